#include "perfdb.hpp"

#include <cstdio>
#include <fstream>
#include <sstream>

#include "core.hpp"

namespace primkit {

void PerfDb::set(const std::string& key, const std::string& solver, const std::string& values) {
    records_[key][solver] = values;
}

std::optional<std::string> PerfDb::get(const std::string& key, const std::string& solver) const {
    const auto rec = records_.find(key);
    if (rec == records_.end()) return std::nullopt;
    const auto it = rec->second.find(solver);
    if (it == rec->second.end()) return std::nullopt;
    return it->second;
}

namespace {
[[noreturn]] void parse_fail(int line, const std::string& what) {
    throw_error(ErrorCode::ParseError, "perf-db line " + std::to_string(line) + ": " + what);
}
}  // namespace

PerfDb PerfDb::parse(const std::string& text) {
    PerfDb db;
    std::size_t pos = 0;
    int lineno = 0;
    while (pos <= text.size()) {
        const std::size_t nl = text.find('\n', pos);
        if (nl == std::string::npos && pos == text.size()) break;
        std::string line = text.substr(pos, nl == std::string::npos ? std::string::npos : nl - pos);
        pos = nl == std::string::npos ? text.size() + 1 : nl + 1;
        ++lineno;
        if (line.empty() || line[0] == '#') continue;
        const std::size_t eq = line.find('=');
        if (eq == std::string::npos || eq == 0) parse_fail(lineno, "missing '=' in '" + line + "'");
        const std::string key = line.substr(0, eq);
        if (db.records_.count(key)) parse_fail(lineno, "duplicate key '" + key + "'");
        std::map<std::string, std::string> entries;
        const std::string rest = line.substr(eq + 1);
        std::size_t p = 0;
        // ';'-separated solver entries; an empty trailing segment is ignored
        while (p < rest.size()) {
            std::size_t semi = rest.find(';', p);
            if (semi == std::string::npos) semi = rest.size();
            const std::string part = rest.substr(p, semi - p);
            p = semi + 1;
            const std::size_t colon = part.find(':');
            if (colon == std::string::npos || colon == 0)
                parse_fail(lineno, "bad entry '" + part + "'");
            entries[part.substr(0, colon)] = part.substr(colon + 1);
        }
        if (entries.empty()) parse_fail(lineno, "no solver entries in '" + line + "'");
        db.records_[key] = std::move(entries);
    }
    return db;
}

PerfDb PerfDb::load(const std::filesystem::path& path) {
    std::ifstream in(path);
    if (!in) throw_error(ErrorCode::IoError, "cannot read " + path.string());
    std::ostringstream ss;
    ss << in.rdbuf();
    return parse(ss.str());
}

std::string PerfDb::serialize() const {
    std::string out;
    for (const auto& [key, entries] : records_) {
        out += key;
        out += '=';
        bool first = true;
        for (const auto& [solver, values] : entries) {
            if (!first) out += ';';
            first = false;
            out += solver + ':' + values;
        }
        out += '\n';
    }
    return out;
}

void PerfDb::save(const std::filesystem::path& path) const {
    const std::string tmp = path.string() + ".tmp";
    {
        std::ofstream out(tmp, std::ios::trunc);
        if (!out) throw_error(ErrorCode::IoError, "cannot write " + tmp);
        out << serialize();
    }
    std::error_code ec;
    std::filesystem::rename(tmp, path, ec);
    if (ec) throw_error(ErrorCode::IoError, "cannot rename " + tmp);
}

PlanCache::PlanCache(std::filesystem::path disk_dir) : dir_(std::move(disk_dir)) {
    if (dir_.empty()) return;
    std::error_code ec;
    std::filesystem::create_directories(dir_, ec);
    if (ec) dir_.clear();  // unwritable -> memory-only cache
}

PlanCache::Stats PlanCache::stats() const {
    std::lock_guard<std::mutex> lock(mu_);
    return stats_;
}

void PlanCache::reset_stats() {
    std::lock_guard<std::mutex> lock(mu_);
    stats_ = Stats{};
}

std::string PlanCache::hash_key(const std::string& problem_key, const std::string& solver_name,
                                const std::string& config_values) {
    // 64-bit FNV-1a over "key|solver|values": stable across processes
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (const std::string* part : {&problem_key, &solver_name, &config_values}) {
        if (part != &problem_key) {
            h ^= static_cast<unsigned char>('|');
            h *= 0x100000001b3ull;
        }
        for (unsigned char ch : *part) {
            h ^= ch;
            h *= 0x100000001b3ull;
        }
    }
    char buf[32];
    std::snprintf(buf, sizeof(buf), "%llx", static_cast<unsigned long long>(h));
    return buf;
}

std::shared_ptr<void> PlanCache::get_or_build(const std::string& cache_key,
                                              const std::string& descriptor, const Build& build,
                                              const Materialize& materialize) {
    std::lock_guard<std::mutex> lock(mu_);
    if (auto it = mem_.find(cache_key); it != mem_.end()) {
        ++stats_.memory_hits;
        return it->second;
    }
    const std::string header = "primkit-plan v" + std::to_string(kPlanVersion);
    const auto path = dir_ / (cache_key + ".plan");
    if (!dir_.empty()) {
        std::ifstream in(path);
        if (in) {
            std::string first;
            std::getline(in, first);
            std::ostringstream body;
            body << in.rdbuf();
            if (first == header && body.str() == descriptor) {
                try {
                    auto plan = materialize(body.str());
                    ++stats_.disk_hits;
                    mem_[cache_key] = plan;
                    return plan;
                } catch (const std::exception&) {
                    // foreign or corrupt entry: rebuild below
                }
            }
        }
    }
    auto plan = build();
    ++stats_.builds;
    mem_[cache_key] = plan;
    if (!dir_.empty()) {
        const std::string tmp = path.string() + ".tmp";
        std::ofstream out(tmp, std::ios::trunc);
        if (out) {
            out << header << '\n' << descriptor;
            out.close();
            std::error_code ec;
            std::filesystem::rename(tmp, path, ec);
        }
    }
    return plan;
}

}  // namespace primkit
