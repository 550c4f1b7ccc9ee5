// Performance database and two-level plan cache.
//
// File formats are bit-compatible with the reference so tuned records and
// cache directories move between the CPU reference and this library:
//   perf-db   `<problem-key>=<solver>:<v1>,<v2>[;<solver>:...]`, '#' comments,
//             sorted by key on save, tmp + rename (proj/src/core/perfdb.cpp:24-98)
//   plan file `<fnv1a-hex>.plan` = "primkit-plan v1\n" + descriptor
//             (proj/src/core/plan_cache.cpp:27-90)
#pragma once

#include <filesystem>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <string>

namespace primkit {

class PerfDb {
public:
    void set(const std::string& problem_key, const std::string& solver,
             const std::string& values);
    std::optional<std::string> get(const std::string& problem_key,
                                   const std::string& solver) const;
    bool empty() const { return records_.empty(); }
    std::size_t size() const { return records_.size(); }

    static PerfDb parse(const std::string& text);
    static PerfDb load(const std::filesystem::path& path);
    std::string serialize() const;
    void save(const std::filesystem::path& path) const;

private:
    std::map<std::string, std::map<std::string, std::string>> records_;
};

class PlanCache {
public:
    struct Stats {
        std::uint64_t builds = 0;
        std::uint64_t memory_hits = 0;
        std::uint64_t disk_hits = 0;
    };
    static constexpr int kPlanVersion = 1;

    explicit PlanCache(std::filesystem::path disk_dir);
    const std::filesystem::path& disk_dir() const { return dir_; }
    Stats stats() const;
    void reset_stats();

    using Build = std::function<std::shared_ptr<void>()>;
    using Materialize = std::function<std::shared_ptr<void>(const std::string&)>;
    std::shared_ptr<void> get_or_build(const std::string& cache_key, const std::string& descriptor,
                                       const Build& build, const Materialize& materialize);

    static std::string hash_key(const std::string& problem_key, const std::string& solver_name,
                                const std::string& config_values);

private:
    std::filesystem::path dir_;
    mutable std::mutex mu_;
    std::map<std::string, std::shared_ptr<void>> mem_;
    Stats stats_;
};

}  // namespace primkit
