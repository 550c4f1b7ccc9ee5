// primkit-driver: benchmark / tuning front end over the primkit C ABI, the
// B200 build's counterpart of the reference CLI (proj/tools/driver.cpp:169-441,
// MIOpenDriver-style flag letters). It links only libprimkit.so, so every
// solver it times runs on the GPU.
//
//   conv    Find over every applicable solver; report per-solver median time
//           and the speed-up against Im2colGemm (driver.cpp:169-266)
//   tune    tune every applicable tunable solver into a perf-db file
//           (driver.cpp:268-312)
//   fusion  fused vs unfused execution of a CBA / CBNA / NA plan, checked
//           element-wise before timing (driver.cpp:328-441)
//
// Reports: "# primkit-report v1" CSV (default) or JSON (--json); the report
// path is printed on success. Exit codes: 0 ok, 1 runtime error, 2 usage.
// PRIMKIT_FAKE_CLOCK=1 makes timings deterministic (injected handle clock).
// Additive flag: --bf16 runs the problem with bf16 storage (tcgen05 paths).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "primkit/primkit.h"

namespace {

struct Usage {
    std::string msg;
};

// ---- command line ---------------------------------------------------------------
struct Args {
    std::map<std::string, std::string> opt;  // "-c" -> "8", "--json" -> ""
    std::vector<std::string> seen;
    bool has(const std::string& k) const { return opt.count(k) != 0; }
    std::string str(const std::string& k, const std::string& dflt) const {
        auto it = opt.find(k);
        return it == opt.end() ? dflt : it->second;
    }
    int64_t num(const std::string& k, int64_t dflt) const {
        auto it = opt.find(k);
        if (it == opt.end()) return dflt;
        char* end = nullptr;
        const long long v = std::strtoll(it->second.c_str(), &end, 10);
        if (!end || *end) throw Usage{"option " + k + " expects an integer, got '" + it->second + "'"};
        return v;
    }
    double real(const std::string& k, double dflt) const {
        auto it = opt.find(k);
        if (it == opt.end()) return dflt;
        char* end = nullptr;
        const double v = std::strtod(it->second.c_str(), &end);
        if (!end || *end) throw Usage{"option " + k + " expects a number, got '" + it->second + "'"};
        return v;
    }
};

const char* kProblemOpts[] = {"-n", "-c", "-H", "-W", "-k", "-y", "-x", "-p",
                              "-q", "-u", "-v", "-l", "-j", "-g"};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& valued,
           const std::vector<std::string>& flags) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string k = argv[i];
        if (k == "--out") k = "-o";
        if (std::find(flags.begin(), flags.end(), k) != flags.end()) {
            a.opt[k] = "";
            continue;
        }
        if (std::find(valued.begin(), valued.end(), k) == valued.end())
            throw Usage{"unknown option '" + k + "'"};
        if (i + 1 >= argc) throw Usage{"option " + k + " needs a value"};
        a.opt[k] = argv[++i];
    }
    return a;
}

struct Problem {
    int64_t n = 1, c = 0, h = 0, w = 0, k = 0, y = 3, x = 3;
    int64_t pad_h = 0, pad_w = 0, stride_h = 1, stride_w = 1, dil_h = 1, dil_w = 1, groups = 1;
    int direction = 1;
    bool bf16 = false;
};

Problem problem_of(const Args& a, bool with_direction, bool k_required) {
    for (const char* req : {"-c", "-H", "-W"})
        if (!a.has(req)) throw Usage{std::string(req) + " is required"};
    if (k_required && !a.has("-k")) throw Usage{"-k is required"};
    Problem p;
    p.n = a.num("-n", 1);
    p.c = a.num("-c", 0);
    p.h = a.num("-H", 0);
    p.w = a.num("-W", 0);
    p.k = a.num("-k", 0);
    p.y = a.num("-y", 3);
    p.x = a.num("-x", 3);
    p.pad_h = a.num("-p", 0);
    p.pad_w = a.num("-q", 0);
    p.stride_h = a.num("-u", 1);
    p.stride_w = a.num("-v", 1);
    p.dil_h = a.num("-l", 1);
    p.dil_w = a.num("-j", 1);
    p.groups = a.num("-g", 1);
    p.bf16 = a.has("--bf16");
    if (with_direction) {
        p.direction = (int)a.num("-F", 1);
        if (p.direction != 1 && p.direction != 2 && p.direction != 4)
            throw Usage{"-F must be 1, 2 or 4"};
    }
    return p;
}

primkit_conv_problem to_c(const Problem& f) {
    primkit_conv_problem p;
    std::memset(&p, 0, sizeof(p));
    p.n = f.n;
    p.c = f.c;
    p.h = f.h;
    p.w = f.w;
    p.k = f.k;
    p.y = f.y;
    p.x = f.x;
    p.pad_h = f.pad_h;
    p.pad_w = f.pad_w;
    p.stride_h = f.stride_h;
    p.stride_w = f.stride_w;
    p.dilation_h = f.dil_h;
    p.dilation_w = f.dil_w;
    p.groups = f.groups;
    p.direction = f.direction == 2   ? PRIMKIT_DIR_BACKWARD_DATA
                  : f.direction == 4 ? PRIMKIT_DIR_BACKWARD_WEIGHTS
                                     : PRIMKIT_DIR_FORWARD;
    p.mode = PRIMKIT_CONV_CONVOLUTION;
    p.etype = f.bf16 ? PRIMKIT_BF16 : PRIMKIT_F32;
    return p;
}

// Run label of the paper's Fig. 5: Y-X-C-H-W-K-padH-padW.
std::string label(const Problem& f) {
    std::ostringstream os;
    os << f.y << '-' << f.x << '-' << f.c << '-' << f.h << '-' << f.w << '-' << f.k << '-'
       << f.pad_h << '-' << f.pad_w;
    return os.str();
}

std::string fixed(double v, int digits) {
    char b[64];
    std::snprintf(b, sizeof(b), "%.*f", digits, v);
    return b;
}

[[noreturn]] void fail(const std::string& what) {
    std::cerr << "error: " << what << "\n";
    std::exit(1);
}

void check(primkit_status s) {
    if (s != PRIMKIT_STATUS_OK) fail(primkit_last_error());
}

struct Handle {
    primkit_handle* h = nullptr;
    Handle() {
        check(primkit_handle_create(&h));
        const char* fake = std::getenv("PRIMKIT_FAKE_CLOCK");
        if (fake && *fake && std::strcmp(fake, "0") != 0) check(primkit_handle_use_fake_clock(h));
    }
    ~Handle() { primkit_handle_destroy(h); }
};

// U(-1, 1) from std::mt19937_64 (the reference's seed scheme: data seed s, next operand s + 1)
std::vector<float> uniform(size_t count, uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<float> d(-1.0f, 1.0f);
    std::vector<float> v(count);
    for (float& f : v) f = d(rng);
    return v;
}

size_t count4(const int64_t d[4]) { return (size_t)(d[0] * d[1] * d[2] * d[3]); }

std::string json_escape(const std::string& s) {
    std::string o;
    for (char ch : s) {
        if (ch == '"' || ch == '\\') o += '\\';
        o += ch;
    }
    return o;
}

void write_report(const std::string& path, bool json, const std::vector<std::string>& cols,
                  const std::vector<std::vector<std::string>>& rows) {
    std::ofstream os(path, std::ios::trunc);
    if (!os) fail("cannot write " + path);
    if (json) {
        os << "{\n  \"schema\": \"primkit-report v1\",\n  \"rows\": [";
        for (size_t r = 0; r < rows.size(); ++r) {
            os << (r ? "," : "") << "\n    {";
            for (size_t i = 0; i < cols.size(); ++i)
                os << (i ? ", " : "") << "\"" << cols[i] << "\": \"" << json_escape(rows[r][i])
                   << "\"";
            os << "}";
        }
        os << (rows.empty() ? "]\n}\n" : "\n  ]\n}\n");
    } else {
        os << "# primkit-report v1\n";
        for (size_t i = 0; i < cols.size(); ++i) os << (i ? "," : "") << cols[i];
        os << "\n";
        for (const auto& row : rows) {
            for (size_t i = 0; i < row.size(); ++i) os << (i ? "," : "") << row[i];
            os << "\n";
        }
    }
    std::cout << path << "\n";
}

std::vector<std::string> solver_names(primkit_handle* h) {
    int n = 0;
    check(primkit_solver_count(h, &n));
    std::vector<std::string> out;
    for (int i = 0; i < n; ++i) {
        char name[64];
        check(primkit_solver_name(h, i, name, sizeof(name)));
        out.push_back(name);
    }
    return out;
}

// ---- conv -------------------------------------------------------------------------
int cmd_conv(const Args& a) {
    const Problem f = problem_of(a, true, true);
    const std::string out = a.str("-o", "report.csv");
    const bool json = a.has("--json");
    const uint64_t seed = (uint64_t)a.num("--seed", 1);
    Handle g;
    const primkit_conv_problem p = to_c(f);
    // operands: the result dims of the other directions (driver.cpp:186-211)
    primkit_conv_problem fwd = p;
    fwd.direction = PRIMKIT_DIR_FORWARD;
    int64_t y_dims[4];
    check(primkit_conv_output_dims(&fwd, y_dims));
    const int64_t x_dims[4] = {p.n, p.c, p.h, p.w};
    const int64_t w_dims[4] = {p.k, p.c / (p.groups ? p.groups : 1), p.y, p.x};
    const int64_t* ad = p.direction == PRIMKIT_DIR_FORWARD ? x_dims : y_dims;
    const int64_t* bd = p.direction == PRIMKIT_DIR_BACKWARD_WEIGHTS ? x_dims : w_dims;
    const auto A = uniform(count4(ad), seed);
    const auto B = uniform(count4(bd), seed + 1);
    size_t ws = 0;
    for (const auto& s : solver_names(g.h)) {
        int ok = 0;
        if (primkit_solver_is_applicable(g.h, s.c_str(), &p, &ok) != PRIMKIT_STATUS_OK || !ok)
            continue;
        uint64_t b = 0;
        if (primkit_solver_workspace_bytes(g.h, s.c_str(), &p, &b) == PRIMKIT_STATUS_OK)
            ws = std::max<size_t>(ws, b);
    }
    primkit_algo_perf perf[16];
    int found = 0;
    check(primkit_find_convolution(g.h, &p, A.data(), B.data(), ws, perf, 16, &found));
    found = std::min(found, 16);
    double base = 0.0;
    for (int i = 0; i < found; ++i)
        if (std::strcmp(perf[i].solver_name, "Im2colGemm") == 0) base = perf[i].time_ms;
    std::vector<std::vector<std::string>> rows;
    for (int i = 0; i < found; ++i)
        rows.push_back({label(f), perf[i].solver_name, fixed(perf[i].time_ms, 6),
                        std::to_string(perf[i].workspace_bytes),
                        fixed(base > 0.0 ? base / perf[i].time_ms : 1.0, 4)});
    write_report(out, json, {"label", "solver", "median_ms", "workspace_bytes", "speedup_vs_im2colgemm"},
                 rows);
    return 0;
}

// ---- tune -------------------------------------------------------------------------
int cmd_tune(const Args& a) {
    const Problem f = problem_of(a, true, true);
    const std::string db = a.str("--db", "perf.db");
    const int64_t budget = a.num("--budget", 0);
    const bool exhaustive = a.has("--exhaustive");
    Handle g;
    const primkit_conv_problem p = to_c(f);
    if (std::ifstream(db).good()) check(primkit_perfdb_load(g.h, db.c_str()));
    int tuned = 0;
    for (const auto& s : solver_names(g.h)) {
        int ok = 0, tunable = 0;
        primkit_solver_is_applicable(g.h, s.c_str(), &p, &ok);
        primkit_solver_is_tunable(g.h, s.c_str(), &tunable);
        if (!ok || !tunable) continue;
        int64_t evals = 0;
        check(primkit_tune(g.h, &p, s.c_str(), budget, exhaustive ? 1 : 0, &evals));
        ++tuned;
    }
    if (!tuned) {
        std::cerr << "warning: no tunable solver applies to this problem; database untouched\n";
        return 1;
    }
    check(primkit_perfdb_save(g.h, db.c_str()));
    std::cout << db << "\n";
    return 0;
}

// ---- fusion -----------------------------------------------------------------------
double median5(primkit_handle* h, const std::function<void()>& fn) {
    fn();
    std::vector<double> t;
    for (int i = 0; i < 5; ++i) {
        double t0 = 0, t1 = 0;
        primkit_handle_now_ms(h, &t0);
        fn();
        primkit_handle_now_ms(h, &t1);
        t.push_back(t1 - t0);
    }
    std::sort(t.begin(), t.end());
    return t[2];
}

int cmd_fusion(const Args& a) {
    const Problem f = problem_of(a, false, false);
    const std::string combo = a.str("--combo", "CBA");
    const std::string algo_s = a.str("--algo", "Direct");
    const std::string act_s = a.str("--act", "relu");
    const float alpha = (float)a.real("--alpha", 0.01);
    const std::string out = a.str("-o", "fusion.csv");
    const bool json = a.has("--json");
    const uint64_t seed = (uint64_t)a.num("--seed", 1);
    if (combo != "CBA" && combo != "CBNA" && combo != "NA")
        throw Usage{"--combo must be CBA, CBNA or NA"};
    primkit_conv_algo algo;
    if (algo_s == "Direct")
        algo = PRIMKIT_ALGO_DIRECT;
    else if (algo_s == "Winograd")
        algo = PRIMKIT_ALGO_WINOGRAD;
    else
        throw Usage{"unknown fusion algorithm '" + algo_s + "'"};
    static const std::map<std::string, primkit_activation> acts = {
        {"relu", PRIMKIT_ACT_RELU}, {"leakyrelu", PRIMKIT_ACT_LEAKY_RELU},
        {"sigmoid", PRIMKIT_ACT_SIGMOID}, {"tanh", PRIMKIT_ACT_TANH}};
    if (!acts.count(act_s)) throw Usage{"unknown activation '" + act_s + "'"};
    const bool conv = combo != "NA";
    if (conv && f.k <= 0) throw Usage{"-k is required for conv fusions"};

    Handle g;
    const primkit_element_type et = f.bf16 ? PRIMKIT_BF16 : PRIMKIT_F32;
    const int64_t in_dims[4] = {f.n, f.c, f.h, f.w};
    primkit_fusion_plan* plan = nullptr;
    check(primkit_fusion_plan_create(in_dims, et, &plan));
    struct PlanGuard {
        primkit_fusion_plan* p;
        ~PlanGuard() { primkit_fusion_plan_destroy(p); }
    } guard{plan};
    if (conv) {
        const int64_t fd[4] = {f.k, f.c / (f.groups ? f.groups : 1), f.y, f.x};
        check(primkit_fusion_add_conv(plan, fd, f.pad_h, f.pad_w, f.stride_h, f.stride_w, f.groups,
                                      algo));
        check(primkit_fusion_add_bias(plan, f.k));
    }
    if (combo != "CBA") check(primkit_fusion_add_batchnorm(plan, PRIMKIT_BN_SPATIAL));
    check(primkit_fusion_add_activation(plan, acts.at(act_s), alpha));
    check(primkit_fusion_compile(g.h, plan));
    int64_t od[4];
    check(primkit_fusion_output_dims(plan, od));
    const int64_t bnc = conv ? f.k : f.c;
    const auto filt = uniform((size_t)(f.k * (f.c / (f.groups ? f.groups : 1)) * f.y * f.x), seed);
    const auto bias = uniform((size_t)std::max<int64_t>(f.k, 0), seed + 1);
    const auto gamma = uniform((size_t)bnc, seed + 2), beta = uniform((size_t)bnc, seed + 3);
    const auto mean = uniform((size_t)bnc, seed + 4);
    auto var = uniform((size_t)bnc, seed + 5);
    for (float& v : var) v = 1.0f + std::fabs(v);
    check(primkit_fusion_set_args(plan, conv ? filt.data() : nullptr, conv ? bias.data() : nullptr,
                                  gamma.data(), beta.data(), mean.data(), var.data(), 1e-5f,
                                  nullptr));
    const auto input = uniform(count4(in_dims), seed + 6);
    std::vector<float> fused(count4(od)), unfused(count4(od));
    primkit_counters cf{}, cu{};
    check(primkit_handle_reset_counters(g.h));
    check(primkit_fusion_execute(g.h, plan, input.data(), fused.data(), 0));
    check(primkit_handle_counters(g.h, &cf));
    check(primkit_handle_reset_counters(g.h));
    check(primkit_fusion_execute(g.h, plan, input.data(), unfused.data(), 1));
    check(primkit_handle_counters(g.h, &cu));
    // fused vs per-op pipeline, before any timing (1e-5 f32; bf16 stores round once
    // in the fused path and after every op in the unfused one)
    const float tol = f.bf16 ? 2e-2f : 1e-5f;
    for (size_t i = 0; i < fused.size(); ++i)
        if (std::fabs(fused[i] - unfused[i]) / std::max(1.0f, std::fabs(unfused[i])) > tol)
            fail("fused and unfused results diverge at element " + std::to_string(i));
    const double tf = median5(g.h, [&] { primkit_fusion_execute(g.h, plan, input.data(), fused.data(), 0); });
    const double tu = median5(g.h, [&] { primkit_fusion_execute(g.h, plan, input.data(), unfused.data(), 1); });
    write_report(out, json, {"label", "pipeline", "median_ms", "buffer_roundtrips", "speedup_vs_unfused"},
                 {{label(f), combo + "/fused", fixed(tf, 6), std::to_string(cf.buffer_roundtrips),
                   fixed(tf > 0 ? tu / tf : 1.0, 4)},
                  {label(f), combo + "/unfused", fixed(tu, 6), std::to_string(cu.buffer_roundtrips),
                   fixed(1.0, 4)}});
    return 0;
}

const char* kUsage =
    "usage: primkit-driver <conv|tune|fusion> [options]\n"
    "  problem: -n N -c C -H H -W W -k K -y R -x S -p padH -q padW -u strideH -v strideW\n"
    "           -l dilH -j dilW -g groups [--bf16]\n"
    "  conv   : -F 1|2|4 (fwd, bwd data, bwd weights) [-o report.csv] [--json] [--seed S]\n"
    "  tune   : -F 1|2|4 [--db perf.db] [--budget B] [--exhaustive]\n"
    "  fusion : [--combo CBA|CBNA|NA] [--algo Direct|Winograd] [--act relu|leakyrelu|sigmoid|tanh]\n"
    "           [--alpha A] [-o fusion.csv] [--json] [--seed S]\n";

}  // namespace

int main(int argc, char** argv) {
    if (argc >= 2 && (!std::strcmp(argv[1], "-h") || !std::strcmp(argv[1], "--help"))) {
        std::cout << kUsage;
        return 0;
    }
    try {
        if (argc < 2) throw Usage{"a subcommand is required"};
        const std::string cmd = argv[1];
        std::vector<std::string> valued(std::begin(kProblemOpts), std::end(kProblemOpts));
        std::vector<std::string> flags = {"--bf16"};
        if (cmd == "conv") {
            valued.insert(valued.end(), {"-F", "-o", "--seed"});
            flags.push_back("--json");
            return cmd_conv(parse(argc, argv, 2, valued, flags));
        }
        if (cmd == "tune") {
            valued.insert(valued.end(), {"-F", "--db", "--budget"});
            flags.push_back("--exhaustive");
            return cmd_tune(parse(argc, argv, 2, valued, flags));
        }
        if (cmd == "fusion") {
            valued.insert(valued.end(), {"--combo", "--algo", "--act", "--alpha", "-o", "--seed"});
            flags.push_back("--json");
            return cmd_fusion(parse(argc, argv, 2, valued, flags));
        }
        throw Usage{"unknown subcommand '" + cmd + "'"};
    } catch (const Usage& u) {
        std::cerr << "error: " << u.msg << "\n\n" << kUsage;
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
