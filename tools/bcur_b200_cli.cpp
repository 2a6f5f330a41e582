// bcur_b200 — the reference CLI's hot-path commands (tools/bcur_main.cpp) on the B200 library.
//
//   decompose  blockcur.cpp:54-133 (Algorithm 1, boosted): a ".bcur" matrix → the JSON report
//              of serialize.cpp:110-122 (+ "config"), optionally written with U.bcur to --out-dir
//   scores     block leverage at rank k (randomized range finder on the GPU in place of the
//              reference's exact SVD) with the score diagnostics → write_scores_csv's CSV
//   css        north star: block column subset selection (block_css) → JSON
//
// Exit codes as the reference (bcur_main.cpp:617-641): 0 success, 2 input / validation
// failure, 3 numerical failure; errors are one JSON line on stderr.
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <variant>
#include <vector>

#include "bcur_b200.hpp"

namespace {

using namespace bcur;

// ---------------------------------------------------------------- minimal ordered JSON
struct Json {
    enum Kind { Null, Bool, Int, Num, Str, Arr, Obj } kind = Null;
    bool b = false;
    long long i = 0;
    double d = 0.0;
    std::string s;
    std::vector<Json> a;
    std::vector<std::pair<std::string, Json>> o;
    Json() = default;
    Json(bool v) : kind(Bool), b(v) {}
    Json(int v) : kind(Int), i(v) {}
    Json(long v) : kind(Int), i(v) {}
    Json(long long v) : kind(Int), i(v) {}
    Json(unsigned long v) : kind(Int), i((long long)v) {}
    Json(unsigned long long v) : kind(Int), i((long long)v) {}
    Json(double v) : kind(Num), d(v) {}
    Json(const char* v) : kind(Str), s(v) {}
    Json(std::string v) : kind(Str), s(std::move(v)) {}
    static Json array() { Json j; j.kind = Arr; return j; }
    static Json object() { Json j; j.kind = Obj; return j; }
    Json& operator[](const std::string& k) {
        if (kind != Obj) kind = Obj;
        for (auto& kv : o)
            if (kv.first == k) return kv.second;
        o.emplace_back(k, Json());
        return o.back().second;
    }
    void push(Json v) {
        kind = Arr;
        a.push_back(std::move(v));
    }
    static std::string num(double v) {
        if (std::isnan(v) || std::isinf(v)) return "null";
        char buf[64];
        auto r = std::to_chars(buf, buf + sizeof buf, v);
        std::string t(buf, r.ptr);
        if (t.find_first_of(".e") == std::string::npos) t += ".0";
        return t;
    }
    static std::string str(const std::string& v) {
        std::string t = "\"";
        for (char ch : v) {
            if (ch == '"' || ch == '\\') t += '\\';
            t += ch;
        }
        return t + "\"";
    }
    // ind < 0: compact (nlohmann's dump()), else pretty with ind spaces (dump(ind))
    void dump(std::ostream& out, int ind, int level) const {
        if (ind < 0) {
            switch (kind) {
                case Arr:
                    out << "[";
                    for (size_t t = 0; t < a.size(); ++t) {
                        if (t) out << ",";
                        a[t].dump(out, ind, level);
                    }
                    out << "]";
                    return;
                case Obj:
                    out << "{";
                    for (size_t t = 0; t < o.size(); ++t) {
                        if (t) out << ",";
                        out << str(o[t].first) << ":";
                        o[t].second.dump(out, ind, level);
                    }
                    out << "}";
                    return;
                default: break;
            }
        }
        const int in_ = ind < 0 ? 0 : ind;
        const std::string pad(in_ * (level + 1), ' '), end(in_ * level, ' ');
        switch (kind) {
            case Null: out << "null"; break;
            case Bool: out << (b ? "true" : "false"); break;
            case Int: out << i; break;
            case Num: out << num(d); break;
            case Str: out << str(s); break;
            case Arr:
                if (a.empty()) { out << "[]"; break; }
                out << "[\n";
                for (size_t t = 0; t < a.size(); ++t) {
                    out << pad;
                    a[t].dump(out, ind, level + 1);
                    out << (t + 1 < a.size() ? ",\n" : "\n");
                }
                out << end << "]";
                break;
            case Obj:
                if (o.empty()) { out << "{}"; break; }
                out << "{\n";
                for (size_t t = 0; t < o.size(); ++t) {
                    out << pad << str(o[t].first) << ": ";
                    o[t].second.dump(out, ind, level + 1);
                    out << (t + 1 < o.size() ? ",\n" : "\n");
                }
                out << end << "}";
                break;
        }
    }
    std::string dump(int ind = 2) const {
        std::ostringstream os;
        dump(os, ind, 0);
        return os.str();
    }
};

constexpr int kSchemaVersion = 1;  // serialize.hpp:11

// serialize.cpp:19-32, 47-61, 75-87
Json plan_json(const SamplingPlan& p) {
    Json j;
    j["schema_version"] = kSchemaVersion;
    j["type"] = "block_plan";
    j["mode"] = to_string(p.mode);
    j["seed"] = (unsigned long long)p.seed;
    j["g"] = (long long)p.draws.size();
    Json d = Json::array();
    for (const BlockDraw& x : p.draws) {
        Json e;
        e["block"] = (long long)x.block;
        e["probability"] = x.probability;
        e["scale"] = x.scale;
        d.push(e);
    }
    j["draws"] = d;
    return j;
}
Json row_plan_json(const RowPlan& p) {
    Json j;
    j["schema_version"] = kSchemaVersion;
    j["type"] = "row_plan";
    j["mode"] = to_string(p.mode);
    j["seed"] = (unsigned long long)p.seed;
    j["source_rows"] = (long long)p.source_rows;
    j["r"] = (long long)p.draws.size();
    Json d = Json::array();
    for (const RowDraw& x : p.draws) {
        Json e;
        e["row"] = (long long)x.row;
        e["probability"] = x.probability;
        e["scale"] = x.scale;
        d.push(e);
    }
    j["draws"] = d;
    return j;
}
Json report_json(const ErrorReport& r) {
    Json j;
    j["variant"] = r.variant == UVariant::full ? "U" : "U_k";
    j["k"] = (long long)r.k;
    j["abs_err"] = r.abs_err;
    j["rel_to_A"] = r.rel_to_a;
    j["rel_to_best_k"] = r.rel_to_best_k ? Json(*r.rel_to_best_k) : Json();
    return j;
}

void print_error(const char* type, const std::string& msg) {
    Json j;
    j["schema_version"] = kSchemaVersion;
    Json e;
    e["type"] = type;
    e["message"] = msg;
    j["error"] = e;
    std::cerr << j.dump(-1) << "\n";
}

// ------------------------------------------------------------------- arguments
struct Args {
    std::map<std::string, std::string> kv;
    std::vector<std::string> flags;
    bool has(const std::string& k) const { return kv.count(k) > 0; }
    bool flag(const std::string& f) const { return std::find(flags.begin(), flags.end(), f) != flags.end(); }
    std::string get(const std::string& k, const std::string& def = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? def : it->second;
    }
    long long num(const std::string& k, long long def) const {
        if (!has(k)) return def;
        try {
            return std::stoll(get(k));
        } catch (...) {
            throw std::invalid_argument("--" + k + " expects an integer");
        }
    }
    double real(const std::string& k, double def) const {
        if (!has(k)) return def;
        try {
            return std::stod(get(k));
        } catch (...) {
            throw std::invalid_argument("--" + k + " expects a number");
        }
    }
};
Args parse(int argc, char** argv, int first) {
    Args a;
    static const char* kFlags[] = {"distinct-rows"};
    for (int i = first; i < argc; ++i) {
        std::string t = argv[i];
        if (t.rfind("--", 0) != 0) throw std::invalid_argument("unexpected argument '" + t + "'");
        t = t.substr(2);
        const auto eq = t.find('=');
        if (eq != std::string::npos) {
            a.kv[t.substr(0, eq)] = t.substr(eq + 1);
            continue;
        }
        bool is_flag = false;
        for (const char* f : kFlags) is_flag = is_flag || t == f;
        if (is_flag) {
            a.flags.push_back(t);
        } else {
            if (i + 1 >= argc) throw std::invalid_argument("--" + t + " needs a value");
            a.kv[t] = argv[++i];
        }
    }
    return a;
}
BlockPartition partition(const Args& a, Index n) {
    if (a.has("boundaries")) {
        std::vector<Index> cuts;
        std::stringstream ss(a.get("boundaries"));
        std::string tok;
        while (std::getline(ss, tok, ',')) cuts.push_back(std::stoll(tok));
        return BlockPartition::from_boundaries(n, cuts);
    }
    if (a.num("block-size", 0) > 0) return BlockPartition::equal_blocks(n, a.num("block-size", 0));
    throw std::invalid_argument("a partition is required: pass --block-size or --boundaries");
}
SamplingMode mode_of(const std::string& m) {
    if (m == "with_replacement" || m == "with") return SamplingMode::with_replacement;
    if (m == "without_replacement" || m == "without") return SamplingMode::without_replacement;
    throw std::invalid_argument("unknown sampling mode '" + m + "'");
}
int dtype_of(const Args& a) {
    const std::string d = a.get("dtype", "f64");
    if (d == "f64") return BCUR_F64;
    if (d == "f32") return BCUR_F32;
    throw std::invalid_argument("--dtype must be f64 or f32");
}
std::string input_of(const Args& a) {
    if (!a.has("input")) throw std::invalid_argument("--input is required");
    int64_t r = 0, c = 0;
    detail::check(bcur_bcur_header(a.get("input").c_str(), &r, &c));  // ParseError before any device work
    return a.get("input");
}

// ------------------------------------------------------------------ commands
int run_decompose(const Args& a) {  // bcur_main.cpp:98-144
    const std::string in = input_of(a);
    const Index k = a.num("k", 0), r = a.num("r", 0), g = a.num("g", 0);
    Index t = a.num("t", 1);
    const double delta = a.real("delta", 0.0);
    if (delta > 0.0) {  // blockcur.cpp:146-151
        if (!(delta < 1.0)) throw std::invalid_argument("boost_trials: delta must be in (0, 1)");
        t = (Index)std::ceil(std::log(1.0 / delta));
    }
    CurOptions opts;
    opts.block_mode = mode_of(a.get("mode", "with_replacement"));
    opts.distinct_rows = a.flag("distinct-rows");
    if (a.get("row-mode", "uniform") != "uniform")
        throw std::invalid_argument("row sampling 'leverage' needs the exact SVD of A (not on this path)");
    auto A = DeviceMatrix::load_binary(in, dtype_of(a));
    const BlockPartition part = partition(a, A.cols());
    Rng rng((std::uint64_t)a.num("seed", 0));
    const std::uint64_t seed = rng.seed();
    const CurResult res = block_cur_boosted(A, part, k, r, g, t, opts, rng);
    Index c = 0;
    for (const BlockDraw& d : res.block_plan.draws) c += part.width(d.block);
    Json rep;
    rep["schema_version"] = kSchemaVersion;
    Json shapes;
    auto pair = [](Index x, Index y) {
        Json p = Json::array();
        p.push((long long)x);
        p.push((long long)y);
        return p;
    };
    shapes["C"] = pair(A.rows(), c);
    shapes["U"] = pair(c, r);
    shapes["R"] = pair(r, A.cols());
    shapes["W"] = pair(r, c);
    rep["shapes"] = shapes;
    rep["row_plan"] = row_plan_json(res.row_plan);
    rep["block_plan"] = plan_json(res.block_plan);
    Json metrics = Json::array();
    metrics.push(report_json(res.metrics_u));
    metrics.push(report_json(res.metrics_uk));
    rep["metrics"] = metrics;
    Json te = Json::array();
    for (double e : res.trial_errors) te.push(e);
    rep["trial_errors"] = te;
    Json cfg;
    cfg["command"] = "decompose";
    cfg["input"] = in;
    cfg["k"] = (long long)k;
    cfg["r"] = (long long)r;
    cfg["g"] = (long long)g;
    cfg["t"] = (long long)t;
    cfg["delta"] = delta;
    cfg["seed"] = (unsigned long long)seed;
    cfg["mode"] = to_string(opts.block_mode);
    cfg["row_mode"] = "uniform";
    cfg["distinct_rows"] = opts.distinct_rows;
    cfg["blocks"] = (long long)part.num_blocks();
    rep["config"] = cfg;
    const std::string text = rep.dump(2);
    if (a.has("out-dir")) {
        const std::filesystem::path dir(a.get("out-dir"));
        std::filesystem::create_directories(dir);
        std::ofstream(dir / "report.json") << text << "\n";
        auto U = DeviceMatrix::upload(res.u);
        U.save_binary((dir / "U.bcur").string());
    }
    std::cout << text << "\n";
    return 0;
}

int run_scores(const Args& a) {  // bcur_main.cpp:158-190 (randomized subspace in place of svd(a))
    const std::string in = input_of(a);
    const Index k = a.num("k", 0);
    auto A = DeviceMatrix::load_binary(in, dtype_of(a));
    const BlockPartition part = partition(a, A.cols());
    if (k < 1 || k > std::min(A.rows(), A.cols())) throw std::invalid_argument("scores: need 1 <= k <= min(m, n)");
    Device& dev = Device::current();
    Rng rng((std::uint64_t)a.num("seed", 0));
    const std::uint64_t key = bcur_omega_key(rng.seed());  // the library's sketch key (as block_css)
    bcur_dmat hv = nullptr, hu = nullptr;
    int64_t keff = 0;
    detail::check(bcur_range_finder(dev.handle(), A.handle(), k, a.num("p", 10), a.num("q", 2), key, &hv, &hu, nullptr,
                                    &keff));
    DeviceMatrix V(hv), U(hu);
    if (keff == 0) throw ZeroMatrix("scores: input matrix is identically zero");
    const ScoreVector scores = block_leverage(V, part);
    const auto off = part.offsets();
    std::vector<double> sr((size_t)part.num_blocks());
    double alpha = NAN, mu = NAN;
    const bcur_status st = bcur_block_diagnostics(dev.handle(), V.handle(), U.handle(), off.data(), part.num_blocks(),
                                                  sr.data(), &alpha, &mu);
    if (st != BCUR_OK && st != BCUR_E_ZERO_BLOCK) detail::check(st);  // ZeroBlock: alpha stays NaN (as the reference)
    if (st == BCUR_E_ZERO_BLOCK) alpha = NAN;
    Json cfg;
    cfg["command"] = "scores";
    cfg["input"] = in;
    cfg["k"] = (long long)k;
    cfg["blocks"] = (long long)part.num_blocks();
    std::ostringstream out;
    out.precision(17);
    out << "# config=" << cfg.dump(-1) << "\n";
    double total = 0.0;
    for (Index g = 0; g < part.num_blocks(); ++g) total += scores.scores(g);
    out << "# normalizer=" << scores.normalizer << "\n# sum_scores=" << total << "\n# block_stable_rank=" << alpha
        << "\n# incoherence=" << mu << "\nblock,start,end,width,score,probability\n";
    for (Index g = 0; g < part.num_blocks(); ++g) {
        const Index b = off[(size_t)g], e = off[(size_t)g + 1];
        out << g << ',' << b << ',' << e << ',' << (e - b) << ',' << scores.scores(g) << ',' << scores.scores(g) / total
            << "\n";
    }
    if (a.has("output")) {
        std::ofstream f(a.get("output"));
        if (!f) throw ParseError("cannot write " + a.get("output"));
        f << out.str();
    } else {
        std::cout << out.str();
    }
    return 0;
}

int run_css(const Args& a) {  // north star: block_css
    const std::string in = input_of(a);
    auto A = DeviceMatrix::load_binary(in, dtype_of(a));
    const BlockPartition part = partition(a, A.cols());
    CssOptions o;
    o.p = a.num("p", 10);
    o.q = a.num("q", 2);
    o.mode = mode_of(a.get("mode", "without_replacement"));
    o.materialize_c = false;
    Rng rng((std::uint64_t)a.num("seed", 0));
    const CssResult res = block_css(A, part, a.num("k", 0), a.num("g", 0), rng, o);
    Json j;
    j["schema_version"] = kSchemaVersion;
    j["block_plan"] = plan_json(res.plan);
    j["abs_err"] = res.projection_error;
    j["a_norm"] = res.report.a_norm;
    j["rel_err"] = res.report.rel_err;
    j["normalizer"] = res.scores.normalizer;
    std::cout << j.dump(2) << "\n";
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2 || !std::strcmp(argv[1], "--help") || !std::strcmp(argv[1], "-h")) {
        std::printf("usage: bcur_b200 decompose|scores|css --input A.bcur (--block-size S | --boundaries c1,c2,..)\n"
                    "  decompose --k K --r R --g G [--t T | --delta D] [--seed N] [--mode with|without]\n"
                    "            [--distinct-rows] [--dtype f64|f32] [--out-dir DIR]\n"
                    "  scores    --k K [--p P] [--q Q] [--seed N] [--dtype f64|f32] [--output FILE]\n"
                    "  css       --k K --g G [--p P] [--q Q] [--seed N] [--mode with|without] [--dtype f64|f32]\n");
        return argc < 2 ? 2 : 0;
    }
    const std::string cmd = argv[1];
    try {
        const Args a = parse(argc, argv, 2);
        if (cmd == "decompose") return run_decompose(a);
        if (cmd == "scores") return run_scores(a);
        if (cmd == "css") return run_css(a);
        throw std::invalid_argument("unknown command '" + cmd + "'");
    } catch (const ParseError& e) {
        print_error("ParseError", e.what());
        return 2;
    } catch (const DimensionMismatch& e) {
        print_error("DimensionMismatch", e.what());
        return 2;
    } catch (const DeviceError& e) {
        print_error("DeviceError", e.what());
        return 3;
    } catch (const Error& e) {  // numerical: ZeroMatrix, InvalidBasis, DegenerateR, IterationFailure, ...
        print_error("NumericalError", e.what());
        return 3;
    } catch (const std::out_of_range& e) {
        print_error("OutOfRange", e.what());
        return 2;
    } catch (const std::invalid_argument& e) {
        print_error("InvalidArgument", e.what());
        return 2;
    } catch (const std::exception& e) {
        print_error("Error", e.what());
        return 2;
    }
}
