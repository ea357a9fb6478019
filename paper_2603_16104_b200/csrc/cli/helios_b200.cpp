// helios_b200 — `helios run` (tools/helios_main.cpp:48-115) on the B200
// executor, self-contained: the workflow / inputs / profile JSON, binding,
// rewrites, the cache-aware planner, simulate() and the reports all come from
// libhelium_b200.so through its C ABI (hk_run_workflow). Same flags, files and
// byte-stable reports as the reference CLI; plus --engine
// none|tiny|tiny_f32|llama3_8b|qwen25_32b (default none: the reference's
// synthetic LLM body) and --device N. Exit codes: 0 ok, 1 run error, 2 usage.
// (integration/helios_b200_main.cpp is the variant a maintainer links against
// the reference library instead.)
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "helium_b200.h"

namespace {

struct Spec {
    int workers = 1;
    std::vector<std::size_t> capacities = {4096};
    std::uint64_t seed = 0;
    bool stochastic = false;
    bool collect_trace = false;
    std::size_t block = 16, prefill_budget = 0, pin_threshold = 200;
    double alpha = 0;
};

std::string slurp(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open " + path);
    std::ostringstream ss;
    ss << f.rdbuf();
    return ss.str();
}

void emit(const std::string& path, const std::string& content) {
    if (path.empty() || path == "-") {
        std::cout << content;
        return;
    }
    std::ofstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot write " + path);
    f << content;
}

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct RunArgs {
    std::string workflow, inputs, profile;
    Spec spec;
    std::string scheduler = "cache_aware";
    std::vector<std::size_t> capacities;
    bool no_prune = false, no_merge = false, no_prompt_cache = false, no_pin = false, no_sim = false;
    std::string cache_file, out, format = "json", calls_out, trace_out, outputs_out, schedule_out;
    std::string engine = "none";
    int device = 0;
};

template <class T>
T number(const std::string& opt, const std::string& v) {
    try {
        std::size_t used = 0;
        T x;
        if constexpr (std::is_floating_point_v<T>)
            x = static_cast<T>(std::stod(v, &used));
        else if constexpr (std::is_signed_v<T>)
            x = static_cast<T>(std::stoll(v, &used));
        else
            x = static_cast<T>(std::stoull(v, &used));
        if (used != v.size()) throw std::invalid_argument(v);
        return x;
    } catch (const std::exception&) {
        throw Usage(opt + ": " + v + " is not a number");
    }
}

RunArgs parse_run(int argc, char** argv) {
    RunArgs a;
    if (const char* s = std::getenv("HELIOS_SEED")) a.spec.seed = number<std::uint64_t>("HELIOS_SEED", s);
    const std::map<std::string, bool*> flags{{"--stochastic", &a.spec.stochastic}, {"--no-prune", &a.no_prune},
                                             {"--no-cse", &a.no_merge},           {"--no-prompt-cache", &a.no_prompt_cache},
                                             {"--no-proactive-kv", &a.no_pin},    {"--no-sim", &a.no_sim},
                                             {"--trace", &a.spec.collect_trace}};
    for (int i = 2; i < argc; ++i) {
        std::string opt = argv[i], val;
        bool has_val = false;
        if (const auto eq = opt.find('='); opt.rfind("--", 0) == 0 && eq != std::string::npos) {
            val = opt.substr(eq + 1);
            opt = opt.substr(0, eq);
            has_val = true;
        }
        if (auto f = flags.find(opt); f != flags.end()) {
            if (has_val) throw Usage(opt + " takes no value");
            *f->second = true;
            continue;
        }
        if (!has_val) {
            if (i + 1 >= argc) throw Usage(opt + " needs a value");
            val = argv[++i];
        }
        if (opt == "--workflow") a.workflow = val;
        else if (opt == "--inputs") a.inputs = val;
        else if (opt == "--profile") a.profile = val;
        else if (opt == "--workers") a.spec.workers = number<int>(opt, val);
        else if (opt == "--capacity") {
            std::stringstream ss(val);
            for (std::string c; std::getline(ss, c, ',');) a.capacities.push_back(number<std::size_t>(opt, c));
        } else if (opt == "--scheduler") a.scheduler = val;
        else if (opt == "--seed") a.spec.seed = number<std::uint64_t>(opt, val);
        else if (opt == "--block") a.spec.block = number<std::size_t>(opt, val);
        else if (opt == "--prefill-budget") a.spec.prefill_budget = number<std::size_t>(opt, val);
        else if (opt == "--pin-threshold") a.spec.pin_threshold = number<std::size_t>(opt, val);
        else if (opt == "--alpha") a.spec.alpha = number<double>(opt, val);
        else if (opt == "--cache-file") a.cache_file = val;
        else if (opt == "--out") a.out = val;
        else if (opt == "--format") {
            if (val != "json" && val != "csv") throw Usage("--format: " + val + " not in {json,csv}");
            a.format = val;
        } else if (opt == "--calls-out") a.calls_out = val;
        else if (opt == "--trace-out") a.trace_out = val;
        else if (opt == "--outputs-out") a.outputs_out = val;
        else if (opt == "--schedule-out") a.schedule_out = val;
        else if (opt == "--engine") a.engine = val;
        else if (opt == "--device") a.device = number<int>(opt, val);
        else throw Usage("the following argument was not expected: " + opt);
    }
    for (const auto* req : {&a.workflow, &a.inputs, &a.profile})
        if (req->empty()) throw Usage("--workflow, --inputs and --profile are required");
    return a;
}


hk_engine* make_engine(const RunArgs& a) {
    if (a.engine == "none") return nullptr;
    hk_model_config mc{};
    if (a.engine == "tiny" || a.engine == "tiny_f32")
        mc = hk_model_config{2, 256, 2, 1, 128, 768, 32768, 0, 10000.0f, 1e-5f, 0, a.engine == "tiny_f32" ? 1u : 0u, 0};
    else if (a.engine == "llama3_8b")
        mc = hk_model_config{32, 4096, 32, 8, 128, 14336, 128256, 0, 500000.0f, 1e-5f, 0, 0, 0};
    else if (a.engine == "qwen25_32b")
        mc = hk_model_config{64, 5120, 40, 8, 128, 27648, 152064, 1, 1000000.0f, 1e-6f, 0, 0, 0};
    else
        throw Usage("--engine: " + a.engine + " not in {none,tiny,tiny_f32,llama3_8b,qwen25_32b}");
    const std::vector<std::size_t>& caps = a.capacities.empty() ? a.spec.capacities : a.capacities;
    std::uint64_t cap = 0;
    for (std::size_t c : caps) cap = std::max<std::uint64_t>(cap, c);
    const std::uint32_t calls = 600;
    hk_engine_config ec{a.device, static_cast<std::uint32_t>(a.spec.workers),
                        static_cast<std::uint32_t>(cap / a.spec.block + calls * 80 + 64),
                        static_cast<std::uint32_t>(a.spec.block), calls, 8192 + 512, 12288, 1};
    hk_engine* e = hk_engine_create(&mc, &ec);
    if (!e) throw std::runtime_error(std::string("hk_engine_create: ") + hk_last_error());
    return e;
}

std::string report(const hk_run* r, int which, bool document) {
    const std::size_t n = document ? hk_run_document(r, which, nullptr, 0) : hk_run_report(r, which, nullptr, 0);
    std::string s(n, '\0');
    if (document)
        hk_run_document(r, which, s.data(), s.size());
    else
        hk_run_report(r, which, s.data(), s.size());
    if (!s.empty() && s.back() == '\0') s.pop_back();
    return s;
}

int do_run(RunArgs& a) {
    const std::string wf = slurp(a.workflow), in = slurp(a.inputs), prof = slurp(a.profile);
    if (!a.capacities.empty()) a.spec.capacities = a.capacities;
    if (!a.trace_out.empty()) a.spec.collect_trace = true;
    const bool substitute = !a.no_prompt_cache;
    hk_pcache* cache = nullptr;
    if (!a.cache_file.empty() && substitute) {
        std::ifstream probe(a.cache_file);
        if (probe.good()) {
            const std::string doc = slurp(a.cache_file);
            cache = hk_pcache_load(doc.data(), doc.size());
        } else {
            cache = hk_pcache_create(65536);
        }
        if (!cache) throw std::runtime_error(hk_last_error());
    }
    std::vector<std::uint64_t> caps(a.spec.capacities.begin(), a.spec.capacities.end());
    hk_workflow_spec ws{a.spec.workers, caps.data(), caps.size(), a.scheduler.c_str(), a.spec.seed,
                        a.spec.stochastic ? 1 : 0, a.no_prune ? 0 : 1, a.no_merge ? 0 : 1, substitute ? 1 : 0,
                        a.no_pin ? 0 : 1, a.spec.pin_threshold, 0.5, a.spec.block, a.spec.prefill_budget, a.spec.alpha,
                        a.no_sim ? 0 : 1, a.spec.collect_trace ? 1 : 0, 0};
    hk_engine* eng = a.no_sim ? nullptr : make_engine(a);
    hk_run* r = hk_run_workflow(wf.c_str(), in.c_str(), prof.c_str(), &ws, cache, eng);
    if (eng) hk_engine_destroy(eng);
    if (!r) {
        const std::string err = hk_last_error();
        if (cache) hk_pcache_destroy(cache);
        throw std::runtime_error(err);
    }
    if (cache) {
        std::string doc(hk_pcache_save(cache, nullptr, 0), '\0');
        hk_pcache_save(cache, doc.data(), doc.size());
        doc.pop_back();
        emit(a.cache_file, doc);
        hk_pcache_destroy(cache);
    }
    emit(a.out, a.format == "csv" ? report(r, 1, false) : report(r, 0, true));
    if (!a.calls_out.empty()) emit(a.calls_out, report(r, 1, false));
    if (!a.trace_out.empty()) emit(a.trace_out, report(r, 2, false));
    if (!a.outputs_out.empty()) emit(a.outputs_out, report(r, 1, true));
    if (!a.schedule_out.empty()) emit(a.schedule_out, report(r, 2, true));
    hk_run_free(r);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2 || std::string(argv[1]) != "run") {
        std::cerr << "usage: " << argv[0] << " run --workflow W --inputs I --profile P [options]\n"
                  << "  (the `run` subcommand of helios, tools/helios_main.cpp:48-115, executed on the B200)\n";
        return 2;
    }
    try {
        RunArgs a = parse_run(argc, argv);
        return do_run(a);
    } catch (const Usage& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
