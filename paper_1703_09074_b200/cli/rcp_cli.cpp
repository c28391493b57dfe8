// SPDX-License-Identifier: MIT
// `rcp` command line front end, the drop-in for the reference CLI
// (/root/reference/proj/tools/main.cpp): same subcommands, options, summary
// line and exit codes, over the B200 library (include/rcp_b200/rcp.hpp, the
// C ABI in include/rcpg.h) and the reference's file formats (io.hpp here).
//
//   rcp synth --shape 100,100,100 --rank 10 [--snr 10] [--seed S] --out x.dten
//             [--truth t.kten] [--csv-export x.csv] [--dtype f64|f32]
//   rcp decompose --in x.dten --rank R [--method als|bcd] [--deterministic]
//             [--oversample P] [--power-iters Q] [--modes 1,2] [--tol T]
//             [--max-iter N] [--seed S] --out m.kten [--trace fit.csv]
//   rcp reconstruct --in m.kten --out x.dten [--csv-export x.csv]
//
// Exit codes (main.cpp:289-311): 0 success (decompose: converged), 2 decompose
// ran to max_iter without converging, 1 on any error (parse errors included).
// Not carried over: `bound`, `bench` (diagnostics sweeps) and `--toy-video`
// (demo generator).
// --dtype is an extension: the fp32 configs are stored as dtype-1 files.
#include <chrono>
#include <cstdio>
#include <iomanip>
#include <iostream>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "rcp_b200/io.hpp"
#include "rcp_b200/rcp.hpp"

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// --name value | --name=value | flags
struct Args {
  std::map<std::string, std::string> kv;
  std::set<std::string> flags;
  bool has(const std::string& k) const { return kv.count(k) || flags.count(k); }
  std::string str(const std::string& k, const std::string& d = "") const {
    auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
  }
};

Args parse(int argc, char** argv, int first, const std::set<std::string>& opts, const std::set<std::string>& flag_names) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string tok = argv[i];
    if (tok.rfind("--", 0) != 0) throw UsageError("The following argument was not expected: " + tok);
    std::string val;
    bool inline_val = false;
    const auto eq = tok.find('=');
    if (eq != std::string::npos) {
      val = tok.substr(eq + 1);
      tok = tok.substr(0, eq);
      inline_val = true;
    }
    if (flag_names.count(tok)) {
      if (inline_val) throw UsageError(tok + ": flag takes no value");
      a.flags.insert(tok);
    } else if (opts.count(tok)) {
      if (!inline_val) {
        if (i + 1 >= argc) throw UsageError(tok + " requires an argument");
        val = argv[++i];
      }
      a.kv[tok] = val;
    } else {
      throw UsageError("The following argument was not expected: " + tok);
    }
  }
  return a;
}

void require(const Args& a, const std::string& k) {
  if (!a.has(k)) throw UsageError(k + " is required");
}

long long to_int(const std::string& k, const std::string& s) {
  try {
    size_t pos = 0;
    const long long v = std::stoll(s, &pos);
    if (pos != s.size()) throw std::invalid_argument(s);
    return v;
  } catch (const std::exception&) {
    throw UsageError(k + ": " + s + " is not an integer");
  }
}
unsigned long long to_u64(const std::string& k, const std::string& s) {
  try {
    size_t pos = 0;
    const unsigned long long v = std::stoull(s, &pos);
    if (pos != s.size() || (!s.empty() && s[0] == '-')) throw std::invalid_argument(s);
    return v;
  } catch (const std::exception&) {
    throw UsageError(k + ": " + s + " is not an unsigned integer");
  }
}
double to_double(const std::string& k, const std::string& s) {
  try {
    size_t pos = 0;
    const double v = std::stod(s, &pos);
    if (pos != s.size()) throw std::invalid_argument(s);
    return v;
  } catch (const std::exception&) {
    throw UsageError(k + ": " + s + " is not a number");
  }
}
std::vector<rcp::Index> to_list(const std::string& k, const std::string& s) {
  std::vector<rcp::Index> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ',')) out.push_back(rcp::Index(to_int(k, item)));
  return out;
}

// ------------------------------------------------------------------ synth
template <typename S>
int synth_as(const Args& a) {
  const rcp::Shape shape = to_list("--shape", a.str("--shape"));
  const rcp::Index rank = rcp::Index(to_int("--rank", a.str("--rank")));
  const std::uint64_t seed = a.has("--seed") ? to_u64("--seed", a.str("--seed")) : 0;
  double snr = 0.0;
  if (a.has("--snr")) {
    snr = to_double("--snr", a.str("--snr"));
    if (!(snr > 0.0)) throw std::invalid_argument("add_noise: snr must be positive");
  }
  auto [tensor, truth] = rcp::random_lowrank<S>(shape, rank, seed, snr, seed);  // main.cpp:45-47: NoiseSpec{snr, seed}
  if (a.has("--truth")) rcp::io::write_kruskal(a.str("--truth"), truth);
  rcp::io::write_tensor(a.str("--out"), tensor);
  if (a.has("--csv-export")) rcp::io::write_tensor_csv(a.str("--csv-export"), tensor);
  return 0;
}

int run_synth(const Args& a) {
  require(a, "--out");
  if (a.has("--toy-video")) throw std::invalid_argument("synth: --toy-video is not part of this build");
  require(a, "--shape");
  require(a, "--rank");
  const std::string dt = a.str("--dtype", "f64");
  if (dt == "f64") return synth_as<double>(a);
  if (dt == "f32") return synth_as<float>(a);
  throw UsageError("--dtype: " + dt + " not in {f64, f32}");
}

// -------------------------------------------------------------- decompose
template <typename S>
int decompose_as(const Args& a) {
  const rcp::Tensor<S> tensor = rcp::io::read_tensor<S>(a.str("--in"));
  rcp::DecomposeConfig cfg;
  cfg.rank = rcp::Index(to_int("--rank", a.str("--rank")));
  const std::string method = a.str("--method", "als");
  if (method != "als" && method != "bcd") throw UsageError("--method: " + method + " not in {als, bcd}");
  cfg.method = method == "bcd" ? rcp::SolveMethod::bcd : rcp::SolveMethod::als;
  cfg.randomized = !a.has("--deterministic");
  cfg.tol = a.has("--tol") ? to_double("--tol", a.str("--tol")) : 1e-5;
  cfg.max_iter = a.has("--max-iter") ? int(to_int("--max-iter", a.str("--max-iter"))) : 500;
  cfg.seed = a.has("--seed") ? to_u64("--seed", a.str("--seed")) : 0;
  cfg.compress.target_rank = cfg.rank;
  cfg.compress.oversampling = a.has("--oversample") ? rcp::Index(to_int("--oversample", a.str("--oversample"))) : 10;
  cfg.compress.power_iterations = a.has("--power-iters") ? int(to_int("--power-iters", a.str("--power-iters"))) : 2;
  cfg.compress.seed = rcp::derive_seed(cfg.seed, rcp::stream_id(rcp::StreamDomain::compress));
  if (a.has("--modes")) {
    std::vector<rcp::Index> zero_based;
    for (rcp::Index m : to_list("--modes", a.str("--modes"))) {
      if (m < 1 || m > tensor.order()) throw std::invalid_argument("decompose: --modes entries are 1-based");
      zero_based.push_back(m - 1);
    }
    cfg.compress.modes = std::move(zero_based);
  }
  const auto t0 = std::chrono::steady_clock::now();
  const auto [model, trace] = rcp::decompose(tensor, cfg);
  const double seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  rcp::io::write_kruskal(a.str("--out"), model);
  if (a.has("--trace")) rcp::io::write_trace_csv(a.str("--trace"), trace);
  std::cout << "method=" << rcp::method_name(cfg.method) << " randomized=" << (cfg.randomized ? "true" : "false")
            << " rank=" << cfg.rank << " iters=" << trace.iterations << " seconds=" << std::setprecision(6) << seconds
            << " error=" << std::setprecision(12) << trace.final_relative_error << '\n';
  return trace.converged ? 0 : 2;
}

int run_decompose(const Args& a) {
  require(a, "--in");
  require(a, "--rank");
  require(a, "--out");
  if (a.has("--deterministic"))
    for (const char* k : {"--oversample", "--power-iters", "--modes"})
      if (a.has(k)) throw UsageError(std::string("--deterministic excludes ") + k);
  return rcp::io::tensor_dtype(a.str("--in")) == 1 ? decompose_as<float>(a) : decompose_as<double>(a);
}

// ------------------------------------------------------------ reconstruct
int run_reconstruct(const Args& a) {
  require(a, "--in");
  require(a, "--out");
  const auto model = rcp::io::read_kruskal<double>(a.str("--in"));
  const auto tensor = rcp::reconstruct(model);
  rcp::io::write_tensor(a.str("--out"), tensor);
  if (a.has("--csv-export")) rcp::io::write_tensor_csv(a.str("--csv-export"), tensor);
  return 0;
}

const char* kUsage =
    "Randomized CP tensor decomposition toolkit (B200)\n"
    "Usage: rcp SUBCOMMAND [OPTIONS]\n"
    "Subcommands:\n"
    "  synth        Generate a synthetic low-rank tensor\n"
    "  decompose    Fit a CP model to a tensor file\n"
    "  reconstruct  Expand a model file to a dense tensor\n";

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "A subcommand is required\n" << kUsage;
    return 1;
  }
  const std::string sub = argv[1];
  if (sub == "--help" || sub == "-h") {
    std::cout << kUsage;
    return 0;
  }
  try {
    if (sub == "synth")
      return run_synth(parse(argc, argv, 2, {"--shape", "--rank", "--snr", "--seed", "--out", "--truth", "--csv-export",
                                             "--dtype"},
                             {"--toy-video"}));
    if (sub == "decompose")
      return run_decompose(parse(argc, argv, 2, {"--in", "--rank", "--method", "--oversample", "--power-iters",
                                                 "--modes", "--tol", "--max-iter", "--seed", "--out", "--trace"},
                                 {"--deterministic"}));
    if (sub == "reconstruct")
      return run_reconstruct(parse(argc, argv, 2, {"--in", "--out", "--csv-export"}, {}));
    throw UsageError("The following argument was not expected: " + sub);
  } catch (const UsageError& e) {
    std::cerr << e.what() << "\nRun with --help for more information.\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}
