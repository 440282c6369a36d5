// `ndconv` command-line drop-in (reference: /root/reference/proj/tools/main.cpp) on the
// B200 library through the C++ drop-in header.  Same subcommands' options, output
// files, `<output>.manifest` key=value lines, trace CSV and exit codes:
//   0 ok, 1 other error, 2 usage, 3 FormatError, 4 ShapeError/BoundsError, 5 NumericError
// (main.cpp:420-438).  The reference parses with CLI11 (absent here), so this file has
// its own small parser for the same option syntax (`--opt value`, `--opt=value`,
// comma-separated lists, flags).
//
//   ndconv [--threads N] convolve --input X --kernel H --output Y
//   ndconv [--threads N] deconv --observed Y --kernel H --shape d1,d2[,d3] --output X
//          [--method pg|rl] [--max-iters N] [--tol T] [--step S] [--seedless]
//          [--trace-csv PATH]
//   ndconv metrics --reference A --estimate B
//   ndconv simulate --outdir D [--phantom lines|texture|PGM] [--size r[,c]] [--lines N]
//          [--psf gaussian|delta] [--psf-size k[,k]] [--sigma S] [--noise-mean M]
//          [--noise-std S] [--seed N]          (phantoms and noise generated on the device)
// verify / matrix (explicit-matrix property checks, O(N^2) host tooling) are not part
// of the B200 build.
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "ndconv_b200/ndconv.hpp"

using namespace ndconv;

namespace {

constexpr const char* kVersion = "0.1.0";

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

bool ends_with(const std::string& s, const std::string& suf) {
  return s.size() >= suf.size() && s.compare(s.size() - suf.size(), suf.size(), suf) == 0;
}

bool is_pgm(const std::string& p) { return ends_with(p, ".pgm"); }

Tensor load_tensor(const std::string& p) { return is_pgm(p) ? io::read_pgm(p) : io::read_tensor(p); }

void store_tensor(const Tensor& t, const std::string& p) {
  if (is_pgm(p))
    io::write_pgm(t, p, /*clamp=*/true);
  else
    io::write_tensor(t, p);
}

class Manifest {
 public:
  void add(const std::string& k, const std::string& v) { e_.emplace_back(k, v); }
  void add_num(const std::string& k, double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.17g", v);
    add(k, b);
  }
  void add_count(const std::string& k, std::size_t v) { add(k, std::to_string(v)); }
  void write(const std::string& path) const {
    std::ofstream out(path);
    if (!out) throw FormatError("cannot write manifest " + path);
    for (const auto& kv : e_) out << kv.first << "=" << kv.second << "\n";
    if (!out) throw FormatError("manifest write failure: " + path);
  }

 private:
  std::vector<std::pair<std::string, std::string>> e_;
};

Manifest header(const std::string& sub) {
  Manifest m;
  m.add("subcommand", sub);
  m.add("version", kVersion);
  return m;
}

std::string shape_csv(const Shape& s) {
  std::string o;
  for (std::size_t i = 0; i < s.ndim(); ++i) o += (i ? "," : "") + std::to_string(s.extent(i));
  return o;
}

// --- option parsing ---------------------------------------------------------------------------
struct Opts {
  std::map<std::string, std::string> kv;
  std::set<std::string> flags;
};

Opts parse_opts(const std::vector<std::string>& args, const std::set<std::string>& valued,
                const std::set<std::string>& flag_names) {
  Opts o;
  for (std::size_t i = 0; i < args.size(); ++i) {
    std::string a = args[i];
    if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument '" + a + "'");
    std::string key = a.substr(2), val;
    const auto eq = key.find('=');
    bool has_val = false;
    if (eq != std::string::npos) {
      val = key.substr(eq + 1);
      key = key.substr(0, eq);
      has_val = true;
    }
    if (flag_names.count(key)) {
      if (has_val) throw UsageError("--" + key + " takes no value");
      o.flags.insert(key);
    } else if (valued.count(key)) {
      if (!has_val) {
        if (i + 1 >= args.size()) throw UsageError("--" + key + " requires a value");
        val = args[++i];
      }
      o.kv[key] = val;
    } else {
      throw UsageError("unknown option --" + key);
    }
  }
  return o;
}

std::string req(const Opts& o, const std::string& k) {
  auto it = o.kv.find(k);
  if (it == o.kv.end()) throw UsageError("--" + k + " is required");
  return it->second;
}

std::size_t to_positive(const std::string& k, const std::string& v) {
  char* end = nullptr;
  const long long x = std::strtoll(v.c_str(), &end, 10);
  if (v.empty() || *end != '\0' || x <= 0) throw UsageError("--" + k + ": expected a positive integer");
  return static_cast<std::size_t>(x);
}

double to_nonneg(const std::string& k, const std::string& v) {
  char* end = nullptr;
  const double x = std::strtod(v.c_str(), &end);
  if (v.empty() || *end != '\0' || !(x >= 0)) throw UsageError("--" + k + ": expected a non-negative number");
  return x;
}

std::size_t to_count(const std::string& k, const std::string& v) {
  char* end = nullptr;
  const long long x = std::strtoll(v.c_str(), &end, 10);
  if (v.empty() || *end != '\0' || x < 0) throw UsageError("--" + k + ": expected a non-negative integer");
  return static_cast<std::size_t>(x);
}

double to_double(const std::string& k, const std::string& v) {
  char* end = nullptr;
  const double x = std::strtod(v.c_str(), &end);
  if (v.empty() || *end != '\0') throw UsageError("--" + k + ": expected a number");
  return x;
}

std::uint64_t to_u64(const std::string& k, const std::string& v) {
  char* end = nullptr;
  if (v.empty() || v[0] == '-') throw UsageError("--" + k + ": expected an unsigned integer");
  const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
  if (*end != '\0') throw UsageError("--" + k + ": expected an unsigned integer");
  return static_cast<std::uint64_t>(x);
}

// Comma-separated list; `positive` rejects zero entries (CLI11 PositiveNumber), `max_n`
// bounds the count (CLI11 expected(1, max_n)).
std::vector<std::size_t> to_list(const std::string& k, const std::string& v, bool positive = true,
                                 std::size_t max_n = 0) {
  std::vector<std::size_t> out;
  std::size_t start = 0;
  while (start <= v.size()) {
    const std::size_t comma = v.find(',', start);
    const std::string item = v.substr(start, comma == std::string::npos ? std::string::npos : comma - start);
    out.push_back(positive ? to_positive(k, item) : to_count(k, item));
    if (comma == std::string::npos) break;
    start = comma + 1;
  }
  if (max_n && out.size() > max_n) throw UsageError("--" + k + ": expected at most " + std::to_string(max_n) + " values");
  return out;
}

void write_trace_csv(const std::string& path, const DeconvReport& r) {
  std::ofstream out(path);
  if (!out) throw FormatError("cannot write trace " + path);
  out << "iter,objective,kkt\n";
  char b[96];
  for (std::size_t k = 1; k < r.objective_trace.size(); ++k) {
    const double kkt = k < r.kkt_trace.size() ? r.kkt_trace[k] : -1.0;
    std::snprintf(b, sizeof b, "%zu,%.17g,%.17g\n", k, r.objective_trace[k], kkt);
    out << b;
  }
  if (!out) throw FormatError("trace write failure: " + path);
}

// --- subcommands ------------------------------------------------------------------------------
int run_convolve(const std::vector<std::string>& args) {
  const Opts o = parse_opts(args, {"input", "kernel", "output"}, {});
  const std::string in = req(o, "input"), ker = req(o, "kernel"), out = req(o, "output");
  const Tensor x = load_tensor(in);
  const Kernel h(load_tensor(ker));
  const Tensor y = conv_full(x, h);
  store_tensor(y, out);
  Manifest m = header("convolve");
  m.add("input", in);
  m.add("kernel", ker);
  m.add("output", out);
  m.add("input_shape", shape_csv(x.shape()));
  m.add("kernel_shape", shape_csv(h.shape()));
  m.add("output_shape", shape_csv(y.shape()));
  m.write(out + ".manifest");
  return 0;
}

int run_deconv(const std::vector<std::string>& args) {
  const Opts o = parse_opts(args, {"observed", "kernel", "shape", "method", "max-iters", "tol", "step",
                                   "trace-csv", "output"},
                            {"seedless"});
  const std::string obs = req(o, "observed"), ker = req(o, "kernel"), out = req(o, "output");
  const std::vector<std::size_t> shape = to_list("shape", req(o, "shape"));
  const std::string method = o.kv.count("method") ? o.kv.at("method") : "pg";
  if (method != "pg" && method != "rl") throw UsageError("--method: expected pg or rl");
  const std::size_t max_iters = o.kv.count("max-iters") ? to_positive("max-iters", o.kv.at("max-iters")) : 500;
  const double tol = o.kv.count("tol") ? to_nonneg("tol", o.kv.at("tol")) : 1e-6;
  const double step = o.kv.count("step") ? to_nonneg("step", o.kv.at("step")) : 0.0;
  const std::string trace = o.kv.count("trace-csv") ? o.kv.at("trace-csv") : "";
  const bool seedless = o.flags.count("seedless") != 0;

  const Tensor y = load_tensor(obs);
  const Kernel h(load_tensor(ker));
  const Shape xs{std::vector<std::size_t>(shape)};
  DeconvReport rep = [&] {
    if (method == "pg") {
      DeconvConfig c;
      c.max_iters = max_iters;
      c.tol_rel_objective = tol;
      if (step > 0.0) c.initial_step = step;
      return deconv_pg(y, h, xs, c);
    }
    RlConfig c;
    c.max_iters = max_iters;
    c.tol_rel_change = tol;
    return deconv_rl(y, h, xs, c);
  }();
  store_tensor(rep.estimate, out);
  if (!trace.empty()) write_trace_csv(trace, rep);
  Manifest m = header("deconv");
  m.add("observed", obs);
  m.add("kernel", ker);
  m.add("output", out);
  m.add("method", method);
  m.add("shape", shape_csv(xs));
  m.add_count("max_iters", max_iters);
  m.add_num("tol", tol);
  m.add_num("step", step);
  m.add("seedless", seedless ? "true" : "false");
  if (!trace.empty()) m.add("trace_csv", trace);
  m.add("stop_reason", to_string(rep.stop_reason));
  m.add_count("iterations_run", rep.iterations_run);
  m.add_num("final_objective", rep.objective_trace.back());
  if (!rep.kkt_trace.empty()) m.add_num("final_kkt", rep.kkt_trace.back());
  if (method == "rl") m.add_count("negative_pixels_clamped", rep.negative_pixels_clamped);
  m.add_num("wall_time_seconds", rep.wall_time_seconds);
  m.write(out + ".manifest");
  if (rep.stop_reason == StopReason::stalled)
    throw NumericError("line search stalled before reaching the tolerance");
  return 0;
}

int run_metrics(const std::vector<std::string>& args) {
  const Opts o = parse_opts(args, {"reference", "estimate"}, {});
  const Tensor a = load_tensor(req(o, "reference"));
  const Tensor b = load_tensor(req(o, "estimate"));
  const double snr = sim::snr_db(a, b);
  if (std::isinf(snr))
    std::printf("inf\n");
  else
    std::printf("%.12f\n", snr);
  return 0;
}

int run_simulate(const std::vector<std::string>& args) {
  const Opts o = parse_opts(args, {"phantom", "size", "lines", "psf", "psf-size", "sigma", "noise-mean", "noise-std",
                                   "seed", "outdir"},
                            {});
  const std::string outdir = req(o, "outdir");
  auto get = [&](const char* k, const char* dflt) { return o.kv.count(k) ? o.kv.at(k) : std::string(dflt); };
  const std::string phantom = get("phantom", "lines"), psf_kind = get("psf", "gaussian");
  const std::vector<std::size_t> size = to_list("size", get("size", "128"), false, 2);
  const std::size_t lines = to_positive("lines", get("lines", "9"));
  std::vector<std::size_t> psf_ext = to_list("psf-size", get("psf-size", "5"), false, 2);
  const double sigma = to_double("sigma", get("sigma", "1.0"));
  const double noise_mean = to_double("noise-mean", get("noise-mean", "0.0"));
  const double noise_std = to_double("noise-std", get("noise-std", "5.0"));
  const std::uint64_t seed = to_u64("seed", get("seed", "1"));

  const std::size_t rows = size.at(0), cols = size.size() > 1 ? size.at(1) : rows;
  const Tensor truth = phantom == "lines"     ? sim::phantom_lines(rows, cols, lines, 255.0)
                       : phantom == "texture" ? sim::phantom_texture(rows, cols)
                                              : io::read_pgm(phantom);  // any PGM serves as a phantom
  if (psf_ext.size() == 1) psf_ext.push_back(psf_ext[0]);
  const Kernel psf = psf_kind == "gaussian" ? sim::gaussian_psf(psf_ext, sigma)
                     : psf_kind == "delta"  ? sim::delta_psf(psf_ext)
                                            : throw Error("unknown --psf kind '" + psf_kind +
                                                          "' (expected gaussian or delta)");
  const Tensor observed = sim::add_gaussian_noise(conv_full(truth, psf), {noise_mean, noise_std, seed});

  std::filesystem::create_directories(outdir);
  const std::filesystem::path dir(outdir);
  io::write_tensor(truth, (dir / "truth.ndt").string());
  io::write_pgm(truth, (dir / "truth.pgm").string(), /*clamp=*/true);
  io::write_tensor(psf.tensor(), (dir / "psf.ndt").string());
  io::write_tensor(observed, (dir / "observed.ndt").string());
  io::write_pgm(observed, (dir / "observed.pgm").string(), /*clamp=*/true);

  Manifest m = header("simulate");
  m.add("phantom", phantom);
  m.add("size", shape_csv(truth.shape()));
  m.add_count("lines", lines);
  m.add("psf", psf_kind);
  m.add("psf_size", shape_csv(psf.shape()));
  m.add_num("sigma", sigma);
  m.add_num("noise_mean", noise_mean);
  m.add_num("noise_std", noise_std);
  m.add("seed", std::to_string(seed));
  m.add("outdir", outdir);
  m.add("truth", (dir / "truth.ndt").string());
  m.add("psf_file", (dir / "psf.ndt").string());
  m.add("observed", (dir / "observed.ndt").string());
  m.add("observed_shape", shape_csv(observed.shape()));
  m.write((dir / "manifest.txt").string());
  return 0;
}

void usage(std::FILE* f) {
  std::fprintf(f,
               "ndconv %s (B200 / sm_100a) -- n-dimensional convolution and deconvolution\n"
               "usage: ndconv [--threads N] <convolve|deconv|metrics|simulate> [options]\n"
               "  convolve --input X --kernel H --output Y\n"
               "  deconv   --observed Y --kernel H --shape d1,d2 --output X [--method pg|rl]\n"
               "           [--max-iters N] [--tol T] [--step S] [--seedless] [--trace-csv P]\n"
               "  metrics  --reference A --estimate B\n"
               "  simulate --outdir D [--phantom lines|texture|P.pgm] [--size r[,c]] [--lines N]\n"
               "           [--psf gaussian|delta] [--psf-size k[,k]] [--sigma S] [--noise-mean M]\n"
               "           [--noise-std S] [--seed N]\n",
               kVersion);
}

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> args(argv + 1, argv + argc);
  std::size_t i = 0;
  try {
    unsigned threads = 1;
    while (i < args.size() && args[i].rfind("--", 0) == 0) {
      const std::string a = args[i];
      if (a == "--help" || a == "-h") {
        usage(stdout);
        return 0;
      }
      if (a == "--threads" || a.rfind("--threads=", 0) == 0) {
        std::string v;
        if (a == "--threads") {
          if (i + 1 >= args.size()) throw UsageError("--threads requires a value");
          v = args[++i];
        } else {
          v = a.substr(10);
        }
        threads = static_cast<unsigned>(to_positive("threads", v));
        ++i;
        continue;
      }
      throw UsageError("unknown option " + a);
    }
    if (i >= args.size()) throw UsageError("a subcommand is required");
    const std::string sub = args[i];
    const std::vector<std::string> rest(args.begin() + i + 1, args.end());
    for (const std::string& r : rest)
      if (r == "--help" || r == "-h") {
        usage(stdout);
        return 0;
      }
    set_max_threads(threads);
    if (sub == "convolve") return run_convolve(rest);
    if (sub == "deconv") return run_deconv(rest);
    if (sub == "metrics") return run_metrics(rest);
    if (sub == "simulate") return run_simulate(rest);
    if (sub == "verify" || sub == "matrix")
      throw UsageError(sub + ": host-side tooling, not part of the B200 build");
    throw UsageError("unknown subcommand '" + sub + "'");
  } catch (const UsageError& e) {
    std::fprintf(stderr, "usage error: %s\n", e.what());
    usage(stderr);
    return 2;
  } catch (const FormatError& e) {
    std::fprintf(stderr, "format error: %s\n", e.what());
    return 3;
  } catch (const ShapeError& e) {
    std::fprintf(stderr, "shape error: %s\n", e.what());
    return 4;
  } catch (const BoundsError& e) {
    std::fprintf(stderr, "bounds error: %s\n", e.what());
    return 4;
  } catch (const NumericError& e) {
    std::fprintf(stderr, "numerical error: %s\n", e.what());
    return 5;
  } catch (const Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "unexpected error: %s\n", e.what());
    return 1;
  }
}
