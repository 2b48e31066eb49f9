// fde_b200: command-line drop-in for the reference's `fde solve` and
// `fde table` (proj/src/cli.cpp:84-211, report writer proj/src/report.cpp:
// 28-80) running the B200 library through its C ABI (include/fde_b200.h).
//
//   fde_b200 solve --example K | --coeff-preset K | --config K  --n N [options]
//   fde_b200 table --table K [--sizes 16 32 64 128] [options]
//
// Same flags, defaults, CSV columns and manifest as the reference; the
// reference's `--n <= 4096` cap becomes the line-kernel limit (n <= 4096 per
// direction).  Extensions: --config K runs BASELINE configuration K (1..5,
// seeded sources), --solver bicgstab, --seed.  Exit codes
// follow the reference (proj/src/cli.cpp:135,473-476): 0 ok, 1 some step did
// not converge or the run failed with an exception (library failures print
// fde_last_error()), 2 usage error.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <ctime>
#include <filesystem>
#include <fstream>
#include <limits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/fde_b200.h"

namespace {

namespace fs = std::filesystem;

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct LibError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void check(int rc, const char* what) {
  if (rc != FDE_OK) throw LibError(std::string(what) + ": " + fde_last_error());
}

std::string dstr(double v) {  // cli.cpp:28-32
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.15g", v);
  return buf;
}
std::string sci(double v) {  // report.cpp:66-70
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.5e", v);
  return buf;
}
std::string fixed3(double v) {  // report.cpp:72-76
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.3f", v);
  return buf;
}

// report.cpp:12-35: <dir>/<command>-<UTC yyyymmdd-hhmmssmmm>.csv
fs::path results_file(const fs::path& dir, const std::string& command) {
  fs::create_directories(dir);
  using namespace std::chrono;
  const auto now = system_clock::now();
  const std::time_t secs = system_clock::to_time_t(now);
  const auto ms = duration_cast<milliseconds>(now.time_since_epoch()) % 1000;
  std::tm tm{};
  gmtime_r(&secs, &tm);
  char buf[40];
  std::snprintf(buf, sizeof buf, "%04d%02d%02d-%02d%02d%02d%03d", tm.tm_year + 1900,
                tm.tm_mon + 1, tm.tm_mday, tm.tm_hour, tm.tm_min, tm.tm_sec, (int)ms.count());
  return dir / (command + "-" + buf + ".csv");
}

std::string json_str(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o + "\"";
}

// report.cpp:37-50: {"command", "parameters" (ordered), "seed", "version"}
void write_manifest(const fs::path& csv, const std::string& command,
                    const std::vector<std::pair<std::string, std::string>>& params,
                    unsigned long long seed) {
  fs::path p = csv;
  p.replace_extension(".manifest");
  std::ofstream out(p);
  if (!out) throw std::runtime_error("cannot write " + p.string());
  out << "{\n  \"command\": " << json_str(command) << ",\n  \"parameters\": {";
  for (size_t i = 0; i < params.size(); ++i)
    out << (i ? "," : "") << "\n    " << json_str(params[i].first) << ": "
        << json_str(params[i].second);
  out << (params.empty() ? "}" : "\n  }") << ",\n  \"seed\": " << seed
      << ",\n  \"version\": \"fde-0.1.0\",\n  \"backend\": \"b200\"\n}\n";
}

struct Csv {
  std::ofstream out;
  explicit Csv(const fs::path& p) : out(p) {
    if (!out) throw std::runtime_error("cannot write " + p.string());
  }
  void comment(const std::string& t) { out << "# " << t << '\n'; }
  void row(const std::vector<std::string>& cells) {
    for (size_t i = 0; i < cells.size(); ++i) out << (i ? "," : "") << cells[i];
    out << '\n';
  }
};

// ---- argument parsing (the subset of CLI11 behaviour the reference uses)
struct Args {
  std::vector<std::string> a;
  size_t i = 0;
  bool more() const { return i < a.size(); }
  std::string flag() { return a[i++]; }
  std::string value(const std::string& f) {
    if (i >= a.size()) throw Usage(f + " needs a value");
    return a[i++];
  }
};
double to_d(const std::string& f, const std::string& v) {
  char* e = nullptr;
  const double d = std::strtod(v.c_str(), &e);
  if (!e || *e) throw Usage(f + ": not a number: " + v);
  return d;
}
long to_l(const std::string& f, const std::string& v) {
  char* e = nullptr;
  const long d = std::strtol(v.c_str(), &e, 10);
  if (!e || *e) throw Usage(f + ": not an integer: " + v);
  return d;
}
void range(const std::string& f, long v, long lo, long hi) {
  if (v < lo || v > hi)
    throw Usage(f + " must be in [" + std::to_string(lo) + ", " + std::to_string(hi) + "]");
}
int precond_id(const std::string& name) {
  if (name == "none") return 0;
  if (name == "p2") return 1;
  if (name == "mgm") return 2;
  if (name == "p2-exact") return 3;
  if (name == "mgm-galerkin") return 4;
  throw Usage("unknown preconditioner: " + name);
}
int coarse_id(const std::string& name) {  // cli.cpp:61-66
  if (name == "lu") return 0;
  if (name == "sweeps") return 1;
  if (name == "none") return 2;
  throw Usage("unknown coarse solve: " + name);
}
double default_alpha(int) { return 1.8; }                          // cli.cpp:39
double default_beta(int which) { return which == 1 ? 1.6 : 1.9; }  // cli.cpp:40

struct March {
  double avg = 0.0, err = std::numeric_limits<double>::quiet_NaN(), wall = 0.0;
  bool has_error = false, converged = true;
};

// time_march + SolveReport (driver.cpp:10-69) through fde_time_march
March march(const fde_problem& p, size_t n, size_t steps, const fde_driver_config& cfg) {
  std::vector<double> u(n * n), res(steps);
  std::vector<size_t> its(steps);
  March r;
  check(fde_time_march(&p, n, n, steps, &cfg, u.data(), its.data(), res.data(), &r.wall),
        "time_march");
  double sum = 0.0;
  for (size_t k = 0; k < steps; ++k) {
    sum += (double)its[k];
    r.converged = r.converged && res[k] <= cfg.tol;  // KrylovResult::converged
  }
  r.avg = steps ? sum / (double)steps : 0.0;
  if (p.preset > 100) {  // manufactured examples have an exact solution
    check(fde_error_inf(&p, n, n, steps, p.t_final, u.data(), &r.err), "error_inf");
    r.has_error = true;
  }
  return r;
}

int cmd_solve(Args& a) {
  int example = 0, preset = 0, config = 0;
  long n = -1, m = 0, restart = 20, max_outer = 100, cycles = 1, coarse_sweeps = 3;
  std::string precond = "none", coarse = "sweeps", out_dir = "results", solver = "gmres";
  double tol = 1e-7, omega = 0.9, alpha = 0.0, beta = 0.0;
  unsigned long long seed = 0;
  std::vector<double> domain;
  while (a.more()) {
    const std::string f = a.flag();
    if (f == "--example") example = (int)to_l(f, a.value(f)), range(f, example, 1, 3);
    else if (f == "--coeff-preset") preset = (int)to_l(f, a.value(f)), range(f, preset, 1, 3);
    else if (f == "--config") config = (int)to_l(f, a.value(f)), range(f, config, 1, 5);
    else if (f == "--n") n = to_l(f, a.value(f)), range(f, n, 1, 4096);
    else if (f == "--m") m = to_l(f, a.value(f)), range(f, m, 0, 1L << 30);
    else if (f == "--precond") precond = a.value(f), precond_id(precond);
    else if (f == "--tol") {
      tol = to_d(f, a.value(f));
      if (!(tol > 0)) throw Usage("--tol must be positive");
    } else if (f == "--restart") restart = to_l(f, a.value(f)), range(f, restart, 1, 10000);
    else if (f == "--max-outer") max_outer = to_l(f, a.value(f)), range(f, max_outer, 1, 100000);
    else if (f == "--omega") {
      omega = to_d(f, a.value(f));
      if (!(omega > 0)) throw Usage("--omega must be positive");
    } else if (f == "--vcycles-per-apply") cycles = to_l(f, a.value(f)), range(f, cycles, 1, 16);
    else if (f == "--coarse") coarse = a.value(f), coarse_id(coarse);
    else if (f == "--coarse-sweeps")
      coarse_sweeps = to_l(f, a.value(f)), range(f, coarse_sweeps, 1, 64);
    else if (f == "--alpha") alpha = to_d(f, a.value(f));
    else if (f == "--beta") beta = to_d(f, a.value(f));
    else if (f == "--domain") {
      for (int k = 0; k < 4; ++k) domain.push_back(to_d(f, a.value(f)));
    } else if (f == "--out-dir") out_dir = a.value(f);
    else if (f == "--solver") {
      solver = a.value(f);
      if (solver != "gmres" && solver != "bicgstab") throw Usage("unknown solver: " + solver);
    } else if (f == "--seed") seed = (unsigned long long)to_l(f, a.value(f));
    else throw Usage("unknown option for solve: " + f);
  }
  if (example == 0 && preset == 0 && config == 0) {
    std::fprintf(stderr, "solve needs --example or --coeff-preset\n");  // cli.cpp:86-89
    return 2;
  }
  fde_problem p{};
  std::string label;
  size_t nn = 0, steps = 0;
  if (config) {  // BASELINE configuration (grid, steps and tau from the config)
    size_t cn = 0, cs = 0;
    check(fde_problem_preset(config, seed, -1, (size_t)m, 0.0, &p, &cn, &cs), "preset");
    nn = n > 0 ? (size_t)n : cn;
    steps = cs;
    label = "config-" + std::to_string(config);
  } else {
    if (n < 0) throw Usage("--n is required");
    const int which = example > 0 ? example : preset;  // cli.cpp:69-82
    const double al = alpha > 0.0 ? alpha : default_alpha(which);
    const double be = beta > 0.0 ? beta : default_beta(which);
    if (domain.empty()) check(fde_problem_example_default(which, al, be, &p), "example");
    else check(fde_problem_example(which, al, be, domain[0], domain[1], domain[2], domain[3], &p),
               "example");
    nn = (size_t)n;
    steps = m > 0 ? (size_t)m : nn;
    label = example > 0 ? std::to_string(example) : "custom-" + std::to_string(which);
  }
  fde_driver_config cfg;
  fde_driver_config_default(&cfg);
  cfg.precond = precond_id(precond);
  cfg.tol = tol;
  cfg.restart = (size_t)restart;
  cfg.max_outer = (size_t)max_outer;
  cfg.omega = omega;
  cfg.cycles = (size_t)cycles;
  cfg.coarse = coarse_id(coarse);
  cfg.coarse_sweeps = (size_t)coarse_sweeps;
  cfg.solver = solver == "bicgstab" ? 1 : 0;
  const March r = march(p, nn, steps, cfg);

  const fs::path csv = results_file(out_dir, "solve");
  {
    Csv w(csv);
    w.row({"example", "n", "precond", "avg_iters", "error_inf", "wall_time"});
    w.row({label, std::to_string(nn), precond, fixed3(r.avg), r.has_error ? sci(r.err) : "nan",
           fixed3(r.wall)});
  }
  std::vector<std::pair<std::string, std::string>> params = {
      {"example", label},
      {"n", std::to_string(nn)},
      {"m", std::to_string(steps)},
      {"precond", precond},
      {"tol", dstr(tol)},
      {"restart", std::to_string(restart)},
      {"omega", dstr(omega)},
      {"vcycles-per-apply", std::to_string(cycles)},
      {"alpha", dstr(p.alpha)},
      {"beta", dstr(p.beta)},
      {"domain", dstr(p.ax) + " " + dstr(p.bx) + " " + dstr(p.ay) + " " + dstr(p.by)}};
  if (solver != "gmres") params.push_back({"solver", solver});
  write_manifest(csv, "solve", params, seed);
  std::printf("%s n=%zu precond=%s avg_iters=%.3f error_inf=%s wall=%.3fs%s\n", label.c_str(), nn,
              precond.c_str(), r.avg, r.has_error ? sci(r.err).c_str() : "n/a", r.wall,
              r.converged ? "" : "  [NOT CONVERGED]");
  std::printf("wrote %s\n", csv.string().c_str());
  return r.converged ? 0 : 1;
}

int cmd_table(Args& a) {  // cli.cpp:151-211
  int table = 0;
  std::vector<size_t> sizes;
  double tol = 1e-7, omega = 0.9;
  long restart = 20, restart_none = 512, cycles = 1;
  std::string out_dir = "results";
  while (a.more()) {
    const std::string f = a.flag();
    if (f == "--table") table = (int)to_l(f, a.value(f)), range(f, table, 1, 3);
    else if (f == "--sizes") {
      while (a.more() && a.a[a.i].rfind("--", 0) != 0) {
        const long s = to_l(f, a.flag());
        if (s != 16 && s != 32 && s != 64 && s != 128) throw Usage("--sizes: 16, 32, 64 or 128");
        sizes.push_back((size_t)s);
      }
    } else if (f == "--tol") tol = to_d(f, a.value(f));
    else if (f == "--restart") restart = to_l(f, a.value(f));
    else if (f == "--restart-none") restart_none = to_l(f, a.value(f));
    else if (f == "--omega") omega = to_d(f, a.value(f));
    else if (f == "--vcycles-per-apply") cycles = to_l(f, a.value(f)), range(f, cycles, 1, 16);
    else if (f == "--out-dir") out_dir = a.value(f);
    else throw Usage("unknown option for table: " + f);
  }
  if (!table) throw Usage("--table is required");
  if (sizes.empty()) sizes = {16, 32, 64, 128};
  std::sort(sizes.begin(), sizes.end());
  sizes.erase(std::unique(sizes.begin(), sizes.end()), sizes.end());
  const std::vector<std::string> columns =
      table == 1 ? std::vector<std::string>{"none", "p2", "p2-exact", "mgm", "mgm-galerkin"}
                 : std::vector<std::string>{"none", "p2", "mgm"};
  fde_problem p{};
  check(fde_problem_example_default(table, default_alpha(table), default_beta(table), &p),
        "example");
  const fs::path csv = results_file(out_dir, "table");
  bool all_ok = true;
  {
    Csv w(csv);
    w.comment("average GMRES iterations per preconditioner, final max-norm error");
    w.comment("P_JLZ column omitted: literature baseline, not reimplemented here");
    std::vector<std::string> header{"n"};
    for (const auto& c : columns) header.push_back(c);
    header.push_back("error_inf");
    w.row(header);
    for (size_t n : sizes) {
      std::vector<std::string> cells{std::to_string(n)};
      double err = std::numeric_limits<double>::quiet_NaN();
      for (const auto& c : columns) {
        fde_driver_config cfg;
        fde_driver_config_default(&cfg);
        cfg.precond = precond_id(c);
        cfg.tol = tol;
        cfg.restart = (size_t)(cfg.precond == 0 ? restart_none : restart);
        cfg.omega = omega;
        cfg.cycles = (size_t)cycles;
        const March r = march(p, n, n, cfg);
        all_ok = all_ok && r.converged;
        cells.push_back(fixed3(r.avg));
        if (r.has_error) err = r.err;
        std::printf("table %d n=%zu precond=%s avg_iters=%.3f wall=%.3fs%s\n", table, n, c.c_str(),
                    r.avg, r.wall, r.converged ? "" : "  [NOT CONVERGED]");
      }
      cells.push_back(sci(err));
      w.row(cells);
    }
  }
  std::string size_list;
  for (size_t n : sizes) size_list += (size_list.empty() ? "" : " ") + std::to_string(n);
  write_manifest(csv, "table",
                 {{"table", std::to_string(table)},
                  {"sizes", size_list},
                  {"tol", dstr(tol)},
                  {"restart", std::to_string(restart)},
                  {"omega", dstr(omega)},
                  {"vcycles-per-apply", std::to_string(cycles)}},
                 0);
  std::printf("wrote %s\n", csv.string().c_str());
  return all_ok ? 0 : 1;
}

const char* kHelp =
    "fde_b200 -- B200 fractional diffusion solver (drop-in for `fde solve` / `fde table`)\n"
    "  solve (--example K | --coeff-preset K | --config K) --n N [--m M]\n"
    "        [--precond none|p2|p2-exact|mgm|mgm-galerkin]\n"
    "        [--tol T] [--restart R] [--max-outer O] [--omega W] [--vcycles-per-apply C]\n"
    "        [--coarse lu|sweeps|none] [--coarse-sweeps S] [--alpha A] [--beta B]\n"
    "        [--domain ax bx ay by] [--solver gmres|bicgstab] [--seed S] [--out-dir DIR]\n"
    "  table --table K [--sizes 16 32 64 128] [--tol T] [--restart R] [--restart-none R]\n"
    "        [--omega W] [--vcycles-per-apply C] [--out-dir DIR]\n";

}  // namespace

int main(int argc, char** argv) {
  Args a;
  for (int i = 1; i < argc; ++i) a.a.emplace_back(argv[i]);
  try {
    if (!a.more() || a.a[0] == "--help" || a.a[0] == "-h") {
      std::fputs(kHelp, a.more() ? stdout : stderr);
      return a.more() ? 0 : 2;
    }
    const std::string cmd = a.flag();
    if (cmd == "solve") return cmd_solve(a);
    if (cmd == "table") return cmd_table(a);
    throw Usage("unknown subcommand: " + cmd);
  } catch (const Usage& e) {
    std::fprintf(stderr, "error: %s\n%s", e.what(), kHelp);
    return 2;
  } catch (const LibError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
