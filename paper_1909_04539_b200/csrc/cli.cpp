// bandsolve_b200 — the benchmark command of the reference's CLI
// (tools/main.cpp:129-278, run_bench) on the GPU library. Same options, the
// same timing CSV schema (problem,variant,n,m,steps,threads,wall_s,
// per_step_mean_s,per_step_std_s,elements) and the same companion
// <out>.speedup.csv (per-system time / each other variant's time per cell),
// so the paper's speed-up surfaces come out of
// one command. Every cell is one bandsolve_bench_run call: the Crank-Nicolson
// time-stepping loop of pde.cpp run_benchmark, each step timed on the device.
//
// Extension: variant "cusparse" (the per-system step with cuSPARSE's
// gtsvInterleavedBatch / gpsvInterleavedBatch, the paper's cuThomasBatch
// baseline). When it is in the list, a second companion
// <out>.speedup_cusparse.csv gives the cuSPARSE time / each other variant's.
//
//   bandsolve_b200 bench [--problem diffusion|hyperdiffusion|both]
//       [--variants shared,persystem,uniform,cusparse] [--n 64,128,256]
//       [--m 64,256,1024] [--steps 1000] [--dt X] [--threads T]
//       [--out bench.csv] [--dump-every D --dump-prefix P]
//   bandsolve_b200 --version
//
// Exit codes as the reference: 0 ok, 1 solver/IO failure, 2 bad arguments,
// 3 IBAT failure.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "../../include/bandsolve.h"

namespace {

enum Exit { kOk = 0, kSolver = 1, kArgs = 2, kIbat = 3 };

std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out(1);
  for (char ch : s) {
    if (ch == ',') out.emplace_back();
    else out.back() += ch;
  }
  return out;
}

bool sizes(const std::string& s, std::vector<size_t>& out) {
  for (const std::string& tok : split(s)) {
    if (tok.empty() || tok.find_first_not_of("0123456789") != std::string::npos) return false;
    const unsigned long long v = std::strtoull(tok.c_str(), nullptr, 10);
    if (v == 0) return false;
    out.push_back(static_cast<size_t>(v));
  }
  return !out.empty();
}

// write to <path>.tmp, then rename: a failed run leaves no partial file
bool write_file(const std::string& path, const std::string& text) {
  const std::string tmp = path + ".tmp";
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return false;
  bool ok = std::fwrite(text.data(), 1, text.size(), f) == text.size();
  ok = (std::fclose(f) == 0) && ok;
  if (ok && std::rename(tmp.c_str(), path.c_str()) == 0) return true;
  std::remove(tmp.c_str());
  return false;
}

std::string companion(const std::string& out, const char* tag) {
  const std::string ext = ".csv";
  if (out.size() > ext.size() && out.compare(out.size() - ext.size(), ext.size(), ext) == 0)
    return out.substr(0, out.size() - ext.size()) + "." + tag + ".csv";
  return out + "." + tag;
}

int exit_for(bandsolve_status st) {
  if (st == BANDSOLVE_OK) return kOk;
  if (st == BANDSOLVE_ERR_BAD_ARG) return kArgs;
  if (st == BANDSOLVE_ERR_BAD_FORMAT || st == BANDSOLVE_ERR_IO) return kIbat;
  return kSolver;
}

struct Variant {
  const char* name;
  int id;
};
const Variant kVariants[] = {{"shared", BANDSOLVE_VARIANT_SHARED},
                             {"persystem", BANDSOLVE_VARIANT_PER_SYSTEM},
                             {"uniform", BANDSOLVE_VARIANT_UNIFORM},
                             {"cusparse", BANDSOLVE_VARIANT_CUSPARSE}};

const char* variant_name(int id) {
  for (const Variant& v : kVariants)
    if (v.id == id) return v.name;
  return "?";
}

struct Options {
  std::string problem = "diffusion", variants = "shared,persystem";
  std::string n_list = "64,128,256", m_list = "64,256,1024";
  long steps = 1000;
  double dt = 0.0;
  int threads = 0;
  std::string out = "bench.csv";
  long dump_every = 0;
  std::string dump_prefix;
};

int usage(FILE* f) {
  std::fprintf(f,
               "usage: bandsolve_b200 bench [--problem diffusion|hyperdiffusion|both]\n"
               "         [--variants shared,persystem,uniform,cusparse] [--n LIST] [--m LIST]\n"
               "         [--steps K] [--dt X] [--threads T] [--out PATH]\n"
               "         [--dump-every D --dump-prefix P]\n"
               "       bandsolve_b200 --version\n");
  return kArgs;
}

int parse(int argc, char** argv, Options& o) {
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    if (k == "--help" || k == "-h") {
      usage(stdout);
      return -1;
    }
    if (i + 1 >= argc) {
      std::fprintf(stderr, "%s needs a value\n", k.c_str());
      return kArgs;
    }
    const std::string v = argv[++i];
    char* end = nullptr;
    if (k == "--problem") o.problem = v;
    else if (k == "--variants") o.variants = v;
    else if (k == "--n") o.n_list = v;
    else if (k == "--m") o.m_list = v;
    else if (k == "--out") o.out = v;
    else if (k == "--dump-prefix") o.dump_prefix = v;
    else if (k == "--steps" || k == "--threads" || k == "--dump-every") {
      const long x = std::strtol(v.c_str(), &end, 10);
      if (end == v.c_str() || *end) {
        std::fprintf(stderr, "%s: not an integer: %s\n", k.c_str(), v.c_str());
        return kArgs;
      }
      if (k == "--steps") o.steps = x;
      else if (k == "--threads") o.threads = static_cast<int>(x);
      else o.dump_every = x;
    } else if (k == "--dt") {
      o.dt = std::strtod(v.c_str(), &end);
      if (end == v.c_str() || *end) {
        std::fprintf(stderr, "--dt: not a number: %s\n", v.c_str());
        return kArgs;
      }
    } else {
      std::fprintf(stderr, "unknown option %s\n", k.c_str());
      return kArgs;
    }
  }
  return kOk;
}

int bench(const Options& o) {
  std::vector<int> problems;
  if (o.problem == "diffusion" || o.problem == "both") problems.push_back(BANDSOLVE_PROBLEM_DIFFUSION);
  if (o.problem == "hyperdiffusion" || o.problem == "both") problems.push_back(BANDSOLVE_PROBLEM_HYPERDIFFUSION);
  if (problems.empty()) {
    std::fprintf(stderr, "unknown problem '%s'\n", o.problem.c_str());
    return kArgs;
  }
  std::vector<int> variants;
  for (const std::string& tok : split(o.variants)) {
    int id = -1;
    for (const Variant& v : kVariants)
      if (tok == v.name) id = v.id;
    if (id < 0) {
      std::fprintf(stderr, "unknown variant '%s'\n", tok.c_str());
      return kArgs;
    }
    variants.push_back(id);
  }
  auto has = [&](int id) {
    for (int v : variants)
      if (v == id) return true;
    return false;
  };
  if (has(BANDSOLVE_VARIANT_UNIFORM) && problems.front() == BANDSOLVE_PROBLEM_DIFFUSION) {
    std::fprintf(stderr, "the uniform variant applies to hyperdiffusion only\n");
    return kArgs;
  }
  std::vector<size_t> ns, ms;
  if (!sizes(o.n_list, ns) || !sizes(o.m_list, ms)) {
    std::fprintf(stderr, "bad --n/--m list\n");
    return kArgs;
  }
  if (o.steps < 1) {
    std::fprintf(stderr, "--steps must be >= 1\n");
    return kArgs;
  }
  if (o.threads > 0) bandsolve_set_threads(o.threads);

  std::string csv = "problem,variant,n,m,steps,threads,wall_s,per_step_mean_s,per_step_std_s,elements\n";
  // (problem, n, m) -> variant -> mean seconds per step
  std::map<std::string, std::map<int, double>> means;
  char line[384];
  for (int problem : problems) {
    const char* pname = problem == BANDSOLVE_PROBLEM_DIFFUSION ? "diffusion" : "hyperdiffusion";
    for (int variant : variants)
      for (size_t n : ns)
        for (size_t m : ms) {
          bandsolve_bench_params p{};
          p.n = n;
          p.m = m;
          p.steps = o.steps;
          p.dt = o.dt;
          p.problem = problem;
          p.variant = variant;
          p.dump_every = o.dump_every;
          p.dump_prefix = o.dump_prefix.empty() ? nullptr : o.dump_prefix.c_str();
          bandsolve_bench_result r{};
          const bandsolve_status st = bandsolve_bench_run(&p, &r);
          if (st != BANDSOLVE_OK) {
            std::fprintf(stderr, "bench cell %s/%s n=%zu m=%zu failed: %s (%s)\n", pname, variant_name(variant), n, m,
                         bandsolve_status_string(st), bandsolve_last_error());
            return exit_for(st);
          }
          std::snprintf(line, sizeof line, "%s,%s,%zu,%zu,%ld,%d,%.9e,%.9e,%.9e,%llu\n", pname,
                        variant_name(variant), n, m, r.steps, r.threads, r.wall_s, r.per_step_mean_s, r.per_step_std_s,
                        static_cast<unsigned long long>(r.elements));
          csv += line;
          std::snprintf(line, sizeof line, "%s,%zu,%zu", pname, n, m);
          means[line][variant] = r.per_step_mean_s;
        }
  }
  if (!write_file(o.out, csv)) {
    std::fprintf(stderr, "cannot write %s\n", o.out.c_str());
    return kSolver;
  }
  // companion tables: base variant's time / each other variant's, per cell
  auto table = [&](int base, const char* column, const char* tag) -> bool {
    if (!has(base) || variants.size() < 2) return true;
    std::string t = std::string("problem,n,m,variant,") + column + "\n";
    for (int problem : problems) {
      const char* pname = problem == BANDSOLVE_PROBLEM_DIFFUSION ? "diffusion" : "hyperdiffusion";
      for (size_t n : ns)
        for (size_t m : ms) {
          std::snprintf(line, sizeof line, "%s,%zu,%zu", pname, n, m);
          const auto& cell = means[line];
          const auto b = cell.find(base);
          if (b == cell.end()) continue;
          for (int v : variants) {
            const auto it = cell.find(v);
            if (v == base || it == cell.end()) continue;
            char row[192];
            std::snprintf(row, sizeof row, "%s,%zu,%zu,%s,%.6f\n", pname, n, m, variant_name(v),
                          b->second / it->second);
            t += row;
          }
        }
    }
    const std::string path = companion(o.out, tag);
    if (write_file(path, t)) return true;
    std::fprintf(stderr, "cannot write %s\n", path.c_str());
    return false;
  };
  if (!table(BANDSOLVE_VARIANT_PER_SYSTEM, "speedup_vs_persystem", "speedup")) return kSolver;
  if (!table(BANDSOLVE_VARIANT_CUSPARSE, "speedup_vs_cusparse", "speedup_cusparse")) return kSolver;
  return kOk;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage(stderr);
  const std::string cmd = argv[1];
  if (cmd == "--version") {
    std::printf("%s\n", bandsolve_version());
    return kOk;
  }
  if (cmd == "--help" || cmd == "-h") {
    usage(stdout);
    return kOk;
  }
  if (cmd != "bench") {
    std::fprintf(stderr, "unknown command '%s' (this tool carries the bench command)\n", cmd.c_str());
    return kArgs;
  }
  Options o;
  const int rc = parse(argc, argv, o);
  if (rc < 0) return kOk;
  if (rc != kOk) return rc;
  return bench(o);
}
