// fpmul_main.cpp -- the `fpmul` command line of the reference (proj/tools/fpmul_main.cpp:
// mul / selftest / bench subcommands, exit codes 0 ok, 1 verification failure, 2 usage or I/O
// error, CSV schema of `bench`) on the B200 backend.  A small hand-written argument parser stands in
// for the reference's vendored CLI11.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "fpmul/io.hpp"
#include "fpmul/polymul.hpp"
#include "fpmul/selftest.hpp"

namespace {

constexpr int kExitOk = 0;
constexpr int kExitVerifyFailure = 1;
constexpr int kExitUsage = 2;

int usage(const std::string& msg) {
  if (!msg.empty()) std::cerr << "error: " << msg << "\n";
  std::cerr << "usage: fpmul_b200 mul IN_A IN_B OUT [--field auto|64|128]\n"
               "       fpmul_b200 selftest [--level quick|full] [--seed N] [--inject-encode-fault]\n"
               "       fpmul_b200 bench --min-log A --max-log B [--reps N] [--csv PATH] [--field auto|64|128]"
               " [--seed N]\n";
  return kExitUsage;
}

struct Args {
  std::vector<std::string> positional;
  std::map<std::string, std::string> opts;
  std::vector<std::string> flags;
};

// "--name value" options (value required) and bare "--flag"s from the given flag list.
bool parse(int argc, char** argv, int first, const std::vector<std::string>& flag_names, Args& out, std::string& err) {
  for (int i = first; i < argc; ++i) {
    const std::string a = argv[i];
    if (a.rfind("--", 0) == 0) {
      bool is_flag = false;
      for (const auto& f : flag_names) is_flag |= (a == f);
      if (is_flag) {
        out.flags.push_back(a);
      } else if (i + 1 < argc) {
        out.opts[a] = argv[++i];
      } else {
        err = "option " + a + " needs a value";
        return false;
      }
    } else {
      out.positional.push_back(a);
    }
  }
  return true;
}

bool parse_field(const std::string& s, fpmul::FieldChoice& f) {
  if (s == "auto") f = fpmul::FieldChoice::kAuto;
  else if (s == "64") f = fpmul::FieldChoice::kGF64;
  else if (s == "128") f = fpmul::FieldChoice::kGF128;
  else return false;
  return true;
}

bool parse_uint(const std::string& s, uint64_t& v) {
  if (s.empty()) return false;
  char* end = nullptr;
  v = std::strtoull(s.c_str(), &end, 10);
  return end && *end == 0;
}

int cmd_mul(const Args& a) {
  if (a.positional.size() != 3) return usage("mul needs IN_A IN_B OUT");
  fpmul::MulOptions opts;
  for (const auto& [k, v] : a.opts) {
    if (k == "--field") {
      if (!parse_field(v, opts.field)) return usage("--field must be auto, 64 or 128");
    } else {
      return usage("unknown option " + k);
    }
  }
  try {
    const fpmul::BitPoly x = fpmul::load_polynomial(a.positional[0]);
    const fpmul::BitPoly y = fpmul::load_polynomial(a.positional[1]);
    const fpmul::BitPoly c = fpmul::fp_polymul(x, y, opts);
    fpmul::store_polynomial(a.positional[2], c);
    std::cout << "product bit length: " << c.max_degree_plus_one() << "\n";
    return kExitOk;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  }
}

int cmd_selftest(const Args& a) {
  fpmul::SelftestOptions opts;
  for (const auto& [k, v] : a.opts) {
    uint64_t n = 0;
    if (k == "--level" && (v == "quick" || v == "full")) opts.level = v == "full" ? fpmul::SelftestLevel::kFull : fpmul::SelftestLevel::kQuick;
    else if (k == "--seed" && parse_uint(v, n)) opts.seed = n;
    else return usage("bad selftest option " + k + " " + v);
  }
  for (const auto& f : a.flags)
    if (f == "--inject-encode-fault") opts.corrupt_encode_matrix = true;
  if (!a.positional.empty()) return usage("selftest takes no positional arguments");
  const auto report = fpmul::run_selftest(opts, std::cout);
  if (!report.ok) {
    std::cerr << "selftest FAILED; failing invariants:\n";
    for (const auto& name : report.failed_invariants) std::cerr << "  " << name << "\n";
    return kExitVerifyFailure;
  }
  std::cout << "selftest passed\n";
  return kExitOk;
}

int cmd_bench(const Args& a) {
  uint64_t min_log = 0, max_log = 0, reps = 100, seed = 1;
  bool have_min = false, have_max = false;
  std::string csv_path, field = "auto";
  for (const auto& [k, v] : a.opts) {
    bool ok = true;
    if (k == "--min-log") ok = have_min = parse_uint(v, min_log);
    else if (k == "--max-log") ok = have_max = parse_uint(v, max_log);
    else if (k == "--reps") ok = parse_uint(v, reps);
    else if (k == "--seed") ok = parse_uint(v, seed);
    else if (k == "--csv") csv_path = v;
    else if (k == "--field") field = v;
    else return usage("unknown option " + k);
    if (!ok) return usage("bad value for " + k);
  }
  fpmul::FieldChoice fc;
  if (!have_min || !have_max) return usage("bench needs --min-log and --max-log");
  if (!parse_field(field, fc)) return usage("--field must be auto, 64 or 128");
  if (min_log > max_log || reps < 3) {
    std::cerr << "error: need min-log <= max-log and reps >= 3\n";
    return kExitUsage;
  }
  std::ostream* out = &std::cout;
  std::ofstream file;
  if (!csv_path.empty()) {
    file.open(csv_path);
    if (!file) {
      std::cerr << "error: cannot open '" << csv_path << "'\n";
      return kExitUsage;
    }
    out = &file;
  }
  // same columns as the reference (fpmul_main.cpp bench): sizes, mean wall time, stage seconds
  *out << "log2_size_words,n_bits,m,reps,mean_s,basiscvt_s,encode_s,butterfly_s,pointwise_s,"
          "ibutterfly_s,decode_s,ibasiscvt_s\n";
  std::mt19937_64 rng(seed);
  for (uint64_t lg = min_log; lg <= max_log; ++lg) {
    const size_t n_bits = size_t{64} << lg;  // padded product length
    fpmul::MulOptions opts;
    opts.field = fc;
    fpmul::StageSeconds stages;
    opts.stage_seconds = &stages;
    fpmul::MulPlan plan;
    try {
      plan = fpmul::plan_mul(n_bits / 2, n_bits / 2, opts.field);
    } catch (const std::exception& e) {
      std::cerr << "error: " << e.what() << "\n";
      return kExitUsage;
    }
    const fpmul::BitPoly x = fpmul::random_bitpoly(n_bits / 2, rng);
    const fpmul::BitPoly y = fpmul::random_bitpoly(n_bits / 2, rng);
    if (lg == min_log) {  // verification hook: an independent transform (the other field) agrees
      fpmul::MulOptions o64, o128;
      o64.field = fpmul::FieldChoice::kGF64;
      o128.field = fpmul::FieldChoice::kGF128;
      bool same = true;
      try {
        same = fpmul::fp_polymul(x, y, o64) == fpmul::fp_polymul(x, y, o128);
      } catch (const std::invalid_argument&) {  // size beyond GF(2^64): compare with itself skipped
      }
      if (!same) {
        std::cerr << "verification FAILED at log2(n/64)=" << lg << ": GF(2^64) and GF(2^128) products differ\n";
        return kExitVerifyFailure;
      }
    }
    stages = fpmul::StageSeconds{};
    double total = 0;
    fpmul::BitPoly sink;
    for (uint64_t r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      sink = fpmul::fp_polymul(x, y, opts);
      total += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    const double inv = 1.0 / static_cast<double>(reps);
    char line[512];
    std::snprintf(line, sizeof line, "%u,%zu,%u,%u,%.9f,%.9f,%.9f,%.9f,%.9f,%.9f,%.9f,%.9f\n",
                  static_cast<unsigned>(lg), n_bits, plan.field_degree, static_cast<unsigned>(reps), total * inv,
                  stages.basiscvt * inv, stages.encode * inv, stages.butterfly * inv, stages.pointwise * inv,
                  stages.ibutterfly * inv, stages.decode * inv, stages.ibasiscvt * inv);
    *out << line << std::flush;
  }
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage("a subcommand is required");
  const std::string cmd = argv[1];
  Args a;
  std::string err;
  if (!parse(argc, argv, 2, {"--inject-encode-fault"}, a, err)) return usage(err);
  if (cmd == "mul") return cmd_mul(a);
  if (cmd == "selftest") return cmd_selftest(a);
  if (cmd == "bench") return cmd_bench(a);
  if (cmd == "--help" || cmd == "-h") {
    usage("");
    return kExitOk;
  }
  return usage("unknown subcommand '" + cmd + "'");
}
