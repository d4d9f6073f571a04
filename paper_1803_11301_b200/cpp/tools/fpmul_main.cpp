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

// `bench`: one CSV row per size 2^k words of padded product (k = min_log .. max_log), columns as the
// reference's schema (fpmul_main.cpp:105-106).  mean_s is the host-measured mean of `reps` calls of
// fp_polymul (host buffers in, product out); the stage columns are the GPU's own per-stage times
// (CUDA events inside the pipeline, summed by StageSeconds) divided by reps.  Before timing, every
// size's operands are checked once against karatsuba_mul -- the word-level carry-less product, an
// algorithm independent of the FFT pipeline -- on a prefix of at most 2^20 bits, so the check runs
// at every size and cannot be skipped.
struct BenchSpec {
  uint64_t lo = 0, hi = 0, reps = 100, seed = 1;
  bool have_lo = false, have_hi = false;
  fpmul::FieldChoice field = fpmul::FieldChoice::kAuto;
  std::string csv;
};

bool read_bench_spec(const Args& a, BenchSpec& b, std::string& why) {
  for (const auto& [k, v] : a.opts) {
    bool ok = true;
    if (k == "--min-log") b.have_lo = ok = parse_uint(v, b.lo);
    else if (k == "--max-log") b.have_hi = ok = parse_uint(v, b.hi);
    else if (k == "--reps") ok = parse_uint(v, b.reps);
    else if (k == "--seed") ok = parse_uint(v, b.seed);
    else if (k == "--csv") b.csv = v;
    else if (k == "--field") ok = parse_field(v, b.field);
    else ok = false;
    if (!ok) {
      why = "bad or unknown bench option " + k;
      return false;
    }
  }
  if (!b.have_lo || !b.have_hi) why = "bench needs --min-log and --max-log";
  else if (b.hi < b.lo) why = "--max-log is below --min-log";
  else if (b.reps < 3) why = "--reps must be at least 3";
  else if (b.hi > 27) why = "--max-log above 27 (2^33-bit products) is not supported";
  return why.empty();
}

fpmul::BitPoly prefix(const fpmul::BitPoly& p, size_t bits) {
  fpmul::BitPoly q = p;
  q.resize_bits(std::min(bits, p.bit_length()));
  return q;
}

int cmd_bench(const Args& a) {
  BenchSpec spec;
  std::string why;
  if (!read_bench_spec(a, spec, why)) return usage(why);
  std::ofstream file;
  if (!spec.csv.empty()) {
    file.open(spec.csv);
    if (!file) return usage("--csv: '" + spec.csv + "' is not writable");
  }
  std::ostream& csv = spec.csv.empty() ? std::cout : file;
  csv << "log2_size_words,n_bits,m,reps,mean_s,basiscvt_s,encode_s,butterfly_s,pointwise_s,"
         "ibutterfly_s,decode_s,ibasiscvt_s\n";
  std::mt19937_64 gen(spec.seed);
  for (uint64_t k = spec.lo; k <= spec.hi; ++k) {
    const size_t product_bits = size_t{64} << k;
    const size_t operand_bits = product_bits / 2;
    fpmul::MulPlan plan;
    try {
      plan = fpmul::plan_mul(operand_bits, operand_bits, spec.field);
    } catch (const std::exception& e) {
      return usage(std::string("size 2^") + std::to_string(k) + " words: " + e.what());
    }
    const fpmul::BitPoly x = fpmul::random_bitpoly(operand_bits, gen);
    const fpmul::BitPoly y = fpmul::random_bitpoly(operand_bits, gen);
    fpmul::MulOptions opts;
    opts.field = spec.field;
    {  // independent cross-check (karatsuba_mul shares no code with the FFT pipeline)
      const size_t cut = std::min<size_t>(operand_bits, size_t{1} << 20);
      const fpmul::BitPoly xs = prefix(x, cut), ys = prefix(y, cut);
      if (!(fpmul::fp_polymul(xs, ys, opts) == fpmul::karatsuba_mul(xs, ys))) {
        std::cerr << "verification FAILED at 2^" << k << " words: fp_polymul differs from karatsuba_mul\n";
        return kExitVerifyFailure;
      }
    }
    fpmul::StageSeconds gpu_stages{};
    opts.stage_seconds = &gpu_stages;
    std::vector<double> wall;
    wall.reserve(spec.reps);
    fpmul::BitPoly last;
    for (uint64_t r = 0; r < spec.reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      last = fpmul::fp_polymul(x, y, opts);
      wall.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    double sum = 0;
    for (double w : wall) sum += w;
    const double per = 1.0 / static_cast<double>(spec.reps);
    const double cols[7] = {gpu_stages.basiscvt, gpu_stages.encode, gpu_stages.butterfly, gpu_stages.pointwise,
                            gpu_stages.ibutterfly, gpu_stages.decode, gpu_stages.ibasiscvt};
    csv << k << ',' << product_bits << ',' << plan.field_degree << ',' << spec.reps << ',';
    csv.setf(std::ios::fixed);
    csv.precision(9);
    csv << sum * per;
    for (double c : cols) csv << ',' << c * per;
    csv.unsetf(std::ios::fixed);
    csv << '\n' << std::flush;
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
