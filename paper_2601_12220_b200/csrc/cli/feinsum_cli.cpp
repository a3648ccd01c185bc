// feinsum — command-line front end of the B200 build.
//
// Same subcommands, options, output bytes and exit codes as the reference
// CLI (/root/reference/proj/tools/feinsum.cpp:52-245, goldens in
// proj/tests/test_cli.cpp), written against the drop-in C++ API
// (include/feinsum/*.hpp, implemented by libfeinsum_b200.so) with its own
// argument parser (the reference uses CLI11, which is not vendored). One
// subcommand is new: `tune` measures a plan's tuned transform on the GPU under
// candidate parameter sets and records each as a fact (device "b200"), the
// tuning loop of SURVEY.md §8(f) item 1.
//
// Exit codes: 0 ok, 1 domain error (malformed input), 2 usage, 3 io.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "feinsum/canonicalize.hpp"
#include "feinsum/factsdb.hpp"
#include "feinsum/notation.hpp"
#include "feinsum/raising.hpp"
#include "feinsum_b200.h"

namespace {

using namespace feinsum;

// ------------------------------------------------------------ arguments --

struct UsageError {
  std::string msg;
};

struct OptSpec {
  std::string name;  // without the leading --
  bool required = false;
};

// Parsed command line of one subcommand: positionals in order, --name value
// (or --name=value) options. Unknown options, missing required ones and extra
// positionals are usage errors (exit 2), as CLI11 reports them.
struct Args {
  std::vector<std::string> pos;
  std::map<std::string, std::string> opt;
  bool help = false;

  static Args parse(int argc, char** argv, int first, const std::vector<std::string>& positionals, int required_pos,
                    const std::vector<OptSpec>& opts) {
    Args a;
    for (int i = first; i < argc; ++i) {
      std::string t = argv[i];
      if (t == "-h" || t == "--help") {
        a.help = true;
        continue;
      }
      if (t.size() > 2 && t.compare(0, 2, "--") == 0) {
        std::string name = t.substr(2), val;
        bool inline_val = false;
        if (auto eq = name.find('='); eq != std::string::npos) {
          val = name.substr(eq + 1);
          name = name.substr(0, eq);
          inline_val = true;
        }
        bool known = false;
        for (const auto& o : opts) known = known || o.name == name;
        if (!known) throw UsageError{"The following argument was not expected: " + t};
        if (!inline_val) {
          if (i + 1 >= argc) throw UsageError{"--" + name + ": 1 required argument missing"};
          val = argv[++i];
        }
        a.opt[name] = val;
        continue;
      }
      if (a.pos.size() >= positionals.size()) throw UsageError{"The following argument was not expected: " + t};
      a.pos.push_back(t);
    }
    if (a.help) return a;
    if (static_cast<int>(a.pos.size()) < required_pos)
      throw UsageError{positionals[a.pos.size()] + " is required"};
    for (const auto& o : opts)
      if (o.required && !a.opt.count(o.name)) throw UsageError{"--" + o.name + " is required"};
    return a;
  }
  std::string get(const std::string& k, const std::string& dflt) const {
    auto it = opt.find(k);
    return it == opt.end() ? dflt : it->second;
  }
  double num(const std::string& k, double dflt) const {
    auto it = opt.find(k);
    if (it == opt.end()) return dflt;
    char* end = nullptr;
    const double v = std::strtod(it->second.c_str(), &end);
    if (end == it->second.c_str() || *end) throw UsageError{"--" + k + ": Value " + it->second + " could not be converted"};
    return v;
  }
  std::int64_t integer(const std::string& k, std::int64_t dflt) const {
    auto it = opt.find(k);
    if (it == opt.end()) return dflt;
    char* end = nullptr;
    const long long v = std::strtoll(it->second.c_str(), &end, 10);
    if (end == it->second.c_str() || *end) throw UsageError{"--" + k + ": Value " + it->second + " could not be converted"};
    return v;
  }
};

const char* kUsage =
    "canonicalize batched einsums and keep tuning facts about them\n"
    "Usage: feinsum SUBCOMMAND [OPTIONS]\n\n"
    "Subcommands:\n"
    "  canonicalize FILE [--format text|key-only]   print the canonical form of an einsum file\n"
    "  isomorphic FIRST SECOND                      decide whether two einsum files agree\n"
    "  match KERNEL REFERENCE                       match a kernel file against a reference einsum\n"
    "  record FILE --device D --wall S [--db P] [--transform T] [--rate R] [--meta M]\n"
    "                                               store a tuning fact for an einsum\n"
    "  retrieve FILE --device D [--db P]            look up the best known fact for an einsum\n"
    "  stats FILE [--device D]                      cost model numbers for an einsum\n"
    "  tune FILE [--db P] [--candidates M1,M2,...] [--reps N] [--warmup N]\n"
    "                                               time the tuned transform on this GPU and record facts\n";

// --------------------------------------------------------------- output --

std::string slurp(const std::string& path) {
  if (path == "-") {
    std::ostringstream ss;
    ss << std::cin.rdbuf();
    return ss.str();
  }
  std::ifstream in(path, std::ios::binary);
  if (!in) throw error(errc::io, "cannot read " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

std::string num(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

void print_map(const char* label, const std::map<std::string, std::string>& m) {
  std::cout << label << ":";
  bool first = true;
  for (const auto& [k, v] : m) {
    std::cout << (first ? " " : ", ") << k << " -> " << v;
    first = false;
  }
  std::cout << "\n";
}

void print_perm(const char* label, const std::vector<int>& p) {
  std::cout << label << ":";
  for (size_t i = 0; i < p.size(); ++i) std::cout << (i ? ", " : " ") << (i + 1) << " -> " << (p[i] + 1);
  std::cout << "\n";
}

// ---------------------------------------------------------- subcommands --

int run_canonicalize(const std::string& file, const std::string& format) {
  BatchedEinsum e = parse_classic(slurp(file));
  CanonResult c = canonicalize(e);
  const std::string key = canonical_key(c.canonical);
  if (format == "key-only") {
    std::cout << key << "\n";
    return 0;
  }
  std::cout << print_classic(c.canonical);
  std::cout << "key: " << key << "\n";
  print_perm("rows (canonical -> input)", c.sigma_row);
  print_perm("slots (canonical -> input)", c.sigma_slot);
  print_map("indices (canonical -> input)", c.sigma_idx);
  print_map("arrays (canonical -> input)", c.sigma_arg);
  return 0;
}

int run_isomorphic(const std::string& f1, const std::string& f2) {
  BatchedEinsum e1 = parse_classic(slurp(f1));
  BatchedEinsum e2 = parse_classic(slurp(f2));
  std::optional<SubstitutionWitness> w = is_isomorphic(e1, e2);
  if (!w) {
    std::cout << "not isomorphic\n";
    return 0;
  }
  std::cout << "isomorphic\n";
  print_perm("rows (first -> second)", w->sigma_row);
  print_perm("slots (first -> second)", w->sigma_slot);
  print_map("indices (second -> first)", w->sigma_idx);
  print_map("arrays (second -> first)", w->sigma_arg);
  return 0;
}

int run_match(const std::string& kfile, const std::string& rfile) {
  FunctionalKernel k = parse_kernel(slurp(kfile));
  BatchedEinsum ref = parse_classic(slurp(rfile));
  MatchResult m = identify_as_einsum(k, ref);
  std::cout << "match\n";
  std::cout << "rows (reference -> statement):";
  for (size_t i = 0; i < m.sigma_row.size(); ++i) std::cout << (i ? ", " : " ") << (i + 1) << " -> " << (m.sigma_row[i] + 1);
  std::cout << "\n";
  print_map("indices (reference -> kernel)", m.sigma_idx);
  print_map("arrays (reference -> kernel)", m.sigma_arg);
  return 0;
}

int run_record(const std::string& file, const Args& a) {
  BatchedEinsum e = parse_classic(slurp(file));
  CanonResult c = canonicalize(e);
  FactRecord r;
  r.canonical_key = canonical_key(c.canonical);
  r.device_id = a.get("device", "");
  r.transform_id = a.get("transform", "baseline");
  r.wall_time_s = a.num("wall", 0.0);
  const double rate = a.num("rate", 0.0);
  r.flop_rate = rate > 0.0 ? rate : flop_count(e) / r.wall_time_s;
  r.meta = a.get("meta", "");
  record_facts(a.get("db", "./feinsum-facts.db"), {r});
  std::cout << "recorded " << r.canonical_key << "\n";
  return 0;
}

int run_retrieve(const std::string& file, const Args& a) {
  BatchedEinsum e = parse_classic(slurp(file));
  const std::string key = canonical_key(canonicalize(e).canonical);
  const std::string device = a.get("device", "");
  std::optional<FactRecord> r = retrieve(a.get("db", "./feinsum-facts.db"), key, device);
  if (!r) {
    std::cout << "no facts for this einsum on " << device << "\n";
    return 0;
  }
  std::cout << "key: " << r->canonical_key << "\n";
  std::cout << "transform: " << r->transform_id << "\n";
  std::cout << "wall_time_s: " << num(r->wall_time_s) << "\n";
  std::cout << "flop_rate: " << num(r->flop_rate) << "\n";
  std::cout << "recorded_at: " << r->recorded_at << "\n";
  if (!r->meta.empty()) std::cout << "meta: " << r->meta << "\n";
  return 0;
}

int run_stats(const std::string& file, const std::string& device) {
  BatchedEinsum e = parse_classic(slurp(file));
  std::cout << "flops: " << num(flop_count(e)) << "\n";
  std::cout << "bytes: " << num(footprint_bytes(e)) << "\n";
  std::cout << "intensity: " << num(arithmetic_intensity(e)) << "\n";
  std::vector<DeviceModel> devs;
  if (!device.empty()) {
    std::optional<DeviceModel> d = device_preset(device);
    if (!d) throw error(errc::usage, "unknown device " + device + " (have: mi250x h100 titanv p100)");
    devs.push_back(*d);
  } else {
    devs = device_presets();
  }
  for (const DeviceModel& d : devs)
    std::cout << "device " << d.id << ": roofline " << num(roofline_flop_rate(e, d)) << ", "
              << (memory_bound(e, d) ? "memory bound" : "compute bound") << "\n";
  return 0;
}

int run_fuzz(std::uint64_t seed, int count) {
  GenParams p;
  for (int t = 0; t < count; ++t) {
    const std::uint64_t s = seed + 1000003ull * static_cast<std::uint64_t>(t);
    BatchedEinsum e = generate_random(p, s);
    Scrambled sc = scramble(e, s ^ 0x9e3779b97f4a7c15ull);
    auto bad = [&](const std::string& what) {
      std::cout << "fuzz case " << t << " (seed " << s << "): " << what << "\n";
      std::cout << "--- original ---\n" << print_classic(e);
      std::cout << "--- scrambled ---\n" << print_classic(sc.e);
      return 1;
    };
    if (!verify_witness(sc.e, e, sc.w)) return bad("scramble witness does not check out");
    CanonResult c1 = canonicalize(e);
    CanonResult c2 = canonicalize(sc.e);
    if (!equals(c1.canonical, c2.canonical)) return bad("canonical forms differ");
    if (!verify_witness(e, c1.canonical, canonical_witness(c1))) return bad("canonicalization witness does not check out");
    if (!equals(canonicalize(c1.canonical).canonical, c1.canonical)) return bad("canonicalize is not idempotent");
  }
  std::cout << "ok: " << count << " cases\n";
  return 0;
}

// ------------------------------------------------------------------ tune --

std::string take_json_string(const std::string& js, const std::string& field) {
  const std::string pat = "\"" + field + "\":\"";
  const auto at = js.find(pat);
  if (at == std::string::npos) return "";
  std::string out;
  for (size_t i = at + pat.size(); i < js.size() && js[i] != '"'; ++i) {
    if (js[i] == '\\' && i + 1 < js.size()) ++i;
    out += js[i];
  }
  return out;
}

double take_json_number(const std::string& js, const std::string& field) {
  const std::string pat = "\"" + field + "\":";
  const auto at = js.find(pat);
  return at == std::string::npos ? 0.0 : std::strtod(js.c_str() + at + pat.size(), nullptr);
}

std::string json_quote(const std::string& s) {
  std::string o = "\"";
  for (char ch : s) {
    if (ch == '"' || ch == '\\') o += '\\';
    o += ch;
  }
  return o + "\"";
}

// default candidates per transform family (fact meta strings; "" = defaults)
std::vector<std::string> default_candidates(const std::string& transform) {
  if (transform == "fem_grad/v1")
    return {"stages=4", "stages=4;te=16", "stages=3;ept=2", "stages=4;ept=2", "stages=3;ept=2;te=64"};
  if (transform == "gett_dmma/v1") return {"stages=2;group=6", "stages=2;group=12", "stages=3;group=12"};
  if (transform == "hex_sumfact/v1") return {"", "v=3", "ne=2", "v=1"};
  if (transform == "tt/v1") return {"", "tc=1"};
  return {""};
}

int run_tune(const std::string& file, const Args& a) {
  const std::string text = slurp(file);
  const bool is_kernel = text.find("stmt ") != std::string::npos;
  BatchedEinsum e = is_kernel ? BatchedEinsum{} : parse_classic(text);
  const std::string db = a.get("db", "./feinsum-facts.db");
  const int reps = static_cast<int>(a.integer("reps", 5));
  const int warmup = static_cast<int>(a.integer("warmup", 2));
  if (fe_device_check() != FE_OK) throw error(errc::io, fe_last_error());

  char* ejs = nullptr;
  if (!is_kernel && fe_parse_classic(text.c_str(), &ejs) != FE_OK) throw error(errc::domain, fe_last_error());
  const std::string einsum_json = ejs ? ejs : "";
  fe_free(ejs);
  auto make = [&](const std::string& options) {
    fe_plan_t plan = nullptr;
    const int st = is_kernel ? fe_plan_create_kernel(text.c_str(), options.c_str(), &plan)
                             : fe_plan_create(einsum_json.c_str(), options.c_str(), &plan);
    if (st != FE_OK) throw error(st == FE_ERR_USAGE ? errc::usage : errc::domain, fe_last_error());
    return plan;
  };
  fe_plan_t base = make("{}");
  char* desc = nullptr;
  fe_plan_describe(base, &desc);
  const std::string info = desc ? desc : "";
  fe_free(desc);
  fe_plan_destroy(base);
  const std::string key = take_json_string(info, "key");
  const std::string transform = take_json_string(info, "transform");
  const double flops = take_json_number(info, "algorithmic_flops");

  std::vector<std::string> cands;
  if (a.opt.count("candidates")) {
    // comma-separated meta strings; empty items mean "defaults" (",," = three)
    const std::string list = a.get("candidates", "");
    size_t from = 0;
    for (;;) {
      const size_t comma = list.find(',', from);
      cands.push_back(list.substr(from, comma == std::string::npos ? std::string::npos : comma - from));
      if (comma == std::string::npos) break;
      from = comma + 1;
    }
  } else {
    cands = default_candidates(transform);
  }
  std::vector<FactRecord> facts;
  std::cout << "key: " << key << "\ntransform: " << transform << "\n";
  for (const std::string& meta : cands) {
    std::string options = "{\"transform\":" + json_quote(transform);
    if (!meta.empty()) options += ",\"meta\":" + json_quote(meta);
    options += "}";
    fe_plan_t plan = make(options);
    double sec = 0.0;
    const int st = fe_plan_time(plan, reps, warmup, 7, &sec);
    fe_plan_destroy(plan);
    if (st != FE_OK) throw error(errc::io, fe_last_error());
    FactRecord r;
    r.canonical_key = key;
    // reduced-precision variants (3xTF32 tensor cores: ~1e-5 against double,
    // above the fp32 bar on some data) are a separate precision class: they
    // are retrieved only by plans created with device "b200-tf32"
    r.device_id = meta.find("tc=1") != std::string::npos ? "b200-tf32" : "b200";
    r.transform_id = transform;
    r.wall_time_s = sec;
    r.flop_rate = sec > 0.0 ? flops / sec : 0.0;
    r.meta = meta;
    facts.push_back(r);
    std::cout << "candidate " << (meta.empty() ? "(defaults)" : meta) << ": " << num(sec) << " s\n";
  }
  record_facts(db, facts);
  std::cout << "recorded " << facts.size() << " facts in " << db << "\n";
  return 0;
}

int dispatch(int argc, char** argv) {
  if (argc < 2) throw UsageError{"A subcommand is required"};
  const std::string sub = argv[1];
  if (sub == "-h" || sub == "--help") {
    std::cout << kUsage;
    return 0;
  }
  auto help = [](const Args& a) {
    if (a.help) std::cout << kUsage;
    return a.help;
  };
  if (sub == "canonicalize") {
    Args a = Args::parse(argc, argv, 2, {"file"}, 1, {{"format"}});
    if (help(a)) return 0;
    const std::string fmt = a.get("format", "text");
    if (fmt != "text" && fmt != "key-only") throw UsageError{"--format: " + fmt + " not in {text,key-only}"};
    return run_canonicalize(a.pos[0], fmt);
  }
  if (sub == "isomorphic") {
    Args a = Args::parse(argc, argv, 2, {"first", "second"}, 2, {});
    if (help(a)) return 0;
    return run_isomorphic(a.pos[0], a.pos[1]);
  }
  if (sub == "match") {
    Args a = Args::parse(argc, argv, 2, {"kernel", "reference"}, 2, {});
    if (help(a)) return 0;
    return run_match(a.pos[0], a.pos[1]);
  }
  if (sub == "record") {
    Args a = Args::parse(argc, argv, 2, {"file"}, 1,
                         {{"db"}, {"device", true}, {"transform"}, {"wall", true}, {"rate"}, {"meta"}});
    if (help(a)) return 0;
    return run_record(a.pos[0], a);
  }
  if (sub == "retrieve") {
    Args a = Args::parse(argc, argv, 2, {"file"}, 1, {{"db"}, {"device", true}});
    if (help(a)) return 0;
    return run_retrieve(a.pos[0], a);
  }
  if (sub == "stats") {
    Args a = Args::parse(argc, argv, 2, {"file"}, 1, {{"device"}});
    if (help(a)) return 0;
    return run_stats(a.pos[0], a.get("device", ""));
  }
  if (sub == "fuzz") {
    Args a = Args::parse(argc, argv, 2, {}, 0, {{"seed"}, {"count"}});
    if (help(a)) return 0;
    return run_fuzz(static_cast<std::uint64_t>(a.integer("seed", 1)), static_cast<int>(a.integer("count", 100)));
  }
  if (sub == "tune") {
    Args a = Args::parse(argc, argv, 2, {"file"}, 1, {{"db"}, {"candidates"}, {"reps"}, {"warmup"}});
    if (help(a)) return 0;
    return run_tune(a.pos[0], a);
  }
  throw UsageError{"The following argument was not expected: " + sub};
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return dispatch(argc, argv);
  } catch (const UsageError& e) {
    std::cerr << e.msg << "\nRun with --help for more information.\n";
    return 2;
  } catch (const feinsum::error& e) {
    std::cerr << "error: " << e.what() << "\n";
    switch (e.kind()) {
      case feinsum::errc::usage: return 2;
      case feinsum::errc::io: return 3;
      default: return 1;
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
