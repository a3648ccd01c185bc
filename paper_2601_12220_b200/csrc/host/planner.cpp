// B200 planner — see planner.hpp for the pipeline. Canonicalization drives
// dispatch exactly as the paper intends: the tuned choice is stored per normal
// form (canonical key -> fact), the kernel family is matched on the canonical
// form, and the sigma maps (canonical -> caller) route the caller's buffers to
// the kernel's roles. Since canonical slot j has the same layout as caller slot
// sigma_slot[j], no data is ever transposed.
#include "planner.hpp"

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <mutex>
#include <numeric>
#include <set>
#include <sstream>

#include "feinsum/notation.hpp"
#include "json.hpp"
#include "einsum_json.hpp"  // after the feinsum headers

namespace feinsum::detail {
std::string key_of_canonical(const BatchedEinsum& e);
}

namespace feb200 {

using feinsum::errc;
using feinsum::error;
using feinsum::Expr;

namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw error(errc::io, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
void cuda_check(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }

}  // namespace

const LeafInfo& leaf_info(const Plan& p, int i) {
  const size_t n = p.leaves.size();
  return static_cast<size_t>(i) < n ? p.leaves[static_cast<size_t>(i)] : p.tab_leaves.at(static_cast<size_t>(i) - n);
}

const char* family_transform(Family f) {
  switch (f) {
    case Family::generic: return "generic/v1";
    case Family::fem_grad: return "fem_grad/v1";
    case Family::gett: return "gett_dmma/v1";
    case Family::tt: return "tt/v1";
    case Family::hex: return "hex_sumfact/v1";
    case Family::path: return "path/v1";
  }
  return "generic/v1";
}

int storage_from_name(const std::string& s) {
  static const std::map<std::string, int> m = {{"f64", ST_F64}, {"f32", ST_F32}, {"c128", ST_C128}, {"c64", ST_C64},
                                               {"i8", ST_I8},   {"i32", ST_I32}, {"i64", ST_I64},   {"f16", ST_F16}};
  auto it = m.find(s);
  if (it == m.end()) throw error(errc::usage, "unknown storage \"" + s + "\"");
  return it->second;
}

const char* storage_name(int st) {
  static const char* names[] = {"f64", "f32", "c128", "c64", "i8", "i32", "i64", "f16"};
  return (st >= 0 && st < 8) ? names[st] : "?";
}

int native_storage(Dtype t) {
  switch (t) {
    case Dtype::int8: return ST_I8;
    case Dtype::int32: return ST_I32;
    case Dtype::int64: return ST_I64;
    case Dtype::float16: return ST_F16;
    case Dtype::float32: return ST_F32;
    case Dtype::float64: return ST_F64;
    case Dtype::complex64: return ST_C64;
    case Dtype::complex128: return ST_C128;
  }
  return ST_F64;
}

namespace {
bool is_complex_dtype(Dtype t) { return t == Dtype::complex64 || t == Dtype::complex128; }
}  // namespace

std::string default_facts_path() {
  Dl_info info{};
  if (dladdr(reinterpret_cast<void*>(&default_facts_path), &info) && info.dli_fname) {
    std::string so = info.dli_fname;
    const auto slash = so.rfind('/');
    const std::string dir = slash == std::string::npos ? "." : so.substr(0, slash);
    return dir + "/../facts/b200.facts";
  }
  return "paper_2601_12220_b200/facts/b200.facts";
}

PlanOptions parse_options(const std::string& json) {
  PlanOptions o;
  if (json.empty()) return o;
  const fejson::Value v = fejson::parse(json);
  if (v.t != fejson::Value::T::object) throw error(errc::usage, "options must be a JSON object");
  if (auto* x = v.find("storage")) {
    o.storage = x->as_str();
    if (o.storage != "native" && o.storage != "wide")
      throw error(errc::usage, "options.storage must be \"native\" or \"wide\"");
  }
  if (auto* x = v.find("leaf_storage"))
    for (const auto& [name, st] : x->o) o.storage_of[name] = st.as_str();
  if (auto* x = v.find("facts")) o.facts_path = x->as_str();
  if (auto* x = v.find("device")) o.device_id = x->as_str();
  if (auto* x = v.find("transform")) o.force_transform = x->as_str();
  if (auto* x = v.find("canonicalize")) o.canonicalize = x->b;
  if (auto* x = v.find("dry_run")) o.dry_run = x->b;
  if (auto* x = v.find("meta")) o.meta_override = x->as_str();
  if (auto* x = v.find("codegen")) o.codegen = x->b;
  return o;
}

// ------------------------------------------------------------- facts index --

namespace {

// In-process index over a facts file: retrieve() semantics (least wall time,
// ties to newest recorded_at, then later row), loaded once per path/mtime.
class FactsIndex {
 public:
  std::optional<feinsum::FactRecord> best(const std::string& path, const std::string& key,
                                          const std::string& device) {
    std::lock_guard<std::mutex> lock(mu_);
    auto& entry = cache_[path];
    if (!entry.loaded) {
      entry.loaded = true;
      try {
        for (auto& r : feinsum::load_facts(path)) {
          auto& slot = entry.best[r.canonical_key + "\x1f" + r.device_id];
          const bool better = !slot || r.wall_time_s < slot->wall_time_s ||
                              (r.wall_time_s == slot->wall_time_s && r.recorded_at >= slot->recorded_at);
          if (better) slot = r;
        }
      } catch (const error&) {
        entry.best.clear();
      }
    }
    auto it = entry.best.find(key + "\x1f" + device);
    if (it == entry.best.end()) return std::nullopt;
    return it->second;
  }
  void invalidate() {
    std::lock_guard<std::mutex> lock(mu_);
    cache_.clear();
  }

 private:
  struct Entry {
    bool loaded = false;
    std::map<std::string, std::optional<feinsum::FactRecord>> best;
  };
  std::mutex mu_;
  std::map<std::string, Entry> cache_;
};

FactsIndex& facts_index() {
  static FactsIndex idx;
  return idx;
}

// ------------------------------------------------------ operand compilation --

void flatten_chain(const Expr& e, char a, char b, std::vector<std::pair<char, const Expr*>>& out) {
  // left-deep chain of a/b operators: ((t0 op t1) op t2) ...
  if (e.kind == Expr::Kind::binary && (e.op == a || e.op == b)) {
    flatten_chain(e.children[0], a, b, out);
    out.emplace_back(e.op, &e.children[1]);
    return;
  }
  out.emplace_back(0, &e);
}

bool uses_sqrt(const Expr& e) {
  if (e.kind == Expr::Kind::unary && e.name == "sqrt") return true;
  for (const Expr& c : e.children)
    if (uses_sqrt(c)) return true;
  return false;
}

struct OperandCompiler {
  Plan& plan;
  std::map<std::string, int> leaf_of;
  bool force_vm = false;
  bool skip_range_check = false;

  explicit OperandCompiler(Plan& p) : plan(p) {
    for (size_t i = 0; i < p.leaves.size(); ++i) leaf_of[p.leaves[i].meta.name] = static_cast<int>(i);
  }

  // epilogue compilation: reads of acc_name are the row's own value
  std::string acc_name;
  LeafInfo acc_info;

  const LeafInfo& leaf_checked(const std::string& name) {
    if (!acc_name.empty() && name == acc_name) return acc_info;
    auto it = leaf_of.find(name);
    if (it == leaf_of.end()) throw error(errc::domain, "no binding for array " + name);
    return plan.leaves[it->second];
  }

  int add_chain(const std::vector<CoefFactor>& f) {
    CoefChain c{};
    c.n = static_cast<int>(f.size());
    for (size_t i = 0; i < f.size(); ++i) c.f[i] = f[i];
    plan.chains.push_back(c);
    return static_cast<int>(plan.chains.size()) - 1;
  }

  // factor classification for the affine path
  enum class FK { scalar, tensor, other };
  FK classify(const Expr& f, const OperandExpr& op, const ArrayMeta& sm, CoefFactor* cf, int* leaf) {
    if (f.kind == Expr::Kind::literal) {
      *cf = CoefFactor{-1, f.literal};
      return FK::scalar;
    }
    if (f.kind != Expr::Kind::access) return FK::other;
    auto it = leaf_of.find(f.name);
    if (it == leaf_of.end()) return FK::other;
    const LeafInfo& L = plan.leaves[it->second];
    if (f.subs.empty() && L.meta.shape.empty()) {
      *cf = CoefFactor{it->second, 0.0};
      return FK::scalar;
    }
    if (f.subs == op.params && L.meta.shape == sm.shape &&
        std::set<std::string>(op.params.begin(), op.params.end()).size() == op.params.size()) {
      *leaf = it->second;
      return FK::tensor;
    }
    return FK::other;
  }

  bool try_affine(const OperandExpr& op, const ArrayMeta& sm, OperandStatic& out) {
    std::vector<std::pair<char, const Expr*>> terms;
    flatten_chain(op.body, '+', '-', terms);
    if (terms.size() > static_cast<size_t>(kMaxAffineTerms)) return false;
    OperandStatic s{};
    s.kind = OPK_AFFINE;
    s.leaf = -1;
    s.ndim = static_cast<int>(op.params.size());
    s.n_terms = static_cast<int>(terms.size());
    const size_t chains_before = plan.chains.size();
    for (size_t t = 0; t < terms.size(); ++t) {
      std::vector<std::pair<char, const Expr*>> factors;
      flatten_chain(*terms[t].second, '*', '*', factors);
      std::vector<CoefFactor> pre, post;
      int leaf = -1;
      for (const auto& [opch, fx] : factors) {
        CoefFactor cf{};
        int lf = -1;
        const FK k = classify(*fx, op, sm, &cf, &lf);
        if (k == FK::other || (k == FK::tensor && leaf >= 0)) {
          plan.chains.resize(chains_before);
          return false;
        }
        if (k == FK::tensor)
          leaf = lf;
        else
          (leaf < 0 ? pre : post).push_back(cf);
      }
      AffineTerm& tm = s.term[t];
      tm.sign = terms[t].first == '-' ? -1 : 1;
      tm.leaf = leaf;
      tm.pre = tm.post0 = tm.post1 = -1;
      if (pre.size() > static_cast<size_t>(kMaxCoefFactors) || post.size() > 2) {
        plan.chains.resize(chains_before);
        return false;
      }
      if (!pre.empty()) tm.pre = add_chain(pre);
      if (!post.empty()) tm.post0 = add_chain({post[0]});
      if (post.size() > 1) tm.post1 = add_chain({post[1]});
    }
    out = s;
    return true;
  }

  int emit(const Expr& e, int depth, const OperandExpr& op, const ArrayMeta& sm) {
    if (depth >= kMaxVmRegs) throw error(errc::usage, "operand expression nests deeper than the device VM's 16 registers");
    VmInstr in{};
    in.dst = depth;
    switch (e.kind) {
      case Expr::Kind::literal:
        in.code = VM_LIT;
        in.imm = e.literal;
        break;
      case Expr::Kind::param: {
        in.code = VM_PARAM;
        const auto it = std::find(op.params.begin(), op.params.end(), e.name);
        in.arg = static_cast<int>(it - op.params.begin());
        break;
      }
      case Expr::Kind::access: {
        const LeafInfo& L = leaf_checked(e.name);
        if (e.subs.size() != L.meta.shape.size())
          throw error(errc::domain, "array " + e.name + " read with " + std::to_string(e.subs.size()) +
                                        " subscripts, has " + std::to_string(L.meta.shape.size()) + " axes");
        VmRead rd{};
        rd.leaf = (!acc_name.empty() && e.name == acc_name) ? kAccLeaf : leaf_of.at(e.name);
        rd.ndim = static_cast<int>(e.subs.size());
        if (rd.ndim > kMaxDims) throw error(errc::usage, "array " + e.name + " has too many axes for the device VM");
        std::int64_t stride = 1;
        for (int d = rd.ndim - 1; d >= 0; --d) {
          const auto it = std::find(op.params.begin(), op.params.end(), e.subs[d]);
          rd.param_of[d] = static_cast<int>(it - op.params.begin());
          rd.stride[d] = stride;
          stride *= L.meta.shape[d];
        }
        plan.reads.push_back(rd);
        in.code = VM_READ;
        in.arg = static_cast<int>(plan.reads.size()) - 1;
        break;
      }
      case Expr::Kind::unary: {
        emit(e.children[0], depth, op, sm);
        in.a = depth;
        if (e.name == "sin") in.code = VM_SIN;
        else if (e.name == "cos") in.code = VM_COS;
        else if (e.name == "exp") in.code = VM_EXP;
        else if (e.name == "sqrt") in.code = VM_SQRT;
        else if (e.name == "reciprocal") in.code = VM_RECIP;
        else throw error(errc::domain, "unknown function " + e.name);
        break;
      }
      case Expr::Kind::binary: {
        emit(e.children[0], depth, op, sm);
        emit(e.children[1], depth + 1, op, sm);
        in.a = depth;
        in.b = depth + 1;
        switch (e.op) {
          case '+': in.code = VM_ADD; break;
          case '-': in.code = VM_SUB; break;
          case '*': in.code = VM_MUL; break;
          case '/': in.code = VM_DIV; break;
          default: throw error(errc::domain, std::string("unknown operator ") + e.op);
        }
        break;
      }
    }
    plan.prog.push_back(in);
    return depth;
  }

  // Reproduce the reference's failure for reads that leave the array: the
  // first offending point in row-major order over the operand's shape.
  void check_ranges(const OperandExpr& op, const ArrayMeta& sm) {
    struct Hit {
      std::int64_t flat;
      std::string name;
      std::int64_t value;
      size_t axis;
    };
    std::optional<Hit> first;
    std::vector<std::int64_t> pstride(op.params.size(), 1);
    for (int k = static_cast<int>(op.params.size()) - 2; k >= 0; --k)
      pstride[k] = pstride[k + 1] * sm.shape[k + 1];
    std::function<void(const Expr&)> walk = [&](const Expr& e) {
      for (const Expr& c : e.children) walk(c);
      if (e.kind != Expr::Kind::access) return;
      auto it = leaf_of.find(e.name);
      if (it == leaf_of.end()) return;
      const ArrayMeta& lm = plan.leaves[it->second].meta;
      for (size_t d = 0; d < e.subs.size() && d < lm.shape.size(); ++d) {
        const auto pit = std::find(op.params.begin(), op.params.end(), e.subs[d]);
        const size_t k = static_cast<size_t>(pit - op.params.begin());
        if (k >= sm.shape.size() || sm.shape[k] <= lm.shape[d]) continue;
        const std::int64_t flat = lm.shape[d] * pstride[k];
        if (!first || flat < first->flat) first = Hit{flat, e.name, lm.shape[d], d};
      }
    };
    walk(op.body);
    if (first)
      throw error(errc::domain, "array " + first->name + " subscript " + std::to_string(first->value) +
                                    " out of range on axis " + std::to_string(first->axis));
  }

  // RowEpilogue of a row with output shape out: always a VM program (run by
  // generated code only); acc must be read pointwise (in-place safe)
  OperandStatic compile_epilogue(const feinsum::RowEpilogue& ep, const ArrayMeta& out, int out_storage) {
    if (ep.op.params.size() != out.shape.size())
      throw error(errc::domain, "epilogue of " + ep.acc + " takes " + std::to_string(ep.op.params.size()) +
                                    " parameters, the output has " + std::to_string(out.shape.size()) + " axes");
    if (leaf_of.count(ep.acc)) throw error(errc::domain, "epilogue value " + ep.acc + " is also a bound array");
    acc_name = ep.acc;
    acc_info = LeafInfo{out, out_storage};
    std::function<void(const Expr&)> check = [&](const Expr& e) {
      for (const Expr& c : e.children) check(c);
      if (e.kind != Expr::Kind::access) return;
      if (e.name == ep.acc) {
        if (e.subs != ep.op.params)
          throw error(errc::domain, "epilogue reads " + ep.acc + " off its own point (only [" +
                                        [&] {
                                          std::string j;
                                          for (const auto& x : ep.op.params) j += (j.empty() ? "" : ",") + x;
                                          return j;
                                        }() + "])");
        return;
      }
      const LeafInfo& L = leaf_checked(e.name);
      if (e.subs.size() != L.meta.shape.size())
        throw error(errc::domain, "array " + e.name + " read with " + std::to_string(e.subs.size()) +
                                      " subscripts, has " + std::to_string(L.meta.shape.size()) + " axes");
    };
    check(ep.op.body);
    check_ranges(ep.op, out);
    OperandStatic s{};
    s.kind = OPK_VM;
    s.ndim = static_cast<int>(out.shape.size());
    s.prog_off = static_cast<int>(plan.prog.size());
    emit(ep.op.body, 0, ep.op, out);
    s.prog_len = static_cast<int>(plan.prog.size()) - s.prog_off;
    if (uses_sqrt(ep.op.body)) throw error(errc::usage, "epilogues are real-valued (no sqrt)");
    acc_name.clear();
    return s;
  }

  OperandStatic compile(const OperandExpr& op, const ArrayMeta& sm) {
    if (op.params.size() != sm.shape.size())
      throw error(errc::domain, "materialize: operand takes " + std::to_string(op.params.size()) +
                                    " parameters, shape has " + std::to_string(sm.shape.size()) + " axes");
    // plain positional read of a same-shaped leaf
    const Expr& b = op.body;
    if (!force_vm && b.kind == Expr::Kind::access && b.subs == op.params) {
      auto it = leaf_of.find(b.name);
      if (it != leaf_of.end() && plan.leaves[it->second].meta.shape == sm.shape &&
          std::set<std::string>(op.params.begin(), op.params.end()).size() == op.params.size()) {
        OperandStatic s{};
        s.kind = OPK_PLAIN;
        s.leaf = it->second;
        s.ndim = static_cast<int>(sm.shape.size());
        return s;
      }
    }
    // validate every read up front (reference messages)
    std::function<void(const Expr&)> check = [&](const Expr& e) {
      for (const Expr& c : e.children) check(c);
      if (e.kind == Expr::Kind::access) {
        const LeafInfo& L = leaf_checked(e.name);
        if (e.subs.size() != L.meta.shape.size())
          throw error(errc::domain, "array " + e.name + " read with " + std::to_string(e.subs.size()) +
                                        " subscripts, has " + std::to_string(L.meta.shape.size()) + " axes");
      }
    };
    check(b);
    if (!skip_range_check) check_ranges(op, sm);
    OperandStatic s{};
    if (!force_vm && try_affine(op, sm, s)) return s;
    s = OperandStatic{};
    s.kind = OPK_VM;
    s.ndim = static_cast<int>(sm.shape.size());
    s.prog_off = static_cast<int>(plan.prog.size());
    emit(b, 0, op, sm);
    s.prog_len = static_cast<int>(plan.prog.size()) - s.prog_off;
    if (uses_sqrt(b)) plan.complex_mode = true;
    return s;
  }
};

// --------------------------------------------------------- pattern matching --

// Match a canonical notation against a role pattern (slots of role letters).
// Finds a slot permutation and index bijection making them equal position by
// position; returns role slot -> canonical slot and role letter -> index.
struct RoleMatch {
  std::vector<int> slot;            // pattern slot -> canonical slot
  std::map<char, std::string> idx;  // role letter -> canonical index
};

std::optional<RoleMatch> match_roles(const BatchedEinsum& c, const std::vector<std::string>& pat_in,
                                     const std::string& pat_out) {
  const int n = c.n();
  if (static_cast<int>(pat_in.size()) != n || c.i_out.size() != pat_out.size()) return std::nullopt;
  std::vector<int> perm(static_cast<size_t>(n));
  std::iota(perm.begin(), perm.end(), 0);
  do {
    std::map<char, std::string> fwd;
    std::map<std::string, char> back;
    bool ok = true;
    auto bind = [&](char role, const std::string& sym) {
      auto [it, fresh] = fwd.insert({role, sym});
      if (!fresh && it->second != sym) return false;
      auto [jt, fresh2] = back.insert({sym, role});
      if (!fresh2 && jt->second != role) return false;
      return true;
    };
    for (int k = 0; k < n && ok; ++k) {
      const std::string& roles = pat_in[k];
      const auto& syms = c.i_in[perm[k]];
      if (roles.size() != syms.size()) {
        ok = false;
        break;
      }
      for (size_t d = 0; d < roles.size() && ok; ++d) ok = bind(roles[d], syms[d]);
    }
    for (size_t d = 0; d < pat_out.size() && ok; ++d) ok = bind(pat_out[d], c.i_out[d]);
    if (ok) return RoleMatch{perm, fwd};
  } while (std::next_permutation(perm.begin(), perm.end()));
  return std::nullopt;
}

bool aligned16(const void* p) { return (reinterpret_cast<std::uintptr_t>(p) & 15u) == 0; }

// Tuned parameter from a fact's meta string "k1=v1;k2=v2" (default if absent).
int meta_int(const std::string& meta, const std::string& key, int dflt) {
  size_t pos = 0;
  while (pos < meta.size()) {
    size_t end = meta.find(';', pos);
    if (end == std::string::npos) end = meta.size();
    const std::string item = meta.substr(pos, end - pos);
    const size_t eq = item.find('=');
    if (eq != std::string::npos && item.substr(0, eq) == key) return std::atoi(item.c_str() + eq + 1);
    pos = end + 1;
  }
  return dflt;
}

// FEM gradient family: J[x,r,e] D[x,i,j] U[e,j] -> Y[r,e,i]
bool bind_fem(Plan& p, std::string* why) {
  const auto m = match_roles(p.canon.canonical, {"xre", "xij", "ej"}, "rei");
  if (!m) {
    *why = "notation is not xre,xij,ej->rei";
    return false;
  }
  if (p.complex_mode) {
    *why = "complex data";
    return false;
  }
  const auto lens = feinsum::index_lengths(p.canon.canonical);
  FemBinding f;
  f.NX = static_cast<int>(lens.at(m->idx.at('x')));
  f.NR = static_cast<int>(lens.at(m->idx.at('r')));
  f.NI = static_cast<int>(lens.at(m->idx.at('i')));
  f.NJ = static_cast<int>(lens.at(m->idx.at('j')));
  f.E = lens.at(m->idx.at('e'));
  f.rows = p.skel.b();
  if (!fem_grad_supported(f.NX, f.NR, f.NI, f.NJ)) {
    *why = "no compiled instance for these extents";
    return false;
  }
  if (f.E % 2 != 0) {
    *why = "odd element count (bulk copies need 16-byte runs)";
    return false;
  }
  if (f.rows > kFemMaxRows) {
    *why = "too many rows";
    return false;
  }
  const int n = p.skel.n();
  int u_tiles = 0;
  int elem_st = -1;
  for (int q = 0; q < f.rows; ++q) {
    const int ur = p.canon.sigma_row[q];
    auto operand = [&](int role) -> const OperandStatic& {
      return p.ops[static_cast<size_t>(ur) * n + p.canon.sigma_slot[m->slot[role]]];
    };
    const OperandStatic& J = operand(0);
    const OperandStatic& D = operand(1);
    const OperandStatic& U = operand(2);
    if (J.kind != OPK_PLAIN || D.kind != OPK_PLAIN) {
      *why = "functional J or D operand";
      return false;
    }
    // one element type for every array of the plan: f64, or f32 (the fp32
    // kernel instance; E % 4 == 0 so its bulk-copy rows stay 16-byte aligned)
    auto same_storage = [&](int st) {
      if (elem_st < 0) elem_st = st;
      return st == elem_st && (st == ST_F64 || (st == ST_F32 && f.E % 4 == 0));
    };
    if (!same_storage(leaf_info(p, J.leaf).storage) || !same_storage(leaf_info(p, D.leaf).storage)) {
      *why = "storage other than uniform f64 / f32 (f32: E % 4 == 0)";
      return false;
    }
    std::vector<AffineTerm> terms;
    if (U.kind == OPK_PLAIN) {
      terms.push_back(AffineTerm{1, -1, U.leaf, -1, -1});
    } else if (U.kind == OPK_AFFINE) {
      for (int t = 0; t < U.n_terms; ++t) {
        if (U.term[t].leaf < 0 || U.term[t].post1 >= 0) {
          *why = "affine U operand with a constant or two post factors";
          return false;
        }
        terms.push_back(U.term[t]);
      }
    } else {
      *why = "U operand needs the VM";
      return false;
    }
    for (const auto& t : terms)
      if (!same_storage(leaf_info(p, t.leaf).storage)) {
        *why = "storage other than uniform f64 / f32 (f32: E % 4 == 0)";
        return false;
      }
    u_tiles += static_cast<int>(terms.size());
    f.j_leaf.push_back(J.leaf);
    f.d_leaf.push_back(D.leaf);
    f.u_terms.push_back(std::move(terms));
    f.out_row.push_back(ur);
    if (!same_storage(p.outputs[ur].storage)) {
      *why = "output storage differs from the inputs'";
      return false;
    }
  }
  f.f32 = elem_st == ST_F32;
  if (u_tiles > kFemMaxUTiles) {
    *why = "too many U tiles";
    return false;
  }
  p.fem = std::move(f);
  return true;
}

std::vector<std::int64_t> row_major_strides(const std::vector<std::int64_t>& shape) {
  std::vector<std::int64_t> st(shape.size(), 1);
  for (int d = static_cast<int>(shape.size()) - 2; d >= 0; --d) st[d] = st[d + 1] * shape[d + 1];
  return st;
}

// Operand usable by the GETT prologue: plain, or coef[alpha] * X (+ coef[beta]).
bool gett_operand(const Plan& p, const OperandStatic& op, int* leaf, int* alpha, int* beta) {
  *alpha = *beta = -1;
  if (op.kind == OPK_PLAIN) {
    *leaf = op.leaf;
  } else if (op.kind == OPK_AFFINE) {
    const AffineTerm& t0 = op.term[0];
    if (t0.leaf < 0 || t0.post0 >= 0 || op.n_terms > 2) return false;
    *leaf = t0.leaf;
    *alpha = t0.pre;
    if (op.n_terms == 2) {
      const AffineTerm& t1 = op.term[1];
      if (t1.leaf >= 0 || t1.sign < 0 || t1.pre < 0) return false;
      *beta = t1.pre;
      if (*alpha < 0) return false;  // x + beta: no multiplier slot to fold it into
    }
  } else {
    return false;
  }
  const int st = leaf_info(p, *leaf).storage;
  return st == ST_F64 || st == ST_F32;
}

// Storage of the GETT roles over all rows (uniform f64 or f32 per role) and
// the operand rows; shared by both binders below.
bool gett_rows(Plan& p, GettBinding& g, int sa, int sb, std::string* why) {
  const BatchedEinsum& c = p.canon.canonical;
  const int n = c.n();
  int a_st = -1, b_st = -1, c_st = -1;
  for (int q = 0; q < c.b(); ++q) {
    const int ur = p.canon.sigma_row[q];
    GettBinding::Row r{};
    r.out_row = ur;
    if (!gett_operand(p, p.ops[static_cast<size_t>(ur) * n + p.canon.sigma_slot[sa]], &r.a_leaf, &r.a_alpha, &r.a_beta) ||
        !gett_operand(p, p.ops[static_cast<size_t>(ur) * n + p.canon.sigma_slot[sb]], &r.b_leaf, &r.b_alpha, &r.b_beta)) {
      *why = "operands are not plain or alpha*X+beta f64 / f32";
      return false;
    }
    const int sa_ = leaf_info(p, r.a_leaf).storage, sb_ = leaf_info(p, r.b_leaf).storage, sc_ = p.outputs[ur].storage;
    if ((a_st >= 0 && sa_ != a_st) || (b_st >= 0 && sb_ != b_st) || (c_st >= 0 && sc_ != c_st)) {
      *why = "mixed storage across rows";
      return false;
    }
    a_st = sa_;
    b_st = sb_;
    c_st = sc_;
    g.rows.push_back(r);
  }
  if (c_st != ST_F64 && c_st != ST_F32) {
    *why = "output storage other than f64 / f32";
    return false;
  }
  g.a_f32 = a_st == ST_F32;
  g.b_f32 = b_st == ST_F32;
  g.c_f32 = c_st == ST_F32;
  return true;
}

// GETT over index groups of one or two indices (matmul-shaped contractions:
// `ab,bc->ac`, `abc,cd->abd`, ...). A group of two indices maps onto the
// kernel's (outer, inner) dims as in bind_gett; a group of one index x of
// extent L is reshaped into (L / s, s) — offsets x * sigma = (x / s) * (s *
// sigma) + (x % s) * sigma, so no data moves. M / N inner extents must fit a
// 72-row box (24..72), K parts must be even; operands whose unit-stride dim is
// not the kernel's (A: kA, B: kB) are repacked per execute as in bind_gett.
bool bind_gett_split(Plan& p, std::string* why) {
  const BatchedEinsum& c = p.canon.canonical;
  if (p.complex_mode || c.n() != 2) {
    *why = "not a 2-operand contraction";
    return false;
  }
  {
    const std::set<std::string> s0(c.i_in[0].begin(), c.i_in[0].end()), s1(c.i_in[1].begin(), c.i_in[1].end()),
        so(c.i_out.begin(), c.i_out.end());
    if (s0.size() != c.i_in[0].size() || s1.size() != c.i_in[1].size() || so.size() != c.i_out.size()) {
      *why = "repeated indices";
      return false;
    }
  }
  // fold indices that stay adjacent (same order) in every array holding them
  // into one (TCCG's 6-index contractions: `dega,gfbc->abcdef` folds de and
  // bc): the row-major offset of the pair is that of one index of the
  // product extent, so no data moves
  std::vector<std::string> L0 = c.i_in[0], L1 = c.i_in[1], LC = c.i_out;
  std::map<std::string, std::int64_t> ex;
  for (const auto& [x, v] : feinsum::index_lengths(c)) ex[x] = v;
  for (bool merged = true; merged;) {
    merged = false;
    std::vector<std::vector<std::string>*> lists = {&L0, &L1, &LC};
    for (auto* L : lists) {
      for (size_t d = 0; d + 1 < L->size() && !merged; ++d) {
        const std::string x = (*L)[d], y = (*L)[d + 1];
        bool ok = true;
        for (auto* M : lists) {
          const auto px = std::find(M->begin(), M->end(), x), py = std::find(M->begin(), M->end(), y);
          if ((px == M->end()) != (py == M->end())) ok = false;  // different groups
          else if (px != M->end() && py != px + 1) ok = false;   // not adjacent in this array
        }
        if (!ok) continue;
        const std::string xy = x + "+" + y;
        ex[xy] = ex.at(x) * ex.at(y);
        for (auto* M : lists) {
          const auto px = std::find(M->begin(), M->end(), x);
          if (px == M->end()) continue;
          *px = xy;
          M->erase(px + 1);
        }
        merged = true;
      }
      if (merged) break;
    }
  }
  const feinsum::IndexList &l0 = L0, &l1 = L1;
  const std::set<std::string> s0(l0.begin(), l0.end()), s1(l1.begin(), l1.end()), so(LC.begin(), LC.end());
  std::vector<std::string> K, M0, N1, Z;  // K in operand 0's order; Z: batch (in A, B and C)
  for (const auto& x : l0) {
    const bool in1 = s1.count(x) > 0, ino = so.count(x) > 0;
    if (in1 && ino) {
      Z.push_back(x);
      continue;
    }
    if (!in1 && !ino) {
      *why = "index summed within one operand";
      return false;
    }
    (in1 ? K : M0).push_back(x);
  }
  if (Z.size() > 1) {
    *why = "more than one batch index";
    return false;
  }
  for (const auto& x : l1) {
    if (s0.count(x)) continue;
    if (!so.count(x)) {
      *why = "index summed within one operand";
      return false;
    }
    N1.push_back(x);
  }
  if (K.empty() || M0.empty() || N1.empty() || K.size() > 2 || M0.size() > 2 || N1.size() > 2) {
    *why = "index groups of one or two (folded) indices only";
    return false;
  }
  const auto& lens = ex;
  auto strides = [&](const std::vector<std::string>& l) {
    std::map<std::string, std::int64_t> m;
    std::int64_t st = 1;
    for (size_t d = l.size(); d-- > 0;) {
      m[l[d]] = st;
      st *= ex.at(l[d]);
    }
    return m;
  };
  const auto st0 = strides(L0), st1 = strides(L1), stc = strides(LC);
  // operand roles: B is the operand holding C's unit-stride index (coalesced
  // C stores run along the kernel's ni)
  const bool swap = std::find(M0.begin(), M0.end(), LC.back()) != M0.end();
  const int sa = swap ? 1 : 0, sb = 1 - sa;
  const auto& stA = swap ? st1 : st0;
  const auto& stB = swap ? st0 : st1;
  const std::vector<std::string>& M = swap ? N1 : M0;
  const std::vector<std::string>& N = swap ? M0 : N1;
  struct VD {
    std::int64_t ext = 1, a = 0, b = 0, c = 0;  // extent, strides in A, B, C
  };
  auto vd_of = [&](const std::string& x) {
    VD v;
    v.ext = lens.at(x);
    v.a = stA.count(x) ? stA.at(x) : 0;
    v.b = stB.count(x) ? stB.at(x) : 0;
    v.c = stc.count(x) ? stc.at(x) : 0;
    return v;
  };
  auto split = [](const VD& v, std::int64_t inner, VD* outer, VD* in) {
    *in = v;
    in->ext = inner;
    *outer = v;
    outer->ext = v.ext / inner;
    outer->a = v.a * inner;
    outer->b = v.b * inner;
    outer->c = v.c * inner;
  };
  // (outer, inner) of an M / N group: inner extent in 24..72 (largest divisor)
  auto mn_dims = [&](const std::vector<std::string>& grp, bool by_c, VD* outer, VD* in) {
    if (grp.size() == 2) {
      VD x = vd_of(grp[0]), y = vd_of(grp[1]);
      const bool y_inner = by_c ? y.c < x.c : (M == grp ? y.a < x.a : y.b < x.b);
      *in = y_inner ? y : x;
      *outer = y_inner ? x : y;
      // the M box dim (72 rows) should be as full as possible: take the other
      // index when the stride-preferred one fills it under 2/3. N keeps C's
      // unit-stride index (coalesced, vectorised epilogue stores) unless it
      // does not fit at all.
      if (!by_c && in->ext < 48 && outer->ext >= 48 && outer->ext <= 72) std::swap(*in, *outer);
      if (!(in->ext >= 24 && in->ext <= 72) && outer->ext >= 24 && outer->ext <= 72) std::swap(*in, *outer);
      return in->ext >= 24 && in->ext <= 72;
    }
    const VD v = vd_of(grp[0]);
    for (std::int64_t d = 72; d >= 24; --d)
      if (v.ext % d == 0) {
        split(v, d, outer, in);
        return true;
      }
    return false;
  };
  VD mo, mi, no, ni, ka, kb;
  if (!mn_dims(M, false, &mo, &mi) || !mn_dims(N, true, &no, &ni)) {
    *why = "M / N extents have no 24..72 inner part";
    return false;
  }
  if (K.size() == 2) {
    VD x = vd_of(K[0]), y = vd_of(K[1]);
    // kA = A's finer-stride K index
    ka = x.a < y.a ? x : y;
    kb = x.a < y.a ? y : x;
  } else {
    // one K index: kA (A's part) inner, kB outer; both even, kA a multiple
    // of the 8-wide A box where possible
    const VD v = vd_of(K[0]);
    std::int64_t best = 0;
    for (std::int64_t d : {8, 16, 32, 64, 4, 2, 24, 40, 48, 56, 12, 20, 28, 36, 44, 6, 10, 14, 18, 22, 26, 30})
      if (v.ext % d == 0 && (v.ext / d) % 2 == 0) {
        best = d;
        break;
      }
    if (!best) {
      *why = "K extent has no even x even split";
      return false;
    }
    split(v, best, &kb, &ka);
  }
  GettBinding g;
  g.ext_mo = mo.ext;
  g.ext_mi = mi.ext;
  g.ext_no = no.ext;
  g.ext_ni = ni.ext;
  g.ext_ka = ka.ext;
  g.ext_kb = kb.ext;
  if (!gett_supported(g.ext_mi, g.ext_ni, g.ext_ka, g.ext_kb)) {
    *why = "extents outside the kernel box (mi, ni in 24..72, even K extents)";
    return false;
  }
  if (!gett_rows(p, g, sa, sb, why)) return false;
  VD zd;  // batch dim (extent 1 when there is none)
  if (!Z.empty()) {
    zd = vd_of(Z[0]);
    for (const auto& r : g.rows)
      if (r.a_alpha >= 0 || r.b_alpha >= 0) {
        *why = "alpha*X+beta operands with a batch index";
        return false;
      }
  }
  g.nz = zd.ext;
  g.c_z = zd.c;
  // A: kA unit stride, other strides even (16-byte TMA strides); B: kB
  g.pack_a = g.a_f32 || ka.a != 1 || mo.a % 2 || mi.a % 2 || kb.a % 2 || zd.a % 2;
  g.pack_b = g.b_f32 || kb.b != 1 || no.b % 2 || ni.b % 2 || ka.b % 2 || zd.b % 2;
  g.a_z_src = zd.a;
  g.b_z_src = zd.b;
  g.a_z = g.pack_a ? g.ext_mo * g.ext_mi * g.ext_kb * g.ext_ka : zd.a;
  g.b_z = g.pack_b ? g.ext_no * g.ext_ni * g.ext_ka * g.ext_kb : zd.b;
  if (g.pack_a) {
    const std::int64_t src[4] = {mo.a, mi.a, kb.a, ka.a};
    std::copy(src, src + 4, g.a_src);
    g.a_kb = g.ext_ka;
    g.a_mi = g.ext_kb * g.ext_ka;
    g.a_mo = g.ext_mi * g.a_mi;
  } else {
    g.a_mo = mo.a;
    g.a_mi = mi.a;
    g.a_kb = kb.a;
  }
  if (g.pack_b) {
    const std::int64_t src[4] = {no.b, ni.b, ka.b, kb.b};
    std::copy(src, src + 4, g.b_src);
    g.b_ka = g.ext_kb;
    g.b_ni = g.ext_ka * g.ext_kb;
    g.b_no = g.ext_ni * g.b_ni;
  } else {
    g.b_no = no.b;
    g.b_ni = ni.b;
    g.b_ka = ka.b;
  }
  g.c_mo = mo.c;
  g.c_mi = mi.c;
  g.c_no = no.c;
  g.c_ni = ni.c;
  auto names = [](const std::vector<std::string>& v) {
    std::string r;
    for (const auto& x : v) r += x;
    return r;
  };
  g.shard_m = M[0].substr(0, M[0].find('+'));  // a folded pair shards along its outer index
  g.role_names = std::string(Z.empty() ? "" : "batch " + Z[0] + " (" + std::to_string(g.nz) + ") ") + "split M=" + names(M) + " (" + std::to_string(g.ext_mo) + "x" + std::to_string(g.ext_mi) + ") N=" +
                 names(N) + " (" + std::to_string(g.ext_no) + "x" + std::to_string(g.ext_ni) + ") K=" + names(K) +
                 " (" + std::to_string(g.ext_kb) + "x" + std::to_string(g.ext_ka) + ")" + (g.pack_a ? " packA" : "") +
                 (g.pack_b ? " packB" : "") + (g.a_f32 || g.b_f32 || g.c_f32 ? " f32io" : "");
  p.gett = std::move(g);
  return true;
}

bool bind_gett4(Plan& p, std::string* why);

// GETT family: the 2+2+2-index TCCG form (bind_gett4), else the split form.
bool bind_gett(Plan& p, std::string* why) {
  std::string w4;
  if (bind_gett4(p, &w4)) return true;
  if (bind_gett_split(p, why)) return true;
  *why = w4 + "; " + *why;
  return false;
}

// 2 slots, pure contraction (every index in exactly two of A, B, C), 2+2+2
// indices, C's unit-stride index on the B side, A's and B's unit-stride
// indices both contracted.
bool bind_gett4(Plan& p, std::string* why) {
  const BatchedEinsum& c = p.canon.canonical;
  if (p.complex_mode || c.n() != 2 || c.i_out.size() != 4) {
    *why = "not a 2-operand 4-index contraction";
    return false;
  }
  const std::set<std::string> s0(c.i_in[0].begin(), c.i_in[0].end()), s1(c.i_in[1].begin(), c.i_in[1].end());
  if (s0.size() != 4 || s1.size() != 4 || c.i_in[0].size() != 4 || c.i_in[1].size() != 4) {
    *why = "repeated indices";
    return false;
  }
  std::set<std::string> K, out(c.i_out.begin(), c.i_out.end());
  for (const auto& x : s0)
    if (s1.count(x)) K.insert(x);
  if (K.size() != 2) {
    *why = "needs exactly two contracted indices";
    return false;
  }
  for (const auto& x : out)
    if (K.count(x)) {
      *why = "batch index";
      return false;
    }
  // ni: the kernel's inner N index (one 72-row TMA box per no value); the
  // output's last index when its extent fits a box (coalesced C stores),
  // else the next output index from the end that does
  const auto lens0 = feinsum::index_lengths(c);
  auto fits = [&](const std::string& x) { return lens0.at(x) >= 24 && lens0.at(x) <= 72; };
  std::string ni = c.i_out.back();
  for (auto it = c.i_out.rbegin(); it != c.i_out.rend(); ++it)
    if (fits(*it)) {
      ni = *it;
      break;
    }
  const int sb = s1.count(ni) ? 1 : 0, sa = 1 - sb;
  const feinsum::IndexList& la = c.i_in[sa];
  const feinsum::IndexList& lb = c.i_in[sb];
  // the kernel wants A's unit-stride index to be one contracted index (kA)
  // and B's the other (kB); an operand that does not comply is repacked per
  // execute (one HBM pass, ~1% of the contraction at TCCG sizes) — this is
  // what lets every TCCG sibling spelling run on the tensor cores
  const std::vector<std::string> Kv(K.begin(), K.end());
  const bool a_ok = K.count(la.back()) > 0;
  bool b_ok = K.count(lb.back()) > 0 && !(a_ok && lb.back() == la.back());
  std::string ka, kb;
  if (a_ok) {
    ka = la.back();
    kb = ka == Kv[0] ? Kv[1] : Kv[0];
    b_ok = b_ok && lb.back() == kb;
  } else if (b_ok) {
    kb = lb.back();
    ka = kb == Kv[0] ? Kv[1] : Kv[0];
  } else {
    ka = Kv[0];
    kb = Kv[1];
  }
  const auto lens = feinsum::index_lengths(c);
  std::vector<std::string> M, N;
  for (const auto& x : la)
    if (!K.count(x)) M.push_back(x);
  for (const auto& x : lb)
    if (!K.count(x)) N.push_back(x);
  std::string mi = M[1], mo = M[0];  // later position = smaller stride in A
  if (!fits(mi) && fits(mo)) std::swap(mi, mo);  // TMA dims take any order
  const std::string no = N[0] == ni ? N[1] : N[0];
  GettBinding g;
  g.pack_a = !a_ok;
  g.pack_b = !b_ok;
  // storage: uniform per role over the rows (f64 or f32); fp32 operands are
  // widened through the pack pass
  {
    const int n = c.n();
    int a_st = -1, b_st = -1, c_st = -1;
    for (int q = 0; q < c.b(); ++q) {
      const int ur = p.canon.sigma_row[q];
      const OperandStatic& oa = p.ops[static_cast<size_t>(ur) * n + p.canon.sigma_slot[sa]];
      const OperandStatic& ob = p.ops[static_cast<size_t>(ur) * n + p.canon.sigma_slot[sb]];
      const int la_leaf = oa.kind == OPK_AFFINE ? oa.term[0].leaf : oa.leaf;
      const int lb_leaf = ob.kind == OPK_AFFINE ? ob.term[0].leaf : ob.leaf;
      if (la_leaf < 0 || lb_leaf < 0 || (oa.kind != OPK_PLAIN && oa.kind != OPK_AFFINE) ||
          (ob.kind != OPK_PLAIN && ob.kind != OPK_AFFINE)) {
        *why = "operands are not plain or alpha*X+beta";
        return false;
      }
      const int sa_ = leaf_info(p, la_leaf).storage, sb_ = leaf_info(p, lb_leaf).storage, sc_ = p.outputs[ur].storage;
      if ((a_st >= 0 && sa_ != a_st) || (b_st >= 0 && sb_ != b_st) || (c_st >= 0 && sc_ != c_st)) {
        *why = "mixed storage across rows";
        return false;
      }
      a_st = sa_;
      b_st = sb_;
      c_st = sc_;
    }
    if ((a_st != ST_F64 && a_st != ST_F32) || (b_st != ST_F64 && b_st != ST_F32) || (c_st != ST_F64 && c_st != ST_F32)) {
      *why = "storage other than f64 / f32";
      return false;
    }
    g.a_f32 = a_st == ST_F32;
    g.b_f32 = b_st == ST_F32;
    g.c_f32 = c_st == ST_F32;
    g.pack_a = g.pack_a || g.a_f32;
    g.pack_b = g.pack_b || g.b_f32;
  }
  g.ext_mo = lens.at(mo);
  g.ext_mi = lens.at(mi);
  g.ext_no = lens.at(no);
  g.ext_ni = lens.at(ni);
  g.ext_ka = lens.at(ka);
  g.ext_kb = lens.at(kb);
  if (!gett_supported(g.ext_mi, g.ext_ni, g.ext_ka, g.ext_kb)) {
    *why = "extents outside the kernel box (mi, ni in 24..72, even K extents)";
    return false;
  }
  auto stride_of = [&](const feinsum::IndexList& l, const std::vector<std::int64_t>& shape, const std::string& s) {
    const auto st = row_major_strides(shape);
    for (size_t d = 0; d < l.size(); ++d)
      if (l[d] == s) return st[d];
    return std::int64_t{0};
  };
  const auto& sha = c.args[0][sa].shape;
  const auto& shb = c.args[0][sb].shape;
  std::vector<std::int64_t> shc;
  for (const auto& s : c.i_out) shc.push_back(lens.at(s));
  // TMA strides must be multiples of 16 bytes: an operand with an odd stride
  // is repacked like a non-compliant one
  if (!g.pack_a && (stride_of(la, sha, mo) % 2 || stride_of(la, sha, mi) % 2 || stride_of(la, sha, kb) % 2)) g.pack_a = true;
  if (!g.pack_b && (stride_of(lb, shb, no) % 2 || stride_of(lb, shb, ni) % 2 || stride_of(lb, shb, ka) % 2)) g.pack_b = true;
  if (g.pack_a) {
    const std::int64_t src[4] = {stride_of(la, sha, mo), stride_of(la, sha, mi), stride_of(la, sha, kb),
                                 stride_of(la, sha, ka)};
    std::copy(src, src + 4, g.a_src);
    g.a_kb = g.ext_ka;
    g.a_mi = g.ext_kb * g.ext_ka;
    g.a_mo = g.ext_mi * g.a_mi;
  } else {
    g.a_mo = stride_of(la, sha, mo);
    g.a_mi = stride_of(la, sha, mi);
    g.a_kb = stride_of(la, sha, kb);
  }
  if (g.pack_b) {
    const std::int64_t src[4] = {stride_of(lb, shb, no), stride_of(lb, shb, ni), stride_of(lb, shb, ka),
                                 stride_of(lb, shb, kb)};
    std::copy(src, src + 4, g.b_src);
    g.b_ka = g.ext_kb;
    g.b_ni = g.ext_ka * g.ext_kb;
    g.b_no = g.ext_ni * g.b_ni;
  } else {
    g.b_no = stride_of(lb, shb, no);
    g.b_ni = stride_of(lb, shb, ni);
    g.b_ka = stride_of(lb, shb, ka);
  }
  g.c_mo = stride_of(c.i_out, shc, mo);
  g.c_mi = stride_of(c.i_out, shc, mi);
  g.c_no = stride_of(c.i_out, shc, no);
  g.c_ni = stride_of(c.i_out, shc, ni);
  g.shard_m = mo;
  g.role_names = "mo=" + mo + " mi=" + mi + " no=" + no + " ni=" + ni + " kA=" + ka + " kB=" + kb +
                 (g.pack_a ? " packA" : "") + (g.pack_b ? " packB" : "") + (g.a_f32 || g.b_f32 || g.c_f32 ? " f32io" : "");
  const int n = c.n();
  for (int q = 0; q < c.b(); ++q) {
    const int ur = p.canon.sigma_row[q];
    GettBinding::Row r{};
    r.out_row = ur;
    if (!gett_operand(p, p.ops[static_cast<size_t>(ur) * n + p.canon.sigma_slot[sa]], &r.a_leaf, &r.a_alpha, &r.a_beta) ||
        !gett_operand(p, p.ops[static_cast<size_t>(ur) * n + p.canon.sigma_slot[sb]], &r.b_leaf, &r.b_alpha, &r.b_beta)) {
      *why = "operands are not plain or alpha*X+beta f64 / f32";
      return false;
    }
    g.rows.push_back(r);
  }
  p.gett = std::move(g);
  return true;
}

// Tensor-train family: G1[i,j] G2[k,l] X[n,j,l] -> Y[n,i,k], 64^4 cores.
bool bind_tt(Plan& p, std::string* why) {
  const auto m = match_roles(p.canon.canonical, {"ij", "kl", "njl"}, "nik");
  if (!m) {
    *why = "notation is not ij,kl,njl->nik";
    return false;
  }
  if (p.complex_mode) {
    *why = "complex data";
    return false;
  }
  const auto lens = feinsum::index_lengths(p.canon.canonical);
  TTBinding t;
  t.nb = lens.at(m->idx.at('n'));
  t.NI = static_cast<int>(lens.at(m->idx.at('i')));
  t.NJ = static_cast<int>(lens.at(m->idx.at('j')));
  t.NK = static_cast<int>(lens.at(m->idx.at('k')));
  t.NL = static_cast<int>(lens.at(m->idx.at('l')));
  if (!tt_supported(t.NI, t.NJ, t.NK, t.NL, false) && !tt_supported(t.NI, t.NJ, t.NK, t.NL, true)) {
    *why = "cores outside 8..64 (or an odd unit-stride extent)";
    return false;
  }
  const int n = p.skel.n();
  int storage = -1;
  for (int q = 0; q < p.skel.b(); ++q) {
    const int ur = p.canon.sigma_row[q];
    TTBinding::Row r{};
    int* dst[3] = {&r.g1, &r.g2, &r.x};
    for (int role = 0; role < 3; ++role) {
      const OperandStatic& op = p.ops[static_cast<size_t>(ur) * n + p.canon.sigma_slot[m->slot[role]]];
      if (op.kind != OPK_PLAIN) {
        *why = "functional operand";
        return false;
      }
      const int st = leaf_info(p, op.leaf).storage;
      if ((st != ST_F64 && st != ST_F32) || (storage >= 0 && st != storage)) {
        *why = "storage must be uniformly f64 or f32";
        return false;
      }
      storage = st;
      *dst[role] = op.leaf;
    }
    if (p.outputs[ur].storage != storage) {
      *why = "output storage differs from the inputs";
      return false;
    }
    r.out_row = ur;
    t.rows.push_back(r);
  }
  t.fp32 = storage == ST_F32;
  if (!tt_supported(t.NI, t.NJ, t.NK, t.NL, t.fp32)) {
    *why = "fp32 cores need a unit-stride extent divisible by 4";
    return false;
  }
  p.tt = std::move(t);
  return true;
}

// Hex sum-factorised family (C2):
//   B1[x,a,i] B2[x,b,m] B3[x,c,n] G[x,y,e,a,b,c] F1[y,a,j] F2[y,b,k] F3[y,c,l] u[e,j,k,l] -> y[e,i,m,n]
// with the 1-D operators and G shared by every row (field).
bool bind_hex(Plan& p, std::string* why) {
  const BatchedEinsum& c = p.canon.canonical;
  if (c.n() != 8 || p.complex_mode) {
    *why = "not an 8-slot real einsum";
    return false;
  }
  const auto m = match_roles(c, {"xai", "xbm", "xcn", "xyeabc", "yaj", "ybk", "ycl", "ejkl"}, "eimn");
  if (!m) {
    *why = "notation is not the sum-factorised hex operator";
    return false;
  }
  const auto lens = feinsum::index_lengths(c);
  HexBinding h;
  h.E = lens.at(m->idx.at('e'));
  h.ND = static_cast<int>(lens.at(m->idx.at('x')));
  h.P = static_cast<int>(lens.at(m->idx.at('a')));
  for (char r : std::string("bcijklmn"))
    if (lens.at(m->idx.at(r)) != h.P) {
      *why = "quadrature and dof extents differ";
      return false;
    }
  if (lens.at(m->idx.at('y')) != h.ND || !hex_supported(h.ND, h.P, h.E, c.b())) {
    *why = "no compiled instance (needs 3 directions, P = 5, even E, <= 8 fields)";
    return false;
  }
  const int n = c.n();
  // pattern slot -> kernel matrix index: slots 0..2 backward (B1..B3), 4..6 forward (F1..F3)
  const int mat_of_slot[8] = {3, 4, 5, -1, 0, 1, 2, -1};
  // one element type: f64, or f32 (the fp32 instance: four-element stages,
  // so E % 4 == 0 below P = 6)
  const int est = p.outputs[0].storage;
  if ((est != ST_F64 && est != ST_F32) || (est == ST_F32 && h.P < 6 && h.E % 4 != 0)) {
    *why = "storage other than uniform f64 / f32 (f32: E % 4 == 0)";
    return false;
  }
  h.f32 = est == ST_F32;
  for (int q = 0; q < c.b(); ++q) {
    const int ur = p.canon.sigma_row[q];
    auto leaf_at = [&](int role) -> int {
      const OperandStatic& op = p.ops[static_cast<size_t>(ur) * n + p.canon.sigma_slot[m->slot[role]]];
      if (op.kind != OPK_PLAIN || leaf_info(p, op.leaf).storage != est) return -1;
      return op.leaf;
    };
    for (int role = 0; role < 8; ++role) {
      const int leaf = leaf_at(role);
      if (leaf < 0) {
        *why = "functional operand or mixed storage";
        return false;
      }
      if (role == 7) {
        h.u.push_back(leaf);
      } else if (role == 3) {
        if (h.g >= 0 && h.g != leaf) {
          *why = "G differs between rows";
          return false;
        }
        h.g = leaf;
      } else {
        int& slot = h.mats[mat_of_slot[role]];
        if (slot >= 0 && slot != leaf) {
          *why = "1-D operators differ between rows";
          return false;
        }
        slot = leaf;
      }
    }
    if (p.outputs[ur].storage != est) {
      *why = "mixed output storage";
      return false;
    }
    h.out_row.push_back(ur);
  }
  p.hex = std::move(h);
  return true;
}

// ------------------------------------------------------------ path FLOPs --

}  // namespace

double optimal_path_flops(const BatchedEinsum& e) {
  const int n = e.n();
  const auto len = feinsum::index_lengths(e);
  std::vector<std::set<std::string>> idx(static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) idx[k].insert(e.i_in[k].begin(), e.i_in[k].end());
  const std::set<std::string> out(e.i_out.begin(), e.i_out.end());
  auto size_of = [&](const std::set<std::string>& s) {
    double v = 1;
    for (const auto& x : s) v *= static_cast<double>(len.at(x));
    return v;
  };
  if (n == 1) {
    // a single operand: one pass over its iteration space if it reduces
    std::set<std::string> all = idx[0];
    const bool reduces = all.size() > out.size() || e.i_in[0].size() != all.size();
    return reduces ? size_of(all) : 0.0;
  }
  if (n > 16) return feinsum::flop_count(e) / std::max(1, e.b());
  const int full = (1 << n) - 1;
  std::vector<std::set<std::string>> keep(static_cast<size_t>(full) + 1);
  for (int s = 1; s <= full; ++s) {
    std::set<std::string> inside, outside = out;
    for (int k = 0; k < n; ++k)
      (s >> k & 1 ? inside : outside).insert(idx[k].begin(), idx[k].end());
    for (const auto& x : inside)
      if (outside.count(x)) keep[s].insert(x);
  }
  std::vector<double> cost(static_cast<size_t>(full) + 1, 0.0);
  for (int s = 1; s <= full; ++s) {
    if ((s & (s - 1)) == 0) continue;  // singleton
    double best = INFINITY;
    for (int a = (s - 1) & s; a > 0; a = (a - 1) & s) {
      const int b = s ^ a;
      if (a < b) continue;  // each split once
      std::set<std::string> all = keep[a];
      all.insert(keep[b].begin(), keep[b].end());
      const bool summed = all.size() > keep[s].size();
      const double c = cost[a] + cost[b] + size_of(all) * (summed ? 2.0 : 1.0);
      best = std::min(best, c);
    }
    cost[s] = best;
  }
  return cost[full];
}

namespace {

double expr_ops(const Expr& e) {
  double c = (e.kind == Expr::Kind::binary || e.kind == Expr::Kind::unary) ? 1.0 : 0.0;
  for (const Expr& x : e.children) c += expr_ops(x);
  return c;
}

void upload_tables(Plan& p, GenericLaunch& g, const BatchedEinsum& e, bool dry_run) {
  std::map<std::string, int> pos;
  {
    std::vector<std::string> syms = e.i_out;
    for (auto& s : feinsum::reduction_indices(e)) syms.push_back(s);
    for (size_t i = 0; i < syms.size(); ++i) pos[syms[i]] = static_cast<int>(i);
  }
  // static blob: ops | slot_pos | slot_stride | slot_ndim | prog | reads | chains
  std::vector<int> slot_pos(static_cast<size_t>(e.n()) * kMaxDims, 0), slot_ndim(static_cast<size_t>(e.n()), 0);
  std::vector<std::int64_t> slot_stride(static_cast<size_t>(e.n()) * kMaxDims, 0);
  for (int k = 0; k < e.n(); ++k) {
    const int nd = static_cast<int>(e.i_in[k].size());
    if (nd > kMaxDims) throw error(errc::usage, "operand with more than 12 axes");
    slot_ndim[k] = nd;
    std::int64_t st = 1;
    for (int d = nd - 1; d >= 0; --d) {
      slot_pos[k * kMaxDims + d] = pos.at(e.i_in[k][d]);
      slot_stride[k * kMaxDims + d] = st;
      st *= e.args[0][k].shape[d];
    }
  }
  auto align = [](size_t x) { return (x + 255) & ~size_t{255}; };
  size_t off = 0;
  const size_t o_ops = off; off = align(off + sizeof(OperandStatic) * p.ops.size());
  const size_t o_pos = off; off = align(off + sizeof(int) * slot_pos.size());
  const size_t o_str = off; off = align(off + sizeof(std::int64_t) * slot_stride.size());
  const size_t o_nd = off; off = align(off + sizeof(int) * slot_ndim.size());
  const size_t o_prog = off; off = align(off + sizeof(VmInstr) * p.prog.size());
  const size_t o_reads = off; off = align(off + sizeof(VmRead) * p.reads.size());
  const size_t o_chains = off; off = align(off + sizeof(CoefChain) * p.chains.size());
  const size_t total = std::max<size_t>(off, 256);
  std::vector<unsigned char> blob(total, 0);
  auto put = [&](size_t at, const void* src, size_t n) {
    if (n) std::memcpy(blob.data() + at, src, n);
  };
  put(o_ops, p.ops.data(), sizeof(OperandStatic) * p.ops.size());
  put(o_pos, slot_pos.data(), sizeof(int) * slot_pos.size());
  put(o_str, slot_stride.data(), sizeof(std::int64_t) * slot_stride.size());
  put(o_nd, slot_ndim.data(), sizeof(int) * slot_ndim.size());
  put(o_prog, p.prog.data(), sizeof(VmInstr) * p.prog.size());
  put(o_reads, p.reads.data(), sizeof(VmRead) * p.reads.size());
  put(o_chains, p.chains.data(), sizeof(CoefChain) * p.chains.size());

  if (dry_run) return;
  cuda_check(cudaGetDevice(&p.device), "cudaGetDevice");
  cuda_check(device_sm_count(&p.sm_count), "device attributes");
  cuda_check(cudaMalloc(&p.d_blob, total), "cudaMalloc(plan tables)");
  cuda_check(cudaMemcpy(p.d_blob, blob.data(), total, cudaMemcpyHostToDevice), "upload plan tables");
  if (!p.chains.empty()) {
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&p.d_coef), sizeof(double) * 2 * p.chains.size()),
               "cudaMalloc(coefficients)");
    // literal-only chains (e.g. C5's 0.5) are folded here with the coefficient
    // kernel's arithmetic (complex left fold, IEEE products, no contraction)
    // and uploaded once, which saves a launch per execute
    bool literal = true;
    for (const auto& ch : p.chains)
      for (int f = 0; f < ch.n; ++f) literal = literal && ch.f[f].leaf < 0;
    if (literal) {
      std::vector<double> host(2 * p.chains.size());
      for (size_t c = 0; c < p.chains.size(); ++c) {
        double re = 0.0, im = 0.0;
        for (int f = 0; f < p.chains[c].n; ++f) {
          const double vr = p.chains[c].f[f].lit, vi = 0.0;
          if (f == 0) {
            re = vr;
            im = vi;
          } else {
            const double nr = re * vr - im * vi, ni = re * vi + im * vr;
            re = nr;
            im = ni;
          }
        }
        host[2 * c] = re;
        host[2 * c + 1] = im;
      }
      cuda_check(cudaMemcpy(p.d_coef, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice),
                 "upload coefficients");
      p.coef_static = true;
    }
  }
  auto* base = static_cast<unsigned char*>(p.d_blob);
  g.ops = reinterpret_cast<const OperandStatic*>(base + o_ops);
  g.slot_pos = reinterpret_cast<const int*>(base + o_pos);
  g.slot_stride = reinterpret_cast<const std::int64_t*>(base + o_str);
  g.slot_ndim = reinterpret_cast<const int*>(base + o_nd);
  g.prog = reinterpret_cast<const VmInstr*>(base + o_prog);
  g.reads = reinterpret_cast<const VmRead*>(base + o_reads);
  g.chains = reinterpret_cast<const CoefChain*>(base + o_chains);
  g.n_chains = static_cast<int>(p.chains.size());
  g.coef = p.d_coef;
}

// Contraction path for einsums of three or more operands with no tuned family
// of their own: the cheapest pairwise order (the DP of optimal_path_flops,
// the opt_einsum convention the roofline counts in) executed as a chain of
// 2-operand plans, each on its own tuned family when one binds (GETT: M / N /
// K / batch groups of one or two indices) and on the generic kernel
// otherwise; taken when the path costs under a quarter of the naive sum.
// Intermediates are plan buffers in the operands' element type (f64 / f32). The summation order differs from the reference's naive
// sum (like every tuned family: the 1e-12 bar); exact on dyadic data while
// partial sums stay below 2^53.
bool bind_path(Plan& p, const PlanOptions& opt, std::string* why) {
  const BatchedEinsum& e = p.skel;
  const int n = e.n();
  if (e.b() > 1 && !p.complex_mode && !p.functional && p.tabs.empty()) {
    // several rows and no family for the whole batch: each row planned on
    // its own (a family, a path or the generic kernel), taken when at least
    // one row gets something better than the generic kernel
    PlanOptions so = opt;
    so.force_transform.clear();
    so.meta_override.clear();
    std::vector<PathStep> steps;
    bool better = false;
    try {
      for (int r = 0; r < e.b(); ++r) {
        BatchedEinsum row;
        row.i_in = e.i_in;
        row.i_out = e.i_out;
        row.args = {e.args[static_cast<size_t>(r)]};
        PathStep ps;
        ps.plan = make_plan(row, so);
        better = better || ps.plan->family != Family::generic;
        for (const auto& L : ps.plan->leaves) {
          int src = -1;
          for (size_t i = 0; i < p.leaves.size(); ++i)
            if (p.leaves[i].meta.name == L.meta.name) src = static_cast<int>(i);
          if (src < 0 || L.storage != p.leaves[static_cast<size_t>(src)].storage) throw error(errc::usage, "row leaf");
          ps.src.push_back(src);
        }
        if (ps.plan->outputs[0].storage != p.outputs[static_cast<size_t>(r)].storage) throw error(errc::usage, "row output");
        ps.out = -1;
        ps.out_row = r;
        steps.push_back(std::move(ps));
      }
    } catch (const std::exception& ex) {
      *why = std::string("path: ") + ex.what();
      return false;
    }
    if (!better) {
      *why = "path: no row has a better plan than the generic kernel";
      return false;
    }
    p.path = std::move(steps);
    p.inter_bytes = 0;
    return true;
  }
  if (e.b() != 1 || n < 2 || n > 12 || p.complex_mode || p.functional || !p.tabs.empty()) {
    *why = "path: one row of 2..12 plain real operands";
    return false;
  }
  // one element type: f64, or f32 (fp32 intermediates, like any fp32 chain)
  const int est = p.outputs[0].storage;
  for (int k = 0; k < n; ++k)
    if (p.ops[static_cast<size_t>(k)].kind != OPK_PLAIN || leaf_info(p, p.ops[static_cast<size_t>(k)].leaf).storage != est ||
        (est != ST_F64 && est != ST_F32)) {
      *why = "path: plain operands, all f64 or all f32";
      return false;
    }
  const std::int64_t esize = est == ST_F32 ? 4 : 8;
  const auto len = feinsum::index_lengths(e);
  std::vector<std::set<std::string>> idx(static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) idx[static_cast<size_t>(k)].insert(e.i_in[k].begin(), e.i_in[k].end());
  const std::set<std::string> out(e.i_out.begin(), e.i_out.end());
  auto size_of = [&](const std::set<std::string>& st) {
    double v = 1;
    for (const auto& x : st) v *= static_cast<double>(len.at(x));
    return v;
  };
  const int full = (1 << n) - 1;
  std::vector<std::set<std::string>> keep(static_cast<size_t>(full) + 1);
  for (int st = 1; st <= full; ++st) {
    std::set<std::string> inside, outside = out;
    for (int k = 0; k < n; ++k) (st >> k & 1 ? inside : outside).insert(idx[k].begin(), idx[k].end());
    for (const auto& x : inside)
      if (outside.count(x)) keep[static_cast<size_t>(st)].insert(x);
  }
  std::vector<double> cost(static_cast<size_t>(full) + 1, 0.0);
  std::vector<int> split(static_cast<size_t>(full) + 1, 0);
  for (int st = 1; st <= full; ++st) {
    if ((st & (st - 1)) == 0) continue;
    double best = INFINITY;
    for (int a = (st - 1) & st; a > 0; a = (a - 1) & st) {
      const int b = st ^ a;
      if (a < b) continue;
      std::set<std::string> all = keep[static_cast<size_t>(a)];
      all.insert(keep[static_cast<size_t>(b)].begin(), keep[static_cast<size_t>(b)].end());
      const double c = cost[static_cast<size_t>(a)] + cost[static_cast<size_t>(b)] +
                       size_of(all) * (all.size() > keep[static_cast<size_t>(st)].size() ? 2.0 : 1.0);
      if (c < best) {
        best = c;
        split[static_cast<size_t>(st)] = a;
      }
    }
    cost[static_cast<size_t>(st)] = best;
  }
  // operands with private or repeated indices are first reduced to the
  // indices they share (a one-operand step: sum / diagonal on the generic
  // kernel); with two operands that is the only reason for a path
  int pre = 0;
  for (int k = 0; k < n; ++k)
    if (keep[static_cast<size_t>(1) << k].size() != e.i_in[static_cast<size_t>(k)].size()) ++pre;
  double pre_cost = 0;
  for (int k = 0; k < n; ++k) pre_cost += size_of(idx[static_cast<size_t>(k)]);
  if ((n == 2 && pre == 0) || (cost[static_cast<size_t>(full)] + pre_cost) * 4.0 >= feinsum::flop_count(e)) {
    *why = "path: no cheaper than the naive sum";
    return false;
  }
  // post-order build: an operand is (index list, meta, source)
  struct Opnd {
    feinsum::IndexList ix;
    ArrayMeta meta;
    int src;  // caller leaf, or -(1 + intermediate id)
  };
  std::vector<PathStep> steps;
  std::vector<std::int64_t> offs;
  std::int64_t bytes = 0;
  PlanOptions so = opt;
  so.force_transform.clear();
  so.meta_override.clear();
  std::function<Opnd(int)> build = [&](int st) -> Opnd {
    // a step over one or two operands into R (index list of st's keep set,
    // or the einsum's output at the root)
    auto make_step = [&](int s2, const std::vector<const Opnd*>& ops) {
      Opnd R;
      if (s2 == full) {
        R.ix = e.i_out;
      } else {
        for (const Opnd* o : ops)
          for (const auto& x : o->ix)
            if (keep[static_cast<size_t>(s2)].count(x) && std::find(R.ix.begin(), R.ix.end(), x) == R.ix.end())
              R.ix.push_back(x);
      }
      const int id = static_cast<int>(offs.size());
      R.meta.name = "_path_t" + std::to_string(id);
      R.meta.dtype = est == ST_F32 ? Dtype::float32 : Dtype::float64;
      for (const auto& x : R.ix) R.meta.shape.push_back(len.at(x));
      BatchedEinsum step;
      step.i_out = R.ix;
      step.args.emplace_back();
      for (const Opnd* o : ops) {
        step.i_in.push_back(o->ix);
        step.args[0].push_back(o->meta);
      }
      PathStep ps;
      ps.plan = make_plan(step, so);
      for (const auto& L : ps.plan->leaves)
        for (const Opnd* o : ops)
          if (L.meta.name == o->meta.name) {
            ps.src.push_back(o->src);
            break;
          }
      if (s2 == full) {
        ps.out = -1;
        R.src = 0;
      } else {
        ps.out = id;
        offs.push_back(bytes);
        bytes += (R.meta.num_elements() * esize + 255) / 256 * 256;
        R.src = -(1 + id);
      }
      steps.push_back(std::move(ps));
      return R;
    };
    if ((st & (st - 1)) == 0) {
      int k = 0;
      while (!(st >> k & 1)) ++k;
      Opnd leaf{e.i_in[static_cast<size_t>(k)], e.args[0][static_cast<size_t>(k)], p.ops[static_cast<size_t>(k)].leaf};
      if (keep[static_cast<size_t>(st)].size() == leaf.ix.size() || st == full) return leaf;
      return make_step(st, {&leaf});  // private / repeated indices reduced first
    }
    const int a = split[static_cast<size_t>(st)], b = st ^ a;
    const Opnd A = build(a), B = build(b);
    return make_step(st, {&A, &B});
  };
  try {
    build(full);
  } catch (const std::exception& ex) {
    *why = std::string("path: ") + ex.what();
    return false;
  }
  p.path = std::move(steps);
  p.inter_off = std::move(offs);
  p.inter_bytes = bytes;
  return true;
}

void finish_plan(Plan& p, const PlanOptions& opt) {
  const BatchedEinsum& e = p.skel;
  if (e.b() > kMaxRows) throw error(errc::usage, "more than 96 rows; spell the batch as an index");
  if (p.leaves.size() > static_cast<size_t>(kMaxLeaves)) throw error(errc::usage, "more than 96 input arrays");

  // outputs: R<row>, widest dtype of the row, i_out shape
  const auto lens = feinsum::index_lengths(e);
  for (int r = 0; r < e.b(); ++r) {
    OutputInfo o;
    o.meta.name = "R" + std::to_string(r + 1);
    o.meta.dtype = e.args[r][0].dtype;
    for (const auto& a : e.args[r])
      if (feinsum::dtype_rank(a.dtype) > feinsum::dtype_rank(o.meta.dtype)) o.meta.dtype = a.dtype;
    for (const auto& s : e.i_out) o.meta.shape.push_back(lens.at(s));
    if (opt.storage == "wide")
      o.storage = p.complex_mode ? ST_C128 : ST_F64;
    else
      o.storage = native_storage(o.meta.dtype);
    p.outputs.push_back(o);
  }

  // costs
  const double row_flops = optimal_path_flops(e);
  p.alg_flops = row_flops * e.b();
  p.ref_flops = feinsum::flop_count(e);
  p.operand_flops = 0;
  if (p.functional)
    for (const auto& [name, op] : p.operand_exprs) {
      std::int64_t count = 1;
      for (const auto& row : e.args)
        for (const auto& a : row)
          if (a.name == name) count = a.num_elements();
      p.operand_flops += expr_ops(op.body) * static_cast<double>(count);
    }
  p.alg_flops += p.operand_flops;
  p.bytes = 0;
  for (const auto& L : p.leaves) p.bytes += static_cast<double>(L.bytes());
  for (const auto& o : p.outputs) p.bytes += static_cast<double>(o.bytes());

  // normal form + key (0-dim operands cannot be encoded: generic path)
  bool encodable = opt.canonicalize;
  for (const auto& a : feinsum::universe(e))
    if (a.dim() == 0) encodable = false;
  if (encodable) {
    // memo keyed by the exact spelling: repeated plans skip the search
    static std::mutex mu;
    static std::map<std::string, CanonResult> memo;
    const std::string spelling = fejson::dump(feinsum::transport::einsum_to_json(e));
    bool hit = false;
    {
      std::lock_guard<std::mutex> lock(mu);
      auto it = memo.find(spelling);
      if (it != memo.end()) {
        p.canon = it->second;
        hit = true;
      }
    }
    if (!hit) {
      p.canon = feinsum::canonicalize(e);
      std::lock_guard<std::mutex> lock(mu);
      if (memo.size() > 4096) memo.clear();
      memo.emplace(spelling, p.canon);
    }
    p.key = feinsum::detail::key_of_canonical(p.canon.canonical);
    p.has_canon = true;
  }

  // kernel choice: forced > fact > first matching family > generic
  std::vector<Family> order = {Family::fem_grad, Family::gett, Family::tt, Family::hex, Family::path};
  auto family_of = [](const std::string& t) -> std::optional<Family> {
    for (Family f : {Family::generic, Family::fem_grad, Family::gett, Family::tt, Family::hex, Family::path})
      if (t == family_transform(f)) return f;
    return std::nullopt;
  };
  std::string why;
  auto try_bind = [&](Family f) -> bool {
    if (!p.has_canon) return f == Family::generic;
    switch (f) {
      case Family::generic: return true;
      case Family::fem_grad: return bind_fem(p, &why);
      case Family::gett: return bind_gett(p, &why);
      case Family::tt: return bind_tt(p, &why);
      case Family::hex: return bind_hex(p, &why);
      case Family::path: return bind_path(p, opt, &why);
      default: return false;
    }
  };
  p.family = Family::generic;
  p.source = "fallback";
  if (!opt.force_transform.empty()) {
    auto f = family_of(opt.force_transform);
    if (!f) throw error(errc::usage, "unknown transform " + opt.force_transform);
    if (!try_bind(*f)) throw error(errc::usage, "transform " + opt.force_transform + " does not apply: " + why);
    p.family = *f;
    p.source = "forced";
  } else {
    std::optional<feinsum::FactRecord> fact;
    if (p.has_canon)
      fact = facts_index().best(opt.facts_path.empty() ? default_facts_path() : opt.facts_path, p.key, opt.device_id);
    if (fact) {
      auto f = family_of(fact->transform_id);
      if (f && try_bind(*f)) {
        p.family = *f;
        p.source = "fact";
        p.meta = fact->meta;
      }
    }
    if (p.source != "fact")
      for (Family f : order)
        if (try_bind(f)) {
          p.family = f;
          p.source = "default";
          break;
        }
  }
  p.transform = family_transform(p.family);
  if (!opt.meta_override.empty()) p.meta = opt.meta_override;
  // tabulated operands back to their programs: the generic kernel (and the
  // generated fem_grad instance) evaluate them in place, no tables
  auto drop_tabs = [&] {
    const size_t bn = static_cast<size_t>(e.b()) * e.n(), nl = p.leaves.size();
    for (size_t i = 0; i < bn; ++i)
      if (p.ops[i].kind == OPK_PLAIN && static_cast<size_t>(p.ops[i].leaf) >= nl)
        p.ops[i] = p.ops[static_cast<size_t>(p.tabs[static_cast<size_t>(p.ops[i].leaf) - nl].op)];
    p.ops.resize(bn);
    p.tabs.clear();
    p.tab_leaves.clear();
  };
  if (p.family == Family::generic && !p.tabs.empty()) drop_tabs();
  // fem_grad with operand programs or epilogues: one generated instance of the
  // kernel body (codegen.cpp) computes the programs in the prologue from the
  // staged leaf tiles and applies the epilogues before the stores
  if (p.family == Family::fem_grad && (!p.tabs.empty() || !p.epilogue.empty())) {
    const FemBinding& f = p.fem;
    int te = meta_int(p.meta, "te", f.NI == 10 ? 32 : (f.NI == 4 ? 64 : 16));
    int ept = meta_int(p.meta, "ept", 1);
    if (ept != 1 && ept != 2) ept = 1;
    if (te < 2 || te > 128 || te % 2 != 0 || te % ept != 0) te = f.NI == 10 ? 32 : (f.NI == 4 ? 64 : 16);
    const bool dsmem = ept == 1 && meta_int(p.meta, "dsmem", 0) != 0;
    std::vector<std::vector<int>> tiles;
    std::vector<int> aux;
    std::string why, log;
    if (!opt.codegen) {
      p.fem_rtc_note = "prebuilt: codegen disabled";
    } else {
      const std::string src = fem_rtc_source(p, te, ept, dsmem, &tiles, &aux, &why);
      void* kern = nullptr;
      bool compiled = false;
      if (!src.empty()) compiled = opt.dry_run ? nvrtc_compiles(src, &log)
                                               : (kern = compile_rtc_kernel(src, "fe_fem_rtc", &log)) != nullptr;
      if (src.empty()) {
        p.fem_rtc_note = "prebuilt: " + why;
      } else if (!compiled) {
        p.fem_rtc_note = "prebuilt: " + log.substr(0, 300);
      } else {
        p.fem_rtc = kern;
        p.fem_rtc_note = "nvrtc";
        p.fem_rtc_te = te;
        p.fem_rtc_ept = ept;
        p.fem_rtc_tiles = tiles;
        p.fem_rtc_aux = aux;
        for (size_t q = 0; q < tiles.size(); ++q) {
          p.fem.u_terms[q].clear();
          for (int leaf : tiles[q]) p.fem.u_terms[q].push_back(AffineTerm{1, -1, leaf, -1, -1});
        }
        drop_tabs();
      }
    }
  }
  // epilogue passes (every family; the generated fem_grad instance fuses
  // them, its runtime fallback to the generic kernel still needs them)
  if (!p.epilogue.empty()) {
    p.epi_pass.assign(static_cast<size_t>(e.b()), Plan::EpiPass{});
    for (int r = 0; r < e.b(); ++r) {
      if (p.epi_ops[static_cast<size_t>(r)].kind != OPK_VM) continue;
      Plan::EpiPass& ep = p.epi_pass[static_cast<size_t>(r)];
      const std::string src = epi_kernel_source(p, p.epi_ops[static_cast<size_t>(r)], p.outputs[static_cast<size_t>(r)].meta,
                                                p.outputs[static_cast<size_t>(r)].storage, &ep.leaf_slots);
      if (src.empty())
        throw error(errc::usage, "epilogue of row " + std::to_string(r) + ": output storage " +
                                     storage_name(p.outputs[static_cast<size_t>(r)].storage) +
                                     " or more than 16 arrays read");
      std::string log;
      const bool ok = opt.dry_run ? nvrtc_compiles(src, &log) : (ep.kernel = compile_rtc_kernel(src, "fe_epi", &log)) != nullptr;
      if (!ok) throw error(errc::io, "epilogue of row " + std::to_string(r) + " does not compile: " + log.substr(0, 300));
    }
  }

  // generic launch (always prepared: it is also the runtime fallback)
  std::vector<std::string> syms = e.i_out;
  for (auto& s : feinsum::reduction_indices(e)) syms.push_back(s);
  if (syms.size() > static_cast<size_t>(kMaxSyms)) throw error(errc::usage, "more than 32 distinct indices");
  GenericLaunch& g = p.gen;
  g = GenericLaunch{};
  g.n_syms = static_cast<int>(syms.size());
  g.n_out = static_cast<int>(e.i_out.size());
  g.b = e.b();
  g.n = e.n();
  g.out_points = 1;
  g.red_points = 1;
  for (size_t i = 0; i < syms.size(); ++i) {
    g.extent[i] = lens.at(syms[i]);
    (static_cast<int>(i) < g.n_out ? g.out_points : g.red_points) *= g.extent[i];
  }
  g.complex_mode = p.complex_mode;
  for (int r = 0; r < e.b(); ++r) g.out_storage[r] = p.outputs[r].storage;

  upload_tables(p, g, e, opt.dry_run);
  if (!opt.dry_run && p.family == Family::path && p.inter_bytes > 0)
    cuda_check(cudaMalloc(&p.d_inter, static_cast<size_t>(p.inter_bytes)), "cudaMalloc(path intermediates)");
  for (size_t k = 0; k < p.tabs.size(); ++k) {
    Plan::TabOperand& t = p.tabs[k];
    const std::string src = tab_kernel_source(p, p.ops[static_cast<size_t>(t.op)], p.tab_leaves[k].meta, &t.leaf_slots);
    std::string log;
    if (!opt.codegen)
      t.codegen = "vm: codegen disabled";
    else if (src.empty())
      t.codegen = "vm: program not expressible (f16 leaf or > 16 leaves)";
    else if (opt.dry_run)
      t.codegen = nvrtc_compiles(src, &log) ? "nvrtc" : "vm: " + log.substr(0, 200);
    else
      t.codegen = (t.kernel = compile_tab_kernel(src, &log)) != nullptr ? "nvrtc" : "vm: " + log.substr(0, 200);
  }
  if (!opt.dry_run && !p.tabs.empty()) {
    const Plan::TabOperand& last = p.tabs.back();
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&p.d_tab), sizeof(double) * static_cast<size_t>(last.offset + last.count)),
               "cudaMalloc(tabulated operands)");
  }
  if (!opt.dry_run && p.family == Family::gett) {
    bool affine = false;
    for (const auto& r : p.gett.rows) affine = affine || r.a_alpha >= 0 || r.b_alpha >= 0;
    if (affine) {
      const size_t n = static_cast<size_t>(p.gett.ext_mo * p.gett.ext_mi + p.gett.ext_no * p.gett.ext_ni);
      cuda_check(cudaMalloc(reinterpret_cast<void**>(&p.d_scratch), n * sizeof(double)), "cudaMalloc(gett scratch)");
    }
    const GettBinding& g = p.gett;
    if (g.pack_a)
      cuda_check(cudaMalloc(reinterpret_cast<void**>(&p.d_pack_a),
                            sizeof(double) * static_cast<size_t>(g.ext_mo * g.ext_mi * g.ext_ka * g.ext_kb * g.nz)),
                 "cudaMalloc(gett packed A)");
    if (g.pack_b)
      cuda_check(cudaMalloc(reinterpret_cast<void**>(&p.d_pack_b),
                            sizeof(double) * static_cast<size_t>(g.ext_no * g.ext_ni * g.ext_ka * g.ext_kb * g.nz)),
                 "cudaMalloc(gett packed B)");
    // split K when the output has too few 144 x 144 tiles to fill the SMs
    // (matmul 512^3: 16 tiles) — slices of the k steps run as separate tiles
    // and a second pass sums them in slice order (fact meta ks=N forces)
    {
      GettBinding& gm = p.gett;
      const std::int64_t tiles = (gm.ext_mo + 1) / 2 * ((gm.ext_no + 1) / 2) * gm.nz;
      const std::int64_t ksteps = (gm.ext_ka + 7) / 8 * ((gm.ext_kb + 3) / 4);
      const std::int64_t csize = gm.ext_mo * gm.ext_mi * gm.ext_no * gm.ext_ni * gm.nz;
      std::int64_t ks = 1;
      if (tiles * 2 <= p.sm_count) ks = std::min<std::int64_t>({16, p.sm_count / tiles, ksteps / 2});
      ks = meta_int(p.meta, "ks", static_cast<int>(ks));
      bool affine = false;
      for (const auto& r : gm.rows) affine = affine || r.a_alpha >= 0 || r.b_alpha >= 0;
      if (ks >= 2 && !affine && ks * csize <= (std::int64_t{1} << 27)) {
        gm.ksplit = static_cast<int>(ks);
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&p.d_ws), sizeof(double) * static_cast<size_t>(ks * csize)),
                   "cudaMalloc(gett split-K workspace)");
      }
    }
    if (g.c_f32)
      cuda_check(cudaMalloc(reinterpret_cast<void**>(&p.d_cbuf),
                            sizeof(double) * static_cast<size_t>(g.ext_mo * g.ext_mi * g.ext_no * g.ext_ni * g.nz)),
                 "cudaMalloc(gett f64 result)");
  }
  // plan-time uploads (tables, literal coefficients) are pageable copies on
  // the legacy stream; executes run on the caller's (possibly non-blocking)
  // stream, so the DMA must be complete before the plan is handed out
  if (!opt.dry_run && p.family == Family::hex) cuda_check(static_cast<cudaError_t>(hex_prepare(p.device)), "hex operator staging");
  // executes that write plan-owned scratch are ordered across streams by an
  // event (see execute), created here so the execute path never allocates
  if (!opt.dry_run && (p.d_tab || p.d_inter || p.d_scratch || p.d_pack_a || p.d_pack_b || p.d_cbuf || p.d_ws ||
                       (!p.chains.empty() && !p.coef_static)))
    cuda_check(cudaEventCreateWithFlags(&p.last_use, cudaEventDisableTiming), "cudaEventCreate(plan scratch)");
  if (!opt.dry_run) cuda_check(cudaStreamSynchronize(cudaStreamLegacy), "plan upload");
}

int leaf_storage_for(const ArrayMeta& m, const PlanOptions& opt) {
  auto it = opt.storage_of.find(m.name);
  if (it != opt.storage_of.end()) return storage_from_name(it->second);
  if (opt.storage == "wide") return is_complex_dtype(m.dtype) ? ST_C128 : ST_F64;
  return native_storage(m.dtype);
}

}  // namespace

Plan::~Plan() {
  if (d_blob) cudaFree(d_blob);
  if (d_coef) cudaFree(d_coef);
  if (d_scratch) cudaFree(d_scratch);
  if (d_pack_a) cudaFree(d_pack_a);
  if (d_pack_b) cudaFree(d_pack_b);
  if (d_cbuf) cudaFree(d_cbuf);
  if (d_ws) cudaFree(d_ws);
  if (last_use) cudaEventDestroy(last_use);
  if (d_tab) cudaFree(d_tab);
  if (d_inter) cudaFree(d_inter);
}

std::unique_ptr<Plan> make_plan(const BatchedEinsum& e, const PlanOptions& opt) {
  feinsum::require_valid(e);
  auto p = std::make_unique<Plan>();
  p->skel = e;
  for (const auto& m : feinsum::universe(e)) {
    LeafInfo L{m, leaf_storage_for(m, opt)};
    if (storage_complex(L.storage)) p->complex_mode = true;
    p->leaves.push_back(L);
  }
  std::map<std::string, int> leaf_of;
  for (size_t i = 0; i < p->leaves.size(); ++i) leaf_of[p->leaves[i].meta.name] = static_cast<int>(i);
  for (int r = 0; r < e.b(); ++r)
    for (int k = 0; k < e.n(); ++k) {
      OperandStatic s{};
      s.kind = OPK_PLAIN;
      s.leaf = leaf_of.at(e.args[r][k].name);
      s.ndim = e.args[r][k].dim();
      p->ops.push_back(s);
    }
  finish_plan(*p, opt);
  return p;
}

std::unique_ptr<Plan> make_functional_plan(const BatchedEinsum& skeleton,
                                           const std::map<std::string, OperandExpr>& operands,
                                           const std::map<std::string, ArrayMeta>& arrays, const PlanOptions& opt,
                                           const std::map<int, feinsum::RowEpilogue>& epilogue) {
  feinsum::require_valid(skeleton);
  auto p = std::make_unique<Plan>();
  p->skel = skeleton;
  p->functional = true;
  p->operand_exprs = operands;
  for (const auto& [name, m] : arrays) {
    LeafInfo L{m, leaf_storage_for(m, opt)};
    if (storage_complex(L.storage)) p->complex_mode = true;
    p->leaves.push_back(L);
  }
  OperandCompiler cc(*p);
  cc.force_vm = opt.force_vm;
  cc.skip_range_check = opt.skip_range_check;
  std::map<std::string, OperandStatic> compiled;
  for (const auto& m : feinsum::universe(skeleton)) {
    auto it = operands.find(m.name);
    if (it == operands.end()) throw error(errc::domain, "no operand expression for " + m.name);
    compiled[m.name] = cc.compile(it->second, m);
  }
  for (int r = 0; r < skeleton.b(); ++r)
    for (int k = 0; k < skeleton.n(); ++k) p->ops.push_back(compiled.at(skeleton.args[r][k].name));
  // row epilogues (extension): compiled against the row's output point
  p->epilogue = epilogue;
  if (!epilogue.empty()) {
    if (p->complex_mode) throw error(errc::usage, "epilogues need a real-valued plan");
    if (!opt.codegen) throw error(errc::usage, "epilogues run as generated code (option codegen: false given)");
    OperandStatic none{};
    none.kind = -1;
    p->epi_ops.assign(static_cast<size_t>(skeleton.b()), none);
    const auto lens = feinsum::index_lengths(skeleton);
    for (const auto& [row, ep] : epilogue) {
      if (row < 0 || row >= skeleton.b()) throw error(errc::domain, "epilogue for row " + std::to_string(row) + " of " +
                                                                          std::to_string(skeleton.b()));
      ArrayMeta out{ep.acc, {}, Dtype::float64};
      for (const auto& ix : skeleton.i_out) out.shape.push_back(lens.at(ix));
      p->epi_ops[static_cast<size_t>(row)] = cc.compile_epilogue(ep, out, ST_F64);
    }
  }
  // real-valued VM operands become tabulated leaves (Plan::tabs); finish_plan
  // drops them again if no tuned family binds
  constexpr std::int64_t kTabBudget = std::int64_t{1} << 30;  // doubles (8 GiB)
  if (!p->complex_mode && !opt.force_vm) {
    std::int64_t off = 0;
    for (const auto& m : feinsum::universe(skeleton)) {
      const OperandStatic c = compiled.at(m.name);
      if (c.kind != OPK_VM || m.dim() == 0) continue;
      if (p->leaves.size() + p->tabs.size() >= static_cast<size_t>(kMaxLeaves)) break;
      if (off + m.num_elements() > kTabBudget) break;
      const int leaf = static_cast<int>(p->leaves.size() + p->tabs.size());
      Plan::TabOperand tab;
      tab.name = m.name;
      tab.op = static_cast<int>(p->ops.size());
      tab.count = m.num_elements();
      tab.offset = off;
      p->tabs.push_back(std::move(tab));
      off += (m.num_elements() + 1) / 2 * 2;  // 16-byte aligned runs
      p->ops.push_back(c);
      ArrayMeta tm = m;
      tm.name = "tabulated " + m.name;
      tm.dtype = Dtype::float64;
      p->tab_leaves.push_back(LeafInfo{tm, ST_F64});
      OperandStatic plain{};
      plain.kind = OPK_PLAIN;
      plain.leaf = leaf;
      plain.ndim = m.dim();
      for (int r = 0; r < skeleton.b(); ++r)
        for (int k = 0; k < skeleton.n(); ++k)
          if (skeleton.args[r][k].name == m.name) p->ops[static_cast<size_t>(r) * skeleton.n() + k] = plain;
    }
  }
  finish_plan(*p, opt);
  return p;
}

namespace {
void execute_on(const Plan& plan, const void* const* d_in, void* const* d_out, void* stream, bool* epi_done);
// recursive: a path plan's execute holds its bucket while it executes its
// step plans, whose addresses can hash to the same bucket (a plain mutex
// self-deadlocked there, intermittently: 1 in 16 per step)
std::recursive_mutex g_scratch_mu[16];

// the rows' epilogues as in-place passes over the outputs (families that do
// not fuse them)
void run_epilogues(const Plan& plan, const void* const* d_in, void* const* d_out, void* stream) {
  for (size_t r = 0; r < plan.epi_pass.size(); ++r) {
    const Plan::EpiPass& ep = plan.epi_pass[r];
    if (!ep.kernel) continue;
    TabArgs args{};
    for (size_t k = 0; k < ep.leaf_slots.size(); ++k) args.leaf[k] = d_in[ep.leaf_slots[k]];
    args.out = static_cast<double*>(d_out[r]);
    args.count = plan.outputs[r].meta.num_elements();
    cuda_check(launch_tab_kernel(ep.kernel, args, plan.sm_count, stream), "generated epilogue kernel");
  }
}
}  // namespace

// Plans that own mutable device scratch (tabulated operands, path
// intermediates, GETT packs / K-sums / split-K workspace, per-execute
// coefficients) serialise their executes: each waits for the previous one, on
// whatever stream it ran, through the plan's last_use event. Plans without
// scratch run concurrently on any number of streams.
void execute(const Plan& plan, const void* const* d_in, void* const* d_out, void* stream) {
  bool epi_done = false;
  if (!plan.last_use) {
    execute_on(plan, d_in, d_out, stream, &epi_done);
    if (!epi_done) run_epilogues(plan, d_in, d_out, stream);
    return;
  }
  std::lock_guard<std::recursive_mutex> lock(g_scratch_mu[(reinterpret_cast<std::uintptr_t>(&plan) >> 6) & 15]);
  auto st = static_cast<cudaStream_t>(stream);
  cuda_check(cudaStreamWaitEvent(st, plan.last_use, 0), "plan scratch ordering");
  execute_on(plan, d_in, d_out, stream, &epi_done);
  if (!epi_done) run_epilogues(plan, d_in, d_out, stream);
  cuda_check(cudaEventRecord(plan.last_use, st), "plan scratch ordering");
}

namespace {
void execute_on(const Plan& plan, const void* const* d_in, void* const* d_out, void* stream, bool* epi_done) {
  const void* all_in[kMaxLeaves];
  const size_t nl = plan.leaves.size(), nt = plan.tabs.size();
  if (nt) {
    for (size_t i = 0; i < nl; ++i) all_in[i] = d_in[i];
    for (size_t k = 0; k < nt; ++k) all_in[nl + k] = plan.d_tab + plan.tabs[k].offset;
    d_in = all_in;
  }
  GenericLaunch g = plan.gen;
  for (size_t i = 0; i < nl + nt; ++i) {
    g.leaves.ptr[i] = d_in[i];
    g.leaves.storage[i] = leaf_info(plan, static_cast<int>(i)).storage;
  }
  for (int r = 0; r < plan.skel.b(); ++r) g.out[r] = d_out[r];
  if (!plan.chains.empty() && !plan.coef_static)
    cuda_check(launch_coef(g.chains, g.n_chains, g.leaves, plan.d_coef, stream), "coefficient kernel");
  for (const Plan::TabOperand& tab : plan.tabs) {
    if (tab.kernel) {
      TabArgs args{};
      for (size_t k = 0; k < tab.leaf_slots.size(); ++k) args.leaf[k] = g.leaves.ptr[tab.leaf_slots[k]];
      args.out = plan.d_tab + tab.offset;
      args.count = tab.count;
      cuda_check(launch_tab_kernel(tab.kernel, args, plan.sm_count, stream), "generated tabulation kernel");
      continue;
    }
    TabulateLaunch t{};
    t.op = plan.gen.ops + tab.op;
    t.prog = plan.gen.prog;
    t.reads = plan.gen.reads;
    t.chains = plan.gen.chains;
    t.n_chains = plan.gen.n_chains;
    t.coef = plan.d_coef;
    const ArrayMeta& m = plan.tab_leaves[static_cast<size_t>(&tab - plan.tabs.data())].meta;
    t.ndim = m.dim();
    for (int d = 0; d < m.dim(); ++d) t.shape[d] = m.shape[d];
    t.first = 0;
    t.count = tab.count;
    t.complex_mode = false;
    t.leaves = g.leaves;
    t.out = plan.d_tab + tab.offset;
    t.real_out = true;
    cuda_check(launch_tabulate(t, stream), "tabulate kernel");
  }

  if (plan.family == Family::path) {
    auto inter = [&](int id) { return static_cast<unsigned char*>(plan.d_inter) + plan.inter_off[static_cast<size_t>(id)]; };
    for (const PathStep& st : plan.path) {
      std::vector<const void*> in;
      for (int src : st.src) in.push_back(src >= 0 ? d_in[src] : inter(-src - 1));
      void* out = st.out < 0 ? d_out[st.out_row] : inter(st.out);
      execute(*st.plan, in.data(), &out, stream);
    }
    return;
  }
  if (plan.family == Family::fem_grad) {
    const FemBinding& f = plan.fem;
    FemGradLaunch L{};
    L.rows = f.rows;
    L.E = f.E;
    L.NX = f.NX;
    L.NR = f.NR;
    L.NI = f.NI;
    L.NJ = f.NJ;
    L.stages = meta_int(plan.meta, "stages", 4);
    L.d_in_smem = meta_int(plan.meta, "dsmem", 0) != 0;
    std::vector<int> jl, dl;
    bool ok = true;
    int u = 0;
    L.plain_u = true;
    for (int q = 0; q < f.rows; ++q) {
      auto idx_of = [](std::vector<int>& v, int leaf) {
        auto it = std::find(v.begin(), v.end(), leaf);
        if (it != v.end()) return static_cast<int>(it - v.begin());
        v.push_back(leaf);
        return static_cast<int>(v.size()) - 1;
      };
      L.row_j[q] = idx_of(jl, f.j_leaf[q]);
      L.row_d[q] = idx_of(dl, f.d_leaf[q]);
      L.row_u_first[q] = u;
      L.row_u_count[q] = static_cast<int>(f.u_terms[q].size());
      if (f.u_terms[q].size() != 1 || f.u_terms[q][0].pre >= 0 || f.u_terms[q][0].post0 >= 0) L.plain_u = false;
      for (const AffineTerm& t : f.u_terms[q]) {
        L.U[u] = static_cast<const double*>(d_in[t.leaf]);
        L.u_sign[u] = t.sign;
        L.u_pre[u] = t.pre;
        L.u_post[u] = t.post0;
        ok = ok && aligned16(L.U[u]);
        ++u;
      }
      L.Y[q] = static_cast<double*>(d_out[f.out_row[q]]);
    }
    L.n_u = u;
    L.n_j = static_cast<int>(jl.size());
    L.n_d = static_cast<int>(dl.size());
    for (size_t a = 0; a < jl.size(); ++a) {
      L.J[a] = static_cast<const double*>(d_in[jl[a]]);
      ok = ok && aligned16(L.J[a]);
    }
    for (size_t a = 0; a < dl.size(); ++a) L.D[a] = static_cast<const double*>(d_in[dl[a]]);
    L.coef = plan.d_coef;
    L.tile_e = meta_int(plan.meta, "te", f.NI == 10 ? 32 : (f.NI == 4 ? 64 : 16));
    L.grid = meta_int(plan.meta, "grid", 0);  // 0: all resident CTAs
    L.ept = meta_int(plan.meta, "ept", 1);
    L.f32 = f.f32;
    L.mma = !f.f32 && meta_int(plan.meta, "mma", 0) != 0 && fem_mma_supported(L.NX, L.NR, L.NI, L.NJ);
    if (ok && plan.fem_rtc) {
      // generated instance: staged tiles per row as generated, aux reads
      int t = 0;
      for (int q = 0; q < f.rows; ++q) {
        L.row_u_first[q] = t;
        L.row_u_count[q] = static_cast<int>(plan.fem_rtc_tiles[static_cast<size_t>(q)].size());
        for (int leaf : plan.fem_rtc_tiles[static_cast<size_t>(q)]) {
          L.U[t] = static_cast<const double*>(d_in[leaf]);
          L.u_sign[t] = 1;
          L.u_pre[t] = L.u_post[t] = -1;
          ok = ok && aligned16(L.U[t]);
          ++t;
        }
      }
      L.n_u = t;
      L.plain_u = false;
      for (size_t k = 0; k < plan.fem_rtc_aux.size(); ++k) L.aux[k] = d_in[plan.fem_rtc_aux[k]];
      if (L.stages < 2) L.stages = 2;  // the pipelined prologue reads one stage ahead
      if (ok) {
        cuda_check(launch_fem_grad_rtc(L, plan.fem_rtc, plan.fem_rtc_te, plan.fem_rtc_ept, stream),
                   "generated fem_grad kernel");
        *epi_done = true;
        return;
      }
    } else if (ok) {
      if (L.mma)
        cuda_check(launch_fem_mma(L, stream), "fem_mma kernel");
      else
        cuda_check(launch_fem_grad(L, stream), "fem_grad kernel");
      return;
    }
  }
  if (plan.family == Family::gett) {
    const GettBinding& b = plan.gett;
    bool ok = true;
    for (const auto& r : b.rows) ok = ok && aligned16(d_in[r.a_leaf]) && aligned16(d_in[r.b_leaf]);
    if (ok) {
      for (const auto& r : b.rows) {
        GettLaunch L{};
        L.ext_mo = b.ext_mo;
        L.ext_mi = b.ext_mi;
        L.ext_no = b.ext_no;
        L.ext_ni = b.ext_ni;
        L.ext_ka = b.ext_ka;
        L.ext_kb = b.ext_kb;
        L.a_mo = b.a_mo;
        L.a_mi = b.a_mi;
        L.a_kb = b.a_kb;
        L.b_no = b.b_no;
        L.b_ni = b.b_ni;
        L.b_ka = b.b_ka;
        L.c_mo = b.c_mo;
        L.c_mi = b.c_mi;
        L.c_no = b.c_no;
        L.c_ni = b.c_ni;
        L.A = static_cast<const double*>(d_in[r.a_leaf]);
        L.B = static_cast<const double*>(d_in[r.b_leaf]);
        if (b.pack_a) {
          const std::int64_t ext[4] = {b.ext_mo, b.ext_mi, b.ext_kb, b.ext_ka};
          cuda_check(b.a_f32 ? permute4_widen(static_cast<const float*>(d_in[r.a_leaf]), plan.d_pack_a, ext, b.a_src, stream,
                                              b.nz, b.a_z_src)
                             : permute4(L.A, plan.d_pack_a, ext, b.a_src, stream, b.nz, b.a_z_src),
                     "gett pack A");
          L.A = plan.d_pack_a;
        }
        if (b.pack_b) {
          const std::int64_t ext[4] = {b.ext_no, b.ext_ni, b.ext_ka, b.ext_kb};
          cuda_check(b.b_f32 ? permute4_widen(static_cast<const float*>(d_in[r.b_leaf]), plan.d_pack_b, ext, b.b_src, stream,
                                              b.nz, b.b_z_src)
                             : permute4(L.B, plan.d_pack_b, ext, b.b_src, stream, b.nz, b.b_z_src),
                     "gett pack B");
          L.B = plan.d_pack_b;
        }
        L.C = b.c_f32 ? plan.d_cbuf : static_cast<double*>(d_out[r.out_row]);
        L.nz = b.nz;
        L.a_z = b.a_z;
        L.b_z = b.b_z;
        L.c_z = b.c_z;
        L.ksplit = b.ksplit;
        L.ws = plan.d_ws;
        L.a_alpha = r.a_alpha;
        L.a_beta = r.a_beta;
        L.b_alpha = r.b_alpha;
        L.b_beta = r.b_beta;
        L.coef = plan.d_coef;
        L.scratch = plan.d_scratch;
        L.stages = meta_int(plan.meta, "stages", 3);
        L.group = meta_int(plan.meta, "group", 12);
        L.grid = meta_int(plan.meta, "grid", 0);
        cuda_check(launch_gett(L, stream), "gett kernel");
        if (b.c_f32)
          cuda_check(narrow_f64_f32(plan.d_cbuf, static_cast<float*>(d_out[r.out_row]),
                                    b.ext_mo * b.ext_mi * b.ext_no * b.ext_ni * b.nz, stream),
                     "gett narrow C");
      }
      return;
    }
  }
  if (plan.family == Family::hex) {
    const HexBinding& h = plan.hex;
    bool ok = aligned16(d_in[h.g]);
    for (int u : h.u) ok = ok && aligned16(d_in[u]);
    if (ok) {
      HexLaunch L{};
      L.E = h.E;
      L.ND = h.ND;
      L.P = h.P;
      L.rows = static_cast<int>(h.u.size());
      L.variant = meta_int(plan.meta, "v", 2);
      L.f32 = h.f32;
      L.ne = meta_int(plan.meta, "ne", 4);
      for (int k = 0; k < 6; ++k) L.mats[k] = static_cast<const double*>(d_in[h.mats[k]]);
      L.G = static_cast<const double*>(d_in[h.g]);
      for (size_t q = 0; q < h.u.size(); ++q) {
        L.U[q] = static_cast<const double*>(d_in[h.u[q]]);
        L.Y[q] = static_cast<double*>(d_out[h.out_row[q]]);
      }
      cuda_check(launch_hex(L, stream), "hex kernel");
      return;
    }
  }
  if (plan.family == Family::tt) {
    const TTBinding& b = plan.tt;
    bool ok = true;
    for (const auto& r : b.rows) ok = ok && aligned16(d_in[r.x]) && aligned16(d_out[r.out_row]);
    if (ok) {
      for (const auto& r : b.rows) {
        TTLaunch L{};
        L.Nb = b.nb;
        L.NI = b.NI;
        L.NJ = b.NJ;
        L.NK = b.NK;
        L.NL = b.NL;
        L.fp32 = b.fp32 ? 1 : 0;
        L.G1 = d_in[r.g1];
        L.G2 = d_in[r.g2];
        L.X = d_in[r.x];
        L.Y = d_out[r.out_row];
        L.x_sj = b.NL;
        L.x_sn = static_cast<std::int64_t>(b.NJ) * b.NL;
        L.y_sn = static_cast<std::int64_t>(b.NI) * b.NK;
        L.stages = meta_int(plan.meta, "stages", 2);
        if (L.fp32 && meta_int(plan.meta, "tc", 0) != 0 && tt_tc_supported(L))
          cuda_check(launch_tt_tc(L, stream), "tt tcgen05 kernel");
        else
          cuda_check(launch_tt(L, stream), "tt kernel");
      }
      return;
    }
  }
  cuda_check(launch_generic(g, stream), "generic kernel");
}
}  // namespace

void tabulate(const Plan& plan, const std::string& name, const void* const* d_in, double* d_out, std::int64_t first,
              std::int64_t count, void* stream) {
  const auto& e = plan.skel;
  int row = -1, slot = -1;
  ArrayMeta meta;
  for (int r = 0; r < e.b() && row < 0; ++r)
    for (int k = 0; k < e.n(); ++k)
      if (e.args[r][k].name == name) {
        row = r;
        slot = k;
        meta = e.args[r][k];
        break;
      }
  if (row < 0) throw error(errc::domain, "no operand named " + name);
  TabulateLaunch t{};
  t.op = plan.gen.ops + (static_cast<size_t>(row) * e.n() + slot);
  for (const Plan::TabOperand& tab : plan.tabs)
    if (tab.name == name) t.op = plan.gen.ops + tab.op;  // the VM original, not its table
  t.prog = plan.gen.prog;
  t.reads = plan.gen.reads;
  t.chains = plan.gen.chains;
  t.n_chains = plan.gen.n_chains;
  t.coef = plan.d_coef;
  t.ndim = meta.dim();
  for (int d = 0; d < meta.dim(); ++d) t.shape[d] = meta.shape[d];
  t.first = first;
  t.count = count;
  t.complex_mode = plan.complex_mode;
  for (size_t i = 0; i < plan.leaves.size(); ++i) {
    t.leaves.ptr[i] = d_in[i];
    t.leaves.storage[i] = plan.leaves[i].storage;
  }
  t.out = d_out;
  if (!plan.chains.empty() && !plan.coef_static)
    cuda_check(launch_coef(t.chains, t.n_chains, t.leaves, plan.d_coef, stream), "coefficient kernel");
  cuda_check(launch_tabulate(t, stream), "tabulate kernel");
}

std::string describe(const Plan& p) {
  using fejson::Value;
  Value v = Value::obj();
  v.set("key", Value::str(p.key));
  v.set("transform", Value::str(p.transform));
  v.set("source", Value::str(p.source));
  v.set("meta", Value::str(p.meta));
  v.set("functional", Value::boolean_(p.functional));
  v.set("complex", Value::boolean_(p.complex_mode));
  // the arithmetic pipe the chosen kernel issues to (roofline denominator)
  const char* pipe = "fma";
  switch (p.family) {
    case Family::fem_grad: pipe = meta_int(p.meta, "mma", 0) ? "dmma" : "dfma"; break;
    case Family::gett: pipe = "dmma"; break;
    case Family::tt: pipe = (p.tt.fp32 && meta_int(p.meta, "tc", 0)) ? "tcgen05_tf32x3" : "dmma"; break;
    case Family::hex: pipe = "dfma"; break;
    case Family::path: pipe = "dmma"; break;
    case Family::generic: pipe = "fma"; break;
  }
  v.set("pipe", Value::str(pipe));
  // kernels one execute launches (tuned path, aligned buffers): the family's
  // kernel per row where it loops over rows, plus the coefficient kernel and
  // GETT's operand passes (row sums for alpha*X+beta, repacks)
  int launches = p.chains.empty() || p.coef_static ? 0 : 1;
  switch (p.family) {
    case Family::fem_grad: launches += 1; break;
    case Family::hex: launches += (meta_int(p.meta, "v", 2) == 1 && p.hex.P == 5) ? 1 : 2; break;  // v2: + operator gather
    case Family::tt: launches += static_cast<int>(p.tt.rows.size()); break;
    case Family::gett:
      for (const auto& r : p.gett.rows) {
        launches += 1 + (p.gett.pack_a ? 1 : 0) + (p.gett.pack_b ? 1 : 0) + (p.gett.c_f32 ? 1 : 0) +
                    (p.gett.ksplit > 1 ? 1 : 0);
        if (r.a_alpha >= 0 || r.b_alpha >= 0) launches += 2;
      }
      break;
    case Family::generic: launches += 1; break;
    case Family::path:
      for (const auto& st : p.path) {
        const std::string d = describe(*st.plan);
        const auto at = d.find("\"launches\":");
        if (at != std::string::npos) launches += std::atoi(d.c_str() + at + 11);
      }
      break;
  }
  launches += static_cast<int>(p.tabs.size());
  const bool epi_fused = p.fem_rtc_note == "nvrtc";
  if (!epi_fused)
    for (const auto& op : p.epi_ops) launches += op.kind == OPK_VM ? 1 : 0;
  v.set("launches", Value::num(launches));
  // extension: row epilogues and the generated fem_grad instance
  Value erows = Value::arr();
  for (const auto& [row, ep] : p.epilogue) erows.push(Value::num(row));
  v.set("epilogue_rows", std::move(erows));
  v.set("epilogue_fused", Value::boolean_(epi_fused && !p.epilogue.empty()));
  if (!p.fem_rtc_note.empty()) v.set("fem_codegen", Value::str(p.fem_rtc_note));
  Value tabs = Value::arr();
  Value gens = Value::arr();
  for (const auto& t : p.tabs) {
    tabs.push(Value::str(t.name));
    gens.push(Value::str(t.codegen));
  }
  v.set("tabulated", std::move(tabs));
  v.set("tab_codegen", std::move(gens));
  Value leaves = Value::arr();
  for (const auto& L : p.leaves) {
    Value x = feinsum::transport::meta_to_json(L.meta);
    x.set("storage", Value::str(storage_name(L.storage)));
    x.set("bytes", Value::num(L.bytes()));
    leaves.push(std::move(x));
  }
  v.set("inputs", std::move(leaves));
  Value outs = Value::arr();
  for (const auto& o : p.outputs) {
    Value x = feinsum::transport::meta_to_json(o.meta);
    x.set("storage", Value::str(storage_name(o.storage)));
    x.set("bytes", Value::num(o.bytes()));
    outs.push(std::move(x));
  }
  v.set("outputs", std::move(outs));
  v.set("algorithmic_flops", Value::dbl(p.alg_flops));
  v.set("operand_flops", Value::dbl(p.operand_flops));
  v.set("reference_flops", Value::dbl(p.ref_flops));
  v.set("bytes", Value::dbl(p.bytes));
  if (p.has_canon) {
    Value c = Value::obj();
    c.set("canonical", feinsum::transport::einsum_to_json(p.canon.canonical));
    c.set("sigma_idx", feinsum::transport::strmap_to_json(p.canon.sigma_idx));
    c.set("sigma_arg", feinsum::transport::strmap_to_json(p.canon.sigma_arg));
    c.set("sigma_row", feinsum::transport::ints_to_json(p.canon.sigma_row));
    c.set("sigma_slot", feinsum::transport::ints_to_json(p.canon.sigma_slot));
    v.set("canon", std::move(c));
  }
  if (p.family == Family::fem_grad) {
    Value f = Value::obj();
    f.set("NX", Value::num(p.fem.NX));
    f.set("NR", Value::num(p.fem.NR));
    f.set("NI", Value::num(p.fem.NI));
    f.set("NJ", Value::num(p.fem.NJ));
    f.set("E", Value::num(p.fem.E));
    v.set("roles", std::move(f));
  }
  if (p.family == Family::gett) {
    Value f = Value::obj();
    f.set("roles", Value::str(p.gett.role_names));
    f.set("tile", Value::str("144x144x32, 12 DMMA warps + 1 TMA warpgroup"));
    v.set("roles", std::move(f));
  }
  return fejson::dump(v);
}

namespace {

// Canonical index each family shards along (element / batch / outer-M axis).
std::string shard_index_of(const Plan& p) {
  const BatchedEinsum& c = p.canon.canonical;
  auto role = [&](const std::vector<std::string>& in, const std::string& out, char r) -> std::string {
    const auto m = match_roles(c, in, out);
    return m ? p.canon.sigma_idx.at(m->idx.at(r)) : std::string();
  };
  switch (p.family) {
    case Family::fem_grad: return role({"xre", "xij", "ej"}, "rei", 'e');
    case Family::tt: return role({"ij", "kl", "njl"}, "nik", 'n');
    case Family::hex:
      return role({"xai", "xbm", "xcn", "xyeabc", "yaj", "ybk", "ycl", "ejkl"}, "eimn", 'e');
    case Family::gett:
      // the outer M index (4-index form: mo; split form: the M group's first)
      return p.canon.sigma_idx.at(p.gett.shard_m);
    case Family::generic:
    case Family::path: break;
  }
  return p.skel.i_out.empty() ? std::string() : p.skel.i_out[0];
}

}  // namespace

int pipe_chunks(const Plan& p, int dflt) {
  if (p.family != Family::gett || p.gett.role_names.rfind("mo=", 0) != 0) return dflt;
  // GETT (4-index form, shards along mo): wave quantisation of each chunk's
  // launch dominates — C3 in 8 chunks of 9 mo is 180 tiles = 2 waves on 148
  // SMs, in 9 chunks of 8 mo 144 tiles = one. Pick the chunk count whose
  // chunks fill whole waves best (ties: closest to the default).
  const std::int64_t n = p.gett.ext_mo, no_tiles = (p.gett.ext_no + 1) / 2;
  const int sms = p.sm_count > 0 ? p.sm_count : 148;
  int best = dflt;
  double best_score = -1.0;
  for (int c = 3; c <= 16 && c <= n; ++c) {
    const std::int64_t mo_c = (n + c - 1) / c;
    const std::int64_t tiles = (mo_c + 1) / 2 * no_tiles;
    const std::int64_t waves = (tiles + sms - 1) / sms;
    const double score = static_cast<double>(tiles) / static_cast<double>(waves * sms) - 0.005 * std::abs(c - dflt);
    if (score > best_score) {
      best_score = score;
      best = c;
    }
  }
  return best;
}

std::unique_ptr<Plan> make_shard(const Plan& full, int rank, int world, const PlanOptions& opt, std::int64_t* lo,
                                 std::int64_t* hi, std::string* axis) {
  if (world < 1 || rank < 0 || rank >= world) throw error(errc::usage, "shard: need 0 <= rank < world");
  const std::string ix = shard_index_of(full);
  if (ix.empty()) throw error(errc::usage, "this einsum has no output index to shard along");
  const auto lens = feinsum::index_lengths(full.skel);
  const std::int64_t n = lens.at(ix);
  // fem_grad moves elements in pairs (16-byte bulk-copy runs); hex in stages
  // of four when the axis allows it (the four-element kernel), else pairs
  std::int64_t unit = 1;
  if (full.family == Family::fem_grad) unit = full.fem.f32 ? 4 : 2;  // fp32: 16-byte bulk-copy rows
  if (full.family == Family::hex) unit = lens.at(ix) % 4 == 0 ? 4 : 2;
  const std::int64_t units = n / unit;
  std::int64_t a = units * rank / world * unit, b = units * (rank + 1) / world * unit;
  if (rank == world - 1) b = n;
  if (b <= a) throw error(errc::usage, "shard: axis " + ix + " (" + std::to_string(n) + ") is too short for " +
                                           std::to_string(world) + " ranks");
  *lo = a;
  *hi = b;
  *axis = ix;

  // the same einsum with the axis restricted to [a, b)
  BatchedEinsum e = full.skel;
  for (auto& row : e.args)
    for (int k = 0; k < e.n(); ++k)
      for (size_t d = 0; d < e.i_in[k].size(); ++d)
        if (e.i_in[k][d] == ix) row[k].shape[d] = b - a;
  if (!feinsum::validate(e).empty())
    throw error(errc::usage, "shard: an array is read both along and across axis " + ix);

  PlanOptions o = opt;
  o.force_transform = full.transform;
  std::unique_ptr<Plan> s;
  if (!full.functional) {
    s = make_plan(e, o);
  } else {
    // slice each leaf on the axes its reads bind to sharded operand axes
    std::map<std::string, ArrayMeta> arrays;
    for (const auto& L : full.leaves) arrays[L.meta.name] = L.meta;
    std::map<std::string, std::vector<bool>> sliced;  // leaf -> axes
    for (const auto& m : feinsum::universe(full.skel)) {
      std::vector<bool> op_axis(static_cast<size_t>(m.dim()), false);
      for (int k = 0; k < full.skel.n(); ++k)
        for (const auto& row : full.skel.args)
          if (row[k].name == m.name)
            for (size_t d = 0; d < full.skel.i_in[k].size(); ++d) op_axis[d] = op_axis[d] || full.skel.i_in[k][d] == ix;
      const OperandExpr& op = full.operand_exprs.at(m.name);
      std::function<void(const Expr&)> walk = [&](const Expr& x) {
        for (const Expr& c : x.children) walk(c);
        if (x.kind != Expr::Kind::access) return;
        auto& flags = sliced[x.name];
        flags.resize(x.subs.size(), false);
        for (size_t d = 0; d < x.subs.size(); ++d) {
          const auto pit = std::find(op.params.begin(), op.params.end(), x.subs[d]);
          const size_t pk = static_cast<size_t>(pit - op.params.begin());
          if (pk < op_axis.size() && op_axis[pk]) flags[d] = true;
        }
      };
      walk(op.body);
    }
    // epilogue reads: subscripts are output indices, sliced where they are the axis
    for (const auto& [row, ep] : full.epilogue) {
      std::function<void(const Expr&)> walk = [&](const Expr& x) {
        for (const Expr& c : x.children) walk(c);
        if (x.kind != Expr::Kind::access || x.name == ep.acc) return;
        auto& flags = sliced[x.name];
        flags.resize(x.subs.size(), false);
        for (size_t d = 0; d < x.subs.size(); ++d) flags[d] = flags[d] || x.subs[d] == ix;
      };
      walk(ep.op.body);
    }
    for (auto& [name, flags] : sliced) {
      auto& meta = arrays.at(name);
      for (size_t d = 0; d < flags.size(); ++d)
        if (flags[d]) {
          if (meta.shape[d] != n) throw error(errc::usage, "shard: array " + name + " is not aligned with " + ix);
          meta.shape[d] = b - a;
        }
    }
    s = make_functional_plan(e, full.operand_exprs, arrays, o, full.epilogue);
  }
  s->meta = full.meta;
  s->source = "shard of " + full.source + " plan " + full.key;
  return s;
}

}  // namespace feb200
