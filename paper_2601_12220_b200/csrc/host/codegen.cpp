// Tabulation kernels generated per operand program and compiled at plan time
// with NVRTC for sm_100a (functional operands as GPU
// code, not an interpreter).
//
// A real-valued VM operand (Plan::tabs) is tabulated at the start of every
// execute. The device VM (operand.cuh, eval_vm_real) interprets the program per
// element — instruction fetch, dispatch, run-time index decomposition — which
// costs ~5x the arithmetic. Here the same program is emitted as straight-line
// CUDA C: compile-time shapes (index decomposition by constant division),
// compile-time read strides, one local per VM register, and exactly the VM's
// rounding (__dadd_rn / __dmul_rn / __ddiv_rn, libdevice sin / cos / exp,
// -fmad=false), so the values are bit-identical to the VM's and therefore to
// the reference's materialize (proj/src/raising.cpp:336-393) for finite data.
//
// NVRTC is loaded with dlopen (no link-time dependency); the cubin is loaded
// context-independently with cudaLibraryLoadData and launched through
// cudaLaunchKernel. Anything unsupported (f16 leaves, > 16 leaves read, NVRTC
// missing, a compile error) leaves the operand on the VM tabulation kernel.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "planner.hpp"

namespace feb200 {

extern const int kRtcHeaderCount;
extern const char* const kRtcHeaderNames[];
extern const char* const kRtcHeaderSources[];

namespace {

struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  bool ok = false;
};

const Nvrtc& nvrtc() {
  static Nvrtc n = [] {
    Nvrtc r;
    void* h = nullptr;
    for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_GLOBAL)) != nullptr) break;
    if (!h) return r;
    r.create = reinterpret_cast<decltype(r.create)>(dlsym(h, "nvrtcCreateProgram"));
    r.compile = reinterpret_cast<decltype(r.compile)>(dlsym(h, "nvrtcCompileProgram"));
    r.log_size = reinterpret_cast<decltype(r.log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
    r.log = reinterpret_cast<decltype(r.log)>(dlsym(h, "nvrtcGetProgramLog"));
    r.cubin_size = reinterpret_cast<decltype(r.cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
    r.cubin = reinterpret_cast<decltype(r.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
    r.destroy = reinterpret_cast<decltype(r.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
    r.ok = r.create && r.compile && r.log_size && r.log && r.cubin_size && r.cubin && r.destroy;
    return r;
  }();
  return n;
}

std::string hexlit(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%a", v);
  return std::string("(") + buf + ")";
}

// element read through pointer expression `base` at offset expression `off`, as double
std::string load_expr(int st, const std::string& base, const std::string& off) {
  const std::string& p = base;
  switch (st) {
    case ST_F64: return "__ldg((const double*)" + p + " + (" + off + "))";
    case ST_F32: return "(double)__ldg((const float*)" + p + " + (" + off + "))";
    case ST_C128: return "__ldg((const double*)" + p + " + 2 * (" + off + "))";
    case ST_C64: return "(double)__ldg((const float*)" + p + " + 2 * (" + off + "))";
    case ST_I8: return "(double)((const signed char*)" + p + ")[" + off + "]";
    case ST_I32: return "(double)__ldg((const int*)" + p + " + (" + off + "))";
    case ST_I64: return "(double)__ldg((const long long*)" + p + " + (" + off + "))";
    default: return "";
  }
}

std::string read_offset(const VmRead& rd) {
  std::string off = "0LL";
  for (int d = 0; d < rd.ndim; ++d)
    off += " + p" + std::to_string(rd.param_of[d]) + " * " + std::to_string(rd.stride[d]) + "LL";
  return off;
}

// slot of `leaf` in `slots` (appended if new; -1 past `cap`)
int slot_of(std::vector<int>* slots, int leaf, int cap) {
  for (size_t k = 0; k < slots->size(); ++k)
    if ((*slots)[k] == leaf) return static_cast<int>(k);
  if (slots->size() >= static_cast<size_t>(cap)) return -1;
  slots->push_back(leaf);
  return static_cast<int>(slots->size()) - 1;
}

// Straight-line CUDA for the VM program of `op`: one double local per VM
// register and exactly the VM's rounding. Operand parameter k is the local
// p<k> (declared by the caller); `read` renders a leaf read as a double
// expression ("" = unsupported). The value ends in r0. False if unsupported.
// fast: exp / sin / cos as fastmath.cuh's range-unchecked straight-line forms,
// each argument's range test and-ed into the caller's `fe_ok` (the caller
// re-evaluates with the checked forms when it is false: same values where
// the fast form applies, so the result never depends on the variant).
bool emit_program(const Plan& p, const OperandStatic& op, const std::function<std::string(const VmRead&)>& read,
                  const std::string& ind, std::ostringstream& s, bool fast = false) {
  s << ind << "double r0 = 0.0";
  for (int r = 1; r < kMaxVmRegs; ++r) s << ", r" << r << " = 0.0";
  s << ";\n";
  for (int pc = op.prog_off; pc < op.prog_off + op.prog_len; ++pc) {
    const VmInstr& in = p.prog[static_cast<size_t>(pc)];
    const std::string dst = "r" + std::to_string(in.dst & (kMaxVmRegs - 1));
    const std::string a = "r" + std::to_string(in.a & (kMaxVmRegs - 1));
    const std::string b = "r" + std::to_string(in.b & (kMaxVmRegs - 1));
    std::string v;
    switch (in.code) {
      case VM_LIT: v = hexlit(in.imm); break;
      case VM_PARAM: v = "(double)p" + std::to_string(in.arg); break;
      case VM_READ:
        v = read(p.reads[static_cast<size_t>(in.arg)]);
        if (v.empty()) return false;
        break;
      case VM_ADD: v = "__dadd_rn(" + a + ", " + b + ")"; break;
      case VM_SUB: v = "__dsub_rn(" + a + ", " + b + ")"; break;
      case VM_MUL: v = "__dmul_rn(" + a + ", " + b + ")"; break;
      case VM_DIV: v = "__ddiv_rn(" + a + ", " + b + ")"; break;
      case VM_SIN:
      case VM_COS:
      case VM_EXP: {
        const char* fn = in.code == VM_SIN ? "sin" : in.code == VM_COS ? "cos" : "exp";
        if (fast) {
          s << ind << "fe_ok = fe_ok & feb200::fe_" << (in.code == VM_EXP ? "exp" : "trig") << "_ok(" << a << ");\n";
          v = std::string("feb200::fe_") + fn + "_fast(" + a + ")";
        } else {
          v = std::string("feb200::fe_") + fn + "(" + a + ")";
        }
        break;
      }
      case VM_RECIP: v = "__ddiv_rn(1.0, " + a + ")"; break;
      default: return false;  // sqrt: complex plans only
    }
    s << ind << dst << " = " << v << ";\n";
  }
  return true;
}

// p<k> locals: row-major decomposition of flat index `t` over `shape`
void emit_decompose(const std::vector<std::int64_t>& shape, const std::string& t, const std::string& ind,
                    std::ostringstream& s) {
  const int nd = static_cast<int>(shape.size());
  s << ind << "long long rem = " << t << ";\n";
  for (int d = nd - 1; d >= 1; --d)
    s << ind << "const long long p" << d << " = rem % " << shape[d] << "LL; rem /= " << shape[d] << "LL;\n";
  if (nd >= 1) s << ind << "const long long p0 = rem;\n";
  s << ind << "(void)rem;\n";
}

}  // namespace

// Source of the tabulation kernel for one operand, or "" if unsupported.
// `leaf_slots` receives the plan leaf index of each kernel leaf slot.
std::string tab_kernel_source(const Plan& p, const OperandStatic& op, const ArrayMeta& meta,
                              std::vector<int>* leaf_slots) {
  std::ostringstream s;
  s << "#include \"fastmath.cuh\"\nstruct TabArgs { const void* leaf[" << kTabLeaves << "]; double* out; long long count; };\n"
    << "extern \"C\" __global__ void __launch_bounds__(256) fe_tab(const TabArgs a) {\n"
    << "  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < a.count;\n"
    << "       t += (long long)gridDim.x * blockDim.x) {\n";
  emit_decompose(meta.shape, "t", "    ", s);
  leaf_slots->clear();
  auto read = [&](const VmRead& rd) -> std::string {
    if (rd.leaf < 0) return "";
    const int slot = slot_of(leaf_slots, rd.leaf, kTabLeaves);
    if (slot < 0) return "";
    return load_expr(leaf_info(p, rd.leaf).storage, "a.leaf[" + std::to_string(slot) + "]", read_offset(rd));
  };
  if (!emit_program(p, op, read, "    ", s)) return "";
  s << "    a.out[t] = r0;\n  }\n}\n";
  return s.str();
}

// Source of the in-place epilogue pass of one row (RowEpilogue): every output
// point t reads its value (acc), runs the program, stores the result.
std::string epi_kernel_source(const Plan& p, const OperandStatic& op, const ArrayMeta& out_meta, int out_storage,
                              std::vector<int>* leaf_slots) {
  if (out_storage != ST_F64 && out_storage != ST_F32) return "";
  const std::string T = out_storage == ST_F64 ? "double" : "float";
  std::ostringstream s;
  s << "#include \"fastmath.cuh\"\nstruct TabArgs { const void* leaf[" << kTabLeaves << "]; double* out; long long count; };\n"
    << "extern \"C\" __global__ void __launch_bounds__(256) fe_epi(const TabArgs a) {\n"
    << "  " << T << "* out = (" << T << "*)a.out;\n"
    << "  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < a.count;\n"
    << "       t += (long long)gridDim.x * blockDim.x) {\n";
  emit_decompose(out_meta.shape, "t", "    ", s);
  s << "    const double acc = (double)out[t];\n";
  leaf_slots->clear();
  auto read = [&](const VmRead& rd) -> std::string {
    if (rd.leaf == kAccLeaf) return "acc";
    if (rd.leaf < 0) return "";
    const int slot = slot_of(leaf_slots, rd.leaf, kTabLeaves);
    if (slot < 0) return "";
    return load_expr(leaf_info(p, rd.leaf).storage, "a.leaf[" + std::to_string(slot) + "]", read_offset(rd));
  };
  if (!emit_program(p, op, read, "    ", s)) return "";
  s << "    out[t] = (" << T << ")r0;\n  }\n}\n";
  return s.str();
}

// Source of a fem_grad instance (fem_grad.cuh's kernel body) with every row's
// U operand built in the prologue from staged leaf tiles — plain, affine, or
// a VM program (the tabulated operand's program, now never written to HBM) —
// and the rows' epilogues applied before the stores. `u_tiles` receives the
// staged leaves per canonical row, `aux` the leaves read through p.aux.
std::string fem_rtc_source(const Plan& p, int te, int ept, bool dsmem, std::vector<std::vector<int>>* u_tiles,
                           std::vector<int>* aux, std::string* why) {
  const FemBinding& f = p.fem;
  const size_t nl = p.leaves.size();
  if (f.f32) {
    *why = "fp32 plans use the prebuilt instances";
    return "";
  }
  u_tiles->assign(static_cast<size_t>(f.rows), {});
  aux->clear();
  const std::vector<std::int64_t> tile_shape{f.E, f.NJ};
  const int kUTile = te * f.NJ;
  // staged tiles: [TE, NJ] runs of [E, NJ] leaves, numbered in row order
  // (a row's tiles are consecutive; the producer streams them every stage)
  std::vector<std::pair<int, int>> staged;  // (row, leaf) in tile order
  auto tile_index = [&](int q, int leaf) {
    for (size_t k = 0; k < staged.size(); ++k)
      if (staged[k].first == q && staged[k].second == leaf) return static_cast<int>(k);
    return -1;
  };
  auto stageable = [&](const VmRead& rd, int p_e, int p_j) {
    if (rd.leaf < 0 || static_cast<size_t>(rd.leaf) >= nl) return false;
    const LeafInfo& L = leaf_info(p, rd.leaf);
    return rd.ndim == 2 && rd.param_of[0] == p_e && rd.param_of[1] == p_j && L.meta.shape == tile_shape &&
           L.storage == ST_F64;
  };
  auto aux_read = [&](const VmRead& rd) -> std::string {
    if (rd.leaf < 0 || static_cast<size_t>(rd.leaf) >= nl) return "";
    const int slot = slot_of(aux, rd.leaf, kFemMaxAux);
    if (slot < 0) return "";
    return load_expr(leaf_info(p, rd.leaf).storage, "p.aux[" + std::to_string(slot) + "]", read_offset(rd));
  };
  // pass 1: the tiles every row stages (U terms / program reads, then the
  // epilogue's [E, NI] reads when NI == NJ), in row order
  std::vector<const OperandStatic*> epi_of(static_cast<size_t>(f.rows), nullptr);
  for (int q = 0; q < f.rows; ++q) {
    auto add = [&](int leaf) {
      if (tile_index(q, leaf) < 0) staged.emplace_back(q, leaf);
    };
    const auto& terms = f.u_terms[static_cast<size_t>(q)];
    const bool program = terms.size() == 1 && static_cast<size_t>(terms[0].leaf) >= nl;
    if (!program) {
      for (const AffineTerm& tm : terms) add(tm.leaf);
    } else {
      const OperandStatic& op = p.ops[static_cast<size_t>(p.tabs[static_cast<size_t>(terms[0].leaf) - nl].op)];
      for (int pc = op.prog_off; pc < op.prog_off + op.prog_len; ++pc) {
        const VmInstr& in = p.prog[static_cast<size_t>(pc)];
        if (in.code == VM_READ && stageable(p.reads[static_cast<size_t>(in.arg)], 0, 1))
          add(p.reads[static_cast<size_t>(in.arg)].leaf);
      }
    }
    const int row = f.out_row[static_cast<size_t>(q)];
    if (static_cast<size_t>(row) < p.epi_ops.size() && p.epi_ops[static_cast<size_t>(row)].kind == OPK_VM) {
      const OperandStatic& op = p.epi_ops[static_cast<size_t>(row)];
      epi_of[static_cast<size_t>(q)] = &op;
      if (f.NI == f.NJ)
        for (int pc = op.prog_off; pc < op.prog_off + op.prog_len; ++pc) {
          const VmInstr& in = p.prog[static_cast<size_t>(pc)];
          if (in.code == VM_READ && stageable(p.reads[static_cast<size_t>(in.arg)], 1, 2))
            add(p.reads[static_cast<size_t>(in.arg)].leaf);
        }
    }
  }
  if (staged.size() > static_cast<size_t>(kFemMaxUTiles)) {
    *why = "too many staged tiles";
    return "";
  }
  for (const auto& [q, leaf] : staged) (*u_tiles)[static_cast<size_t>(q)].push_back(leaf);

  // pass 2: prologue — every staged value of this (v) point is read into a
  // register first (the rows' programs then overlap), then each row's value
  std::ostringstream pro, epi;
  std::vector<int> fast_rows;
  std::vector<std::string> fast_body, slow_body;
  pro << "      const double* __restrict__ sd = (const double*)su;\n";
  for (size_t k = 0; k < staged.size(); ++k)
    pro << "      const double s" << k << " = sd[" << k << " * kUTile + v];\n";
  pro << "@FASTBLOCK@";
  for (int q = 0; q < f.rows; ++q) {
    pro << "      {  // canonical row " << q << "\n";
    const auto& terms = f.u_terms[static_cast<size_t>(q)];
    const bool program = terms.size() == 1 && static_cast<size_t>(terms[0].leaf) >= nl;
    if (!program) {
      // plain / affine: (pre * x) * post per term, folded left to right
      for (size_t t = 0; t < terms.size(); ++t) {
        const AffineTerm& tm = terms[t];
        const std::string x = "s" + std::to_string(tile_index(q, tm.leaf));
        const std::string pre = tm.pre >= 0 ? "__ldg(p.coef + " + std::to_string(2 * tm.pre) + ")" : "1.0";
        const std::string post = tm.post0 >= 0 ? "__ldg(p.coef + " + std::to_string(2 * tm.post0) + ")" : "1.0";
        const std::string term = "__dmul_rn(__dmul_rn(" + pre + ", " + x + "), " + post + ")";
        if (t == 0)
          pro << "        double val = " << term << ";\n";
        else
          pro << "        val = " << (tm.sign > 0 ? "__dadd_rn" : "__dsub_rn") << "(val, " << term << ");\n";
      }
      if (terms.empty()) pro << "        double val = 0.0;\n";
    } else {
      const OperandStatic& op = p.ops[static_cast<size_t>(p.tabs[static_cast<size_t>(terms[0].leaf) - nl].op)];
      auto read = [&](const VmRead& rd) -> std::string {
        if (stageable(rd, 0, 1)) return "s" + std::to_string(tile_index(q, rd.leaf));
        return aux_read(rd);
      };
      bool global_reads = false;
      auto read_chk = [&](const VmRead& rd) -> std::string {
        if (!stageable(rd, 0, 1)) global_reads = true;
        return read(rd);
      };
      std::ostringstream body, fast;
      if (!emit_program(p, op, read_chk, "          ", body)) {
        *why = "operand program of row " + std::to_string(q) + " not expressible";
        return "";
      }
      if (!global_reads && emit_program(p, op, read, "          ", fast, true)) {
        // every read is a staged value (registers, valid for dead points
        // too): this row joins the point's straight-line block of fast
        // forms (emitted after the loop over rows), and only a point whose
        // arguments leave their range re-runs the checked forms
        fast_rows.push_back(q);
        fast_body.push_back(fast.str());
        slow_body.push_back(body.str());
        pro << "        double val = live ? fv" << q << " : 0.0;\n";
      } else {
        pro << "        double val = 0.0;\n        if (live) {\n" << body.str() << "          val = r0;\n        }\n";
      }
    }
    pro << "        uc[" << q << " * kUTile + v] = val;\n      }\n";
    // epilogue of the caller row this canonical row writes
    if (const OperandStatic* op = epi_of[static_cast<size_t>(q)]) {
      auto read = [&](const VmRead& rd) -> std::string {
        if (rd.leaf == kAccLeaf) return "(double)y";
        const int k = f.NI == f.NJ && stageable(rd, 1, 2) ? tile_index(q, rd.leaf) : -1;
        if (k >= 0) return "sd[" + std::to_string(k * kUTile) + " + (e - e0) * " + std::to_string(f.NJ) + " + i]";
        return aux_read(rd);
      };
      std::ostringstream body;
      if (!emit_program(p, *op, read, "        ", body)) {
        *why = "epilogue of row " + std::to_string(f.out_row[static_cast<size_t>(q)]) + " not expressible";
        return "";
      }
      epi << "      case " << q << ": {\n" << body.str() << "        return r0;\n      }\n";
    }
  }
  {
    // the fast block: every fast row's program back to back (no branch
    // between them, so their long dependency chains interleave), one range
    // test for the point, the checked forms only when it fails
    std::ostringstream fb;
    if (!fast_rows.empty()) {
      fb << "      bool fe_ok = true;\n      double";
      for (size_t k = 0; k < fast_rows.size(); ++k) fb << (k ? ", fv" : " fv") << fast_rows[k];
      fb << ";\n";
      for (size_t k = 0; k < fast_rows.size(); ++k)
        fb << "      {\n" << fast_body[k] << "        fv" << fast_rows[k] << " = r0;\n      }\n";
      fb << "      if (!fe_ok) {\n";
      for (size_t k = 0; k < fast_rows.size(); ++k)
        fb << "        {\n" << slow_body[k] << "          fv" << fast_rows[k] << " = r0;\n        }\n";
      fb << "      }\n";
    }
    std::string ps = pro.str();
    ps.replace(ps.find("@FASTBLOCK@"), 11, fb.str());
    pro.str(ps);
  }
  const int consumers = (te * f.NI / ept + 31) / 32 * 32;
  std::ostringstream s;
  s << "#include \"fastmath.cuh\"\n#include \"fem_grad.cuh\"\n"
    << "using namespace feb200;\nusing namespace feb200::fem;\n"
    << "struct GenPro {\n  static constexpr bool kPlain = false;\n  static constexpr bool kPipe = true;\n"
    << "  template <typename T, int kUTile, int kConsumers>\n"
    << "  __device__ static void combine(const FemGradLaunch& p, const T* su, T* uc, const Coef*, int c, long long e0,\n"
    << "                                 long long E) {\n"
    << "    for (int v = c; v < kUTile; v += kConsumers) {\n"
    << "      const long long p0 = e0 + v / " << f.NJ << ";\n"
    << "      const long long p1 = v % " << f.NJ << ";\n"
    << "      const bool live = p0 < E;\n"
    << "      (void)p1; (void)live;\n"
    << pro.str() << "    }\n  }\n};\n"
    << "struct GenEpi {\n  static constexpr bool kIdentity = " << (epi.str().empty() ? "true" : "false") << ";\n"
    << "  template <typename T>\n"
    << "  __device__ static T apply(const FemGradLaunch& p, int q, int r, long long e, int i, T y, const T* su,\n"
    << "                            long long e0) {\n"
    << "    const long long p0 = r, p1 = e, p2 = i;\n"
    << "    const double* __restrict__ sd = (const double*)su;\n"
    << "    (void)p0; (void)p1; (void)p2; (void)p; (void)sd; (void)e0;\n"
    << "    switch (q) {\n" << epi.str() << "      default: return y;\n    }\n  }\n};\n"
    << "extern \"C\" __global__ void __launch_bounds__(" << 32 + consumers << ", " << (dsmem ? 2 : 1) << ")\n"
    << "    fe_fem_rtc(const __grid_constant__ FemGradLaunch p) {\n"
    << "  fem_grad_body<double, " << f.NX << ", " << f.NR << ", " << f.NI << ", " << f.NJ << ", " << te
    << ", GenPro, " << (dsmem ? "true" : "false") << ", " << ept << ", GenEpi>(p);\n}\n";
  return s.str();
}

namespace {

// NVRTC compile to an sm_100a cubin; false (and the log) on failure
bool nvrtc_cubin(const std::string& src, std::vector<char>* cubin, std::string* log) {
  if (std::getenv("FE_DUMP_RTC")) std::fprintf(stderr, "---- generated source ----\n%s\n", src.c_str());
  const Nvrtc& n = nvrtc();
  if (!n.ok) {
    *log = "NVRTC not available";
    return false;
  }
  nvrtcProgram prog;
  // the device headers generated instances include (embedded at build time)
  if (n.create(&prog, src.c_str(), "fe_rtc.cu", kRtcHeaderCount, kRtcHeaderSources, kRtcHeaderNames) !=
      NVRTC_SUCCESS) {
    *log = "nvrtcCreateProgram failed";
    return false;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "-fmad=false", "--std=c++17", "-default-device"};
  const bool ok = n.compile(prog, 4, opts) == NVRTC_SUCCESS;
  size_t ls = 0;
  n.log_size(prog, &ls);
  log->assign(ls, '\0');
  if (ls) n.log(prog, log->data());
  if (ok) {
    size_t cs = 0;
    n.cubin_size(prog, &cs);
    cubin->resize(cs);
    n.cubin(prog, cubin->data());
    // FE_DUMP_CUBIN=<dir>: keep every generated cubin (cuobjdump -sass / -res-usage)
    if (const char* dir = std::getenv("FE_DUMP_CUBIN")) {
      static int seq = 0;
      const std::string path = std::string(dir) + "/fe_rtc_" + std::to_string(seq++) + ".cubin";
      if (FILE* f = std::fopen(path.c_str(), "wb")) {
        std::fwrite(cubin->data(), 1, cubin->size(), f);
        std::fclose(f);
      }
    }
  }
  n.destroy(&prog);
  return ok;
}

}  // namespace

// Compile (memoised by source), load, and return the handle of kernel `name`, or nullptr.
void* compile_rtc_kernel(const std::string& src, const char* name, std::string* log) {
  static std::mutex mu;
  static std::map<std::string, void*> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(src);
  if (it != cache.end()) return it->second;
  std::vector<char> cubin;
  if (!nvrtc_cubin(src, &cubin, log)) return nullptr;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t k = nullptr;
  if (cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
      cudaLibraryGetKernel(&k, lib, name) != cudaSuccess) {
    cudaGetLastError();
    *log = "cudaLibraryLoadData / cudaLibraryGetKernel failed";
    return nullptr;
  }
  cache.emplace(src, reinterpret_cast<void*>(k));  // libraries stay loaded for the process
  return reinterpret_cast<void*>(k);
}

void* compile_tab_kernel(const std::string& src, std::string* log) { return compile_rtc_kernel(src, "fe_tab", log); }

// NVRTC compile only (no device): dry-run plans report whether the emitted
// source compiles for sm_100a.
bool nvrtc_compiles(const std::string& src, std::string* log) {
  static std::mutex mu;
  static std::map<std::string, std::pair<bool, std::string>> memo;
  std::lock_guard<std::mutex> lock(mu);
  auto it = memo.find(src);
  if (it == memo.end()) {
    std::vector<char> cubin;
    std::string l;
    const bool ok = nvrtc_cubin(src, &cubin, &l);
    it = memo.emplace(src, std::make_pair(ok, l)).first;
  }
  *log = it->second.second;
  return it->second.first;
}

int launch_tab_kernel(void* kernel, const TabArgs& args, int sm_count, void* stream) {
  if (args.count == 0) return cudaSuccess;
  std::int64_t blocks = (args.count + 255) / 256;
  const std::int64_t cap = static_cast<std::int64_t>(sm_count) * 8;
  if (blocks > cap) blocks = cap;
  void* params[] = {const_cast<TabArgs*>(&args)};
  return cudaLaunchKernel(reinterpret_cast<const void*>(kernel), dim3(static_cast<unsigned>(blocks)), dim3(256), params,
                          0, static_cast<cudaStream_t>(stream));
}

}  // namespace feb200
