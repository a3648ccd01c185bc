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
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "planner.hpp"

namespace feb200 {

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

// element read of leaf slot k at offset expression `off`, as double
std::string load_expr(int st, int k, const std::string& off) {
  const std::string p = "a.leaf[" + std::to_string(k) + "]";
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

}  // namespace

// Source of the tabulation kernel for one operand, or "" if unsupported.
// `leaf_slots` receives the plan leaf index of each kernel leaf slot.
std::string tab_kernel_source(const Plan& p, const OperandStatic& op, const ArrayMeta& meta,
                              std::vector<int>* leaf_slots) {
  std::ostringstream s;
  const int nd = meta.dim();
  s << "struct TabArgs { const void* leaf[" << kTabLeaves << "]; double* out; long long count; };\n"
    << "extern \"C\" __global__ void __launch_bounds__(256) fe_tab(const TabArgs a) {\n"
    << "  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < a.count;\n"
    << "       t += (long long)gridDim.x * blockDim.x) {\n"
    << "    long long rem = t;\n";
  for (int d = nd - 1; d >= 1; --d)
    s << "    const long long p" << d << " = rem % " << meta.shape[d] << "LL; rem /= " << meta.shape[d] << "LL;\n";
  if (nd >= 1) s << "    const long long p0 = rem;\n";
  for (int r = 0; r < kMaxVmRegs; ++r) s << "    double r" << r << " = 0.0;\n";
  leaf_slots->clear();
  for (int pc = op.prog_off; pc < op.prog_off + op.prog_len; ++pc) {
    const VmInstr& in = p.prog[static_cast<size_t>(pc)];
    const std::string dst = "r" + std::to_string(in.dst & (kMaxVmRegs - 1));
    const std::string a = "r" + std::to_string(in.a & (kMaxVmRegs - 1));
    const std::string b = "r" + std::to_string(in.b & (kMaxVmRegs - 1));
    std::string v;
    switch (in.code) {
      case VM_LIT: v = hexlit(in.imm); break;
      case VM_PARAM: v = "(double)p" + std::to_string(in.arg); break;
      case VM_READ: {
        const VmRead& rd = p.reads[static_cast<size_t>(in.arg)];
        int slot = -1;
        for (size_t k = 0; k < leaf_slots->size(); ++k)
          if ((*leaf_slots)[k] == rd.leaf) slot = static_cast<int>(k);
        if (slot < 0) {
          if (leaf_slots->size() >= static_cast<size_t>(kTabLeaves)) return "";
          slot = static_cast<int>(leaf_slots->size());
          leaf_slots->push_back(rd.leaf);
        }
        std::string off = "0LL";
        for (int d = 0; d < rd.ndim; ++d)
          off += " + p" + std::to_string(rd.param_of[d]) + " * " + std::to_string(rd.stride[d]) + "LL";
        v = load_expr(leaf_info(p, rd.leaf).storage, slot, off);
        if (v.empty()) return "";
        break;
      }
      case VM_ADD: v = "__dadd_rn(" + a + ", " + b + ")"; break;
      case VM_SUB: v = "__dsub_rn(" + a + ", " + b + ")"; break;
      case VM_MUL: v = "__dmul_rn(" + a + ", " + b + ")"; break;
      case VM_DIV: v = "__ddiv_rn(" + a + ", " + b + ")"; break;
      case VM_SIN: v = "sin(" + a + ")"; break;
      case VM_COS: v = "cos(" + a + ")"; break;
      case VM_EXP: v = "exp(" + a + ")"; break;
      case VM_RECIP: v = "__ddiv_rn(1.0, " + a + ")"; break;
      default: return "";  // sqrt: complex plans only
    }
    s << "    " << dst << " = " << v << ";\n";
  }
  s << "    a.out[t] = r0;\n  }\n}\n";
  return s.str();
}

namespace {

// NVRTC compile to an sm_100a cubin; false (and the log) on failure
bool nvrtc_cubin(const std::string& src, std::vector<char>* cubin, std::string* log) {
  const Nvrtc& n = nvrtc();
  if (!n.ok) {
    *log = "NVRTC not available";
    return false;
  }
  nvrtcProgram prog;
  if (n.create(&prog, src.c_str(), "fe_tab.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
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
  }
  n.destroy(&prog);
  return ok;
}

}  // namespace

// Compile (memoised by source), load, and return the kernel handle, or nullptr.
void* compile_tab_kernel(const std::string& src, std::string* log) {
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
      cudaLibraryGetKernel(&k, lib, "fe_tab") != cudaSuccess) {
    cudaGetLastError();
    *log = "cudaLibraryLoadData / cudaLibraryGetKernel failed";
    return nullptr;
  }
  cache.emplace(src, reinterpret_cast<void*>(k));  // libraries stay loaded for the process
  return reinterpret_cast<void*>(k);
}

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
