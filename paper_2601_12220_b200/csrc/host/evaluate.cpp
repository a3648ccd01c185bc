// The drop-in numeric entry points of the reference API — evaluate
// (proj/include/feinsum/core.hpp:141), evaluate_functional, materialize and
// eval_expr (proj/include/feinsum/raising.hpp:38-59) — implemented on the GPU
// through the planner. Host DenseArrays (complex<double>, the reference's
// representation) are uploaded "wide" (f64, or c128 when any value is complex)
// so every value reaches the kernel unrounded; results come back the same way.
// There is deliberately no host evaluation path: without a usable CUDA device
// these functions throw errc::io.
#include <cuda_runtime.h>

#include <deque>
#include <functional>
#include <memory>

#include "feinsum/core.hpp"
#include "feinsum/raising.hpp"
#include "planner.hpp"

namespace feinsum {

namespace {

using feb200::Plan;
using feb200::PlanOptions;

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw error(errc::io, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

void require_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    throw error(errc::io,
                "no usable CUDA device: feinsum-b200 evaluates on sm_100a GPUs only (there is no CPU fallback)");
}

bool has_imag(const DenseArray& a) {
  for (const auto& z : a.data)
    if (z.imag() != 0.0) return true;
  return false;
}

bool complex_dtype(Dtype t) { return t == Dtype::complex64 || t == Dtype::complex128; }

// Device buffers of one call; freed on scope exit.
struct DeviceScratch {
  std::vector<void*> bufs;
  std::deque<std::vector<double>> staged;
  cudaStream_t stream = nullptr;
  ~DeviceScratch() {
    if (stream) cudaStreamSynchronize(stream);
    for (void* b : bufs) cudaFree(b);
    if (stream) cudaStreamDestroy(stream);
  }
  void* alloc(size_t bytes) {
    void* p = nullptr;
    check(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc");
    bufs.push_back(p);
    return p;
  }
};

void* upload(DeviceScratch& ds, const DenseArray& a, int storage) {
  const size_t n = a.data.size();
  if (storage == feb200::ST_C128) {
    void* d = ds.alloc(n * 16);
    check(cudaMemcpyAsync(d, a.data.data(), n * 16, cudaMemcpyHostToDevice, ds.stream), "upload");
    return d;
  }
  // staged real parts live until the stream has consumed them (pageable
  // async copies only guarantee staging, so keep the buffer alive)
  ds.staged.emplace_back(n);
  std::vector<double>& re = ds.staged.back();
  for (size_t i = 0; i < n; ++i) re[i] = a.data[i].real();
  void* d = ds.alloc(n * 8);
  check(cudaMemcpyAsync(d, re.data(), n * 8, cudaMemcpyHostToDevice, ds.stream), "upload");
  return d;
}

std::vector<DenseArray> run(const Plan& plan, const Bindings& bindings) {
  DeviceScratch ds;
  check(cudaStreamCreateWithFlags(&ds.stream, cudaStreamNonBlocking), "cudaStreamCreate");
  std::vector<const void*> ins;
  for (const auto& L : plan.leaves) ins.push_back(upload(ds, bindings.at(L.meta.name), L.storage));
  std::vector<void*> outs;
  for (const auto& o : plan.outputs) outs.push_back(ds.alloc(static_cast<size_t>(o.bytes())));
  feb200::execute(plan, ins.data(), outs.data(), ds.stream);
  std::vector<DenseArray> result;
  for (size_t r = 0; r < plan.outputs.size(); ++r) {
    const auto& o = plan.outputs[r];
    DenseArray a = DenseArray::zeros(o.meta);
    const size_t n = a.data.size();
    if (o.storage == feb200::ST_C128) {
      check(cudaMemcpyAsync(a.data.data(), outs[r], n * 16, cudaMemcpyDeviceToHost, ds.stream), "download");
      check(cudaStreamSynchronize(ds.stream), "download");
    } else {
      std::vector<double> re(n);
      check(cudaMemcpyAsync(re.data(), outs[r], n * 8, cudaMemcpyDeviceToHost, ds.stream), "download");
      check(cudaStreamSynchronize(ds.stream), "download");
      for (size_t i = 0; i < n; ++i) a.data[i] = {re[i], 0.0};
    }
    result.push_back(std::move(a));
  }
  return result;
}

PlanOptions wide_options(const Bindings& bindings, const std::vector<std::string>& names) {
  PlanOptions opt;
  opt.storage = "wide";
  for (const auto& name : names) {
    const DenseArray& a = bindings.at(name);
    opt.storage_of[name] = (complex_dtype(a.meta.dtype) || has_imag(a)) ? "c128" : "f64";
  }
  return opt;
}

// arrays read by operand bodies, with the metadata their bindings carry
std::map<std::string, ArrayMeta> read_arrays(const std::map<std::string, OperandExpr>& ops, const Bindings& b) {
  std::map<std::string, ArrayMeta> arrays;
  std::function<void(const Expr&)> walk = [&](const Expr& e) {
    if (e.kind == Expr::Kind::access) {
      auto it = b.find(e.name);
      if (it != b.end()) arrays.emplace(e.name, it->second.meta);
    }
    for (const Expr& c : e.children) walk(c);
  };
  for (const auto& kv : ops) walk(kv.second.body);
  return arrays;
}

}  // namespace

std::vector<DenseArray> evaluate(const BatchedEinsum& e, const Bindings& bindings) {
  require_valid(e);
  std::vector<std::string> names;
  for (const ArrayMeta& a : universe(e)) {
    auto it = bindings.find(a.name);
    if (it == bindings.end()) throw error(errc::domain, "no binding for array " + a.name);
    if (!(it->second.meta == a))
      throw error(errc::domain, "binding for array " + a.name + " does not match the declared shape/dtype");
    if (static_cast<std::int64_t>(it->second.data.size()) != a.num_elements())
      throw error(errc::domain, "binding for array " + a.name + " has wrong element count");
    names.push_back(a.name);
  }
  require_device();
  auto plan = feb200::make_plan(e, wide_options(bindings, names));
  return run(*plan, bindings);
}

std::vector<DenseArray> evaluate_functional(const FunctionalBatchedEinsum& f, const Bindings& bindings) {
  for (const ArrayMeta& m : universe(f.skeleton))
    if (!f.operand_map.count(m.name)) throw error(errc::domain, "no operand expression for " + m.name);
  require_device();
  auto reads = f.operand_map;  // arrays read by operands and (extension) epilogues
  for (const auto& [row, ep] : f.epilogue) reads["epilogue " + std::to_string(row)] = ep.op;
  auto arrays = read_arrays(reads, bindings);
  for (const auto& [row, ep] : f.epilogue) arrays.erase(ep.acc);
  std::vector<std::string> names;
  for (const auto& kv : arrays) names.push_back(kv.first);
  for (const auto& name : names)
    if (static_cast<std::int64_t>(bindings.at(name).data.size()) != bindings.at(name).meta.num_elements())
      throw error(errc::domain, "binding for array " + name + " has wrong element count");
  auto plan = feb200::make_functional_plan(f.skeleton, f.operand_map, arrays, wide_options(bindings, names),
                                           f.epilogue);
  return run(*plan, bindings);
}

namespace {

// one-slot identity skeleton "p0 p1 ... -> p0 p1 ..." over meta
BatchedEinsum operand_skeleton(const ArrayMeta& meta) {
  BatchedEinsum e;
  IndexList idx;
  for (int d = 0; d < meta.dim(); ++d) idx.push_back("p" + std::to_string(d));
  e.i_out = idx;
  e.i_in = {idx};
  e.args = {{meta}};
  return e;
}

std::vector<std::complex<double>> tabulate_points(const Plan& plan, const Bindings& bindings, const std::string& name,
                                                  std::int64_t first, std::int64_t count) {
  DeviceScratch ds;
  check(cudaStreamCreateWithFlags(&ds.stream, cudaStreamNonBlocking), "cudaStreamCreate");
  std::vector<const void*> ins;
  for (const auto& L : plan.leaves) ins.push_back(upload(ds, bindings.at(L.meta.name), L.storage));
  auto* out = static_cast<double*>(ds.alloc(static_cast<size_t>(count) * 16));
  feb200::tabulate(plan, name, ins.data(), out, first, count, ds.stream);
  std::vector<std::complex<double>> host(static_cast<size_t>(count));
  check(cudaMemcpyAsync(host.data(), out, static_cast<size_t>(count) * 16, cudaMemcpyDeviceToHost, ds.stream),
        "download");
  check(cudaStreamSynchronize(ds.stream), "download");
  return host;
}

}  // namespace

DenseArray materialize(const OperandExpr& op, const ArrayMeta& meta, const Bindings& bindings) {
  if (op.params.size() != meta.shape.size())
    throw error(errc::domain, "materialize: operand takes " + std::to_string(op.params.size()) +
                                  " parameters, shape has " + std::to_string(meta.shape.size()) + " axes");
  require_device();
  std::map<std::string, OperandExpr> ops{{meta.name, op}};
  const auto arrays = read_arrays(ops, bindings);
  std::vector<std::string> names;
  for (const auto& kv : arrays) names.push_back(kv.first);
  PlanOptions opt = wide_options(bindings, names);
  opt.canonicalize = false;
  auto plan = feb200::make_functional_plan(operand_skeleton(meta), ops, arrays, opt);
  DenseArray a = DenseArray::zeros(meta);
  a.data = tabulate_points(*plan, bindings, meta.name, 0, meta.num_elements());
  return a;
}

std::complex<double> eval_expr(const OperandExpr& op, const std::vector<std::int64_t>& at, const Bindings& bindings) {
  if (at.size() != op.params.size())
    throw error(errc::domain, "eval_expr: got " + std::to_string(at.size()) + " values for " +
                                  std::to_string(op.params.size()) + " parameters");
  // validate reads in evaluation order with the actual point (reference messages)
  std::map<std::string, std::int64_t> env;
  for (size_t k = 0; k < at.size(); ++k) env[op.params[k]] = at[k];
  std::function<void(const Expr&)> walk = [&](const Expr& e) {
    for (const Expr& c : e.children) walk(c);
    if (e.kind != Expr::Kind::access) return;
    auto it = bindings.find(e.name);
    if (it == bindings.end()) throw error(errc::domain, "no binding for array " + e.name);
    const auto& shape = it->second.meta.shape;
    if (e.subs.size() != shape.size())
      throw error(errc::domain, "array " + e.name + " read with " + std::to_string(e.subs.size()) +
                                    " subscripts, has " + std::to_string(shape.size()) + " axes");
    for (size_t d = 0; d < e.subs.size(); ++d) {
      const std::int64_t v = env.at(e.subs[d]);
      if (v < 0 || v >= shape[d])
        throw error(errc::domain, "array " + e.name + " subscript " + std::to_string(v) + " out of range on axis " +
                                      std::to_string(d));
    }
  };
  walk(op.body);
  require_device();
  ArrayMeta meta{"point", {}, Dtype::float64};
  std::int64_t flat = 0;
  for (std::int64_t v : at) {
    meta.shape.push_back(v + 1);
    flat = flat * (v + 1) + v;
  }
  std::map<std::string, OperandExpr> ops{{meta.name, op}};
  const auto arrays = read_arrays(ops, bindings);
  std::vector<std::string> names;
  for (const auto& kv : arrays) names.push_back(kv.first);
  PlanOptions opt = wide_options(bindings, names);
  opt.canonicalize = false;
  opt.force_vm = true;
  opt.skip_range_check = true;
  auto plan = feb200::make_functional_plan(operand_skeleton(meta), ops, arrays, opt);
  return tabulate_points(*plan, bindings, meta.name, flat, 1)[0];
}

}  // namespace feinsum
