// extern "C" boundary (include/feinsum_b200.h). Every entry point converts
// exceptions into status codes + a thread-local message, so no C++ exception
// ever crosses the ABI.
#include <algorithm>
#include "feinsum_b200.h"

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>

#include "feinsum/canonicalize.hpp"
#include "feinsum/factsdb.hpp"
#include "feinsum/induced_graph.hpp"
#include "feinsum/notation.hpp"
#include "feinsum/raising.hpp"
#include "json.hpp"
#include "planner.hpp"
#include "einsum_json.hpp"  // after the feinsum headers

using fejson::Value;
using namespace feinsum;

// Pipelined host execution (fe_plan_execute_host on large plans): the plan is
// cut into chunks along its shard axis (fe_plan_shard's sub-plans); chunk k's
// H2D, chunk k-1's kernels and chunk k-2's D2H run concurrently on three
// streams (two copy engines + the SMs), double-buffered device slots.
struct HostPipe {
  struct Slice {
    int pos = -1;  // axis position in the array, -1: replicated (copied once per call)
    std::int64_t outer = 1, inner = 1, n = 0, esize = 8;
  };
  std::vector<std::unique_ptr<feb200::Plan>> parts;
  std::vector<std::int64_t> lo, hi;
  std::vector<Slice> in_slice, out_slice;
  std::vector<void*> rep_in;                    // replicated inputs (full size)
  std::vector<void*> slot_in[2], slot_out[2];   // per-slot chunk buffers (largest chunk)
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  cudaEvent_t start = nullptr, rep_done = nullptr, h2d_done[2] = {}, comp_done[2] = {}, d2h_done[2] = {};
  ~HostPipe() {
    for (void* p : rep_in) cudaFree(p);
    for (int b = 0; b < 2; ++b) {
      for (void* p : slot_in[b]) cudaFree(p);
      for (void* p : slot_out[b]) cudaFree(p);
      if (h2d_done[b]) cudaEventDestroy(h2d_done[b]);
      if (comp_done[b]) cudaEventDestroy(comp_done[b]);
      if (d2h_done[b]) cudaEventDestroy(d2h_done[b]);
    }
    if (start) cudaEventDestroy(start);
    if (rep_done) cudaEventDestroy(rep_done);
    for (cudaStream_t q : {s_h2d, s_comp, s_d2h})
      if (q) cudaStreamDestroy(q);
  }
};

// Row pipeline (fe_plan_execute_host on plans too small to chunk, with
// several rows): each row runs as its own single-row plan, so row r's
// outputs stream back while row r+1 computes and row r+2's private inputs
// upload (C1: the 7.2 MB of outputs no longer wait for the whole batch).
// Single-row plans do each element's arithmetic in the same order, so the
// outputs are bitwise those of the batched execute.
struct RowPipe {
  std::vector<std::unique_ptr<feb200::Plan>> rows;
  std::vector<std::vector<int>> src;   // row plan leaf -> plan leaf
  std::vector<int> first_use;          // plan leaf -> first row that reads it
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  cudaEvent_t start = nullptr;
  std::vector<cudaEvent_t> h2d_done, comp_done, d2h_done;
  ~RowPipe() {
    for (auto* v : {&h2d_done, &comp_done, &d2h_done})
      for (cudaEvent_t e : *v) cudaEventDestroy(e);
    if (start) cudaEventDestroy(start);
    for (cudaStream_t q : {s_h2d, s_comp, s_d2h})
      if (q) cudaStreamDestroy(q);
  }
};

struct fe_plan_s {
  std::unique_ptr<feb200::Plan> plan;
  std::unique_ptr<RowPipe> rowpipe;
  bool rowpipe_tried = false;
  std::string options;  // creation options (sub-plans of the host pipeline reuse them)
  // staging buffers for fe_plan_execute_host, allocated on first use
  std::vector<void*> staged_in, staged_out;
  std::unique_ptr<HostPipe> pipe;
  bool pipe_tried = false;
  ~fe_plan_s() {
    for (void* p : staged_in) cudaFree(p);
    for (void* p : staged_out) cudaFree(p);
  }
};

namespace {

thread_local std::string g_last;

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

int guarded(const std::function<void()>& f) {
  try {
    f();
    return FE_OK;
  } catch (const feinsum::error& e) {
    g_last = e.what();
    return 1 + static_cast<int>(e.kind());
  } catch (const std::bad_alloc&) {
    g_last = "out of host memory";
    return FE_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_last = e.what();
    return FE_ERR_INTERNAL;
  }
}

int cuda_status(int e) {
  if (e == 0) return FE_OK;
  g_last = std::string("CUDA error: ") + cudaGetErrorString(static_cast<cudaError_t>(e));
  return FE_ERR_CUDA;
}

BatchedEinsum ein(const char* js) { return transport::einsum_from_json(fejson::parse(js)); }
void put(char** out, const Value& v) { *out = dup(fejson::dump(v)); }

Value graph_json(const ColoredDigraph& g) {
  Value v = Value::obj();
  v.set("n", Value::num(g.n));
  Value colors = Value::arr();
  for (int c : g.colors) colors.push(Value::num(c));
  v.set("colors", std::move(colors));
  Value edges = Value::arr();
  for (int i = 0; i < g.n; ++i)
    for (int j = 0; j < g.n; ++j)
      if (g.edge(i, j)) {
        Value e = Value::arr();
        e.push(Value::num(i));
        e.push(Value::num(j));
        edges.push(std::move(e));
      }
  v.set("edges", std::move(edges));
  return v;
}

ColoredDigraph graph_from(const Value& v) {
  ColoredDigraph g = ColoredDigraph::empty(static_cast<int>(v.at("n").as_int()));
  size_t k = 0;
  for (const auto& c : v.at("colors").a) g.colors.at(k++) = static_cast<int>(c.as_int());
  for (const auto& e : v.at("edges").a) g.set_edge(static_cast<int>(e.a[0].as_int()), static_cast<int>(e.a[1].as_int()));
  return g;
}

Expr expr_from(const Value& v) {
  Expr e;
  if (auto* x = v.find("lit")) {
    e.kind = Expr::Kind::literal;
    e.literal = x->as_double();
  } else if (auto* x = v.find("param")) {
    e.kind = Expr::Kind::param;
    e.name = x->as_str();
  } else if (auto* x = v.find("read")) {
    e.kind = Expr::Kind::access;
    e.name = x->as_str();
    e.subs = transport::list_from_json(v.at("subs"));
  } else if (auto* x = v.find("fn")) {
    e.kind = Expr::Kind::unary;
    e.name = x->as_str();
    e.children.push_back(expr_from(v.at("x")));
  } else if (auto* x = v.find("op")) {
    e.kind = Expr::Kind::binary;
    e.op = x->as_str().at(0);
    e.children.push_back(expr_from(v.at("l")));
    e.children.push_back(expr_from(v.at("r")));
  } else {
    throw error(errc::usage, "expression node needs one of lit/param/read/fn/op");
  }
  return e;
}

Value canon_json(const CanonResult& c) {
  Value v = Value::obj();
  v.set("canonical", transport::einsum_to_json(c.canonical));
  v.set("sigma_idx", transport::strmap_to_json(c.sigma_idx));
  v.set("sigma_arg", transport::strmap_to_json(c.sigma_arg));
  v.set("sigma_row", transport::ints_to_json(c.sigma_row));
  v.set("sigma_slot", transport::ints_to_json(c.sigma_slot));
  return v;
}

}  // namespace

namespace feinsum::detail {
std::string key_of_canonical(const BatchedEinsum& e);
}

extern "C" {

const char* fe_last_error(void) { return g_last.c_str(); }
void fe_free(void* p) { std::free(p); }
int fe_version(void) { return 1; }

int fe_device_check(void) {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    g_last = std::string("no usable CUDA device (") + cudaGetErrorString(e) + ")";
    return FE_ERR_IO;
  }
  return FE_OK;
}

int fe_parse_classic(const char* text, char** out) {
  return guarded([&] { put(out, transport::einsum_to_json(parse_classic(text))); });
}

int fe_print_classic(const char* js, char** out) {
  return guarded([&] { *out = dup(print_classic(ein(js))); });
}

int fe_validate(const char* js, char** out) {
  return guarded([&] { put(out, transport::list_to_json(validate(ein(js)))); });
}

int fe_canonicalize(const char* js, char** out) {
  return guarded([&] {
    const CanonResult c = canonicalize(ein(js));
    Value v = canon_json(c);
    v.set("key", Value::str(feinsum::detail::key_of_canonical(c.canonical)));
    put(out, v);
  });
}

int fe_canonical_key(const char* js, char** out) {
  return guarded([&] { *out = dup(canonical_key(ein(js))); });
}

int fe_is_isomorphic(const char* a, const char* b, char** out) {
  return guarded([&] {
    const auto w = is_isomorphic(ein(a), ein(b));
    put(out, w ? transport::witness_to_json(*w) : Value{});
  });
}

int fe_brute_force_isomorphic(const char* a, const char* b, uint64_t budget, char** out) {
  return guarded([&] {
    const auto w = brute_force_isomorphic(ein(a), ein(b), budget);
    put(out, w ? transport::witness_to_json(*w) : Value{});
  });
}

int fe_verify_witness(const char* a, const char* b, const char* w, char** out) {
  return guarded([&] {
    std::vector<std::string> why;
    const bool ok =
        verify_witness(ein(a), ein(b), transport::witness_from_json<SubstitutionWitness>(fejson::parse(w)), &why);
    Value v = Value::obj();
    v.set("ok", Value::boolean_(ok));
    v.set("why", transport::list_to_json(why));
    put(out, v);
  });
}

int fe_generate_random(const char* params_js, uint64_t seed, char** out) {
  return guarded([&] {
    GenParams p;
    const Value pv = fejson::parse(params_js);
    auto geti = [&](const char* k, int& dst) {
      if (auto* x = pv.find(k)) dst = static_cast<int>(x->as_int());
    };
    geti("b_min", p.b_min);
    geti("b_max", p.b_max);
    geti("n_min", p.n_min);
    geti("n_max", p.n_max);
    geti("max_indices", p.max_indices);
    geti("max_dim", p.max_dim);
    if (auto* x = pv.find("shape_pool")) {
      p.shape_pool.clear();
      for (const auto& s : x->a) p.shape_pool.push_back(s.as_int());
    }
    if (auto* x = pv.find("dtype_pool")) {
      p.dtype_pool.clear();
      for (const auto& s : x->a) p.dtype_pool.push_back(dtype_from_name(s.as_str()));
    }
    if (auto* x = pv.find("allow_empty_out")) p.allow_empty_out = x->b;
    if (auto* x = pv.find("allow_repeated_index")) p.allow_repeated_index = x->b;
    put(out, transport::einsum_to_json(generate_random(p, seed)));
  });
}

int fe_scramble(const char* js, uint64_t seed, char** out) {
  return guarded([&] {
    const Scrambled s = scramble(ein(js), seed);
    Value v = Value::obj();
    v.set("e", transport::einsum_to_json(s.e));
    v.set("w", transport::witness_to_json(s.w));
    put(out, v);
  });
}

int fe_induced_graph(const char* js, int64_t shuffle_seed, char** out) {
  return guarded([&] {
    std::optional<std::uint64_t> seed;
    if (shuffle_seed >= 0) seed = static_cast<std::uint64_t>(shuffle_seed);
    const InducedGraph ig = to_induced_graph(ein(js), seed);
    Value v = graph_json(ig.graph);
    Value ia = Value::obj(), ii = Value::obj(), io = Value::obj(), ip = Value::obj(), il = Value::obj(),
          idt = Value::obj();
    for (const auto& [k, x] : ig.iota_arg) ia.set(std::to_string(k), Value::str(x));
    for (const auto& [k, x] : ig.iota_index) ii.set(std::to_string(k), Value::str(x));
    for (const auto& [k, x] : ig.iota_output) io.set(std::to_string(k), Value::num(x));
    for (const auto& [k, x] : ig.iota_argpos) ip.set(std::to_string(k), Value::num(x));
    for (const auto& [k, x] : ig.iota_length) il.set(std::to_string(k), Value::num(x));
    for (const auto& [k, x] : ig.iota_dtype) idt.set(std::to_string(k), Value::str(dtype_name(x)));
    v.set("iota_arg", std::move(ia));
    v.set("iota_index", std::move(ii));
    v.set("iota_output", std::move(io));
    v.set("iota_argpos", std::move(ip));
    v.set("iota_length", std::move(il));
    v.set("iota_dtype", std::move(idt));
    put(out, v);
  });
}

int fe_canonical_labeling(const char* graph_js, char** out) {
  return guarded([&] { put(out, transport::ints_to_json(canonical_labeling(graph_from(fejson::parse(graph_js))).perm)); });
}

int fe_check_compliance(const char* graph_js, char** out) {
  return guarded([&] { put(out, transport::list_to_json(check_compliance(graph_from(fejson::parse(graph_js))))); });
}

int fe_raise(const char* fk, char** out) {
  return guarded([&] {
    const FunctionalKernel k = parse_kernel(fk);
    const RaiseResult rr = raise_to_batched_einsum(k);
    Value v = Value::obj();
    v.set("skeleton", transport::einsum_to_json(rr.f.skeleton));
    v.set("sigma_arg", transport::strmap_to_json(rr.sigma_arg));
    v.set("sigma_idx", transport::strmap_to_json(rr.sigma_idx));
    Value fps = Value::obj();
    for (const auto& [name, op] : rr.f.operand_map) fps.set(name, Value::str(fingerprint(op)));
    v.set("fingerprints", std::move(fps));
    v.set("idealized", Value::boolean_(is_idealized(rr.f)));
    v.set("printed", Value::str(print_kernel(k)));
    put(out, v);
  });
}

int fe_identify(const char* fk, const char* js, char** out) {
  return guarded([&] {
    const MatchResult m = identify_as_einsum(parse_kernel(fk), ein(js));
    Value v = Value::obj();
    v.set("sigma_idx", transport::strmap_to_json(m.sigma_idx));
    v.set("sigma_arg", transport::strmap_to_json(m.sigma_arg));
    v.set("sigma_arg_skeleton", transport::strmap_to_json(m.sigma_arg_skeleton));
    v.set("sigma_row", transport::ints_to_json(m.sigma_row));
    put(out, v);
  });
}

int fe_cost(const char* js, char** out) {
  return guarded([&] {
    const BatchedEinsum e = ein(js);
    Value v = Value::obj();
    v.set("flop_count", Value::dbl(flop_count(e)));
    v.set("footprint_bytes", Value::dbl(footprint_bytes(e)));
    v.set("arithmetic_intensity", Value::dbl(arithmetic_intensity(e)));
    v.set("algorithmic_flops", Value::dbl(feb200::optimal_path_flops(e) * e.b()));
    Value presets = Value::obj();
    for (const DeviceModel& d : device_presets()) {
      Value p = Value::obj();
      p.set("roofline_flop_rate", Value::dbl(roofline_flop_rate(e, d)));
      p.set("memory_bound", Value::boolean_(memory_bound(e, d)));
      presets.set(d.id, std::move(p));
    }
    v.set("presets", std::move(presets));
    put(out, v);
  });
}

int fe_record_facts(const char* path, const char* facts_js) {
  return guarded([&] {
    std::vector<FactRecord> batch;
    for (const auto& f : fejson::parse(facts_js).a) {
      FactRecord r;
      r.canonical_key = f.at("canonical_key").as_str();
      r.device_id = f.at("device_id").as_str();
      r.transform_id = f.at("transform_id").as_str();
      r.wall_time_s = f.at("wall_time_s").as_double();
      r.flop_rate = f.at("flop_rate").as_double();
      if (auto* x = f.find("recorded_at")) r.recorded_at = x->as_str();
      if (auto* x = f.find("meta")) r.meta = x->as_str();
      batch.push_back(std::move(r));
    }
    record_facts(path, batch);
  });
}

int fe_retrieve(const char* path, const char* key, const char* device, char** out) {
  return guarded([&] {
    const auto r = retrieve(path, key, device);
    if (!r) {
      put(out, Value{});
      return;
    }
    Value v = Value::obj();
    v.set("canonical_key", Value::str(r->canonical_key));
    v.set("device_id", Value::str(r->device_id));
    v.set("transform_id", Value::str(r->transform_id));
    v.set("wall_time_s", Value::dbl(r->wall_time_s));
    v.set("flop_rate", Value::dbl(r->flop_rate));
    v.set("recorded_at", Value::str(r->recorded_at));
    v.set("meta", Value::str(r->meta));
    put(out, v);
  });
}

// ------------------------------------------------------------------ plans --

int fe_plan_create(const char* js, const char* options, fe_plan_t* out) {
  return guarded([&] {
    auto h = std::make_unique<fe_plan_s>();
    h->plan = feb200::make_plan(ein(js), feb200::parse_options(options ? options : ""));
    h->options = options ? options : "";
    *out = h.release();
  });
}

int fe_plan_create_kernel(const char* fk, const char* options, fe_plan_t* out) {
  return guarded([&] {
    const FunctionalKernel k = parse_kernel(fk);
    const RaiseResult rr = raise_to_batched_einsum(k);
    auto h = std::make_unique<fe_plan_s>();
    h->plan = feb200::make_functional_plan(rr.f.skeleton, rr.f.operand_map, k.arrays,
                                           feb200::parse_options(options ? options : ""), rr.f.epilogue);
    h->options = options ? options : "";
    *out = h.release();
  });
}

int fe_plan_create_functional(const char* js, const char* options, fe_plan_t* out) {
  return guarded([&] {
    const Value v = fejson::parse(js);
    const BatchedEinsum skel = transport::einsum_from_json(v.at("skeleton"));
    std::map<std::string, OperandExpr> ops;
    for (const auto& [name, o] : v.at("operands").o)
      ops[name] = OperandExpr{transport::list_from_json(o.at("params")), expr_from(o.at("body"))};
    std::map<std::string, ArrayMeta> arrays;
    for (const auto& m : v.at("arrays").a) {
      ArrayMeta meta = transport::meta_from_json(m);
      arrays[meta.name] = meta;
    }
    // extension: "epilogue": [{"row": r, "acc": name, "params": [...], "body": expr}, ...]
    std::map<int, RowEpilogue> epi;
    if (const Value* ev = v.find("epilogue"))
      for (const auto& x : ev->a)
        epi[static_cast<int>(x.at("row").as_int())] =
            RowEpilogue{x.at("acc").as_str(),
                        OperandExpr{transport::list_from_json(x.at("params")), expr_from(x.at("body"))}};
    auto h = std::make_unique<fe_plan_s>();
    h->plan = feb200::make_functional_plan(skel, ops, arrays, feb200::parse_options(options ? options : ""), epi);
    h->options = options ? options : "";
    *out = h.release();
  });
}

int fe_plan_describe(fe_plan_t plan, char** out) {
  return guarded([&] { *out = dup(feb200::describe(*plan->plan)); });
}

int fe_plan_num_inputs(fe_plan_t plan) { return static_cast<int>(plan->plan->leaves.size()); }
int fe_plan_num_outputs(fe_plan_t plan) { return static_cast<int>(plan->plan->outputs.size()); }

int fe_plan_execute(fe_plan_t plan, const void* const* d_in, void* const* d_out, void* stream) {
  return guarded([&] {
    if (!plan->plan->d_blob) throw error(errc::usage, "plan was created with dry_run; it cannot execute");
    feb200::execute(*plan->plan, d_in, d_out, stream);
  });
}

namespace {

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw error(errc::io, std::string(what) + ": " + cudaGetErrorString(e));
}

// Slice of `full` along the one axis where `part` differs (shape-only view).
HostPipe::Slice slice_of(const ArrayMeta& full, const ArrayMeta& part, int storage) {
  HostPipe::Slice sl;
  sl.esize = feb200::storage_bytes(storage);
  for (size_t d = 0; d < full.shape.size(); ++d)
    if (full.shape[d] != part.shape[d]) {
      if (sl.pos >= 0) {
        sl.pos = -2;  // more than one sliced axis: not a simple slice
        return sl;
      }
      sl.pos = static_cast<int>(d);
    }
  if (sl.pos >= 0) {
    for (int d = 0; d < sl.pos; ++d) sl.outer *= full.shape[d];
    for (size_t d = sl.pos + 1; d < full.shape.size(); ++d) sl.inner *= full.shape[d];
    sl.n = full.shape[sl.pos];
  }
  return sl;
}

// host <-> chunk buffer copy of rows [lo, hi) of a sliced array: one 2-D copy
// (measured: per-row copies cost ~3 us of copy-engine time each, e.g. C1 in
// two chunks 380 -> 241 us end to end); FE_COPY_ROWS=<n> copies arrays of up
// to n outer rows row by row instead (A/B)
void copy_slice(const HostPipe::Slice& sl, std::int64_t lo, std::int64_t hi, void* dev, void* host, bool h2d,
                cudaStream_t st) {
  const std::int64_t run = (hi - lo) * sl.inner * sl.esize, pitch = sl.n * sl.inner * sl.esize;
  unsigned char* hbase = static_cast<unsigned char*>(host) + lo * sl.inner * sl.esize;
  unsigned char* dbase = static_cast<unsigned char*>(dev);
  static const std::int64_t row_copies = std::getenv("FE_COPY_ROWS") ? std::atoll(std::getenv("FE_COPY_ROWS")) : 0;
  if (sl.outer <= row_copies) {
    for (std::int64_t o = 0; o < sl.outer; ++o) {
      if (h2d)
        cuda_ok(cudaMemcpyAsync(dbase + o * run, hbase + o * pitch, run, cudaMemcpyHostToDevice, st), "H2D");
      else
        cuda_ok(cudaMemcpyAsync(hbase + o * pitch, dbase + o * run, run, cudaMemcpyDeviceToHost, st), "D2H");
    }
  } else if (h2d) {
    cuda_ok(cudaMemcpy2DAsync(dbase, run, hbase, pitch, run, sl.outer, cudaMemcpyHostToDevice, st), "H2D");
  } else {
    cuda_ok(cudaMemcpy2DAsync(hbase, pitch, dbase, run, run, sl.outer, cudaMemcpyDeviceToHost, st), "D2H");
  }
}

// Build the chunk pipeline of a plan, or nothing when it does not pay (small
// plans) or does not apply (no shard axis).
std::unique_ptr<HostPipe> make_pipe(const fe_plan_s& h) {
  const feb200::Plan& p = *h.plan;
  std::int64_t bytes = 0;
  for (const auto& L : p.leaves) bytes += L.bytes();
  for (const auto& O : p.outputs) bytes += O.bytes();
  const char* thr = std::getenv("FE_PIPE_MIN_MB");
  if (bytes < (static_cast<std::int64_t>(thr ? std::atoi(thr) : 64) << 20)) return nullptr;
  // 8 chunks (measured on the suite: 8 and 16 tie, 32 loses to per-chunk
  // launch and copy overheads); FE_PIPE_CHUNKS overrides for experiments
  const int chunks = std::getenv("FE_PIPE_CHUNKS") ? std::max(2, std::atoi(std::getenv("FE_PIPE_CHUNKS")))
                                                  : feb200::pipe_chunks(p, 8);
  auto pipe = std::make_unique<HostPipe>();
  const feb200::PlanOptions opt = feb200::parse_options(h.options);
  try {
    for (int k = 0; k < chunks; ++k) {
      std::int64_t lo = 0, hi = 0;
      std::string axis;
      pipe->parts.push_back(feb200::make_shard(p, k, chunks, opt, &lo, &hi, &axis));
      pipe->lo.push_back(lo);
      pipe->hi.push_back(hi);
    }
  } catch (const error&) {
    return nullptr;  // no shard axis: the serial path
  }
  const feb200::Plan& first = *pipe->parts[0];
  if (first.leaves.size() != p.leaves.size() || first.outputs.size() != p.outputs.size()) return nullptr;
  for (size_t i = 0; i < p.leaves.size(); ++i) {
    if (first.leaves[i].meta.name != p.leaves[i].meta.name || first.leaves[i].storage != p.leaves[i].storage)
      return nullptr;
    pipe->in_slice.push_back(slice_of(p.leaves[i].meta, first.leaves[i].meta, p.leaves[i].storage));
    if (pipe->in_slice.back().pos == -2) return nullptr;
  }
  for (size_t r = 0; r < p.outputs.size(); ++r) {
    pipe->out_slice.push_back(slice_of(p.outputs[r].meta, first.outputs[r].meta, p.outputs[r].storage));
    if (pipe->out_slice.back().pos < 0) return nullptr;  // every output must be cut by the axis
  }
  std::int64_t widest = 0;
  for (int k = 0; k < chunks; ++k) widest = std::max(widest, pipe->hi[k] - pipe->lo[k]);
  auto alloc = [](std::int64_t n) {
    void* d = nullptr;
    cuda_ok(cudaMalloc(&d, static_cast<size_t>(std::max<std::int64_t>(n, 16))), "cudaMalloc");
    return d;
  };
  for (size_t i = 0; i < p.leaves.size(); ++i) {
    const auto& sl = pipe->in_slice[i];
    pipe->rep_in.push_back(sl.pos < 0 ? alloc(p.leaves[i].bytes()) : nullptr);
    for (int b = 0; b < 2; ++b)
      pipe->slot_in[b].push_back(sl.pos < 0 ? nullptr : alloc(sl.outer * widest * sl.inner * sl.esize));
  }
  for (size_t r = 0; r < p.outputs.size(); ++r) {
    const auto& sl = pipe->out_slice[r];
    for (int b = 0; b < 2; ++b) pipe->slot_out[b].push_back(alloc(sl.outer * widest * sl.inner * sl.esize));
  }
  for (cudaStream_t* q : {&pipe->s_h2d, &pipe->s_comp, &pipe->s_d2h})
    cuda_ok(cudaStreamCreateWithFlags(q, cudaStreamNonBlocking), "stream");
  for (cudaEvent_t* e : {&pipe->start, &pipe->rep_done})
    cuda_ok(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
  for (int b = 0; b < 2; ++b)
    for (cudaEvent_t* e : {&pipe->h2d_done[b], &pipe->comp_done[b], &pipe->d2h_done[b]})
      cuda_ok(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
  return pipe;
}

// FE_PIPE_TRACE=1: timing events per pipeline step, printed to stderr after
// the call (debug aid; synchronises)
struct PipeTrace {
  bool on = std::getenv("FE_PIPE_TRACE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> ev;
  void mark(const std::string& what, cudaStream_t q) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, q);
    ev.emplace_back(what, e);
  }
  ~PipeTrace() {
    if (!on || ev.empty()) return;
    for (auto& [what, e] : ev) {
      cudaEventSynchronize(e);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev.front().second, e);
      std::fprintf(stderr, "pipe %-16s %8.3f ms\n", what.c_str(), ms);
    }
    for (auto& kv : ev) cudaEventDestroy(kv.second);
  }
};

void run_pipe(HostPipe& P, const void* const* h_in, void* const* h_out, cudaStream_t s) {
  const int chunks = static_cast<int>(P.parts.size());
  PipeTrace tr;
  tr.mark("start", s);
  cuda_ok(cudaEventRecord(P.start, s), "event");
  for (cudaStream_t q : {P.s_h2d, P.s_comp, P.s_d2h}) cuda_ok(cudaStreamWaitEvent(q, P.start, 0), "wait");
  // replicated inputs once per call
  for (size_t i = 0; i < P.in_slice.size(); ++i)
    if (P.in_slice[i].pos < 0)
      cuda_ok(cudaMemcpyAsync(P.rep_in[i], h_in[i], static_cast<size_t>(P.parts[0]->leaves[i].bytes()),
                              cudaMemcpyHostToDevice, P.s_h2d),
              "H2D");
  tr.mark("replicated h2d", P.s_h2d);
  for (int k = 0; k < chunks; ++k) {
    const int b = k & 1;
    // H2D of chunk k into slot b, once chunk k-2's kernels have read it
    if (k >= 2) cuda_ok(cudaStreamWaitEvent(P.s_h2d, P.comp_done[b], 0), "wait");
    std::vector<const void*> din(P.in_slice.size());
    for (size_t i = 0; i < P.in_slice.size(); ++i) {
      if (P.in_slice[i].pos < 0) {
        din[i] = P.rep_in[i];
        continue;
      }
      copy_slice(P.in_slice[i], P.lo[k], P.hi[k], P.slot_in[b][i], const_cast<void*>(h_in[i]), true, P.s_h2d);
      din[i] = P.slot_in[b][i];
    }
    cuda_ok(cudaEventRecord(P.h2d_done[b], P.s_h2d), "event");
    tr.mark("h2d " + std::to_string(k), P.s_h2d);
    // kernels of chunk k, once its inputs landed and chunk k-2's outputs left
    cuda_ok(cudaStreamWaitEvent(P.s_comp, P.h2d_done[b], 0), "wait");
    if (k >= 2) cuda_ok(cudaStreamWaitEvent(P.s_comp, P.d2h_done[b], 0), "wait");
    feb200::execute(*P.parts[k], din.data(), P.slot_out[b].data(), P.s_comp);
    cuda_ok(cudaEventRecord(P.comp_done[b], P.s_comp), "event");
    tr.mark("comp " + std::to_string(k), P.s_comp);
    // D2H of chunk k's outputs
    cuda_ok(cudaStreamWaitEvent(P.s_d2h, P.comp_done[b], 0), "wait");
    for (size_t r = 0; r < P.out_slice.size(); ++r)
      copy_slice(P.out_slice[r], P.lo[k], P.hi[k], P.slot_out[b][r], h_out[r], false, P.s_d2h);
    cuda_ok(cudaEventRecord(P.d2h_done[b], P.s_d2h), "event");
    tr.mark("d2h " + std::to_string(k), P.s_d2h);
  }
  // the caller's stream resumes after the last D2H (and with it everything)
  cuda_ok(cudaStreamWaitEvent(s, P.d2h_done[(chunks - 1) & 1], 0), "wait");
  cuda_ok(cudaStreamWaitEvent(s, P.d2h_done[chunks & 1], 0), "wait");
}

}  // namespace

// Row pipeline of a plan, or nothing (one row, functional / complex / path
// plans, or a row that does not plan on its own leaves)
std::unique_ptr<RowPipe> make_rowpipe(const fe_plan_s& h) {
  const feb200::Plan& p = *h.plan;
  if (std::getenv("FE_NO_ROWPIPE") || p.skel.b() < 2 || p.functional || p.complex_mode || !p.tabs.empty() ||
      p.family == feb200::Family::path || p.family == feb200::Family::generic)
    return nullptr;
  auto rp = std::make_unique<RowPipe>();
  const feb200::PlanOptions opt = feb200::parse_options(h.options);
  rp->first_use.assign(p.leaves.size(), -1);
  try {
    for (int r = 0; r < p.skel.b(); ++r) {
      BatchedEinsum row;
      row.i_in = p.skel.i_in;
      row.i_out = p.skel.i_out;
      row.args = {p.skel.args[static_cast<size_t>(r)]};
      rp->rows.push_back(feb200::make_plan(row, opt));
      const feb200::Plan& rpl = *rp->rows.back();
      if (rpl.family != p.family || rpl.outputs[0].storage != p.outputs[static_cast<size_t>(r)].storage) return nullptr;
      std::vector<int> src;
      for (const auto& L : rpl.leaves) {
        int k = -1;
        for (size_t i = 0; i < p.leaves.size(); ++i)
          if (p.leaves[i].meta.name == L.meta.name && p.leaves[i].storage == L.storage) k = static_cast<int>(i);
        if (k < 0) return nullptr;
        if (rp->first_use[static_cast<size_t>(k)] < 0) rp->first_use[static_cast<size_t>(k)] = r;
        src.push_back(k);
      }
      rp->src.push_back(std::move(src));
    }
  } catch (const error&) {
    return nullptr;
  }
  for (cudaStream_t* q : {&rp->s_h2d, &rp->s_comp, &rp->s_d2h})
    cuda_ok(cudaStreamCreateWithFlags(q, cudaStreamNonBlocking), "stream");
  cuda_ok(cudaEventCreateWithFlags(&rp->start, cudaEventDisableTiming), "event");
  for (auto* v : {&rp->h2d_done, &rp->comp_done, &rp->d2h_done}) {
    v->resize(rp->rows.size());
    for (cudaEvent_t& e : *v) cuda_ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  }
  return rp;
}

int fe_plan_execute_host(fe_plan_t plan, const void* const* h_in, void* const* h_out, void* stream) {
  return guarded([&] {
    const feb200::Plan& p = *plan->plan;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!plan->pipe_tried) {
      plan->pipe_tried = true;
      plan->pipe = make_pipe(*plan);
    }
    if (plan->pipe) {
      run_pipe(*plan->pipe, h_in, h_out, s);
      return;
    }
    auto ensure = [](std::vector<void*>& bufs, size_t i, std::int64_t bytes) {
      if (bufs.size() <= i) bufs.resize(i + 1, nullptr);
      if (!bufs[i]) {
        const cudaError_t e = cudaMalloc(&bufs[i], static_cast<size_t>(bytes > 0 ? bytes : 16));
        if (e != cudaSuccess) throw error(errc::io, std::string("cudaMalloc: ") + cudaGetErrorString(e));
      }
      return bufs[i];
    };
    if (!plan->rowpipe_tried) {
      plan->rowpipe_tried = true;
      plan->rowpipe = make_rowpipe(*plan);
    }
    if (RowPipe* rp = plan->rowpipe.get()) {
      // H2D of row r's not yet uploaded leaves | row r's kernels | row r's D2H
      // on three streams; all device buffers are the plan's staging ones
      cuda_ok(cudaEventRecord(rp->start, s), "event");
      for (cudaStream_t q : {rp->s_h2d, rp->s_comp, rp->s_d2h}) cuda_ok(cudaStreamWaitEvent(q, rp->start, 0), "wait");
      for (size_t r = 0; r < rp->rows.size(); ++r) {
        for (size_t i = 0; i < p.leaves.size(); ++i)
          if (rp->first_use[i] == static_cast<int>(r))
            cuda_ok(cudaMemcpyAsync(ensure(plan->staged_in, i, p.leaves[i].bytes()), h_in[i],
                                    static_cast<size_t>(p.leaves[i].bytes()), cudaMemcpyHostToDevice, rp->s_h2d),
                    "H2D");
        cuda_ok(cudaEventRecord(rp->h2d_done[r], rp->s_h2d), "event");
        cuda_ok(cudaStreamWaitEvent(rp->s_comp, rp->h2d_done[r], 0), "wait");
        std::vector<const void*> din;
        for (int k : rp->src[r]) din.push_back(plan->staged_in[static_cast<size_t>(k)]);
        void* dout = ensure(plan->staged_out, r, p.outputs[r].bytes());
        feb200::execute(*rp->rows[r], din.data(), &dout, rp->s_comp);
        cuda_ok(cudaEventRecord(rp->comp_done[r], rp->s_comp), "event");
        cuda_ok(cudaStreamWaitEvent(rp->s_d2h, rp->comp_done[r], 0), "wait");
        cuda_ok(cudaMemcpyAsync(h_out[r], dout, static_cast<size_t>(p.outputs[r].bytes()), cudaMemcpyDeviceToHost,
                                rp->s_d2h),
                "D2H");
        cuda_ok(cudaEventRecord(rp->d2h_done[r], rp->s_d2h), "event");
      }
      cuda_ok(cudaStreamWaitEvent(s, rp->d2h_done.back(), 0), "wait");
      return;
    }
    std::vector<const void*> din;
    for (size_t i = 0; i < p.leaves.size(); ++i) {
      void* d = ensure(plan->staged_in, i, p.leaves[i].bytes());
      const cudaError_t e = cudaMemcpyAsync(d, h_in[i], static_cast<size_t>(p.leaves[i].bytes()),
                                            cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) throw error(errc::io, std::string("H2D: ") + cudaGetErrorString(e));
      din.push_back(d);
    }
    std::vector<void*> dout;
    for (size_t r = 0; r < p.outputs.size(); ++r) dout.push_back(ensure(plan->staged_out, r, p.outputs[r].bytes()));
    feb200::execute(p, din.data(), dout.data(), stream);
    for (size_t r = 0; r < p.outputs.size(); ++r) {
      const cudaError_t e = cudaMemcpyAsync(h_out[r], dout[r], static_cast<size_t>(p.outputs[r].bytes()),
                                            cudaMemcpyDeviceToHost, s);
      if (e != cudaSuccess) throw error(errc::io, std::string("D2H: ") + cudaGetErrorString(e));
    }
  });
}

int fe_plan_tabulate(fe_plan_t plan, const char* operand, const void* const* d_in, double* d_out, int64_t first,
                     int64_t count, void* stream) {
  return guarded([&] { feb200::tabulate(*plan->plan, operand, d_in, d_out, first, count, stream); });
}

int fe_plan_shard(fe_plan_t plan, int rank, int world, const char* options, fe_plan_t* out, int64_t* lo, int64_t* hi,
                  char** axis) {
  return guarded([&] {
    std::string ax;
    auto h = std::make_unique<fe_plan_s>();
    h->plan = feb200::make_shard(*plan->plan, rank, world, feb200::parse_options(options ? options : ""), lo, hi, &ax);
    *axis = dup(ax);
    *out = h.release();
  });
}

int fe_plan_destroy(fe_plan_t plan) {
  delete plan;
  return FE_OK;
}

int fe_plan_time(fe_plan_t plan, int reps, int warmup, uint64_t seed, double* seconds) {
  return guarded([&] {
    const feb200::Plan& p = *plan->plan;
    auto check = [](cudaError_t e, const char* what) {
      if (e != cudaSuccess) throw error(errc::io, std::string(what) + ": " + cudaGetErrorString(e));
    };
    std::vector<void*> ins(p.leaves.size(), nullptr), outs(p.outputs.size(), nullptr);
    void* flush = nullptr;
    constexpr std::int64_t kFlush = std::int64_t{256} << 20;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    auto release = [&] {
      for (void* q : ins) cudaFree(q);
      for (void* q : outs) cudaFree(q);
      cudaFree(flush);
      if (e0) cudaEventDestroy(e0);
      if (e1) cudaEventDestroy(e1);
    };
    try {
      for (size_t i = 0; i < ins.size(); ++i) {
        const std::int64_t n = std::max<std::int64_t>(p.leaves[i].bytes(), 16);
        check(cudaMalloc(&ins[i], static_cast<size_t>(n)), "cudaMalloc");
        check(static_cast<cudaError_t>(feb200::fill_dyadic(ins[i], p.leaves[i].storage, p.leaves[i].meta.num_elements(),
                                                           seed * 1000 + i, nullptr)),
              "fill");
      }
      for (size_t r = 0; r < outs.size(); ++r)
        check(cudaMalloc(&outs[r], static_cast<size_t>(std::max<std::int64_t>(p.outputs[r].bytes(), 16))), "cudaMalloc");
      check(cudaMalloc(&flush, kFlush), "cudaMalloc");
      check(cudaEventCreate(&e0), "event");
      check(cudaEventCreate(&e1), "event");
      for (int w = 0; w < warmup; ++w) feb200::execute(p, ins.data(), outs.data(), nullptr);
      double total = 0.0;
      for (int r = 0; r < reps; ++r) {
        check(static_cast<cudaError_t>(feb200::flush_l2(flush, kFlush, nullptr)), "flush");
        check(cudaEventRecord(e0, nullptr), "event");
        feb200::execute(p, ins.data(), outs.data(), nullptr);
        check(cudaEventRecord(e1, nullptr), "event");
        check(cudaEventSynchronize(e1), "sync");
        float ms = 0.f;
        check(cudaEventElapsedTime(&ms, e0, e1), "event");
        total += ms * 1e-3;
      }
      *seconds = reps > 0 ? total / reps : 0.0;
    } catch (...) {
      release();
      throw;
    }
    release();
  });
}

int fe_fill_dyadic(void* d_ptr, int storage, int64_t count, uint64_t seed, void* stream) {
  return cuda_status(feb200::fill_dyadic(d_ptr, storage, count, seed, stream));
}

int fe_flush_l2(void* d_scratch, int64_t bytes, void* stream) {
  return cuda_status(feb200::flush_l2(d_scratch, bytes, stream));
}

int fe_fp64_peak(int which, double* tflops) { return cuda_status(feb200::fp64_peak(which, tflops)); }

int fe_launch_probe(void* stream) { return cuda_status(feb200::launch_probe(stream)); }

int fe_sm_count(void) {
  int n = 0;
  if (feb200::device_sm_count(&n) != 0) return -1;
  return n;
}

}  // extern "C"
