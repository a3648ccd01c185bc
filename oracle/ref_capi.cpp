// TEST ORACLE — not product code. A C-ABI shim over the UNMODIFIED reference
// library (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/). Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it, and only as the checker or
// the timed CPU baseline — never as part of the product path.
//
// Every entry point returns 0 on success or 1 + feinsum::errc on failure
// (domain=1, usage=2, io=3; 9 = non-feinsum exception); the message is in
// ref_last_error(). Structured results are JSON strings freed by ref_free().
// Arrays cross as interleaved complex<double> (numpy complex128) because the
// reference evaluator holds every dtype as complex<double>
// (proj/include/feinsum/core.hpp:125-134).

#include <cstdint>
#include <cstring>
#include <string>

#include "feinsum/canonicalize.hpp"
#include "feinsum/core.hpp"
#include "feinsum/factsdb.hpp"
#include "feinsum/graph_canon.hpp"
#include "feinsum/induced_graph.hpp"
#include "feinsum/notation.hpp"
#include "feinsum/raising.hpp"
#include "feinsum/rng.hpp"
#include "ref_json.hpp"

using namespace feinsum;
using oj::Value;

namespace {

thread_local std::string g_err;

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const feinsum::error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.kind());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

BatchedEinsum ein(const char* js) { return ot::einsum_from_json(oj::parse(js)); }

Value canon_to_json(const CanonResult& c) {
  Value v = Value::obj();
  v.set("canonical", ot::einsum_to_json(c.canonical));
  v.set("sigma_idx", ot::strmap_to_json(c.sigma_idx));
  v.set("sigma_arg", ot::strmap_to_json(c.sigma_arg));
  v.set("sigma_row", ot::ints_to_json(c.sigma_row));
  v.set("sigma_slot", ot::ints_to_json(c.sigma_slot));
  return v;
}

Value graph_to_json(const ColoredDigraph& g) {
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

ColoredDigraph graph_from_json(const Value& v) {
  ColoredDigraph g = ColoredDigraph::empty(static_cast<int>(v.at("n").as_int()));
  int k = 0;
  for (const auto& c : v.at("colors").a) g.colors[k++] = static_cast<int>(c.as_int());
  for (const auto& e : v.at("edges").a)
    g.set_edge(static_cast<int>(e.a[0].as_int()), static_cast<int>(e.a[1].as_int()));
  return g;
}

void put(char** out, const Value& v) { *out = dup(oj::dump(v)); }

Bindings bind_universe(const BatchedEinsum& e, const double* const* in_c) {
  Bindings b;
  size_t k = 0;
  for (const ArrayMeta& m : universe(e)) {
    DenseArray a = DenseArray::zeros(m);
    const double* src = in_c[k++];
    for (size_t i = 0; i < a.data.size(); ++i) a.data[i] = {src[2 * i], src[2 * i + 1]};
    b.emplace(m.name, std::move(a));
  }
  return b;
}

void write_rows(const std::vector<DenseArray>& rows, double* const* out_c) {
  for (size_t r = 0; r < rows.size(); ++r)
    for (size_t i = 0; i < rows[r].data.size(); ++i) {
      out_c[r][2 * i] = rows[r].data[i].real();
      out_c[r][2 * i + 1] = rows[r].data[i].imag();
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(char* p) { std::free(p); }

int ref_parse_classic(const char* text, char** out) {
  return guard([&] { put(out, ot::einsum_to_json(parse_classic(text))); });
}

int ref_print_classic(const char* js, char** out) {
  return guard([&] { *out = dup(print_classic(ein(js))); });
}

int ref_validate(const char* js, char** out) {
  return guard([&] { put(out, ot::list_to_json(validate(ein(js)))); });
}

int ref_canonicalize(const char* js, char** out) {
  return guard([&] {
    CanonResult c = canonicalize(ein(js));
    Value v = canon_to_json(c);
    v.set("key", Value::str(canonical_key(c.canonical)));
    put(out, v);
  });
}

int ref_canonical_key(const char* js, char** out) {
  return guard([&] { *out = dup(canonical_key(ein(js))); });
}

int ref_generate_random(const char* params_js, std::uint64_t seed, char** out) {
  return guard([&] {
    GenParams p;
    Value pv = oj::parse(params_js);
    if (auto* x = pv.find("b_min")) p.b_min = static_cast<int>(x->as_int());
    if (auto* x = pv.find("b_max")) p.b_max = static_cast<int>(x->as_int());
    if (auto* x = pv.find("n_min")) p.n_min = static_cast<int>(x->as_int());
    if (auto* x = pv.find("n_max")) p.n_max = static_cast<int>(x->as_int());
    if (auto* x = pv.find("max_indices")) p.max_indices = static_cast<int>(x->as_int());
    if (auto* x = pv.find("max_dim")) p.max_dim = static_cast<int>(x->as_int());
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
    put(out, ot::einsum_to_json(generate_random(p, seed)));
  });
}

int ref_scramble(const char* js, std::uint64_t seed, char** out) {
  return guard([&] {
    Scrambled s = scramble(ein(js), seed);
    Value v = Value::obj();
    v.set("e", ot::einsum_to_json(s.e));
    v.set("w", ot::witness_to_json(s.w));
    put(out, v);
  });
}

int ref_is_isomorphic(const char* a, const char* b, char** out) {
  return guard([&] {
    auto w = is_isomorphic(ein(a), ein(b));
    put(out, w ? ot::witness_to_json(*w) : Value{});
  });
}

int ref_brute_force_isomorphic(const char* a, const char* b, std::uint64_t budget, char** out) {
  return guard([&] {
    auto w = brute_force_isomorphic(ein(a), ein(b), budget);
    put(out, w ? ot::witness_to_json(*w) : Value{});
  });
}

int ref_verify_witness(const char* a, const char* b, const char* w, char** out) {
  return guard([&] {
    std::vector<std::string> why;
    bool ok = verify_witness(ein(a), ein(b),
                             ot::witness_from_json<SubstitutionWitness>(oj::parse(w)), &why);
    Value v = Value::obj();
    v.set("ok", Value::boolean_(ok));
    v.set("why", ot::list_to_json(why));
    put(out, v);
  });
}

int ref_induced_graph(const char* js, std::int64_t shuffle_seed, char** out) {
  return guard([&] {
    std::optional<std::uint64_t> seed;
    if (shuffle_seed >= 0) seed = static_cast<std::uint64_t>(shuffle_seed);
    InducedGraph ig = to_induced_graph(ein(js), seed);
    Value v = graph_to_json(ig.graph);
    Value ia = Value::obj(), ii = Value::obj(), io = Value::obj(), ip = Value::obj(),
          il = Value::obj(), idt = Value::obj();
    for (auto& [k, x] : ig.iota_arg) ia.set(std::to_string(k), Value::str(x));
    for (auto& [k, x] : ig.iota_index) ii.set(std::to_string(k), Value::str(x));
    for (auto& [k, x] : ig.iota_output) io.set(std::to_string(k), Value::num(x));
    for (auto& [k, x] : ig.iota_argpos) ip.set(std::to_string(k), Value::num(x));
    for (auto& [k, x] : ig.iota_length) il.set(std::to_string(k), Value::num(x));
    for (auto& [k, x] : ig.iota_dtype) idt.set(std::to_string(k), Value::str(dtype_name(x)));
    v.set("iota_arg", std::move(ia));
    v.set("iota_index", std::move(ii));
    v.set("iota_output", std::move(io));
    v.set("iota_argpos", std::move(ip));
    v.set("iota_length", std::move(il));
    v.set("iota_dtype", std::move(idt));
    put(out, v);
  });
}

int ref_canonical_labeling(const char* graph_js, char** out) {
  return guard([&] {
    Relabeling r = canonical_labeling(graph_from_json(oj::parse(graph_js)));
    put(out, ot::ints_to_json(r.perm));
  });
}

int ref_check_compliance(const char* graph_js, char** out) {
  return guard([&] {
    put(out, ot::list_to_json(check_compliance(graph_from_json(oj::parse(graph_js)))));
  });
}

int ref_evaluate(const char* js, const double* const* in_c, double* const* out_c) {
  return guard([&] {
    BatchedEinsum e = ein(js);
    write_rows(evaluate(e, bind_universe(e, in_c)), out_c);
  });
}

// Kernel text -> raise_to_batched_einsum -> evaluate_functional. in_c holds
// the kernel's declared arrays in name order (FunctionalKernel::arrays is a
// std::map); out_c one buffer per statement row of the raised skeleton.
int ref_eval_kernel(const char* fk, const double* const* in_c, double* const* out_c) {
  return guard([&] {
    FunctionalKernel k = parse_kernel(fk);
    RaiseResult rr = raise_to_batched_einsum(k);
    Bindings b;
    size_t i = 0;
    for (const auto& [name, m] : k.arrays) {
      DenseArray a = DenseArray::zeros(m);
      const double* src = in_c[i++];
      for (size_t t = 0; t < a.data.size(); ++t) a.data[t] = {src[2 * t], src[2 * t + 1]};
      b.emplace(name, std::move(a));
    }
    write_rows(evaluate_functional(rr.f, b), out_c);
  });
}

int ref_raise(const char* fk, char** out) {
  return guard([&] {
    FunctionalKernel k = parse_kernel(fk);
    RaiseResult rr = raise_to_batched_einsum(k);
    Value v = Value::obj();
    v.set("skeleton", ot::einsum_to_json(rr.f.skeleton));
    v.set("sigma_arg", ot::strmap_to_json(rr.sigma_arg));
    v.set("sigma_idx", ot::strmap_to_json(rr.sigma_idx));
    Value fps = Value::obj();
    for (const auto& [name, op] : rr.f.operand_map) fps.set(name, Value::str(fingerprint(op)));
    v.set("fingerprints", std::move(fps));
    v.set("idealized", Value::boolean_(is_idealized(rr.f)));
    v.set("printed", Value::str(print_kernel(k)));
    put(out, v);
  });
}

int ref_identify(const char* fk, const char* js, char** out) {
  return guard([&] {
    MatchResult m = identify_as_einsum(parse_kernel(fk), ein(js));
    Value v = Value::obj();
    v.set("sigma_idx", ot::strmap_to_json(m.sigma_idx));
    v.set("sigma_arg", ot::strmap_to_json(m.sigma_arg));
    v.set("sigma_arg_skeleton", ot::strmap_to_json(m.sigma_arg_skeleton));
    v.set("sigma_row", ot::ints_to_json(m.sigma_row));
    put(out, v);
  });
}

int ref_cost(const char* js, char** out) {
  return guard([&] {
    BatchedEinsum e = ein(js);
    Value v = Value::obj();
    v.set("flop_count", Value::dbl(flop_count(e)));
    v.set("footprint_bytes", Value::dbl(footprint_bytes(e)));
    v.set("arithmetic_intensity", Value::dbl(arithmetic_intensity(e)));
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

int ref_record_facts(const char* path, const char* facts_js) {
  return guard([&] {
    std::vector<FactRecord> batch;
    for (const auto& f : oj::parse(facts_js).a) {
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

int ref_retrieve(const char* path, const char* key, const char* device, char** out) {
  return guard([&] {
    auto r = retrieve(path, key, device);
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

// test::random_bindings (proj/tests/test_util.hpp:19-29): one mt19937_64
// stream, arrays filled back to back in universe order, value m/2^19 - 1.
void ref_random_fill(std::uint64_t seed, int n_arrays, const std::int64_t* sizes, double** out) {
  std::mt19937_64 rng(seed);
  for (int a = 0; a < n_arrays; ++a)
    for (std::int64_t i = 0; i < sizes[a]; ++i)
      out[a][i] = static_cast<double>(draw_below(rng, 1u << 20)) / (1u << 19) - 1.0;
}

}  // extern "C"
