// The C++ drop-in: code written against the reference headers
// (proj/include/feinsum/*.hpp) compiles unchanged against include/feinsum and
// links libfeinsum_b200.so. Checks mirror the reference's own doctest cases
// (proj/tests/test_core.cpp, test_canonicalize.cpp, test_notation.cpp,
// test_raising.cpp, test_factsdb.cpp) with a minimal assertion harness
// (doctest is not vendored). `dropin_test host` runs the host-side checks,
// `dropin_test gpu` adds evaluate()/evaluate_functional() on the device.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <unistd.h>

#include "feinsum/canonicalize.hpp"
#include "feinsum/core.hpp"
#include "feinsum/factsdb.hpp"
#include "feinsum/notation.hpp"
#include "feinsum/raising.hpp"
#include "feinsum/rng.hpp"

using namespace feinsum;

static int failures = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (!(cond)) {                                                       \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
      ++failures;                                                        \
    }                                                                    \
  } while (0)

static ArrayMeta am(std::string n, std::vector<std::int64_t> s, Dtype t = Dtype::float64) {
  return ArrayMeta{std::move(n), std::move(s), t};
}

// test::random_bindings (proj/tests/test_util.hpp:19-29)
static Bindings random_bindings(const BatchedEinsum& e, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  Bindings b;
  for (const auto& a : universe(e)) {
    DenseArray arr = DenseArray::zeros(a);
    for (auto& x : arr.data) x = {static_cast<double>(draw_below(rng, 1u << 20)) / (1u << 19) - 1.0, 0.0};
    b.emplace(a.name, std::move(arr));
  }
  return b;
}

static void host_checks() {
  // worked golden (test_canonicalize.cpp:23-39, test_notation.cpp:126-130)
  auto e1 = make_batched("ij,ik->i", {{am("A", {72, 18}), am("B", {72, 18})}});
  auto c = canonicalize(e1);
  CHECK(c.canonical == make_batched("ab,ac->a", {{am("A0", {72, 18}), am("A1", {72, 18})}}));
  CHECK((c.sigma_idx == std::map<std::string, std::string>{{"a", "i"}, {"b", "j"}, {"c", "k"}}));
  CHECK(c.sigma_row == std::vector<int>{0});
  CHECK((c.sigma_slot == std::vector<int>{0, 1}));
  CHECK(canonical_key(c.canonical) == "FE1|b=1|n=2|out=a|in=ab;ac|rows=A0,A1|A0=float64:72x18|A1=float64:72x18");
  CHECK(verify_witness(e1, c.canonical, canonical_witness(c)));
  // batched key (test_notation.cpp:131-135)
  auto sq = parse_classic(
      "einsum: ij,j->i\nrow: A,B\nrow: A,C\narray: A float64 96x4\narray: B float64 4\narray: C float64 4\n");
  CHECK(canonical_key(canonicalize(sq).canonical) ==
        "FE1|b=2|n=2|out=b|in=ba;a|rows=A0,A1;A0,A2|A0=float64:96x4|A1=float64:4|A2=float64:4");
  // scramble sweep (test_canonicalize.cpp:106-118)
  GenParams p;
  for (std::uint64_t seed = 500; seed < 560; ++seed) {
    auto e = generate_random(p, seed);
    auto s = scramble(e, seed * 31 + 7);
    CHECK(verify_witness(s.e, e, s.w));
    CHECK(canonicalize(s.e).canonical == canonicalize(e).canonical);
  }
  // errors carry the reference wording
  try {
    canonical_key(e1);
    CHECK(false);
  } catch (const error& err) {
    CHECK(std::string(err.what()) == "canonical_key wants a canonical form; canonicalize first");
    CHECK(err.kind() == errc::domain);
  }
  // kernel identification (Alg. 2) on the squared kernel fixture
  const char* fk =
      "domain: i0<96 i1<4\n"
      "def u(i,j) := P[i,j]*P[i,j]\n"
      "def v(i) := 3*cos(Q[i])+5\n"
      "def w(i) := sin(R[i])\n"
      "array: P float64 96x4\narray: Q float64 4\narray: R float64 4\n"
      "stmt y1[i0] = sum([i1], u(i0,i1)*v(i1))\n"
      "stmt y2[i0] = sum([i1], u(i0,i1)*w(i1))\n";
  auto m = identify_as_einsum(parse_kernel(fk), sq);
  CHECK(m.sigma_row.size() == 2);
  // facts: record, retrieve the cheapest (test_factsdb.cpp:172-205)
  char tmpl[] = "/tmp/fe_facts_XXXXXX";
  const int fd = mkstemp(tmpl);
  close(fd);
  std::remove(tmpl);
  const std::string path = tmpl;
  const std::string key = canonical_key(c.canonical);
  record_facts(path, {FactRecord{key, "b200", "gett_dmma/v1", 2.0, 1.0, "2026-01-01T00:00:00.000000Z", "a"},
                      FactRecord{key, "b200", "generic/v1", 1.0, 2.0, "2026-01-01T00:00:00.000000Z", "b"}});
  auto best = retrieve(path, key, "b200");
  CHECK(best && best->transform_id == "generic/v1");
  CHECK(!retrieve(path, key, "h100"));
  std::remove(path.c_str());
  std::remove((path + ".lock").c_str());
  // cost model (test_factsdb.cpp:207-237)
  auto mm = make_batched("ik,kj->ij", {{am("A", {10, 4}), am("B", {4, 10})}});
  CHECK(flop_count(mm) == 2.0 * 10 * 4 * 10);
  CHECK(footprint_bytes(mm) == (40 + 40 + 100) * 8.0);
}

static void gpu_checks() {
  // evaluate vs a hand-rolled matmul (test_core.cpp:154-174)
  auto e = make_batched("ik,kj->ij", {{am("A", {10, 4}), am("B", {4, 10})}});
  auto bind = random_bindings(e, 42);
  auto got = evaluate(e, bind);
  CHECK(got.size() == 1 && got[0].meta.name == "R1" && got[0].meta.shape == (std::vector<std::int64_t>{10, 10}));
  const auto& A = bind.at("A").data;
  const auto& B = bind.at("B").data;
  double worst = 0;
  for (int i = 0; i < 10; ++i)
    for (int j = 0; j < 10; ++j) {
      std::complex<double> s = 0.0;
      for (int k = 0; k < 4; ++k) s += A[i * 4 + k] * B[k * 10 + j];
      worst = std::max(worst, std::abs(got[0].data[i * 10 + j] - s) / std::max(1.0, std::abs(s)));
    }
  CHECK(worst < 1e-13);
  // complex without conjugation: (i)(i) + (1)(2) = 1 exactly
  auto ec = make_batched("i,i->", {{am("x", {2}, Dtype::complex128), am("y", {2}, Dtype::complex128)}});
  Bindings bc;
  bc["x"] = DenseArray{am("x", {2}, Dtype::complex128), {{0, 1}, {1, 0}}};
  bc["y"] = DenseArray{am("y", {2}, Dtype::complex128), {{0, 1}, {2, 0}}};
  CHECK(evaluate(ec, bc)[0].data[0] == std::complex<double>(1.0, 0.0));
  // widest dtype per row (test_core.cpp:211-218)
  auto ew = make_batched("i,i->i", {{am("x", {3}, Dtype::float32), am("y", {3}, Dtype::float64)},
                                    {am("x", {3}, Dtype::float32), am("z", {3}, Dtype::int8)}});
  auto rw = evaluate(ew, random_bindings(ew, 17));
  CHECK(rw[0].meta.dtype == Dtype::float64 && rw[1].meta.dtype == Dtype::float32);
  // missing binding message
  try {
    evaluate(make_batched("i->i", {{am("x", {5})}}), {});
    CHECK(false);
  } catch (const error& err) {
    CHECK(std::string(err.what()) == "no binding for array x");
  }
  // functional operands: squared kernel vs a hand loop (test_raising.cpp:291-317)
  const char* fk =
      "domain: i0<96 i1<4\n"
      "def u(i,j) := P[i,j]*P[i,j]\n"
      "def v(i) := 3*cos(Q[i])+5\n"
      "def w(i) := sin(R[i])\n"
      "array: P float64 96x4\narray: Q float64 4\narray: R float64 4\n"
      "stmt y1[i0] = sum([i1], u(i0,i1)*v(i1))\n"
      "stmt y2[i0] = sum([i1], u(i0,i1)*w(i1))\n";
  auto k = parse_kernel(fk);
  auto rr = raise_to_batched_einsum(k);
  BatchedEinsum carrier{{"i"}, {{"i", "j"}, {"j"}, {"j"}}, {{k.arrays.at("P"), k.arrays.at("Q"), k.arrays.at("R")}}};
  auto fb = random_bindings(carrier, 5);
  auto fr = evaluate_functional(rr.f, fb);
  const auto& P = fb.at("P").data;
  const auto& Q = fb.at("Q").data;
  const auto& R = fb.at("R").data;
  worst = 0;
  for (int i = 0; i < 96; ++i) {
    std::complex<double> s1 = 0, s2 = 0;
    for (int j = 0; j < 4; ++j) {
      const auto u = P[i * 4 + j] * P[i * 4 + j];
      s1 += u * (3.0 * std::cos(Q[j]) + 5.0);
      s2 += u * std::sin(R[j]);
    }
    worst = std::max({worst, std::abs(fr[0].data[i] - s1), std::abs(fr[1].data[i] - s2)});
  }
  CHECK(worst < 1e-12);
  // eval_expr / materialize (device tabulation)
  auto one = eval_expr(k.defs.at("v"), {2}, fb);
  CHECK(std::abs(one - (3.0 * std::cos(Q[2]) + 5.0)) < 1e-14);
  auto mat = materialize(k.defs.at("u"), ArrayMeta{"u", {96, 4}, Dtype::float64}, fb);
  CHECK(mat.data[7] == P[7] * P[7]);
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "host";
  host_checks();
  if (mode == "gpu") gpu_checks();
  std::printf("%s: %d failure(s)\n", mode.c_str(), failures);
  return failures == 0 ? 0 : 1;
}
