/* TEST ORACLE — not product code. Plain-C restatement of the reference dense
 * evaluator feinsum::evaluate (proj/src/core.cpp:269-358) for ONE row, used
 * by tests/ to pin the restatement against oracle/_ref and as a second,
 * independent checker. Only tests/, smoke() and bench.py's cpu_baseline leg
 * may call it.
 *
 * Semantics restated from the reference:
 *  - loop symbols = i_out, then the reduction indices in first-occurrence
 *    order (core.cpp:281-293); the caller passes each operand's per-dim
 *    loop-symbol position and row-major stride (core.cpp:309-324);
 *  - for every output point (odometer, last output symbol fastest,
 *    core.cpp:350-354) and every reduction point (odometer, last reduction
 *    symbol fastest, core.cpp:343-346) the term is the complex product of the
 *    slot values, left to right from 1+0i (core.cpp:335-340);
 *  - the terms of one output point are added with pairwise_sum: <= 8 terms
 *    sequentially from 0+0i, otherwise split at n/2 (core.cpp:259-267).
 * Complex multiply is the schoolbook (ac-bd, ad+bc) form, which is what the
 * reference build computes for finite inputs (no FMA contraction: compiled
 * with -ffp-contract=off, like oracle/_ref).
 */
#include <stdint.h>
#include <stdlib.h>

typedef struct {
  double re, im;
} cplx;

static cplx pairwise(const cplx* p, int64_t n) {
  if (n <= 8) {
    cplx s = {0.0, 0.0};
    for (int64_t i = 0; i < n; ++i) {
      s.re += p[i].re;
      s.im += p[i].im;
    }
    return s;
  }
  int64_t h = n / 2;
  cplx a = pairwise(p, h), b = pairwise(p + h, n - h);
  cplx s = {a.re + b.re, a.im + b.im};
  return s;
}

/* n_syms loop symbols with extents; the first n_out are output symbols.
 * Slot k has ndim[k] dims; pos/stride are flattened over slots (offset =
 * sum of ndim of earlier slots). data[k] points to interleaved complex
 * doubles. out receives prod(output extents) interleaved complex values.
 * Returns 0, or -1 on allocation failure. */
int port_evaluate_row(int n_syms, const int64_t* extent, int n_out, int n_slots, const int* ndim,
                      const int* pos, const int64_t* stride, const double* const* data,
                      double* out) {
  int64_t out_points = 1, red_points = 1;
  for (int i = 0; i < n_syms; ++i) {
    if (i < n_out)
      out_points *= extent[i];
    else
      red_points *= extent[i];
  }
  cplx* terms = (cplx*)malloc(sizeof(cplx) * (size_t)(red_points > 0 ? red_points : 1));
  int64_t* val = (int64_t*)calloc((size_t)(n_syms > 0 ? n_syms : 1), sizeof(int64_t));
  if (!terms || !val) {
    free(terms);
    free(val);
    return -1;
  }
  for (int64_t op = 0; op < out_points; ++op) {
    for (int64_t rp = 0; rp < red_points; ++rp) {
      cplx prod = {1.0, 0.0};
      int base = 0;
      for (int k = 0; k < n_slots; ++k) {
        int64_t off = 0;
        for (int d = 0; d < ndim[k]; ++d) off += val[pos[base + d]] * stride[base + d];
        base += ndim[k];
        double c = data[k][2 * off], dd = data[k][2 * off + 1];
        double a = prod.re, b = prod.im;
        volatile double ac = a * c, bd = b * dd, ad = a * dd, bc = b * c;
        prod.re = ac - bd;
        prod.im = ad + bc;
      }
      terms[rp] = prod;
      for (int i = n_syms; i-- > n_out;) {
        if (++val[i] < extent[i]) break;
        val[i] = 0;
      }
    }
    cplx s = pairwise(terms, red_points);
    out[2 * op] = s.re;
    out[2 * op + 1] = s.im;
    for (int i = n_out; i-- > 0;) {
      if (++val[i] < extent[i]) break;
      val[i] = 0;
    }
  }
  free(terms);
  free(val);
  return 0;
}
