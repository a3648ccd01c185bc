/* feinsum B200 — C-ABI of the evaluation path.
 *
 * This is the thin, plain-pointer boundary the north star asks for: the C++
 * drop-in (the include/feinsum headers, same signatures as the reference headers)
 * and the Python mirror (paper_2601_12220_b200/feinsum.py) both sit on it.
 * No torch or C++ types cross it: structured values travel as JSON text,
 * arrays as raw device (or host) pointers, streams as cudaStream_t cast to
 * void*.
 *
 * The reference has no FFI of its own: its public C++ API is
 * the contract. Each entry point below names the reference function it
 * replaces or exposes (file:line under /root/reference/proj).
 *
 * Status codes: 0 ok; 1 + feinsum::errc (1 domain, 2 usage, 3 io); 4 CUDA
 * error; 5 internal. The message of the last failure on the calling thread is
 * fe_last_error(). Returned strings are heap-allocated: release with fe_free.
 */
#ifndef FEINSUM_B200_H_
#define FEINSUM_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FE_OK 0
#define FE_ERR_DOMAIN 1
#define FE_ERR_USAGE 2
#define FE_ERR_IO 3
#define FE_ERR_CUDA 4
#define FE_ERR_INTERNAL 5

/* storage codes of device buffers (see DESIGN.md §data layout) */
#define FE_ST_F64 0
#define FE_ST_F32 1
#define FE_ST_C128 2
#define FE_ST_C64 3
#define FE_ST_I8 4
#define FE_ST_I32 5
#define FE_ST_I64 6
#define FE_ST_F16 7

typedef struct fe_plan_s* fe_plan_t;

const char* fe_last_error(void);
void fe_free(void* p);
int fe_version(void);
/* FE_OK when a CUDA device is usable, FE_ERR_IO otherwise (message says why) */
int fe_device_check(void);

/* ---- host side: normal forms, keys, retrieval (JSON in / JSON out) ---- */

/* parse_classic, notation.hpp:33 / notation.cpp:137 */
int fe_parse_classic(const char* es_text, char** out_einsum_json);
/* print_classic, notation.hpp:34 / notation.cpp:235 */
int fe_print_classic(const char* einsum_json, char** out_text);
/* validate, core.hpp:70 / core.cpp:63 -> JSON list of messages */
int fe_validate(const char* einsum_json, char** out_json);
/* canonicalize, canonicalize.hpp:25 / canonicalize.cpp:11 ->
 * {"canonical","sigma_idx","sigma_arg","sigma_row","sigma_slot","key"} */
int fe_canonicalize(const char* einsum_json, char** out_json);
/* canonical_key, notation.hpp:44 / notation.cpp:251 (input must be canonical) */
int fe_canonical_key(const char* einsum_json, char** out_key);
/* is_isomorphic, canonicalize.hpp:35 -> witness JSON or null */
int fe_is_isomorphic(const char* a_json, const char* b_json, char** out_json);
/* brute_force_isomorphic, canonicalize.hpp:41 */
int fe_brute_force_isomorphic(const char* a_json, const char* b_json, uint64_t budget, char** out_json);
/* verify_witness, canonicalize.hpp:31 -> {"ok":bool,"why":[...]} */
int fe_verify_witness(const char* a_json, const char* b_json, const char* w_json, char** out_json);
/* generate_random / scramble, canonicalize.hpp:57-69 */
int fe_generate_random(const char* params_json, uint64_t seed, char** out_json);
int fe_scramble(const char* einsum_json, uint64_t seed, char** out_json);
/* to_induced_graph / canonical_labeling / check_compliance (graph JSON:
 * {"n","colors","edges":[[i,j],...], iota maps}) */
int fe_induced_graph(const char* einsum_json, int64_t shuffle_seed, char** out_json);
int fe_canonical_labeling(const char* graph_json, char** out_json);
int fe_check_compliance(const char* graph_json, char** out_json);
/* parse_kernel + raise_to_batched_einsum, raising.hpp:91-103 */
int fe_raise(const char* fk_text, char** out_json);
/* identify_as_einsum (Alg. 2), raising.hpp:119 */
int fe_identify(const char* fk_text, const char* einsum_json, char** out_json);
/* flop_count / footprint_bytes / roofline presets, factsdb.hpp:43-60,
 * plus the B200 algorithmic (optimal pairwise path) FLOP count */
int fe_cost(const char* einsum_json, char** out_json);
/* record_facts / retrieve, factsdb.hpp:31-36 */
int fe_record_facts(const char* path, const char* facts_json);
int fe_retrieve(const char* path, const char* key, const char* device, char** out_json);

/* ---- device side: plans (replace evaluate, core.hpp:141, and
 *      evaluate_functional, raising.hpp:58) ---- */

/* options JSON (all optional): {"storage": "native"|"wide", "leaf_storage": {name: "f64"|...},
 *  "facts": path, "device": "b200", "transform": "generic/v1"|..., "meta": "k=v;...",
 *  "codegen": true|false (NVRTC tabulation kernels for non-affine operands; false: device VM),
 *  "dry_run": true (plan on the host only)} */
int fe_plan_create(const char* einsum_json, const char* options_json, fe_plan_t* out);
/* .fk kernel text: inputs = declared arrays in name order, one output per stmt */
int fe_plan_create_kernel(const char* fk_text, const char* options_json, fe_plan_t* out);
/* {"skeleton": einsum, "operands": {name: {"params": [...], "body": expr}},
 *  "arrays": [meta, ...]} with expr = {"lit":x} | {"param":p} |
 *  {"read":A,"subs":[...]} | {"fn":f,"x":expr} | {"op":"+","l":expr,"r":expr} */
int fe_plan_create_functional(const char* json, const char* options_json, fe_plan_t* out);
/* key, transform, source, inputs/outputs (name, shape, dtype, storage,
 * bytes), FLOP and byte counts, canonical form and sigma maps */
int fe_plan_describe(fe_plan_t plan, char** out_json);
int fe_plan_num_inputs(fe_plan_t plan);
int fe_plan_num_outputs(fe_plan_t plan);
/* stream-ordered; never allocates; d_in in describe().inputs order, d_out one
 * buffer per caller row */
int fe_plan_execute(fe_plan_t plan, const void* const* d_in, void* const* d_out, void* stream);
/* end-to-end: host inputs -> H2D -> kernels -> D2H into host outputs, ordered
 * on `stream` (device staging buffers are owned by the plan; not
 * synchronized). Plans above 64 MB run as a pipeline of chunks (8; GETT: by wave fill) along the
 * shard axis: chunk k's H2D, chunk k-1's kernels and chunk k-2's D2H overlap
 * on internal streams (host buffers should be pinned for the copies to
 * overlap); smaller plans with several rows (plain real operands) run one
 * single-row plan per row so row r's D2H overlaps row r+1's kernels; either
 * way the outputs equal fe_plan_execute's bitwise and `stream` resumes after
 * the last D2H. Not for concurrent calls on one plan (the staging buffers and
 * pipelines are the plan's). */
int fe_plan_execute_host(fe_plan_t plan, const void* const* h_in, void* const* h_out, void* stream);
/* tabulate one skeleton operand (materialize, raising.hpp:43) into
 * interleaved complex doubles */
int fe_plan_tabulate(fe_plan_t plan, const char* operand, const void* const* d_in, double* d_out, int64_t first,
                     int64_t count, void* stream);
/* shard of a plan for rank/world along the family's element/batch axis;
 * writes the half-open range [lo, hi) and the axis name */
int fe_plan_shard(fe_plan_t plan, int rank, int world, const char* options_json, fe_plan_t* out, int64_t* lo,
                  int64_t* hi, char** axis);
int fe_plan_destroy(fe_plan_t plan);
/* mean device time (CUDA events, L2 flushed before every run) of one execute
 * on synthetic dyadic inputs allocated and filled on the current device; the
 * measurement the tuner records as a fact's wall_time_s */
int fe_plan_time(fe_plan_t plan, int reps, int warmup, uint64_t seed, double* out_seconds);

/* ---- device utilities for tests and benches ---- */
/* deterministic dyadic values m/2^19 - 1 (the reference's random_bindings
 * value grid) written on the device */
int fe_fill_dyadic(void* d_ptr, int storage, int64_t count, uint64_t seed, void* stream);
/* overwrite `bytes` of scratch (>= L2 size), then read it back, to evict L2
 * between timed runs and leave it clean */
int fe_flush_l2(void* d_scratch, int64_t bytes, void* stream);
int fe_sm_count(void);
/* measured FP64 throughput of the current device, TFLOP/s: which = 0 DFMA,
 * 1 DMMA (the FP64 roofline denominator; MEASURED_PEAKS.json has none),
 * 2 half the warps each (shared datapath?), 100 + w: DFMA with w warps/SM */
int fe_fp64_peak(int which, double* tflops);
/* launch one empty kernel on `stream` (the launch-latency floor a timed
 * single execute cannot go below) */
int fe_launch_probe(void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FEINSUM_B200_H_ */
