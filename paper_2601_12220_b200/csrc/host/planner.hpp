// B200 planner: turns a (functional) batched einsum into an executable plan.
//
//   parse -> validate -> canonicalize (normal form + sigma maps)
//         -> canonical key -> tuning facts (device "b200")
//         -> kernel family matched on the canonical form, operands routed to
//            the caller's buffers by the sigma maps (pointer permutation only)
//         -> sm_100a launch
//
// Functional operands are compiled once per plan into device programs
// (affine fast path or a register VM) that the kernels evaluate in their
// operand prologue. Every plan also carries the generic-kernel launch so any
// einsum runs on the GPU; there is no host evaluation path.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "feinsum/canonicalize.hpp"
#include "feinsum/core.hpp"
#include "feinsum/factsdb.hpp"
#include "feinsum/raising.hpp"
#include "../kernels/launch.h"

struct CUevent_st;
namespace feb200 {

using feinsum::ArrayMeta;
using feinsum::BatchedEinsum;
using feinsum::CanonResult;
using feinsum::Dtype;
using feinsum::OperandExpr;

enum class Family { generic, fem_grad, gett, tt, hex, path };
const char* family_transform(Family f);  // "generic/v1", "fem_grad/v1", ...

struct PlanOptions {
  std::string storage = "native";              // "native" | "wide"
  std::map<std::string, std::string> storage_of;  // per-leaf override: f64 c128 f32 c64 ...
  std::string facts_path;                     // default: bundled facts/b200.facts
  std::string device_id = "b200";
  std::string force_transform;                // e.g. "generic/v1"
  bool canonicalize = true;
  bool force_vm = false;      // internal: point evaluation (eval_expr)
  bool skip_range_check = false;
  bool dry_run = false;       // plan without touching the device (CPU tests)
  std::string meta_override;  // tuner: run these parameters instead of the fact's
  bool codegen = true;        // NVRTC tabulation kernels for VM operands (false: device VM)
};

PlanOptions parse_options(const std::string& json);

struct LeafInfo {
  ArrayMeta meta;
  int storage;
  std::int64_t bytes() const { return meta.num_elements() * storage_bytes(storage); }
};

struct OutputInfo {
  ArrayMeta meta;  // name R<row>, widest dtype of the row, shape of i_out
  int storage;
  std::int64_t bytes() const { return meta.num_elements() * storage_bytes(storage); }
};

// Roles of the FEM-gradient family bound to the caller's operands.
struct FemBinding {
  int NX, NR, NI, NJ;
  std::int64_t E;
  int rows;
  // per canonical row: leaf indices / output row
  std::vector<int> j_leaf, d_leaf, out_row;
  std::vector<std::vector<AffineTerm>> u_terms;  // per row; leaf indices
  bool f32 = false;  // every array float32 (fp32 kernel instance)
};

// Roles of the GETT family (dense 2-operand contraction on DMMA).
struct GettBinding {
  std::int64_t ext_mo = 0, ext_mi = 0, ext_no = 0, ext_ni = 0, ext_ka = 0, ext_kb = 0;
  std::int64_t a_mo = 0, a_mi = 0, a_kb = 0, b_no = 0, b_ni = 0, b_ka = 0;
  std::int64_t c_mo = 0, c_mi = 0, c_no = 0, c_ni = 0;
  std::string role_names;  // "mo=a mi=b ..." for describe()
  std::string shard_m;     // canonical name of the M index shards split (outer M index)
  // operands whose unit-stride index is not their contracted one are repacked
  // per execute into a plan buffer laid out [mo][mi][kB][kA] (A) or
  // [no][ni][kA][kB] (B); *_src are the source strides in that dim order
  bool pack_a = false, pack_b = false;
  // fp32 operands are widened into the pack buffers (the reference computes
  // float32 in double, so the f64 DMMA path is its arithmetic); an fp32
  // output is accumulated in d_cbuf and narrowed once
  bool a_f32 = false, b_f32 = false, c_f32 = false;
  // batch index (in A, B and C; split form only): nz values; kernel strides
  // a_z / b_z (after a repack: the packed block size), source strides for
  // the repack, C stride
  std::int64_t nz = 1, a_z = 0, b_z = 0, a_z_src = 0, b_z_src = 0, c_z = 0;
  int ksplit = 1;  // split-K slices for small tile counts (plan workspace d_ws)
  std::int64_t a_src[4] = {0, 0, 0, 0}, b_src[4] = {0, 0, 0, 0};
  struct Row {
    int a_leaf, b_leaf, out_row;
    int a_alpha, a_beta, b_alpha, b_beta;
  };
  std::vector<Row> rows;
};

// Roles of the tensor-train family: Y[n,i,k] = sum G1[i,j] G2[k,l] X[n,j,l].
struct TTBinding {
  std::int64_t nb = 0;
  int NI = 0, NJ = 0, NK = 0, NL = 0;
  bool fp32 = false;
  struct Row {
    int g1, g2, x, out_row;
  };
  std::vector<Row> rows;
};

// Roles of the hex sum-factorised family (C2).
struct HexBinding {
  std::int64_t E = 0;
  int ND = 0, P = 0;
  int mats[6] = {-1, -1, -1, -1, -1, -1};  // leaf of F1 F2 F3 B1 B2 B3
  int g = -1;
  std::vector<int> u, out_row;  // per canonical row
  bool f32 = false;             // every array float32 (fp32 instance of the v2 kernel)
};

struct Plan;

// One pairwise step of a contraction path (Family::path): a 2-operand plan
// whose inputs are caller arrays or earlier intermediates.
struct PathStep {
  std::unique_ptr<Plan> plan;
  std::vector<int> src;  // per step-plan input: caller leaf (>= 0) or intermediate -(1 + id)
  int out = -1;          // intermediate id, or -1: the caller's output out_row
  int out_row = 0;
};

struct Plan {
  // ---- what is computed ----
  BatchedEinsum skel;  // the caller's einsum (skeleton if functional)
  bool functional = false;
  std::map<std::string, OperandExpr> operand_exprs;  // functional: skeleton name -> expr
  std::vector<LeafInfo> leaves;    // execution inputs, in order
  std::vector<OutputInfo> outputs; // one per caller row, in caller row order
  std::vector<OperandStatic> ops;  // [row * n + slot], caller order
  std::vector<VmInstr> prog;
  std::vector<VmRead> reads;
  std::vector<CoefChain> chains;
  bool complex_mode = false;

  // VM operands of a real-valued functional plan are tabulated at the start of
  // every execute into plan buffers (the reference's materialize, on the
  // device, bit-identical values) and read as plain f64 leaves, so the tuned
  // families take them too. Synthetic leaf k has index leaves.size() + k; its
  // program is the VM original kept at ops[op]. Empty when the plan runs the
  // generic kernel (which evaluates the programs in place).
  struct TabOperand {
    std::string name;  // skeleton operand
    int op;            // index of the VM original in ops (past the b * n slots)
    std::int64_t count, offset;  // elements, offset in d_tab (doubles)
    void* kernel = nullptr;       // NVRTC-compiled tabulation kernel (codegen.cpp), or the VM
    std::vector<int> leaf_slots;  // its leaf slots -> plan leaf indices
    std::string codegen;          // "nvrtc" | "vm: <why>"
  };
  std::vector<TabOperand> tabs;
  std::vector<LeafInfo> tab_leaves;
  double* d_tab = nullptr;

  // ---- normal form and retrieval ----
  bool has_canon = false;
  CanonResult canon;
  std::string key;
  std::string transform;  // chosen kernel family
  std::string meta;       // tuned parameters (fact meta or defaults)
  std::string source;     // "fact" | "default" | "forced" | "fallback"
  Family family = Family::generic;
  FemBinding fem;
  GettBinding gett;
  TTBinding tt;
  HexBinding hex;
  // contraction path (n >= 3 operands, every step on a tuned family)
  std::vector<PathStep> path;
  std::vector<std::int64_t> inter_off;  // intermediate id -> byte offset in d_inter
  std::int64_t inter_bytes = 0;
  void* d_inter = nullptr;

  // ---- costs ----
  double alg_flops = 0, operand_flops = 0, bytes = 0, ref_flops = 0;

  // ---- device state ----
  int device = 0;
  void* d_blob = nullptr;
  double* d_coef = nullptr;
  bool coef_static = false;     // every chain is literal: coefficients uploaded once, no per-execute kernel
  double* d_scratch = nullptr;  // family workspace (GETT affine K-sums)
  double* d_pack_a = nullptr;   // GETT repacked operands (see GettBinding)
  double* d_pack_b = nullptr;
  double* d_cbuf = nullptr;     // GETT f64 result staging for fp32 outputs
  double* d_ws = nullptr;       // GETT split-K partial tiles
  // ---- extension: row epilogues (RowEpilogue) and the generated fem_grad
  // instance (codegen.cpp) that fuses operand programs and epilogues ----
  std::map<int, feinsum::RowEpilogue> epilogue;  // caller row -> post-op, as given
  std::vector<OperandStatic> epi_ops;  // per caller row: OPK_VM program (acc reads leaf kAccLeaf), or kind -1
  struct EpiPass {
    void* kernel = nullptr;            // NVRTC in-place pass over the row's output
    std::vector<int> leaf_slots;
  };
  std::vector<EpiPass> epi_pass;       // per caller row (unfused families)
  void* fem_rtc = nullptr;             // generated fem_grad instance (prologue programs + epilogues), or null
  int fem_rtc_te = 0, fem_rtc_ept = 0;
  std::vector<std::vector<int>> fem_rtc_tiles;  // per canonical row: staged U leaf tiles
  std::vector<int> fem_rtc_aux;                 // FemGradLaunch::aux slot -> plan leaf
  std::string fem_rtc_note;                     // describe(): "nvrtc" or why not
  ::CUevent_st* last_use = nullptr;  // cudaEvent_t; orders executes that share the scratch above (null: no scratch)
  GenericLaunch gen{};  // pointers filled per execution
  int sm_count = 148;

  ~Plan();
};

// VmRead::leaf of an epilogue's read of its own row value (RowEpilogue::acc).
constexpr int kAccLeaf = -2;

// Generated tabulation kernels (codegen.cpp).
constexpr int kTabLeaves = 16;
struct TabArgs {
  const void* leaf[kTabLeaves];
  double* out;
  long long count;
};
std::string tab_kernel_source(const Plan& p, const OperandStatic& op, const ArrayMeta& meta,
                              std::vector<int>* leaf_slots);
std::string epi_kernel_source(const Plan& p, const OperandStatic& op, const ArrayMeta& out_meta, int out_storage,
                              std::vector<int>* leaf_slots);
std::string fem_rtc_source(const Plan& p, int te, int ept, bool dsmem, std::vector<std::vector<int>>* u_tiles,
                           std::vector<int>* aux, std::string* why);
void* compile_tab_kernel(const std::string& src, std::string* log);
void* compile_rtc_kernel(const std::string& src, const char* name, std::string* log);
bool nvrtc_compiles(const std::string& src, std::string* log);
int launch_tab_kernel(void* kernel, const TabArgs& args, int sm_count, void* stream);

// Leaf i of the plan: a caller input, or (i >= leaves.size()) a tabulated operand.
const LeafInfo& leaf_info(const Plan& p, int i);

std::unique_ptr<Plan> make_plan(const BatchedEinsum& e, const PlanOptions& opt);
std::unique_ptr<Plan> make_functional_plan(const BatchedEinsum& skeleton,
                                           const std::map<std::string, OperandExpr>& operands,
                                           const std::map<std::string, ArrayMeta>& arrays,
                                           const PlanOptions& opt,
                                           const std::map<int, feinsum::RowEpilogue>& epilogue = {});

// Enqueue the plan on `stream` with device pointers (inputs in plan->leaves
// order, outputs in caller row order). Stream-ordered, allocation-free.
void execute(const Plan& plan, const void* const* d_in, void* const* d_out, void* stream);

// Shard plan for rank/world along the family's shard axis.
std::unique_ptr<Plan> make_shard(const Plan& full, int rank, int world, const PlanOptions& opt,
                                 std::int64_t* lo, std::int64_t* hi, std::string* axis);

// Chunks of the host pipeline (fe_plan_execute_host) for this plan.
int pipe_chunks(const Plan& p, int dflt);

std::string describe(const Plan& plan);  // JSON

// Algorithmic FLOPs of one row: cheapest pairwise contraction order.
double optimal_path_flops(const BatchedEinsum& e);

// Tabulate one operand program on the device (materialize / eval_expr).
void tabulate(const Plan& plan, const std::string& skeleton_name, const void* const* d_in, double* d_out,
              std::int64_t first, std::int64_t count, void* stream);

// Storage code <-> name ("f64", "c128", ...), and the native storage of a dtype.
int storage_from_name(const std::string& s);
const char* storage_name(int st);
int native_storage(Dtype t);

// Bundled facts file path (next to the shared library).
std::string default_facts_path();

}  // namespace feb200
