// Host <-> device launch contracts of the sm_100a kernels. Plain C++ structs
// (no CUDA headers) shared by the planner (host .cpp) and the kernels (.cu).
// The planner fills these from a Plan; each launch_* function enqueues its
// kernel(s) on the given stream and returns a cudaError_t as int.
#pragma once

#include "rtc_std.h"

namespace feb200 {

// Device storage of an array. NATIVE storage follows the declared dtype; the
// DenseArray drop-in uploads "wide" (F64/C128) so values survive unrounded,
// exactly as the reference holds them (complex<double> for every dtype).
enum Storage : int {
  ST_F64 = 0,
  ST_F32 = 1,
  ST_C128 = 2,
  ST_C64 = 3,
  ST_I8 = 4,
  ST_I32 = 5,
  ST_I64 = 6,
  ST_F16 = 7,
};

inline int storage_bytes(int s) {
  switch (s) {
    case ST_F64: return 8;
    case ST_F32: return 4;
    case ST_C128: return 16;
    case ST_C64: return 8;
    case ST_I8: return 1;
    case ST_I32: return 4;
    case ST_I64: return 8;
    case ST_F16: return 2;
  }
  return 0;
}
inline bool storage_complex(int s) { return s == ST_C128 || s == ST_C64; }

constexpr int kMaxSyms = 32;
constexpr int kMaxDims = 12;
constexpr int kMaxLeaves = 96;
constexpr int kMaxRows = 96;
constexpr int kMaxAffineTerms = 4;
constexpr int kMaxVmRegs = 16;

// ---- operand programs (static, uploaded once per plan) ----

enum OperandKind : int { OPK_PLAIN = 0, OPK_AFFINE = 1, OPK_VM = 2 };

// value = fold_{t} (acc (+|-) term_t), term = [coef[pre] *] leaf[flat] [* coef[post0]] [* coef[post1]]
// A term with leaf < 0 is the constant coef[pre].
struct AffineTerm {
  int sign;   // +1 add, -1 subtract (ignored for the first term)
  int pre;    // coefficient slot or -1
  int leaf;   // leaf index or -1
  int post0;  // coefficient slot or -1
  int post1;  // coefficient slot or -1
};

struct OperandStatic {
  int kind;
  int leaf;     // OPK_PLAIN: leaf index
  int n_terms;  // OPK_AFFINE
  AffineTerm term[kMaxAffineTerms];
  int prog_off, prog_len;  // OPK_VM: instruction range in the program table
  int ndim;                // operand rank (number of parameters)
};

enum VmCode : int {
  VM_LIT = 0,    // r[dst] = imm
  VM_PARAM,      // r[dst] = params[arg]
  VM_READ,       // r[dst] = leaf read, descriptor reads[arg]
  VM_ADD,
  VM_SUB,
  VM_MUL,
  VM_DIV,
  VM_SIN,
  VM_COS,
  VM_EXP,
  VM_SQRT,
  VM_RECIP,
};

struct VmInstr {
  int code;
  int dst, a, b;
  int arg;
  double imm;
};

struct VmRead {
  int leaf;
  int ndim;
  int param_of[kMaxDims];           // which operand parameter indexes each axis
  std::int64_t stride[kMaxDims];    // row-major strides of the leaf
};

// Coefficient chains for affine operands: coef[c] = f0 * f1 * ... (left fold),
// each factor a literal or a 0-dim leaf read. Evaluated by a tiny kernel at the
// start of every execution (leaf pointers change per call).
struct CoefFactor {
  int leaf;    // -1 = literal
  double lit;
};
constexpr int kMaxCoefFactors = 4;
struct CoefChain {
  int n;
  CoefFactor f[kMaxCoefFactors];
};

// ---- generic strided evaluator (any einsum; bit-exact order) ----

struct LeafTable {
  const void* ptr[kMaxLeaves];
  int storage[kMaxLeaves];
};

struct GenericLaunch {
  // device pointers into the plan's static blob
  const OperandStatic* ops;   // [b * n], row-major over (row, slot)
  const int* slot_pos;        // [n * kMaxDims]
  const std::int64_t* slot_stride;  // [n * kMaxDims]
  const int* slot_ndim;       // [n]
  const VmInstr* prog;
  const VmRead* reads;
  const CoefChain* chains;
  int n_chains;
  double* coef;               // device scratch [n_chains * 2] (re, im)
  int n_syms, n_out, b, n;
  std::int64_t extent[kMaxSyms];
  std::int64_t out_points, red_points;
  bool complex_mode;
  int out_storage[kMaxRows];  // per row: ST_F64/ST_C128/...
  LeafTable leaves;
  void* out[kMaxRows];
};

int launch_generic(const GenericLaunch& p, void* stream);

// Tabulate one operand over its shape (materialize / eval_expr).
struct TabulateLaunch {
  const OperandStatic* op;
  const VmInstr* prog;
  const VmRead* reads;
  const CoefChain* chains;
  int n_chains;
  double* coef;
  int ndim;
  std::int64_t shape[kMaxDims];
  std::int64_t count;        // points to produce
  std::int64_t first;        // flat index of the first point
  bool complex_mode;
  LeafTable leaves;
  double* out;               // interleaved complex (re, im) per point
  bool real_out;             // or: one double (re) per point (tabulated operands)
};

int launch_tabulate(const TabulateLaunch& p, void* stream);

// ---- K1: FEM gradient  y[q][r,e,i] = sum_{x,j} J_q[x,r,e] D_q[x,i,j] U_q[e,j] ----
// Canonical layouts: J [NX, NR, E], D [NX, NI, NJ], U leaves [E, NJ],
// Y [NR, E, NI] (all row-major). U_q is an affine combination of staged leaf
// tiles (plain operand = one term, no coefficients).
constexpr int kFemMaxRows = 16;
constexpr int kFemMaxUTiles = 32;
constexpr int kFemMaxAux = 16;

struct FemGradLaunch {
  int rows;
  std::int64_t E;
  int NX, NR, NI, NJ;
  int tile_e;  // elements per pipeline stage
  int stages;
  int grid;    // persistent CTAs
  int n_j, n_d, n_u;
  const double* J[kFemMaxRows];  // distinct J arrays
  const double* D[kFemMaxRows];  // distinct D arrays
  int row_j[kFemMaxRows], row_d[kFemMaxRows];
  const double* U[kFemMaxUTiles];  // staged U leaves, grouped by row
  int u_sign[kFemMaxUTiles], u_pre[kFemMaxUTiles], u_post[kFemMaxUTiles];
  int row_u_first[kFemMaxRows], row_u_count[kFemMaxRows];
  bool plain_u;        // every row: one term, no coefficients
  bool d_in_smem;      // D read from shared memory (2 CTAs/SM) instead of registers
  bool mma;            // fem_mma.cu: inner contraction on DMMA (fp64 tensor cores)
  int ept;             // elements per consumer thread (1 or 2)
  bool f32;            // J, D, U, Y are float (pointers reinterpreted); E % 4 == 0
  const double* coef;  // interleaved complex coefficients (real part used)
  double* Y[kFemMaxRows];
  // plan-time generated instances (codegen.cpp): arrays the fused operand
  // programs / epilogues read outside the staged tiles
  const void* aux[kFemMaxAux];
};

int launch_fem_grad(const FemGradLaunch& p, void* stream);
// an NVRTC-compiled instance (codegen.cpp) of the same kernel body with tile
// shape (te, ept): grid, block and shared memory sized like the prebuilt ones
int launch_fem_grad_rtc(const FemGradLaunch& p, void* kernel, int te, int ept, void* stream);
bool fem_grad_supported(int NX, int NR, int NI, int NJ);
int launch_fem_mma(const FemGradLaunch& p, void* stream);
bool fem_mma_supported(int NX, int NR, int NI, int NJ);

// evaluate coefficient chains into coef (interleaved complex)
int launch_coef(const CoefChain* chains, int n_chains, const LeafTable& leaves, double* coef, void* stream);

// ---- K3: dense 2-operand contraction (TCCG GETT) on DMMA ----
// C[mo,mi,no,ni] = sum_{kA,kB} A[mo,mi,kB,kA] B[no,ni,kA,kB], roles bound to
// arbitrary index positions through strides (elements). kA is A's unit-stride
// index, kB is B's; ni is the tile index of C (unit stride for vector stores).
struct GettLaunch {
  std::int64_t ext_mo, ext_mi, ext_no, ext_ni, ext_ka, ext_kb;
  std::int64_t a_mo, a_mi, a_kb;  // A strides (a_ka == 1)
  std::int64_t b_no, b_ni, b_ka;  // B strides (b_kb == 1)
  std::int64_t c_mo, c_mi, c_no, c_ni;
  const double* A;
  const double* B;
  double* C;
  // optional affine prologue: value = coef[alpha] * x + coef[beta] (-1 = none)
  int a_alpha, a_beta, b_alpha, b_beta;
  const double* coef;
  double* scratch;  // ext_mo*ext_mi + ext_no*ext_ni doubles (affine operands' K-sums)
  int stages, group, grid;
  // batch: an index of A, B and C (nz values, strides a_z / b_z / c_z; no
  // affine operands); nz <= 1 = none
  std::int64_t nz, a_z, b_z, c_z;
  // split K (small tile counts): ksplit slices into ws (ksplit x the dense
  // C size, C's strides), summed into C by a second pass; 0 / 1 = off
  int ksplit;
  double* ws;
};

int launch_gett(const GettLaunch& p, void* stream);
bool gett_supported(std::int64_t ext_mi, std::int64_t ext_ni, std::int64_t ext_ka, std::int64_t ext_kb);

// ---- K4: tensor-train layer  Y[n,i,k] = sum_{j,l} G1[i,j] G2[k,l] X[n,j,l] ----
// Layouts: G1 [i,j], G2 [k,l] row-major; X [n,j,l] with unit l stride; Y [n,i,k].
struct TTLaunch {
  std::int64_t Nb;  // batch (samples)
  int NI, NJ, NK, NL;
  int fp32;  // 1: float storage (fp64 accumulation), 0: double
  const void* G1;
  const void* G2;
  const void* X;
  void* Y;
  std::int64_t x_sj, x_sn, y_sn;
  int stages;
};

int launch_tt(const TTLaunch& p, void* stream);
bool tt_supported(int NI, int NJ, int NK, int NL, bool fp32);
// fp32 on the tcgen05 tensor cores (3xTF32), tt_tc.cu
int launch_tt_tc(const TTLaunch& p, void* stream);
bool tt_tc_supported(const TTLaunch& p);

// ---- K5: hex sum-factorized operator ----
// y_q[e,i,m,n] = sum B1[x,a,i] B2[x,b,m] B3[x,c,n] G[x,y,e,a,b,c]
//                    F1[y,a,j] F2[y,b,k] F3[y,c,l] u_q[e,j,k,l]
// (C2 uses B_d = F_d = A_d). Layouts as written, row-major.
struct HexLaunch {
  std::int64_t E;
  int ND;    // 3 directions
  int P;     // points = dofs per direction (5 for P4)
  int rows;  // fields, <= 8
  const double* mats[6];  // F1 F2 F3 B1 B2 B3, each [ND, P, P]
  const double* G;        // [ND, ND, E, P, P, P]
  const double* U[8];
  double* Y[8];
  int variant;  // 2 (default): constant-bank operators, plane/line passes, C/A of consecutive stages merged
                //   when rows == 8; 3: the three-barrier v2 kernel; 5: merged without the pass-B split;
                //   1: register-plane passes
  int ne;       // v2 elements per stage: 4 (default when E % 4 == 0) or 2
  bool f32;     // every array float (pointers reinterpreted; v2 only, E % 4 == 0 below Q = 6)
};

int launch_hex(const HexLaunch& p, void* stream);
int hex_prepare(int device);  // plan time: operator staging + ordering event
bool hex_supported(int nd, int p, std::int64_t E, int rows);

// ---- utilities ----
int device_sm_count(int* out);
int fill_dyadic(void* ptr, int storage, std::int64_t count, std::uint64_t seed, void* stream);
int flush_l2(void* scratch, std::int64_t bytes, void* stream);
// dst[i0][i1][i2][i3] (contiguous, extents ext[0..3]) = src[sum_d i_d * src_stride[d]]:
// repacks a strided operand into a kernel's layout (GETT operands whose
// unit-stride index is not a contracted one)
// nz > 1: a batch of nz blocks, src stride src_z, packed back to back in dst
int permute4(const double* src, double* dst, const std::int64_t ext[4], const std::int64_t src_stride[4], void* stream,
             std::int64_t nz = 1, std::int64_t src_z = 0);
// the same from an fp32 source, widened to fp64; and a dense fp64 -> fp32 copy
int permute4_widen(const float* src, double* dst, const std::int64_t ext[4], const std::int64_t src_stride[4], void* stream,
                   std::int64_t nz = 1, std::int64_t src_z = 0);
int narrow_f64_f32(const double* src, float* dst, std::int64_t n, void* stream);
// which: 0 = DFMA (CUDA cores), 1 = DMMA m8n8k4 (FP64 tensor cores)
int fp64_peak(int which, double* tflops);
int launch_probe(void* stream);

}  // namespace feb200
