/*
 * gfb.h -- C ABI of the B200 gradient-program engine (libgfb.so).
 *
 * The reference executes forward and reverse-mode programs with a scalar
 * Python tree-walking interpreter (gradflow, pkg/src/gradflow/interpreter.py).
 * The host lowering in paper_2509_02197_b200/lowering.py walks the same IR
 * and issues these entry points instead; each one replaces one interpreter
 * routine, cited per entry below.
 *
 * Conventions
 *   - plain C types only: device pointers, int64 extents/offsets, doubles;
 *   - every call is asynchronous on the given cudaStream_t (passed as void*);
 *   - no allocation inside a call: workspaces are passed in;
 *   - return 0 on success, a GFB_E* status otherwise (launch/config errors);
 *   - arithmetic-domain faults inside kernels (x/0, log(<=0), ...) are
 *     reported through the device error word `err` (GFB_EBIT_* bits), which
 *     the host reads after the stream synchronises and maps to the
 *     reference's DomainError (pkg/src/gradflow/errors.py:56).
 */
#ifndef GFB_H
#define GFB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GFB_ABI_VERSION 12

#define GFB_MAX_PARAMS 8    /* map parameters (iteration-space rank) */
#define GFB_MAX_RANK 8      /* array rank */
#define GFB_MAX_INPUTS 8    /* operands read by one tasklet */
#define GFB_MAX_OUTPUTS 8   /* outputs written by one tasklet */
#define GFB_MAX_CODE 128    /* bytecode length (all outputs together) */
#define GFB_MAX_CONSTS 24
#define GFB_MAX_TAPS 32     /* taps of one linear stencil */
#define GFB_MAX_SRCS 4      /* source arrays of one linear stencil */

enum gfb_dtype { GFB_F32 = 0, GFB_F64 = 1 };

enum gfb_status {
  GFB_OK = 0,
  GFB_EINVAL = 1,      /* malformed descriptor */
  GFB_ECUDA = 2,       /* CUDA launch failure */
  GFB_EUNSUPPORTED = 3 /* shape outside what the kernel family handles */
};

/* device error word bits (eager domain errors, reference symexpr.py:81-133) */
#define GFB_EBIT_DIV0 0x1u
#define GFB_EBIT_LOG 0x2u
#define GFB_EBIT_SQRT 0x4u
#define GFB_EBIT_POW 0x8u
#define GFB_EBIT_IDIV0 0x10u
#define GFB_EBIT_MOD0 0x20u

/* tasklet bytecode (postfix; one segment per output connector) */
enum gfb_op {
  GFB_OP_IN = 0,    /* push input operand [arg] at the current point */
  GFB_OP_CONST = 1, /* push consts[arg] */
  GFB_OP_ADD, GFB_OP_SUB, GFB_OP_MUL, GFB_OP_DIV, GFB_OP_IDIV, GFB_OP_MOD,
  GFB_OP_MIN, GFB_OP_MAX, GFB_OP_POW,
  GFB_OP_NEG, GFB_OP_SIN, GFB_OP_COS, GFB_OP_EXP, GFB_OP_LOG, GFB_OP_SQRT,
  GFB_OP_TANH, GFB_OP_ABS, GFB_OP_SIGN,
  GFB_OP_COUNT
};

/*
 * Map iteration space (reference MapNode, ir.py:107-116): parameter p runs
 * over [lo_p, hi_p) with step st_p, where lo_p / hi_p are affine in the
 * earlier parameters (triangular spaces):
 *     lo_p = lo0[p] + sum_{q<p} loc[p][q] * x_q     (same for hi)
 * box_lo/box_ext is the host-computed bounding box the thread grid covers.
 */
typedef struct {
  int32_t nparams;
  int32_t triangular; /* 0: ranges independent (box == space) */
  int64_t lo0[GFB_MAX_PARAMS];
  int64_t hi0[GFB_MAX_PARAMS];
  int64_t step[GFB_MAX_PARAMS];
  int64_t loc[GFB_MAX_PARAMS][GFB_MAX_PARAMS];
  int64_t hic[GFB_MAX_PARAMS][GFB_MAX_PARAMS];
  int64_t box_lo[GFB_MAX_PARAMS];
  int64_t box_ext[GFB_MAX_PARAMS]; /* number of points along p in the box */
} gfb_space;

/* One memlet endpoint: element offset = c0 + sum_p s[p] * x_p (elements). */
typedef struct {
  void *base;
  int32_t dtype;
  int32_t _pad;
  int64_t c0;
  int64_t s[GFB_MAX_PARAMS];
} gfb_operand;

/*
 * Pointwise map: one thread per iteration point, every output written by the
 * point that computes it (reference Executor._exec_map + _exec_tasklet,
 * interpreter.py:478-507, :405-426). Host lowering guarantees the outputs are
 * point-private (injective subsets, no cross-point read-after-write), so the
 * per-point read-all-then-write order of the reference is preserved.
 *   wcr[o] = 0 overwrite, 1 sum (plain read-modify-write), 2 sum (atomic)
 */
typedef struct {
  gfb_space space;
  int32_t n_in, n_out;
  int32_t compute_f64;
  int32_t ncode;
  gfb_operand in[GFB_MAX_INPUTS];
  gfb_operand out[GFB_MAX_OUTPUTS];
  int32_t wcr[GFB_MAX_OUTPUTS];
  int32_t code_start[GFB_MAX_OUTPUTS];
  int32_t code_len[GFB_MAX_OUTPUTS];
  uint8_t code[GFB_MAX_CODE];
  uint8_t arg[GFB_MAX_CODE];
  double consts[GFB_MAX_CONSTS];
  uint32_t *err;
} gfb_map_desc;

/*
 * Gather pass: the scatter-add outputs of one map that land in one array D
 * (wcr="sum" memlets, reference autodiff.py:1053-1060) executed output-
 * stationary and atomic-free. Thread groups own target elements y of D inside
 * ybox; for each contributing output memlet ("term") the map parameters are
 * split into pivots (solved from y) and free parameters (looped):
 *     x_piv = (y_row - off_row - sum_{q != piv} C[row][q] x_q) / C[row][piv]
 * Every candidate point is range- and step-checked against the space.
 * Result: D[y] = base(y) + sum_terms sum_points body(x), where base(y) is
 *     clear_mode 0: D[y]                    (accumulate)
 *     clear_mode 1: 0                       (target known zero: overwrite)
 *     clear_mode 2: y in clear box ? 0 : D[y]  (folded pending gradient clear)
 * Large free loops split over `nsplit` CTAs per target tile; partials then go
 * to `workspace` ([nsplit][|ybox|] of the target dtype) and gfb_gather_launch
 * finishes them with a deterministic second pass.
 */
typedef struct {
  int32_t row_of[GFB_MAX_PARAMS];   /* -1: free parameter, else pivot row */
  int32_t order[GFB_MAX_PARAMS];    /* evaluation order of the pivots */
  int32_t npiv;
  int32_t code_start, code_len;
  int32_t _pad;
  int64_t C[GFB_MAX_RANK][GFB_MAX_PARAMS]; /* subset coefficients (-1,0,1) */
  int64_t off[GFB_MAX_RANK];
} gfb_term;

typedef struct {
  gfb_space space;
  int32_t rank;        /* rank of D */
  int32_t dtype;       /* dtype of D */
  int32_t compute_f64;
  int32_t n_in;
  int32_t n_terms;
  int32_t clear_mode;
  int32_t lanes_on_free; /* 1: a warp cooperates on one target (coalesced free loop) */
  int32_t nsplit;
  void *dst;
  int64_t dst_strides[GFB_MAX_RANK];
  int64_t ybox_lo[GFB_MAX_RANK];
  int64_t ybox_ext[GFB_MAX_RANK];
  int64_t clear_lo[GFB_MAX_RANK];
  int64_t clear_hi[GFB_MAX_RANK];
  int64_t free_lo[GFB_MAX_PARAMS];  /* per term-free parameter loop box */
  int64_t free_ext[GFB_MAX_PARAMS];
  gfb_operand in[GFB_MAX_INPUTS];
  gfb_term terms[4];
  uint8_t code[GFB_MAX_CODE];
  uint8_t arg[GFB_MAX_CODE];
  double consts[GFB_MAX_CONSTS];
  void *workspace;
  uint32_t *err;
} gfb_gather_desc;

/*
 * Linear stencil sweep (fast path for maps whose tasklet is a constant-
 * coefficient linear combination of shifted reads, and for the gather form
 * of their adjoints; reference adj_map autodiff.py:962-1081):
 *     D[y] = base(y) + sum_t [y in mask_t] * coef_t * S_{src_t}[y + delta_t]
 * for y in [lo, hi) (rank <= 3, row-major, innermost dimension contiguous).
 * base(y) follows gfb_gather_desc.clear_mode; mode 3 = pure overwrite of the
 * region (forward sweep).
 */
typedef struct {
  int32_t rank;
  int32_t dtype;
  int32_t clear_mode; /* 0 acc, 1/3 overwrite, 2 folded clear */
  int32_t ntaps;
  void *dst;
  const void *src[GFB_MAX_SRCS];
  int64_t dims[3];    /* dims of D (all arrays share the same dims) */
  int64_t lo[3], hi[3];
  int64_t clear_lo[3], clear_hi[3];
  int32_t tap_src[GFB_MAX_TAPS];
  int32_t tap_masked[GFB_MAX_TAPS];
  int64_t tap_delta[GFB_MAX_TAPS][3];
  int64_t tap_mlo[GFB_MAX_TAPS][3];
  int64_t tap_mhi[GFB_MAX_TAPS][3];
  double tap_coef[GFB_MAX_TAPS];
} gfb_stencil_desc;

/*
 * Radius-1 star stencil sweep (positions 0 centre, 1/2 -/+ dim0, 3/4 -/+
 * dim1, 5/6 -/+ dim2; rank 2 arrays omit dim0): one linear map sweep
 *   D[y] = base(y) + sum_p [y in mask_p] coef_p * S[y + e_p]   for y in [lo, hi)
 * with base(y) as in gfb_stencil_desc (mode 0 acc, 1/3 zero, 2 folded clear).
 */
typedef struct {
  double coef[7];
  int32_t present; /* bit p: tap at position p */
  int32_t masked;  /* bit p: tap p carries a mask box */
  int32_t mode;
  int32_t _pad;
  int64_t mlo[7][3], mhi[7][3];
  int64_t lo[3], hi[3];
  int64_t clo[3], chi[3];
} gfb_star_op;

/*
 * Fused pair of star sweeps (one jacobi_2d / heat_3d timestep, forward or
 * adjoint): X = a(Y) then Z = b(X), in one pass. X is staged in shared
 * memory with a one-point halo; Z is written to `zout` (a ping-pong buffer
 * when Z aliases Y); X is written to `xout` only if `xwrite`, and never
 * inside the dead box (values the next writer overwrites unread).
 * Elements outside a's / b's region take the old X / Z values.
 */
/* gfb_star_pair_desc.flags: outside the op's region Z (X) is a copy of its
 * old value; when the host knows the target twin already holds equal values
 * there (ping-pong buffers after both were initialised), the copy is skipped */
#define GFB_STAR_SKIP_ZCOPY 1
#define GFB_STAR_SKIP_XCOPY 2

typedef struct {
  int32_t rank;   /* 2 or 3 */
  int32_t dtype;
  int32_t xwrite;
  int32_t flags;  /* GFB_STAR_SKIP_* */
  int64_t dims[3];
  gfb_star_op a, b;
  const void *y, *xold;
  void *xout;
  const void *zold;
  void *zout;
  int64_t dead_lo[3], dead_hi[3];
  /* slab decomposition along the outermost dimension (rank 3 only): the
   * arrays hold global planes [plane0, plane0 + dims[0]); Z (and X) are
   * produced for local planes [zlo, zhi). Single device: 0, 0, dims[0]. */
  int64_t plane0, zlo, zhi;
  int64_t global_d0;
  /* planes per CTA of the 3-D kernel (0: chosen from the launch's size) */
  int64_t tpm_hint;
} gfb_star_pair_desc;

/*
 * Affine product contraction (implicit GEMM; fast path of the gather pass
 * for wcr="sum" maps whose tasklet is a scaled product of two reads with
 * affine subsets, e.g. convolution forward / input / weight adjoints):
 *     D[m, n] = base(m, n) + scale * sum_k A[ta(m) + ta(k)] * B[tb(n) + tb(k)]
 * over the flattened output coordinates split into m (those A depends on)
 * and n (those only B depends on) and the flattened free parameters k.
 * A product is counted only when every constraint holds:
 *     lo[c] <= cm[c](m) + ck[c](k) < hi[c]   for c < ncm   (A side)
 *     lo[c] <= cn[c](n) + ck[c](k) < hi[c]   for ncm <= c < ncm + ncn
 * (pivot parameters of the reparameterised scatter staying in their box).
 * Index tables are int32 device arrays, one entry per m / n / k:
 *   mtab[m] = {A offset, D offset, inside clear box, cm[0..ncm)}
 *   ntab[n] = {B offset, D offset, inside clear box, cn[0..ncn)}
 *   ktab[k] = {A offset, B offset, ck[0..ncm+ncn)}
 * base follows gfb_gather_desc.clear_mode (a clear-box point needs both its
 * m and n bits). nsplit > 1 splits k; fp64 partials go to the workspace
 * (nsplit * M * N doubles) and a second pass adds them in a fixed order.
 */
typedef struct {
  int32_t dtype;
  int32_t clear_mode;
  int32_t ncm, ncn;
  int32_t a_kfast;   /* bit 0: A contiguous along k (else along m): load layout;
                        bit 1: 16-byte quads along that direction (fp32: offsets
                        consecutive and 4-aligned, constraints equal within a quad) */
  int32_t b_nfast;   /* bit 0: B contiguous along n (else along k); bit 1 as above */
  int32_t nsplit;
  int32_t mstride, nstride, kstride;  /* int32 words per table entry */
  int64_t M, N, K;
  double scale;
  const void *a, *b;
  void *d;
  const int32_t *mtab, *ntab, *ktab;
  int32_t lo[4], hi[4];
  void *workspace;
} gfb_contract_desc;

/*
 * Vectorised map (pointwise and single-dimension reductions). The host folds
 * the iteration box into `ndim` loop dimensions (innermost last, adjacent
 * dimensions merged when every operand's strides allow) with zero-based loop
 * coordinates k: element offset = c0 + sum_d s[d] * k_d. Each warp owns a row
 * (all but the innermost coordinate, decomposed once) and 32 * vec points of
 * the innermost one; the tasklet bytecode runs on a register stack of static
 * depth (code[pc] = op | depth_before << 6 | arg << 10), vec points per lane.
 *   mode 0: pointwise; out[o] (wcr 0 store, 1 add) per point
 *   mode 1: out[0] = base + sum over the innermost dimension (warp per row)
 *   mode 2: ndim == 2; out[0] = base + sum over dimension 0 (columns along
 *           dimension 1; nsplit row ranges, fp64 partials in the workspace)
 * base follows gfb_gather_desc.clear_mode with the clear box in loop
 * coordinates of the kept dimensions.
 */
#define GFB_M2_DIMS 8
#define GFB_M2_OUTS 4
#define GFB_M2_DEPTH 6
typedef struct {
  const void *base;
  int32_t dtype;
  int32_t _pad;
  int64_t c0;
  int64_t s[GFB_M2_DIMS];
} gfb_m2_operand;

typedef struct {
  int32_t mode;
  int32_t compute_f64;
  int32_t ndim;
  int32_t vec;
  int32_t n_in, n_out;
  int32_t clear_mode;
  int32_t nsplit;
  int64_t ext[GFB_M2_DIMS];
  gfb_m2_operand in[GFB_MAX_INPUTS];
  gfb_m2_operand out[GFB_M2_OUTS];
  int32_t wcr[GFB_M2_OUTS];
  int32_t code_start[GFB_M2_OUTS];
  int32_t code_len[GFB_M2_OUTS];
  uint32_t code[GFB_MAX_CODE];
  double consts[GFB_MAX_CONSTS];
  int64_t clear_lo[GFB_M2_DIMS], clear_hi[GFB_M2_DIMS];
  void *workspace;
  uint32_t *err;
} gfb_map2_desc;

/* ---- entry points --------------------------------------------------- */

int gfb_abi_version(void);
const char *gfb_last_error(void);
int gfb_device_sm_count(void);
/* sizes of gfb_space, gfb_operand, gfb_map_desc, gfb_term, gfb_gather_desc,
 * gfb_stencil_desc, gfb_star_op, gfb_star_pair_desc, gfb_contract_desc,
 * gfb_map2_desc, gfb_wave_desc (binding layout check); returns the count
 * written */
int gfb_struct_sizes(int64_t *out, int32_t cap);

/* replaces Executor._exec_map / _exec_tasklet (interpreter.py:478-507, 405-426) */
int gfb_map_launch(const gfb_map_desc *d, void *stream);

/*
 * Sequential loop nest of one tasklet (reference _exec_loop / run_level over
 * LoopRegions whose body is a single scalar tasklet, interpreter.py:221-330,
 * 396-426), executed by hyperplanes: the nest's iteration space is map.space
 * (one parameter per loop, box_lo = first iterate, step = the loop's step,
 * so box index k_p is the execution order of loop p); points with
 * sum_p c[p] * k_p == h form hyperplane h. The host proves (lowering.py,
 * ProgramRun._wavefront) that every pair of iterations touching one element
 * (at least one of them writing) lies on different hyperplanes in
 * execution order, so hyperplanes h = 0 .. hmax run in order with their
 * points in parallel (one cooperative launch, a grid barrier between
 * hyperplanes), and the result is the sequential nest's, element for
 * element. `solve` is a parameter with c != 0 (its index is solved from h).
 */
typedef struct {
  gfb_map_desc map;
  int64_t c[GFB_MAX_PARAMS];
  int64_t hmax;
  int32_t solve;
  int32_t _pad;
} gfb_wave_desc;

int gfb_wave_launch(const gfb_wave_desc *d, void *stream);
/* replaces the wcr="sum" scatter of _exec_tasklet (interpreter.py:422-423) */
int gfb_gather_launch(const gfb_gather_desc *d, void *stream);
int64_t gfb_gather_workspace_bytes(const gfb_gather_desc *d);
/* linear stencil fast path of _exec_map (interpreter.py:478-507) */
int gfb_stencil_launch(const gfb_stencil_desc *d, void *stream);
/* product-contraction fast path of the wcr="sum" scatter (interpreter.py:
 * 422-423, 478-507): implicit GEMM over index tables */
int gfb_contract_launch(const gfb_contract_desc *d, void *stream);
/* vectorised pointwise map / one-dimensional reduction (see gfb_map2_desc);
 * replaces _exec_map / _exec_tasklet (interpreter.py:478-507, 405-426) */
int gfb_map2_launch(const gfb_map2_desc *d, void *stream);
int64_t gfb_map2_workspace_bytes(const gfb_map2_desc *d);

/* fused forward / adjoint timestep of a radius-1 stencil program (two
 * consecutive _exec_map sweeps, interpreter.py:478-507) */
int gfb_star_pair_launch(const gfb_star_pair_desc *d, void *stream);

/* reduce_sum library node (interpreter.py:447-451): out (=|+=) sum(x[0:n]).
 * workspace >= gfb_reduce_workspace_bytes(n) bytes; deterministic order. */
int64_t gfb_reduce_workspace_bytes(int64_t n);
int gfb_reduce_sum(const void *x, int32_t xdtype, int64_t n, void *out,
                   int32_t odtype, int32_t accumulate, void *workspace,
                   void *stream);

/* ew_unary / ew_binary library nodes (interpreter.py:452-463, 553-597):
 *   out[i] (= | +=) op(a[i] [, b[i]]); `op` is a gfb_op code, `c` the scale
 *   constant; a scalar operand (n_a == 1) broadcasts. */
int gfb_elementwise(int32_t op, double c, const void *a, int64_t n_a,
                    const void *b, int64_t n_b, void *out, int64_t n,
                    int32_t dtype, int32_t accumulate, uint32_t *err,
                    void *stream);

/* fill / broadcast (reduce_sum adjoint map, autodiff.py:940-960; zero-init on
 * first touch, interpreter.py:171-189): out[i] (= | +=) scale * (*src or 1). */
int gfb_broadcast(const void *src, int32_t src_dtype, double scale, void *out,
                  int64_t n, int32_t dtype, int32_t accumulate, void *stream);

/* box fill: D[y] = value for y in [lo, hi) (rank <= 3); materialised
 * pending gradient clear (autodiff.py:735-740) */
int gfb_fill_box(void *dst, int32_t dtype, int32_t rank, const int64_t *dims,
                 const int64_t *lo, const int64_t *hi, double value,
                 void *stream);

/* matmul library node (interpreter.py:433-446; adjoint jobs autodiff.py:
 * 780-802): C (= | +=) op(A) @ op(B), row-major, op = transpose if t*.
 * fp64 runs on the DMMA tensor path, fp32 on the FFMA path. */
int64_t gfb_matmul_workspace_bytes(int32_t dtype, int32_t ta, int32_t tb, int64_t M,
                                   int64_t N, int64_t K);
int gfb_matmul(int32_t dtype, int32_t ta, int32_t tb, int64_t M, int64_t N,
               int64_t K, const void *A, int64_t lda, const void *B,
               int64_t ldb, void *C, int64_t ldc, int32_t accumulate,
               void *workspace, void *stream);

/* one-pass matrix-vector pair over a row-major A[R, C] (lda elements per
 * row): r (= | +=) A u and c (= | +=) A^T v in a single streaming read of A.
 * Replaces two N==1 matmul library nodes over the same matrix
 * (interpreter.py:433-446) -- atax forward t = A x, y = A^T t (chain = 1:
 * v is the new r), bicg forward s = A^T r, q = A p, and both adjoint pairs
 * (autodiff.py:780-802). Either half may be absent (u = r = NULL, or
 * c = NULL). Needs 16-byte aligned A / u, C and lda multiples of the 16-byte
 * vector width; gfb_matvec_pair_usable() says whether a shape qualifies.
 * Workspace: gfb_matvec_pair_workspace_bytes() (column partials). */
int64_t gfb_matvec_pair_workspace_bytes(int32_t dtype, int64_t R, int64_t C,
                                        int32_t has_col);
int gfb_matvec_pair_usable(int32_t dtype, int64_t R, int64_t C, int64_t lda,
                           const void *A, const void *u);
int gfb_matvec_pair(int32_t dtype, int64_t R, int64_t C, const void *A,
                    int64_t lda, const void *u, void *r, int32_t r_acc,
                    const void *v, void *c, int32_t c_acc, int32_t chain,
                    void *workspace, void *stream);

/* fused outer-product adjoints into one matrix gradient (autodiff.py:
 * 780-802, two K==1 matmul jobs with the same target):
 * C[i,j] (= | +=) u1[i] v1[j] + u2[i] v2[j]; u2 = v2 = NULL for rank 1.
 * Unit-stride vectors; v*, C 16-byte aligned, N and ldc multiples of the
 * 16-byte vector width. */
int gfb_rank2(int32_t dtype, int64_t M, int64_t N, const void *u1,
              const void *v1, const void *u2, const void *v2, void *C,
              int64_t ldc, int32_t accumulate, void *stream);

/* device-to-device copy of n elements (tape snapshots, interpreter.py:371-386) */
int gfb_copy(void *dst, const void *src, int64_t bytes, void *stream);

/* halo planes for slab decomposition (multi-GPU stencils): pack/unpack
 * `nplanes` contiguous outer-dimension planes starting at plane `p0`. */
int gfb_plane_copy(void *dst, const void *src, int64_t plane_elems,
                   int32_t dtype, int64_t nplanes, void *stream);

/* K15: the halo exchange of a slab-decomposed stencil timestep over NCCL
 * (the engine's Python path posts the same exchange through
 * torch.distributed, decomp.HaloOp). Each array is a contiguous local slab
 * whose outermost dimension holds [own_lo - width, own_hi + width) halo and
 * owned planes; the owned planes next to each neighbour are sent and the
 * neighbour's are received into the halo:
 *   lower: send [own_lo, own_lo + w)  recv [own_lo - w, own_lo)
 *   upper: send [own_hi - w, own_hi)  recv [own_hi, own_hi + w)
 * all in one NCCL group on `stream`. `nccl_comm` is the caller's ncclComm_t;
 * NCCL is resolved at run time (the libnccl.so.2 already in the process, or
 * the system one), so the library has no link-time NCCL dependency. */
#define GFB_MAX_HALO 4
typedef struct {
  void *base;           /* local slab, contiguous, halo planes included */
  int64_t plane_bytes;  /* bytes of one outermost-dimension plane */
  int64_t planes;       /* local planes (halo included) */
  int64_t own_lo, own_hi;
  int64_t width;        /* halo planes per side */
} gfb_halo_array;

typedef struct {
  int32_t n;            /* arrays exchanged in one group (<= GFB_MAX_HALO) */
  int32_t lower, upper; /* neighbour ranks in the communicator; -1: none */
  int32_t _pad;
  gfb_halo_array a[GFB_MAX_HALO];
} gfb_halo_desc;

int gfb_halo_exchange(const gfb_halo_desc *d, void *nccl_comm, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* GFB_H */
