/* dash_b200.h — C ABI of the B200-native DASH optimizer step (arXiv 2602.02016).
 *
 * Every entry point is stream-ordered on the caller's CUDA stream (`stream` is a cudaStream_t passed
 * as void*), takes device pointers and plain sizes, and never allocates: scratch comes from a
 * caller-owned workspace whose size is given by the matching *_ws_bytes query.  Return codes:
 *     DASH_OK = 0, DASH_EINVAL = 1 (bad argument), DASH_ENONFINITE = 2, DASH_ECUDA = 3.
 * Python binding: paper_2602_02016_b200/_lib.py (ctypes); see INTEGRATION.md.
 *
 * Each function names the reference interface it replaces (paths relative to
 * /root/reference/pkg/src/blockshampoo/).
 */
#ifndef DASH_B200_H_
#define DASH_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DASH_OK 0
#define DASH_EINVAL 1
#define DASH_ENONFINITE 2
#define DASH_ECUDA 3

/* A stack of `nmat` rows x cols matrices in split-f16 form:
 *   value = (hi + lo) * 2^exp[m], hi/lo fp16 planes of rows x ld, ld % 64 == 0, padding zero.
 * Layout of `data`: [nmat][2][rows][ld] (plane 0 = hi, plane 1 = lo). */
typedef struct dash_stack {
  uint16_t* data;
  int nmat, rows, cols, ld;
  int* exp;           /* [nmat] power-of-two exponents */
  uint32_t* amax;     /* [nmat] float bit patterns of max |value| (NaN bits = non-finite seen) */
} dash_stack;

/* One gradient block of a 2-D layer (or one chunk of a 1-D layer, as a rows x 1 matrix) in the flat
 * parameter space, with the preconditioner slots it feeds (shampoo.py:176-230: SlotRef(group, slot)). */
typedef struct dash_block {
  long long off;            /* flat offset of element (r0, c0) */
  int ld;                   /* row stride of the layer (1-D chunks: 1) */
  int rows, cols;           /* block shape (1-D chunk: len x 1) */
  int group_l, slot_l;      /* left preconditioner */
  int group_r, slot_r;      /* right preconditioner (-1 for 1-D chunks) */
} dash_block;

/* Opaque per-structure plan: owns the grouped-GEMM job tables of one optimizer structure. */
typedef struct dash_plan dash_plan;

/* Library / build identification. */
const char* dash_version(void);
int dash_device_sms(void);
/* Instrumentation: number of kernels this library has launched (process lifetime), and optional
 * CUDA-event timing of every tcgen05 GEMM launch on its own stream (algorithmic flops = 2 M N K per job). */
unsigned long long dash_launch_count(void);
void dash_gemm_timing(int enable);
int dash_gemm_timing_read(int* launches, double* ms, double* flops);
/* Per-launch detail of the timed GEMM launches: up to `cap` entries of (ms, algorithmic flops = 2 M N K per
 * job, issued tensor-core flops = tiles x 2 x 256 x 128 x padded K x passes, tiles); returns the number
 * written (or -status on error). */
int dash_gemm_timing_list(int cap, double* ms, double* flops, double* issued, int* tiles);

/* ---------------------------------------------------------------- dense primitives (linalg.py)
 * dash_split: fp32 stack (src[m*src_mat_stride + r*src_ld + c]) -> split-f16 stack.
 *   Replaces the storage side of linalg.quantize (linalg.py:75-79) for the tensor-core modes. */
int dash_split(const float* src, long long src_mat_stride, int src_ld, const dash_stack* dst, void* stream);
/* dash_unsplit: split-f16 stack -> fp32 (dst[m*dst_mat_stride + r*dst_ld + c]). */
int dash_unsplit(const dash_stack* src, float* dst, long long dst_mat_stride, int dst_ld, void* stream);

/* dash_bmm: C[m] = alpha * op(A[m]) @ op(B[m]) for every m (linalg.bmm, linalg.py:105-114).
 *   trans_a/trans_b: 1 = use the transpose of the stored matrix.  passes: 3 = split-f16 products
 *   (fp32-class), 1 = fp16 hi*hi only.  C may be null if f_out (fp32, [m*f_mat_stride + r*f_ld + c])
 *   is given, and vice versa. */
size_t dash_bmm_ws_bytes(int nmat);
int dash_bmm(const dash_stack* a, int trans_a, const dash_stack* b, int trans_b, const dash_stack* c,
             float* f_out, long long f_mat_stride, int f_ld, float alpha, int passes, void* ws,
             size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- inverse-root solvers (roots.py)
 * Inputs are split stacks of square blocks a (N x B x B); the solvers run on a_hat = a * inv_scale[m]
 * (inv_scale may be NULL = 1), i.e. the reference's a / scales (shampoo.py:326).  Per-block reports are
 * written to device arrays iters[N], resid[N] (float), conv[N] (0/1) exactly as IterationReport
 * (roots.py:32-36).  tol = 0 is fixed-iteration mode.  passes: 3 = split-f16 (fp32-class), 4 = split-f16
 * accumulated in 16 K ranges per tile, each drained from TMEM into fp32 registers (FULL64: B = 1024 Newton-DB
 * error ~14x smaller, ~20% slower), 1 = fp16.
 * stall > 0 (used when the requested tolerance is below the rounding floor of the arithmetic): a block whose
 * residual stops decreasing (r_k >= r_{k-1}) once r_{k-1} <= stall is frozen as converged at that floor;
 * stall = 0 keeps the reference's rules exactly (non-finite, r <= tol, divergence watch).
 *
 * dash_ndb: batched Newton-Denman-Beavers (roots.batched_newton_db, roots.py:262-305):
 *   y <- a_hat^(1/2), z <- a_hat^(-1/2). */
size_t dash_ndb_ws_bytes(int n, int b);
int dash_ndb(const dash_stack* a, const float* inv_scale, const dash_stack* y, const dash_stack* z, float tol,
             float stall, int max_iters, int passes, int* iters, float* resid, int* conv, void* ws, size_t ws_bytes,
             void* stream);
/* dash_cn: batched coupled Newton (roots.batched_coupled_newton, roots.py:216-259): x <- a_hat^(-1/p),
 *   p in {2, 4}, c = CnConfig.resolved_c (roots.py:53-56). */
/* dash_ndb_upper: dash_ndb leaving y and z in upper pair-block storage (only the 256x256 blocks on or above
 *   the block diagonal are valid, diagonal blocks complete) -- the optimizer completes only the
 *   output it reads; the input a may itself be upper-stored (dash_ndb accepts that too).  dash_fill_lower
 *   completes such a stack in place (lower blocks <- transposed upper);
 *   both are plain dash_ndb / a no-op when the iterates are stored complete (DASH_NDB_UP=0, DASH_KB=32).
 *   outputs: the outputs the caller reads (1 = y, 2 = z, 3 = both); the last iteration computes only those
 *   (the other stack then holds an earlier iterate). */
int dash_ndb_upper(const dash_stack* a, const float* inv_scale, const dash_stack* y, const dash_stack* z, float tol,
                   float stall, int max_iters, int passes, int outputs, int* iters, float* resid, int* conv, void* ws,
                   size_t ws_bytes, void* stream);
int dash_fill_lower(const dash_stack* s, void* stream);
size_t dash_cn_ws_bytes(int n, int b);
int dash_cn(const dash_stack* a, const float* inv_scale, int p, float c, const dash_stack* x, float tol,
            float stall, int max_iters, int passes, int* iters, float* resid, int* conv, void* ws, size_t ws_bytes,
            void* stream);
/* dash_scale_stack: v = value * mult[m]^pw -> fp32 f_out and/or split dst (the root rescale
 *   roots * scales^(-1/p), shampoo.py:348, with mult = 1/scale and pw = 1/p).  gate (device int, may be
 *   NULL): nothing is written unless *gate != 0 (a group that failed its scale checks keeps its roots).
 *   src_upper: src is in upper pair-block storage (dash_ndb_upper output); the lower blocks are read
 *   transposed, so the outputs are complete without a dash_fill_lower pass. */
int dash_scale_stack(const dash_stack* src, const float* mult, float pw, float* f_out, long long f_mat_stride,
                     int f_ld, const dash_stack* dst, const int* gate, int src_upper, void* stream);
/* dash_scale_check: the refresh's scale checks for one group, on the device (shampoo.py:324-325,
 *   spectral.py:99-107): status[m] == 2 (pool collapsed twice) -> code 2 (DegenerateSpectrumError), a
 *   non-positive / non-finite scale[m] -> code 1 (ConvergenceError).  err[2] is shared by the groups of one
 *   refresh (zeroed by the caller): the first failing group stores (code, group); *ok = 1 iff no group failed
 *   so far (the commit gate of dash_scale_stack / dash_clenshaw).  status may be NULL (Frobenius). */
int dash_scale_check(const float* scale, const int* status, int n, int group, int* ok, int* err, void* stream);
/* dash_clenshaw: optimized matrix Clenshaw of a Chebyshev series (chebyshev.batched_clenshaw_matrix,
 *   chebyshev.py:137-184) on S = 2 a inv_scale - I with coefficients coeffs[0..degree] (fit on the host,
 *   chebyshev.py:46-84), result * mult[m] -> fp32 f_out ([m][B][B]) and/or split out.  d-1 products.
 *   gate (may be NULL): the final product writes the outputs only when *gate != 0. */
size_t dash_cheb_ws_bytes(int n, int b);
int dash_clenshaw(const dash_stack* a, const float* inv_scale, const float* mult, const double* coeffs, int degree,
                  float* f_out, const dash_stack* out, int passes, const int* gate, void* ws, size_t ws_bytes,
                  void* stream);

/* ---------------------------------------------------------------- optimizer step (shampoo.py)
 * dash_plan_create: register the block table (matrix blocks first, then 1-D chunks), the groups'
 * fp32 EMA stacks gema[g] ([gsize][gdim][gdim]) and split root stacks groot[g], and the flat buffers
 * (grad/adam/mom over the flat parameter space; gsm/gsv split gradient stacks; tm split temp; um/uv fp32
 * update stacks; pn_part/un_part/gamax/graft_s per-block scratch).  Builds and uploads the statistics and
 * apply GEMM job tables into ws (size dash_plan_ws_bytes).  Returns NULL on error (status set). */
size_t dash_plan_ws_bytes(int nb_m, int nb_v);
dash_plan* dash_plan_create(const dash_block* blocks, int nb_m, int nb_v, int block_size, int ngroups,
                            const int* gdim, const int* gsize, float* const* gema, const dash_stack* groot,
                            float* grad, float* adam, float* mom, const dash_stack* gsm, const dash_stack* gsv,
                            const dash_stack* tm, float* um, float* uv, float* pn_part, float* un_part,
                            uint32_t* gamax, float* graft_s, float beta_lr, int passes, void* ws, size_t ws_bytes,
                            void* stream, int* status);
void dash_plan_destroy(dash_plan* p);
/* Owner-only optimizer state (block sharding; PAPER.md:114 keeps each block's Adam / momentum on its owner):
 * d_offsets (device, nb_m + nb_v entries, multiples of 4, caller-owned, must outlive the plan's use) gives each
 * block's base in a packed adam / mom buffer holding the blocks back to back (row-major inside a block).
 * NULL (the default) indexes adam / mom like the flat parameter space. */
int dash_plan_set_state_offsets(dash_plan* p, const long long* d_offsets);
int dash_plan_un_stride(const dash_plan* p);
int dash_prep_parts(void);
/* Length of each block's slice of the apply-norm partial buffer (`un_part`) for a given block size. */
int dash_apply_partials(int block_size);
/* accumulate (shampoo.py:238-278): Adam / momentum EMA, block split of the gradient, L/R statistics EMA
 * as grouped tcgen05 GEMMs, and the per-block graft-direction norms |P_b|^2 for n_acc = t + 1. */
int dash_plan_accumulate(dash_plan* p, float beta2, float beta1, int n_acc, float graft_eps, void* stream);
/* apply + graft (shampoo.py:380-403): U = rootL G rootR (1-D: rootL g), s_b = |P_b| / |U_b|,
 * theta_out = theta_in - eta s_b U_b. */
int dash_plan_apply(dash_plan* p, const float* theta_in, float* theta_out, float eta, void* stream);
/* Per-group refresh helpers (shampoo.py:312-349): symmetrize the EMA (linalg.symmetrize) and collect
 * max|a| / sum(a^2) partials of a = ema + eps I; split a; Frobenius scale; pooled power iteration
 * (spectral.py:87-117, block seeds block_seed(seed, i), NumPy-identical start vectors).
 * status[i]: 0 ok, 1 non-positive scale, 2 pool collapsed twice.  seed_index (device, nullable): global
 * block index used for block i's child seed (block sharding keeps the 1-GPU pools).  vec_out (device,
 * nullable, [n][d]): the selected normalized pool vector (spectral.py:108-112); a zero matrix gives
 * lambda = 0 and its first start vector (spectral.py:99-101). */
int dash_group_sym(float* ema, int n, int d, float eps, uint32_t* amax, float* fro_part, void* stream);
int dash_group_split_a(const float* ema, float eps, const dash_stack* a, void* stream);
int dash_fro_scale(const float* fro_part, int n, float* scale, float* inv_scale, void* stream);
int dash_power_iteration(const float* ema, int n, int d, float eps, int pool, int iters, unsigned long long seed,
                         float* scale, float* inv_scale, int* status, const int* seed_index, float* vec_out,
                         void* stream);
/* Same result from the solver's split stack a = ema + eps I (d a multiple of 128, <= 1024): tensor-core
 * matvecs (tcgen05, one d/128-CTA cluster per two blocks, pool in shared memory; passes 1..iters multiply the
 * fp16 plane of a, the Rayleigh-quotient pass the full split a).  Blocks whose pool collapses are re-run by
 * dash_power_iteration's kernel on ema (zero matrix -> lambda 0, reseeded retry); ema may be NULL, leaving
 * status 3 for them.  Replaces the inner loop of spectral.multi_power_iteration (spectral.py:77-112). */
int dash_power_iteration_split(const dash_stack* a, const float* ema, float eps, int pool, int iters,
                               unsigned long long seed, float* scale, float* inv_scale, int* status,
                               const int* seed_index, void* stream);
/* dash_jacobi_eigh: batched cyclic Jacobi eigendecomposition in float64 (eigensolver.eigh / _jacobi,
 *   eigensolver.py:53-124): the reference's round-robin schedule of disjoint pairs, dead-pair skip
 *   0.1 tol |A|_F / d, convergence when the off-diagonal norm <= tol |A|_F, at most max_sweeps sweeps.
 *   a: n x d x d float64 symmetric blocks (d <= 1024); lam: n x d eigenvalues ascending; q: n x d x d
 *   eigenvectors in columns; sweeps / status (nullable): sweeps run, 0 converged / 1 not converged.
 *   ws: dash_jacobi_ws_bytes(n, d) bytes (working copies of A and V). */
size_t dash_jacobi_ws_bytes(int n, int d);
int dash_jacobi_eigh(const double* a, int n, int d, double tol, int max_sweeps, double* lam, double* q, int* sweeps,
                     int* status, void* ws, size_t ws_bytes, void* stream);
/* Block sharding exchange: copy blocks[b] (device table) of the flat space to/from the block-major
 * packed buffer at offsets pos[b] (device), around the all-gather of updated parameter shards. */
int dash_pack_blocks(const dash_block* blocks, int n, const long long* pos, const float* flat, float* packed,
                     void* stream);
int dash_unpack_blocks(const dash_block* blocks, int n, const long long* pos, const float* packed, float* flat,
                       void* stream);
/* spectral.block_seed (spectral.py:53-55), host side. */
unsigned long long dash_block_seed(unsigned long long seed, unsigned long long index);
/* First `count` draws of default_rng(seed).uniform(-1, 1), computed on the device (double). */
int dash_uniform_pm1(unsigned long long seed, int count, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DASH_B200_H_ */
