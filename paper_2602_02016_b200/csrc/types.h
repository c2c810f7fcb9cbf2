// Shared host/device data structures of the DASH B200 engine.
//
// Matrix storage ("split-f16 stack"): a stack of `nmat` matrices of `rows x cols`, each stored as two
// fp16 planes (hi, lo) of `rows x ld` (ld = cols rounded up to 64, zero padded) plus a per-matrix
// power-of-two exponent e and a running max-abs `amax`:
//     value[m][r][c] = (hi[m][r][c] + lo[m][r][c]) * 2^e[m]
// hi = RN16(x * 2^-e), lo = RN16(x * 2^-e - hi).  e is chosen so |x| * 2^-e < 2^15, which keeps both
// planes in the fp16 normal range for every entry within 2^-18 of the matrix max (22-bit significand,
// i.e. fp32-class accuracy) -- see DESIGN.md "split-f16 format".
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#include <cuda_fp16.h>
#define DASH_HD __host__ __device__
#else
#define DASH_HD
struct __half { unsigned short x; };
#endif

namespace dash {

constexpr int kTileM = 256;   // output tile rows (CTA pair, tcgen05 cta_group::2, 128 rows per CTA)
constexpr int kTileN = 128;   // output tile columns (64 B rows staged per CTA)
constexpr int kPartialsPerTile = 16;  // EPI_APPLY: 2 CTAs x 4 TMEM lane quarters x 2 column halves
constexpr int kTileK = 64;    // fp16 elements per 128-byte swizzle row
constexpr int kLdAlign = 64;  // leading-dimension padding of split stacks (elements)
constexpr int kEExp = -13;    // fixed exponent of identity-like Newton factors E (|E| < 8)

enum EpiOp : int {
  EPI_SPLIT = 0,       // C = alpha * alpha_p[mat] * acc                 -> split (+ optional fp32)
  EPI_NDB_E = 1,       // E = 1.5 I - 0.5 acc (E = I when inactive)     -> split, residual max|E-I|
  EPI_EMA = 2,         // F = beta * F_in + (1 - beta) * acc            -> fp32 only
  EPI_CHEB = 3,        // B = 2 acc - S + c I                           -> split
  EPI_CHEB_FINAL = 4,  // R = (acc - S + c I) * alpha_p[mat]            -> fp32 + split
  EPI_APPLY = 5,       // U = acc                                       -> fp32, per-tile sum(U^2)
  EPI_CN_M = 6,        // M = acc -> split, residual max|M-I|, and corr C = (1+1/p) I - M/p -> split #2
};

// One output matrix of a grouped GEMM: C[M x N] = op(A)[M x K] * op(B)[K x N], then epilogue.
// Operand majorness (tcgen05 terms): A K-major = stored row-major M x K; A MN-major = stored K x M.
//                                    B K-major = stored N x K;           B MN-major = stored K x N.
struct GemmJob {
  // ---- operands (TMA maps index into the map table; mat = coordinate along the stack)
  int a_map, b_map;
  int a_map32, b_map32;  // the same operands with 32-wide K boxes (K-block 32 kernel variant)
  int a_mat, b_mat;
  int a_mn, b_mn;
  int M, N, K;
  int tiles_n;  // ceil(N / kTileN)
  int tile_start;  // first global tile index of this job
  int tiles_n2, tile_start2;  // the same for 256-wide pair tiles (launches of symmetric jobs only)
  int op;
  int out_mat;     // index into per-matrix epilogue arrays (resid, active, alpha_p)
  int c_ld;        // split output leading dim
  int f_ld;        // fp32 output / input leading dim
  int s_ld;        // side split input leading dim
  int sym;         // 1: C is symmetric (M == N): only tiles on/above the diagonal run, the epilogue mirrors
  // Upper pair-block storage of symmetric matrices (K-block 64 launches): a stack flagged `up` holds only the
  // 256x256 pair blocks on or above the block diagonal (diagonal pair blocks complete).  a_up / b_up: read a
  // lower k-block of the operand as the transposed upper one (a_mapT = the A map of the other majorness;
  // B uses the same 64x64 map with swapped coordinates).  c_up: the epilogue mirrors only inside diagonal
  // pair blocks.
  int a_up, b_up, c_up, a_mapT;
  const int* a_exp;  const unsigned* a_amax;   // exponent / amax of the A matrix
  const int* b_exp;  const unsigned* b_amax;
  // ---- TMA store maps of the split outputs (-1: direct stores): c_map / c2_map box 64 x 32 x 2 planes
  //      (128-byte swizzle), c_tmap / c2_tmap box 32 x 64 x 2 planes (transposed mirror of symmetric jobs)
  int c_map, c_tmap, c2_map, c2_tmap;
  int c_rows, c_cols;  // dims of the output stack (TMA stores only when the job covers it exactly)
  int c_mat, c2_mat;   // matrix index of the outputs within their stacks (TMA coordinate)
  int s_map, s_mat;    // TMA load map (box 64 x 32 x 2 planes, 128-byte swizzle) + matrix of the side input, or -1
  int f_map, f_tmap, f_mat;  // fp32 output (and EPI_EMA input) maps: box 32 x 32 (128-byte swizzle) and 32 x 64
  int f_rows, f_cols;        // (transposed mirror), or -1; f_rows x f_cols = dims of the fp32 matrices
  // ---- split output (hi plane; lo plane at +c_plane elements)
  __half* c_hi; long long c_plane; int* c_exp; unsigned* c_amax;
  // ---- second split output (EPI_CN_M correction factor)
  __half* c2_hi; long long c2_plane; int* c2_exp; unsigned* c2_amax;
  // ---- fp32 output / input
  float* f_out; const float* f_in;
  // ---- side split input (EPI_CHEB*: B_{k+2})
  const __half* s_hi; long long s_plane; const int* s_exp; const unsigned* s_amax;
  // ---- scalars
  float alpha; float beta; float gamma; float pad1;
  const float* alpha_p;   // per-matrix multiplier (indexed by out_mat) or null
  const float* gamma_p;   // launch-wide scalar overriding gamma (EPI_CHEB: c_k) or null
  unsigned* resid;        // per-matrix residual accumulator (indexed by out_mat) or null
  const int* active;      // per-matrix active flag (indexed by out_mat) or null
  float* partial;         // EPI_APPLY: per-(tile, quarter) partial sums, indexed by local tile
};

}  // namespace dash
