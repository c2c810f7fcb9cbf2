// Optimizer-step kernels: gradient prep (Adam / momentum EMA + graft-direction norms + block max),
// gradient blocking into split stacks, preconditioner symmetrization, pooled power iteration,
// and the grafted parameter update.  Plus the `dash_plan` that owns the per-structure GEMM job
// tables (statistics EMA and the L^(-1/4) G R^(-1/4) apply) so a step launches a fixed set of kernels.
//
// Reference: shampoo.py:238-278 (accumulate), :294-298 (_group_scales), :352-404 (graft_scale, step),
// spectral.py:53-117 (block_seed, start vectors, pooled power iteration).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "engine.h"
#include "elem.cuh"
#include "ptx.cuh"
#include "rng.cuh"

namespace cg = cooperative_groups;

namespace dash {

constexpr int kPrepParts = 16;  // CTAs per block in the elementwise passes (fixed -> deterministic sums)

__device__ __forceinline__ int exp_for_amax(float amax) {
  if (!(amax > 0.f) || !(amax < 3.0e38f)) return 0;
  int x;
  frexpf(amax, &x);
  return x - 15;
}

template <int NT>
__device__ double block_sum_d(double v, double* sh) {
  v = warp_sum_d(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < NT / 32; ++i) t += sh[i];  // fixed order
  __syncthreads();
  return t;
}

// ---------------------------------------------------------------------------- gradient prep
// adam <- b2 adam + (1-b2) g^2 ; mom <- b1 mom + (1-b1) g ; P = num / (eps + sqrt(adam * bc2_inv))
// with num = g (b1 == 0) or mom * bc1_inv; per-block partial sum(P^2) and max|g|.
__global__ void __launch_bounds__(256) prep_kernel(const dash_block* __restrict__ blocks, const float* __restrict__ g,
                                                   float* __restrict__ adam, float* __restrict__ mom, float beta2,
                                                   float beta1, float bc1_inv, float bc2_inv, float geps,
                                                   float* __restrict__ pn_part, unsigned* __restrict__ gamax,
                                                   const long long* __restrict__ sofs) {
  __shared__ double sh[8];
  const int b = blockIdx.y, p = blockIdx.x;
  const dash_block blk = blocks[b];
  // optimizer state index of block element e: the flat parameter index (sofs == NULL) or, for an owner-only
  // state (block sharding), the block's packed base + e (block-major, row-major inside the block)
  const long long sb = sofs ? sofs[b] : -1;
  const long long total = static_cast<long long>(blk.rows) * blk.cols;
  const long long per = (total + kPrepParts - 1) / kPrepParts;
  const long long e0 = p * per, e1 = min(total, e0 + per);
  double pn = 0.0;
  float mx = 0.f;
  auto one = [&](long long i, long long si) {
    const float gv = g[i];
    const float a = beta2 * adam[si] + (1.f - beta2) * gv * gv;
    adam[si] = a;
    float num = gv;
    if (mom) {
      const float m = beta1 * mom[si] + (1.f - beta1) * gv;
      mom[si] = m;
      num = m * bc1_inv;
    }
    const float pv = num / (geps + sqrtf(a * bc2_inv));
    pn += static_cast<double>(pv) * pv;
    float av = fabsf(gv);
    if (!(av <= 3.0e38f)) av = __uint_as_float(0x7fc00000u);
    mx = nonneg_max(mx, av);
  };
  // rows of 4-aligned 4-multiple width (every 2-D block and 1-D chunk of the DASH shapes): 16-byte accesses
  const bool contiguous = blk.ld == blk.cols || blk.rows == 1;
  const long long w = contiguous ? total : blk.cols;  // elements per contiguous run
  if (w % 4 == 0 && blk.off % 4 == 0 && blk.ld % 4 == 0 && (e0 % 4 == 0) && (per % 4 == 0) && (sb < 0 || sb % 4 == 0)) {
    for (long long e = e0 + 4 * threadIdx.x; e < e1; e += 4 * blockDim.x) {
      const long long r = contiguous ? 0 : e / blk.cols, c = contiguous ? e : e % blk.cols;
      const long long i = blk.off + r * blk.ld + c;
      const long long si = sb < 0 ? i : sb + e;
      const float4 g4 = *reinterpret_cast<const float4*>(g + i);
      float4 a4 = *reinterpret_cast<const float4*>(adam + si);
      const float gv[4] = {g4.x, g4.y, g4.z, g4.w};
      float av4[4] = {a4.x, a4.y, a4.z, a4.w};
      float num[4] = {gv[0], gv[1], gv[2], gv[3]};
      if (mom) {
        float4 m4 = *reinterpret_cast<const float4*>(mom + si);
        float mv[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          mv[k] = beta1 * mv[k] + (1.f - beta1) * gv[k];
          num[k] = mv[k] * bc1_inv;
        }
        *reinterpret_cast<float4*>(mom + si) = make_float4(mv[0], mv[1], mv[2], mv[3]);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        av4[k] = beta2 * av4[k] + (1.f - beta2) * gv[k] * gv[k];
        const float pv = num[k] / (geps + sqrtf(av4[k] * bc2_inv));
        pn += static_cast<double>(pv) * pv;
        float aa = fabsf(gv[k]);
        if (!(aa <= 3.0e38f)) aa = __uint_as_float(0x7fc00000u);
        mx = nonneg_max(mx, aa);
      }
      *reinterpret_cast<float4*>(adam + si) = make_float4(av4[0], av4[1], av4[2], av4[3]);
    }
  } else {
    for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const int r = static_cast<int>(e / blk.cols), c = static_cast<int>(e % blk.cols);
      const long long i = blk.off + static_cast<long long>(r) * blk.ld + c;
      one(i, sb < 0 ? i : sb + e);
    }
  }
  const double t = block_sum_d<256>(pn, sh);
  if (threadIdx.x == 0) pn_part[b * kPrepParts + p] = static_cast<float>(t);
  mx = warp_max_nonneg(mx);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(gamax + b, mx);
}

// Copy block b of the flat gradient into slot b of a split stack (zero padded), exponent from max|g|.
__global__ void __launch_bounds__(256) grad_split_kernel(const dash_block* __restrict__ blocks,
                                                         const float* __restrict__ g, dash_stack st,
                                                         const unsigned* __restrict__ gamax) {
  const int b = blockIdx.y;
  const dash_block blk = blocks[b];
  const float amax = __uint_as_float(gamax[b]);
  const int e = exp_for_amax(amax);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st.exp[b] = e;
    st.amax[b] = gamax[b];
  }
  const float inv = ldexpf(1.f, -e);
  __half* hi = mat_hi(st, b);
  const bool vec = blk.cols % 8 == 0 && blk.ld % 4 == 0 && blk.off % 4 == 0;
  for_chunks8(st.rows, st.ld, [&](int r, int c) {
    float v[8];
    const float* src = g + blk.off + static_cast<long long>(r) * blk.ld + c;
    if (r < blk.rows && vec && c + 8 <= blk.cols) {
      const float4 x0 = __ldg(reinterpret_cast<const float4*>(src));
      const float4 x1 = __ldg(reinterpret_cast<const float4*>(src) + 1);
      v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w; v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = (r < blk.rows && c + k < blk.cols) ? src[k] : 0.f;
    }
    store_split8(hi, mat_plane(st), static_cast<long long>(r) * st.ld + c, v, inv);
  });
}

// ---------------------------------------------------------------------------- preconditioner stats
// In-place symmetrization ema <- (ema + ema^T) / 2 of an (n, d, d) stack (linalg.symmetrize), plus
// per-block max|a| and sum(a^2) partials of a = ema + eps I (inputs of the solver split / Frobenius scale).
// CTA p of a block walks the upper-triangle 32 x 32 tile pairs p, p + kPrepParts, ...: both tiles are read
// coalesced into shared memory, averaged, and written back coalesced (the mirror through the transpose
// buffer); the partial sums are per CTA and combined in a fixed order (deterministic).
__global__ void __launch_bounds__(256) sym_kernel(float* __restrict__ ema, int d, float eps,
                                                  unsigned* __restrict__ amax, float* __restrict__ fro_part) {
  __shared__ float t1[32][33], t2[32][33];
  __shared__ double sh[8];
  const int m = blockIdx.y, p = blockIdx.x;
  float* a = ema + static_cast<long long>(m) * d * d;
  const int nt = (d + 31) / 32, npairs = nt * (nt + 1) / 2;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double fro = 0.0;
  float mx = 0.f;
  for (int tp = p; tp < npairs; tp += kPrepParts) {
    int ti = 0, rem = tp;
    while (rem >= nt - ti) { rem -= nt - ti; ++ti; }
    const int tj = ti + rem;
    const int r0 = ti * 32, c0 = tj * 32;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int y = ty + 8 * k;
      t1[y][tx] = (r0 + y < d && c0 + tx < d) ? a[static_cast<long long>(r0 + y) * d + c0 + tx] : 0.f;
      t2[y][tx] = (c0 + y < d && r0 + tx < d) ? a[static_cast<long long>(c0 + y) * d + r0 + tx] : 0.f;
    }
    __syncthreads();
    const bool diag = ti == tj;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int y = ty + 8 * k;
      const int r = r0 + y, c = c0 + tx;
      const float v = (t1[y][tx] + t2[tx][y]) * 0.5f;  // X[r][c] and X[c][r]
      if (r < d && c < d) {
        a[static_cast<long long>(r) * d + c] = v;
        const float av = (r == c) ? v + eps : v;
        fro += (diag ? 1.0 : 2.0) * static_cast<double>(av) * av;
        mx = nonneg_max(mx, fabsf(av));
      }
    }
    __syncthreads();
    if (!diag) {  // mirror: row c0 + y of the lower tile = column of the averaged upper tile
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int y = ty + 8 * k;
        const int r = c0 + y, c = r0 + tx;
        if (r < d && c < d) a[static_cast<long long>(r) * d + c] = (t1[tx][y] + t2[y][tx]) * 0.5f;
      }
    }
    __syncthreads();
  }
  const double t = block_sum_d<256>(fro, sh);
  if (threadIdx.x == 0) fro_part[m * kPrepParts + p] = static_cast<float>(t);
  mx = warp_max_nonneg(mx);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(amax + m, mx);
}

// a = ema + eps I -> split stack (exponent from the exact max computed by sym_kernel).
__global__ void __launch_bounds__(256) a_split_kernel(const float* __restrict__ ema, float eps, dash_stack st) {
  const int m = blockIdx.y;
  const int d = st.rows;
  const int e = exp_for_amax(__uint_as_float(st.amax[m]));
  if (blockIdx.x == 0 && threadIdx.x == 0) st.exp[m] = e;
  const float inv = ldexpf(1.f, -e);
  const float* a = ema + static_cast<long long>(m) * d * d;
  __half* hi = mat_hi(st, m);
  const bool vec = (d & 7) == 0;
  for_chunks8(d, st.ld, [&](int r, int c) {
    float v[8];
    const float* src = a + static_cast<long long>(r) * d + c;
    if (vec && c + 8 <= d) {
      const float4 x0 = __ldg(reinterpret_cast<const float4*>(src));
      const float4 x1 = __ldg(reinterpret_cast<const float4*>(src) + 1);
      v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w; v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = c + i < d ? __ldg(src + i) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (r == c + i) v[i] += eps;
    store_split8(hi, mat_plane(st), static_cast<long long>(r) * st.ld + c, v, inv);
  });
}

// Frobenius scale (shampoo.py:296): s = sqrt(sum a^2), fixed-order reduction of the partials.
__global__ void fro_scale_kernel(const float* __restrict__ fro_part, int n, float* __restrict__ scale,
                                 float* __restrict__ inv_scale) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  double t = 0.0;
  for (int p = 0; p < kPrepParts; ++p) t += fro_part[m * kPrepParts + p];
  const float s = static_cast<float>(sqrt(t));
  scale[m] = s;
  inv_scale[m] = s > 0.f ? 1.f / s : 0.f;
}

// ---------------------------------------------------------------------------- power iteration
constexpr int kPiPool = 16;

// Block m's pool seed: block_seed(seed, i) with i = seed_index[m] (global block index under block sharding) or
// m (spectral.py:117); seed_index[m] < 0 means "seed is the block's own seed" (multi_power_iteration).
__device__ __forceinline__ uint64_t pi_block_seed(unsigned long long seed, const int* seed_index, int m) {
  const int i = seed_index ? seed_index[m] : m;
  return i < 0 ? static_cast<uint64_t>(seed) : rng::block_seed(seed, static_cast<uint64_t>(i));
}

// ---------------------------------------------------------------------------- power iteration v2
// A thread-block cluster of C CTAs per block (C = ceil(d / 128) <= 8) splits the rows of A; every CTA
// streams its row slab of A once per iteration (the 4 MB block stays L2-resident across the 31 passes
// because only ~18 blocks are in flight), keeps the full pool V (d x 16, fp32) in shared memory, and the
// clusters exchange column norms and the new V rows through distributed shared memory.  A is symmetric,
// so the slab A[rows, k] is read as the contiguous row segment A[k, rows].
//
// Matvec thread tile: 4 rows x all 16 pool columns, 8 interleaved k-splits (one per warp: k = w, w + 8, ...).
// Each k costs one coalesced 16-byte global load of A per thread (512 B per warp) and four broadcast
// shared loads of V[k] for 64 FMAs, so the loop is FMA-bound instead of shared-memory bound; the eight
// k-split partials are summed in a fixed order (deterministic, batch-independent).
constexpr int kPi2Threads = 256;
constexpr int kPi2Cols = 16;      // pool columns per thread
constexpr int kPi2R = 128;       // max rows per CTA (32 row groups of 4)
constexpr int kPi2Splits = 8;     // interleaved k splits (one per warp)
constexpr int kPi2Ahead = 4;     // k steps of A prefetched into registers

struct Pi2Smem {
  static size_t bytes(int d) {
    return sizeof(float) * (2 * static_cast<size_t>(d) * kPiPool + static_cast<size_t>(kPi2Splits) * kPi2R * kPiPool +
                            kPi2R * kPiPool) +
           sizeof(double) * (8 * kPiPool * 3 + kPi2Threads) + 64;
  }
};

// A[k, row0 + r4 .. + 3] (== A[rows, k] by symmetry); k is clamped into range and out-of-range steps are
// zeroed by a select, so the unrolled k loop has no branches.  VEC: d, row0 and nr are multiples of 4.
template <bool VEC>
__device__ __forceinline__ float4 pi2_load_a(const float* __restrict__ a, int d, int k, int row0, int r4, int nr) {
  const int kc = k < d ? k : d - 1;
  const float* src = a + static_cast<long long>(kc) * d + row0;
  float4 x;
  if (VEC) {
    x = __ldg(reinterpret_cast<const float4*>(src + (r4 < nr ? r4 : 0)));
    if (r4 >= nr) x = make_float4(0.f, 0.f, 0.f, 0.f);
  } else {
    x.x = r4 < nr ? __ldg(src + r4) : 0.f;
    x.y = r4 + 1 < nr ? __ldg(src + r4 + 1) : 0.f;
    x.z = r4 + 2 < nr ? __ldg(src + r4 + 2) : 0.f;
    x.w = r4 + 3 < nr ? __ldg(src + r4 + 3) : 0.f;
  }
  if (k >= d) x = make_float4(0.f, 0.f, 0.f, 0.f);
  return x;
}

// W[r][0..15] = sum_k (A + eps I)[row0 + r][k] V[k][0..15] for this CTA's rows; the eps I term is added
// as eps V[row0 + r] in the fixed-order reduction.
template <bool VEC>
__device__ void pi2_matvec(const float* __restrict__ a, int d, float eps, int row0, int nr, const float* __restrict__ v,
                           float* __restrict__ red, float* __restrict__ w) {
  const int t = threadIdx.x, rg = t & 31, ks = (t >> 5) % kPi2Splits, ch = (t >> 5) / kPi2Splits, r4 = 4 * rg;
  float acc[4][kPi2Cols];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < kPi2Cols; ++j) acc[i][j] = 0.f;
  if (VEC && d % (kPi2Splits * kPi2Ahead) == 0 && nr == kPi2R) {
    // fast path (every DASH block size): no tail, full slab -> pointer-stepped loads, no selects
    const long long st4 = static_cast<long long>(kPi2Splits) * d / 4;  // float4 stride between my k steps
    const float4* p = reinterpret_cast<const float4*>(a + static_cast<long long>(ks) * d + row0 + r4);
    const float4* vks = reinterpret_cast<const float4*>(v) + ks * (kPiPool / 4) + ch * (kPi2Cols / 4);
    float4 pre[kPi2Ahead];
#pragma unroll
    for (int u = 0; u < kPi2Ahead; ++u) pre[u] = __ldg(p + u * st4);
    const int rounds = d / (kPi2Splits * kPi2Ahead);
    const int vstep = kPi2Splits * (kPiPool / 4);  // float4 stride of V between my consecutive k steps
    float4 vn[kPi2Cols / 4];                        // V row of the next k step (shared loads one step ahead)
#pragma unroll
    for (int j4 = 0; j4 < kPi2Cols / 4; ++j4) vn[j4] = vks[j4];
    for (int rd = 0; rd < rounds; ++rd) {
      const bool more = rd + 1 < rounds;
      const float4* pn = p + static_cast<long long>(kPi2Ahead) * (rd + 1) * st4;
#pragma unroll
      for (int u = 0; u < kPi2Ahead; ++u) {
        const float4 av = pre[u];
        if (more) pre[u] = __ldg(pn + u * st4);
        float4 vc[kPi2Cols / 4];
#pragma unroll
        for (int j4 = 0; j4 < kPi2Cols / 4; ++j4) vc[j4] = vn[j4];
        if (more || u + 1 < kPi2Ahead) {
          const float4* vk = vks + (kPi2Ahead * rd + u + 1) * vstep;
#pragma unroll
          for (int j4 = 0; j4 < kPi2Cols / 4; ++j4) vn[j4] = vk[j4];
        }
        const float ar[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
        for (int j4 = 0; j4 < kPi2Cols / 4; ++j4) {
          const float4 vv = vc[j4];
          const float vr[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][4 * j4 + j] = fmaf(ar[i], vr[j], acc[i][4 * j4 + j]);
        }
      }
    }
  } else {
  float4 pre[kPi2Ahead];
#pragma unroll
  for (int u = 0; u < kPi2Ahead; ++u) pre[u] = pi2_load_a<VEC>(a, d, ks + kPi2Splits * u, row0, r4, nr);
  for (int k0 = ks; k0 < d; k0 += kPi2Splits * kPi2Ahead) {
#pragma unroll
    for (int u = 0; u < kPi2Ahead; ++u) {
      const int k = k0 + kPi2Splits * u;
      const float4 av = pre[u];
      pre[u] = pi2_load_a<VEC>(a, d, k + kPi2Splits * kPi2Ahead, row0, r4, nr);
      const float4* vk = reinterpret_cast<const float4*>(v + (k < d ? k : 0) * kPiPool + ch * kPi2Cols);
      const float ar[4] = {av.x, av.y, av.z, av.w};  // zero when k >= d
#pragma unroll
      for (int j4 = 0; j4 < kPi2Cols / 4; ++j4) {
        const float4 vv = vk[j4];
        const float vr[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][4 * j4 + j] = fmaf(ar[i], vr[j], acc[i][4 * j4 + j]);
      }
    }
  }
  }
  // partials [split][row][16] -> fixed-order sum over the splits (+ eps V)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float4* dst = reinterpret_cast<float4*>(red + (ks * kPi2R + r4 + i) * kPiPool + ch * kPi2Cols);
#pragma unroll
    for (int j4 = 0; j4 < kPi2Cols / 4; ++j4)
      dst[j4] = make_float4(acc[i][4 * j4], acc[i][4 * j4 + 1], acc[i][4 * j4 + 2], acc[i][4 * j4 + 3]);
  }
  __syncthreads();
  for (int e = t; e < nr * kPiPool; e += kPi2Threads) {
    float x = 0.f;
#pragma unroll
    for (int s2 = 0; s2 < kPi2Splits; ++s2) x += red[s2 * kPi2R * kPiPool + e];
    w[e] = fmaf(eps, v[row0 * kPiPool + e], x);
  }
  __syncthreads();
}

// Cluster-wide fixed-order column sums: out[j] = sum over ranks q of (sum over my rows of f(x, y)).
__device__ void pi2_colsum(cg::cluster_group& cl, int C, int q, const float* __restrict__ x, int xstride,
                           const float* __restrict__ y, int nr, double* stripes, double* slots, double* out) {
  const int t = threadIdx.x, j = t % kPiPool, s = t / kPiPool;  // 16 stripes
  double acc = 0.0;
  for (int r = s; r < nr; r += kPi2Threads / kPiPool) {
    const double xv = x[r * xstride + j];
    acc += xv * (y ? static_cast<double>(y[r * kPiPool + j]) : xv);
  }
  stripes[s * kPiPool + j] = acc;
  __syncthreads();
  if (t < kPiPool) {
    double p = 0.0;
    for (int i = 0; i < kPi2Threads / kPiPool; ++i) p += stripes[i * kPiPool + t];
    for (int dst = 0; dst < C; ++dst) {
      double* remote = cl.map_shared_rank(slots, dst);
      remote[q * kPiPool + t] = p;
    }
  }
  cl.sync();
  if (t < kPiPool) {
    double tot = 0.0;
    for (int i = 0; i < C; ++i) tot += slots[i * kPiPool + t];
    out[t] = tot;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kPi2Threads, 1) pi2_kernel(const float* __restrict__ ema, int d, float eps, int pool,
                                                             int iters, unsigned long long seed,
                                                             float* __restrict__ scale, float* __restrict__ inv_scale,
                                                             int* __restrict__ status,
                                                             const int* __restrict__ seed_index, int exp_flags,
                                                             float* __restrict__ vec_out, int retry_only) {
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks());
  const int q = static_cast<int>(cl.block_rank());
  const int m = blockIdx.x / C;
  // retry mode: only blocks the tensor-core kernel flagged (status 3, collapsed pool) run; the whole cluster of
  // every other block leaves before touching distributed shared memory
  if (retry_only && status[m] != 3) return;
  const int R = ((d + C - 1) / C + 3) / 4 * 4;  // rows per CTA, a multiple of 4 (16-byte aligned slabs)
  const bool vec = d % 4 == 0;
  const int row0 = q * R;
  const int nr = max(0, min(R, d - row0));
  extern __shared__ __align__(16) unsigned char pi2_raw[];
  float* vbuf = reinterpret_cast<float*>(pi2_raw);                 // [2][d][16]
  float* red = vbuf + 2 * d * kPiPool;                              // [splits][R][16]
  float* w = red + kPi2Splits * kPi2R * kPiPool;                    // [R][16]
  double* stripes = reinterpret_cast<double*>(w + kPi2R * kPiPool);  // [16][16]
  double* slots = stripes + kPi2Threads;                            // [8][16]
  double* colv = slots + 8 * kPiPool;                               // [16]
  double* qv = colv + kPiPool;                                      // [16]
  double* vv = qv + kPiPool;                                        // [16]
  const float* a = ema + static_cast<long long>(m) * d * d;
  uint64_t bseed = pi_block_seed(seed, seed_index, m);
  // start vectors for my rows into w: element (j, i) is draw j*d + i of default_rng(sd); colv <- column |.|^2
  auto draw_start = [&](uint64_t sd) {
    const int per = (nr + 15) / 16;  // rows per (j, chunk) task
    for (int task = threadIdx.x; task < kPiPool * 16; task += kPi2Threads) {
      const int j = task / 16, c = task % 16;
      const int r0 = c * per, r1 = min(nr, r0 + per);
      if (r0 >= r1) continue;
      if (j < pool) {
        rng::Pcg64 g;
        g.seed(sd);
        g.advance(static_cast<uint64_t>(j) * d + row0 + r0);
        for (int r = r0; r < r1; ++r) w[r * kPiPool + j] = static_cast<float>(g.uniform_pm1());
      } else {
        for (int r = r0; r < r1; ++r) w[r * kPiPool + j] = 0.f;
      }
    }
    __syncthreads();
    pi2_colsum(cl, C, q, w, kPiPool, nullptr, nr, stripes, slots, colv);
  };
  float lam = 0.f;
  int st = 0, best = -1;
  bool zero_matrix = false;
  const float* vfinal = vbuf;
  for (int attempt = 0; attempt < 2; ++attempt) {
    float* v = vbuf;
    draw_start(bseed);
    // normalize (zero norm -> 1) and broadcast my rows of V0 to every CTA of the cluster
    for (int i = threadIdx.x; i < nr * kPiPool; i += kPi2Threads) {
      const int j = i % kPiPool;
      double n = sqrt(colv[j]);
      if (n == 0.0) n = 1.0;
      const float x = static_cast<float>(w[i] / n);
      for (int dst = 0; dst < C; ++dst) cl.map_shared_rank(v, dst)[row0 * kPiPool + i] = x;
    }
    cl.sync();
    int cur = 0;
    for (int it = 0; it < iters; ++it) {
      const float* vc = vbuf + cur * d * kPiPool;
      float* vn = vbuf + (cur ^ 1) * d * kPiPool;
      if (exp_flags & 1) {  // experiment: skip the matvec (W = V)
        for (int i = threadIdx.x; i < nr * kPiPool; i += kPi2Threads) w[i] = vc[row0 * kPiPool + i];
        __syncthreads();
      } else {
        if (vec) pi2_matvec<true>(a, d, eps, row0, nr, vc, red, w);
        else pi2_matvec<false>(a, d, eps, row0, nr, vc, red, w);
      }
      pi2_colsum(cl, C, q, w, kPiPool, nullptr, nr, stripes, slots, colv);
      for (int i = threadIdx.x; i < nr * kPiPool; i += kPi2Threads) {
        const double n = sqrt(colv[i % kPiPool]);
        const float x = n > 0.0 ? static_cast<float>(w[i] / n) : 0.f;
        for (int dst = 0; dst < C; ++dst) cl.map_shared_rank(vn, dst)[row0 * kPiPool + i] = x;
      }
      cl.sync();
      cur ^= 1;
    }
    const float* vc = vbuf + cur * d * kPiPool;
    vfinal = vc;
    if (vec) pi2_matvec<true>(a, d, eps, row0, nr, vc, red, w);  // A V once more for the quotients
    else pi2_matvec<false>(a, d, eps, row0, nr, vc, red, w);
    pi2_colsum(cl, C, q, vc + row0 * kPiPool, kPiPool, w, nr, stripes, slots, qv);
    pi2_colsum(cl, C, q, vc + row0 * kPiPool, kPiPool, nullptr, nr, stripes, slots, vv);
    // every CTA evaluates the (identical) selection; rank 0 writes the result
    best = -1;
    double bq = 0.0;
    bool any = false;
    for (int j = 0; j < pool; ++j) {
      if (vv[j] > 0.0) {
        if (!any || qv[j] > bq) { bq = qv[j]; best = j; }
        any = true;
      }
    }
    if (any && bq != 0.0) {
      lam = static_cast<float>(bq / vv[best]);
      break;
    }
    if (attempt == 0) {
      // collapsed pool: the zero matrix yields lambda = 0 with the first start vector (spectral.py:99-101)
      int nz = 0;
      if (eps != 0.f) nz = 1;
      for (long long i = threadIdx.x; !nz && i < static_cast<long long>(nr) * d; i += kPi2Threads)
        nz = a[static_cast<long long>(row0) * d + i] != 0.f;
      nz = __syncthreads_or(nz);
      if (threadIdx.x == 0)
        for (int dst = 0; dst < C; ++dst) cl.map_shared_rank(slots, dst)[q * kPiPool] = nz ? 1.0 : 0.0;
      cl.sync();
      double tot = 0.0;
      for (int i = 0; i < C; ++i) tot += slots[i * kPiPool];
      cl.sync();
      if (tot == 0.0) {
        zero_matrix = true;
        lam = 0.f;
        break;
      }
      bseed = rng::block_seed(bseed, 0x5EEDull);
      st = 1;
    } else {
      st = 2;
    }
    cl.sync();
  }
  if (vec_out) {  // the selected (normalized) vector, or the first start vector of a zero matrix
    float* out = vec_out + static_cast<long long>(m) * d + row0;
    if (zero_matrix) {
      cl.sync();
      draw_start(pi_block_seed(seed, seed_index, m));
      const double n = colv[0] > 0.0 ? sqrt(colv[0]) : 1.0;
      for (int r = threadIdx.x; r < nr; r += kPi2Threads) out[r] = static_cast<float>(w[r * kPiPool] / n);
    } else if (best >= 0 && vv[best] > 0.0) {
      const double n = sqrt(vv[best]);
      for (int r = threadIdx.x; r < nr; r += kPi2Threads)
        out[r] = static_cast<float>(vfinal[(row0 + r) * kPiPool + best] / n);
    }
  }
  if (q == 0 && threadIdx.x == 0) {
    const float s = 2.f * lam;
    scale[m] = s;
    inv_scale[m] = s > 0.f ? 1.f / s : 0.f;
    if (status) status[m] = (st == 2) ? 2 : (s > 0.f ? 0 : 1);
  }
  cl.sync();  // keep every CTA's shared memory alive until all remote writes are done
}

static int pi2_launch(const float* ema, int n, int d, float eps, int pool, int iters, unsigned long long seed,
                      float* scale, float* inv_scale, int* status, const int* seed_index, float* vec_out,
                      cudaStream_t st, int retry_only = 0) {
  int C = (d + kPi2R - 1) / kPi2R;
  if (C > 8) return DASH_EINVAL;
  if (C < 1) C = 1;
  const size_t smem = Pi2Smem::bytes(d);
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(pi2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(n * C));
  cfg.blockDim = dim3(kPi2Threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = C;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  static const int exp_flags = getenv("DASH_PI_EXP") ? atoi(getenv("DASH_PI_EXP")) : 0;  // experiment knob
  cudaError_t e = cudaLaunchKernelEx(&cfg, pi2_kernel, ema, d, eps, pool, iters, seed, scale, inv_scale, status,
                                     seed_index, exp_flags, vec_out, retry_only);
  note_launch();
  return e == cudaSuccess ? DASH_OK : DASH_ECUDA;
}

int pi_retry_launch(const float* ema, int n, int d, float eps, int pool, int iters, unsigned long long seed,
                    float* scale, float* inv_scale, int* status, const int* seed_index, cudaStream_t st) {
  return pi2_launch(ema, n, d, eps, pool, iters, seed, scale, inv_scale, status, seed_index, nullptr, st, 1);
}

// ---------------------------------------------------------------------------- grafted update
// theta_out = theta_in - eta * s_b * U with s_b = |P_b| / |U_b| (0 if |U_b| = 0) (shampoo.py:352-359, :393).
__global__ void __launch_bounds__(256) update_kernel(const dash_block* __restrict__ blocks, int nb_m, int bsz,
                                                     const float* __restrict__ pn_part,
                                                     const float* __restrict__ un_part, int un_stride,
                                                     const float* __restrict__ um, const float* __restrict__ uv,
                                                     const float* __restrict__ theta_in, float* __restrict__ theta_out,
                                                     float eta, float* __restrict__ graft_s) {
  const int b = blockIdx.y;
  const dash_block blk = blocks[b];
  __shared__ float coef;
  if (threadIdx.x == 0) {
    double pn = 0.0, un = 0.0;
    for (int p = 0; p < kPrepParts; ++p) pn += pn_part[b * kPrepParts + p];
    const int ntiles = ((blk.rows + kTileM - 1) / kTileM) * ((blk.cols + kTileN - 1) / kTileN) * kPartialsPerTile;
    for (int i = 0; i < ntiles; ++i) un += un_part[static_cast<long long>(b) * un_stride + i];
    const double s = un == 0.0 ? 0.0 : sqrt(pn) / sqrt(un);
    coef = static_cast<float>(static_cast<double>(eta) * s);
    if (graft_s && blockIdx.x == 0) graft_s[b] = static_cast<float>(s);
  }
  __syncthreads();
  const float k = coef;
  const float* u = b < nb_m ? um + static_cast<long long>(b) * bsz * bsz : uv + static_cast<long long>(b - nb_m) * bsz;
  const int uld = b < nb_m ? bsz : 1;
  const long long total = static_cast<long long>(blk.rows) * blk.cols;
  if (blk.cols % 4 == 0 && blk.ld % 4 == 0 && blk.off % 4 == 0 && uld % 4 == 0) {  // 16-byte accesses
    const int c4n = blk.cols / 4;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total / 4;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
      const int r = static_cast<int>(e / c4n), c = static_cast<int>(e % c4n) * 4;
      const long long i = blk.off + static_cast<long long>(r) * blk.ld + c;
      const float4 t = __ldg(reinterpret_cast<const float4*>(theta_in + i));
      const float4 uu = __ldg(reinterpret_cast<const float4*>(u + static_cast<long long>(r) * uld + c));
      *reinterpret_cast<float4*>(theta_out + i) = make_float4(t.x - k * uu.x, t.y - k * uu.y, t.z - k * uu.z,
                                                              t.w - k * uu.w);
    }
  } else {
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
      const int r = static_cast<int>(e / blk.cols), c = static_cast<int>(e % blk.cols);
      const long long i = blk.off + static_cast<long long>(r) * blk.ld + c;
      theta_out[i] = theta_in[i] - k * u[static_cast<long long>(r) * uld + c];
    }
  }
}

// ---------------------------------------------------------------------------- shard exchange
// Block-major packing of (a subset of) the flat parameter space: block b occupies
// packed[pos[b] .. pos[b] + rows*cols) in row-major order.  Used around the NCCL all-gather of the
// updated parameter shards (one rank owns each gradient block).
template <bool PACK>
__global__ void __launch_bounds__(256) pack_kernel(const dash_block* __restrict__ blocks,
                                                   const long long* __restrict__ pos, float* __restrict__ flat,
                                                   float* __restrict__ packed) {
  const int b = blockIdx.y;
  const dash_block blk = blocks[b];
  const long long total = static_cast<long long>(blk.rows) * blk.cols;
  const long long base = pos[b];
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / blk.cols), c = static_cast<int>(e % blk.cols);
    const long long i = blk.off + static_cast<long long>(r) * blk.ld + c;
    if (PACK) packed[base + e] = flat[i];
    else flat[i] = packed[base + e];
  }
}

// ---------------------------------------------------------------------------- plan
}  // namespace dash

struct dash_plan {
  int nb_m = 0, nb_v = 0, bsz = 0, ngroups = 0;
  std::vector<dash_block> hblocks;  // matrix blocks then vector chunks
  std::vector<int> gdim, gsize;
  std::vector<float*> gema;
  std::vector<dash_stack> groot;
  dash_block* dblocks = nullptr;
  float *grad = nullptr, *adam = nullptr, *mom = nullptr, *um = nullptr, *uv = nullptr;
  float *pn_part = nullptr, *un_part = nullptr, *graft_s = nullptr;
  unsigned* gamax = nullptr;
  const long long* sofs = nullptr;  // owner-only optimizer state: per-block packed offsets (device, caller-owned)
  int un_stride = 0;
  dash_stack gsm{}, gsv{}, tm{};
  dash::UploadedGemm g_stats, g_apply1, g_apply2;
  float beta_lr = 0.95f;
  int passes = 3;
};

namespace dash {

static int un_stride_for(int bsz) {
  return kPartialsPerTile * ((bsz + kTileM - 1) / kTileM) * ((bsz + kTileN - 1) / kTileN);
}

static void set_dims(GemmJob& j, int M, int N, int K) {
  j.M = M;
  j.N = N;
  j.K = K;
  j.tiles_n = (N + kTileN - 1) / kTileN;
  j.tiles_n2 = (N + 255) / 256;
}

static dash_stack slot_stack(const dash_stack& s) { return s; }

size_t plan_ws_bytes(int nb_m, int nb_v) {
  const int nb = nb_m + nb_v;
  return Arena::need(sizeof(dash_block) * nb) + JobBuilder::bytes_for(64, 2 * nb) +
         JobBuilder::bytes_for(64, nb) * 2 + 8192;
}

}  // namespace dash

using namespace dash;

extern "C" {

size_t dash_plan_ws_bytes(int nb_m, int nb_v) { return plan_ws_bytes(nb_m, nb_v); }

dash_plan* dash_plan_create(const dash_block* blocks, int nb_m, int nb_v, int block_size, int ngroups,
                            const int* gdim, const int* gsize, float* const* gema, const dash_stack* groot,
                            float* grad, float* adam, float* mom, const dash_stack* gsm, const dash_stack* gsv,
                            const dash_stack* tm, float* um, float* uv, float* pn_part, float* un_part,
                            unsigned* gamax, float* graft_s, float beta_lr, int passes, void* ws, size_t ws_bytes,
                            void* stream, int* status) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto fail = [&](int code) -> dash_plan* {
    if (status) *status = code;
    return nullptr;
  };
  if (!blocks || nb_m < 0 || nb_v < 0 || nb_m + nb_v == 0 || block_size < 1 || ngroups < 1 || !grad || !adam ||
      !pn_part || !un_part || !gamax || (passes != 1 && passes != 3 && passes != 4))
    return fail(DASH_EINVAL);
  if ((nb_m && (!stack_ok(gsm) || !stack_ok(tm) || !um)) || (nb_v && (!stack_ok(gsv) || !uv))) return fail(DASH_EINVAL);
  dash_plan* p = new dash_plan();
  p->nb_m = nb_m;
  p->nb_v = nb_v;
  p->bsz = block_size;
  p->ngroups = ngroups;
  p->hblocks.assign(blocks, blocks + nb_m + nb_v);
  p->gdim.assign(gdim, gdim + ngroups);
  p->gsize.assign(gsize, gsize + ngroups);
  p->gema.assign(gema, gema + ngroups);
  p->groot.assign(groot, groot + ngroups);
  p->grad = grad; p->adam = adam; p->mom = mom; p->um = um; p->uv = uv;
  p->pn_part = pn_part; p->un_part = un_part; p->gamax = gamax; p->graft_s = graft_s;
  if (nb_m) { p->gsm = *gsm; p->tm = *tm; }
  if (nb_v) p->gsv = *gsv;
  p->un_stride = un_stride_for(block_size);
  p->beta_lr = beta_lr;
  p->passes = passes;
  Arena ar(ws, ws_bytes);
  const int nb = nb_m + nb_v;
  p->dblocks = ar.take_n<dash_block>(nb);
  if (!ar.ok) { delete p; return fail(DASH_EINVAL); }
  cudaMemcpyAsync(p->dblocks, p->hblocks.data(), sizeof(dash_block) * nb, cudaMemcpyHostToDevice, st);
  // ---- statistics EMA jobs: L = G G^T, R = G^T G per matrix block, L = g g^T per vector chunk
  JobBuilder js, j1, j2;
  for (int b = 0; b < nb; ++b) {
    const dash_block& k = p->hblocks[b];
    const bool mat = b < nb_m;
    const dash_stack& gs = mat ? p->gsm : p->gsv;
    const int sidx = mat ? b : b - nb_m;
    if (k.group_l < 0 || k.group_l >= ngroups || (mat && (k.group_r < 0 || k.group_r >= ngroups))) {
      delete p;
      return fail(DASH_EINVAL);
    }
    GemmJob j;
    // L
    if (!js.operands(j, gs, sidx, 0, gs, sidx, 1, false)) { delete p; return fail(DASH_EINVAL); }
    set_dims(j, k.rows, k.rows, k.cols);
    j.op = EPI_EMA;
    j.beta = beta_lr;
    {
      const int d = p->gdim[k.group_l];
      js.set_fout(j, p->gema[k.group_l], p->gsize[k.group_l], d, d, k.slot_l, true);
    }
    // G G^T (and G^T G, g g^T) is symmetric: only the tiles on / above the diagonal run, the epilogue writes the
    // transposed tile below (the EMA input of a lower tile is the transpose of its upper one)
    j.sym = j.f_map >= 0 ? 1 : 0;
    js.push(j);
    if (mat) {  // R
      if (!js.operands(j, gs, sidx, 1, gs, sidx, 0, false)) { delete p; return fail(DASH_EINVAL); }
      set_dims(j, k.cols, k.cols, k.rows);
      j.op = EPI_EMA;
      j.beta = beta_lr;
      const int d = p->gdim[k.group_r];
      js.set_fout(j, p->gema[k.group_r], p->gsize[k.group_r], d, d, k.slot_r, true);
      j.sym = j.f_map >= 0 ? 1 : 0;
      js.push(j);
    }
    // ---- apply jobs
    const dash_stack& rl = p->groot[k.group_l];
    if (mat) {
      // T = rootL G_b  (split, into tm slot b)
      if (!j1.operands(j, rl, k.slot_l, 0, gs, sidx, 0, false)) { delete p; return fail(DASH_EINVAL); }
      set_dims(j, k.rows, k.cols, k.rows);
      j.op = EPI_SPLIT;
      j.out_mat = b;
      j1.set_out(j, p->tm, b);
      j1.push(j);
      // U = T rootR  (fp32 block layout + per-tile sum(U^2))
      const dash_stack& rr = p->groot[k.group_r];
      if (!j2.operands(j, p->tm, b, 0, rr, k.slot_r, 0, false)) { delete p; return fail(DASH_EINVAL); }
      set_dims(j, k.rows, k.cols, k.cols);
      j.op = EPI_APPLY;
      j.out_mat = b;
      j2.set_fout(j, p->um, p->nb_m, block_size, block_size, b);
      j.partial = p->un_part + static_cast<long long>(b) * p->un_stride;
      j2.push(j);
    } else {
      // u = rootL g_c (vector chunk)
      if (!j1.operands(j, rl, k.slot_l, 0, gs, sidx, 0, false)) { delete p; return fail(DASH_EINVAL); }
      set_dims(j, k.rows, 1, k.rows);
      j.op = EPI_APPLY;
      j.out_mat = b;
      j.f_out = p->uv + static_cast<long long>(sidx) * block_size;
      j.f_ld = 1;
      j.partial = p->un_part + static_cast<long long>(b) * p->un_stride;
      j1.push(j);
    }
  }
  if (!js.upload(ar, st, &p->g_stats) || !j1.upload(ar, st, &p->g_apply1) || !j2.upload(ar, st, &p->g_apply2)) {
    delete p;
    return fail(DASH_EINVAL);
  }
  if (status) *status = cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_ECUDA;
  return p;
}

void dash_plan_destroy(dash_plan* p) { delete p; }

int dash_plan_set_state_offsets(dash_plan* p, const long long* d_offsets) {
  if (!p) return DASH_EINVAL;
  p->sofs = d_offsets;
  return DASH_OK;
}

// accumulate (shampoo.py:238-278) + graft-direction norms for step index t (n_acc = t + 1).
int dash_plan_accumulate(dash_plan* p, float beta2, float beta1, int n_acc, float graft_eps, void* stream) {
  if (!p) return DASH_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nb = p->nb_m + p->nb_v;
  const float bc1_inv = p->mom ? static_cast<float>(1.0 / (1.0 - std::pow(static_cast<double>(beta1), n_acc))) : 1.f;
  const float bc2_inv = static_cast<float>(1.0 / (1.0 - std::pow(static_cast<double>(beta2), n_acc)));
  cudaMemsetAsync(p->gamax, 0, sizeof(unsigned) * nb, st);
  prep_kernel<<<dim3(kPrepParts, nb), 256, 0, st>>>(p->dblocks, p->grad, p->adam, p->mom, beta2, beta1, bc1_inv,
                                                   bc2_inv, graft_eps, p->pn_part, p->gamax, p->sofs);
  note_launch();
  if (p->nb_m) {
    grad_split_kernel<<<dim3(32, p->nb_m), 256, 0, st>>>(p->dblocks, p->grad, p->gsm, p->gamax);
    note_launch();
  }
  if (p->nb_v) {
    grad_split_kernel<<<dim3(4, p->nb_v), 256, 0, st>>>(p->dblocks + p->nb_m, p->grad, p->gsv, p->gamax + p->nb_m);
    note_launch();
  }
  if (int rc = p->g_stats.run(p->passes, st)) return rc;
  return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_ECUDA;
}

// Symmetrize one group's EMA stack and (optionally) emit a = ema + eps I as a split stack.
int dash_group_sym(float* ema, int n, int d, float eps, unsigned* amax, float* fro_part, void* stream) {
  if (!ema || n < 1 || d < 1 || !amax || !fro_part) return DASH_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaMemsetAsync(amax, 0, sizeof(unsigned) * n, st);
  sym_kernel<<<dim3(kPrepParts, n), 256, 0, st>>>(ema, d, eps, amax, fro_part);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_ECUDA;
}

int dash_group_split_a(const float* ema, float eps, const dash_stack* a, void* stream) {
  if (!ema || !stack_ok(a) || a->rows != a->cols) return DASH_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  long long el = static_cast<long long>(a->rows) * a->ld;
  int gx = static_cast<int>(std::min<long long>(64, std::max<long long>(1, el / 4096)));
  a_split_kernel<<<dim3(gx, a->nmat), 256, 0, st>>>(ema, eps, *a);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_ECUDA;
}

int dash_fro_scale(const float* fro_part, int n, float* scale, float* inv_scale, void* stream) {
  if (!fro_part || n < 1 || !scale || !inv_scale) return DASH_EINVAL;
  fro_scale_kernel<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(fro_part, n, scale, inv_scale);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_ECUDA;
}

int dash_power_iteration(const float* ema, int n, int d, float eps, int pool, int iters, unsigned long long seed,
                         float* scale, float* inv_scale, int* status, const int* seed_index, float* vec_out,
                         void* stream) {
  if (!ema || n < 1 || d < 1 || d > 1024 || pool < 1 || pool > kPiPool || iters < 1 || !scale || !inv_scale)
    return DASH_EINVAL;
  // cluster kernel: the rows of every block split over ceil(d / 128) <= 8 CTAs
  return pi2_launch(ema, n, d, eps, pool, iters, seed, scale, inv_scale, status, seed_index, vec_out,
                    static_cast<cudaStream_t>(stream));
}

// Apply L^(-1/4) G R^(-1/4) (1-D: L^(-1/2) g) and the grafted update theta_out = theta_in - eta s_b U_b.
int dash_plan_apply(dash_plan* p, const float* theta_in, float* theta_out, float eta, void* stream) {
  if (!p || !theta_in || !theta_out) return DASH_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = p->g_apply1.run(p->passes, st)) return rc;
  if (int rc = p->g_apply2.run(p->passes, st)) return rc;
  const int nb = p->nb_m + p->nb_v;
  update_kernel<<<dim3(16, nb), 256, 0, st>>>(p->dblocks, p->nb_m, p->bsz, p->pn_part, p->un_part, p->un_stride,
                                             p->um, p->uv, theta_in, theta_out, eta, p->graft_s);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_ECUDA;
}

int dash_plan_un_stride(const dash_plan* p) { return p ? p->un_stride : -1; }
int dash_prep_parts(void) { return kPrepParts; }
int dash_apply_partials(int block_size) { return block_size > 0 ? un_stride_for(block_size) : -1; }

int dash_pack_blocks(const dash_block* blocks, int n, const long long* pos, const float* flat, float* packed,
                     void* stream) {
  if (n < 0 || (n && (!blocks || !pos || !flat || !packed))) return DASH_EINVAL;
  if (n) {
    pack_kernel<true><<<dim3(16, n), 256, 0, static_cast<cudaStream_t>(stream)>>>(blocks, pos, const_cast<float*>(flat),
                                                                                 packed);
    note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_ECUDA;
}

int dash_unpack_blocks(const dash_block* blocks, int n, const long long* pos, const float* packed, float* flat,
                       void* stream) {
  if (n < 0 || (n && (!blocks || !pos || !flat || !packed))) return DASH_EINVAL;
  if (n) {
    pack_kernel<false><<<dim3(16, n), 256, 0, static_cast<cudaStream_t>(stream)>>>(blocks, pos, flat,
                                                                                  const_cast<float*>(packed));
    note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_ECUDA;
}

unsigned long long dash_block_seed(unsigned long long seed, unsigned long long index) {
  return rng::block_seed(seed, index);
}

// First `count` draws of default_rng(seed).uniform(-1, 1) computed on the device (test hook for the
// NumPy-compatible stream used by the power iteration).
__global__ void uniform_kernel(unsigned long long seed, int count, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  rng::Pcg64 g;
  g.seed(seed);
  g.advance(static_cast<uint64_t>(i));
  out[i] = g.uniform_pm1();
}

int dash_uniform_pm1(unsigned long long seed, int count, double* out, void* stream) {
  if (count < 0 || !out) return DASH_EINVAL;
  if (count) uniform_kernel<<<(count + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, count, out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_ECUDA;
}

}  // extern "C"
