// Batched inverse-root solvers: Newton-Denman-Beavers (NDB) and Coupled Newton (CN) with per-block
// freezing, divergence watch and reports, all device-resident (no host round trip per iteration).
//
// Reference semantics: roots.py:216-305 (batched_coupled_newton / batched_newton_db), the watch
// roots.py:71-86, the max-norm residual roots.py:212-213.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <vector>

#include "engine.h"
#include "elem.cuh"
#include "ptx.cuh"
#include "solver.h"

namespace dash {

// ---------------------------------------------------------------------------- per-block state
struct BlockState {  // struct-of-arrays in the workspace
  int* active;       // [n]
  float* hist;       // [n * 4] last residuals (oldest first)
  int* hlen;         // [n]
  float* last;       // [n] most recent residual (report for never-frozen blocks)
  unsigned* resid;   // [n] residual accumulator (float bits, atomicMax)
  int* n_active;     // [1]
  int* par;          // [1] which ping-pong buffer holds the latest iterate (flips only when GEMMs ran)
};

static bool take_state(Arena& ar, int n, BlockState* s) {
  s->active = ar.take_n<int>(n);
  s->hist = ar.take_n<float>(4 * n);
  s->hlen = ar.take_n<int>(n);
  s->last = ar.take_n<float>(n);
  s->resid = ar.take_n<unsigned>(n);
  s->n_active = ar.take_n<int>(1);
  s->par = ar.take_n<int>(1);
  return ar.ok;
}

static size_t state_bytes(int n) {
  return Arena::need(4 * n) * 3 + Arena::need(16 * n) + Arena::need(4 * n) + 2 * Arena::need(4);
}

__global__ void state_init_kernel(BlockState s, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    s.active[i] = 1;
    s.hlen[i] = 0;
    s.resid[i] = 0u;
    s.last[i] = __uint_as_float(0x7f800000u);
    if (i == 0) {
      *s.n_active = n;
      *s.par = 0;
    }
  }
}

__global__ void set_par_kernel(int* par, int v) { *par = v; }

// Zero up to three amax arrays, but only when the gated GEMMs that refill them will run.
__global__ void zero_amax_gated_kernel(const int* gate, int n, unsigned* a, unsigned* b, unsigned* c) {
  if (gate && *gate == 0) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (a) a[i] = 0u;
    if (b) b[i] = 0u;
    if (c) c[i] = 0u;
  }
}

static void zero_amax(const int* gate, int n, unsigned* a, unsigned* b, unsigned* c, cudaStream_t st) {
  zero_amax_gated_kernel<<<(n + 255) / 256, 256, 0, st>>>(gate, n, a, b, c);
  note_launch();
}

// _DivergenceWatch.update (roots.py:77-86): keep 4 residuals, trip on 3 strict rises with >10x growth.
__device__ bool watch_push(float* h, int* hl, float r) {
  int n = *hl;
  if (n < 4) {
    h[n] = r;
    *hl = ++n;
  } else {
    h[0] = h[1]; h[1] = h[2]; h[2] = h[3]; h[3] = r;
  }
  return n == 4 && h[3] > h[2] && h[2] > h[1] && h[1] > h[0] && h[3] > 10.f * h[0];
}

// One iteration's freeze decisions in reference order (roots.py:291-301, and :274-280 when first).
// stall > 0 (a tolerance below the precision floor, see SolverConfig): a block whose residual stops decreasing
// (r_k >= r_{k-1}) once r_{k-1} <= stall has reached the rounding floor of the arithmetic and is frozen as
// converged there (checked after the non-finite and tolerance rules, before the watch).
// z0..z2 (nullable): amax arrays of the next iteration's GEMM outputs, zeroed here when blocks stay active (the
// gated GEMMs refill them), which saves two launches per Newton-DB iteration.
__global__ void freeze_kernel(BlockState s, int n, int k, float tol, float stall, int first, int* iters,
                              float* resid_out, int* conv, int* newly_frozen, unsigned* z0 = nullptr,
                              unsigned* z1 = nullptr, unsigned* z2 = nullptr) {
  __shared__ int cnt;
  if (threadIdx.x == 0) {
    cnt = 0;
    if (!first && *s.n_active > 0) *s.par ^= 1;  // this iteration's (gated) GEMMs ran
  }
  __syncthreads();
  int local = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const float r = __uint_as_float(s.resid[i]);
    s.resid[i] = 0u;
    if (newly_frozen) newly_frozen[i] = 0;
    if (!s.active[i]) continue;
    const float prev = s.last[i];
    s.last[i] = r;
    bool stop = false, ok = false;
    if (first) {
      if (r <= tol) { stop = true; ok = true; }
      else watch_push(s.hist + 4 * i, s.hlen + i, r);
    } else if (!isfinite(r)) {
      stop = true;
    } else if (r <= tol) {
      stop = true; ok = true;
    } else if (stall > 0.f && r >= prev && prev <= stall) {
      stop = true; ok = true;
    } else if (watch_push(s.hist + 4 * i, s.hlen + i, r)) {
      stop = true;
    }
    if (stop) {
      s.active[i] = 0;
      iters[i] = k;
      resid_out[i] = r;
      conv[i] = ok ? 1 : 0;
      if (newly_frozen) newly_frozen[i] = 1;
    } else {
      ++local;
    }
  }
  atomicAdd(&cnt, local);
  __syncthreads();
  if (threadIdx.x == 0) *s.n_active = cnt;
  if (cnt > 0)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      if (z0) z0[i] = 0u;
      if (z1) z1[i] = 0u;
      if (z2) z2[i] = 0u;
    }
}

// Reports of blocks still active after the loop: (max_iters, last residual, False) (roots.py:302-304).
__global__ void finish_kernel(BlockState s, int n, int max_iters, int* iters, float* resid_out, int* conv) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (s.active[i]) {
      iters[i] = max_iters;
      resid_out[i] = s.last[i];
      conv[i] = 0;
    }
  }
}

// ---------------------------------------------------------------------------- elementwise kernels
// NDB closed-form first iteration (roots.py:267-271): E1 = 1.5 I - 0.5 a_hat, Z1 = E1,
// residual max|E1 - I|; a_hat = a * inv_scale[m].
// upper = 1: E1 / Z1 are consumed only as upper pair-block operands, so only those blocks of `a` are read
// and written (the input may itself be upper-stored, e.g. the first solve's Y of an inverse 4th root).
__global__ void ndb_first_kernel(dash_stack a, const float* __restrict__ inv_scale, dash_stack e, dash_stack z,
                                 unsigned* __restrict__ resid, int upper) {
  const int m = blockIdx.y;
  const int n = a.rows;
  const float sa = ldexpf(1.f, a.exp[m]) * (inv_scale ? inv_scale[m] : 1.f);
  const float inv_e = ldexpf(1.f, -kEExp);
  const __half* ah = mat_hi(a, m);
  __half* eh = mat_hi(e, m);
  __half* zh = mat_hi(z, m);
  float rmax = 0.f, amax = 0.f;
  bool ovf = false;
  for_chunks8(n, a.ld, [&](int r, int c) {
    if (upper && (r >> 8) > (c >> 8)) return;  // lower pair block (never read)
    float v[8];
    load_split8(ah, mat_plane(a), static_cast<long long>(r) * a.ld + c, sa, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float d = (r == c + i) ? 1.f : 0.f;
      const float ev = (c + i < n) ? 1.5f * d - 0.5f * v[i] : 0.f;
      v[i] = ev;
      rmax = nonneg_max(rmax, fabsf(ev - d));
      amax = nonneg_max(amax, fabsf(ev));
    }
    ovf |= store_split8(eh, mat_plane(e), static_cast<long long>(r) * e.ld + c, v, inv_e);
    store_split8(zh, mat_plane(z), static_cast<long long>(r) * z.ld + c, v, inv_e);
  });
  if (ovf) { rmax = __uint_as_float(0x7fc00000u); amax = rmax; }
  rmax = warp_max_nonneg(rmax);
  amax = warp_max_nonneg(amax);
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(resid + m, rmax);
    atomic_max_nonneg(e.amax + m, amax);
    atomic_max_nonneg(z.amax + m, amax);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    e.exp[m] = kEExp;
    z.exp[m] = kEExp;
  }
}

// CN initial state (roots.py:228-229): X0 = I / c, M0 = a_hat / c^p, and the first correction
// C1 = (1 + 1/p) I - M0 / p (roots.py:236); residual slot unused here.
__global__ void cn_first_kernel(dash_stack a, const float* __restrict__ inv_scale, float inv_c, float inv_cp,
                                float p, dash_stack x, dash_stack mm, dash_stack corr) {
  const int m = blockIdx.y;
  const int n = a.rows;
  const float sa = ldexpf(1.f, a.exp[m]) * (inv_scale ? inv_scale[m] : 1.f);
  const float inv_e = ldexpf(1.f, -kEExp);
  // M0 exponent from its exact bound: max|M0| <= amax_a * sa_scale / c^p
  const float bound_m = __uint_as_float(a.amax[m]) * (inv_scale ? inv_scale[m] : 1.f) * inv_cp;
  int em = 0;
  if (bound_m > 0.f && bound_m < 3.0e38f) { frexpf(bound_m, &em); em -= 15; }
  const float inv_m = ldexpf(1.f, -em);
  const __half* ah = mat_hi(a, m);
  __half* xh = mat_hi(x, m);
  __half* mh = mat_hi(mm, m);
  __half* ch = mat_hi(corr, m);
  float amax_m = 0.f, amax_c = 0.f;
  for_chunks8(n, a.ld, [&](int r, int c) {
    float av[8], xv[8], mv[8], cv[8];
    load_split8(ah, mat_plane(a), static_cast<long long>(r) * a.ld + c, sa, av);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool in = c + i < n;
      const float d = (r == c + i) ? 1.f : 0.f;
      mv[i] = in ? av[i] * inv_cp : 0.f;
      cv[i] = in ? (1.f + 1.f / p) * d - mv[i] / p : 0.f;
      xv[i] = d * inv_c;
      amax_m = nonneg_max(amax_m, fabsf(mv[i]));
      amax_c = nonneg_max(amax_c, fabsf(cv[i]));
    }
    store_split8(xh, mat_plane(x), static_cast<long long>(r) * x.ld + c, xv, inv_e);
    store_split8(mh, mat_plane(mm), static_cast<long long>(r) * mm.ld + c, mv, inv_m);
    store_split8(ch, mat_plane(corr), static_cast<long long>(r) * corr.ld + c, cv, inv_e);
  });
  amax_m = warp_max_nonneg(amax_m);
  amax_c = warp_max_nonneg(amax_c);
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(mm.amax + m, amax_m);
    atomic_max_nonneg(corr.amax + m, amax_c);
    atomic_max_nonneg(x.amax + m, inv_c);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    x.exp[m] = kEExp;
    mm.exp[m] = em;
    corr.exp[m] = kEExp;
  }
}

// Rewrite the correction factor of blocks that froze this iteration to I (roots.py:236 for k+1).
__global__ void reset_identity_kernel(dash_stack s, const int* __restrict__ flags) {
  const int m = blockIdx.y;
  if (!flags[m]) return;
  const int n = s.rows;
  __half* h = reinterpret_cast<__half*>(s.data) + static_cast<long long>(m) * 2 * n * s.ld;
  __half* l = h + static_cast<long long>(n) * s.ld;
  const float one = ldexpf(1.f, -kEExp);
  const long long total = static_cast<long long>(n) * n;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / n), c = static_cast<int>(i % n);
    const long long o = static_cast<long long>(r) * s.ld + c;
    h[o] = __float2half_rn(r == c ? one : 0.f);
    l[o] = __float2half_rn(0.f);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s.exp[m] = kEExp;
    s.amax[m] = __float_as_uint(1.f);
  }
}

// value * mult[m] -> fp32 (f_out, optional) and split (dst, optional).  Used for the root rescale
// roots * scale^(-1/p) (shampoo.py:348).
__global__ void scale_stack_kernel(dash_stack src, const float* __restrict__ mult, float pw, float* __restrict__ f_out,
                                   long long f_mat_stride, int f_ld, dash_stack dst, int has_dst,
                                   const int* __restrict__ gate) {
  if (gate && *gate == 0) return;  // the group failed its scale checks: keep the previous roots
  const int m = blockIdx.y;
  const int rows = src.rows, cols = src.cols;
  const float mu = mult ? (pw == 1.f ? mult[m] : static_cast<float>(pow(static_cast<double>(mult[m]), static_cast<double>(pw)))) : 1.f;
  const float sc = ldexpf(1.f, src.exp[m]) * mu;
  int e = 0;
  const float bound = __uint_as_float(src.amax[m]) * fabsf(mu);
  if (bound > 0.f && bound < 3.0e38f) { frexpf(bound, &e); e -= 15; }
  const float inv = ldexpf(1.f, -e);
  const __half* sh = mat_hi(src, m);
  __half* dh = has_dst ? mat_hi(dst, m) : nullptr;
  float amax = 0.f;
  for_chunks8(rows, src.ld, [&](int r, int c) {
    float v[8];
    load_split8(sh, mat_plane(src), static_cast<long long>(r) * src.ld + c, sc, v);
    if (f_out) {
      float* fo = f_out + m * f_mat_stride + static_cast<long long>(r) * f_ld + c;
      if (c + 8 <= cols && (f_ld & 3) == 0 && ((m * f_mat_stride) & 3) == 0) {
        reinterpret_cast<float4*>(fo)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4*>(fo)[1] = make_float4(v[4], v[5], v[6], v[7]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) if (c + i < cols) fo[i] = v[i];
      }
    }
    if (has_dst) {
      store_split8(dh, mat_plane(dst), static_cast<long long>(r) * dst.ld + c, v, inv);
#pragma unroll
      for (int i = 0; i < 8; ++i) amax = nonneg_max(amax, fabsf(v[i]));
    }
  });
  if (has_dst) {
    amax = warp_max_nonneg(amax);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(dst.amax + m, amax);
    if (blockIdx.x == 0 && threadIdx.x == 0) dst.exp[m] = e;
  }
}

// scale_stack of an upper pair-block stored source (the Newton-DB root as it leaves the solver): every 64 x 64
// destination tile stages its source tile in shared memory with 16-byte loads -- the tile itself on / above the
// block diagonal, the transposed upper tile below it -- so the completion pass (fill_lower) is fused away; the
// outputs are written as 8-column vectors like scale_stack_kernel, with the same arithmetic (bit-identical).
constexpr int kSuT = 64, kSuPad = 8;  // tile edge; padding of the staged rows (halves)
__global__ void __launch_bounds__(256) scale_stack_upper_kernel(dash_stack src, const float* __restrict__ mult,
                                                                float pw, float* __restrict__ f_out,
                                                                long long f_mat_stride, int f_ld, dash_stack dst,
                                                                int has_dst, const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  __shared__ __align__(16) __half th[kSuT][kSuT + kSuPad], tl[kSuT][kSuT + kSuPad];
  const int m = blockIdx.z;
  const int rows = src.rows, cols = src.cols;
  const int r0 = blockIdx.y * kSuT, c0 = blockIdx.x * kSuT;
  const bool lower = (r0 >> 8) > (c0 >> 8);
  const int sr0 = lower ? c0 : r0, sc0 = lower ? r0 : c0;  // source tile (upper storage)
  const float mu = mult ? (pw == 1.f ? mult[m] : static_cast<float>(pow(static_cast<double>(mult[m]), static_cast<double>(pw)))) : 1.f;
  const float sc = ldexpf(1.f, src.exp[m]) * mu;
  int e = 0;
  const float bound = __uint_as_float(src.amax[m]) * fabsf(mu);
  if (bound > 0.f && bound < 3.0e38f) { frexpf(bound, &e); e -= 15; }
  const float inv = ldexpf(1.f, -e);
  const __half* sh = mat_hi(src, m);
  const long long sp = mat_plane(src);
  // stage: 64 rows x 8 chunks of 8 halves per plane; src.ld is a multiple of 64, so chunks never straddle a row
  for (int t = threadIdx.x; t < kSuT * (kSuT / 8); t += blockDim.x) {
    const int i = t >> 3, c8 = (t & 7) * 8;
    const int r = sr0 + i;
    uint4 h = make_uint4(0, 0, 0, 0), l = h;
    if (r < rows && sc0 + c8 < src.ld) {
      const long long off = static_cast<long long>(r) * src.ld + sc0 + c8;
      h = __ldg(reinterpret_cast<const uint4*>(sh + off));
      l = __ldg(reinterpret_cast<const uint4*>(sh + sp + off));
    }
    *reinterpret_cast<uint4*>(&th[i][c8]) = h;
    *reinterpret_cast<uint4*>(&tl[i][c8]) = l;
  }
  __syncthreads();
  __half* dh = has_dst ? mat_hi(dst, m) : nullptr;
  const long long dp = has_dst ? mat_plane(dst) : 0;
  float amax = 0.f;
  for (int t = threadIdx.x; t < kSuT * (kSuT / 8); t += blockDim.x) {
    const int i = t >> 3, c8 = (t & 7) * 8;
    const int r = r0 + i, c = c0 + c8;
    if (r >= rows || c >= (has_dst ? dst.ld : cols)) continue;  // (padding columns of dst are written as zeros)
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const __half h = lower ? th[c8 + k][i] : th[i][c8 + k];
      const __half l = lower ? tl[c8 + k][i] : tl[i][c8 + k];
      v[k] = (c + k < cols) ? (__half2float(h) + __half2float(l)) * sc : 0.f;
    }
    if (f_out) {
      float* fo = f_out + m * f_mat_stride + static_cast<long long>(r) * f_ld + c;
      if (c + 8 <= cols && (f_ld & 3) == 0 && ((m * f_mat_stride) & 3) == 0) {
        reinterpret_cast<float4*>(fo)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4*>(fo)[1] = make_float4(v[4], v[5], v[6], v[7]);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) if (c + k < cols) fo[k] = v[k];
      }
    }
    if (has_dst && c < dst.ld) {
      store_split8(dh, dp, static_cast<long long>(r) * dst.ld + c, v, inv);
#pragma unroll
      for (int k = 0; k < 8; ++k) amax = nonneg_max(amax, fabsf(v[k]));
    }
  }
  if (has_dst) {
    amax = warp_max_nonneg(amax);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(dst.amax + m, amax);
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) dst.exp[m] = e;
  }
}

static dim3 egrid(const dash_stack& s) {
  long long el = static_cast<long long>(s.rows) * s.cols;
  long long b = (el + 255) / 256;
  b = std::min<long long>(std::max<long long>(b, 1), 64);
  return dim3(static_cast<unsigned>(b), static_cast<unsigned>(s.nmat));
}

static int cuda_ok() { return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_ECUDA; }

int scale_stack(const dash_stack& src, const float* mult, float pw, float* f_out, long long f_mat_stride, int f_ld,
                const dash_stack* dst, const int* gate, int src_upper, cudaStream_t st) {
  dash_stack d{};
  if (dst) {
    d = *dst;
    zero_amax(gate, d.nmat, d.amax, nullptr, nullptr, st);
  }
  if (src_upper && ndb_upper_storage()) {
    const dim3 grid((src.ld + kSuT - 1) / kSuT, (src.rows + kSuT - 1) / kSuT, src.nmat);
    scale_stack_upper_kernel<<<grid, 256, 0, st>>>(src, mult, pw, f_out, f_mat_stride, f_ld, d, dst ? 1 : 0, gate);
  } else {
    scale_stack_kernel<<<egrid(src), 256, 0, st>>>(src, mult, pw, f_out, f_mat_stride, f_ld, d, dst ? 1 : 0, gate);
  }
  note_launch();
  return cuda_ok();
}

// Scale checks of one group in reference order (shampoo.py:324-325, spectral.py:99-107), decided on the device:
// a collapsed pool (status 2) is a DegenerateSpectrumError (code 2), a non-positive or non-finite scale a
// ConvergenceError (code 1).  The first failing group records (code, group) in err[0..1]; ok[0] = 1 lets this
// group's roots be committed (gated rescale / final Clenshaw product) only while no group has failed so far,
// which is where the reference's refresh loop would have raised.
__global__ void scale_check_kernel(const float* __restrict__ scale, const int* __restrict__ status, int n, int group,
                                   int* __restrict__ ok, int* __restrict__ err) {
  __shared__ int code;
  if (threadIdx.x == 0) code = 0;
  __syncthreads();
  int c = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (status && status[i] == 2) c = max(c, 2);
    const float s = scale[i];
    if (!(s > 0.f) || !isfinite(s)) c = max(c, 1);
  }
  if (c) atomicMax(&code, c);
  __syncthreads();
  if (threadIdx.x == 0) {
    // the degenerate-spectrum check runs first in the reference (PI raises inside _group_scales)
    const int cc = code;
    const bool clean = err[0] == 0;
    if (clean && cc) {
      err[0] = cc;
      err[1] = group;
    }
    ok[0] = (clean && !cc) ? 1 : 0;
  }
}

int scale_check(const float* scale, const int* status, int n, int group, int* ok, int* err, cudaStream_t st) {
  scale_check_kernel<<<1, 256, 0, st>>>(scale, status, n, group, ok, err);
  note_launch();
  return cuda_ok();
}

// dst <- src when *par == want (device-decided: the host does not know how many gated iterations ran).
__global__ void copy_if_kernel(const int* par, int want, dash_stack dst, dash_stack src) {
  if (*par != want) return;
  const long long n16 = static_cast<long long>(src.nmat) * 2 * src.rows * src.ld / 8;  // uint4 = 8 halves
  const uint4* s = reinterpret_cast<const uint4*>(src.data);
  uint4* d = reinterpret_cast<uint4*>(dst.data);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n16;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    d[i] = s[i];
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < src.nmat; m += gridDim.x * blockDim.x) {
    dst.exp[m] = src.exp[m];
    dst.amax[m] = src.amax[m];
  }
}

static void copy_stack_if(const int* par, int want, const dash_stack& dst, const dash_stack& src, cudaStream_t st) {
  copy_if_kernel<<<1024, 256, 0, st>>>(par, want, dst, src);
  note_launch();
}

// Every solver operand is symmetric in exact arithmetic, so B could be loaded K-major (as its transpose):
// DASH_SYMB=1 does that.  Off by default: the 128x128 diagonal sub-blocks of the iterates are computed
// independently and are only symmetric to rounding, and on ill-conditioned blocks the Newton iterations
// amplify that difference (Y error 3.6e-6 -> 7.5e-5 at cond 1e3) for a 2.6% gain.  Making the diagonal
// sub-blocks exactly symmetric instead (upper copied onto lower in the epilogue) was tried and is worse: a
// cond-1e3 block then trips the divergence watch in tolerance mode (iteration 17, residual 6e-3).
static const int kSymB = getenv("DASH_SYMB") ? atoi(getenv("DASH_SYMB")) : 0;

// Upper pair-block storage of the Newton iterates (types.h): the iterates Y, Z, E are symmetric, so the
// launches store only the 256x256 pair blocks on/above the diagonal and read lower operand blocks transposed
// (K-block 64 launches only; DASH_NDB_UP=0 stores full matrices).  The solver's outputs are completed at the
// end by fill_lower_kernel.
bool ndb_upper_storage() {
  static const int on = getenv("DASH_NDB_UP") ? atoi(getenv("DASH_NDB_UP")) : 1;
  return on && gemm_kblock() == 64;
}
// passes = 4 (FULL64) launches run the K-block 32 kernel (gemm_launch), which reads operands complete
bool ndb_upper_storage(int passes) { return passes != 4 && ndb_upper_storage(); }

// Lower pair blocks of an upper-stored split stack <- transposes of the upper ones (both planes), through
// 32x32 shared-memory tiles (coalesced reads and writes).
__global__ void fill_lower_kernel(dash_stack s) {
  __shared__ uint16_t t[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;  // destination tile (lower pair block)
  if ((r0 >> 8) <= (c0 >> 8)) return;
  uint16_t* base = reinterpret_cast<uint16_t*>(s.data) + static_cast<size_t>(blockIdx.z) * s.rows * s.ld;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = c0 + i, c = r0 + static_cast<int>(threadIdx.x);
    t[i][threadIdx.x] = (r < s.rows && c < s.cols) ? base[static_cast<size_t>(r) * s.ld + c] : 0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + static_cast<int>(threadIdx.x);
    if (r < s.rows && c < s.cols) base[static_cast<size_t>(r) * s.ld + c] = t[threadIdx.x][i];
  }
}

int fill_lower(const dash_stack& s, cudaStream_t st) {
  if (!ndb_upper_storage()) return DASH_OK;  // the iterates were stored complete
  const dim3 grid((s.cols + 31) / 32, (s.rows + 31) / 32, 2 * s.nmat);
  fill_lower_kernel<<<grid, dim3(32, 8), 0, st>>>(s);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_ECUDA;
}

// ---------------------------------------------------------------------------- NDB
size_t ndb_ws_bytes(int n, int b) {  // NOLINT
  const size_t stacks = 3 * stack_bytes(n, b, b);
  const size_t jobs = 4 * JobBuilder::bytes_for(32, 2 * n) + 3 * JobBuilder::bytes_for(32, n);
  return stacks + jobs + state_bytes(n) + 4096;
}

// need: the outputs the caller reads (1 = y, 2 = z, 3 = both).  The last iteration computes only those (the
// optimizer reads Y of the first p = 4 chain and Z otherwise, shampoo.py:332-340): one product fewer per chain.
int ndb_solve(const dash_stack& a, const float* inv_scale, const dash_stack& y_out, const dash_stack& z_out,
              float tol, float stall, int max_iters, int passes, int* iters, float* resid_out, int* conv, void* ws,
              size_t ws_bytes, cudaStream_t st, int* products, bool complete, int need) {
  if (need < 1 || need > 3) return DASH_EINVAL;
  const int n = a.nmat;
  Arena ar(ws, ws_bytes);
  dash_stack e, y2, z2;
  if (!arena_stack(ar, a, &e) || !arena_stack(ar, a, &y2) || !arena_stack(ar, a, &z2)) return DASH_EINVAL;
  for (const dash_stack* t : std::initializer_list<const dash_stack*>{&e, &y2, &z2, &y_out, &z_out}) zero_padding(*t, st);
  BlockState s;
  if (!take_state(ar, n, &s)) return DASH_EINVAL;
  // ping-pong: (Y, Z) at even iterations live in (y_out, z_out), odd ones in (y2, z2)
  const dash_stack ys[2] = {y_out, y2};
  const dash_stack zs[2] = {z_out, z2};
  UploadedGemm g_first, g_e[2], g_yz[2], g_last[2];
  const int up = ndb_upper_storage(passes) ? 1 : 0;
  {
    JobBuilder jb;  // Y1 = (a E1) * inv_scale
    for (int m = 0; m < n; ++m) {
      GemmJob j;
      if (!jb.operands(j, a, m, 0, e, m, kSymB)) return DASH_EINVAL;
      j.op = EPI_SPLIT;
      j.out_mat = m;
      j.sym = 1;
      j.a_up = j.b_up = j.c_up = up;  // a may itself be upper-stored; E1 is
      j.alpha_p = inv_scale;
      jb.set_out(j, ys[1], m);
      jb.push(j);
    }
    if (!jb.upload(ar, st, &g_first)) return DASH_EINVAL;
  }
  for (int par = 0; par < 2; ++par) {
    const dash_stack& yc = ys[par];
    const dash_stack& zc = zs[par];
    const dash_stack& yn = ys[par ^ 1];
    const dash_stack& zn = zs[par ^ 1];
    JobBuilder je;  // E = 1.5 I - 0.5 Z Y   (E = I for frozen blocks)
    for (int m = 0; m < n; ++m) {
      GemmJob j;
      if (!je.operands(j, zc, m, 0, yc, m, kSymB)) return DASH_EINVAL;
      j.op = EPI_NDB_E;
      j.out_mat = m;
      j.sym = 1;
      j.a_up = j.b_up = j.c_up = up;
      j.active = s.active;
      j.resid = s.resid;
      je.set_out(j, e, m);
      je.push(j);
    }
    if (!je.upload(ar, st, &g_e[par])) return DASH_EINVAL;
    JobBuilder jy;  // Y' = Y E, Z' = E Z  (reference order, roots.py:288-289)
    for (int m = 0; m < n; ++m) {
      GemmJob j;
      if (!jy.operands(j, yc, m, 0, e, m, kSymB)) return DASH_EINVAL;
      j.op = EPI_SPLIT;
      j.out_mat = m;
      j.sym = 1;
      j.a_up = j.b_up = j.c_up = up;
      jy.set_out(j, yn, m);
      jy.push(j);
      if (!jy.operands(j, e, m, 0, zc, m, kSymB)) return DASH_EINVAL;
      j.op = EPI_SPLIT;
      j.out_mat = m;
      j.sym = 1;
      j.a_up = j.b_up = j.c_up = up;
      jy.set_out(j, zn, m);
      jy.push(j);
    }
    if (!jy.upload(ar, st, &g_yz[par])) return DASH_EINVAL;
    if (need != 3) {  // the last iteration: the read output only
      JobBuilder jl;
      for (int m = 0; m < n; ++m) {
        GemmJob j;
        if (need == 1 ? !jl.operands(j, yc, m, 0, e, m, kSymB) : !jl.operands(j, e, m, 0, zc, m, kSymB))
          return DASH_EINVAL;
        j.op = EPI_SPLIT;
        j.out_mat = m;
        j.sym = 1;
        j.a_up = j.b_up = j.c_up = up;
        jl.set_out(j, need == 1 ? yn : zn, m);
        jl.push(j);
      }
      if (!jl.upload(ar, st, &g_last[par])) return DASH_EINVAL;
    }
  }
  int np = 0;
  state_init_kernel<<<(n + 255) / 256, 256, 0, st>>>(s, n);
  note_launch();
  // ---- iteration 1 (closed form): E1, Z1 = E1 into (e, z2); Y1 = a_hat E1 into y2
  cudaMemsetAsync(e.amax, 0, sizeof(unsigned) * n, st);
  cudaMemsetAsync(z2.amax, 0, sizeof(unsigned) * n, st);
  cudaMemsetAsync(y2.amax, 0, sizeof(unsigned) * n, st);
  ndb_first_kernel<<<egrid(a), 256, 0, st>>>(a, inv_scale, e, z2, s.resid, up);
  note_launch();
  if (int rc = g_first.run(passes, st)) return rc;
  ++np;
  // each freeze also zeroes the amax arrays the next iteration's (gated) GEMMs fill: E and the Y / Z pair of
  // parity par ^ 1 (iteration k reads (Y, Z)[par] and writes (Y, Z)[par ^ 1])
  freeze_kernel<<<1, 1024, 0, st>>>(s, n, 1, tol, stall, 1, iters, resid_out, conv, nullptr, e.amax,
                                    ys[0].amax, zs[0].amax);
  note_launch();
  set_par_kernel<<<1, 1, 0, st>>>(s.par, 1);  // Y1, Z1 live in the scratch pair
  int par = 1;
  note_launch();
  for (int k = 2; k <= max_iters; ++k) {
    if (int rc = g_e[par].run(passes, st, s.n_active)) return rc;
    const bool last_only = k == max_iters && need != 3;
    if (int rc = (last_only ? g_last[par] : g_yz[par]).run(passes, st, s.n_active)) return rc;
    np += last_only ? 2 : 3;
    const bool more = k < max_iters;  // the next iteration writes (Y, Z)[par] (par flips below)
    freeze_kernel<<<1, 1024, 0, st>>>(s, n, k, tol, stall, 0, iters, resid_out, conv, nullptr,
                                      more ? e.amax : nullptr, more ? ys[par].amax : nullptr,
                                      more ? zs[par].amax : nullptr);
    note_launch();
    par ^= 1;
  }
  finish_kernel<<<(n + 255) / 256, 256, 0, st>>>(s, n, max_iters, iters, resid_out, conv);
  note_launch();
  if (need & 1) copy_stack_if(s.par, 1, y_out, y2, st);  // final iterate in the scratch pair -> outputs
  if (need & 2) copy_stack_if(s.par, 1, z_out, z2, st);
  if (up && complete) {  // (complete = false: the caller completes only the outputs it reads)
    if (need & 1) fill_lower(y_out, st);
    if (need & 2) fill_lower(z_out, st);
  }
  if (products) *products = np;
  return cuda_ok();
}

// ---------------------------------------------------------------------------- Coupled Newton
size_t cn_ws_bytes(int n, int b) {
  const size_t stacks = 6 * stack_bytes(n, b, b);
  const size_t jobs = 2 * (3 * JobBuilder::bytes_for(32, 2 * n)) + JobBuilder::bytes_for(32, n) * 2;
  return stacks + jobs + state_bytes(n) + Arena::need(4 * n) + 4096;
}

// X <- X C ; C2 = C C ; [C4 = C2 C2] ; M <- C^p M with residual max|M - I| and the next correction
// C = (1 + 1/p) I - M / p fused into the M epilogue (roots.py:235-242).
int cn_solve(const dash_stack& a, const float* inv_scale, int p, float c, const dash_stack& x_out, float tol,
             float stall, int max_iters, int passes, int* iters, float* resid_out, int* conv, void* ws, size_t ws_bytes,
             cudaStream_t st, int* products) {
  const int n = a.nmat;
  Arena ar(ws, ws_bytes);
  dash_stack x2, m1, m2, corr, cp;
  if (!arena_stack(ar, a, &x2) || !arena_stack(ar, a, &m1) || !arena_stack(ar, a, &m2) ||
      !arena_stack(ar, a, &corr) || !arena_stack(ar, a, &cp))
    return DASH_EINVAL;
  dash_stack c4 = cp;
  if (p == 4 && !arena_stack(ar, a, &c4)) return DASH_EINVAL;
  for (const dash_stack* t : std::initializer_list<const dash_stack*>{&x2, &m1, &m2, &corr, &cp, &c4, &x_out}) zero_padding(*t, st);
  BlockState s;
  if (!take_state(ar, n, &s)) return DASH_EINVAL;
  int* newly = ar.take_n<int>(n);
  if (!ar.ok) return DASH_EINVAL;
  const dash_stack xs[2] = {x_out, x2};
  const dash_stack ms[2] = {m1, m2};
  const int up = ndb_upper_storage(passes) ? 1 : 0;  // X, M, C are polynomials in a: upper pair-block storage
  UploadedGemm g_xc[2], g_c4, g_m[2];
  for (int par = 0; par < 2; ++par) {
    JobBuilder j1;  // X' = X C and C2 = C C in one launch
    for (int m = 0; m < n; ++m) {
      GemmJob j;
      if (!j1.operands(j, xs[par], m, 0, corr, m, kSymB)) return DASH_EINVAL;
      j.op = EPI_SPLIT; j.out_mat = m; j.sym = 1;
      j.a_up = j.b_up = j.c_up = up;
      j1.set_out(j, xs[par ^ 1], m);
      j1.push(j);
      if (!j1.operands(j, corr, m, 0, corr, m, kSymB)) return DASH_EINVAL;
      j.op = EPI_SPLIT; j.out_mat = m; j.sym = 1;
      j.a_up = j.b_up = j.c_up = up;
      j1.set_out(j, cp, m);
      j1.push(j);
    }
    if (!j1.upload(ar, st, &g_xc[par])) return DASH_EINVAL;
    JobBuilder j3;  // M' = C^p M, residual, next correction
    const dash_stack& cpow = (p == 4) ? c4 : cp;
    for (int m = 0; m < n; ++m) {
      GemmJob j;
      if (!j3.operands(j, cpow, m, 0, ms[par], m, kSymB)) return DASH_EINVAL;
      j.op = EPI_CN_M; j.out_mat = m; j.sym = 1;
      j.a_up = j.b_up = j.c_up = up;
      j.beta = static_cast<float>(p);
      j.active = s.active;
      j.resid = s.resid;
      j3.set_out(j, ms[par ^ 1], m);
      j3.set_out2(j, corr, m);
      j3.push(j);
    }
    if (!j3.upload(ar, st, &g_m[par])) return DASH_EINVAL;
  }
  if (p == 4) {
    JobBuilder j2;
    for (int m = 0; m < n; ++m) {
      GemmJob j;
      if (!j2.operands(j, cp, m, 0, cp, m, kSymB)) return DASH_EINVAL;
      j.op = EPI_SPLIT; j.out_mat = m; j.sym = 1;
      j.a_up = j.b_up = j.c_up = up;
      j2.set_out(j, c4, m);
      j2.push(j);
    }
    if (!j2.upload(ar, st, &g_c4)) return DASH_EINVAL;
  }
  state_init_kernel<<<(n + 255) / 256, 256, 0, st>>>(s, n);
  note_launch();
  cudaMemsetAsync(ms[0].amax, 0, sizeof(unsigned) * n, st);
  cudaMemsetAsync(corr.amax, 0, sizeof(unsigned) * n, st);
  cudaMemsetAsync(xs[0].amax, 0, sizeof(unsigned) * n, st);
  const float cpow_p = (p == 4) ? c * c * c * c : c * c;
  cn_first_kernel<<<egrid(a), 256, 0, st>>>(a, inv_scale, 1.f / c, 1.f / cpow_p, static_cast<float>(p), xs[0], ms[0],
                                            corr);
  note_launch();
  int par = 0, np = 0;
  for (int k = 1; k <= max_iters; ++k) {
    zero_amax(s.n_active, n, xs[par ^ 1].amax, cp.amax, nullptr, st);
    if (int rc = g_xc[par].run(passes, st, s.n_active)) return rc;
    if (p == 4) {
      zero_amax(s.n_active, n, c4.amax, nullptr, nullptr, st);
      if (int rc = g_c4.run(passes, st, s.n_active)) return rc;
    }
    zero_amax(s.n_active, n, ms[par ^ 1].amax, corr.amax, nullptr, st);
    if (int rc = g_m[par].run(passes, st, s.n_active)) return rc;
    np += (p == 4) ? 4 : 3;
    freeze_kernel<<<1, 1024, 0, st>>>(s, n, k, tol, stall, 0, iters, resid_out, conv, newly);
    note_launch();
    reset_identity_kernel<<<egrid(a), 256, 0, st>>>(corr, newly);
    note_launch();
    par ^= 1;
  }
  finish_kernel<<<(n + 255) / 256, 256, 0, st>>>(s, n, max_iters, iters, resid_out, conv);
  note_launch();
  copy_stack_if(s.par, 1, x_out, x2, st);
  if (up) fill_lower(x_out, st);
  if (products) *products = np;
  return cuda_ok();
}

// ---------------------------------------------------------------------------- Chebyshev / Clenshaw
// Optimized Clenshaw (chebyshev.py:156-184): S = 2 a/s - I, B_d = c_d I, B_{d-1} = 2 c_d S + c_{d-1} I,
// B_k = 2 S B_{k+1} - B_{k+2} + c_k I (k = d-2..1), out = (S B_1 - B_2 + c_0 I) * s^(-1/p).
__device__ __forceinline__ int exp_bound(float b) {
  if (!(b > 0.f) || !(b < 3.0e38f)) return 0;
  int x;
  frexpf(b, &x);
  return x - 15;
}

__global__ void cheb_first_kernel(dash_stack a, const float* __restrict__ inv_scale, float cd, float cd1,
                                  dash_stack s_out, dash_stack bd1, dash_stack bd) {
  const int m = blockIdx.y;
  const int n = a.rows;
  const float is = inv_scale ? inv_scale[m] : 1.f;
  const float sa = ldexpf(1.f, a.exp[m]) * is;
  const float bound_s = 2.f * __uint_as_float(a.amax[m]) * is + 1.f;
  const int es = exp_bound(bound_s), e1 = exp_bound(2.f * fabsf(cd) * bound_s + fabsf(cd1)),
            e0 = exp_bound(fabsf(cd) > 0.f ? fabsf(cd) : 1.f);
  const float inv_s = ldexpf(1.f, -es), inv_1 = ldexpf(1.f, -e1), inv_0 = ldexpf(1.f, -e0);
  const __half* ah = mat_hi(a, m);
  __half* sh = mat_hi(s_out, m);
  __half* h1 = mat_hi(bd1, m);
  __half* h0 = mat_hi(bd, m);
  float ms = 0.f, m1 = 0.f;
  for_chunks8(n, a.ld, [&](int r, int c) {
    float sv[8], b1[8], b0[8];
    load_split8(ah, mat_plane(a), static_cast<long long>(r) * a.ld + c, sa, sv);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool in = c + i < n;
      const float d = (r == c + i) ? 1.f : 0.f;
      sv[i] = in ? 2.f * sv[i] - d : 0.f;
      b1[i] = in ? 2.f * cd * sv[i] + cd1 * d : 0.f;
      b0[i] = cd * d;
      ms = nonneg_max(ms, fabsf(sv[i]));
      m1 = nonneg_max(m1, fabsf(b1[i]));
    }
    store_split8(sh, mat_plane(s_out), static_cast<long long>(r) * s_out.ld + c, sv, inv_s);
    store_split8(h1, mat_plane(bd1), static_cast<long long>(r) * bd1.ld + c, b1, inv_1);
    store_split8(h0, mat_plane(bd), static_cast<long long>(r) * bd.ld + c, b0, inv_0);
  });
  ms = warp_max_nonneg(ms);
  m1 = warp_max_nonneg(m1);
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(s_out.amax + m, ms);
    atomic_max_nonneg(bd1.amax + m, m1);
    atomic_max_nonneg(bd.amax + m, fabsf(cd));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s_out.exp[m] = es;
    bd1.exp[m] = e1;
    bd.exp[m] = e0;
  }
}

size_t cheb_ws_bytes(int n, int b) {
  return 4 * stack_bytes(n, b, b) + 4 * JobBuilder::bytes_for(32, n) + Arena::need(4 * 1024) + 4096;
}

__global__ void pick_scalar_kernel(float* dst, const float* src, int k) { *dst = src[k]; }


int cheb_solve(const dash_stack& a, const float* inv_scale, const float* mult, const double* coeffs, int degree,
               float* f_out, const dash_stack* out_split, int passes, const int* gate, void* ws, size_t ws_bytes,
               cudaStream_t st) {
  const int n = a.nmat;
  if (degree < 2 || degree > 1000) return DASH_EINVAL;
  Arena ar(ws, ws_bytes);
  dash_stack sm, bb[3];
  if (!arena_stack(ar, a, &sm) || !arena_stack(ar, a, &bb[0]) || !arena_stack(ar, a, &bb[1]) ||
      !arena_stack(ar, a, &bb[2]))
    return DASH_EINVAL;
  float* d_coef = ar.take_n<float>(degree + 2);  // [0..degree] coefficients, [degree+1] current c_k
  if (!ar.ok) return DASH_EINVAL;
  float* cur = d_coef + degree + 1;
  std::vector<float> hc(degree + 2, 0.f);
  for (int k = 0; k <= degree; ++k) hc[k] = static_cast<float>(coeffs[k]);
  cudaMemcpyAsync(d_coef, hc.data(), sizeof(float) * hc.size(), cudaMemcpyHostToDevice, st);
  for (const dash_stack* t : std::initializer_list<const dash_stack*>{&sm, &bb[0], &bb[1], &bb[2]}) zero_padding(*t, st);
  // rotation r holds the jobs for every k with k % 3 == r: B_k = 2 S B_{k+1} - B_{k+2} + c_k I.  The B_k are
  // polynomials in S, stored as upper pair blocks (the side input is read only at stored positions); the
  // final product reads B_1 that way and writes complete outputs.
  const int up = ndb_upper_storage(passes) ? 1 : 0;
  UploadedGemm g_rot[3], g_fin;
  for (int r = 0; r < 3; ++r) {
    JobBuilder jb;
    for (int m = 0; m < n; ++m) {
      GemmJob j;
      if (!jb.operands(j, sm, m, 0, bb[(r + 1) % 3], m, kSymB)) return DASH_EINVAL;
      j.op = EPI_CHEB;
      j.out_mat = m;
      j.sym = 1;
      j.b_up = j.c_up = up;
      j.gamma_p = cur;
      jb.set_side(j, bb[(r + 2) % 3], m);
      jb.set_out(j, bb[r], m);
      jb.push(j);
    }
    if (!jb.upload(ar, st, &g_rot[r])) return DASH_EINVAL;
  }
  {  // out = (S B_1 - B_2 + c_0 I) * mult
    JobBuilder jb;
    for (int m = 0; m < n; ++m) {
      GemmJob j;
      if (!jb.operands(j, sm, m, 0, bb[1], m, kSymB)) return DASH_EINVAL;
      j.op = EPI_CHEB_FINAL;
      j.out_mat = m;
      j.sym = 1;
      j.b_up = up;
      j.gamma = hc[0];
      j.alpha_p = mult;
      jb.set_side(j, bb[2], m);
      if (out_split) jb.set_out(j, *out_split, m);
      if (f_out) jb.set_fout(j, f_out, n, a.rows, a.rows, m);
      jb.push(j);
    }
    if (!jb.upload(ar, st, &g_fin)) return DASH_EINVAL;
  }
  for (int r = 0; r < 3; ++r) cudaMemsetAsync(bb[r].amax, 0, sizeof(unsigned) * n, st);
  cudaMemsetAsync(sm.amax, 0, sizeof(unsigned) * n, st);
  cheb_first_kernel<<<egrid(a), 256, 0, st>>>(a, inv_scale, hc[degree], hc[degree - 1], sm, bb[(degree - 1) % 3],
                                              bb[degree % 3]);
  note_launch();
  for (int k = degree - 2; k >= 1; --k) {
    pick_scalar_kernel<<<1, 1, 0, st>>>(cur, d_coef, k);
    note_launch();
    cudaMemsetAsync(bb[k % 3].amax, 0, sizeof(unsigned) * n, st);
    if (int rc = g_rot[k % 3].run(passes, st)) return rc;
  }
  if (out_split) zero_amax(gate, n, out_split->amax, nullptr, nullptr, st);
  if (int rc = g_fin.run(passes, st, gate)) return rc;  // the outputs are written only when *gate != 0
  return cuda_ok();
}

}  // namespace dash
