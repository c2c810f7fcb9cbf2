// Persistent grouped tcgen05 GEMM over split-f16 stacks with DASH epilogues (sm_100a).
//
// One CTA per SM, 6 warps:
//   warp 0      TMA producer   (elected lane): global -> smem ring of STAGES k-blocks
//   warp 1      MMA issuer     (elected lane): tcgen05.mma 128x256x16, fp32 accumulators in TMEM
//   warps 2..5  epilogue       tcgen05.ld -> fused DASH epilogue -> global (split fp16 / fp32)
// TMEM holds two 128x256 fp32 accumulators (512 columns) so the epilogue of tile t overlaps the
// MMAs of tile t+1.  With PASSES == 3 every k-block issues hi*hi + hi*lo + lo*hi (split-f16
// products: fp32-class accuracy at 1/3 of the fp16 tensor rate); PASSES == 1 issues hi*hi only.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "ptx.cuh"
#include "types.h"
#include "engine.h"

namespace dash {

// First global tile of a job in the NT-wide tiling (NT = 128: tile_start, NT = 256: tile_start2).
template <int NT>
__device__ __forceinline__ int job_tile_start(const GemmJob& j) {
  return NT == 128 ? j.tile_start : j.tile_start2;
}

template <int NT>
__device__ __forceinline__ int find_job(const GemmJob* __restrict__ jobs, int njobs, int tile, int uniform = 0) {
  if (uniform) return tile / uniform;  // every job has `uniform` tiles (stacked solver launches)
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(NT == 128 ? &jobs[mid].tile_start : &jobs[mid].tile_start2) <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ int exp_from_bound(float b) {
  if (!(b > 0.f) || !(b < 3.0e38f)) return 0;
  int x;
  frexpf(b, &x);
  return x - 15;  // b * 2^-e = m * 2^15 with m in [0.5, 1)
}

__device__ __forceinline__ float amax_of(const unsigned* p) {
  return p ? __uint_as_float(*p) : 0.f;
}

// Split a value (already scaled by 2^-e) into fp16 hi/lo.
__device__ __forceinline__ void split_scaled(float y, __half& h, __half& l) {
  h = __float2half_rn(y);
  l = __float2half_rn(y - __half2float(h));
}

// Store W (16 or 32) consecutive values of row r (cols c0..c0+W-1) as split fp16; masked variant for edges.
template <int W>
__device__ __forceinline__ void store_split(__half* hi, long long plane, int ld, int r, int c0, int M, int N,
                                            const float (&x)[W], float inv_scale, bool& overflow) {
  if (r >= M) return;
  __half* ph = hi + static_cast<long long>(r) * ld + c0;
  __half* pl = ph + plane;
  if (c0 + W <= N) {
    uint32_t hw[W / 2], lw[W / 2];
#pragma unroll
    for (int i = 0; i < W / 2; ++i) {
      __half h0, l0, h1, l1;
      split_scaled(x[2 * i] * inv_scale, h0, l0);
      split_scaled(x[2 * i + 1] * inv_scale, h1, l1);
      overflow |= __hisinf(h0) | __hisinf(h1) | __hisnan(h0) | __hisnan(h1);
      hw[i] = static_cast<uint32_t>(__half_as_ushort(h0)) | (static_cast<uint32_t>(__half_as_ushort(h1)) << 16);
      lw[i] = static_cast<uint32_t>(__half_as_ushort(l0)) | (static_cast<uint32_t>(__half_as_ushort(l1)) << 16);
    }
    uint4* dh = reinterpret_cast<uint4*>(ph);
    uint4* dl = reinterpret_cast<uint4*>(pl);
#pragma unroll
    for (int i = 0; i < W / 8; ++i) {
      dh[i] = make_uint4(hw[4 * i], hw[4 * i + 1], hw[4 * i + 2], hw[4 * i + 3]);
      dl[i] = make_uint4(lw[4 * i], lw[4 * i + 1], lw[4 * i + 2], lw[4 * i + 3]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) {
      if (c0 + i < N) {
        __half h, l;
        split_scaled(x[i] * inv_scale, h, l);
        overflow |= __hisinf(h) | __hisnan(h);
        ph[i] = h;
        pl[i] = l;
      }
    }
  }
}

// ============================================================================ CTA-pair kernel
// One thread-block cluster of 2 CTAs (a TPC pair) computes a 256 x 128 output tile with
// tcgen05.mma.cta_group::2 (M = 256, N = 128, K = 16 per instruction): each CTA stages its 128 rows of A
// and its 64 rows of B (N/2) per k-block; the leader CTA issues the MMAs; each CTA's TMEM receives its
// 128 output rows.
//
// TMEM = 4 slots of 128 fp32 columns, each with its own full/empty barrier pair.  tcgen05 accumulation
// truncates, so its error grows linearly with the number of MMAs summed into one accumulator
// (profiles/r1_accumulation_error.log): a tile with nacc accumulators sends k-blocks
// [c*per, (c+1)*per) to slot c (per = ceil(nk / nacc)) and the epilogue sums the partials in fp32.
// Because each slot is committed as soon as its K range is done, the epilogue drains slot 0 while the
// MMAs of slots 1..3 still run, and the next tile only waits for the slot it starts in -- the TMEM read
// overlaps the tensor work instead of stalling it.  nacc = 1 (fp16 mode) keeps 4 tiles in flight.
//
// Symmetric jobs (jb.sym, C = C^T in exact arithmetic: every Newton / Chebyshev iterate is a polynomial
// in the block) run only the tiles on or above the block diagonal; the epilogue stores each strictly-upper
// 128 x 128 sub-block twice (direct and transposed) and drops the one below-diagonal sub-block of each
// diagonal tile, so every output element has exactly one writer (deterministic).
constexpr int kPairM = kTileM, kHalf = kTileM / 2;
constexpr int kNaccDefault = 4;   // split-f16 accumulation (env DASH_NACC): 1 = one accumulator, 2 = main +
                                   // correction, 4 / 8 / 16 = ring of that many K ranges per tile (4: the
                                   // EMULATED32 default, as fast as 2 and ~4x more accurate; 16: FULL64)
constexpr int kEpiWarps = 8;     // 2 per TMEM lane quarter, 64 columns each
constexpr int kSlots = 4;         // TMEM accumulator slots (4 x 128 columns = all 512)
constexpr int kRing = 8;          // tile-index ring shared by the pair (dynamic scheduling)
constexpr int kPrefetch = 4;      // k-blocks prefetched into L2 ahead of the producer
constexpr int kRingConsumers = 2 + 2 * 8;  // leader MMA + peer producer + epilogue warps of both CTAs
constexpr int kThreads2 = 64 + 32 * kEpiWarps;

// KB = K-block (64: 128-byte swizzled K rows; 32: 64-byte swizzle, twice the stages in the same shared memory
// -> more bytes in flight per unit of MMA time, i.e. more tolerance to HBM/L2 latency).
// NT = pair tile width (128 or 256).  A 256 x 256 pair tile halves the shared-memory bytes per flop (the
// 256 x 128 tile needs ~156 B/clk of the 128 B/clk an SM's shared memory delivers for split products) at the
// price of one accumulator per tile (2 TMEM sets of 256 columns), so it serves fp16 launches and split
// launches that accept single-accumulator error.
#ifndef DASH_P3_STAGES  // experiment overrides (build-time)
#define DASH_P3_STAGES 3
#endif
#ifndef DASH_EPI_WARP_BYTES
#define DASH_EPI_WARP_BYTES 8192
#endif
template <int PASSES, int KB, int NT = 128>
struct Gemm2Cfg {
  static constexpr int kPlanes = PASSES == 3 ? 2 : 1;
  static constexpr int kABytes = kHalf * KB * 2;         // 16 / 8 KB per plane (128 rows of A)
  static constexpr int kBBytes = (NT / 2) * KB * 2;      // 8 / 4 KB per plane per 64 rows of B (NT / 2 rows)
  static constexpr int kStageBytes = (kABytes + kBBytes) * kPlanes;
  static constexpr int kEpiBytes = kEpiWarps * DASH_EPI_WARP_BYTES;  // per epilogue warp: 32 x 64 split tile (2 planes)
  // NT = 256: as many stages as the 227 KB of shared memory holds
  static constexpr int kStages = NT == 128 ? (PASSES == 3 ? DASH_P3_STAGES : 6) * (64 / KB)
                                           : ((232448 - kEpiBytes - 1024 - 512) / kStageBytes < 10
                                                  ? (232448 - kEpiBytes - 1024 - 512) / kStageBytes : 10);
  static constexpr int kSmemBytes = kStages * kStageBytes + kEpiBytes + 1024 + 512;
  static_assert(kSmemBytes <= 232448, "shared memory per CTA");
  static_assert((2 * kStages + 2 * kSlots + kEpiWarps + 2 * kRing) * 8 + kRing * 4 + 4 <= 512, "barrier block");
};

// Upper pair-block storage: is the k-block (256-block kp) of an operand whose 256-row/col block is `blk` a
// lower block?  K-major operands are stored (rows = blk, cols = k); MN-major ones (rows = k, cols = blk).
__device__ __forceinline__ bool upper_flip(int mn, int blk, int kp) { return mn ? kp > blk : blk > kp; }

// Tile `local` of a job -> (256-row tile ti, NT-column tile tj).  Symmetric jobs enumerate, per row tile
// I, only the column tiles that reach the diagonal: J >= 2I (NT = 128) or J >= I (NT = 256).
template <int NT>
__device__ __forceinline__ void tile_coords(const GemmJob& jb, int local, int& ti, int& tj) {
  constexpr int step = 256 / NT;
  const int tn = NT == 128 ? jb.tiles_n : jb.tiles_n2;
  if (!jb.sym) {
    ti = local / tn;
    tj = local - ti * tn;
    return;
  }
  int i = 0, row = tn;
  while (local >= row) {
    local -= row;
    ++i;
    row -= step;
  }
  ti = i;
  tj = step * i + local;
}

// Transposed store of 32 values of row r (cols c0..c0+31) into rows c0.. of column r (symmetric mirror).
template <int W>
__device__ __forceinline__ void store_split_T(__half* hi, long long plane, int ld, int r, int c0, int N,
                                              const float (&x)[W], float inv_scale) {
#pragma unroll
  for (int i = 0; i < W; ++i) {
    if (c0 + i < N) {
      __half h, l;
      split_scaled(x[i] * inv_scale, h, l);
      __half* ph = hi + static_cast<long long>(c0 + i) * ld + r;
      ph[0] = h;
      ph[plane] = l;
    }
  }
}

struct EpiCtx {
  int op, mat, r, M, N;
  bool inactive, row_ok, store, mirror;
  float sc, mul, gam, inv_out, inv_e, side_scale, cn_a, cn_b;
  float amax, amax2, resid;
  double sumsq;
  bool ovf, ovf2;
  const uint8_t* sbuf;  // side input tile staged in shared memory by TMA (direct swizzled layout) or null
  const uint8_t* fbuf;  // EPI_EMA: fp32 input tile staged by TMA ([2][32 rows][32 floats], swizzled) or null
  bool f_tma;           // fp32 output goes through the staged bulk store (skip direct stores)
  int lane, lc0;        // lane (= row within the warp tile) and first column of the warp tile
};

// fp32 tile staging: [half][32 rows][32 floats], 128-byte swizzle (two {32, 32, 1} boxes per 64-column tile).
__device__ __forceinline__ int f32_off(int lane, int col) {  // col in [0, 64)
  const int h = col >> 5, w = col & 31;
  return h * 4096 + lane * 128 + (((w >> 2) ^ (lane & 7)) << 4) + (w & 3) * 4;
}

template <int W>
__device__ __forceinline__ void put_split(const EpiCtx& cx, __half* hi, long long plane, int ld, int c0,
                                          const float (&x)[W], float inv, bool& ovf) {
  if (!cx.store) return;
  store_split<W>(hi, plane, ld, cx.r, c0, cx.M, cx.N, x, inv, ovf);
  if (cx.mirror && cx.r < cx.M) store_split_T<W>(hi, plane, ld, cx.r, c0, cx.N, x, inv);
}

template <int W>
__device__ __forceinline__ void put_f32(const EpiCtx& cx, float* f, int ld, int c0, const float (&x)[W]) {
  if (!cx.store || cx.r >= cx.M) return;
  float* fo = f + static_cast<long long>(cx.r) * ld + c0;
#pragma unroll
  for (int i = 0; i < W; ++i) if (c0 + i < cx.N) fo[i] = x[i];
  if (cx.mirror) {
#pragma unroll
    for (int i = 0; i < W; ++i) if (c0 + i < cx.N) f[static_cast<long long>(c0 + i) * ld + cx.r] = x[i];
  }
}

// Apply the fused DASH epilogue to W consecutive columns c0.. of row cx.r (x holds the fp32 product).
template <int W>
__device__ __forceinline__ void epi_piece(const GemmJob& jb, EpiCtx& cx, int c0, float (&x)[W], bool split_now) {
  const int r = cx.r;
  switch (cx.op) {
    case EPI_SPLIT: {
#pragma unroll
      for (int i = 0; i < W; ++i) {
        x[i] *= cx.sc * cx.mul;
        if (cx.row_ok && c0 + i < cx.N) cx.amax = nonneg_max(cx.amax, fabsf(x[i]));
      }
      if (jb.c_hi && split_now) put_split<W>(cx, jb.c_hi, jb.c_plane, jb.c_ld, c0, x, cx.inv_out, cx.ovf);
      if (jb.f_out && !cx.f_tma) put_f32<W>(cx, jb.f_out, jb.f_ld, c0, x);
    } break;
    case EPI_NDB_E: {
#pragma unroll
      for (int i = 0; i < W; ++i) {
        const float d = (r == c0 + i) ? 1.f : 0.f;
        float e = 1.5f * d - 0.5f * (x[i] * cx.sc);
        if (cx.inactive) e = d;
        x[i] = e;
        if (cx.row_ok && c0 + i < cx.N) {
          cx.resid = nonneg_max(cx.resid, fabsf(e - d));
          cx.amax = nonneg_max(cx.amax, fabsf(e));
        }
      }
      if (split_now) put_split<W>(cx, jb.c_hi, jb.c_plane, jb.c_ld, c0, x, cx.inv_out, cx.ovf);
    } break;
    case EPI_EMA: {  // never symmetric (host); fp32 read-modify-write
      const float b = jb.beta, omb = 1.f - jb.beta;
      if (cx.fbuf) {   // staged input; the output is staged + bulk-stored by the caller (values stay in x)
#pragma unroll
        for (int i4 = 0; i4 < W / 4; ++i4) {
          const float4 fi = *reinterpret_cast<const float4*>(cx.fbuf + f32_off(cx.lane, c0 - cx.lc0 + 4 * i4));
          x[4 * i4] = b * fi.x + omb * (x[4 * i4] * cx.sc);
          x[4 * i4 + 1] = b * fi.y + omb * (x[4 * i4 + 1] * cx.sc);
          x[4 * i4 + 2] = b * fi.z + omb * (x[4 * i4 + 2] * cx.sc);
          x[4 * i4 + 3] = b * fi.w + omb * (x[4 * i4 + 3] * cx.sc);
        }
      } else if (cx.row_ok) {
        const float* fi = jb.f_in + static_cast<long long>(r) * jb.f_ld + c0;
        float* fo = jb.f_out + static_cast<long long>(r) * jb.f_ld + c0;
#pragma unroll
        for (int i = 0; i < W; ++i)
          if (c0 + i < cx.N) fo[i] = b * fi[i] + omb * (x[i] * cx.sc);
      }
    } break;
    case EPI_APPLY: {  // never symmetric (host)
#pragma unroll
      for (int i = 0; i < W; ++i) x[i] *= cx.sc;
      if (cx.row_ok) {
        float* fo = jb.f_out + static_cast<long long>(r) * jb.f_ld + c0;
#pragma unroll
        for (int i = 0; i < W; ++i)
          if (c0 + i < cx.N) {
            const float u = x[i];
            if (!cx.f_tma) fo[i] = u;
            cx.sumsq += static_cast<double>(u) * u;
          }
      }
    } break;
    case EPI_CHEB:
    case EPI_CHEB_FINAL: {
      const bool fin = cx.op == EPI_CHEB_FINAL;
      if (!fin && cx.sbuf && cx.row_ok && c0 + W <= cx.N) {
        // full piece, staged side input: paired conversions, fused 2 (x sc) - s (exact scalings, one rounding,
        // the same value as the general path), the diagonal term only where the diagonal crosses the piece
        const float ss = cx.side_scale, s2 = 2.f * cx.sc;
#pragma unroll
        for (int c8 = 0; c8 < W / 8; ++c8) {
          const int ch = (c0 - cx.lc0) / 8 + c8;
          const int off = cx.lane * 128 + ((ch ^ (cx.lane & 7)) << 4);
          const uint4 h = *reinterpret_cast<const uint4*>(cx.sbuf + off);
          const uint4 l = *reinterpret_cast<const uint4*>(cx.sbuf + 4096 + off);
          const uint32_t hw[4] = {h.x, h.y, h.z, h.w}, lw[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) {
            const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&hw[e2]));
            const float2 lf = __half22float2(*reinterpret_cast<const __half2*>(&lw[e2]));
            const int i = 8 * c8 + 2 * e2;
            x[i] = fmaf(x[i], s2, -fmaf(hf.x, ss, lf.x * ss));
            x[i + 1] = fmaf(x[i + 1], s2, -fmaf(hf.y, ss, lf.y * ss));
          }
        }
        const int di = r - c0;
        if (static_cast<unsigned>(di) < static_cast<unsigned>(W)) {
#pragma unroll
          for (int i = 0; i < W; ++i)
            if (i == di) x[i] += cx.gam;
        }
#pragma unroll
        for (int i = 0; i < W; ++i) cx.amax = nonneg_max(cx.amax, fabsf(x[i]));
        if (jb.c_hi && split_now) put_split<W>(cx, jb.c_hi, jb.c_plane, jb.c_ld, c0, x, cx.inv_out, cx.ovf);
        break;
      }
      __half svh[W], svl[W];
      if (cx.sbuf) {  // W consecutive columns = W / 8 swizzled 16-byte chunks of this lane's row
#pragma unroll
        for (int c8 = 0; c8 < W / 8; ++c8) {
          const int ch = (c0 - cx.lc0) / 8 + c8;
          const int off = cx.lane * 128 + ((ch ^ (cx.lane & 7)) << 4);
          const uint4 h = *reinterpret_cast<const uint4*>(cx.sbuf + off);
          const uint4 l = *reinterpret_cast<const uint4*>(cx.sbuf + 4096 + off);
          const __half* hp = reinterpret_cast<const __half*>(&h);
          const __half* lp = reinterpret_cast<const __half*>(&l);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            svh[8 * c8 + e] = hp[e];
            svl[8 * c8 + e] = lp[e];
          }
        }
      } else {
        const __half* sh = jb.s_hi + static_cast<long long>(r) * jb.s_ld + c0;
        const __half* sl = sh + jb.s_plane;
#pragma unroll
        for (int i = 0; i < W; ++i) {
          const bool ok = cx.row_ok && c0 + i < cx.N;
          svh[i] = ok ? sh[i] : __float2half(0.f);
          svl[i] = ok ? sl[i] : __float2half(0.f);
        }
      }
#pragma unroll
      for (int i = 0; i < W; ++i) {
        float sv = 0.f;
        if (cx.row_ok && c0 + i < cx.N) sv = (__half2float(svh[i]) + __half2float(svl[i])) * cx.side_scale;
        const float d = (r == c0 + i) ? cx.gam : 0.f;
        const float y = fin ? (x[i] * cx.sc - sv + d) * cx.mul : 2.f * (x[i] * cx.sc) - sv + d;
        x[i] = y;
        if (cx.row_ok && c0 + i < cx.N) cx.amax = nonneg_max(cx.amax, fabsf(y));
      }
      if (jb.c_hi && split_now) put_split<W>(cx, jb.c_hi, jb.c_plane, jb.c_ld, c0, x, cx.inv_out, cx.ovf);
      if (jb.f_out && !cx.f_tma) put_f32<W>(cx, jb.f_out, jb.f_ld, c0, x);
    } break;
    case EPI_CN_M: {
      float cc[W];
#pragma unroll
      for (int i = 0; i < W; ++i) {
        const float d = (r == c0 + i) ? 1.f : 0.f;
        const float m = x[i] * cx.sc;
        x[i] = m;
        float c = cx.cn_a * d - cx.cn_b * m;
        if (cx.inactive) c = d;
        cc[i] = c;
        if (cx.row_ok && c0 + i < cx.N) {
          cx.resid = nonneg_max(cx.resid, fabsf(m - d));
          cx.amax = nonneg_max(cx.amax, fabsf(m));
          cx.amax2 = nonneg_max(cx.amax2, fabsf(c));
        }
      }
      if (split_now) {
        put_split<W>(cx, jb.c_hi, jb.c_plane, jb.c_ld, c0, x, cx.inv_out, cx.ovf);
        put_split<W>(cx, jb.c2_hi, jb.c2_plane, jb.c_ld, c0, cc, cx.inv_e, cx.ovf2);
      }
    } break;
    default: break;
  }
}

// ---- SMEM-staged split stores (bulk tensor store per epilogue warp: 32 rows x 64 columns x 2 planes)
// Direct layout: [plane][32 rows][128 B], 128-byte swizzle (16-byte chunk ch of row r at chunk ch ^ (r & 7)),
// matching a {64, 32, 2, 1} tensor map with CU_TENSOR_MAP_SWIZZLE_128B.  f(v, col) gives the stored value.
template <class F>
__device__ __forceinline__ void stage_direct(uint8_t* buf, const float (&acc)[64], int lane, int c0, float inv,
                                             F f, bool& ovf) {
#pragma unroll
  for (int ch = 0; ch < 8; ++ch) {
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      // paired round-to-nearest conversions (bitwise the scalar split): hi = rn(y), lo = rn(y - hi); the hi
      // half overflows (inf) or is NaN exactly when !(|y| < 65520)
      const float y0 = f(acc[8 * ch + 2 * i], c0 + 8 * ch + 2 * i) * inv;
      const float y1 = f(acc[8 * ch + 2 * i + 1], c0 + 8 * ch + 2 * i + 1) * inv;
      const __half2 h = __floats2half2_rn(y0, y1);
      const float2 hf = __half22float2(h);
      const __half2 l = __floats2half2_rn(y0 - hf.x, y1 - hf.y);
      ovf |= !(fabsf(y0) < 65520.f) | !(fabsf(y1) < 65520.f);
      hw[i] = *reinterpret_cast<const uint32_t*>(&h);
      lw[i] = *reinterpret_cast<const uint32_t*>(&l);
    }
    const int off = lane * 128 + ((ch ^ (lane & 7)) << 4);
    *reinterpret_cast<uint4*>(buf + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(buf + 4096 + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
}

// Transposed layout: [plane][64 rows (= columns c0..c0+63)][32 columns (= this warp's rows) x 2 B], no swizzle,
// matching a {32, 64, 2, 1} tensor map.  Built from the direct layout already in `buf` (after its bulk store
// has read it): every lane reloads its own row, then writes it as a column -- one contiguous 64-byte row of
// the transposed tile per column and warp.
__device__ __forceinline__ void stage_transpose_in_place(uint8_t* buf, int lane) {
  uint32_t hv[32], lv[32];
#pragma unroll
  for (int ch = 0; ch < 8; ++ch) {
    const int off = lane * 128 + ((ch ^ (lane & 7)) << 4);
    const uint4 h = *reinterpret_cast<const uint4*>(buf + off);
    const uint4 l = *reinterpret_cast<const uint4*>(buf + 4096 + off);
    hv[4 * ch] = h.x; hv[4 * ch + 1] = h.y; hv[4 * ch + 2] = h.z; hv[4 * ch + 3] = h.w;
    lv[4 * ch] = l.x; lv[4 * ch + 1] = l.y; lv[4 * ch + 2] = l.z; lv[4 * ch + 3] = l.w;
  }
  __syncwarp();
  uint16_t* bh = reinterpret_cast<uint16_t*>(buf) + lane;
#pragma unroll
  for (int j = 0; j < 64; ++j) {
    const int sh = (j & 1) * 16;
    bh[j * 32] = static_cast<uint16_t>(hv[j >> 1] >> sh);
    bh[2048 + j * 32] = static_cast<uint16_t>(lv[j >> 1] >> sh);
  }
}

// Mirror of a staged 32 x 64 split tile written straight to global memory (DASH_EXP knob 32): every lane
// reloads its own row from the staged buffer (read-only, concurrent with the tile's bulk store), lane pairs
// swap one packed (hi, lo) element per column pair, each lane stores two 4-byte words of the transposed tile.
__device__ __forceinline__ void store_mirror_from_stage(const uint8_t* buf, __half* c_hi, long long plane, int ld,
                                                        int r0, int c0, int N, int lane) {
  uint32_t hv[32], lv[32];
#pragma unroll
  for (int ch = 0; ch < 8; ++ch) {
    const int off = lane * 128 + ((ch ^ (lane & 7)) << 4);
    const uint4 h = *reinterpret_cast<const uint4*>(buf + off);
    const uint4 l = *reinterpret_cast<const uint4*>(buf + 4096 + off);
    hv[4 * ch] = h.x; hv[4 * ch + 1] = h.y; hv[4 * ch + 2] = h.z; hv[4 * ch + 3] = h.w;
    lv[4 * ch] = l.x; lv[4 * ch + 1] = l.y; lv[4 * ch + 2] = l.z; lv[4 * ch + 3] = l.w;
  }
  const bool even = (lane & 1) == 0;
  uint16_t* base = reinterpret_cast<uint16_t*>(c_hi);
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const uint32_t e0 = __byte_perm(hv[j], lv[j], 0x5410), e1 = __byte_perm(hv[j], lv[j], 0x7632);
    const uint32_t recv = __shfl_xor_sync(0xffffffffu, even ? e1 : e0, 1);
    const int col = c0 + 2 * j + (even ? 0 : 1);
    const int row = r0 + (lane & ~1);
    const uint32_t lo_e = even ? e0 : recv, hi_e = even ? recv : e1;
    const uint32_t wh = __byte_perm(lo_e, hi_e, 0x5410), wl = __byte_perm(lo_e, hi_e, 0x7632);
    if (col < N) {
      uint16_t* p = base + static_cast<long long>(col) * ld + row;
      *reinterpret_cast<uint32_t*>(p) = wh;
      *reinterpret_cast<uint32_t*>(p + plane) = wl;
    }
  }
}

__device__ __forceinline__ void stage_direct_f32(uint8_t* buf, const float (&acc)[64], int lane) {
#pragma unroll
  for (int c4 = 0; c4 < 16; ++c4)
    *reinterpret_cast<float4*>(buf + f32_off(lane, 4 * c4)) =
        make_float4(acc[4 * c4], acc[4 * c4 + 1], acc[4 * c4 + 2], acc[4 * c4 + 3]);
}

// Transposed fp32 tile [64 rows (= columns)][32 floats (= this warp's rows)], no swizzle ({32, 64, 1} box).
__device__ __forceinline__ void stage_transposed_f32(uint8_t* buf, const float (&acc)[64], int lane) {
  float* b = reinterpret_cast<float*>(buf) + lane;
#pragma unroll
  for (int j = 0; j < 64; ++j) b[j * 32] = acc[j];
}

template <int PASSES, int KB, int NT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    dash_gemm2_kernel(const GemmJob* __restrict__ jobs, int njobs, int total_tiles,
                      const CUtensorMap* __restrict__ maps, const int* __restrict__ gate, int nacc_in, int uniform,
                      int* __restrict__ tile_counter, unsigned long long* __restrict__ prof) {
  // prof (DASH_GEMM_DEBUG & 2, diagnostics): clock64 cycles per role spent waiting on each barrier kind:
  // [0] producer on empty, [1] MMA on tempty, [2] MMA on full, [3] epilogue on tfull, [4] epilogue on
  // bulk-store reads, [5] producer total, [6] MMA total, [7] epilogue total (summed over warps)
  unsigned long long pw0 = 0, pw1 = 0;
  const long long t_start = clock64();
  using C = Gemm2Cfg<PASSES, KB, NT>;
  constexpr int kPN = NT;                    // pair tile columns = TMEM columns per accumulator slot
  constexpr int kRounds = NT / 128;          // epilogue passes over a tile (128 columns each)
  constexpr uint32_t kSl = 512 / NT;         // TMEM slots
  const int nacc_req = NT == 128 ? (nacc_in & 0xff) : 1;
  // ring mode (split products, nacc_req = R >= 4): the K loop of a tile is cut into R ranges ("units"); unit u of
  // the launch accumulates in TMEM slot u % 4 and the epilogue adds it into registers (fp32, round to nearest)
  // and releases the slot, so each truncating tensor-core accumulation chain is K / R long while the four slots
  // keep the MMA running ahead of the epilogue
  const bool ring = PASSES == 3 && nacc_req >= 4;
  const int nring = ring ? nacc_req : 0;
  const int nacc = ring ? static_cast<int>(kSl) : nacc_req;  // accumulators per tile (1, 2 or 4; 1 for NT = 256)
  const bool mc = PASSES == 3 && nacc == 2;  // main (hi*hi) + correction (hi*lo + lo*hi) accumulators
  const bool mc4 = PASSES == 3 && nacc == 4 && !ring;  // three K-range main accumulators + correction
  const int xp = nacc_in >> 8;  // DASH_EXP knobs: timing 1 hi planes only, 2 no epilogue, 4 no staging, 8 no bulk stores, 16 L2 prefetch; 32 mirror via global stores (valid, 2-3% slower); 64 / 128 plain (unhinted) split stores / operand loads; 256 no side-input load
  const uint32_t nsets = kSl / nacc;         // tiles in flight in TMEM

  if (gate && *gate == 0) return;  // uniform across the grid (and thus across each pair)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes + C::kEpiBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + kSlots;
  uint64_t* sbar = tempty + kSlots;  // per epilogue warp: side-input TMA load
  uint64_t* tq_full = sbar + kEpiWarps;   // tile ring: index published (both CTAs' copies)
  uint64_t* tq_empty = tq_full + kRing;   // tile ring: every consumer read it (leader's copy used)
  int* tile_ring = reinterpret_cast<int*>(tq_empty + kRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tile_ring + kRing);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();  // 0 = leader (issues the pair MMAs)

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);   // leader's arrive_expect_tx (both CTAs' TMA bytes land here)
      mbar_init(&empty[s], 1);  // pair-MMA commit (multicast to both CTAs)
    }
    for (int a = 0; a < kSlots; ++a) {
      mbar_init(&tfull[a], 1);                // pair-MMA commit (multicast)
      mbar_init(&tempty[a], 2 * kEpiWarps);   // every epilogue warp of both CTAs (leader's copy used)
    }
    for (int w = 0; w < kEpiWarps; ++w) mbar_init(&sbar[w], 1);
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&tq_full[i], 1);
      mbar_init(&tq_empty[i], kRingConsumers);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc2<512>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Dynamic tile scheduling: the leader's producer draws tiles from a global atomic counter (the pairs stay
  // within a few tiles of each other, so every matrix's operands are read from HBM about once and reused
  // from L2) and publishes them through a ring in both CTAs; -1 ends the stream.
  const uint32_t leader_tq_empty = mapa_shared(smem_u32(tq_empty), 0);
  auto next_tile = [&](uint32_t i) -> int {  // consumer side (one thread)
    const uint32_t slot = i % kRing;
    mbar_wait_cluster(&tq_full[slot], (i / kRing) & 1u);
    const int tile = ld_acquire_shared(&tile_ring[slot]);  // completes before the (relaxed) release of the slot
    mbar_arrive_remote_relaxed(leader_tq_empty + slot * 8);
    return tile;
  };

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer (both CTAs)
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t peer_ring = mapa_shared(smem_u32(tile_ring), 1);
      const uint32_t peer_full = mapa_shared(smem_u32(tq_full), 1);
      const uint64_t pol_load = l2_policy_evict_last();
      for (uint32_t it = 0;; ++it) {
        int tile;
        if (rank == 0) {
          const uint32_t slot = it % kRing;
          mbar_wait_cluster(&tq_empty[slot], ((it / kRing) & 1u) ^ 1u);
          tile = atomicAdd(tile_counter, 1);
          if (tile >= total_tiles) {
            tile = -1;
            // the last pair to run dry re-arms the counters for the next launch on this stream
            if (atomicAdd(tile_counter + 1, 1) == static_cast<int>(gridDim.x / 2) - 1) {
              tile_counter[0] = 0;
              tile_counter[1] = 0;
              __threadfence();
            }
          }
          tile_ring[slot] = tile;
          st_cluster_u32(peer_ring + slot * 4, static_cast<uint32_t>(tile));
          mbar_arrive(&tq_full[slot]);
          mbar_arrive_remote(peer_full + slot * 8);
        } else {
          tile = next_tile(it);
        }
        if (tile < 0) break;
        const GemmJob& jb = jobs[find_job<NT>(jobs, njobs, tile, uniform)];
        int ti, tj;
        tile_coords<NT>(jb, tile - job_tile_start<NT>(jb), ti, tj);
        const int am = ti * kPairM + kHalf * static_cast<int>(rank);
        const int bn = tj * kPN + (kPN / 2) * static_cast<int>(rank);
        const int nk = (jb.K + KB - 1) / KB;
        const CUtensorMap* amap = maps + (KB == 64 ? jb.a_map : jb.a_map32);
        const CUtensorMap* bmap = maps + (KB == 64 ? jb.b_map : jb.b_map32);
        const CUtensorMap* amapT = maps + jb.a_mapT;
        const int a_mn = jb.a_mn, b_mn = jb.b_mn, a_mat = jb.a_mat, b_mat = jb.b_mat;
        const int a_up = KB == 64 ? jb.a_up : 0, b_up = KB == 64 ? jb.b_up : 0;
        // L2 prefetch kPrefetch k-blocks beyond the shared-memory ring: the ring only covers ~3 k-blocks of
        // MMA time, less than an HBM miss, and every tile's first touch of an operand block misses L2
        auto prefetch = [&](int kb) {
          const int k0 = kb * KB;
          for (int p = 0; p < C::kPlanes; ++p) {
            if (!a_mn) {
              tma_prefetch_4d(amap, k0, am, p, a_mat);
            } else {
              tma_prefetch_4d(amap, am, k0, p, a_mat);
              tma_prefetch_4d(amap, am + 64, k0, p, a_mat);
            }
            for (int h = 0; h < NT / 128; ++h) {
              if (!b_mn) tma_prefetch_4d(bmap, k0, bn + 64 * h, p, b_mat);
              else tma_prefetch_4d(bmap, bn + 64 * h, k0, p, b_mat);
            }
          }
        };
        if (xp & 16)  // experiment knob: L2 prefetch ahead of the ring (measured: no gain)
          for (int kb = 0; kb < kPrefetch && kb < nk; ++kb) prefetch(kb);
        for (int kb = 0; kb < nk; ++kb) {
          if ((xp & 16) && kb + kPrefetch < nk) prefetch(kb + kPrefetch);
          {
            const long long w0 = prof ? clock64() : 0;
            mbar_wait(&empty[stage], phase ^ 1);
            if (prof) pw0 += clock64() - w0;
          }
          const int nplanes = (xp & 1) ? 1 : C::kPlanes;  // experiment knob: hi planes only (timing)
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * C::kStageBytes / C::kPlanes * nplanes);
          uint8_t* sA = smem + stage * C::kStageBytes;
          uint8_t* sB = sA + C::kABytes * C::kPlanes;
          const int k0 = kb * KB;
          auto load = [&](void* dst, const CUtensorMap* map, int x0, int x1, int pl, int mat) {
            if (!(xp & 128)) tma2_load_4d_hint(dst, map, &full[stage], x0, x1, pl, mat, pol_load);  // L2 evict-last
            else tma2_load_4d(dst, map, &full[stage], x0, x1, pl, mat);
          };
          // upper pair-block storage: a lower k-block is read as the transposed upper one (other majorness)
          const bool fa = a_up && upper_flip(a_mn, ti, k0 >> 8);
          const bool fb = b_up && upper_flip(b_mn, bn >> 8, k0 >> 8);
          const int ea_mn = a_mn ^ static_cast<int>(fa), eb_mn = b_mn ^ static_cast<int>(fb);
          const CUtensorMap* am_cur = fa ? amapT : amap;
#pragma unroll
          for (int p = 0; p < C::kPlanes; ++p) {
            if (p >= nplanes) break;
            uint8_t* a_dst = sA + p * C::kABytes;
            uint8_t* b_dst = sB + p * C::kBBytes;
            if (!ea_mn) {
              load(a_dst, am_cur, k0, am, p, a_mat);
            } else {
              load(a_dst, am_cur, am, k0, p, a_mat);
              load(a_dst + 64 * KB * 2, am_cur, am + 64, k0, p, a_mat);
            }
            // B: NT / 2 rows per CTA as 64-row boxes (K-major: consecutive 8-row groups; MN-major: 64-column
            // groups KB * 128 B apart, the LBO of the descriptor)
#pragma unroll
            for (int h = 0; h < NT / 128; ++h) {
              if (!eb_mn) load(b_dst + h * 64 * KB * 2, bmap, k0, bn + 64 * h, p, b_mat);
              else load(b_dst + h * 64 * KB * 2, bmap, bn + 64 * h, k0, p, b_mat);
            }
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (leader CTA only)
    // The whole warp runs the loop (warp-uniform control flow); one elected lane issues each MMA / commit.
    if (rank == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t t = 0;
      uint32_t ucount = 0;  // ring mode: accumulation units issued so far
      for (;; ++t) {
        int tile = 0;
        if (lane == 0) tile = next_tile(t);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile < 0) break;
        const GemmJob& jb = jobs[find_job<NT>(jobs, njobs, tile, uniform)];
        const int nk = (jb.K + KB - 1) / KB;
        int ti, tj;
        tile_coords<NT>(jb, tile - job_tile_start<NT>(jb), ti, tj);
        const int a_up = KB == 64 ? jb.a_up : 0, b_up = KB == 64 ? jb.b_up : 0;
        const int bpb = (tj * kPN) >> 8;  // 256-block of this tile's B rows (the same for both CTAs)
        // Split products keep the cross terms hi*lo + lo*hi (2^-11 smaller) in their own "correction" slot, the
        // last one of the tile, so they never truncate against the full-size sum.  The hi*hi terms go to
        // `nmain` slots by K range: nacc == 2 -> one main slot over the whole K; nacc == 4 -> three main slots of
        // K / 3 each (shorter truncating accumulation chains, FULL64).  Unsplit products (fp16, or DASH_NACC=1)
        // put every pass into slot c = K range c of nacc.
        const int per_us = ring ? (nk * (KB / 16) + nring - 1) / nring : 0;  // k steps per ring unit
        if (ring && per_us % (KB / 16) == 0) {  // ---- ring mode, units of whole k blocks (the usual case)
          const int per_u = per_us / (KB / 16);
          uint32_t u = ucount;  // the current unit (counters, not divisions: this loop is issue-latency bound)
          int kin = 0;          // k-blocks of the current unit issued
          for (int kb = 0; kb < nk; ++kb) {
            const bool first = kin == 0;
            const uint32_t slot = u % kSl;
            if (first) {
              const long long w0 = prof ? clock64() : 0;
              mbar_wait(&tempty[slot], ((u / kSl) & 1u) ^ 1u);
              if (prof) pw0 += clock64() - w0;
              tc_fence_after();
            }
            const int a_mn = jb.a_mn ^ static_cast<int>(a_up && upper_flip(jb.a_mn, ti, (kb * KB) >> 8));
            const int b_mn = jb.b_mn ^ static_cast<int>(b_up && upper_flip(jb.b_mn, bpb, (kb * KB) >> 8));
            const uint32_t idesc = umma_idesc_f16(kPairM, kPN, a_mn, b_mn);
            const uint32_t a_lbo = a_mn ? KB * 128u : 16u, b_lbo = b_mn ? KB * 128u : 16u;
            const uint32_t a_kstep = a_mn ? 2048u : 32u, b_kstep = b_mn ? 2048u : 32u;
            const uint32_t a_sbo = a_mn ? 1024u : (KB == 64 ? 1024u : 512u), b_sbo = b_mn ? 1024u : (KB == 64 ? 1024u : 512u);
            const uint32_t a_lay = a_mn ? 2u : (KB == 64 ? 2u : 4u), b_lay = b_mn ? 2u : (KB == 64 ? 2u : 4u);
            {
              const long long w0 = prof ? clock64() : 0;
              mbar_wait(&full[stage], phase);
              if (prof) pw1 += clock64() - w0;
            }
            tc_fence_after();
            const uint32_t a_base = smem_u32(smem + stage * C::kStageBytes);
            const uint32_t b_base = a_base + C::kABytes * C::kPlanes;
#pragma unroll
            for (int k = 0; k < KB / 16; ++k) {
#pragma unroll
              for (int p = 0; p < PASSES; ++p) {
                const uint32_t ap = (p == 2) ? 1u : 0u, bp = (p == 1) ? 1u : 0u;
                const uint64_t ad = umma_sdesc(a_base + ap * C::kABytes + k * a_kstep, a_lbo, a_sbo, a_lay);
                const uint64_t bd = umma_sdesc(b_base + bp * C::kBBytes + k * b_kstep, b_lbo, b_sbo, b_lay);
                umma2_f16_elect(tmem_base + slot * kPN, ad, bd, idesc, (first && k == 0 && p == 0) ? 0u : 1u);
              }
            }
            umma2_commit_mc_elect(&empty[stage]);
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
            if (++kin == per_u || kb == nk - 1) {
              umma2_commit_mc_elect(&tfull[slot]);
              ++u;
              kin = 0;
            }
          }
          ucount = u;
          continue;
        }
        if (ring) {  // ---- ring mode, units of per_u 16-wide k steps (shorter than a k block: FULL64, B <= 512)
          const int per_u = per_us;
          uint32_t u = ucount;
          int kin = 0;          // k steps of the current unit issued
          for (int kb = 0; kb < nk; ++kb) {
            const int a_mn = jb.a_mn ^ static_cast<int>(a_up && upper_flip(jb.a_mn, ti, (kb * KB) >> 8));
            const int b_mn = jb.b_mn ^ static_cast<int>(b_up && upper_flip(jb.b_mn, bpb, (kb * KB) >> 8));
            const uint32_t idesc = umma_idesc_f16(kPairM, kPN, a_mn, b_mn);
            const uint32_t a_lbo = a_mn ? KB * 128u : 16u, b_lbo = b_mn ? KB * 128u : 16u;
            const uint32_t a_kstep = a_mn ? 2048u : 32u, b_kstep = b_mn ? 2048u : 32u;
            const uint32_t a_sbo = a_mn ? 1024u : (KB == 64 ? 1024u : 512u), b_sbo = b_mn ? 1024u : (KB == 64 ? 1024u : 512u);
            const uint32_t a_lay = a_mn ? 2u : (KB == 64 ? 2u : 4u), b_lay = b_mn ? 2u : (KB == 64 ? 2u : 4u);
            {
              const long long w0 = prof ? clock64() : 0;
              mbar_wait(&full[stage], phase);
              if (prof) pw1 += clock64() - w0;
            }
            tc_fence_after();
            const uint32_t a_base = smem_u32(smem + stage * C::kStageBytes);
            const uint32_t b_base = a_base + C::kABytes * C::kPlanes;
#pragma unroll
            for (int k = 0; k < KB / 16; ++k) {
              const uint32_t slot = u % kSl;
              if (kin == 0) {
                const long long w0 = prof ? clock64() : 0;
                mbar_wait(&tempty[slot], ((u / kSl) & 1u) ^ 1u);
                if (prof) pw0 += clock64() - w0;
                tc_fence_after();
              }
#pragma unroll
              for (int p = 0; p < PASSES; ++p) {
                const uint32_t ap = (p == 2) ? 1u : 0u, bp = (p == 1) ? 1u : 0u;
                const uint64_t ad = umma_sdesc(a_base + ap * C::kABytes + k * a_kstep, a_lbo, a_sbo, a_lay);
                const uint64_t bd = umma_sdesc(b_base + bp * C::kBBytes + k * b_kstep, b_lbo, b_sbo, b_lay);
                umma2_f16_elect(tmem_base + slot * kPN, ad, bd, idesc, (kin == 0 && p == 0) ? 0u : 1u);
              }
              if (++kin == per_u || (kb == nk - 1 && k == KB / 16 - 1)) {
                umma2_commit_mc_elect(&tfull[slot]);
                ++u;
                kin = 0;
              }
            }
            umma2_commit_mc_elect(&empty[stage]);
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
          }
          ucount = u;
          continue;
        }
        const int nmain = mc ? 1 : (mc4 ? 3 : nacc);
        const int per = (nk + nmain - 1) / nmain;  // k-blocks per main slot
        const bool corr = mc || mc4;
        // K-major: 128-byte (KB 64) or 64-byte (KB 32) swizzled rows, 8-row groups 1024 / 512 B apart, 32 B per
        // 16-wide k step; MN-major: 128-byte rows along M/N, 64-column groups KB * 128 B apart, 2 KB per k step
        constexpr uint32_t kSbo = KB == 64 ? 1024u : 512u, kLay = KB == 64 ? 2u : 4u;
        const uint32_t base = (t % nsets) * static_cast<uint32_t>(nacc);
        const uint32_t corr_slot = base + static_cast<uint32_t>(nacc - 1);
        const uint32_t d_corr = tmem_base + corr_slot * kPN;
        const uint32_t use_par = ((t / nsets) & 1u) ^ 1u;
        int c = 0, kin = 0;  // main slot and k-blocks issued into it (counters: no divisions in the issue loop)
        for (int kb = 0; kb < nk; ++kb) {
          const bool first = kin == 0;
          const uint32_t slot = base + static_cast<uint32_t>(c);
          if (first || (corr && kb == 0)) {
            const long long w0 = prof ? clock64() : 0;
            if (first) mbar_wait(&tempty[slot], use_par);
            if (corr && kb == 0) mbar_wait(&tempty[corr_slot], use_par);
            if (prof) pw0 += clock64() - w0;
            tc_fence_after();
          }
          const uint32_t d_tmem = tmem_base + slot * kPN;
          // operand majorness of this k-block (flipped for lower blocks of upper pair-block storage)
          const int a_mn = jb.a_mn ^ static_cast<int>(a_up && upper_flip(jb.a_mn, ti, (kb * KB) >> 8));
          const int b_mn = jb.b_mn ^ static_cast<int>(b_up && upper_flip(jb.b_mn, bpb, (kb * KB) >> 8));
          const uint32_t idesc = umma_idesc_f16(kPairM, kPN, a_mn, b_mn);
          const uint32_t a_lbo = a_mn ? KB * 128u : 16u, b_lbo = b_mn ? KB * 128u : 16u;
          const uint32_t a_kstep = a_mn ? 2048u : 32u, b_kstep = b_mn ? 2048u : 32u;
          const uint32_t a_sbo = a_mn ? 1024u : kSbo, b_sbo = b_mn ? 1024u : kSbo;
          const uint32_t a_lay = a_mn ? 2u : kLay, b_lay = b_mn ? 2u : kLay;
          {
            const long long w0 = prof ? clock64() : 0;
            mbar_wait(&full[stage], phase);
            if (prof) pw1 += clock64() - w0;
          }
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem + stage * C::kStageBytes);
          const uint32_t b_base = a_base + C::kABytes * C::kPlanes;
#pragma unroll
          for (int k = 0; k < KB / 16; ++k) {
#pragma unroll
            for (int p = 0; p < PASSES; ++p) {
              const uint32_t ap = (p == 2) ? 1u : 0u;  // pass 2: A_lo * B_hi
              const uint32_t bp = (p == 1) ? 1u : 0u;  // pass 1: A_hi * B_lo
              const uint64_t ad = umma_sdesc(a_base + ap * C::kABytes + k * a_kstep, a_lbo, a_sbo, a_lay);
              const uint64_t bd = umma_sdesc(b_base + bp * C::kBBytes + k * b_kstep, b_lbo, b_sbo, b_lay);
              const bool to_corr = corr && p > 0;
              // a slot's first write overwrites (main: pass 0 of its first k step; correction: pass 1 of k-block 0)
              const uint32_t fresh = to_corr ? ((kb == 0 && k == 0 && p == 1) ? 0u : 1u)
                                             : ((first && k == 0 && p == 0) ? 0u : 1u);
              umma2_f16_elect(to_corr ? d_corr : d_tmem, ad, bd, idesc, fresh);
            }
          }
          umma2_commit_mc_elect(&empty[stage]);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
          if (++kin == per || kb == nk - 1) {  // this main slot's K range is complete
            umma2_commit_mc_elect(&tfull[slot]);
            ++c;
            kin = 0;
          }
          if (corr && kb == nk - 1) umma2_commit_mc_elect(&tfull[corr_slot]);
        }
        // main slots without k-blocks (nk < nmain): keep every slot's phase in step
        for (; c < nmain; ++c) {
          const uint32_t slot = base + static_cast<uint32_t>(c);
          mbar_wait(&tempty[slot], use_par);
          tc_fence_after();
          umma2_commit_mc_elect(&tfull[slot]);
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2..9 of both CTAs)
    const int q = warp & 3;                         // TMEM lane quarter (warps 2..9 -> 2, 3, 0, 1, 2, 3, 0, 1)
    const int hc = static_cast<int>(warp - 2) >> 2;  // column half (64 columns) of this warp
    uint8_t* ebuf = smem + C::kStages * C::kStageBytes + (warp - 2) * 8192;  // 1024-aligned staging tile
    uint32_t sphase = 0;
    const uint32_t leader_tempty = mapa_shared(smem_u32(tempty), 0);
    const uint64_t pol_store = l2_policy_evict_first();
    auto wait_reads = [&]() {  // lane 0: this warp's bulk stores have read the staging buffer
      const long long w0 = prof ? clock64() : 0;
      bulk_wait_read0();
      if (prof) pw1 += clock64() - w0;
    };
    // split tile bulk store, L2 evict-first (its next reader is a later launch; keep the operands resident)
    auto store4 = [&](int map, int x0, int x1, int mat) {
      if (!(xp & 64)) tma_store_4d_hint(maps + map, ebuf, x0, x1, 0, mat, pol_store);
      else tma_store_4d(maps + map, ebuf, x0, x1, 0, mat);
    };
    uint32_t t = 0;
    uint32_t ucount = 0;  // ring mode: accumulation units drained so far
    for (;; ++t) {
      int tile = 0;
      if (lane == 0) tile = next_tile(t);
      tile = __shfl_sync(0xffffffffu, tile, 0);
      if (tile < 0) break;
      const GemmJob& jb = jobs[find_job<NT>(jobs, njobs, tile, uniform)];
      const int local = tile - job_tile_start<NT>(jb);
      int ti, tj;
      tile_coords<NT>(jb, local, ti, tj);
      const int m0 = ti * kPairM;
      // NT = 256: two rounds over 128-column halves; TMEM is released after the last one
      for (int rd = 0; rd < kRounds; ++rd) {
        const int n0 = tj * kPN + 128 * rd;
        const int nk = (jb.K + KB - 1) / KB;
        const int nmain = mc ? 1 : (mc4 ? 3 : nacc);
        const int per = (nk + nmain - 1) / nmain;
        const int used_main = (nk + per - 1) / per;  // main slots with k-blocks; the correction slot is the last
        const uint32_t base = (t % nsets) * static_cast<uint32_t>(nacc);
        const uint32_t use_par = (t / nsets) & 1u;
        const bool side_tma = jb.s_map >= 0;
        const bool f_tma = jb.f_map >= 0;
        const bool fin_tma = f_tma && jb.op == EPI_EMA;
        __syncwarp();                 // every lane is done with the previous tile's staging buffer
        const bool side_load = side_tma && !(xp & 256);  // (knob 256: timing without the side-input load)
        if ((side_load || fin_tma) && lane == 0) {  // stage the side / fp32 input tile while the MMAs run
          wait_reads();          // the previous tile's bulk stores have read the buffer
          mbar_arrive_expect_tx(&sbar[warp - 2], 8192);
          const int tc0 = n0 + 64 * hc, tr0 = m0 + kHalf * static_cast<int>(rank) + 32 * q;
          if (side_tma) {
            tma_load_4d(ebuf, maps + jb.s_map, &sbar[warp - 2], tc0, tr0, 0, jb.s_mat);
          } else {
            tma_load_3d(ebuf, maps + jb.f_map, &sbar[warp - 2], tc0, tr0, jb.f_mat);
            tma_load_3d(ebuf + 4096, maps + jb.f_map, &sbar[warp - 2], tc0 + 32, tr0, jb.f_mat);
          }
        }
        float acc[64];
        // ring mode: drain the tile's units in issue order (unit u -> slot u % kSl), summing in registers
        const int nsteps = nk * (KB / 16), per_us = ring ? (nsteps + nring - 1) / nring : 1;
        const int nunits = ring ? (nsteps + per_us - 1) / per_us : nacc;
        for (int c = 0; c < nunits; ++c) {
          if (ring) {
            const uint32_t u = ucount + static_cast<uint32_t>(c), slot = u % kSl;
            const long long w0 = prof ? clock64() : 0;
            mbar_wait(&tfull[slot], (u / kSl) & 1u);
            if (prof) pw0 += clock64() - w0;
            tc_fence_after();
            const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + slot * kPN + 64 * hc;
  #pragma unroll
            for (int j = 0; j < 2; ++j) {
              float v[32];
              tmem_ld32(taddr + 32 * j, v);
  #pragma unroll
              for (int i = 0; i < 32; ++i) acc[32 * j + i] = (c == 0) ? v[i] : acc[32 * j + i] + v[i];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote_relaxed(leader_tempty + slot * 8);
            continue;
          }
          const uint32_t slot = base + static_cast<uint32_t>(c);
          if (rd == 0) {
            const long long w0 = prof ? clock64() : 0;
            mbar_wait(&tfull[slot], use_par);
            if (prof) pw0 += clock64() - w0;
            tc_fence_after();
          }
          if (c < used_main || ((mc || mc4) && c == nacc - 1)) {
            const uint32_t taddr =
                tmem_base + (static_cast<uint32_t>(q * 32) << 16) + slot * kPN + 128 * rd + 64 * hc;
  #pragma unroll
            for (int j = 0; j < 2; ++j) {
              float v[32];
              tmem_ld32(taddr + 32 * j, v);
  #pragma unroll
              for (int i = 0; i < 32; ++i) acc[32 * j + i] = (c == 0) ? v[i] : acc[32 * j + i] + v[i];
            }
          }
          if (rd == kRounds - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote_relaxed(leader_tempty + slot * 8);
          }
        }
        if (ring) ucount += static_cast<uint32_t>(nunits);
        // ---- fused epilogue on the fp32 sums
        EpiCtx cx;
        cx.op = jb.op;
        cx.mat = jb.out_mat;
        cx.r = m0 + kHalf * static_cast<int>(rank) + q * 32 + static_cast<int>(lane);
        cx.M = jb.M;
        cx.N = jb.N;
        // symmetric job: this CTA's 128 x 128 sub-block (row block 2 ti + rank, column block n0 / 128)
        const int rb = 2 * ti + static_cast<int>(rank), cb = n0 / 128;
        cx.store = !jb.sym || rb <= cb;
        cx.mirror = jb.sym && rb < cb && (!jb.c_up || (rb >> 1) == (cb >> 1));
        cx.row_ok = cx.r < jb.M && cx.store;
        const int ea = jb.a_exp ? __ldg(jb.a_exp) : 0;
        const int eb = jb.b_exp ? __ldg(jb.b_exp) : 0;
        cx.sc = ldexpf(1.f, ea + eb);
        cx.mul = jb.alpha * (jb.alpha_p ? __ldg(jb.alpha_p + cx.mat) : 1.f);
        cx.inactive = jb.active && __ldg(jb.active + cx.mat) == 0;
        cx.gam = jb.gamma_p ? *jb.gamma_p : jb.gamma;
        const float prod_bound = static_cast<float>(jb.K) * amax_of(jb.a_amax) * amax_of(jb.b_amax);
        cx.side_scale = jb.s_hi ? ldexpf(1.f, __ldg(jb.s_exp)) : 0.f;
        int e_out = 0;
        switch (cx.op) {
          case EPI_SPLIT: e_out = exp_from_bound(prod_bound * fabsf(cx.mul)); break;
          case EPI_NDB_E: e_out = kEExp; break;
          case EPI_CHEB: e_out = exp_from_bound(2.f * prod_bound + amax_of(jb.s_amax) + fabsf(cx.gam)); break;
          case EPI_CHEB_FINAL:
            e_out = exp_from_bound((prod_bound + amax_of(jb.s_amax) + fabsf(cx.gam)) * fabsf(cx.mul));
            break;
          case EPI_CN_M: e_out = exp_from_bound(prod_bound); break;
          default: break;
        }
        if (m0 == 0 && n0 == 0 && rank == 0 && threadIdx.x == 64) {
          if (jb.c_exp) *jb.c_exp = e_out;
          if (jb.c2_exp) *jb.c2_exp = kEExp;
        }
        cx.inv_out = ldexpf(1.f, -e_out);
        cx.inv_e = ldexpf(1.f, -kEExp);
        cx.cn_a = 1.f + 1.f / jb.beta;
        cx.cn_b = 1.f / jb.beta;
        cx.amax = cx.amax2 = cx.resid = 0.f;
        cx.sumsq = 0.0;
        cx.ovf = cx.ovf2 = false;
        const bool tma_out = jb.c_map >= 0;
        cx.sbuf = nullptr;
        cx.fbuf = nullptr;
        cx.f_tma = f_tma;
        cx.lane = static_cast<int>(lane);
        cx.lc0 = n0 + 64 * hc;
        if (side_tma || fin_tma) {
          if (side_load || fin_tma) {
            mbar_wait(&sbar[warp - 2], sphase);
            sphase ^= 1u;
          }
          if (side_tma) cx.sbuf = ebuf;
          else cx.fbuf = ebuf;
        }
  #pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c0 = n0 + 64 * hc + 16 * j;
          float (&v)[16] = *reinterpret_cast<float(*)[16]>(&acc[16 * j]);  // in place: final values stay in acc
          // (a symmetric job's sub-block below the diagonal is neither stored nor reduced: skip its math)
          if (c0 < jb.N && cx.store && !(xp & 2)) epi_piece<16>(jb, cx, c0, v, !tma_out);
        }
        if ((tma_out || f_tma) && cx.store && !(xp & 2)) {
          // ---- staged bulk-tensor stores of the split output(s), direct and (symmetric jobs) mirrored
          const int r0 = m0 + kHalf * static_cast<int>(rank) + 32 * q;
          const int c0 = n0 + 64 * hc;
          const int lr = static_cast<int>(lane);
          auto ident = [](float v, int) { return v; };
          if (tma_out) {
          if (lane == 0) wait_reads();  // this warp's previous stores have read the buffer
          __syncwarp();                      // (and every lane is done with the staged side input)
          if (!(xp & 4)) stage_direct(ebuf, acc, lr, c0, cx.inv_out, ident, cx.ovf);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && !(xp & 8)) {
            store4(jb.c_map, c0, r0, jb.c_mat);
            bulk_commit();
          }
          if (cx.mirror && (xp & 32)) {
            store_mirror_from_stage(ebuf, jb.c_hi, jb.c_plane, jb.c_ld, r0, c0, cx.N, lr);
          } else if (cx.mirror) {
            if (lane == 0) wait_reads();
            __syncwarp();
            stage_transpose_in_place(ebuf, lr);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              store4(jb.c_tmap, r0, c0, jb.c_mat);
              bulk_commit();
            }
          }
          if (jb.c2_map >= 0) {  // EPI_CN_M: next correction C = (1 + 1/p) I - M / p (I when frozen)
            const int r = cx.r;
            const float ca = cx.cn_a, cb = cx.cn_b;
            const bool inact = cx.inactive;
            auto corr = [r, ca, cb, inact](float m, int col) {
              const float d = (r == col) ? 1.f : 0.f;
              return inact ? d : ca * d - cb * m;
            };
            if (lane == 0) wait_reads();
            __syncwarp();
            stage_direct(ebuf, acc, lr, c0, cx.inv_e, corr, cx.ovf2);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              store4(jb.c2_map, c0, r0, jb.c2_mat);
              bulk_commit();
            }
            if (cx.mirror && (xp & 32)) {
              store_mirror_from_stage(ebuf, jb.c2_hi, jb.c2_plane, jb.c_ld, r0, c0, cx.N, lr);
            } else if (cx.mirror) {
              if (lane == 0) wait_reads();
              __syncwarp();
              stage_transpose_in_place(ebuf, lr);
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                store4(jb.c2_tmap, r0, c0, jb.c2_mat);
                bulk_commit();
              }
            }
          }
          }  // tma_out
          if (f_tma) {  // fp32 output: direct tile (two swizzled 32 x 32 boxes) and, if symmetric, its mirror
            if (lane == 0) wait_reads();
            __syncwarp();
            stage_direct_f32(ebuf, acc, lr);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_3d(maps + jb.f_map, ebuf, c0, r0, jb.f_mat);
              tma_store_3d(maps + jb.f_map, ebuf + 4096, c0 + 32, r0, jb.f_mat);
              bulk_commit();
            }
            if (cx.mirror) {
              if (lane == 0) wait_reads();
              __syncwarp();
              stage_transposed_f32(ebuf, acc, lr);
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_3d(maps + jb.f_tmap, ebuf, r0, c0, jb.f_mat);
                bulk_commit();
              }
            }
          }
        }
        // per-matrix reductions (max is order independent -> deterministic)
        float am = cx.ovf ? __uint_as_float(0x7fc00000u) : cx.amax;
        float am2 = cx.ovf2 ? __uint_as_float(0x7fc00000u) : cx.amax2;
        float rs = cx.resid;
        am = warp_max_nonneg(am);
        am2 = warp_max_nonneg(am2);
        rs = warp_max_nonneg(rs);
        if (lane == 0 && cx.store) {
          if (jb.c_amax) atomic_max_nonneg(jb.c_amax, am);
          if (jb.c2_amax) atomic_max_nonneg(jb.c2_amax, am2);
          if (jb.resid && !cx.inactive)
            atomic_max_nonneg(jb.resid + cx.mat, (cx.op == EPI_NDB_E || cx.op == EPI_CN_M) && cx.ovf
                                                     ? __uint_as_float(0x7fc00000u) : rs);
        }
        if (cx.op == EPI_APPLY) {  // (never in NT = 256 launches: the host keeps them to symmetric jobs)
          const double sacc = warp_sum_d(cx.sumsq);
          if (lane == 0) jb.partial[local * kPartialsPerTile + rank * 8 + hc * 4 + q] = static_cast<float>(sacc);
        }
      }  // round
    }
    if (lane == 0) bulk_wait0();  // bulk stores complete before the CTA retires
  }
  if (prof && lane == 0 && (warp >= 2 || warp == 0 || rank == 0)) {
    const unsigned long long tot = clock64() - t_start;
    if (warp == 0) { atomicAdd(prof + 0, pw0); atomicAdd(prof + 5, tot); }
    else if (warp == 1) { atomicAdd(prof + 1, pw0); atomicAdd(prof + 2, pw1); atomicAdd(prof + 6, tot); }
    else { atomicAdd(prof + 3, pw0); atomicAdd(prof + 4, pw1); atomicAdd(prof + 7, tot); }
  }
  tc_fence_before();
  cluster_sync_all();  // no CTA of the pair may exit while its peer still uses its TMEM / barriers
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2<512>(tmem_base);
  }
}

// ---------------------------------------------------------------------------- host launcher
constexpr int kMaxDevices = 64;
static int g_nacc = 0;
static int g_dbg = -1;
static int g_exp = -1;
static int g_kb = 0;
constexpr int kKbDefault = 64;   // K-block of the launches (env DASH_KB = 32 | 64)
constexpr int kWideDefault = 1;  // 256-wide tiles for fp16 launches of symmetric jobs (env DASH_NT)

// Launch accounting + optional CUDA-event timing of every GEMM launch (bench / roofline hooks).
struct GemmTimer {
  bool on = false;
  std::vector<cudaEvent_t> ev;  // start/stop pairs
  std::vector<double> flops, issued;
  std::vector<int> tiles;
  size_t used = 0;
};
static GemmTimer g_timer;        // diagnostics (bench / roofline hooks); guarded by g_timer_mu
static std::mutex g_timer_mu;
std::atomic<unsigned long long> g_launches{0};

void note_launch(int n) { g_launches += static_cast<unsigned long long>(n); }

static int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev < 0 ? 0 : (dev >= kMaxDevices ? kMaxDevices - 1 : dev);
}

template <int PASSES, int KB, int NT = 128>
static void launch_variant(int grid2, cudaStream_t stream, const GemmJob* d_jobs, int njobs, int total_tiles,
                           const CUtensorMap* d_maps, const int* gate, int flags, int uniform, int* counter,
                           unsigned long long* prof) {
  static std::once_flag attr[kMaxDevices];  // the attribute is per device; set once per device, thread-safe
  std::call_once(attr[current_device()], [] {
    cudaFuncSetAttribute(dash_gemm2_kernel<PASSES, KB, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Gemm2Cfg<PASSES, KB, NT>::kSmemBytes);
  });
  dash_gemm2_kernel<PASSES, KB, NT><<<grid2, kThreads2, Gemm2Cfg<PASSES, KB, NT>::kSmemBytes, stream>>>(
      d_jobs, njobs, total_tiles, d_maps, gate, flags, uniform, counter, prof);
}

int gemm_kblock() {
  if (g_kb == 0) {
    const char* e = getenv("DASH_KB");
    g_kb = e ? atoi(e) : kKbDefault;
    if (g_kb != 32 && g_kb != 64) g_kb = kKbDefault;
  }
  return g_kb;
}

// 256-wide pair tiles (DASH_NT): 0 never, 1 fp16 launches (default), 2 fp16 and split launches
static int wide_mode() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("DASH_NT");
    m = !e ? kWideDefault : atoi(e) == 128 ? 0 : atoi(e) == 256 ? 1 : atoi(e) == 2562 ? 2 : kWideDefault;
  }
  return m;
}

// counter: the launch's pair of device ints (tile counter, finished pairs) for the dynamic tile scheduler,
// carved from the caller's workspace and zeroed at upload; the kernel re-arms both to zero when it finishes,
// so the same uploaded launch can run back to back on one stream.
int gemm_launch(const GemmJob* d_jobs, int njobs, int total_tiles, const CUtensorMap* d_maps, int passes,
                cudaStream_t stream, int* counter, const int* gate, double flops, int uniform, double issued,
                const GemmWide* wide) {
  if (total_tiles <= 0) return 0;
  if (!counter) return 1;
  // passes = 4: the split 3-pass products in ring mode with 16 K ranges per tile (FULL64: each truncating
  // tensor-core accumulation chain covers K / 16; B = 1024 Newton-DB error ~14x smaller than the main +
  // correction default, ~20% slower); otherwise the DASH_NACC default
  int nacc_req = 0;
  int kb_force = 0;
  if (passes == 4) {  // FULL64: 32-wide K blocks and one ring unit per K block (32-long truncating chains)
    passes = 3;
    nacc_req = 32;
    kb_force = 32;
    issued *= 0.75;
  }
  const int wm = wide_mode();
  const bool use_wide = wide && wide->tiles > 0 && (passes == 1 ? wm >= 1 : wm >= 2);
  if (use_wide) {
    total_tiles = wide->tiles;
    uniform = wide->uniform;
    issued = wide->issued1 * passes;
  }
  ++g_launches;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  std::unique_lock<std::mutex> timer_lock(g_timer_mu, std::defer_lock);
  if (g_timer.on) timer_lock.lock();
  if (g_timer.on) {
    if (g_timer.used + 2 > g_timer.ev.size()) {
      for (int i = 0; i < 256; ++i) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        g_timer.ev.push_back(e);
      }
    }
    e0 = g_timer.ev[g_timer.used];
    e1 = g_timer.ev[g_timer.used + 1];
    g_timer.used += 2;
    g_timer.flops.push_back(flops);
    g_timer.issued.push_back(issued);
    g_timer.tiles.push_back(total_tiles);
    cudaEventRecord(e0, stream);
  }
  if (g_dbg < 0) {
    const char* e = getenv("DASH_GEMM_DEBUG");
    g_dbg = e ? atoi(e) : 0;
  }
  if (g_exp < 0) {
    const char* e = getenv("DASH_EXP");
    g_exp = e ? atoi(e) : 0;
  }
  if (g_nacc == 0) {
    const char* e = getenv("DASH_NACC");
    g_nacc = e ? atoi(e) : kNaccDefault;
    if (g_nacc != 1 && g_nacc != 2 && g_nacc != 4 && g_nacc != 8 && g_nacc != 16) g_nacc = kNaccDefault;
  }
  int num_sms = 0;
  cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, current_device());
  cudaError_t err;
  const int grid2 = 2 * (total_tiles < num_sms / 2 ? total_tiles : num_sms / 2);  // CTA pairs
  static unsigned long long* prof = nullptr;  // DASH_GEMM_DEBUG=2 diagnostics only
  if ((g_dbg & 2) && !prof) {
    cudaMalloc(&prof, 8 * sizeof(unsigned long long));
    cudaMemset(prof, 0, 8 * sizeof(unsigned long long));
  }
  if (g_kb == 0) {
    const char* e = getenv("DASH_KB");
    g_kb = e ? atoi(e) : kKbDefault;
    if (g_kb != 32 && g_kb != 64) g_kb = kKbDefault;
  }
  const int flags = (passes == 3 ? (nacc_req ? nacc_req : g_nacc) : 1) | (g_exp << 8);
  const int kb = kb_force ? kb_force : g_kb;
  if (use_wide && passes == 3 && kb == 64) launch_variant<3, 64, 256>(grid2, stream, d_jobs, njobs, total_tiles, d_maps, gate, flags, uniform, counter, prof);
  else if (use_wide && passes == 3) launch_variant<3, 32, 256>(grid2, stream, d_jobs, njobs, total_tiles, d_maps, gate, flags, uniform, counter, prof);
  else if (use_wide && kb == 64) launch_variant<1, 64, 256>(grid2, stream, d_jobs, njobs, total_tiles, d_maps, gate, flags, uniform, counter, prof);
  else if (use_wide) launch_variant<1, 32, 256>(grid2, stream, d_jobs, njobs, total_tiles, d_maps, gate, flags, uniform, counter, prof);
  else if (passes == 3 && kb == 64) launch_variant<3, 64>(grid2, stream, d_jobs, njobs, total_tiles, d_maps, gate, flags, uniform, counter, prof);
  else if (passes == 3) launch_variant<3, 32>(grid2, stream, d_jobs, njobs, total_tiles, d_maps, gate, flags, uniform, counter, prof);
  else if (kb == 64) launch_variant<1, 64>(grid2, stream, d_jobs, njobs, total_tiles, d_maps, gate, flags, uniform, counter, prof);
  else launch_variant<1, 32>(grid2, stream, d_jobs, njobs, total_tiles, d_maps, gate, flags, uniform, counter, prof);
  if (e1) cudaEventRecord(e1, stream);
  if (prof) {  // diagnostics: per-launch wait-cycle breakdown (serialises the stream)
    unsigned long long h[8];
    cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    cudaMemsetAsync(prof, 0, sizeof(h), stream);
    auto pct = [](unsigned long long a, unsigned long long b) { return b ? 100.0 * a / b : 0.0; };
    fprintf(stderr,
            "[gemm] passes=%d nt=%d tiles=%d  producer: empty-wait %.1f%%  mma: tempty-wait %.1f%% full-wait %.1f%%"
            "  epilogue: tfull-wait %.1f%% store-read-wait %.1f%%\n",
            passes, use_wide ? 256 : 128, total_tiles, pct(h[0], h[5]), pct(h[1], h[6]), pct(h[2], h[6]),
            pct(h[3], h[7]), pct(h[4], h[7]));
  }
  err = cudaGetLastError();
  return err == cudaSuccess ? 0 : 3;
}

void gemm_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(g_timer_mu);
  g_timer.on = on != 0;
  g_timer.used = 0;
  g_timer.flops.clear();
  g_timer.issued.clear();
  g_timer.tiles.clear();
}

int gemm_timing_list(int cap, double* ms, double* flops, double* issued, int* tiles) {
  std::lock_guard<std::mutex> lk(g_timer_mu);
  const int k = static_cast<int>(g_timer.used / 2);
  const int n = k < cap ? k : cap;
  for (int i = 0; i < n; ++i) {
    float x = 0.f;
    if (cudaEventSynchronize(g_timer.ev[2 * i + 1]) != cudaSuccess) return -3;
    cudaEventElapsedTime(&x, g_timer.ev[2 * i], g_timer.ev[2 * i + 1]);
    ms[i] = x;
    flops[i] = g_timer.flops[i];
    issued[i] = g_timer.issued[i];
    tiles[i] = g_timer.tiles[i];
  }
  return n;
}

// Synchronises on the recorded events; returns launches timed, total ms and total algorithmic flops.
int gemm_timing_read(int* n, double* ms, double* flops) {
  std::lock_guard<std::mutex> lk(g_timer_mu);
  double t = 0.0, f = 0.0;
  const int k = static_cast<int>(g_timer.used / 2);
  for (int i = 0; i < k; ++i) {
    float x = 0.f;
    if (cudaEventSynchronize(g_timer.ev[2 * i + 1]) != cudaSuccess) return 3;
    cudaEventElapsedTime(&x, g_timer.ev[2 * i], g_timer.ev[2 * i + 1]);
    t += x;
    f += g_timer.flops[i];
  }
  *n = k;
  *ms = t;
  *flops = f;
  return 0;
}

}  // namespace dash
