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

#include <cstdlib>
#include <vector>

#include "ptx.cuh"
#include "types.h"

namespace dash {

__device__ __forceinline__ int find_job(const GemmJob* __restrict__ jobs, int njobs, int tile, int uniform = 0) {
  if (uniform) return tile / uniform;  // every job has `uniform` tiles (stacked solver launches)
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(&jobs[mid].tile_start) <= tile) lo = mid; else hi = mid - 1;
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

// Store 32 consecutive values of row r (cols c0..c0+31) as split fp16; masked variant for edges.
__device__ __forceinline__ void store_split32(__half* hi, long long plane, int ld, int r, int c0, int M, int N,
                                              const float (&x)[32], float inv_scale, bool& overflow) {
  if (r >= M) return;
  __half* ph = hi + static_cast<long long>(r) * ld + c0;
  __half* pl = ph + plane;
  if (c0 + 32 <= N) {
    uint32_t hw[16], lw[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
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
    for (int i = 0; i < 4; ++i) {
      dh[i] = make_uint4(hw[4 * i], hw[4 * i + 1], hw[4 * i + 2], hw[4 * i + 3]);
      dl[i] = make_uint4(lw[4 * i], lw[4 * i + 1], lw[4 * i + 2], lw[4 * i + 3]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
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

__device__ __forceinline__ void load_split32(const __half* hi, long long plane, int ld, int r, int c0, int M,
                                             int N, float scale, float (&x)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = 0.f;
  if (r >= M) return;
  const __half* ph = hi + static_cast<long long>(r) * ld + c0;
  const __half* pl = ph + plane;
  if (c0 + 32 <= N) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint4 h = __ldg(reinterpret_cast<const uint4*>(ph) + i);
      uint4 l = __ldg(reinterpret_cast<const uint4*>(pl) + i);
      const __half2* h2 = reinterpret_cast<const __half2*>(&h);
      const __half2* l2 = reinterpret_cast<const __half2*>(&l);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float2 fh = __half22float2(h2[k]);
        float2 fl = __half22float2(l2[k]);
        x[8 * i + 2 * k] = (fh.x + fl.x) * scale;
        x[8 * i + 2 * k + 1] = (fh.y + fl.y) * scale;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (c0 + i < N) x[i] = (__half2float(ph[i]) + __half2float(pl[i])) * scale;
  }
}

// ============================================================================ v2: CTA-pair kernel
// One thread-block cluster of 2 CTAs (a TPC pair) computes a 256 x 128 output tile with
// tcgen05.mma.cta_group::2 (M = 256, N = 128, K = 16 per instruction): each CTA stages its 128 rows of A
// and its 64 rows of B (N/2) per k-block; the leader CTA issues the MMAs; each CTA's TMEM receives its
// 128 output rows.  tcgen05 accumulation truncates, so its error grows linearly with the number of
// MMAs summed into one accumulator (profiles/r1_accumulation_error.log): k-block kb therefore goes to
// accumulator kb % nacc of the tile (nacc x 128 TMEM columns) and the 4 epilogue warps sum the nacc
// partials in fp32 registers (one row x 128 columns per thread).  nacc = 4 (split-f16 modes) cuts the
// Newton-DB error 3.6x for ~9% time; nacc = 1 keeps 4 tiles in flight in TMEM.
constexpr int kPairM = kTileM, kPairN = kTileN, kHalf = kTileM / 2, kHalfN = kTileN / 2;
constexpr int kNaccDefault = 4;   // interleaved TMEM accumulators per tile, split-f16 (env DASH_NACC = 1, 2, 4)
constexpr int kEpiWarps = 4;
constexpr int kAccBufs = 4;       // TMEM accumulation buffers (4 x 128 columns = all 512)
constexpr int kThreads2 = 64 + 32 * kEpiWarps;

template <int PASSES>
struct Gemm2Cfg {
  static constexpr int kPlanes = PASSES == 3 ? 2 : 1;
  static constexpr int kABytes = kHalf * kTileK * 2;   // 16 KB per plane (128 rows of A)
  static constexpr int kBBytes = kHalfN * kTileK * 2;  // 8 KB per plane (64 rows of B)
  static constexpr int kStageBytes = (kABytes + kBBytes) * kPlanes;
  static constexpr int kStages = PASSES == 3 ? 4 : 8;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 512;
};

struct EpiCtx {
  int op, mat, r, M, N;
  bool inactive, row_ok;
  float sc, mul, gam, inv_out, inv_e, side_scale, cn_a, cn_b;
  float amax, amax2, resid;
  double sumsq;
  bool ovf, ovf2;
};

// Apply the fused DASH epilogue to 32 consecutive columns c0.. of row cx.r (x holds the fp32 product).
__device__ __forceinline__ void epi_piece(const GemmJob& jb, EpiCtx& cx, int c0, float (&x)[32]) {
  const int r = cx.r;
  switch (cx.op) {
    case EPI_SPLIT: {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        x[i] *= cx.sc * cx.mul;
        if (cx.row_ok && c0 + i < cx.N) cx.amax = nonneg_max(cx.amax, fabsf(x[i]));
      }
      if (jb.c_hi) store_split32(jb.c_hi, jb.c_plane, jb.c_ld, r, c0, cx.M, cx.N, x, cx.inv_out, cx.ovf);
      if (jb.f_out && cx.row_ok) {
        float* fo = jb.f_out + static_cast<long long>(r) * jb.f_ld + c0;
#pragma unroll
        for (int i = 0; i < 32; ++i) if (c0 + i < cx.N) fo[i] = x[i];
      }
    } break;
    case EPI_NDB_E: {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float d = (r == c0 + i) ? 1.f : 0.f;
        float e = 1.5f * d - 0.5f * (x[i] * cx.sc);
        if (cx.inactive) e = d;
        x[i] = e;
        if (cx.row_ok && c0 + i < cx.N) {
          cx.resid = nonneg_max(cx.resid, fabsf(e - d));
          cx.amax = nonneg_max(cx.amax, fabsf(e));
        }
      }
      store_split32(jb.c_hi, jb.c_plane, jb.c_ld, r, c0, cx.M, cx.N, x, cx.inv_out, cx.ovf);
    } break;
    case EPI_EMA: {
      if (cx.row_ok) {
        const float* fi = jb.f_in + static_cast<long long>(r) * jb.f_ld + c0;
        float* fo = jb.f_out + static_cast<long long>(r) * jb.f_ld + c0;
        const float b = jb.beta, omb = 1.f - jb.beta;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < cx.N) fo[i] = b * fi[i] + omb * (x[i] * cx.sc);
      }
    } break;
    case EPI_APPLY: {
      if (cx.row_ok) {
        float* fo = jb.f_out + static_cast<long long>(r) * jb.f_ld + c0;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < cx.N) {
            const float u = x[i] * cx.sc;
            fo[i] = u;
            cx.sumsq += static_cast<double>(u) * u;
          }
      }
    } break;
    case EPI_CHEB:
    case EPI_CHEB_FINAL: {
      const bool fin = cx.op == EPI_CHEB_FINAL;
      const __half* sh = jb.s_hi + static_cast<long long>(r) * jb.s_ld + c0;
      const __half* sl = sh + jb.s_plane;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        float sv = 0.f;
        if (cx.row_ok && c0 + i < cx.N) sv = (__half2float(sh[i]) + __half2float(sl[i])) * cx.side_scale;
        const float d = (r == c0 + i) ? cx.gam : 0.f;
        const float y = fin ? (x[i] * cx.sc - sv + d) * cx.mul : 2.f * (x[i] * cx.sc) - sv + d;
        x[i] = y;
        if (cx.row_ok && c0 + i < cx.N) cx.amax = nonneg_max(cx.amax, fabsf(y));
      }
      if (jb.c_hi) store_split32(jb.c_hi, jb.c_plane, jb.c_ld, r, c0, cx.M, cx.N, x, cx.inv_out, cx.ovf);
      if (jb.f_out && cx.row_ok) {
        float* fo = jb.f_out + static_cast<long long>(r) * jb.f_ld + c0;
#pragma unroll
        for (int i = 0; i < 32; ++i) if (c0 + i < cx.N) fo[i] = x[i];
      }
    } break;
    case EPI_CN_M: {
      float cc[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
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
      store_split32(jb.c_hi, jb.c_plane, jb.c_ld, r, c0, cx.M, cx.N, x, cx.inv_out, cx.ovf);
      store_split32(jb.c2_hi, jb.c2_plane, jb.c_ld, r, c0, cx.M, cx.N, cc, cx.inv_e, cx.ovf2);
    } break;
    default: break;
  }
}

template <int PASSES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    dash_gemm2_kernel(const GemmJob* __restrict__ jobs, int njobs, int total_tiles,
                      const CUtensorMap* __restrict__ maps, const int* __restrict__ gate, int nacc_in, int uniform) {
  using C = Gemm2Cfg<PASSES>;
  const uint32_t nacc = static_cast<uint32_t>(nacc_in);      // accumulators per tile (1, 2 or 4)
  const uint32_t nsets = kAccBufs / nacc;                     // tiles in flight in TMEM

  if (gate && *gate == 0) return;  // uniform across the grid (and thus across each pair)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + kAccBufs;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + kAccBufs);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();  // 0 = leader (issues the pair MMAs)
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);   // leader's arrive_expect_tx (both CTAs' TMA bytes land here)
      mbar_init(&empty[s], 1);  // pair-MMA commit (multicast to both CTAs)
    }
    for (int a = 0; a < kAccBufs; ++a) {
      mbar_init(&tfull[a], 1);                // pair-MMA commit (multicast)
      mbar_init(&tempty[a], 2 * kEpiWarps);   // every epilogue warp of both CTAs (leader's copy used)
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc2<kAccBufs * kPairN>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer (both CTAs)
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = pair; tile < total_tiles; tile += npairs) {
        const GemmJob& jb = jobs[find_job(jobs, njobs, tile, uniform)];
        const int local = tile - jb.tile_start;
        const int am = (local / jb.tiles_n) * kPairM + kHalf * static_cast<int>(rank);
        const int bn = (local % jb.tiles_n) * kPairN + kHalfN * static_cast<int>(rank);
        const int nk = (jb.K + kTileK - 1) / kTileK;
        const CUtensorMap* amap = maps + jb.a_map;
        const CUtensorMap* bmap = maps + jb.b_map;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * C::kStageBytes);
          uint8_t* sA = smem + stage * C::kStageBytes;
          uint8_t* sB = sA + C::kABytes * C::kPlanes;
          const int k0 = kb * kTileK;
#pragma unroll
          for (int p = 0; p < C::kPlanes; ++p) {
            uint8_t* a_dst = sA + p * C::kABytes;
            uint8_t* b_dst = sB + p * C::kBBytes;
            if (!jb.a_mn) {
              tma2_load_4d(a_dst, amap, &full[stage], k0, am, p, jb.a_mat);
            } else {
              tma2_load_4d(a_dst, amap, &full[stage], am, k0, p, jb.a_mat);
              tma2_load_4d(a_dst + 8192, amap, &full[stage], am + 64, k0, p, jb.a_mat);
            }
            if (!jb.b_mn) tma2_load_4d(b_dst, bmap, &full[stage], k0, bn, p, jb.b_mat);
            else tma2_load_4d(b_dst, bmap, &full[stage], bn, k0, p, jb.b_mat);
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (leader CTA only)
    // k-block kb of a tile accumulates into accumulator (kb % nacc) of the tile's buffer set; the
    // accumulators are summed in fp32 by the epilogue, so each one holds only K / nacc of the sum.
    if (rank == 0 && elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t t = 0;
      for (int tile = pair; tile < total_tiles; tile += npairs, ++t) {
        const GemmJob& jb = jobs[find_job(jobs, njobs, tile, uniform)];
        const int nk = (jb.K + kTileK - 1) / kTileK;
        const uint32_t idesc = umma_idesc_f16(kPairM, kPairN, jb.a_mn, jb.b_mn);
        const uint32_t a_lbo = jb.a_mn ? 8192u : 16u, b_lbo = jb.b_mn ? 8192u : 16u;
        const uint32_t a_kstep = jb.a_mn ? 2048u : 32u, b_kstep = jb.b_mn ? 2048u : 32u;
        const uint32_t set = t % nsets;
        mbar_wait(&tempty[set], ((t / nsets) & 1u) ^ 1u);
        tc_fence_after();
        for (int kb = 0; kb < nk; ++kb) {
          const uint32_t d_tmem = tmem_base + (set * nacc + static_cast<uint32_t>(kb % nacc)) * kPairN;
          const bool first = kb < nacc;
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem + stage * C::kStageBytes);
          const uint32_t b_base = a_base + C::kABytes * C::kPlanes;
#pragma unroll
          for (int k = 0; k < kTileK / 16; ++k) {
#pragma unroll
            for (int p = 0; p < PASSES; ++p) {
              const uint32_t ap = (p == 2) ? 1u : 0u;  // pass 2: A_lo * B_hi
              const uint32_t bp = (p == 1) ? 1u : 0u;  // pass 1: A_hi * B_lo
              const uint64_t ad = umma_sdesc(a_base + ap * C::kABytes + k * a_kstep, a_lbo, 1024);
              const uint64_t bd = umma_sdesc(b_base + bp * C::kBBytes + k * b_kstep, b_lbo, 1024);
              umma2_f16(d_tmem, ad, bd, idesc, (first && k == 0 && p == 0) ? 0u : 1u);
            }
          }
          umma2_commit_mc(&empty[stage]);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
        umma2_commit_mc(&tfull[set]);
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2..9, both CTAs)
    const int q = warp & 3;  // TMEM lane quarter of this warp (warps 2..5 -> 2, 3, 0, 1)
    const int half = 0;
    const uint32_t leader_tempty = mapa_shared(smem_u32(tempty), 0);
    uint32_t t = 0;
    for (int tile = pair; tile < total_tiles; tile += npairs, ++t) {
      const GemmJob& jb = jobs[find_job(jobs, njobs, tile, uniform)];
      const int local = tile - jb.tile_start;
      const int m0 = (local / jb.tiles_n) * kPairM;
      const int n0 = (local % jb.tiles_n) * kPairN;
      const int nk = (jb.K + kTileK - 1) / kTileK;
      const uint32_t set = t % nsets;
      const int used = nk < static_cast<int>(nacc) ? nk : static_cast<int>(nacc);
      float acc[128];
      mbar_wait(&tfull[set], (t / nsets) & 1u);
      tc_fence_after();
      for (int c = 0; c < used; ++c) {
        const uint32_t taddr =
            tmem_base + (static_cast<uint32_t>(q * 32) << 16) + (set * nacc + static_cast<uint32_t>(c)) * kPairN;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float v[32];
          tmem_ld32(taddr + 32 * j, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[32 * j + i] = (c == 0) ? v[i] : acc[32 * j + i] + v[i];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(leader_tempty + set * 8);
      // ---- fused epilogue on the fp32 sums
      EpiCtx cx;
      cx.op = jb.op;
      cx.mat = jb.out_mat;
      cx.r = m0 + kHalf * static_cast<int>(rank) + q * 32 + static_cast<int>(lane);
      cx.M = jb.M;
      cx.N = jb.N;
      cx.row_ok = cx.r < jb.M;
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
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c0 = n0 + kHalf * half + 32 * j;
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = acc[32 * j + i];
        if (c0 < jb.N) epi_piece(jb, cx, c0, v);
      }
      // per-matrix reductions (max is order independent -> deterministic)
      float am = cx.ovf ? __uint_as_float(0x7fc00000u) : cx.amax;
      float am2 = cx.ovf2 ? __uint_as_float(0x7fc00000u) : cx.amax2;
      float rs = cx.resid;
      am = warp_max_nonneg(am);
      am2 = warp_max_nonneg(am2);
      rs = warp_max_nonneg(rs);
      (void)half;
      if (lane == 0) {
        if (jb.c_amax) atomic_max_nonneg(jb.c_amax, am);
        if (jb.c2_amax) atomic_max_nonneg(jb.c2_amax, am2);
        if (jb.resid && !cx.inactive)
          atomic_max_nonneg(jb.resid + cx.mat, (cx.op == EPI_NDB_E || cx.op == EPI_CN_M) && cx.ovf
                                                   ? __uint_as_float(0x7fc00000u) : rs);
      }
      if (cx.op == EPI_APPLY) {
        const double sacc = warp_sum_d(cx.sumsq);
        if (lane == 0) jb.partial[local * kPartialsPerTile + rank * 4 + q] = static_cast<float>(sacc);
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();  // no CTA of the pair may exit while its peer still uses its TMEM / barriers
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2<kAccBufs * kPairN>(tmem_base);
  }
}

// ---------------------------------------------------------------------------- host launcher
static int g_num_sms = 0;
static int g_nacc = 0;
static int g_dbg = -1;

// Launch accounting + optional CUDA-event timing of every GEMM launch (bench / roofline hooks).
struct GemmTimer {
  bool on = false;
  std::vector<cudaEvent_t> ev;  // start/stop pairs
  std::vector<double> flops;
  size_t used = 0;
};
static GemmTimer g_timer;
unsigned long long g_launches = 0;

void note_launch(int n) { g_launches += static_cast<unsigned long long>(n); }

int gemm_launch(const GemmJob* d_jobs, int njobs, int total_tiles, const CUtensorMap* d_maps, int passes,
                cudaStream_t stream, const int* gate, double flops, int uniform) {
  if (total_tiles <= 0) return 0;
  ++g_launches;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
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
    cudaEventRecord(e0, stream);
  }
  if (g_dbg < 0) {
    const char* e = getenv("DASH_GEMM_DEBUG");
    g_dbg = e ? atoi(e) : 0;
  }
  if (g_nacc == 0) {
    const char* e = getenv("DASH_NACC");
    g_nacc = e ? atoi(e) : kNaccDefault;
    if (g_nacc != 1 && g_nacc != 2 && g_nacc != 4) g_nacc = kNaccDefault;
  }
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = total_tiles < g_num_sms ? total_tiles : g_num_sms;
  cudaError_t err;
  const int grid2 = 2 * (total_tiles < g_num_sms / 2 ? total_tiles : g_num_sms / 2);  // CTA pairs
  (void)grid;
  if (passes == 3) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(dash_gemm2_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, Gemm2Cfg<3>::kSmemBytes);
      attr = true;
    }
    dash_gemm2_kernel<3><<<grid2, kThreads2, Gemm2Cfg<3>::kSmemBytes, stream>>>(d_jobs, njobs, total_tiles, d_maps,
                                                                                gate, g_nacc, uniform);
  } else {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(dash_gemm2_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, Gemm2Cfg<1>::kSmemBytes);
      attr = true;
    }
    dash_gemm2_kernel<1><<<grid2, kThreads2, Gemm2Cfg<1>::kSmemBytes, stream>>>(d_jobs, njobs, total_tiles, d_maps,
                                                                                gate, 1, uniform);
  }
  if (e1) cudaEventRecord(e1, stream);
  err = cudaGetLastError();
  return err == cudaSuccess ? 0 : 3;
}

void gemm_timing_enable(int on) {
  g_timer.on = on != 0;
  g_timer.used = 0;
  g_timer.flops.clear();
}

// Synchronises on the recorded events; returns launches timed, total ms and total algorithmic flops.
int gemm_timing_read(int* n, double* ms, double* flops) {
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
