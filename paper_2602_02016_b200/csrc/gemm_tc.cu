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

#include <vector>

#include "ptx.cuh"
#include "types.h"

namespace dash {

template <int PASSES>
struct GemmCfg {
  static constexpr int kPlanes = PASSES == 3 ? 2 : 1;
  static constexpr int kABytes = kTileM * kTileK * 2;  // 16 KB per plane
  static constexpr int kBBytes = kTileN * kTileK * 2;  // 32 KB per plane
  static constexpr int kStageBytes = (kABytes + kBBytes) * kPlanes;
  static constexpr int kStages = PASSES == 3 ? 2 : 4;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;
};

__device__ __forceinline__ int find_job(const GemmJob* __restrict__ jobs, int njobs, int tile) {
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

template <int PASSES>
__global__ void __launch_bounds__(192, 1)
    dash_gemm_kernel(const GemmJob* __restrict__ jobs, int njobs, int total_tiles,
                     const CUtensorMap* __restrict__ maps, const int* __restrict__ gate) {
  using C = GemmCfg<PASSES>;
  if (gate && *gate == 0) return;  // nothing active (uniform across the grid)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const GemmJob& jb = jobs[find_job(jobs, njobs, tile)];
        const int local = tile - jb.tile_start;
        const int m0 = (local / jb.tiles_n) * kTileM;
        const int n0 = (local % jb.tiles_n) * kTileN;
        const int nk = (jb.K + kTileK - 1) / kTileK;
        const CUtensorMap* am = maps + jb.a_map;
        const CUtensorMap* bm = maps + jb.b_map;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
          uint8_t* sA = smem + stage * C::kStageBytes;
          uint8_t* sB = sA + C::kABytes * C::kPlanes;
          const int k0 = kb * kTileK;
#pragma unroll
          for (int p = 0; p < C::kPlanes; ++p) {
            uint8_t* a_dst = sA + p * C::kABytes;
            uint8_t* b_dst = sB + p * C::kBBytes;
            if (!jb.a_mn) {
              tma_load_4d(a_dst, am, &full[stage], k0, m0, p, jb.a_mat);
            } else {
              tma_load_4d(a_dst, am, &full[stage], m0, k0, p, jb.a_mat);
              tma_load_4d(a_dst + 8192, am, &full[stage], m0 + 64, k0, p, jb.a_mat);
            }
            if (!jb.b_mn) {
              tma_load_4d(b_dst, bm, &full[stage], k0, n0, p, jb.b_mat);
            } else {
#pragma unroll
              for (int j = 0; j < 4; ++j) tma_load_4d(b_dst + j * 8192, bm, &full[stage], n0 + 64 * j, k0, p, jb.b_mat);
            }
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int t = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++t) {
        const GemmJob& jb = jobs[find_job(jobs, njobs, tile)];
        const int nk = (jb.K + kTileK - 1) / kTileK;
        const uint32_t idesc = umma_idesc_f16(kTileM, kTileN, jb.a_mn, jb.b_mn);
        const uint32_t a_lbo = jb.a_mn ? 8192u : 16u;
        const uint32_t b_lbo = jb.b_mn ? 8192u : 16u;
        const uint32_t a_kstep = jb.a_mn ? 2048u : 32u;
        const uint32_t b_kstep = jb.b_mn ? 2048u : 32u;
        const int acc = t & 1;
        mbar_wait(&tempty[acc], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kTileN;
        for (int kb = 0; kb < nk; ++kb) {
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
              umma_f16(d_tmem, ad, bd, idesc, (kb | k | p) != 0);
            }
          }
          umma_commit(&empty[stage]);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2..5)
    const int q = warp & 3;  // TMEM lane quarter accessible by this warp
    int t = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++t) {
      const GemmJob& jb = jobs[find_job(jobs, njobs, tile)];
      const int local = tile - jb.tile_start;
      const int m0 = (local / jb.tiles_n) * kTileM;
      const int n0 = (local % jb.tiles_n) * kTileN;
      const int r = m0 + q * 32 + static_cast<int>(lane);
      const int op = jb.op;
      const int mat = jb.out_mat;
      // product scale: acc * 2^(ea + eb) is the true A*B entry
      const int ea = jb.a_exp ? __ldg(jb.a_exp) : 0;
      const int eb = jb.b_exp ? __ldg(jb.b_exp) : 0;
      const float sc = ldexpf(1.f, ea + eb);
      float mul = jb.alpha * (jb.alpha_p ? __ldg(jb.alpha_p + mat) : 1.f);
      const bool inactive = jb.active && __ldg(jb.active + mat) == 0;
      const float gam = jb.gamma_p ? *jb.gamma_p : jb.gamma;
      // output exponent
      const float prod_bound = static_cast<float>(jb.K) * amax_of(jb.a_amax) * amax_of(jb.b_amax);
      int e_out = 0, e_side = 0;
      float side_scale = 0.f;
      if (jb.s_hi) {
        e_side = __ldg(jb.s_exp);
        side_scale = ldexpf(1.f, e_side);
      }
      switch (op) {
        case EPI_SPLIT: e_out = exp_from_bound(prod_bound * fabsf(mul)); break;
        case EPI_NDB_E: e_out = kEExp; break;
        case EPI_CHEB:
          e_out = exp_from_bound(2.f * prod_bound + amax_of(jb.s_amax) + fabsf(gam));
          break;
        case EPI_CHEB_FINAL:
          e_out = exp_from_bound((prod_bound + amax_of(jb.s_amax) + fabsf(gam)) * fabsf(mul));
          break;
        case EPI_CN_M: e_out = exp_from_bound(prod_bound); break;
        default: break;
      }
      if (jb.c_exp && m0 == 0 && n0 == 0 && threadIdx.x == 64) *jb.c_exp = e_out;
      if (jb.c2_exp && m0 == 0 && n0 == 0 && threadIdx.x == 64) *jb.c2_exp = kEExp;
      const float inv_out = ldexpf(1.f, -e_out);
      const float inv_e = ldexpf(1.f, -kEExp);

      const int acc = t & 1;
      mbar_wait(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();

      float amax_loc = 0.f, amax2_loc = 0.f, resid_loc = 0.f;
      double sumsq = 0.0;
      bool ovf = false, ovf2 = false;
      const float cn_a = 1.f + 1.f / jb.beta;  // EPI_CN_M: beta carries p
      const float cn_b = 1.f / jb.beta;
#pragma unroll 1
      for (int j = 0; j < kTileN / 32; ++j) {
        const int c0 = n0 + 32 * j;
        if (c0 >= jb.N) break;  // warp-uniform
        float v[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * kTileN + 32 * j, v);
        const bool row_ok = r < jb.M;
        switch (op) {
          case EPI_SPLIT: {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              v[i] *= sc * mul;
              if (row_ok && c0 + i < jb.N) amax_loc = nonneg_max(amax_loc, fabsf(v[i]));
            }
            if (jb.c_hi) store_split32(jb.c_hi, jb.c_plane, jb.c_ld, r, c0, jb.M, jb.N, v, inv_out, ovf);
            if (jb.f_out && row_ok) {
              float* fo = jb.f_out + static_cast<long long>(r) * jb.f_ld + c0;
#pragma unroll
              for (int i = 0; i < 32; ++i) if (c0 + i < jb.N) fo[i] = v[i];
            }
          } break;
          case EPI_NDB_E: {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float d = (r == c0 + i) ? 1.f : 0.f;
              float e = 1.5f * d - 0.5f * (v[i] * sc);
              if (inactive) e = d;
              v[i] = e;
              if (row_ok && c0 + i < jb.N) {
                resid_loc = nonneg_max(resid_loc, fabsf(e - d));
                amax_loc = nonneg_max(amax_loc, fabsf(e));
              }
            }
            store_split32(jb.c_hi, jb.c_plane, jb.c_ld, r, c0, jb.M, jb.N, v, inv_out, ovf);
          } break;
          case EPI_EMA: {
            if (row_ok) {
              const float* fi = jb.f_in + static_cast<long long>(r) * jb.f_ld + c0;
              float* fo = jb.f_out + static_cast<long long>(r) * jb.f_ld + c0;
              const float b = jb.beta, omb = 1.f - jb.beta;
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (c0 + i < jb.N) fo[i] = b * fi[i] + omb * (v[i] * sc);
            }
          } break;
          case EPI_APPLY: {
            if (row_ok) {
              float* fo = jb.f_out + static_cast<long long>(r) * jb.f_ld + c0;
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (c0 + i < jb.N) {
                  const float u = v[i] * sc;
                  fo[i] = u;
                  sumsq += static_cast<double>(u) * u;
                }
            }
          } break;
          case EPI_CHEB:
          case EPI_CHEB_FINAL: {
            float s[32];
            load_split32(jb.s_hi, jb.s_plane, jb.s_ld, r, c0, jb.M, jb.N, side_scale, s);
            const bool fin = op == EPI_CHEB_FINAL;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float d = (r == c0 + i) ? gam : 0.f;
              float x = fin ? (v[i] * sc - s[i] + d) * mul : 2.f * (v[i] * sc) - s[i] + d;
              v[i] = x;
              if (row_ok && c0 + i < jb.N) amax_loc = nonneg_max(amax_loc, fabsf(x));
            }
            if (jb.c_hi) store_split32(jb.c_hi, jb.c_plane, jb.c_ld, r, c0, jb.M, jb.N, v, inv_out, ovf);
            if (jb.f_out && row_ok) {
              float* fo = jb.f_out + static_cast<long long>(r) * jb.f_ld + c0;
#pragma unroll
              for (int i = 0; i < 32; ++i) if (c0 + i < jb.N) fo[i] = v[i];
            }
          } break;
          case EPI_CN_M: {
            float cc[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float d = (r == c0 + i) ? 1.f : 0.f;
              const float m = v[i] * sc;
              v[i] = m;
              float c = cn_a * d - cn_b * m;
              if (inactive) c = d;
              cc[i] = c;
              if (row_ok && c0 + i < jb.N) {
                resid_loc = nonneg_max(resid_loc, fabsf(m - d));
                amax_loc = nonneg_max(amax_loc, fabsf(m));
                amax2_loc = nonneg_max(amax2_loc, fabsf(c));
              }
            }
            store_split32(jb.c_hi, jb.c_plane, jb.c_ld, r, c0, jb.M, jb.N, v, inv_out, ovf);
            store_split32(jb.c2_hi, jb.c2_plane, jb.c_ld, r, c0, jb.M, jb.N, cc, inv_e, ovf2);
          } break;
          default: break;
        }
      }
      // accumulator drained: hand TMEM back to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);

      // per-matrix reductions (max is order independent -> deterministic)
      if (ovf) amax_loc = __uint_as_float(0x7fc00000u);
      if (ovf2) amax2_loc = __uint_as_float(0x7fc00000u);
      amax_loc = warp_max_nonneg(amax_loc);
      amax2_loc = warp_max_nonneg(amax2_loc);
      resid_loc = warp_max_nonneg(resid_loc);
      if (lane == 0) {
        if (jb.c_amax) atomic_max_nonneg(jb.c_amax, amax_loc);
        if (jb.c2_amax) atomic_max_nonneg(jb.c2_amax, amax2_loc);
        if (jb.resid && !inactive) atomic_max_nonneg(jb.resid + mat, op == EPI_NDB_E || op == EPI_CN_M
                                                                          ? (ovf ? __uint_as_float(0x7fc00000u) : resid_loc)
                                                                          : resid_loc);
      }
      if (op == EPI_APPLY) {
        const double s = warp_sum_d(sumsq);
        if (lane == 0) jb.partial[local * 4 + q] = static_cast<float>(s);
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

// ---------------------------------------------------------------------------- host launcher
static int g_num_sms = 0;

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
                cudaStream_t stream, const int* gate, double flops) {
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
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = total_tiles < g_num_sms ? total_tiles : g_num_sms;
  cudaError_t err;
  if (passes == 3) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(dash_gemm_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<3>::kSmemBytes);
      attr = true;
    }
    dash_gemm_kernel<3><<<grid, 192, GemmCfg<3>::kSmemBytes, stream>>>(d_jobs, njobs, total_tiles, d_maps, gate);
  } else {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(dash_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<1>::kSmemBytes);
      attr = true;
    }
    dash_gemm_kernel<1><<<grid, 192, GemmCfg<1>::kSmemBytes, stream>>>(d_jobs, njobs, total_tiles, d_maps, gate);
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
