// Pooled power iteration on the tensor cores (spectral.py:67-117).
//
// One cluster of C = d / 128 CTAs per two blocks (d in {128, ..., 1024}).  CTA q owns rows [128q, 128q + 128) of
// the solver input a = ema + eps I (the Newton solver's split-f16 stack) of both blocks and keeps each block's
// pool V (d x 16, fp16) in shared memory as the K-major B operand of tcgen05.mma (M = 128 rows, N = 16 pool
// vectors, K = d).  The producer warp streams the CTA's A slabs through one 5-stage ring of 32-wide K blocks
// (64-byte swizzle; the blocks stay L2-resident across the 31 passes), alternating the two blocks pass by
// pass, and the MMA warp alternates with it: while one block's row warps exchange its pool across the cluster,
// the tensor cores run the other block's pass, so the per-pass cluster round trip is hidden behind work.
//
// Precision: passes 1..iters multiply the fp16 (hi) plane of a by the fp16 pool (one MMA per 16-wide k step;
// the power iteration only needs the direction); the last pass -- the one whose products give the Rayleigh
// quotients -- multiplies the full split a (hi + lo planes, main + correction accumulators), and the quotient
// is evaluated for exactly the stored pool vector, so lambda is the Rayleigh quotient v^T a v / v^T v of a
// vector within fp16 rounding of the reference's (second-order error in lambda).
//
// One cluster exchange per iteration: every CTA publishes W / s with the fixed bound s = sqrt(d) max|a| (|W_i| <=
// |a_i|_2 |v|_2, so the stored pool stays inside the fp16 range) together with its partial sums of W^2; one bulk
// shared::cluster copy per peer carries both.  After the exchange every CTA knows |W|_2 exactly and applies
// f = s / |W|_2 per column to the next product, so the pool it multiplies is the reference's normalised
// v = W / |W| (zero columns stay zero).  Pools and partials are double-buffered by exchange parity per block.
// Start vectors are the NumPy PCG64 streams (rng.cuh).  A collapsed pool is flagged (status 3) and re-run by the
// fp32 cluster kernel (step.cu), which implements the zero-matrix answer and the reseeded retry.
#include <cuda.h>
#include <cstdlib>
#include <mutex>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "engine.h"
#include "ptx.cuh"
#include "rng.cuh"

namespace dash {

constexpr int kPtStages = 5;
constexpr int kPtSlots = 2;                     // blocks interleaved per cluster
constexpr int kPtThreads = 64 + 128 * kPtSlots; // warp 0 TMA producer, warp 1 MMA, 4 row warps per slot
constexpr int kPtPool = 16;
constexpr int kPtKB = 32;                       // K block of the A ring (64-byte swizzle)
constexpr int kPtAPlane = 128 * kPtKB * 2;      // 8 KB: one plane of a 128 x 32 A tile
constexpr int kPtAStage = 2 * kPtAPlane;        // 16 KB (hi plane; + lo plane in the final pass)
constexpr int kPtVkb = kPtPool * 128;           // 2 KB: [16 rows][128 B] of V^T (fp16) for one 64-wide k-block
constexpr int kVExp = -14;                      // |stored v| <= 1 -> v * 2^14 < 2^15
constexpr int kPiRetry = 3;                     // status: pool collapsed, re-run by the reference-exact kernel
#ifndef PT_SLEEPY_WAIT
#define PT_WAIT mbar_wait_spin  // the per-pass handoffs are latency-critical: spin, do not suspend
#else
#define PT_WAIT mbar_wait
#endif

struct PtLayout {
  int d, nkb;
  size_t v_off, vbuf_bytes, pn_off, dbl_off, bar_off, bytes;
  __host__ __device__ explicit PtLayout(int d_) : d(d_), nkb(d_ / 64) {
    v_off = static_cast<size_t>(kPtStages) * kPtAStage;
    vbuf_bytes = static_cast<size_t>(nkb) * kPtVkb;                      // one pool buffer (32 KB at d = 1024)
    pn_off = v_off + static_cast<size_t>(kPtSlots) * 2 * vbuf_bytes;     // [slot][2 parity][8 ranks][16] doubles
    dbl_off = pn_off + sizeof(double) * kPtSlots * 2 * 8 * kPtPool;      // [slot][4 warps][2][16] doubles
    bar_off = dbl_off + sizeof(double) * kPtSlots * 4 * 2 * kPtPool;
    bytes = bar_off + 512 + 1024;  // barriers + alignment slack
  }
};

// TMA tile load with an L2 cache policy (the hi plane of a is re-read every pass: evict-last; the quotient pass
// reads it for the last time: evict-first)
__device__ __forceinline__ void pt_load_4d(void* smem_dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2,
                                           int c3, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void bulk_copy_to_peer(uint32_t dst_cluster, const void* src, uint32_t bytes,
                                                  uint32_t bar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst_cluster),
               "r"(smem_u32(src)), "r"(bytes), "r"(bar_cluster)
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// named barrier of one slot's 128 row threads (ids 1, 2)
__device__ __forceinline__ void rows_sync(int slot) {
  asm volatile("bar.sync %0, 128;" ::"r"(1 + slot) : "memory");
}

// Cluster-wide fixed-order sums of nv x 16 per-row values (rows = the 128 threads of one slot's row warps):
// lanes -> warp (shuffle butterfly), warps 0..3 in order, then ranks 0..C-1 in order.  Lane j < 16 of row warp 0
// writes its sum into slot[par][q] of every CTA and arrives (relaxed, after one cluster fence) on that CTA's
// red[par] (16 C arrivals per phase).  `par` alternates slot buffers and barriers between consecutive sums.
__device__ void pt_cluster_sum(const double (&x)[2][kPtPool], int nv, double* wpart, double* slots, uint64_t* red,
                               int par, uint32_t& red_phase, int C, int q, int rw, int lane, int slot,
                               double (&out)[2][kPtPool]) {
  rows_sync(slot);  // the previous reduction's reader of wpart is done
  for (int s = 0; s < nv; ++s)
#pragma unroll
    for (int j = 0; j < kPtPool; ++j) {
      double t = x[s][j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) wpart[(rw * 2 + s) * kPtPool + j] = t;
    }
  rows_sync(slot);
  double* my = slots + static_cast<size_t>(par) * 8 * 2 * kPtPool;
  if (rw == 0 && lane < kPtPool) {
    double t[2] = {0.0, 0.0};
    for (int s = 0; s < nv; ++s)
      for (int w = 0; w < 4; ++w) t[s] += wpart[(w * 2 + s) * kPtPool + lane];
    for (int dst = 0; dst < C; ++dst)
      for (int s = 0; s < nv; ++s) {
        const uint32_t ra = mapa_shared(smem_u32(my + (q * 2 + s) * kPtPool + lane), static_cast<uint32_t>(dst));
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(t[s]) : "memory");
      }
    asm volatile("fence.acq_rel.cluster;" ::: "memory");  // one fence for all C destinations, then relaxed arrives
    for (int dst = 0; dst < C; ++dst)
      mbar_arrive_remote_relaxed(mapa_shared(smem_u32(&red[par]), static_cast<uint32_t>(dst)));
  }
  mbar_wait_cluster(&red[par], (red_phase >> par) & 1u);
  red_phase ^= 1u << par;
  for (int s = 0; s < nv; ++s)
#pragma unroll
    for (int j = 0; j < kPtPool; ++j) {
      double t = 0.0;
      for (int r = 0; r < C; ++r) t += my[(r * 2 + s) * kPtPool + j];
      out[s][j] = t;
    }
}

// Element (n, k) of V^T (pool vector n, row k) in the 128-byte-swizzled K-major operand layout (fp16).
__device__ __forceinline__ uint32_t pt_v_off(int n, int k) {
  const int kb = k >> 6, kk = k & 63;
  return kb * kPtVkb + (n >> 3) * 1024 + (n & 7) * 128 + ((((kk >> 3) ^ (n & 7))) << 4) + (kk & 7) * 2;
}

// Intra-CTA fixed-order column sums of w^2 over the 128 rows (warp shuffles, then warps 0..3 in order); valid in
// lanes 0..15 of row warp 0 (lane j holds column j).
__device__ __forceinline__ double pt_cta_colsum(const float (&w)[kPtPool], double* wpart, int rw, int lane, int slot) {
  rows_sync(slot);  // previous users of wpart are done
  // transpose-reduce: at offset o the lane pair (l, l ^ o) splits its remaining columns in halves, each lane
  // keeps one half and adds the partner's copy of it (16 + 8 + 4 + 2 + 1 values; fixed order)
  double t[kPtPool];
#pragma unroll
  for (int j = 0; j < kPtPool; ++j) t[j] = static_cast<double>(w[j]) * w[j];
  int col = 0;
#pragma unroll
  for (int o = 16, n = kPtPool / 2; o > 1; o >>= 1, n >>= 1) {
    const bool hi = (lane & o) != 0;
#pragma unroll
    for (int j = 0; j < n; ++j) {
      const double send = hi ? t[j] : t[j + n];
      const double keep = hi ? t[j + n] : t[j];
      t[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
    col += hi ? n : 0;
  }
  t[0] += __shfl_xor_sync(0xffffffffu, t[0], 1);  // lanes l, l ^ 1 now both hold column `col`
  if ((lane & 1) == 0) wpart[rw * kPtPool + col] = t[0];
  rows_sync(slot);
  double sum = 0.0;
  if (rw == 0 && lane < kPtPool)
    for (int w4 = 0; w4 < 4; ++w4) sum += wpart[w4 * kPtPool + lane];
  return sum;
}

// Pooled power iteration on the tensor cores, two blocks interleaved per cluster (file header).  Passes
// 0..iters-1 multiply the fp16 (hi) plane of a by the fp16 pool (one MMA per 16-wide k step); the final pass,
// whose products give the Rayleigh quotients, multiplies the full split a (hi and lo planes, two MMAs) by the
// same stored pool, and the quotient is evaluated for exactly that stored vector: lambda = v^T a v / v^T v.
__global__ void __launch_bounds__(kPtThreads, 1)
    pi_tc_kernel(const __grid_constant__ CUtensorMap amap, dash_stack a, int pool, int iters, unsigned long long seed,
                 float* __restrict__ scale, float* __restrict__ inv_scale, int* __restrict__ status,
                 const int* __restrict__ seed_index) {
  const int d = a.rows;
  const PtLayout L(d);
  const int C = d / 128;
  const int q = static_cast<int>(cluster_rank());
  const int cluster = blockIdx.x / C;
  const int row0 = q * 128;
  int mblk[kPtSlots];
#pragma unroll
  for (int s = 0; s < kPtSlots; ++s) mblk[s] = cluster * kPtSlots + s < a.nmat ? cluster * kPtSlots + s : -1;
  extern __shared__ uint8_t pt_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(pt_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* empty = full + kPtStages;
  uint64_t* tfull = empty + kPtStages;  // [slot]
  uint64_t* vbar = tfull + kPtSlots;    // [slot]
  uint64_t* red = vbar + kPtSlots;      // [slot][2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red + 2 * kPtSlots);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPtStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kPtSlots; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&vbar[s], 1);
      mbar_init(&red[2 * s], kPtPool * C);
      mbar_init(&red[2 * s + 1], kPtPool * C);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<32 * kPtSlots>(tmem_slot);
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nkb = d / kPtKB;  // 32-wide A blocks per pass (a multiple of 4)

  if (warp == 0) {
    // ---------------------------------------------------------------- A slab producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t keep = l2_policy_evict_last(), drop = l2_policy_evict_first();
      for (int it = 0; it <= iters; ++it) {
        const bool fin = it == iters;
        for (int s = 0; s < kPtSlots; ++s) {
          if (mblk[s] < 0) continue;
          // a stage holds two 32-wide k blocks of the hi plane (passes 1..iters) or the hi + lo planes of one
          // k block (the quotient pass): 16 KB per stage either way, 80 KB in flight
          for (int i = 0; i < (fin ? nkb : nkb / 2); ++i) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], kPtAStage);
            uint8_t* dst = smem + stage * kPtAStage;
            if (fin) {
              pt_load_4d(dst, &amap, &full[stage], i * kPtKB, row0, 0, mblk[s], drop);
              pt_load_4d(dst + kPtAPlane, &amap, &full[stage], i * kPtKB, row0, 1, mblk[s], drop);
            } else {
              pt_load_4d(dst, &amap, &full[stage], 2 * i * kPtKB, row0, 0, mblk[s], keep);
              pt_load_4d(dst + kPtAPlane, &amap, &full[stage], (2 * i + 1) * kPtKB, row0, 0, mblk[s], keep);
            }
            if (++stage == kPtStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (whole warp, elected lane)
    const uint32_t idesc = umma_idesc_f16(128, kPtPool, 0, 0);
    int stage = 0;
    uint32_t phase = 0, vphase = 0;
    for (int it = 0; it <= iters; ++it) {
      const bool fin = it == iters;
      for (int s = 0; s < kPtSlots; ++s) {
        if (mblk[s] < 0) continue;
        PT_WAIT(&vbar[s], (vphase >> s) & 1u);
        vphase ^= 1u << s;
        tc_fence_after();
        const uint8_t* vcur = smem + L.v_off + (static_cast<size_t>(s) * 2 + (it & 1)) * L.vbuf_bytes;
        const uint32_t acc = tmem + 32u * s;
        for (int i = 0; i < (fin ? nkb : nkb / 2); ++i) {
          PT_WAIT(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem + stage * kPtAStage);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            // quotient pass: half h = plane (hi -> main, lo -> correction accumulator) of k block i;
            // other passes: half h = hi plane of k block 2 i + h, all into the main accumulator
            const int kb = fin ? i : 2 * i + h;
            const uint32_t v_base = smem_u32(vcur + (kb >> 1) * kPtVkb) + (kb & 1) * 64;  // 32 of 64 k columns
#pragma unroll
            for (int k = 0; k < kPtKB / 16; ++k) {
              const uint64_t ad = umma_sdesc(a_base + h * kPtAPlane + k * 32, 16, 512, 4);  // 64-byte swizzle
              const uint64_t bd = umma_sdesc(v_base + k * 32, 16, 1024);
              const uint32_t fresh = (i == 0 && k == 0 && (fin || h == 0)) ? 0u : 1u;
              const uint32_t d_acc = acc + ((fin && h) ? 16u : 0u);
              asm volatile(
                  "{\n\t.reg .pred pp, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 pp, %4, 0;\n\t"
                  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, pp;\n\t}\n" ::"r"(d_acc),
                  "l"(ad), "l"(bd), "r"(idesc), "r"(fresh));
            }
          }
          asm volatile(
              "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
                  smem_u32(&empty[stage]))
              : "memory");
          if (++stage == kPtStages) { stage = 0; phase ^= 1; }
        }
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
                smem_u32(&tfull[s]))
            : "memory");
      }
    }
  } else {
    // ---------------------------------------------------------------- row warps of one slot: start vectors,
    // norms, pool exchange, quotients
    const int slot = (static_cast<int>(warp) - 2) / 4;
    const int rw = (static_cast<int>(warp) - 2) % 4;            // 0..3 (order of the fixed reductions)
    const int m = mblk[slot];
    if (m >= 0) {
      const int row = 32 * static_cast<int>(warp & 3) + static_cast<int>(lane);  // TMEM lane = CTA row
      const int kg = row0 + row;                                // global row = K index of V
      const uint32_t taddr = tmem + 32u * slot + (static_cast<uint32_t>(32 * (warp & 3)) << 16);
      uint8_t* vsm = smem + L.v_off + static_cast<size_t>(slot) * 2 * L.vbuf_bytes;  // [2 parity][nkb][16][128 B]
      double* pn = reinterpret_cast<double*>(smem + L.pn_off) + slot * 2 * 8 * kPtPool;
      double* wpart = reinterpret_cast<double*>(smem + L.dbl_off) + slot * 4 * 2 * kPtPool;
      uint64_t* my_red = red + 2 * slot;
      const float sa = ldexpf(1.f, __ldg(a.exp + m) + kVExp);
      const float amax_a = __uint_as_float(__ldg(a.amax + m));
      // |W_i| <= |a_i|_2 <= sqrt(d) max|a| <= sfix, a power of two: the stored pool W / sfix is an exact scaling
      const double sfix =
          amax_a > 0.f ? ldexp(1.0, ilogb(sqrt(static_cast<double>(d)) * static_cast<double>(amax_a)) + 1) : 1.0;
      const float inv_sfix = static_cast<float>(1.0 / sfix);
      const int sidx = seed_index ? seed_index[m] : m;
      const uint64_t bseed = sidx < 0 ? static_cast<uint64_t>(seed) : rng::block_seed(seed, static_cast<uint64_t>(sidx));
      const uint32_t vbar_peer0 = smem_u32(&vbar[slot]);
      const uint32_t my_slice = static_cast<uint32_t>(row0 / 64) * kPtVkb;  // my 2 k-blocks (4 KB) of a pool buffer
      int par = 0;
      uint32_t tphase = 0, red_phase = 0, vphase = 0, ex = 0;
      float v[kPtPool];   // my row of the true pool of the current pass (the stored fp16 value times f)
      float vs[kPtPool];  // my row of the stored pool, fp16-rounded (true pool = vs * f)

      // store my row (fp16, fixed exponent) + my partial sums into pool / partial buffer `ex & 1` and push both
      // to every peer (one exchange; completes vbar there together with everyone else's pushes)
      auto publish = [&](double partial) {
        const float inv = ldexpf(1.f, -kVExp);
        uint8_t* vb = vsm + (ex & 1) * L.vbuf_bytes;
        __half* vh = reinterpret_cast<__half*>(vb);
#pragma unroll
        for (int n = 0; n < kPtPool; ++n) {
          const __half h = __float2half_rn(vs[n] * inv);
          vh[pt_v_off(n, kg) / 2] = h;
          vs[n] = __half2float(h) * ldexpf(1.f, kVExp);  // the value the tensor cores multiply
        }
        double* pslot = pn + ((ex & 1) * 8 + q) * kPtPool;
        if (rw == 0 && lane < kPtPool) pslot[lane] = partial;
        fence_proxy_async_smem();
        rows_sync(slot);
        if (rw == 0 && lane == 0) {
          mbar_arrive_expect_tx(&vbar[slot], static_cast<uint32_t>(C - 1) * (2 * kPtVkb + kPtPool * 8));
          for (int dst = 0; dst < C; ++dst) {
            if (dst == q) continue;
            const uint32_t pb = mapa_shared(vbar_peer0, static_cast<uint32_t>(dst));
            bulk_copy_to_peer(mapa_shared(smem_u32(vb) + my_slice, static_cast<uint32_t>(dst)), vb + my_slice,
                              2 * kPtVkb, pb);
            bulk_copy_to_peer(mapa_shared(smem_u32(pslot), static_cast<uint32_t>(dst)), pslot, kPtPool * 8, pb);
          }
        }
        ++ex;
      };

      // ---- start vectors: element (j, i) of the pool is draw j*d + i of default_rng(bseed) (spectral.py:67-74)
      double x[2][kPtPool], tot[2][kPtPool];
      {
        rng::Pcg64 g;  // seeded once; draw j*d + kg for pool vector j (one draw, then d - 1 steps ahead)
        g.seed(bseed);
        g.advance(static_cast<uint64_t>(kg));
#pragma unroll
        for (int j = 0; j < kPtPool; ++j) {
          float w0 = 0.f;
          if (j < pool) {
            w0 = static_cast<float>(g.uniform_pm1());
            if (j + 1 < pool) g.advance(static_cast<uint64_t>(d) - 1);
          }
          v[j] = w0;
          x[0][j] = static_cast<double>(w0) * w0;
        }
      }
      // the start reduction borrows the pool buffer of parity 1 (first written by the second exchange)
      pt_cluster_sum(x, 1, wpart, reinterpret_cast<double*>(vsm + L.vbuf_bytes), my_red, par, red_phase, C, q, rw,
                     static_cast<int>(lane), slot, tot);
      par ^= 1;
#pragma unroll
      for (int j = 0; j < kPtPool; ++j) {
        double n = sqrt(tot[0][j]);
        if (n == 0.0) n = 1.0;
        vs[j] = static_cast<float>(v[j] / n);  // stored = true pool (|v| <= 1) for the first pass
      }
      publish(0.0);
      float f[kPtPool];
#pragma unroll
      for (int j = 0; j < kPtPool; ++j) f[j] = 1.f;
      for (int it = 0; it <= iters; ++it) {
        // ---- the pool of this pass has been exchanged: its column scale f (pass >= 1) from the partials
        PT_WAIT(&vbar[slot], vphase);
        vphase ^= 1;
        if (it > 0) {
          const double* pp = pn + ((ex - 1) & 1) * 8 * kPtPool;
          float fl = 0.f;  // lane j < 16: the scale of pool column j, then broadcast
          if (lane < kPtPool) {
            double nsq = 0.0;
            for (int r = 0; r < C; ++r) nsq += pp[r * kPtPool + lane];  // ranks in order
            const double nn = sqrt(nsq);
            fl = nn > 0.0 ? static_cast<float>(sfix / nn) : 0.f;
          }
#pragma unroll
          for (int j = 0; j < kPtPool; ++j) f[j] = __shfl_sync(0xffffffffu, fl, j);
        }
#pragma unroll
        for (int j = 0; j < kPtPool; ++j) v[j] = vs[j] * f[j];
        // ---- W = a v for my row: (a vs) * f (the lo-plane accumulator only in the final pass)
        PT_WAIT(&tfull[slot], tphase);
        tphase ^= 1;
        tc_fence_after();
        float mn[kPtPool], cr[kPtPool], w[kPtPool];
        tmem_ld16(taddr, mn);
        if (it == iters) {
          tmem_ld16(taddr + 16, cr);
        } else {
#pragma unroll
          for (int j = 0; j < kPtPool; ++j) cr[j] = 0.f;
        }
        tc_fence_before();
#pragma unroll
        for (int j = 0; j < kPtPool; ++j) w[j] = (mn[j] + cr[j]) * sa * f[j];
        if (it < iters) {
          const double partial = pt_cta_colsum(w, wpart, rw, static_cast<int>(lane), slot);
#pragma unroll
          for (int j = 0; j < kPtPool; ++j) vs[j] = w[j] * inv_sfix;  // exact (power-of-two scale)
          publish(partial);
        } else {
#pragma unroll
          for (int j = 0; j < kPtPool; ++j) {
            x[0][j] = static_cast<double>(v[j]) * w[j];
            x[1][j] = static_cast<double>(v[j]) * v[j];
          }
          // the final reduction borrows the pool buffer that no MMA reads any more
          pt_cluster_sum(x, 2, wpart, reinterpret_cast<double*>(vsm + (ex & 1) * L.vbuf_bytes), my_red, par,
                         red_phase, C, q, rw, static_cast<int>(lane), slot, tot);
          par ^= 1;
        }
      }
      // ---- selection by Rayleigh quotient q_j / |v_j|^2 (spectral.py:104-112)
      double bq = 0.0;
      bool any = false;
      for (int j = 0; j < pool; ++j) {
        if (tot[1][j] > 0.0) {
          const double r = tot[0][j] / tot[1][j];
          if (!any || r > bq) bq = r;
          any = true;
        }
      }
      if (q == 0 && rw == 0 && lane == 0) {
        const bool ok = any && bq != 0.0;
        const float s2 = ok ? 2.f * static_cast<float>(bq) : 0.f;
        scale[m] = s2;
        inv_scale[m] = s2 > 0.f ? 1.f / s2 : 0.f;
        // a collapsed pool (all columns dead or every quotient 0) is re-run by the reference-exact kernel, which
        // implements the zero-matrix answer and the reseeded retry (spectral.py:99-107)
        if (status) status[m] = ok ? (s2 > 0.f ? 0 : 1) : kPiRetry;
      }
    }
  }
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<32 * kPtSlots>(tmem);
  }
}

int pi_tc_launch(const dash_stack& a, int pool, int iters, unsigned long long seed, float* scale, float* inv_scale,
                 int* status, const int* seed_index, cudaStream_t st) {
  const int d = a.rows;
  if (d % 128 != 0 || d < 128 || d > 1024 || a.cols != d || pool > kPtPool || pool < 1 || iters < 1)
    return DASH_EINVAL;
  const int C = d / 128;
  CUtensorMap map;  // A slab tiles: 32 k x 128 rows, 64-byte swizzle
  if (!make_stack_map(a, 128, &map, kPtKB, 1, 64)) return DASH_ECUDA;
  const PtLayout L(d);
  static std::once_flag attr[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(attr[dev & 63], [] {
    cudaFuncSetAttribute(pi_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(PtLayout(1024).bytes));
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>((a.nmat + kPtSlots - 1) / kPtSlots * C));
  cfg.blockDim = dim3(kPtThreads);
  cfg.dynamicSmemBytes = L.bytes;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = C;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, pi_tc_kernel, map, a, pool, iters, seed, scale, inv_scale, status,
                                     seed_index);
  note_launch();
  return e == cudaSuccess ? DASH_OK : DASH_ECUDA;
}

}  // namespace dash

extern "C" int dash_power_iteration_split(const dash_stack* a, const float* ema, float eps, int pool, int iters,
                                          unsigned long long seed, float* scale, float* inv_scale, int* status,
                                          const int* seed_index, void* stream) {
  if (!dash::stack_ok(a) || !scale || !inv_scale || !status) return DASH_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = dash::pi_tc_launch(*a, pool, iters, seed, scale, inv_scale, status, seed_index, st)) return rc;
  // blocks whose pool collapsed (status 3) are re-run from scratch by the fp32 cluster kernel, which implements
  // the zero-matrix answer and the reseeded retry; every other cluster of that launch exits at once
  if (!ema) return DASH_OK;
  return dash::pi_retry_launch(ema, a->nmat, a->rows, eps, pool, iters, seed, scale, inv_scale, status, seed_index,
                               st);
}
