// Pooled power iteration on the tensor cores (spectral.py:67-117).
//
// One cluster of C = d / 128 CTAs per block (d in {128, ..., 1024}).  CTA q owns rows [128q, 128q + 128) of
// the solver input a = ema + eps I (already a split-f16 stack, the Newton solver's input) and keeps the pool
// V (d x 16, split f16) in shared memory as the K-major B operand of tcgen05.mma (M = 128 rows, N = 16 pool
// vectors, K = d, hi*hi + hi*lo + lo*hi into a main and a correction accumulator).  The producer warp streams
// the CTA's A slab through a 5-stage ring of 32-wide K blocks (64-byte swizzle; the 4 MB block stays
// L2-resident across the 31 passes) and the MMA warp runs 3 d / 16 instructions per pass.
//
// One cluster exchange per iteration: instead of normalising W = A v before publishing (which needs the
// global column norms first, i.e. a second cluster round trip), every CTA publishes W / s with the fixed
// bound s = sqrt(d) max|a| (|W_i| <= |a_i|_2 |v|_2, so the stored pool stays inside the fp16 range) together
// with its partial sums of W^2; one bulk shared::cluster copy per peer carries both.  After the exchange
// every CTA knows |W|_2 exactly and applies f = s / |W|_2 per column to the next product, so the pool it
// multiplies is exactly the reference's normalised v = W / |W| (zero columns stay zero).  The pool and the
// partials are double-buffered by exchange parity, so a fast peer never overwrites data a slow CTA's MMA or
// epilogue still reads.  Start vectors are the NumPy PCG64 streams (rng.cuh); the quotients and the selection
// follow the fp32 kernel (step.cu): lambda = q_j / (v_j . v_j) of the best column.
#include <cuda.h>
#include <cstdlib>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "engine.h"
#include "ptx.cuh"
#include "rng.cuh"

namespace dash {

constexpr int kPtStages = 5;
constexpr int kPtThreads = 192;                 // warp 0 TMA producer, warp 1 MMA, warps 2..5 rows
constexpr int kPtPool = 16;
constexpr int kPtKB = 32;                       // K block of the A ring (64-byte swizzle)
constexpr int kPtAPlane = 128 * kPtKB * 2;      // 8 KB: one plane of a 128 x 32 A tile
constexpr int kPtAStage = 2 * kPtAPlane;        // 16 KB
constexpr int kPtVkb = 2 * kPtPool * 128;       // 4 KB: [plane][16 rows][128 B] of V^T for one 64-wide k-block
constexpr int kVExp = -14;                      // |stored v| <= 1 -> v * 2^14 < 2^15

struct PtLayout {
  int d, nkb;
  size_t v_off, vbuf_bytes, pn_off, dbl_off, bar_off, bytes;
  __host__ __device__ explicit PtLayout(int d_) : d(d_), nkb(d_ / 64) {
    v_off = static_cast<size_t>(kPtStages) * kPtAStage;
    vbuf_bytes = static_cast<size_t>(nkb) * kPtVkb;                    // one pool buffer (64 KB at d = 1024)
    pn_off = v_off + 2 * vbuf_bytes;                                   // [2 parity][8 ranks][16] doubles
    dbl_off = pn_off + sizeof(double) * 2 * 8 * kPtPool;               // [4 warps][2][16] doubles
    bar_off = dbl_off + sizeof(double) * 4 * 2 * kPtPool;
    bytes = bar_off + 256 + 1024;  // barriers + alignment slack
  }
};

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

__device__ __forceinline__ void rows_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Cluster-wide fixed-order sums of nv x 16 per-row values (rows = the 128 threads of warps 2..5): lanes ->
// warp (shuffle butterfly), warps 0..3 in order, then ranks 0..C-1 in order.  Only the row warps take part
// (the producer / MMA warps keep streaming), so the exchange is mbarrier based: lane j < 16 of warp 0 writes
// its sum into slot[par][q] of every CTA and arrives (release, cluster scope) on that CTA's red[par]
// (16 C arrivals per phase).  `par` alternates slot buffers and barriers between consecutive reductions.
__device__ void pt_cluster_sum(const double (&x)[2][kPtPool], int nv, double* wpart, double* slots, uint64_t* red,
                               int par, uint32_t& red_phase, int C, int q, int rw, int lane,
                               double (&out)[2][kPtPool]) {
  rows_sync();  // the previous reduction's reader of wpart is done
  for (int s = 0; s < nv; ++s)
#pragma unroll
    for (int j = 0; j < kPtPool; ++j) {
      double t = x[s][j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) wpart[(rw * 2 + s) * kPtPool + j] = t;
    }
  rows_sync();
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

// Element (n, k) of V^T (pool vector n, row k) in the swizzled K-major operand layout, plane p.
__device__ __forceinline__ uint32_t pt_v_off(int n, int k, int p) {
  const int kb = k >> 6, kk = k & 63;
  return kb * kPtVkb + p * (kPtPool * 128) + (n >> 3) * 1024 + (n & 7) * 128 + ((((kk >> 3) ^ (n & 7))) << 4) +
         (kk & 7) * 2;
}

// Intra-CTA fixed-order column sums over the 128 rows (warp shuffles, then warps 0..3 in order); the result is
// valid in lanes 0..15 of row warp 0 (lane j holds column j).
__device__ __forceinline__ double pt_cta_colsum(const float (&w)[kPtPool], double* wpart, int rw, int lane) {
  rows_sync();  // previous users of wpart are done
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
  rows_sync();
  double sum = 0.0;
  if (rw == 0 && lane < kPtPool)
    for (int w4 = 0; w4 < 4; ++w4) sum += wpart[w4 * kPtPool + lane];
  return sum;
}

__global__ void __launch_bounds__(kPtThreads, 1)
    pi_tc_kernel(const __grid_constant__ CUtensorMap amap, dash_stack a, int pool, int iters, unsigned long long seed,
                 float* __restrict__ scale, float* __restrict__ inv_scale, int* __restrict__ status,
                 const int* __restrict__ seed_index, int xp) {
  const int d = a.rows;
  const PtLayout L(d);
  const int C = d / 128;
  const int q = static_cast<int>(cluster_rank());
  const int m = blockIdx.x / C;
  const int row0 = q * 128;
  extern __shared__ uint8_t pt_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(pt_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* vsm = smem + L.v_off;                                  // [2 parity][nkb][plane][16][128 B]
  double* pn = reinterpret_cast<double*>(smem + L.pn_off);        // [2 parity][8 ranks][16]
  double* wpart = reinterpret_cast<double*>(smem + L.dbl_off);    // [4 warps][2][16]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* empty = full + kPtStages;
  uint64_t* tfull = empty + kPtStages;
  uint64_t* vbar = tfull + 1;
  uint64_t* abar = vbar + 1;  // attempt decided (producer / MMA learn whether to run another attempt)
  uint64_t* red = abar + 1;   // [2] cluster reduction barriers (start / final quotients)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red + 2);
  int* again = reinterpret_cast<int*>(tmem_slot + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPtStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(vbar, 1);
    mbar_init(abar, 1);
    mbar_init(&red[0], kPtPool * C);
    mbar_init(&red[1], kPtPool * C);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<32>(tmem_slot);
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nkb = d / kPtKB;  // 32-wide A blocks per pass
  const int passes_per_attempt = iters + 1;

  if (warp == 0) {
    // ---------------------------------------------------------------- A slab producer (all attempts)
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int attempt = 0;; ++attempt) {
        for (int it = 0; it < passes_per_attempt; ++it)
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (xp & 5) {  // experiment: no A loads (MMA reads stale shared memory)
              mbar_arrive(&full[stage]);
            } else {
              mbar_arrive_expect_tx(&full[stage], kPtAStage);
              uint8_t* dst = smem + stage * kPtAStage;
              tma_load_4d(dst, &amap, &full[stage], kb * kPtKB, row0, 0, m);
              tma_load_4d(dst + kPtAPlane, &amap, &full[stage], kb * kPtKB, row0, 1, m);
            }
            if (++stage == kPtStages) { stage = 0; phase ^= 1; }
          }
        mbar_wait(abar, attempt & 1);
        if (!*reinterpret_cast<volatile int*>(again)) break;
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (whole warp, elected lane)
    const uint32_t idesc = umma_idesc_f16(128, kPtPool, 0, 0);
    int stage = 0;
    uint32_t phase = 0, vphase = 0, ex = 0;
    for (int attempt = 0;; ++attempt) {
      for (int it = 0; it < passes_per_attempt; ++it, ++ex) {
        mbar_wait(vbar, vphase);
        vphase ^= 1;
        tc_fence_after();
        uint8_t* vcur = vsm + (ex & 1) * L.vbuf_bytes;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem + stage * kPtAStage);
          const uint32_t v_base = smem_u32(vcur + (kb >> 1) * kPtVkb) + (kb & 1) * 64;  // 32 of the 64 k columns
#pragma unroll
          for (int k = 0; k < kPtKB / 16; ++k)
#pragma unroll
            for (int p = 0; p < 3; ++p) {
              if ((xp & 2) && !(kb == 0 && k == 0 && p <= 1)) continue;  // experiment: (almost) no MMAs
              const uint32_t ap = (p == 2) ? 1u : 0u, bp = (p == 1) ? 1u : 0u;
              const uint64_t ad = umma_sdesc(a_base + ap * kPtAPlane + k * 32, 16, 512, 4);  // 64-byte swizzle
              const uint64_t bd = umma_sdesc(v_base + bp * (kPtPool * 128) + k * 32, 16, 1024);
              const uint32_t fresh = (kb == 0 && k == 0 && p <= 1) ? 0u : 1u;
              asm volatile(
                  "{\n\t.reg .pred pp, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 pp, %4, 0;\n\t"
                  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, pp;\n\t}\n" ::"r"(
                      tmem + (p ? 16u : 0u)),
                  "l"(ad), "l"(bd), "r"(idesc), "r"(fresh));
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
                smem_u32(tfull))
            : "memory");
      }
      mbar_wait(abar, attempt & 1);
      if (!*reinterpret_cast<volatile int*>(again)) break;
    }
  } else {
    // ---------------------------------------------------------------- row warps: start vectors, norms, pool
    const int rw = static_cast<int>(warp) - 2;               // 0..3 (order of the fixed reductions)
    const int row = 32 * static_cast<int>(warp & 3) + static_cast<int>(lane);  // TMEM lane = CTA row
    const int kg = row0 + row;                                // global row = K index of V
    const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * (warp & 3)) << 16);
    const float sa = ldexpf(1.f, __ldg(a.exp + m) + kVExp);
    float amax_a = __uint_as_float(__ldg(a.amax + m));
    // |W_i| <= |a_i|_2 <= sqrt(d) max|a| <= sfix, a power of two: the stored pool W / sfix is an exact scaling
    const double sfix =
        amax_a > 0.f ? ldexp(1.0, ilogb(sqrt(static_cast<double>(d)) * static_cast<double>(amax_a)) + 1) : 1.0;
    const float inv_sfix = static_cast<float>(1.0 / sfix);
    uint64_t bseed = rng::block_seed(seed, static_cast<uint64_t>(seed_index ? seed_index[m] : m));
    const uint32_t vbar_peer0 = smem_u32(vbar);
    const uint32_t my_slice = static_cast<uint32_t>(row0 / 64) * kPtVkb;  // my 2 k-blocks (8 KB) of a pool buffer
    int par = 0;
    uint32_t tphase = 0, red_phase = 0, vphase = 0, ex = 0;
    float lam = 0.f;
    int st = 0;
    float v[kPtPool];   // my row of the (true, normalised) pool of the current pass
    float vs[kPtPool];  // my row of the stored pool (true pool = vs * f)

    // write my stored row (split, fixed exponent) + my partial sums into pool / partial buffer `ex & 1` and push
    // both to every peer (one exchange; completes vbar there together with everyone else's pushes)
    auto publish = [&](double partial) {
      const float inv = ldexpf(1.f, -kVExp);
      uint8_t* vb = vsm + (ex & 1) * L.vbuf_bytes;
      __half* vh = reinterpret_cast<__half*>(vb);
#pragma unroll
      for (int n = 0; n < kPtPool; ++n) {
        const float y = vs[n] * inv;
        const __half h = __float2half_rn(y);
        const __half l = __float2half_rn(y - __half2float(h));
        vh[pt_v_off(n, kg, 0) / 2] = h;
        vh[pt_v_off(n, kg, 1) / 2] = l;
      }
      double* pslot = pn + ((ex & 1) * 8 + q) * kPtPool;
      if (rw == 0 && lane < kPtPool) pslot[lane] = partial;
      fence_proxy_async_smem();
      rows_sync();
      if (rw == 0 && lane == 0) {
        mbar_arrive_expect_tx(vbar, static_cast<uint32_t>(C - 1) * (2 * kPtVkb + kPtPool * 8));
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

    for (int attempt = 0; attempt < 2; ++attempt) {
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
      // the start reduction borrows the pool buffer of the next exchange parity as its slot area
      double* slots0 = reinterpret_cast<double*>(vsm + ((ex + 1) & 1) * L.vbuf_bytes);
      pt_cluster_sum(x, 1, wpart, slots0, red, par, red_phase, C, q, rw, static_cast<int>(lane), tot);
      par ^= 1;
#pragma unroll
      for (int j = 0; j < kPtPool; ++j) {
        double n = sqrt(tot[0][j]);
        if (n == 0.0) n = 1.0;
        v[j] = static_cast<float>(v[j] / n);
        vs[j] = v[j];  // stored = true pool (|v| <= 1) for the first pass
      }
      publish(0.0);
      float f[kPtPool];
#pragma unroll
      for (int j = 0; j < kPtPool; ++j) f[j] = 1.f;
      for (int it = 0; it <= iters; ++it) {
        // ---- the pool of this pass has been exchanged: its column scale f (pass >= 1) from the partials
        mbar_wait(vbar, vphase);
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
          for (int j = 0; j < kPtPool; ++j) {
            f[j] = __shfl_sync(0xffffffffu, fl, j);
            v[j] = vs[j] * f[j];
          }
        }
        // ---- W = A v for my row: (A vs) * f (main + correction accumulators)
        mbar_wait(tfull, tphase);
        tphase ^= 1;
        tc_fence_after();
        float mn[kPtPool], cr[kPtPool], w[kPtPool];
        tmem_ld16(taddr, mn);
        tmem_ld16(taddr + 16, cr);
        tc_fence_before();
#pragma unroll
        for (int j = 0; j < kPtPool; ++j) w[j] = (mn[j] + cr[j]) * sa * f[j];
        if (it < iters) {
          const double partial = pt_cta_colsum(w, wpart, rw, static_cast<int>(lane));
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
          double* slots1 = reinterpret_cast<double*>(vsm + (ex & 1) * L.vbuf_bytes);
          pt_cluster_sum(x, 2, wpart, slots1, red, par, red_phase, C, q, rw, static_cast<int>(lane), tot);
          par ^= 1;
        }
      }
      // ---- selection by Rayleigh quotient q_j / |v_j|^2 (the reference's pool is normalised, so this is its
      // argmax of q_j), lambda = q / |v|^2 (spectral.py:104-112)
      int best = -1;
      double bq = 0.0;
      bool any = false;
      for (int j = 0; j < pool; ++j) {
        if (tot[1][j] > 0.0) {
          const double r = tot[0][j] / tot[1][j];
          if (!any || r > bq) { bq = r; best = j; }
          any = true;
        }
      }
      const bool done = (any && bq != 0.0) || attempt == 1 || (xp & 4);  // knob 4: never retry (timing)
      if (any && bq != 0.0) lam = static_cast<float>(bq);
      else if (attempt == 0) { bseed = rng::block_seed(bseed, 0x5EEDull); st = 1; }
      else st = 2;
      (void)best;
      rows_sync();
      if (rw == 0 && lane == 0) {
        *reinterpret_cast<volatile int*>(again) = done ? 0 : 1;
        mbar_arrive(abar);
      }
      if (done) break;
    }
    if (q == 0 && rw == 0 && lane == 0) {
      const float s2 = 2.f * lam;
      scale[m] = s2;
      inv_scale[m] = s2 > 0.f ? 1.f / s2 : 0.f;
      if (status) status[m] = (st == 2) ? 2 : (s2 > 0.f ? 0 : 1);
    }
  }
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<32>(tmem);
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
  static size_t attr = 0;
  if (L.bytes > attr) {
    cudaFuncSetAttribute(pi_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(L.bytes));
    if (C > 8) cudaFuncSetAttribute(pi_tc_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = L.bytes;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(a.nmat * C));
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
  static const int xp = getenv("DASH_PI_EXP") ? atoi(getenv("DASH_PI_EXP")) : 0;  // experiment knobs
  cudaError_t e = cudaLaunchKernelEx(&cfg, pi_tc_kernel, map, a, pool, iters, seed, scale, inv_scale, status,
                                     seed_index, xp);
  note_launch();
  return e == cudaSuccess ? DASH_OK : DASH_ECUDA;
}

}  // namespace dash

extern "C" int dash_power_iteration_split(const dash_stack* a, int pool, int iters, unsigned long long seed,
                                          float* scale, float* inv_scale, int* status, const int* seed_index,
                                          void* stream) {
  if (!dash::stack_ok(a) || !scale || !inv_scale) return DASH_EINVAL;
  return dash::pi_tc_launch(*a, pool, iters, seed, scale, inv_scale, status, seed_index,
                            static_cast<cudaStream_t>(stream));
}
