// Batched cyclic Jacobi eigensolver in float64 (eigensolver.py:53-124) -- the EVD solver option, the config-2
// comparator and the FULL64 optimizer's re-solve of blocks its fp32-class Newton iteration cannot converge.
//
// One CTA per matrix.  A sweep visits every unordered index pair once in n - 1 (n even) rounds of disjoint
// pairs, the reference's circle-method schedule (eigensolver.py:53-68): round r pairs position i with position
// m - 1 - i of the player list [0, r-rotated 1..m-1].  Per round:
//   1. thread k of the n/2 pairs computes the rotation of pair (p, q) from a_pp, a_qq, a_pq exactly as the
//      reference does (tau, t, c, s in IEEE float64, explicit _rn intrinsics: no FMA contraction), or the
//      identity when |a_pq| <= skip (a "dead" pair, eigensolver.py:95-97);
//   2. A <- R A R^T applied tile by tile: the 2 x 2 tile (pair I rows, pair J columns) becomes
//      R_I A_IJ R_J^T, row rotation first and column rotation second -- the reference's two half-updates
//      (:101-106), fused into one pass over A (tiles are disjoint, so the update is in place);
//   3. V <- V R^T (:107-109), one pass over V.
// After each sweep the off-diagonal Frobenius norm is compared with tol * |A0|_F (:86-111).  Converged
// eigenvalues are sorted ascending with a stable rank (np.argsort kind="stable") and the eigenvector columns
// permuted with them (:114-116).  A and V live in the caller's workspace (float64, L2-resident for the block
// sizes the optimizer uses at small batch), the rotation parameters in shared memory.
#include <cuda_runtime.h>

#include <cmath>

#include "engine.h"

namespace dash {

constexpr int kEvdThreads = 1024;
constexpr int kEvdMaxDim = 1024;

// position -> player of round r (players[0] fixed, players[1..m-1] rotated right by r)
__device__ __forceinline__ int evd_player(int pos, int r, int m) {
  return pos == 0 ? 0 : ((pos - 1 - r) % (m - 1) + (m - 1)) % (m - 1) + 1;
}

__device__ double evd_block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kEvdThreads / 32; ++i) t += red[i];  // fixed order
  __syncthreads();
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  return red[0];
}

__global__ void __launch_bounds__(kEvdThreads) jacobi_kernel(const double* __restrict__ in, int d, double tol,
                                                               int max_sweeps, double* __restrict__ lam_out,
                                                               double* __restrict__ q_out, int* __restrict__ sweeps_out,
                                                               int* __restrict__ status, double* __restrict__ work) {
  __shared__ double cs[kEvdMaxDim / 2], sn[kEvdMaxDim / 2];
  __shared__ int pp[kEvdMaxDim / 2], qq[kEvdMaxDim / 2];
  __shared__ double red[kEvdThreads / 32];
  __shared__ int rank_s[kEvdMaxDim];
  const int mtx = blockIdx.x;
  const long long dd = static_cast<long long>(d) * d;
  const double* a0 = in + mtx * dd;
  double* a = work + mtx * 2 * dd;  // working copy of A
  double* v = a + dd;               // accumulated rotations
  double fro = 0.0;
  for (long long i = threadIdx.x; i < dd; i += kEvdThreads) {
    const double x = a0[i];
    a[i] = x;
    v[i] = (i / d == i % d) ? 1.0 : 0.0;
    fro += x * x;
  }
  const double thresh = tol * sqrt(evd_block_sum(fro, red));
  const double skip = 0.1 * thresh / d;
  const int m = (d % 2 == 0) ? d : d + 1;
  const int half = m / 2;
  auto offdiag = [&]() {
    double t = 0.0;
    for (long long i = threadIdx.x; i < dd; i += kEvdThreads)
      if (i / d != i % d) t += a[i] * a[i];
    return sqrt(evd_block_sum(t, red));
  };
  int sweeps = 0;
  bool converged = d == 1 || offdiag() <= thresh;
  while (!converged && sweeps < max_sweeps) {
    ++sweeps;
    for (int r = 0; r < m - 1; ++r) {
      // ---- 1. rotations of this round's pairs (identity for padded or dead pairs)
      for (int k = threadIdx.x; k < half; k += kEvdThreads) {
        const int x = evd_player(k, r, m), y = evd_player(m - 1 - k, r, m);
        double c = 1.0, s = 0.0;
        // an odd dimension pads the schedule with a dummy player: its partner is a lone index that is not
        // rotated this round (q = -1) but still receives the other pairs' row / column rotations
        int p = min(x, y), q = max(x, y);
        if (q >= d) {
          q = -1;
        } else {
          const double apq = a[static_cast<long long>(p) * d + q];
          if (fabs(apq) > skip) {
            const double app = a[static_cast<long long>(p) * d + p], aqq = a[static_cast<long long>(q) * d + q];
            const double tau = __ddiv_rn(__dsub_rn(aqq, app), __dmul_rn(2.0, apq));
            double t;
            if (tau == 0.0) {
              t = 1.0;
            } else {
              const double sq = __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(tau, tau)));
              t = __ddiv_rn(tau > 0.0 ? 1.0 : -1.0, __dadd_rn(fabs(tau), sq));
            }
            c = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(t, t))));
            s = __dmul_rn(t, c);
          }
        }
        cs[k] = c;
        sn[k] = s;
        pp[k] = p;
        qq[k] = q;
      }
      __syncthreads();
      // ---- 2. A <- R A R^T, one 2 x 2 tile (pair I rows, pair J columns) per work item
      const long long tiles = static_cast<long long>(half) * half;
      for (long long t = threadIdx.x; t < tiles; t += kEvdThreads) {
        const int I = static_cast<int>(t / half), J = static_cast<int>(t % half);
        const int pi = pp[I], qi = qq[I], pj = pp[J], qj = qq[J];  // qi / qj = -1: a lone (unrotated) index
        const double ci = cs[I], si = sn[I], cj = cs[J], sj = sn[J];
        if (si == 0.0 && sj == 0.0) continue;  // both rotations are the identity
        double* r0 = a + static_cast<long long>(pi) * d;
        double* r1 = a + static_cast<long long>(qi < 0 ? pi : qi) * d;
        const double x00 = r0[pj], x01 = qj >= 0 ? r0[qj] : 0.0;
        const double x10 = qi >= 0 ? r1[pj] : 0.0, x11 = (qi >= 0 && qj >= 0) ? r1[qj] : 0.0;
        // rows (eigensolver.py:101-103): p' = c p - s q, q' = s p + c q
        const double y00 = __dsub_rn(__dmul_rn(ci, x00), __dmul_rn(si, x10));
        const double y01 = __dsub_rn(__dmul_rn(ci, x01), __dmul_rn(si, x11));
        const double y10 = __dadd_rn(__dmul_rn(si, x00), __dmul_rn(ci, x10));
        const double y11 = __dadd_rn(__dmul_rn(si, x01), __dmul_rn(ci, x11));
        // columns (:104-106)
        r0[pj] = __dsub_rn(__dmul_rn(cj, y00), __dmul_rn(sj, y01));
        if (qj >= 0) r0[qj] = __dadd_rn(__dmul_rn(sj, y00), __dmul_rn(cj, y01));
        if (qi >= 0) {
          r1[pj] = __dsub_rn(__dmul_rn(cj, y10), __dmul_rn(sj, y11));
          if (qj >= 0) r1[qj] = __dadd_rn(__dmul_rn(sj, y10), __dmul_rn(cj, y11));
        }
      }
      // ---- 3. V <- V R^T (:107-109)
      const long long vitems = static_cast<long long>(d) * half;
      for (long long t = threadIdx.x; t < vitems; t += kEvdThreads) {
        const int row = static_cast<int>(t / half), J = static_cast<int>(t % half);
        const int pj = pp[J], qj = qq[J];
        if (qj < 0 || sn[J] == 0.0) continue;  // lone index or identity rotation
        const double c = cs[J], s = sn[J];
        double* vr = v + static_cast<long long>(row) * d;
        const double vp = vr[pj], vq = vr[qj];
        vr[pj] = __dsub_rn(__dmul_rn(c, vp), __dmul_rn(s, vq));
        vr[qj] = __dadd_rn(__dmul_rn(s, vp), __dmul_rn(c, vq));
      }
      __syncthreads();
    }
    converged = offdiag() <= thresh;
  }
  // ---- eigenvalues ascending (stable), eigenvector columns permuted alike
  for (int i = threadIdx.x; i < d; i += kEvdThreads) {
    const double li = a[static_cast<long long>(i) * d + i];
    int rk = 0;
    for (int j = 0; j < d; ++j) {
      const double lj = a[static_cast<long long>(j) * d + j];
      rk += (lj < li) || (lj == li && j < i);
    }
    rank_s[i] = rk;
    lam_out[static_cast<long long>(mtx) * d + rk] = li;
  }
  __syncthreads();
  double* qo = q_out + mtx * dd;
  for (long long t = threadIdx.x; t < dd; t += kEvdThreads) {
    const int row = static_cast<int>(t / d), col = static_cast<int>(t % d);
    qo[static_cast<long long>(row) * d + rank_s[col]] = v[t];
  }
  if (threadIdx.x == 0) {
    if (sweeps_out) sweeps_out[mtx] = sweeps;
    if (status) status[mtx] = converged ? 0 : 1;
  }
}

}  // namespace dash

extern "C" {

size_t dash_jacobi_ws_bytes(int n, int d) { return 2 * static_cast<size_t>(n) * d * d * sizeof(double) + 256; }

int dash_jacobi_eigh(const double* a, int n, int d, double tol, int max_sweeps, double* lam, double* q, int* sweeps,
                     int* status, void* ws, size_t ws_bytes, void* stream) {
  if (!a || !lam || !q || n < 1 || d < 1 || d > dash::kEvdMaxDim || max_sweeps < 0 || !(tol >= 0.0) || !ws)
    return DASH_EINVAL;
  if (ws_bytes < dash_jacobi_ws_bytes(n, d)) return DASH_EINVAL;
  dash::jacobi_kernel<<<n, dash::kEvdThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      a, d, tol, max_sweeps, lam, q, sweeps, status, static_cast<double*>(ws));
  dash::note_launch();
  return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_ECUDA;
}

}  // extern "C"
