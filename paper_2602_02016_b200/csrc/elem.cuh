// Vectorised helpers of the HBM-bound split-stack kernels: every thread moves 8 consecutive columns
// (one 16-byte word per fp16 plane), rows are walked with a per-matrix grid-stride loop.
#pragma once
#include <cuda_fp16.h>

#include <cstdint>

#include "../../include/dash_b200.h"
#include "ptx.cuh"

namespace dash {

// Calls f(r, c) for every 8-column chunk (c = 0, 8, ...) of a rows x ld matrix; grid.x CTAs share a matrix.
template <class F>
__device__ __forceinline__ void for_chunks8(int rows, int ld, F f) {
  const int cpr = ld >> 3;
  const int total = rows * cpr;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int r = i / cpr;
    f(r, (i - r * cpr) << 3);
  }
}

// 8 values (hi + lo) * scale from the split planes at element offset `off` of the hi plane.
__device__ __forceinline__ void load_split8(const __half* hi, long long plane, long long off, float scale,
                                            float (&v)[8]) {
  const uint4 h = __ldg(reinterpret_cast<const uint4*>(hi + off));
  const uint4 l = __ldg(reinterpret_cast<const uint4*>(hi + plane + off));
  const __half2* h2 = reinterpret_cast<const __half2*>(&h);
  const __half2* l2 = reinterpret_cast<const __half2*>(&l);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 a = __half22float2(h2[k]), b = __half22float2(l2[k]);
    v[2 * k] = (a.x + b.x) * scale;
    v[2 * k + 1] = (a.y + b.y) * scale;
  }
}

// Split 8 values (times inv = 2^-e) into the two planes; returns true when a hi part overflowed.
__device__ __forceinline__ bool store_split8(__half* hi, long long plane, long long off, const float (&v)[8],
                                             float inv) {
  uint32_t hw[4], lw[4];
  bool ovf = false;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float y0 = v[2 * k] * inv, y1 = v[2 * k + 1] * inv;
    const __half h0 = __float2half_rn(y0), h1 = __float2half_rn(y1);
    const __half l0 = __float2half_rn(y0 - __half2float(h0)), l1 = __float2half_rn(y1 - __half2float(h1));
    ovf |= __hisinf(h0) | __hisinf(h1) | __hisnan(h0) | __hisnan(h1);
    hw[k] = static_cast<uint32_t>(__half_as_ushort(h0)) | (static_cast<uint32_t>(__half_as_ushort(h1)) << 16);
    lw[k] = static_cast<uint32_t>(__half_as_ushort(l0)) | (static_cast<uint32_t>(__half_as_ushort(l1)) << 16);
  }
  *reinterpret_cast<uint4*>(hi + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
  *reinterpret_cast<uint4*>(hi + plane + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  return ovf;
}

__device__ __forceinline__ __half* mat_hi(const dash_stack& s, int m) {
  return reinterpret_cast<__half*>(s.data) + static_cast<long long>(m) * 2 * s.rows * s.ld;
}
__device__ __forceinline__ long long mat_plane(const dash_stack& s) { return static_cast<long long>(s.rows) * s.ld; }

}  // namespace dash
