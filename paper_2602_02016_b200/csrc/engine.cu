// Host runtime of the DASH engine: TMA descriptor creation, split/unsplit kernels, grouped GEMM
// job assembly, and the dense-primitive part of the C ABI (include/dash_b200.h).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <vector>

#include "engine.h"
#include "ptx.cuh"

namespace dash {

// ---------------------------------------------------------------------------- TMA descriptors
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_stack_map(const dash_stack& s, int box_rows, CUtensorMap* out, int box_cols, int box_planes, int swz) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(s.ld), static_cast<cuuint64_t>(s.rows), 2,
                        static_cast<cuuint64_t>(s.nmat)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(s.ld) * 2, static_cast<cuuint64_t>(s.rows) * s.ld * 2,
                           2ull * s.rows * s.ld * 2};
  cuuint32_t box[4] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows),
                       static_cast<cuuint32_t>(box_planes), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, s.data, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_f32_map(const float* base, int nmat, int rows, int ld, int box_cols, int box_rows, bool swz,
                  CUtensorMap* out) {
  auto fn = encode_fn();
  if (!fn || ld % 4 != 0 || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(nmat)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 4, static_cast<cuuint64_t>(rows) * ld * 4};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool stack_ok(const dash_stack* s) {
  return s && s->data && s->nmat > 0 && s->rows > 0 && s->cols > 0 && s->ld >= s->cols && s->ld % kLdAlign == 0 &&
         s->exp && s->amax;
}

// ---------------------------------------------------------------------------- split / unsplit
__global__ void amax_kernel(const float* __restrict__ src, long long mat_stride, int ld, int rows, int cols,
                            unsigned* __restrict__ amax) {
  const int m = blockIdx.y;
  const float* base = src + m * mat_stride;
  const long long total = static_cast<long long>(rows) * cols;
  float mx = 0.f;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / cols), c = static_cast<int>(i % cols);
    float v = fabsf(base[static_cast<long long>(r) * ld + c]);
    if (!(v <= 3.0e38f)) v = __uint_as_float(0x7fc00000u);
    mx = nonneg_max(mx, v);
  }
  mx = warp_max_nonneg(mx);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(amax + m, mx);
}

__device__ __forceinline__ int exp_for_max(float amax) {
  if (!(amax > 0.f) || !(amax < 3.0e38f)) return 0;
  int x;
  frexpf(amax, &x);
  return x - 15;
}

__global__ void split_kernel(const float* __restrict__ src, long long mat_stride, int src_ld, int rows, int cols,
                             __half* __restrict__ dst, int ld, const unsigned* __restrict__ amax,
                             int* __restrict__ exp_out) {
  const int m = blockIdx.y;
  const int e = exp_for_max(__uint_as_float(amax[m]));
  if (blockIdx.x == 0 && threadIdx.x == 0) exp_out[m] = e;
  const float inv = ldexpf(1.f, -e);
  const float* s = src + m * mat_stride;
  __half* hi = dst + static_cast<long long>(m) * 2 * rows * ld;
  __half* lo = hi + static_cast<long long>(rows) * ld;
  const long long total = static_cast<long long>(rows) * ld;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / ld), c = static_cast<int>(i % ld);
    float y = 0.f;
    if (c < cols) y = s[static_cast<long long>(r) * src_ld + c] * inv;
    const __half h = __float2half_rn(y);
    hi[i] = h;
    lo[i] = __float2half_rn(y - __half2float(h));
  }
}

__global__ void unsplit_kernel(const __half* __restrict__ src, int rows, int cols, int ld,
                               const int* __restrict__ exps, float* __restrict__ dst, long long mat_stride,
                               int dst_ld) {
  const int m = blockIdx.y;
  const float sc = ldexpf(1.f, exps[m]);
  const __half* hi = src + static_cast<long long>(m) * 2 * rows * ld;
  const __half* lo = hi + static_cast<long long>(rows) * ld;
  float* d = dst + m * mat_stride;
  const long long total = static_cast<long long>(rows) * cols;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / cols), c = static_cast<int>(i % cols);
    const long long o = static_cast<long long>(r) * ld + c;
    d[static_cast<long long>(r) * dst_ld + c] = (__half2float(hi[o]) + __half2float(lo[o])) * sc;
  }
}

static dim3 grid_for(long long elems, int nmat) {
  long long b = (elems + 255) / 256;
  if (b > 1024) b = 1024;
  if (b < 1) b = 1;
  return dim3(static_cast<unsigned>(b), static_cast<unsigned>(nmat));
}

int split_stack(const float* src, long long mat_stride, int src_ld, const dash_stack& d, cudaStream_t st) {
  cudaMemsetAsync(d.amax, 0, sizeof(unsigned) * d.nmat, st);
  amax_kernel<<<grid_for(static_cast<long long>(d.rows) * d.cols, d.nmat), 256, 0, st>>>(
      src, mat_stride, src_ld, d.rows, d.cols, d.amax);
  note_launch();
  split_kernel<<<grid_for(static_cast<long long>(d.rows) * d.ld, d.nmat), 256, 0, st>>>(
      src, mat_stride, src_ld, d.rows, d.cols, reinterpret_cast<__half*>(d.data), d.ld, d.amax, d.exp);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_ECUDA;
}

int unsplit_stack(const dash_stack& s, float* dst, long long mat_stride, int dst_ld, cudaStream_t st) {
  unsplit_kernel<<<grid_for(static_cast<long long>(s.rows) * s.cols, s.nmat), 256, 0, st>>>(
      reinterpret_cast<const __half*>(s.data), s.rows, s.cols, s.ld, s.exp, dst, mat_stride, dst_ld);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_ECUDA;
}

// ---------------------------------------------------------------------------- job assembly
int JobBuilder::add_map(const dash_stack& s, int box_rows, int box_cols, int box_planes, int swz) {
  for (size_t i = 0; i < map_keys.size(); ++i) {
    const MapKey& k = map_keys[i];
    if (k.data == s.data && k.box == box_rows && k.box_cols == box_cols && k.planes == box_planes && k.swz == swz &&
        k.nmat == s.nmat && k.rows == s.rows && k.ld == s.ld)
      return static_cast<int>(i);
  }
  CUtensorMap m;
  if (!make_stack_map(s, box_rows, &m, box_cols, box_planes, swz)) return -1;
  maps.push_back(m);
  map_keys.push_back(MapKey{s.data, box_rows, s.nmat, s.rows, s.ld, box_cols, box_planes, swz});
  return static_cast<int>(maps.size()) - 1;
}

// Fill operand fields of `j` for C = op(A) op(B); returns false on a shape mismatch or map failure.
bool JobBuilder::operands(GemmJob& j, const dash_stack& a, int am, int trans_a, const dash_stack& b, int bm,
                          int trans_b, bool check) {
  const int M = trans_a ? a.cols : a.rows;
  const int K = trans_a ? a.rows : a.cols;
  const int Kb = trans_b ? b.cols : b.rows;
  const int N = trans_b ? b.rows : b.cols;
  if (check && K != Kb) return false;
  std::memset(&j, 0, sizeof(j));
  j.a_mn = trans_a ? 1 : 0;  // stored K x M -> MN-major
  j.b_mn = trans_b ? 0 : 1;  // stored K x N -> MN-major; stored N x K -> K-major
  j.a_map = add_map(a, j.a_mn ? 64 : kTileM / 2);  // each CTA of the pair: 128 rows of A, 64 rows of B
  j.b_map = add_map(b, 64);
  j.a_mapT = add_map(a, j.a_mn ? kTileM / 2 : 64);  // the other majorness (upper pair-block storage reads)
  // K-block 32 variant (deeper pipeline): K-major boxes 32 wide with 64-byte swizzle, MN-major boxes 32 deep
  j.a_map32 = j.a_mn ? add_map(a, 32, 64, 1, 128) : add_map(a, kTileM / 2, 32, 1, 64);
  j.b_map32 = j.b_mn ? add_map(b, 32, 64, 1, 128) : add_map(b, 64, 32, 1, 64);
  if (j.a_map < 0 || j.b_map < 0 || j.a_map32 < 0 || j.b_map32 < 0) return false;
  j.a_mat = am;
  j.b_mat = bm;
  j.M = M;
  j.N = N;
  j.K = K;
  j.tiles_n = (N + kTileN - 1) / kTileN;
  j.tiles_n2 = (N + 255) / 256;
  j.a_exp = a.exp + am;
  j.a_amax = a.amax + am;
  j.b_exp = b.exp + bm;
  j.b_amax = b.amax + bm;
  j.alpha = 1.f;
  j.c_map = j.c_tmap = j.c2_map = j.c2_tmap = -1;
  j.s_map = -1;
  j.f_map = j.f_tmap = -1;
  return true;
}

void JobBuilder::set_out(GemmJob& j, const dash_stack& c, int cm) {
  j.c_hi = reinterpret_cast<__half*>(c.data) + static_cast<long long>(cm) * 2 * c.rows * c.ld;
  j.c_plane = static_cast<long long>(c.rows) * c.ld;
  j.c_ld = c.ld;
  j.c_exp = c.exp + cm;
  j.c_amax = c.amax + cm;
  j.c_rows = c.rows;
  j.c_cols = c.cols;
  j.c_mat = cm;
  j.c_map = add_map(c, 32, 64, 2, true);
  j.c_tmap = add_map(c, 64, 32, 2, false);
}

int JobBuilder::add_f32_map(const float* base, int nmat, int rows, int ld, int box_cols, int box_rows, bool swz) {
  for (size_t i = 0; i < map_keys.size(); ++i) {
    const MapKey& k = map_keys[i];
    if (k.data == base && k.planes == -1 && k.box == box_rows && k.box_cols == box_cols && k.swz == swz &&
        k.nmat == nmat && k.rows == rows && k.ld == ld)
      return static_cast<int>(i);
  }
  CUtensorMap m;
  if (!make_f32_map(base, nmat, rows, ld, box_cols, box_rows, swz, &m)) return -1;
  maps.push_back(m);
  map_keys.push_back(MapKey{base, box_rows, nmat, rows, ld, box_cols, -1, swz});
  return static_cast<int>(maps.size()) - 1;
}

void JobBuilder::set_fout(GemmJob& j, float* base, int nmat, int rows, int ld, int mat, bool is_input) {
  j.f_out = base + static_cast<long long>(mat) * rows * ld;
  j.f_ld = ld;
  if (is_input) j.f_in = j.f_out;
  j.f_mat = mat;
  j.f_rows = rows;
  j.f_cols = ld;
  static const int no_tma = getenv("DASH_NO_TMA_STORE") ? atoi(getenv("DASH_NO_TMA_STORE")) : 0;
  j.f_map = no_tma ? -1 : add_f32_map(base, nmat, rows, ld, 32, 32, true);
  j.f_tmap = no_tma ? -1 : add_f32_map(base, nmat, rows, ld, 32, 64, false);
  if (j.f_map < 0 || j.f_tmap < 0) j.f_map = j.f_tmap = -1;
}

void JobBuilder::set_side(GemmJob& j, const dash_stack& s, int m) {
  j.s_hi = reinterpret_cast<const __half*>(s.data) + static_cast<long long>(m) * 2 * s.rows * s.ld;
  j.s_plane = static_cast<long long>(s.rows) * s.ld;
  j.s_ld = s.ld;
  j.s_exp = s.exp + m;
  j.s_amax = s.amax + m;
  j.s_mat = m;
  static const int no_tma = getenv("DASH_NO_TMA_STORE") ? atoi(getenv("DASH_NO_TMA_STORE")) : 0;
  j.s_map = no_tma ? -1 : add_map(s, 32, 64, 2, true);
}

void JobBuilder::set_out2(GemmJob& j, const dash_stack& c, int cm) {
  j.c2_hi = reinterpret_cast<__half*>(c.data) + static_cast<long long>(cm) * 2 * c.rows * c.ld;
  j.c2_plane = static_cast<long long>(c.rows) * c.ld;
  j.c2_exp = c.exp + cm;
  j.c2_amax = c.amax + cm;
  j.c2_mat = cm;
  j.c2_map = add_map(c, 32, 64, 2, true);
  j.c2_tmap = add_map(c, 64, 32, 2, false);
}

int job_tiles(const GemmJob& j, int nt) {
  const int tm = (j.M + kTileM - 1) / kTileM;
  const int tn = nt == 128 ? j.tiles_n : j.tiles_n2, step = 256 / nt;
  if (!j.sym) return tm * tn;
  int n = 0;  // symmetric: column tiles J >= 2I (nt 128) / J >= I (nt 256) of every 256-row tile I (tile_coords)
  for (int i = 0; i < tm; ++i) n += tn - step * i;
  return n;
}

void JobBuilder::push(GemmJob& j) {
  static const int no_sym = getenv("DASH_NO_SYM") ? atoi(getenv("DASH_NO_SYM")) : 0;  // diagnostic knob
  // symmetric jobs: solver products (split outputs, mirrored as split tiles) and the statistics EMA (fp32 in / out,
  // mirrored through the transposed fp32 map; needs the TMA-staged fp32 path)
  if (j.sym && (no_sym || j.M != j.N || j.op == EPI_APPLY || (j.op == EPI_EMA && (j.f_map < 0 || j.f_tmap < 0))))
    j.sym = 0;
  // TMA-staged split stores need the job to cover its output matrix exactly (padding stays zero)
  static const int no_tma = getenv("DASH_NO_TMA_STORE") ? atoi(getenv("DASH_NO_TMA_STORE")) : 0;
  if (no_tma || !j.c_hi || j.M != j.c_rows || j.N != j.c_cols || j.c_map < 0 || j.c_tmap < 0 ||
      (j.c2_hi && (j.c2_map < 0 || j.c2_tmap < 0)))
    j.c_map = j.c_tmap = j.c2_map = j.c2_tmap = -1;
  j.tile_start = tiles;
  tiles += job_tiles(j);
  j.tile_start2 = tiles2;
  tiles2 += job_tiles(j, 256);
  all_sym = all_sym && j.sym;
  jobs.push_back(j);
}

size_t JobBuilder::bytes_for(int nmaps, int njobs) {  // maps + jobs + the scheduler counters + alignment
  return static_cast<size_t>(nmaps) * sizeof(CUtensorMap) + static_cast<size_t>(njobs) * sizeof(GemmJob) + 384;
}

bool JobBuilder::upload(Arena& ar, cudaStream_t st, UploadedGemm* out) {
  *out = UploadedGemm{};
  if (jobs.empty()) return true;
  const size_t mb = maps.size() * sizeof(CUtensorMap), jb = jobs.size() * sizeof(GemmJob);
  uint8_t* d = static_cast<uint8_t*>(ar.take(mb + jb));
  int* counter = ar.take_n<int>(2);
  if (!d || !counter) return false;
  if (cudaMemsetAsync(counter, 0, 2 * sizeof(int), st) != cudaSuccess) return false;
  out->counter = counter;
  staging.resize(mb + jb);
  std::memcpy(staging.data(), maps.data(), mb);
  std::memcpy(staging.data() + mb, jobs.data(), jb);
  if (cudaMemcpyAsync(d, staging.data(), mb + jb, cudaMemcpyHostToDevice, st) != cudaSuccess) return false;
  out->maps = reinterpret_cast<const CUtensorMap*>(d);
  out->jobs = reinterpret_cast<const GemmJob*>(d + mb);
  out->njobs = static_cast<int>(jobs.size());
  out->tiles = tiles;
  out->flops = 0.0;
  for (const GemmJob& j : jobs) out->flops += 2.0 * j.M * static_cast<double>(j.N) * j.K;
  out->uniform = uniform_tiles();
  out->issued1 = issued_per_pass();
  out->wide = wide();
  return true;
}

GemmWide JobBuilder::wide() const {
  GemmWide w;
  if (jobs.empty() || !all_sym) return w;
  w.tiles = tiles2;
  w.uniform = uniform_tiles(256);
  for (const GemmJob& j : jobs)
    w.issued1 += static_cast<double>(job_tiles(j, 256)) * 2.0 * kTileM * 256 * ((j.K + kTileK - 1) / kTileK) * kTileK;
  return w;
}

double JobBuilder::issued_per_pass() const {
  double f = 0.0;
  for (const GemmJob& j : jobs)
    f += static_cast<double>(job_tiles(j)) * 2.0 * kTileM * kTileN * ((j.K + kTileK - 1) / kTileK) * kTileK;
  return f;
}

int JobBuilder::uniform_tiles(int nt) const {
  if (jobs.empty()) return 0;
  auto start = [nt](const GemmJob& j) { return nt == 128 ? j.tile_start : j.tile_start2; };
  const int total = nt == 128 ? tiles : tiles2;
  const int t0 = jobs.size() > 1 ? start(jobs[1]) - start(jobs[0]) : total;
  for (size_t i = 0; i < jobs.size(); ++i) {
    const int next = i + 1 < jobs.size() ? start(jobs[i + 1]) : total;
    if (next - start(jobs[i]) != t0 || start(jobs[i]) != static_cast<int>(i) * t0) return 0;
  }
  return t0;
}

size_t stack_bytes(int nmat, int rows, int cols) {
  const int ld = (cols + kLdAlign - 1) / kLdAlign * kLdAlign;
  return Arena::need(static_cast<size_t>(nmat) * 2 * rows * ld * 2) + 2 * Arena::need(sizeof(int) * nmat);
}

bool arena_stack(Arena& ar, const dash_stack& like, dash_stack* out) {
  *out = like;
  out->ld = (like.cols + kLdAlign - 1) / kLdAlign * kLdAlign;
  out->data = static_cast<uint16_t*>(ar.take(static_cast<size_t>(like.nmat) * 2 * like.rows * out->ld * 2));
  out->exp = ar.take_n<int>(like.nmat);
  out->amax = ar.take_n<uint32_t>(like.nmat);
  return ar.ok;
}

void zero_padding(const dash_stack& s, cudaStream_t st) {
  // K-major TMA loads read the padding columns [cols, ld): they must hold zeros.
  if (s.cols == s.ld) return;
  cudaMemset2DAsync(reinterpret_cast<uint16_t*>(s.data) + s.cols, static_cast<size_t>(s.ld) * 2, 0,
                    static_cast<size_t>(s.ld - s.cols) * 2, static_cast<size_t>(s.nmat) * 2 * s.rows, st);
}

int JobBuilder::launch(void* ws, size_t ws_bytes, int passes, cudaStream_t st) {
  if (jobs.empty()) return DASH_OK;
  const size_t need = bytes_for(static_cast<int>(maps.size()), static_cast<int>(jobs.size()));
  if (!ws || ws_bytes < need) return DASH_EINVAL;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ws) + 127) & ~uintptr_t(127));
  CUtensorMap* d_maps = reinterpret_cast<CUtensorMap*>(base);
  GemmJob* d_jobs = reinterpret_cast<GemmJob*>(base + maps.size() * sizeof(CUtensorMap));
  // one host staging block -> one H2D copy
  staging.resize(maps.size() * sizeof(CUtensorMap) + jobs.size() * sizeof(GemmJob));
  std::memcpy(staging.data(), maps.data(), maps.size() * sizeof(CUtensorMap));
  std::memcpy(staging.data() + maps.size() * sizeof(CUtensorMap), jobs.data(), jobs.size() * sizeof(GemmJob));
  if (cudaMemcpyAsync(base, staging.data(), staging.size(), cudaMemcpyHostToDevice, st) != cudaSuccess)
    return DASH_ECUDA;
  int* counter = reinterpret_cast<int*>((reinterpret_cast<uintptr_t>(base + staging.size()) + 127) & ~uintptr_t(127));
  if (cudaMemsetAsync(counter, 0, 2 * sizeof(int), st) != cudaSuccess) return DASH_ECUDA;
  double fl = 0.0;
  for (const GemmJob& j : jobs) fl += 2.0 * j.M * static_cast<double>(j.N) * j.K;
  const GemmWide w = wide();
  return gemm_launch(d_jobs, static_cast<int>(jobs.size()), tiles, d_maps, passes, st, counter, nullptr, fl,
                     uniform_tiles(), issued_per_pass() * passes, &w);
}

}  // namespace dash

// ============================================================================ C ABI
using namespace dash;

extern "C" {

const char* dash_version(void) { return "dash-b200 0.1 (sm_100a tcgen05)"; }

unsigned long long dash_launch_count(void) { return g_launches; }
void dash_gemm_timing(int enable) { gemm_timing_enable(enable); }
int dash_gemm_timing_read(int* launches, double* ms, double* flops) {
  if (!launches || !ms || !flops) return DASH_EINVAL;
  return gemm_timing_read(launches, ms, flops);
}

int dash_gemm_timing_list(int cap, double* ms, double* flops, double* issued, int* tiles) {
  if (cap < 0 || (cap > 0 && (!ms || !flops || !issued || !tiles))) return -DASH_EINVAL;
  return gemm_timing_list(cap, ms, flops, issued, tiles);
}

int dash_device_sms(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

int dash_split(const float* src, long long src_mat_stride, int src_ld, const dash_stack* dst, void* stream) {
  if (!src || !stack_ok(dst) || src_ld < dst->cols) return DASH_EINVAL;
  return split_stack(src, src_mat_stride, src_ld, *dst, static_cast<cudaStream_t>(stream));
}

int dash_unsplit(const dash_stack* src, float* dst, long long dst_mat_stride, int dst_ld, void* stream) {
  if (!stack_ok(src) || !dst || dst_ld < src->cols) return DASH_EINVAL;
  return unsplit_stack(*src, dst, dst_mat_stride, dst_ld, static_cast<cudaStream_t>(stream));
}

size_t dash_bmm_ws_bytes(int nmat) { return JobBuilder::bytes_for(16, nmat); }

int dash_bmm(const dash_stack* a, int trans_a, const dash_stack* b, int trans_b, const dash_stack* c,
             float* f_out, long long f_mat_stride, int f_ld, float alpha, int passes, void* ws, size_t ws_bytes,
             void* stream) {
  if (!stack_ok(a) || !stack_ok(b) || (c && !stack_ok(c)) || (!c && !f_out)) return DASH_EINVAL;
  if (a->nmat != b->nmat || (c && c->nmat != a->nmat) || (passes != 1 && passes != 3 && passes != 4)) return DASH_EINVAL;
  const int M = trans_a ? a->cols : a->rows;
  const int N = trans_b ? b->rows : b->cols;
  if (c && (c->rows != M || c->cols != N)) return DASH_EINVAL;
  if (f_out && f_ld < N) return DASH_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  JobBuilder jb;
  if (c) cudaMemsetAsync(c->amax, 0, sizeof(unsigned) * c->nmat, st);
  for (int m = 0; m < a->nmat; ++m) {
    GemmJob j;
    if (!jb.operands(j, *a, m, trans_a, *b, m, trans_b)) return DASH_EINVAL;
    j.op = EPI_SPLIT;
    j.alpha = alpha;
    j.out_mat = m;
    if (c) jb.set_out(j, *c, m);
    if (f_out) {
      j.f_out = f_out + m * f_mat_stride;
      j.f_ld = f_ld;
    }
    jb.push(j);
  }
  return jb.launch(ws, ws_bytes, passes, st);
}

}  // extern "C"
