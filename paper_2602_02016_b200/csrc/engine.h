// Internal host-side interfaces shared by the DASH engine translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <vector>

#include "../../include/dash_b200.h"
#include "types.h"

namespace dash {

// swz: 0 none, 64 = 64-byte swizzle, anything else = 128-byte swizzle
bool make_stack_map(const dash_stack& s, int box_rows, CUtensorMap* out, int box_cols = kTileK, int box_planes = 1,
                    int swz = 128);
bool stack_ok(const dash_stack* s);
int job_tiles(const GemmJob& j, int nt = 128);  // tiles the kernel runs for one job (fewer when j.sym)
int split_stack(const float* src, long long mat_stride, int src_ld, const dash_stack& d, cudaStream_t st);
int unsplit_stack(const dash_stack& s, float* dst, long long mat_stride, int dst_ld, cudaStream_t st);
// The same launch tiled with 256-wide pair tiles (only when every job is symmetric: no per-tile partials).
struct GemmWide {
  int tiles = 0, uniform = 0;
  double issued1 = 0.0;
};
int gemm_launch(const GemmJob* d_jobs, int njobs, int total_tiles, const CUtensorMap* d_maps, int passes,
                cudaStream_t stream, int* counter, const int* gate = nullptr, double flops = 0.0, int uniform = 0,
                double issued = 0.0, const GemmWide* wide = nullptr);
void note_launch(int n = 1);  // count non-GEMM kernel launches
// fp32 cluster power iteration re-run for the blocks whose status is 3 (collapsed tensor-core pool)
int pi_retry_launch(const float* ema, int n, int d, float eps, int pool, int iters, unsigned long long seed,
                    float* scale, float* inv_scale, int* status, const int* seed_index, cudaStream_t st);
int gemm_kblock();            // K-block of the GEMM launches (64, or 32 under DASH_KB=32)
extern std::atomic<unsigned long long> g_launches;
void gemm_timing_enable(int on);
int gemm_timing_read(int* n, double* ms, double* flops);
int gemm_timing_list(int cap, double* ms, double* flops, double* issued, int* tiles);

// A grouped GEMM whose maps + jobs already live in device memory.
struct UploadedGemm {
  const GemmJob* jobs = nullptr;
  const CUtensorMap* maps = nullptr;
  int njobs = 0, tiles = 0;
  int uniform = 0;     // tiles per job when all jobs have the same count (O(1) tile -> job), else 0
  double flops = 0.0;   // algorithmic: sum over jobs of 2 M N K
  double issued1 = 0.0; // tensor-core flops issued per pass (tiles x 2 x 256 x 128 x padded K)
  GemmWide wide;        // 256-wide tiling (tiles = 0: not eligible)
  int* counter = nullptr;  // the dynamic scheduler's 2 device ints (in the caller's workspace)
  int run(int passes, cudaStream_t st, const int* gate = nullptr) const {
    return njobs ? gemm_launch(jobs, njobs, tiles, maps, passes, st, counter, gate, flops, uniform,
                               issued1 * passes, &wide)
                 : 0;
  }
};

// Bump allocator over a caller-owned workspace (128-byte aligned slices).
struct Arena {
  uint8_t* base = nullptr;
  size_t cap = 0, used = 0;
  bool ok = true;
  Arena(void* p, size_t n) : base(static_cast<uint8_t*>(p)), cap(n) {}
  void* take(size_t n) {
    size_t off = (used + 127) & ~size_t(127);
    if (!base || off + n > cap) { ok = false; return nullptr; }
    used = off + n;
    return base + off;
  }
  template <class T> T* take_n(size_t count) { return static_cast<T*>(take(count * sizeof(T))); }
  static size_t need(size_t n) { return ((n + 127) & ~size_t(127)); }
};

// Split stack carved from an arena (same nmat/rows/cols as `like`).
bool arena_stack(Arena& ar, const dash_stack& like, dash_stack* out);
size_t stack_bytes(int nmat, int rows, int cols);
void zero_padding(const dash_stack& s, cudaStream_t st);

// Collects tensor maps + jobs of one grouped GEMM launch and uploads them into a workspace.
struct JobBuilder {
  struct MapKey {
    const void* data;
    int box, nmat, rows, ld;
    int box_cols, planes;
    int swz;
  };
  std::vector<CUtensorMap> maps;
  std::vector<MapKey> map_keys;
  std::vector<GemmJob> jobs;
  std::vector<uint8_t> staging;
  int tiles = 0;
  int tiles2 = 0;        // the same jobs in 256-wide pair tiles
  bool all_sym = true;   // every job symmetric (256-wide tiling allowed)

  void clear() {
    maps.clear();
    map_keys.clear();
    jobs.clear();
    tiles = 0;
    tiles2 = 0;
    all_sym = true;
  }
  int add_map(const dash_stack& s, int box_rows, int box_cols = kTileK, int box_planes = 1, int swz = 128);
  // check = false: the caller overrides M/N/K afterwards (sub-matrices of zero-padded slots)
  bool operands(GemmJob& j, const dash_stack& a, int am, int trans_a, const dash_stack& b, int bm, int trans_b,
                bool check = true);
  void set_out(GemmJob& j, const dash_stack& c, int cm);
  void set_out2(GemmJob& j, const dash_stack& c, int cm);  // second split output (EPI_CN_M correction)
  void set_side(GemmJob& j, const dash_stack& s, int m);   // split side input (EPI_CHEB*: B_{k+2})
  // fp32 output matrix `mat` of a contiguous (nmat, rows, ld) stack (EPI_EMA: also the input), TMA-staged
  void set_fout(GemmJob& j, float* base, int nmat, int rows, int ld, int mat, bool is_input = false);
  int add_f32_map(const float* base, int nmat, int rows, int ld, int box_cols, int box_rows, bool swz);
  void push(GemmJob& j);
  static size_t bytes_for(int nmaps, int njobs);
  int launch(void* ws, size_t ws_bytes, int passes, cudaStream_t st);
  int uniform_tiles(int nt = 128) const;
  GemmWide wide() const;
  double issued_per_pass() const;
  // Upload maps + jobs into the arena (one H2D copy); the builder may be reused afterwards.
  bool upload(Arena& ar, cudaStream_t st, UploadedGemm* out);
  size_t upload_bytes() const { return bytes_for(static_cast<int>(maps.size()), static_cast<int>(jobs.size())); }
};

}  // namespace dash
