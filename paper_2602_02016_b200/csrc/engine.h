// Internal host-side interfaces shared by the DASH engine translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/dash_b200.h"
#include "types.h"

namespace dash {

bool make_stack_map(const dash_stack& s, int box_rows, CUtensorMap* out);
bool stack_ok(const dash_stack* s);
int split_stack(const float* src, long long mat_stride, int src_ld, const dash_stack& d, cudaStream_t st);
int unsplit_stack(const dash_stack& s, float* dst, long long mat_stride, int dst_ld, cudaStream_t st);
int gemm_launch(const GemmJob* d_jobs, int njobs, int total_tiles, const CUtensorMap* d_maps, int passes,
                cudaStream_t stream);

// Collects tensor maps + jobs of one grouped GEMM launch and uploads them into a workspace.
struct JobBuilder {
  struct MapKey {
    const void* data;
    int box, nmat, rows, ld;
  };
  std::vector<CUtensorMap> maps;
  std::vector<MapKey> map_keys;
  std::vector<GemmJob> jobs;
  std::vector<uint8_t> staging;
  int tiles = 0;

  void clear() {
    maps.clear();
    map_keys.clear();
    jobs.clear();
    tiles = 0;
  }
  int add_map(const dash_stack& s, int box_rows);
  bool operands(GemmJob& j, const dash_stack& a, int am, int trans_a, const dash_stack& b, int bm, int trans_b);
  void set_out(GemmJob& j, const dash_stack& c, int cm);
  void push(GemmJob& j);
  static size_t bytes_for(int nmaps, int njobs);
  int launch(void* ws, size_t ws_bytes, int passes, cudaStream_t st);
};

}  // namespace dash
