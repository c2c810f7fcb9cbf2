// Internal solver entry points (C++), wrapped by the C ABI in capi.cu.
#pragma once
#include <cuda_runtime.h>

#include "../../include/dash_b200.h"

namespace dash {

size_t ndb_ws_bytes(int n, int b);
bool ndb_upper_storage();
bool ndb_upper_storage(int passes);  // false for passes = 4 (FULL64 runs the K-block 32 kernel)   // the NDB iterates use upper pair-block storage (types.h)
int fill_lower(const dash_stack& s, cudaStream_t st);  // lower pair blocks <- transposed upper ones
int ndb_solve(const dash_stack& a, const float* inv_scale, const dash_stack& y_out, const dash_stack& z_out,
              float tol, float stall, int max_iters, int passes, int* iters, float* resid_out, int* conv, void* ws,
              size_t ws_bytes, cudaStream_t st, int* products, bool complete = true, int need = 3);
size_t cn_ws_bytes(int n, int b);
int cn_solve(const dash_stack& a, const float* inv_scale, int p, float c, const dash_stack& x_out, float tol,
             float stall, int max_iters, int passes, int* iters, float* resid_out, int* conv, void* ws, size_t ws_bytes,
             cudaStream_t st, int* products);
size_t cheb_ws_bytes(int n, int b);
int cheb_solve(const dash_stack& a, const float* inv_scale, const float* mult, const double* coeffs, int degree,
               float* f_out, const dash_stack* out_split, int passes, const int* gate, void* ws, size_t ws_bytes,
               cudaStream_t st);
int scale_stack(const dash_stack& src, const float* mult, float pw, float* f_out, long long f_mat_stride, int f_ld,
                const dash_stack* dst, const int* gate, int src_upper, cudaStream_t st);
int scale_check(const float* scale, const int* status, int n, int group, int* ok, int* err, cudaStream_t st);

}  // namespace dash
