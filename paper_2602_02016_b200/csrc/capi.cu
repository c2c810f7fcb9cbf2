// C ABI of the solver layer (include/dash_b200.h).
#include "engine.h"
#include "solver.h"

using namespace dash;

static bool square_same(const dash_stack* a, const dash_stack* b) {
  return stack_ok(a) && stack_ok(b) && a->rows == a->cols && b->nmat == a->nmat && b->rows == a->rows &&
         b->cols == a->cols;
}

extern "C" {

size_t dash_ndb_ws_bytes(int n, int b) { return ndb_ws_bytes(n, b); }

int dash_ndb(const dash_stack* a, const float* inv_scale, const dash_stack* y, const dash_stack* z, float tol,
             float stall, int max_iters, int passes, int* iters, float* resid, int* conv, void* ws, size_t ws_bytes,
             void* stream) {
  if (!square_same(a, y) || !square_same(a, z) || max_iters < 1 || tol < 0.f || stall < 0.f || !iters || !resid || !conv ||
      (passes != 1 && passes != 3 && passes != 4))
    return DASH_EINVAL;
  if (ws_bytes < ndb_ws_bytes(a->nmat, a->rows)) return DASH_EINVAL;
  return ndb_solve(*a, inv_scale, *y, *z, tol, stall, max_iters, passes, iters, resid, conv, ws, ws_bytes,
                   static_cast<cudaStream_t>(stream), nullptr);
}

int dash_ndb_upper(const dash_stack* a, const float* inv_scale, const dash_stack* y, const dash_stack* z, float tol,
                   float stall, int max_iters, int passes, int outputs, int* iters, float* resid, int* conv, void* ws,
                   size_t ws_bytes, void* stream) {
  if (!square_same(a, y) || !square_same(a, z) || max_iters < 1 || tol < 0.f || stall < 0.f || !iters || !resid || !conv ||
      (passes != 1 && passes != 3 && passes != 4) || outputs < 1 || outputs > 3)
    return DASH_EINVAL;
  if (ws_bytes < ndb_ws_bytes(a->nmat, a->rows)) return DASH_EINVAL;
  return ndb_solve(*a, inv_scale, *y, *z, tol, stall, max_iters, passes, iters, resid, conv, ws, ws_bytes,
                   static_cast<cudaStream_t>(stream), nullptr, false, outputs);
}

int dash_fill_lower(const dash_stack* s, void* stream) {
  if (!stack_ok(s) || s->rows != s->cols) return DASH_EINVAL;
  return fill_lower(*s, static_cast<cudaStream_t>(stream));
}

size_t dash_cn_ws_bytes(int n, int b) { return cn_ws_bytes(n, b); }

int dash_cn(const dash_stack* a, const float* inv_scale, int p, float c, const dash_stack* x, float tol,
            float stall, int max_iters, int passes, int* iters, float* resid, int* conv, void* ws, size_t ws_bytes,
            void* stream) {
  if (!square_same(a, x) || (p != 2 && p != 4) || !(c > 0.f) || max_iters < 1 || tol < 0.f || stall < 0.f || !iters ||
      !resid || !conv || (passes != 1 && passes != 3 && passes != 4))
    return DASH_EINVAL;
  if (ws_bytes < cn_ws_bytes(a->nmat, a->rows)) return DASH_EINVAL;
  return cn_solve(*a, inv_scale, p, c, *x, tol, stall, max_iters, passes, iters, resid, conv, ws, ws_bytes,
                  static_cast<cudaStream_t>(stream), nullptr);
}

int dash_scale_stack(const dash_stack* src, const float* mult, float pw, float* f_out, long long f_mat_stride,
                     int f_ld, const dash_stack* dst, const int* gate, int src_upper, void* stream) {
  if (!stack_ok(src) || (dst && !square_same(src, dst) && !(stack_ok(dst) && dst->rows == src->rows &&
                                                              dst->cols == src->cols && dst->nmat == src->nmat)))
    return DASH_EINVAL;
  if (!f_out && !dst) return DASH_EINVAL;
  return scale_stack(*src, mult, pw, f_out, f_mat_stride, f_ld, dst, gate, src_upper,
                     static_cast<cudaStream_t>(stream));
}

int dash_scale_check(const float* scale, const int* status, int n, int group, int* ok, int* err, void* stream) {
  if (!scale || n < 1 || !ok || !err) return DASH_EINVAL;
  return scale_check(scale, status, n, group, ok, err, static_cast<cudaStream_t>(stream));
}

size_t dash_cheb_ws_bytes(int n, int b) { return cheb_ws_bytes(n, b); }

int dash_clenshaw(const dash_stack* a, const float* inv_scale, const float* mult, const double* coeffs, int degree,
                  float* f_out, const dash_stack* out, int passes, const int* gate, void* ws, size_t ws_bytes,
                  void* stream) {
  if (!stack_ok(a) || a->rows != a->cols || !coeffs || degree < 2 || (!f_out && !out) ||
      (out && !square_same(a, out)) || (passes != 1 && passes != 3 && passes != 4))
    return DASH_EINVAL;
  if (ws_bytes < cheb_ws_bytes(a->nmat, a->rows)) return DASH_EINVAL;
  return cheb_solve(*a, inv_scale, mult, coeffs, degree, f_out, out, passes, gate, ws, ws_bytes,
                    static_cast<cudaStream_t>(stream));
}

}  // extern "C"
