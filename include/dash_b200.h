/* dash_b200.h — C ABI of the B200-native DASH optimizer step (arXiv 2602.02016).
 *
 * Every entry point is stream-ordered on the caller's CUDA stream (`stream` is a cudaStream_t passed
 * as void*), takes device pointers and plain sizes, and never allocates: scratch comes from a
 * caller-owned workspace whose size is given by the matching *_ws_bytes query.  Return codes:
 *     DASH_OK = 0, DASH_EINVAL = 1 (bad argument), DASH_ENONFINITE = 2, DASH_ECUDA = 3.
 * Python binding: paper_2602_02016_b200/_lib.py (ctypes); see INTEGRATION.md.
 *
 * Each function names the reference interface it replaces (paths relative to
 * /root/reference/pkg/src/blockshampoo/).
 */
#ifndef DASH_B200_H_
#define DASH_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DASH_OK 0
#define DASH_EINVAL 1
#define DASH_ENONFINITE 2
#define DASH_ECUDA 3

/* A stack of `nmat` rows x cols matrices in split-f16 form:
 *   value = (hi + lo) * 2^exp[m], hi/lo fp16 planes of rows x ld, ld % 64 == 0, padding zero.
 * Layout of `data`: [nmat][2][rows][ld] (plane 0 = hi, plane 1 = lo). */
typedef struct dash_stack {
  uint16_t* data;
  int nmat, rows, cols, ld;
  int* exp;           /* [nmat] power-of-two exponents */
  uint32_t* amax;     /* [nmat] float bit patterns of max |value| (NaN bits = non-finite seen) */
} dash_stack;

/* Library / build identification. */
const char* dash_version(void);
int dash_device_sms(void);

/* ---------------------------------------------------------------- dense primitives (linalg.py)
 * dash_split: fp32 stack (src[m*src_mat_stride + r*src_ld + c]) -> split-f16 stack.
 *   Replaces the storage side of linalg.quantize (linalg.py:75-79) for the tensor-core modes. */
int dash_split(const float* src, long long src_mat_stride, int src_ld, const dash_stack* dst, void* stream);
/* dash_unsplit: split-f16 stack -> fp32 (dst[m*dst_mat_stride + r*dst_ld + c]). */
int dash_unsplit(const dash_stack* src, float* dst, long long dst_mat_stride, int dst_ld, void* stream);

/* dash_bmm: C[m] = alpha * op(A[m]) @ op(B[m]) for every m (linalg.bmm, linalg.py:105-114).
 *   trans_a/trans_b: 1 = use the transpose of the stored matrix.  passes: 3 = split-f16 products
 *   (fp32-class), 1 = fp16 hi*hi only.  C may be null if f_out (fp32, [m*f_mat_stride + r*f_ld + c])
 *   is given, and vice versa. */
size_t dash_bmm_ws_bytes(int nmat);
int dash_bmm(const dash_stack* a, int trans_a, const dash_stack* b, int trans_b, const dash_stack* c,
             float* f_out, long long f_mat_stride, int f_ld, float alpha, int passes, void* ws,
             size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DASH_B200_H_ */
