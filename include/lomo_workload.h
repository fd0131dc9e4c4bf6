/* lomo_workload.h -- fused elementwise kernels of the benchmark decoder.
 *
 * These are NOT part of the LOMO update path (include/lomo_b200.h).  They
 * implement the non-GEMM layers of workloads.Llama -- RMSNorm, rotary
 * position embedding, SwiGLU -- as one kernel per layer per direction, so
 * that the config-3 training step (LLaMA-7B) is not
 * dominated by eager PyTorch's chains of elementwise launches.  Same
 * conventions as lomo_b200.h: extern "C", plain pointers, async on `stream`,
 * 0 = ok, LOMO_E_ARG on bad arguments, cudaError_t otherwise.
 *
 * Storage dtype: LOMO_F16 or LOMO_BF16 (lomo_dtype); arithmetic in fp32 with
 * one rounding per output element.  Rows are contiguous, h % 8 == 0.
 */
#ifndef LOMO_WORKLOAD_H
#define LOMO_WORKLOAD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* y[r,:] = round(round(x[r,:] * rstd[r]) * w),  rstd[r] = 1/sqrt(mean(x[r,:]^2) + eps).
 * rstd (fp32, rows) is saved for the backward.  h <= 8192. */
int lomo_wl_rmsnorm_fwd(const void* x, const void* w, void* y, float* rstd, int64_t rows,
                        int h, int dtype, float eps, void* stream);

/* dx = rstd * (dt - n * mean(dt * n)),  n = x * rstd,  dt = dy * w;
 * dw = sum_r dy * round(n).  `partial` is fp32 scratch of
 * lomo_wl_rmsnorm_partial_rows(rows) * h floats (deterministic two-stage
 * reduction, no atomics). */
int lomo_wl_rmsnorm_bwd(const void* dy, const void* x, const void* w, const float* rstd,
                        void* dx, void* dw, float* partial, int64_t rows, int h, int dtype,
                        void* stream);
int lomo_wl_rmsnorm_partial_rows(int64_t rows);

/* The decoder's residual add fused into the norm that follows it:
 * hout = round(x + r) (the residual stream), then y = rmsnorm(hout) as above.
 * The backward's counterpart adds the residual stream's other gradient:
 * dx = round(round(rmsnorm_bwd) + dres), the sum autograd would form. */
int lomo_wl_add_rmsnorm_fwd(const void* x, const void* r, const void* w, void* hout, void* y,
                            float* rstd, int64_t rows, int h, int dtype, float eps,
                            void* stream);
int lomo_wl_rmsnorm_bwd_add(const void* dy, const void* x, const void* w, const float* rstd,
                            const void* dres, void* dx, void* dw, float* partial, int64_t rows,
                            int h, int dtype, void* stream);

/* Rotary embedding of q and k in [rows = b*s, heads, dh] layout, position
 * = row % seq; cos/sin are [seq, dh] tables in the storage dtype.
 * direction 0: out = x*cos + rotate_half(x)*sin (forward);
 * direction 1: the transpose (backward).  q/k may not alias qo/ko. */
int lomo_wl_rope(const void* q, const void* k, void* qo, void* ko, const void* cos,
                 const void* sin, int64_t rows, int seq, int heads, int dh, int dtype,
                 int direction, void* stream);

/* lomo_wl_rope with input rows `ld_in` and output rows `ld_out` elements
 * apart: the forward reads q/k as views of a fused [rows, 3*heads*dh] QKV
 * projection, the backward writes dq/dk straight into d(qkv). */
int lomo_wl_rope_ld(const void* q, const void* k, int64_t ld_in, void* qo, void* ko,
                    int64_t ld_out, const void* cos, const void* sin, int64_t rows, int seq,
                    int heads, int dh, int dtype, int direction, void* stream);

/* The fused-QKV backward in one launch: dq/dk ([batch*seq, heads, dh],
 * contiguous) through the rotary transpose into dqkv[:, 0:2h], and dv (a
 * [batch, heads, seq, dh] tensor with element strides dv_stride_b/h/s, dh
 * contiguous) copied into dqkv[:, 2h:3h]; dqkv is [batch*seq, 3h]. */
int lomo_wl_qkv_rope_bwd(const void* dq, const void* dk, const void* dv, int64_t dv_stride_b,
                         int64_t dv_stride_h, int64_t dv_stride_s, void* dqkv, const void* cos,
                         const void* sin, int64_t batch, int seq, int heads, int dh, int dtype,
                         void* stream);

/* Mean token cross entropy over logits [rows, V] (V % 8 == 0), int64
 * targets: the forward writes the per-row log-sum-exp (fp32, for the
 * backward) and the per-row loss (the caller averages it); the backward
 * writes dlogits = grad * (softmax - onehot) * inv_rows in the logits' dtype,
 * grad read from device memory (fp32 scalar). */
int lomo_wl_ce_fwd(const void* logits, const int64_t* targets, float* lse, float* loss_rows,
                   int64_t rows, int V, int dtype, void* stream);
int lomo_wl_ce_bwd(const void* logits, const int64_t* targets, const float* lse,
                   const float* grad_dev, float inv_rows, void* dlogits, int64_t rows, int V,
                   int dtype, void* stream);

/* SwiGLU over a fused gate/up projection gu [rows, 2f] (gate = gu[:, :f],
 * up = gu[:, f:]): out [rows, f] = silu(gate) * up; the backward writes
 * dgu [rows, 2f] in the same layout. */
int lomo_wl_swiglu_gu_fwd(const void* gu, void* out, int64_t rows, int64_t f, int dtype,
                          void* stream);
int lomo_wl_swiglu_gu_bwd(const void* dout, const void* gu, void* dgu, int64_t rows, int64_t f,
                          int dtype, void* stream);

/* out = silu(g) * u;  backward: dg = dout*u*silu'(g), du = dout*silu(g). */
int lomo_wl_swiglu_fwd(const void* g, const void* u, void* out, int64_t n, int dtype,
                       void* stream);
int lomo_wl_swiglu_bwd(const void* dout, const void* g, const void* u, void* dg, void* du,
                       int64_t n, int dtype, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LOMO_WORKLOAD_H */
