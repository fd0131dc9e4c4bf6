// Fused elementwise layers of the benchmark decoder (workloads.Llama):
// RMSNorm, rotary embedding, SwiGLU -- forward and backward, one kernel each.
//
// Not on the LOMO update path.  They exist because the config-3 training
// step (LLaMA-7B, fp16, seq 1024) spent ~1/3 of its GPU time in eager
// PyTorch's chains of small elementwise kernels around the GEMMs (profiles/
// r01_summary.md); each layer here is a single HBM pass: 16-byte vector
// loads/stores, fp32 arithmetic, one rounding per output.  Reductions are
// fixed-order (no atomics), so results are run-to-run deterministic.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "lomo_b200.h"
#include "lomo_workload.h"

namespace wl {

constexpr int kThreads = 256;
constexpr int kRmsMaxVec = 4;       // RMSNorm: h <= kThreads * 4 vectors * 8 = 8192
constexpr int kTargetCtas = 296;    // RMSNorm backward: 2 CTAs per B200 SM

__device__ __forceinline__ float tof(__half x) { return __half2float(x); }
__device__ __forceinline__ float tof(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T fromf(float x);
template <> __device__ __forceinline__ __half fromf<__half>(float x) { return __float2half_rn(x); }
template <> __device__ __forceinline__ __nv_bfloat16 fromf<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}
template <typename T> __device__ __forceinline__ float rnd(float x) { return tof(fromf<T>(x)); }

template <typename T>
union Vec8 {
  uint4 u;
  T e[8];
};

__device__ __forceinline__ uint4 ld_nc(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// fixed-order block sum, result broadcast to every thread
__device__ __forceinline__ float block_sum(float v, float* sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();  // sm reuse across calls
  if (l == 0) sm[w] = v;
  __syncthreads();
  float r = 0.f;
#pragma unroll
  for (int i = 0; i < kThreads / 32; ++i) r += sm[i];
  return r;
}

// ---------------------------------------------------------------- RMSNorm
// ADD: the residual add of the decoder fused in front, hout = round(x + r)
// (the same rounding as the separate add), normalised from registers.
template <typename T, int kMaxVec, bool ADD = false>
__global__ void __launch_bounds__(kThreads)
    rms_fwd(const T* __restrict__ x, const T* __restrict__ w, T* __restrict__ y,
            float* __restrict__ rstd, int h, float eps, const T* __restrict__ res = nullptr,
            T* __restrict__ hout = nullptr) {
  __shared__ float sm[kThreads / 32];
  const int nv = h / 8;
  const size_t row = blockIdx.x;
  const uint4* xv = reinterpret_cast<const uint4*>(x + row * h);
  Vec8<T> X[kMaxVec];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kMaxVec; ++k) {
    const int i = threadIdx.x + k * kThreads;
    if (i < nv) {
      X[k].u = ld_nc(xv + i);
      if (ADD) {
        Vec8<T> Rv;
        Rv.u = ld_nc(reinterpret_cast<const uint4*>(res + row * h) + i);
#pragma unroll
        for (int e = 0; e < 8; ++e) X[k].e[e] = fromf<T>(tof(X[k].e[e]) + tof(Rv.e[e]));
        reinterpret_cast<uint4*>(hout + row * h)[i] = X[k].u;
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) ss = fmaf(tof(X[k].e[e]), tof(X[k].e[e]), ss);
    }
  }
  const float r = rsqrtf(block_sum(ss, sm) / (float)h + eps);
  if (threadIdx.x == 0) rstd[row] = r;
  const uint4* wv = reinterpret_cast<const uint4*>(w);
  uint4* yv = reinterpret_cast<uint4*>(y + row * h);
#pragma unroll
  for (int k = 0; k < kMaxVec; ++k) {
    const int i = threadIdx.x + k * kThreads;
    if (i < nv) {
      Vec8<T> W, Y;
      W.u = wv[i];
#pragma unroll
      for (int e = 0; e < 8; ++e)
        Y.e[e] = fromf<T>(rnd<T>(tof(X[k].e[e]) * r) * tof(W.e[e]));
      yv[i] = Y.u;
    }
  }
}

// One CTA per `rpc` consecutive rows, taken R rows at a time: all R rows'
// x and dy loads are issued before any arithmetic, their R dot products share
// one block reduction, and the CTA's dw partial stays in registers until the
// end (written once).
template <int R>
__device__ __forceinline__ void block_sum_r(float (&v)[R], float* sm) {  // sm: R * 8 floats
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[r] += __shfl_xor_sync(0xffffffffu, v[r], o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0)
#pragma unroll
    for (int r = 0; r < R; ++r) sm[r * (kThreads / 32) + w] = v[r];
  __syncthreads();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < kThreads / 32; ++i) t += sm[r * (kThreads / 32) + i];
    v[r] = t;
  }
}

// ADD: dx = round(round(rms_bwd) + dres) -- the residual stream's two
// gradient contributions summed as autograd would, without a separate add.
template <typename T, int kMaxVec, int R, bool ADD = false>
__global__ void __launch_bounds__(kThreads)
    rms_bwd(const T* __restrict__ dy, const T* __restrict__ x, const T* __restrict__ w,
            const float* __restrict__ rstd, T* __restrict__ dx, float* __restrict__ partial,
            int64_t rows, int h, int rpc, const T* __restrict__ dres = nullptr) {
  __shared__ float sm[R * (kThreads / 32)];
  const int nv = h / 8;
  const uint4* wv = reinterpret_cast<const uint4*>(w);
  float DW[kMaxVec][8];
  Vec8<T> Wt[kMaxVec];
#pragma unroll
  for (int k = 0; k < kMaxVec; ++k) {
    const int i = threadIdx.x + k * kThreads;
    Wt[k].u = i < nv ? wv[i] : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int e = 0; e < 8; ++e) DW[k][e] = 0.f;
  }
  const int64_t r0 = (int64_t)blockIdx.x * rpc;
  const int64_t r1 = min(r0 + rpc, rows);
  for (int64_t rb = r0; rb < r1; rb += R) {
    Vec8<T> X[R][kMaxVec], D[R][kMaxVec];
    float rs[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t row = rb + r;
      rs[r] = row < r1 ? rstd[row] : 0.f;
#pragma unroll
      for (int k = 0; k < kMaxVec; ++k) {
        const int i = threadIdx.x + k * kThreads;
        if (row < r1 && i < nv) {
          X[r][k].u = ld_nc(reinterpret_cast<const uint4*>(x + row * h) + i);
          D[r][k].u = ld_nc(reinterpret_cast<const uint4*>(dy + row * h) + i);
        } else {
          X[r][k].u = make_uint4(0, 0, 0, 0);
          D[r][k].u = make_uint4(0, 0, 0, 0);
        }
      }
    }
    float dot[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      dot[r] = 0.f;
#pragma unroll
      for (int k = 0; k < kMaxVec; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float n = tof(X[r][k].e[e]) * rs[r];
          const float d = tof(D[r][k].e[e]);
          const float dt = rnd<T>(d * tof(Wt[k].e[e]));  // grad of round(n) * w w.r.t. round(n)
          DW[k][e] = fmaf(d, rnd<T>(n), DW[k][e]);        // grad w.r.t. w
          dot[r] = fmaf(dt, n, dot[r]);
        }
    }
    block_sum_r<R>(dot, sm);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t row = rb + r;
      const float m = dot[r] / (float)h;
#pragma unroll
      for (int k = 0; k < kMaxVec; ++k) {
        const int i = threadIdx.x + k * kThreads;
        if (row < r1 && i < nv) {
          Vec8<T> O, Rg;
          if (ADD) Rg.u = ld_nc(reinterpret_cast<const uint4*>(dres + row * h) + i);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float n = tof(X[r][k].e[e]) * rs[r];
            const float dt = rnd<T>(tof(D[r][k].e[e]) * tof(Wt[k].e[e]));
            O.e[e] = fromf<T>(rs[r] * (dt - n * m));
            if (ADD) O.e[e] = fromf<T>(tof(O.e[e]) + tof(Rg.e[e]));
          }
          reinterpret_cast<uint4*>(dx + row * h)[i] = O.u;
        }
      }
    }
  }
  float* pr = partial + (size_t)blockIdx.x * h;
#pragma unroll
  for (int k = 0; k < kMaxVec; ++k) {
    const int i = threadIdx.x + k * kThreads;
    if (i < nv) {
      float4* p4 = reinterpret_cast<float4*>(pr + (size_t)i * 8);
      p4[0] = make_float4(DW[k][0], DW[k][1], DW[k][2], DW[k][3]);
      p4[1] = make_float4(DW[k][4], DW[k][5], DW[k][6], DW[k][7]);
    }
  }
}

// dw[j] = sum over the CTA partials.  32 columns x 8 row-slices per CTA: each
// warp sums every 8th partial row of its 32 columns (independent loads in
// flight), then warp 0 adds the 8 slice sums in slice order (deterministic).
template <typename T>
__global__ void __launch_bounds__(kThreads)
    rms_dw_reduce(const float* __restrict__ partial, T* __restrict__ dw, int nparts, int h) {
  __shared__ float sm[kThreads / 32][33];
  const int lane = threadIdx.x & 31, slice = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (j < h) {
#pragma unroll 4
    for (int c = slice; c < nparts; c += kThreads / 32) s += partial[(size_t)c * h + j];
  }
  sm[slice][lane] = s;
  __syncthreads();
  if (slice == 0 && j < h) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < kThreads / 32; ++i) t += sm[i][lane];
    dw[j] = fromf<T>(t);
  }
}

// ---------------------------------------------------------------- rotary
// one thread per (tensor, row, head, 8-element group of the first half)
template <typename T>
__global__ void __launch_bounds__(kThreads)
    rope(const T* __restrict__ q, const T* __restrict__ k, T* __restrict__ qo,
         T* __restrict__ ko, const T* __restrict__ cs, const T* __restrict__ sn, int64_t rows,
         int seq, int heads, int dh, int bwd, int64_t ld_in, int64_t ld_out) {
  const int half = dh / 2, gph = half / 8;
  const int64_t per_tensor = rows * heads * gph;
  const int64_t total = 2 * per_tensor;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const bool is_k = t >= per_tensor;
    const int64_t u = is_k ? t - per_tensor : t;
    const int gi = (int)(u % gph);
    const int64_t rh = u / gph;              // row * heads + head
    const int pos = (int)((rh / heads) % seq);
    const T* src = (is_k ? k : q) + (rh / heads) * ld_in + (rh % heads) * dh;
    T* dst = (is_k ? ko : qo) + (rh / heads) * ld_out + (rh % heads) * dh;
    Vec8<T> X1, X2, C1, C2, S1, S2, O1, O2;
    X1.u = ld_nc(src + gi * 8);
    X2.u = ld_nc(src + half + gi * 8);
    const T* cr = cs + (size_t)pos * dh;
    const T* sr = sn + (size_t)pos * dh;
    C1.u = *reinterpret_cast<const uint4*>(cr + gi * 8);
    C2.u = *reinterpret_cast<const uint4*>(cr + half + gi * 8);
    S1.u = *reinterpret_cast<const uint4*>(sr + gi * 8);
    S2.u = *reinterpret_cast<const uint4*>(sr + half + gi * 8);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float x1 = tof(X1.e[e]), x2 = tof(X2.e[e]);
      const float c1 = tof(C1.e[e]), c2 = tof(C2.e[e]);
      const float s1 = tof(S1.e[e]), s2 = tof(S2.e[e]);
      if (!bwd) {  // out = x*cos + cat(-x2, x1)*sin
        O1.e[e] = fromf<T>(x1 * c1 - x2 * s1);
        O2.e[e] = fromf<T>(x2 * c2 + x1 * s2);
      } else {     // its transpose
        O1.e[e] = fromf<T>(x1 * c1 + x2 * s2);
        O2.e[e] = fromf<T>(x2 * c2 - x1 * s1);
      }
    }
    *reinterpret_cast<uint4*>(dst + gi * 8) = O1.u;
    *reinterpret_cast<uint4*>(dst + half + gi * 8) = O2.u;
  }
}

// The fused-QKV backward in one launch: the rotary transpose of dq/dk
// (contiguous [rows, heads, dh]) into d(qkv)[:, 0:2h] and the copy of dv
// (any [b, heads, s, dh] strides with dh contiguous, as SDPA returns it) into
// d(qkv)[:, 2h:3h].  One thread per 8-element group, as in `rope`.
template <typename T>
__global__ void __launch_bounds__(kThreads)
    qkv_bwd(const T* __restrict__ dq, const T* __restrict__ dk, const T* __restrict__ dv,
            int64_t vsb, int64_t vsh, int64_t vss, T* __restrict__ dqkv,
            const T* __restrict__ cs, const T* __restrict__ sn, int64_t rows, int seq, int heads,
            int dh) {
  const int half = dh / 2, gph = half / 8, gv = dh / 8;
  const int64_t per_rot = rows * heads * gph;      // per rotated tensor
  const int64_t total = 2 * per_rot + rows * heads * gv;
  const int64_t h = (int64_t)heads * dh, ld = 3 * h;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t >= 2 * per_rot) {  // dv copy
      const int64_t u = t - 2 * per_rot;
      const int gi = (int)(u % gv);
      const int64_t rh = u / gv;
      const int64_t row = rh / heads, hd = rh % heads;
      const int64_t b = row / seq, sp = row % seq;
      const uint4 x = ld_nc(dv + b * vsb + hd * vsh + sp * vss + gi * 8);
      *reinterpret_cast<uint4*>(dqkv + row * ld + 2 * h + hd * dh + gi * 8) = x;
      continue;
    }
    const bool is_k = t >= per_rot;
    const int64_t u = is_k ? t - per_rot : t;
    const int gi = (int)(u % gph);
    const int64_t rh = u / gph;
    const int pos = (int)((rh / heads) % seq);
    const T* src = (is_k ? dk : dq) + rh * dh;
    T* dst = dqkv + (rh / heads) * ld + (is_k ? h : 0) + (rh % heads) * dh;
    Vec8<T> X1, X2, C1, C2, S1, S2, O1, O2;
    X1.u = ld_nc(src + gi * 8);
    X2.u = ld_nc(src + half + gi * 8);
    const T* cr = cs + (size_t)pos * dh;
    const T* sr = sn + (size_t)pos * dh;
    C1.u = *reinterpret_cast<const uint4*>(cr + gi * 8);
    C2.u = *reinterpret_cast<const uint4*>(cr + half + gi * 8);
    S1.u = *reinterpret_cast<const uint4*>(sr + gi * 8);
    S2.u = *reinterpret_cast<const uint4*>(sr + half + gi * 8);
#pragma unroll
    for (int e = 0; e < 8; ++e) {  // the transpose of the forward rotation
      const float x1 = tof(X1.e[e]), x2 = tof(X2.e[e]);
      O1.e[e] = fromf<T>(x1 * tof(C1.e[e]) + x2 * tof(S2.e[e]));
      O2.e[e] = fromf<T>(x2 * tof(C2.e[e]) - x1 * tof(S1.e[e]));
    }
    *reinterpret_cast<uint4*>(dst + gi * 8) = O1.u;
    *reinterpret_cast<uint4*>(dst + half + gi * 8) = O2.u;
  }
}

// ---------------------------------------------------------------- cross entropy
// Mean token cross entropy over fp16/bf16 logits [rows, V] (the decoder's
// loss, ops.py:332-352 semantics: mean over positions), one CTA per row.
// Forward: lse[r] = max + log(sum exp(x - max)), loss_rows[r] = lse - x[t_r].
// Backward: dlogits = g * (exp(x - lse) - onehot) * inv_rows, g the upstream
// gradient read from device memory (it carries the loss scale), one rounding.
__device__ __forceinline__ void row_max_sum(float& m, float& sexp, float* sm_m, float* sm_s) {
  // combine (max, sum exp) pairs: warp shuffle, then across warps in order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, sexp, o);
    const float mm = fmaxf(m, m2);
    sexp = (m == -INFINITY ? 0.f : sexp * __expf(m - mm)) +
           (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
    m = mm;
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) {
    sm_m[w] = m;
    sm_s[w] = sexp;
  }
  __syncthreads();
  float M = -INFINITY, S = 0.f;
#pragma unroll
  for (int i = 0; i < kThreads / 32; ++i) {
    const float mm = fmaxf(M, sm_m[i]);
    S = (M == -INFINITY ? 0.f : S * __expf(M - mm)) +
        (sm_m[i] == -INFINITY ? 0.f : sm_s[i] * __expf(sm_m[i] - mm));
    M = mm;
  }
  m = M;
  sexp = S;
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
    ce_fwd(const T* __restrict__ logits, const int64_t* __restrict__ tgt, int V,
           float* __restrict__ lse, float* __restrict__ loss_rows) {
  __shared__ float sm_m[kThreads / 32], sm_s[kThreads / 32];
  const int64_t r = blockIdx.x;
  const uint4* xv = reinterpret_cast<const uint4*>(logits + r * V);
  const int nv = V / 8;
  float m = -INFINITY, se = 0.f;
  for (int i = threadIdx.x; i < nv; i += kThreads) {
    Vec8<T> X;
    X.u = ld_nc(xv + i);
    float vm = -INFINITY;
#pragma unroll
    for (int e = 0; e < 8; ++e) vm = fmaxf(vm, tof(X.e[e]));
    const float mm = fmaxf(m, vm);
    float acc = (m == -INFINITY) ? 0.f : se * __expf(m - mm);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc += __expf(tof(X.e[e]) - mm);
    se = acc;
    m = mm;
  }
  row_max_sum(m, se, sm_m, sm_s);
  if (threadIdx.x == 0) {
    const float l = m + __logf(se);
    lse[r] = l;
    loss_rows[r] = l - tof(logits[r * V + tgt[r]]);
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
    ce_bwd(const T* __restrict__ logits, const int64_t* __restrict__ tgt,
           const float* __restrict__ lse, const float* __restrict__ gptr, float inv_rows,
           T* __restrict__ dlogits, int V) {
  const int64_t r = blockIdx.x;
  const float g = *gptr * inv_rows, l = lse[r];
  const int64_t t = tgt[r];
  const uint4* xv = reinterpret_cast<const uint4*>(logits + r * V);
  uint4* dv = reinterpret_cast<uint4*>(dlogits + r * V);
  const int nv = V / 8;
  for (int i = threadIdx.x; i < nv; i += kThreads) {
    Vec8<T> X, D;
    X.u = ld_nc(xv + i);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float p = __expf(tof(X.e[e]) - l);
      D.e[e] = fromf<T>(g * (p - ((int64_t)(i * 8 + e) == t ? 1.f : 0.f)));
    }
    dv[i] = D.u;
  }
}

// ---------------------------------------------------------------- SwiGLU
__device__ __forceinline__ float sigmoidf_(float g) { return 1.f / (1.f + __expf(-g)); }

template <typename T>
__global__ void __launch_bounds__(kThreads)
    swiglu_fwd(const T* __restrict__ g, const T* __restrict__ u, T* __restrict__ out,
               int64_t nvec) {
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  const uint4* uv = reinterpret_cast<const uint4*>(u);
  uint4* ov = reinterpret_cast<uint4*>(out);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    Vec8<T> G, U, O;
    G.u = ld_nc(gv + i);
    U.u = ld_nc(uv + i);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float x = tof(G.e[e]);
      O.e[e] = fromf<T>(x * sigmoidf_(x) * tof(U.e[e]));
    }
    ov[i] = O.u;
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
    swiglu_bwd(const T* __restrict__ dout, const T* __restrict__ g, const T* __restrict__ u,
               T* __restrict__ dg, T* __restrict__ du, int64_t nvec) {
  const uint4* dv = reinterpret_cast<const uint4*>(dout);
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  const uint4* uv = reinterpret_cast<const uint4*>(u);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    Vec8<T> D, G, U, DG, DU;
    D.u = ld_nc(dv + i);
    G.u = ld_nc(gv + i);
    U.u = ld_nc(uv + i);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float x = tof(G.e[e]), d = tof(D.e[e]), y = tof(U.e[e]);
      const float s = sigmoidf_(x);
      DU.e[e] = fromf<T>(d * x * s);
      DG.e[e] = fromf<T>(d * y * s * (1.f + x * (1.f - s)));
    }
    reinterpret_cast<uint4*>(dg)[i] = DG.u;
    reinterpret_cast<uint4*>(du)[i] = DU.u;
  }
}

// Fused gate/up layout: gu[r, 0:f] = gate, gu[r, f:2f] = up (one GEMM output);
// out[r, :] = silu(gate) * up, and the backward writes d(gu) in the same
// layout, so neither direction needs a split or a concatenation copy.
template <typename T>
__global__ void __launch_bounds__(kThreads)
    swiglu_gu_fwd(const T* __restrict__ gu, T* __restrict__ out, int64_t rows, int64_t fv) {
  const int64_t total = rows * fv;  // fv = f / 8 vectors per row half
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / fv, c = i - r * fv;
    const uint4* row = reinterpret_cast<const uint4*>(gu) + r * 2 * fv;
    Vec8<T> G, U, O;
    G.u = ld_nc(row + c);
    U.u = ld_nc(row + fv + c);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float x = tof(G.e[e]);
      O.e[e] = fromf<T>(x * sigmoidf_(x) * tof(U.e[e]));
    }
    reinterpret_cast<uint4*>(out)[i] = O.u;
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
    swiglu_gu_bwd(const T* __restrict__ dout, const T* __restrict__ gu, T* __restrict__ dgu,
                  int64_t rows, int64_t fv) {
  const int64_t total = rows * fv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / fv, c = i - r * fv;
    const uint4* row = reinterpret_cast<const uint4*>(gu) + r * 2 * fv;
    uint4* drow = reinterpret_cast<uint4*>(dgu) + r * 2 * fv;
    Vec8<T> D, G, U, DG, DU;
    D.u = ld_nc(reinterpret_cast<const uint4*>(dout) + i);
    G.u = ld_nc(row + c);
    U.u = ld_nc(row + fv + c);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float x = tof(G.e[e]), d = tof(D.e[e]), y = tof(U.e[e]);
      const float s = sigmoidf_(x);
      DU.e[e] = fromf<T>(d * x * s);
      DG.e[e] = fromf<T>(d * y * s * (1.f + x * (1.f - s)));
    }
    drow[c] = DG.u;
    drow[fv + c] = DU.u;
  }
}

inline int grid_for(int64_t work) {
  // enough CTAs to fill 148 SMs x 8 resident CTAs, no more than the work
  const int64_t cap = 148 * 8;
  const int64_t need = (work + kThreads - 1) / kThreads;
  return (int)(need < cap ? (need > 0 ? need : 1) : cap);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <template <typename> class F, typename... A>
int dispatch(int dtype, A... a) {
  if (dtype == LOMO_F16) return F<__half>::run(a...);
  if (dtype == LOMO_BF16) return F<__nv_bfloat16>::run(a...);
  return LOMO_E_ARG;
}

inline int status() { return (int)cudaGetLastError(); }

template <typename T>
struct RmsFwd {
  static int run(const void* x, const void* w, void* y, float* rstd, int64_t rows, int h,
                 float eps, const void* res, void* hout, cudaStream_t s) {
    // vectors per thread as a template constant: registers hold the row
#define WL_RMS_FWD(NV)                                                                       \
  if (res) rms_fwd<T, NV, true><<<(unsigned)rows, kThreads, 0, s>>>(                         \
      (const T*)x, (const T*)w, (T*)y, rstd, h, eps, (const T*)res, (T*)hout);               \
  else rms_fwd<T, NV><<<(unsigned)rows, kThreads, 0, s>>>((const T*)x, (const T*)w, (T*)y, \
                                                          rstd, h, eps)
    switch ((h / 8 + kThreads - 1) / kThreads) {
      case 1: WL_RMS_FWD(1); break;
      case 2: WL_RMS_FWD(2); break;
      case 3: WL_RMS_FWD(3); break;
      default: WL_RMS_FWD(4); break;
    }
#undef WL_RMS_FWD
    return status();
  }
};

inline int rms_rows_per_cta(int64_t rows) { return (int)((rows + kTargetCtas - 1) / kTargetCtas); }

template <typename T>
struct RmsBwd {
  static int run(const void* dy, const void* x, const void* w, const float* rstd, void* dx,
                 void* dw, float* partial, int64_t rows, int h, const void* dres,
                 cudaStream_t s) {
    const int rpc = rms_rows_per_cta(rows);
    const int nparts = (int)((rows + rpc - 1) / rpc);
#define WL_RMS_BWD(NV, R)                                                                   \
  if (dres) rms_bwd<T, NV, R, true><<<nparts, kThreads, 0, s>>>(                            \
      (const T*)dy, (const T*)x, (const T*)w, rstd, (T*)dx, partial, rows, h, rpc,          \
      (const T*)dres);                                                                      \
  else rms_bwd<T, NV, R><<<nparts, kThreads, 0, s>>>((const T*)dy, (const T*)x, (const T*)w, \
                                                     rstd, (T*)dx, partial, rows, h, rpc)
    switch ((h / 8 + kThreads - 1) / kThreads) {  // rows in flight x vectors <= 8
      case 1: WL_RMS_BWD(1, 4); break;
      case 2: WL_RMS_BWD(2, 2); break;
      case 3: WL_RMS_BWD(3, 2); break;
      default: WL_RMS_BWD(4, 2); break;
    }
#undef WL_RMS_BWD
    rms_dw_reduce<T><<<(h + 31) / 32, kThreads, 0, s>>>(partial, (T*)dw, nparts, h);
    return status();
  }
};

template <typename T>
struct Rope {
  static int run(const void* q, const void* k, void* qo, void* ko, const void* c,
                 const void* sn, int64_t rows, int seq, int heads, int dh, int bwd,
                 int64_t ld_in, int64_t ld_out, cudaStream_t s) {
    const int64_t work = 2 * rows * heads * (dh / 16);
    rope<T><<<grid_for(work), kThreads, 0, s>>>((const T*)q, (const T*)k, (T*)qo, (T*)ko,
                                                (const T*)c, (const T*)sn, rows, seq, heads, dh,
                                                bwd, ld_in, ld_out);
    return status();
  }
};

template <typename T>
struct SwigluFwd {
  static int run(const void* g, const void* u, void* o, int64_t n, cudaStream_t s) {
    swiglu_fwd<T><<<grid_for(n / 8), kThreads, 0, s>>>((const T*)g, (const T*)u, (T*)o, n / 8);
    return status();
  }
};

template <typename T>
struct SwigluBwd {
  static int run(const void* d, const void* g, const void* u, void* dg, void* du, int64_t n,
                 cudaStream_t s) {
    swiglu_bwd<T><<<grid_for(n / 8), kThreads, 0, s>>>((const T*)d, (const T*)g, (const T*)u,
                                                       (T*)dg, (T*)du, n / 8);
    return status();
  }
};

template <typename T>
struct QkvBwd {
  static int run(const void* dq, const void* dk, const void* dv, int64_t vsb, int64_t vsh,
                 int64_t vss, void* dqkv, const void* c, const void* sn, int64_t rows, int seq,
                 int heads, int dh, cudaStream_t s) {
    const int64_t work = rows * heads * (2 * (dh / 16) + dh / 8);  // threads of qkv_bwd
    qkv_bwd<T><<<grid_for(work), kThreads, 0, s>>>((const T*)dq, (const T*)dk, (const T*)dv, vsb,
                                                   vsh, vss, (T*)dqkv, (const T*)c,
                                                   (const T*)sn, rows, seq, heads, dh);
    return status();
  }
};

template <typename T>
struct Ce {
  static int run(const void* logits, const int64_t* tgt, float* lse, float* loss_rows,
                 const float* g, float inv_rows, void* dlogits, int64_t rows, int V, int bwd,
                 cudaStream_t s) {
    if (!bwd)
      ce_fwd<T><<<(unsigned)rows, kThreads, 0, s>>>((const T*)logits, tgt, V, lse, loss_rows);
    else
      ce_bwd<T><<<(unsigned)rows, kThreads, 0, s>>>((const T*)logits, tgt, lse, g, inv_rows,
                                                    (T*)dlogits, V);
    return status();
  }
};

template <typename T>
struct SwigluGu {
  static int run(const void* a, const void* b, void* c, int64_t rows, int64_t f, int bwd,
                 cudaStream_t s) {
    const int64_t fv = f / 8;
    if (!bwd)
      swiglu_gu_fwd<T><<<grid_for(rows * fv), kThreads, 0, s>>>((const T*)a, (T*)c, rows, fv);
    else
      swiglu_gu_bwd<T><<<grid_for(rows * fv), kThreads, 0, s>>>((const T*)a, (const T*)b, (T*)c,
                                                               rows, fv);
    return status();
  }
};

}  // namespace wl

extern "C" {

int lomo_wl_rmsnorm_partial_rows(int64_t rows) {
  if (rows <= 0) return 0;
  const int rpc = wl::rms_rows_per_cta(rows);
  return (int)((rows + rpc - 1) / rpc);
}

int lomo_wl_rmsnorm_fwd(const void* x, const void* w, void* y, float* rstd, int64_t rows, int h,
                        int dtype, float eps, void* stream) {
  if (rows < 0 || h <= 0 || h % 8 || h > wl::kThreads * wl::kRmsMaxVec * 8) return LOMO_E_ARG;
  if (rows == 0) return 0;
  if (!x || !w || !y || !rstd || !wl::aligned16(x) || !wl::aligned16(w) || !wl::aligned16(y))
    return LOMO_E_ARG;
  return wl::dispatch<wl::RmsFwd>(dtype, x, w, y, rstd, rows, h, eps, (const void*)nullptr,
                                  (void*)nullptr, (cudaStream_t)stream);
}

int lomo_wl_add_rmsnorm_fwd(const void* x, const void* r, const void* w, void* hout, void* y,
                            float* rstd, int64_t rows, int h, int dtype, float eps,
                            void* stream) {
  if (rows < 0 || h <= 0 || h % 8 || h > wl::kThreads * wl::kRmsMaxVec * 8) return LOMO_E_ARG;
  if (rows == 0) return 0;
  if (!x || !r || !w || !hout || !y || !rstd) return LOMO_E_ARG;
  if (!wl::aligned16(x) || !wl::aligned16(r) || !wl::aligned16(w) || !wl::aligned16(hout) ||
      !wl::aligned16(y))
    return LOMO_E_ARG;
  return wl::dispatch<wl::RmsFwd>(dtype, x, w, y, rstd, rows, h, eps, r, hout,
                                  (cudaStream_t)stream);
}

int lomo_wl_rmsnorm_bwd(const void* dy, const void* x, const void* w, const float* rstd,
                        void* dx, void* dw, float* partial, int64_t rows, int h, int dtype,
                        void* stream) {
  if (rows <= 0 || h <= 0 || h % 8 || h > wl::kThreads * wl::kRmsMaxVec * 8) return LOMO_E_ARG;
  if (!dy || !x || !w || !rstd || !dx || !dw || !partial) return LOMO_E_ARG;
  if (!wl::aligned16(dy) || !wl::aligned16(x) || !wl::aligned16(w) || !wl::aligned16(dx) ||
      !wl::aligned16(partial))
    return LOMO_E_ARG;
  return wl::dispatch<wl::RmsBwd>(dtype, dy, x, w, rstd, dx, dw, partial, rows, h,
                                  (const void*)nullptr, (cudaStream_t)stream);
}

int lomo_wl_rmsnorm_bwd_add(const void* dy, const void* x, const void* w, const float* rstd,
                            const void* dres, void* dx, void* dw, float* partial, int64_t rows,
                            int h, int dtype, void* stream) {
  if (rows <= 0 || h <= 0 || h % 8 || h > wl::kThreads * wl::kRmsMaxVec * 8) return LOMO_E_ARG;
  if (!dy || !x || !w || !rstd || !dres || !dx || !dw || !partial) return LOMO_E_ARG;
  if (!wl::aligned16(dy) || !wl::aligned16(x) || !wl::aligned16(w) || !wl::aligned16(dx) ||
      !wl::aligned16(dres) || !wl::aligned16(partial))
    return LOMO_E_ARG;
  return wl::dispatch<wl::RmsBwd>(dtype, dy, x, w, rstd, dx, dw, partial, rows, h, dres,
                                  (cudaStream_t)stream);
}

int lomo_wl_rope(const void* q, const void* k, void* qo, void* ko, const void* cos,
                 const void* sin, int64_t rows, int seq, int heads, int dh, int dtype,
                 int direction, void* stream) {
  if (rows < 0 || seq <= 0 || heads <= 0 || dh <= 0 || dh % 16 || (direction & ~1))
    return LOMO_E_ARG;
  if (rows == 0) return 0;
  if (!q || !k || !qo || !ko || !cos || !sin || q == qo || k == ko) return LOMO_E_ARG;
  if (!wl::aligned16(q) || !wl::aligned16(k) || !wl::aligned16(qo) || !wl::aligned16(ko) ||
      !wl::aligned16(cos) || !wl::aligned16(sin))
    return LOMO_E_ARG;
  return wl::dispatch<wl::Rope>(dtype, q, k, qo, ko, cos, sin, rows, seq, heads, dh, direction,
                                (int64_t)heads * dh, (int64_t)heads * dh, (cudaStream_t)stream);
}

int lomo_wl_rope_ld(const void* q, const void* k, int64_t ld_in, void* qo, void* ko,
                    int64_t ld_out, const void* cos, const void* sin, int64_t rows, int seq,
                    int heads, int dh, int dtype, int direction, void* stream) {
  if (rows < 0 || seq <= 0 || heads <= 0 || dh <= 0 || dh % 16 || (direction & ~1))
    return LOMO_E_ARG;
  if (ld_in < (int64_t)heads * dh || ld_in % 8 || ld_out < (int64_t)heads * dh || ld_out % 8)
    return LOMO_E_ARG;
  if (rows == 0) return 0;
  if (!q || !k || !qo || !ko || !cos || !sin || q == qo || k == ko) return LOMO_E_ARG;
  if (!wl::aligned16(q) || !wl::aligned16(k) || !wl::aligned16(qo) || !wl::aligned16(ko) ||
      !wl::aligned16(cos) || !wl::aligned16(sin))
    return LOMO_E_ARG;
  return wl::dispatch<wl::Rope>(dtype, q, k, qo, ko, cos, sin, rows, seq, heads, dh, direction,
                                ld_in, ld_out, (cudaStream_t)stream);
}

int lomo_wl_qkv_rope_bwd(const void* dq, const void* dk, const void* dv, int64_t dv_stride_b,
                         int64_t dv_stride_h, int64_t dv_stride_s, void* dqkv, const void* cos,
                         const void* sin, int64_t batch, int seq, int heads, int dh, int dtype,
                         void* stream) {
  if (batch < 0 || seq <= 0 || heads <= 0 || dh <= 0 || dh % 16) return LOMO_E_ARG;
  if (batch == 0) return 0;
  if (!dq || !dk || !dv || !dqkv || !cos || !sin) return LOMO_E_ARG;
  if (!wl::aligned16(dq) || !wl::aligned16(dk) || !wl::aligned16(dv) || !wl::aligned16(dqkv) ||
      !wl::aligned16(cos) || !wl::aligned16(sin))
    return LOMO_E_ARG;
  if (dv_stride_b % 8 || dv_stride_h % 8 || dv_stride_s % 8) return LOMO_E_ARG;
  return wl::dispatch<wl::QkvBwd>(dtype, dq, dk, dv, dv_stride_b, dv_stride_h, dv_stride_s, dqkv,
                                  cos, sin, batch * (int64_t)seq, seq, heads, dh,
                                  (cudaStream_t)stream);
}

int lomo_wl_ce_fwd(const void* logits, const int64_t* targets, float* lse, float* loss_rows,
                   int64_t rows, int V, int dtype, void* stream) {
  if (rows < 0 || V <= 0 || V % 8 || rows > INT32_MAX) return LOMO_E_ARG;
  if (rows == 0) return 0;
  if (!logits || !targets || !lse || !loss_rows || !wl::aligned16(logits)) return LOMO_E_ARG;
  return wl::dispatch<wl::Ce>(dtype, logits, targets, lse, loss_rows, (const float*)nullptr, 0.f,
                              (void*)nullptr, rows, V, 0, (cudaStream_t)stream);
}

int lomo_wl_ce_bwd(const void* logits, const int64_t* targets, const float* lse,
                   const float* grad_dev, float inv_rows, void* dlogits, int64_t rows, int V,
                   int dtype, void* stream) {
  if (rows < 0 || V <= 0 || V % 8 || rows > INT32_MAX) return LOMO_E_ARG;
  if (rows == 0) return 0;
  if (!logits || !targets || !lse || !grad_dev || !dlogits || !wl::aligned16(logits) ||
      !wl::aligned16(dlogits))
    return LOMO_E_ARG;
  return wl::dispatch<wl::Ce>(dtype, logits, targets, (float*)lse, (float*)nullptr, grad_dev,
                              inv_rows, dlogits, rows, V, 1, (cudaStream_t)stream);
}

int lomo_wl_swiglu_gu_fwd(const void* gu, void* out, int64_t rows, int64_t f, int dtype,
                          void* stream) {
  if (rows < 0 || f <= 0 || f % 8) return LOMO_E_ARG;
  if (rows == 0) return 0;
  if (!gu || !out || !wl::aligned16(gu) || !wl::aligned16(out)) return LOMO_E_ARG;
  return wl::dispatch<wl::SwigluGu>(dtype, gu, (const void*)nullptr, out, rows, f, 0,
                                    (cudaStream_t)stream);
}

int lomo_wl_swiglu_gu_bwd(const void* dout, const void* gu, void* dgu, int64_t rows, int64_t f,
                          int dtype, void* stream) {
  if (rows < 0 || f <= 0 || f % 8) return LOMO_E_ARG;
  if (rows == 0) return 0;
  if (!dout || !gu || !dgu || !wl::aligned16(dout) || !wl::aligned16(gu) || !wl::aligned16(dgu))
    return LOMO_E_ARG;
  return wl::dispatch<wl::SwigluGu>(dtype, dout, gu, dgu, rows, f, 1, (cudaStream_t)stream);
}

int lomo_wl_swiglu_fwd(const void* g, const void* u, void* out, int64_t n, int dtype,
                       void* stream) {
  if (n < 0 || n % 8) return LOMO_E_ARG;
  if (n == 0) return 0;
  if (!g || !u || !out || !wl::aligned16(g) || !wl::aligned16(u) || !wl::aligned16(out))
    return LOMO_E_ARG;
  return wl::dispatch<wl::SwigluFwd>(dtype, g, u, out, n, (cudaStream_t)stream);
}

int lomo_wl_swiglu_bwd(const void* dout, const void* g, const void* u, void* dg, void* du,
                       int64_t n, int dtype, void* stream) {
  if (n < 0 || n % 8) return LOMO_E_ARG;
  if (n == 0) return 0;
  if (!dout || !g || !u || !dg || !du || !wl::aligned16(dout) || !wl::aligned16(g) ||
      !wl::aligned16(u) || !wl::aligned16(dg) || !wl::aligned16(du))
    return LOMO_E_ARG;
  return wl::dispatch<wl::SwigluBwd>(dtype, dout, g, u, dg, du, n, (cudaStream_t)stream);
}

}  // extern "C"
