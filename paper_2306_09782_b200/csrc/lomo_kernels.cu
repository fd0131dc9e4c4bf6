// lomo_kernels.cu -- sm_100a kernels behind include/lomo_b200.h.
//
// K1  lomo_fused_update        p <- round(p - lr * coef * clip(g * inv_scale))
//     reference: optim.py:52-54 (apply_update), tensor.py:30-38,74-81 (write-back
//     rounding), stabilize.py:163-176 (value clip hook), stabilize.py:215-224
//     (update_hook).  HBM-bound streaming kernel, 6 B/elem at 16-bit storage.
// K2  lomo_probe               sumsq[slot] = sum((g*inv_scale)^2), overflow flag
//     reference: stabilize.py:190-200 (probe_hook).  2 B/elem at 16-bit.
// K3a lomo_finalize_norm       N, clip coef, skip, LossScaler.on_overflow
//     reference: stabilize.py:201-213, 94-127, 155-159.
// K3b lomo_scaler_on_clean     LossScaler.on_clean (stabilize.py:123-127, :228-229)
// K4  lomo_fused_rs_update / _probe(_keep), lomo_fused_mc_*: the sharded
//     mode's reduce-scatter fused with K1 / K2 over peer memory (CUDA-IPC P2P
//     loads, or NVLS multimem.ld_reduce).
//
// Design notes:
//  * Each launch processes ONE tensor as it arrives from autograd (the LOMO
//    contract: a gradient is consumed the moment it exists, tape.py:387-405).
//  * 128-bit LDG/STG: g is read through the non-coherent path with
//    L1::no_allocate (read exactly once), p is read and written with
//    streaming hints.  K1: one 256-vector tile per CTA, grid = ceil(n/tile),
//    the block scheduler balances the tiles; K2: 16 KB tiles, 6 CTAs/SM.
//  * PDL between launches; LOMO_CHAINED launches (a K1 / K2 right after one
//    on other tensors) run before griddepcontrol.wait and wait at their end.
//  * Determinism: K2 reduces per thread (fixed element order), per warp
//    (xor shuffles), per CTA (fixed warp order) into its own partial slot;
//    K3a sums each slot's partials in CTA order, then the slots in delivery
//    order -- no float atomics.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>

#include <type_traits>

#include "lomo_b200.h"

namespace lomo_k {

constexpr int kThreads = 256;
// K2: 16-byte loads in flight per thread; the tile is kThreads x kUnroll
// vectors (16 KB).  tools/k1_state_ab.cu, LLaMA-7B probe pass, 8 alternating
// rounds: 16 KB tiles 6.12 TB/s against 5.86-5.93 for 32 KB tiles (8 loads
// per thread) -- smaller tiles spread each 32-90 MB gradient over more CTAs,
// so the grid's last wave is shorter.
constexpr int kUnroll = 4;

// --------------------------------------------------------------------------
// device info (grid sizing)
// --------------------------------------------------------------------------
struct DevInfo {
  int sms = 0;
};

DevInfo g_dev[64];

const DevInfo& dev_info() {
  int d = 0;
  cudaGetDevice(&d);
  DevInfo& di = g_dev[d & 63];
  if (di.sms == 0) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    di.sms = sms > 0 ? sms : 148;
  }
  return di;
}

// --------------------------------------------------------------------------
// 128-bit memory ops with cache hints
// --------------------------------------------------------------------------
__device__ __forceinline__ uint4 ld_stream_ro(const void* ptr) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(ptr));
  return r;
}
__device__ __forceinline__ uint4 ld_stream_rw(const void* ptr) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(ptr));
  return r;
}
__device__ __forceinline__ void st_stream(void* ptr, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(ptr), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Programmatic dependent launch: every kernel waits for its stream
// predecessor's completion (and memory flush) before touching memory, and
// lets its own dependents be scheduled as soon as all its CTAs are running,
// which hides the launch latency between the back-to-back per-tensor launches
// of one backward pass.  Both are no-ops for a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// --------------------------------------------------------------------------
// storage <-> math conversions
// --------------------------------------------------------------------------
template <typename T>
struct St;
template <>
struct St<float> {
  static constexpr int kDtype = LOMO_F32;
};
template <>
struct St<double> {
  static constexpr int kDtype = LOMO_F64;
};
template <>
struct St<__half> {
  static constexpr int kDtype = LOMO_F16;
};
template <>
struct St<__nv_bfloat16> {
  static constexpr int kDtype = LOMO_BF16;
};

template <typename M, typename T>
__device__ __forceinline__ M to_m(T v);
template <>
__device__ __forceinline__ float to_m<float, float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_m<float, double>(double v) { return (float)v; }
template <>
__device__ __forceinline__ float to_m<float, __half>(__half v) { return __half2float(v); }
template <>
__device__ __forceinline__ float to_m<float, __nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
template <>
__device__ __forceinline__ double to_m<double, float>(float v) { return (double)v; }
template <>
__device__ __forceinline__ double to_m<double, double>(double v) { return v; }
template <>
__device__ __forceinline__ double to_m<double, __half>(__half v) {
  return (double)__half2float(v);  // exact
}
template <>
__device__ __forceinline__ double to_m<double, __nv_bfloat16>(__nv_bfloat16 v) {
  // exact.  (Integer widening for normals/zeros with a conversion fallback
  // measured 0.54 of peak over the f64-math pass against 0.85 for this --
  // the per-element branches cost more than the F2F pipe.)
  return (double)__bfloat162float(v);
}

// Round-to-nearest-even store, overflow to +-inf (tensor.py:30-38 for f16;
// the bf16 rule is this framework's restatement, see oracle/lomo_oracle.py).
template <typename T, typename M>
__device__ __forceinline__ T from_m(M v);
template <>
__device__ __forceinline__ float from_m<float, float>(float v) { return v; }
template <>
__device__ __forceinline__ float from_m<float, double>(double v) { return __double2float_rn(v); }
template <>
__device__ __forceinline__ double from_m<double, float>(float v) { return (double)v; }
template <>
__device__ __forceinline__ double from_m<double, double>(double v) { return v; }
template <>
__device__ __forceinline__ __half from_m<__half, float>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ __half from_m<__half, double>(double v) {
  __half r;
  asm("cvt.rn.f16.f64 %0, %1;" : "=h"(*reinterpret_cast<unsigned short*>(&r)) : "d"(v));
  return r;
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_m<__nv_bfloat16, float>(float v) {
  return __float2bfloat16_rn(v);
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_m<__nv_bfloat16, double>(double v) {
  __nv_bfloat16 r;
  asm("cvt.rn.bf16.f64 %0, %1;" : "=h"(*reinterpret_cast<unsigned short*>(&r)) : "d"(v));
  return r;
}

// --------------------------------------------------------------------------
// the per-element update (stabilize.py:217-224 then optim.py:52-54)
// --------------------------------------------------------------------------
template <typename M>
struct UpdArgs {
  M lr;         // learning rate (held in M: fp32 constant in F32 mode)
  M clip;       // > 0: value clip threshold
  M decay;      // 1 - lr*wd (only used when has_wd)
  M inv_scale;  // 1 / loss scale (exact power of two)
  M coef;       // global-norm clip coefficient
  M wd;         // weight decay (decay recomputed when lr comes from the state)
  bool use_scale, use_coef, use_clip, has_wd;
};

// NaN-propagating clamp (np.clip semantics: NaN stays NaN).
template <typename M>
__device__ __forceinline__ M clamp_nan(M g, M c) {
  return g < -c ? -c : (g > c ? c : g);
}

__device__ __forceinline__ float upd_elem(float p, float g, const UpdArgs<float>& a) {
  if (a.use_scale) g = g * a.inv_scale;
  if (a.use_clip) g = clamp_nan(g, a.clip);
  if (a.use_coef) g = g * a.coef;
  if (a.has_wd) p = p * a.decay;
  return __fmaf_rn(-a.lr, g, p);  // one rounding of p - lr*g
}

__device__ __forceinline__ double upd_elem(double p, double g, const UpdArgs<double>& a) {
  // exactly the reference's float64 sequence: g/scale (exact for a power of
  // two), clip, *norm_scale, then p - (lr*g) with two roundings (no FMA).
  if (a.use_scale) g = __dmul_rn(g, a.inv_scale);
  if (a.use_clip) g = clamp_nan(g, a.clip);
  if (a.use_coef) g = __dmul_rn(g, a.coef);
  if (a.has_wd) p = __dmul_rn(p, a.decay);
  return __dsub_rn(p, __dmul_rn(a.lr, g));
}

template <typename T>
union Vec16 {
  uint4 u;
  T e[16 / sizeof(T)];
};

template <typename T, typename M>
__device__ __forceinline__ uint4 upd_vec(const uint4& pv, const uint4& gv,
                                         const UpdArgs<M>& a) {
  Vec16<T> P, G, O;
  P.u = pv;
  G.u = gv;
#pragma unroll
  for (int k = 0; k < (int)(16 / sizeof(T)); ++k) {
    M r = upd_elem(to_m<M>(P.e[k]), to_m<M>(G.e[k]), a);
    O.e[k] = from_m<T, M>(r);
  }
  return O.u;
}

__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_launch_dependents();
}

// Bulk L2 prefetch (TMA unit; 16-byte aligned, multiple of 16 bytes).  Issued
// BEFORE griddepcontrol.wait: a PDL-launched CTA becomes resident while the
// previous grid drains, and its tile's DRAM fetch then overlaps that drain.
// Memory-model safe: it only fills L2, the point of coherence -- a line the
// previous grid is still writing is updated in L2 by that write, and the
// real loads come after the wait (and bypass L1).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes)
                          : "memory");
}

// Step-state scalars (skip, 1/scale, clip coefficient, lr).  Kernels issue
// their data loads BEFORE calling this: the loads do not depend on the
// state, so the state read's L2 latency overlaps them.  Reading the state
// first put one dependent L2 round trip in front of every CTA's loads --
// with one 4 KB tile per CTA that cost K1 a third of its bandwidth whenever
// a state flag was set (9.7 vs 6.2 ms over the LLaMA-7B pass,
// tools/k1_context.py).
// The pass-2 record: fp32 copies of skip / 1/scale / clip coefficient / lr,
// 32 bytes right after the 128-byte header (include/lomo_b200.h).  Every
// state kernel that changes one of those fields republishes it
// (publish_rec), so the fp32-math kernels read their four step constants
// with ONE 16-byte load per warp.  The values are exactly the (float) casts
// the f64 fields would get, so the update's bits are unchanged.
struct K1Rec {
  int32_t skip;
  float inv_scale, coef, lr;
};
constexpr size_t kRecBytes = 32;
static_assert(sizeof(lomo_state) + kRecBytes == LOMO_STATE_SLOTS_OFFSET, "state layout");
__host__ __device__ __forceinline__ const K1Rec* rec_of(const lomo_state* s) {
  return reinterpret_cast<const K1Rec*>(reinterpret_cast<const char*>(s) + sizeof(lomo_state));
}
__device__ __forceinline__ void publish_rec(lomo_state* s) {
  K1Rec* r = const_cast<K1Rec*>(rec_of(s));
  r->skip = s->skip;
  r->inv_scale = (float)s->inv_scale;
  r->coef = (float)s->clip_coef;
  r->lr = (float)s->lr;
}

// Step-state scalars (skip, 1/scale, clip coefficient, lr).  Kernels issue
// their data loads BEFORE calling this: the loads do not depend on the
// state, so the state read's L2 latency overlaps them.  Reading the state
// first put one dependent L2 round trip in front of every CTA's loads --
// with one 4 KB tile per CTA that cost K1 a third of its bandwidth whenever
// a state flag was set (9.7 vs 6.2 ms over the LLaMA-7B pass,
// tools/k1_context.py).
template <typename M>
__device__ __forceinline__ bool resolve_args(UpdArgs<M>& a, unsigned flags,
                                             const lomo_state* st) {
  if (st == nullptr) return true;
  if constexpr (std::is_same<M, float>::value) {
    // fp32 math: lane 0 loads the 16-byte pass-2 record, the warp shares it
    // by four 32-bit shuffles (tools/k1_state_ab.cu: 6.11 ms per LLaMA-7B
    // pass vs 6.20 for four f64 header loads + f64 shuffles, 6.08 flag-free)
    uint4 r = make_uint4(0u, 0u, 0u, 0u);
    if ((threadIdx.x & 31) == 0)
      asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                   : "l"(rec_of(st)));
    r.x = __shfl_sync(0xffffffffu, r.x, 0);
    r.y = __shfl_sync(0xffffffffu, r.y, 0);
    r.z = __shfl_sync(0xffffffffu, r.z, 0);
    r.w = __shfl_sync(0xffffffffu, r.w, 0);
    if ((flags & LOMO_USE_SKIP) && r.x) return false;
    if (flags & LOMO_USE_SCALE) a.inv_scale = __uint_as_float(r.y);
    if (flags & LOMO_USE_COEF) a.coef = __uint_as_float(r.z);
    if (flags & LOMO_LR_FROM_STATE) {
      a.lr = __uint_as_float(r.w);
      if (a.has_wd) {  // decay from the f64 lr, as the f64 path computes it
        double lr;
        asm volatile("ld.global.f64 %0, [%1];" : "=d"(lr) : "l"(&st->lr));
        a.decay = (float)(1.0 - lr * (double)a.wd);
      }
    }
    return true;
  } else {
    // f64 math: four independent plain loads from one 128-byte line, all in
    // flight together (the state was written by an earlier kernel: after the
    // PDL wait, no volatile/strong access is needed -- a volatile read of
    // `skip` compiled to LDG.STRONG.SYS and serialised a second round trip).
    // One lane per warp loads, the warp shares by shuffle.
    int32_t skip = 0;
    double inv_scale = 0.0, coef = 0.0, lr = 0.0;
    if ((threadIdx.x & 31) == 0) {
      asm volatile("ld.global.s32 %0, [%1];" : "=r"(skip) : "l"(&st->skip));
      asm volatile("ld.global.f64 %0, [%1];" : "=d"(inv_scale) : "l"(&st->inv_scale));
      asm volatile("ld.global.f64 %0, [%1];" : "=d"(coef) : "l"(&st->clip_coef));
      asm volatile("ld.global.f64 %0, [%1];" : "=d"(lr) : "l"(&st->lr));
    }
    skip = __shfl_sync(0xffffffffu, skip, 0);
    inv_scale = __shfl_sync(0xffffffffu, inv_scale, 0);
    coef = __shfl_sync(0xffffffffu, coef, 0);
    lr = __shfl_sync(0xffffffffu, lr, 0);
    if ((flags & LOMO_USE_SKIP) && skip) return false;
    if (flags & LOMO_USE_SCALE) a.inv_scale = (M)inv_scale;
    if (flags & LOMO_USE_COEF) a.coef = (M)coef;
    if (flags & LOMO_LR_FROM_STATE) {
      a.lr = (M)lr;
      a.decay = (M)(1.0 - lr * (double)a.wd);
    }
    return true;
  }
}

template <typename M>
__device__ __forceinline__ bool load_args(UpdArgs<M>& a, unsigned flags,
                                          const lomo_state* st) {
  pdl_enter();
  return resolve_args(a, flags, st);
}

// Vector body: `nvec` 16-byte vectors starting at p/g (16-B aligned), plus
// scalar head/tail elements handled by CTA 0.
//
// One tile of kThreads x kK1Vec 16-byte vectors per CTA, no loop: the grid
// holds ceil(nvec / tile) CTAs and the hardware block scheduler hands tiles
// to SMs as earlier CTAs retire.  That dynamic balance removes the CTA-spread
// tail a persistent/chunked grid pays (tools/k1_variants.cu: 6.70 TB/s for
// this layout vs 5.85 TB/s for one chunk per resident CTA on the LLaMA-7B
// pass), and with PDL the next tensor's tiles start as soon as this grid
// drains.
constexpr int kK1Vec = 1;

// CHAIN (LOMO_CHAINED): the previous launch on the stream is a K1 on other
// tensors, so nothing this CTA reads or writes depends on it: the tile's
// loads, the update and the stores run BEFORE griddepcontrol.wait, while the
// previous grid drains, and dependents are released at entry.  The wait at
// the end keeps stream order: this grid completes only after its
// predecessor has (tools/k1_state_ab.cu: 5.83-6.03 ms per LLaMA-7B pass
// against 6.03-6.16 waiting first).
template <typename T, typename M, bool CHAIN>
__global__ void __launch_bounds__(kThreads)
    k1_update(T* __restrict__ p, const T* __restrict__ g, int64_t n, int head,
              int64_t nvec, UpdArgs<M> a, unsigned flags, const lomo_state* st) {
  constexpr int V = 16 / sizeof(T);
  uint4* pv = reinterpret_cast<uint4*>(p + head);
  const uint4* gv = reinterpret_cast<const uint4*>(g + head);
  // (no L2 prefetch here, unlike K2: measured 5 % slower with every CTA
  // prefetching its 4 KB tiles, and 6 % slower with only the first wave)
  if (CHAIN) {
    pdl_launch_dependents();
  } else {
    pdl_enter();
  }
  const int64_t base = (int64_t)blockIdx.x * (kThreads * kK1Vec) + threadIdx.x;
  uint4 P[kK1Vec], G[kK1Vec];
#pragma unroll
  for (int u = 0; u < kK1Vec; ++u) {
    const int64_t i = base + (int64_t)u * kThreads;
    if (i < nvec) {
      G[u] = ld_stream_ro(gv + i);
      P[u] = ld_stream_rw(pv + i);
    }
  }
  if (!resolve_args(a, flags, st)) {  // overlaps the loads above
    if (CHAIN) pdl_wait();
    return;
  }

  if (blockIdx.x == 0) {  // scalar head (before the first aligned vector) and tail
    const int64_t tail0 = head + nvec * V;
    const int64_t ntail = n - tail0;
    for (int64_t i = threadIdx.x; i < head + ntail; i += blockDim.x) {
      const int64_t e = i < head ? i : tail0 + (i - head);
      p[e] = from_m<T, M>(upd_elem(to_m<M>(p[e]), to_m<M>(g[e]), a));
    }
  }
#pragma unroll
  for (int u = 0; u < kK1Vec; ++u) {
    const int64_t i = base + (int64_t)u * kThreads;
    if (i < nvec) st_stream(pv + i, upd_vec<T, M>(P[u], G[u], a));
  }
  if (CHAIN) pdl_wait();
}

// Fallback when p and g have different 16-byte misalignment: scalar, still
// coalesced (consecutive threads touch consecutive elements).
template <typename T, typename M>
__global__ void __launch_bounds__(kThreads)
    k1_update_scalar(T* __restrict__ p, const T* __restrict__ g, int64_t n, UpdArgs<M> a,
                     unsigned flags, const lomo_state* st) {
  if (!load_args(a, flags, st)) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = from_m<T, M>(upd_elem(to_m<M>(p[i]), to_m<M>(g[i]), a));
}

// Multi-tensor variant (small tensors coalesced into one launch): the
// pointer tables travel BY VALUE in the kernel parameter block, blockIdx.y
// selects the tensor.
constexpr int kMulti = 64;
struct MultiTable {
  void* p[kMulti];
  const void* g[kMulti];
  int64_t n[kMulti];
  int32_t slot[kMulti];
  int count;
};

template <typename T, typename M>
__global__ void __launch_bounds__(kThreads)
    k1_update_multi(const __grid_constant__ MultiTable tab, UpdArgs<M> a, unsigned flags,
                    const lomo_state* st) {
  constexpr int V = 16 / sizeof(T);
  if (!load_args(a, flags, st)) return;
  T* p = static_cast<T*>(tab.p[blockIdx.y]);
  const T* g = static_cast<const T*>(tab.g[blockIdx.y]);
  const int64_t n = tab.n[blockIdx.y];
  const bool aligned = ((((uintptr_t)p) | ((uintptr_t)g)) & 15) == 0;
  const int64_t nvec = aligned ? n / V : 0;
  uint4* pv = reinterpret_cast<uint4*>(p);
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x)
    st_stream(pv + i, upd_vec<T, M>(ld_stream_rw(pv + i), ld_stream_ro(gv + i), a));
  for (int64_t i = nvec * V + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = from_m<T, M>(upd_elem(to_m<M>(p[i]), to_m<M>(g[i]), a));
}

// --------------------------------------------------------------------------
// Row-sparse form for an embedding table (the reference's embedding VJP is a
// dense scatter-add, ops.py; its LOMO update leaves every row the batch did
// not touch unchanged, since p - lr*0 == p exactly): the gradient is kept as
// one aggregated row per distinct token id.
// --------------------------------------------------------------------------
// Aggregate: `sorted` are the batch's token ids after a stable sort, `perm`
// the positions they came from.  Position j that starts a run of equal ids
// sums that run's dy rows in sorted (= token) order in fp32 and stores the
// row rounded to the storage dtype, with idx[j] = id; every other position
// stores a zero row and idx[j] = -1.  Fixed size, no host sync, deterministic.
template <typename T>
__global__ void __launch_bounds__(kThreads)
    k_rows_aggregate(const int64_t* __restrict__ sorted, const int64_t* __restrict__ perm,
                     const T* __restrict__ dy, int64_t ntok, int64_t h, T* __restrict__ rows,
                     int64_t* __restrict__ idx) {
  pdl_enter();
  const int64_t j = blockIdx.x;
  const int64_t id = sorted[j];
  const bool head = j == 0 || sorted[j - 1] != id;
  if (threadIdx.x == 0) idx[j] = head ? id : -1;
  int64_t end = j + 1;
  if (head)
    while (end < ntok && sorted[end] == id) ++end;
  constexpr int V = 16 / sizeof(T);
  if ((h % V) == 0 && (((uintptr_t)dy | (uintptr_t)rows) & 15) == 0) {  // 16-byte vectors
    for (int64_t c = threadIdx.x; c < h / V; c += blockDim.x) {
      float acc[V];
#pragma unroll
      for (int e = 0; e < V; ++e) acc[e] = 0.f;
      if (head)
        for (int64_t k = j; k < end; ++k) {
          Vec16<T> D;
          D.u = ld_stream_ro(reinterpret_cast<const uint4*>(dy + perm[k] * h) + c);
#pragma unroll
          for (int e = 0; e < V; ++e) acc[e] += to_m<float>(D.e[e]);
        }
      Vec16<T> O;
#pragma unroll
      for (int e = 0; e < V; ++e) O.e[e] = from_m<T, float>(acc[e]);
      reinterpret_cast<uint4*>(rows + j * h)[c] = O.u;
    }
    return;
  }
  for (int64_t c = threadIdx.x; c < h; c += blockDim.x) {
    float acc = 0.f;
    if (head)
      for (int64_t k = j; k < end; ++k) acc += to_m<float>(dy[perm[k] * h + c]);
    rows[j * h + c] = from_m<T, float>(acc);
  }
}

// Update: p[idx[j], :] <- the K1 arithmetic with rows[j, :], for idx[j] >= 0.
template <typename T, typename M>
__global__ void __launch_bounds__(kThreads)
    k1_rows(T* __restrict__ p, const T* __restrict__ rows, const int64_t* __restrict__ idx,
            int64_t h, UpdArgs<M> a, unsigned flags, const lomo_state* st) {
  if (!load_args(a, flags, st)) return;
  const int64_t r = idx[blockIdx.x];
  if (r < 0) return;  // CTA-uniform
  T* pr = p + r * h;
  const T* gr = rows + (int64_t)blockIdx.x * h;
  constexpr int V = 16 / sizeof(T);
  const bool vec = (h % V) == 0 && (((uintptr_t)pr | (uintptr_t)gr) & 15) == 0;
  if (vec) {  // 128-bit path (rows of a 16-byte-multiple width)
    uint4* pv = reinterpret_cast<uint4*>(pr);
    const uint4* gv = reinterpret_cast<const uint4*>(gr);
    for (int64_t c = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; c < h / V;
         c += (int64_t)gridDim.y * blockDim.x)
      pv[c] = upd_vec<T, M>(pv[c], ld_stream_ro(gv + c), a);
    return;
  }
  for (int64_t c = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; c < h;
       c += (int64_t)gridDim.y * blockDim.x)
    pr[c] = from_m<T, M>(upd_elem(to_m<M>(pr[c]), to_m<M>(gr[c]), a));
}

// --------------------------------------------------------------------------
// K2: probe -- deterministic sum of squares + non-finite flag
// --------------------------------------------------------------------------
__device__ __forceinline__ lomo_state* hdr(void* s) { return reinterpret_cast<lomo_state*>(s); }
// state block layout (include/lomo_b200.h): header | sumsq[nslots] |
// nblocks[nslots] (int32, padded to 8 B) | partials[nslots][PER_SLOT]
__host__ __device__ __forceinline__ size_t nblocks_words(int nslots) {
  return (size_t)(nslots + 1) / 2;  // int32 pairs -> 8-byte words
}
__device__ __forceinline__ double* slots_of(lomo_state* s) {
  return reinterpret_cast<double*>(reinterpret_cast<char*>(s) + LOMO_STATE_SLOTS_OFFSET);
}
__device__ __forceinline__ int32_t* nblocks_of(lomo_state* s) {
  return reinterpret_cast<int32_t*>(slots_of(s) + s->nslots);
}
__device__ __forceinline__ double* partials_of(lomo_state* s, int slot) {
  return slots_of(s) + s->nslots + nblocks_words(s->nslots) +
         (size_t)slot * LOMO_PROBE_BLOCKS_PER_SLOT;
}
// One CTA's partial of norm slot `slot` (thread 0).  A slot outside
// [0, nslots) writes nothing and raises the sticky state->error (the host
// turns it into LOMO_E_SLOT at the step's status read).
__device__ __forceinline__ void put_partial(lomo_state* st, int slot, double v, int nblocks,
                                            int nslots) {
  if ((unsigned)slot >= (unsigned)nslots) {
    st->error = 1;
    return;
  }
  double* s = slots_of(st);
  s[nslots + nblocks_words(nslots) + (size_t)slot * LOMO_PROBE_BLOCKS_PER_SLOT + blockIdx.x] = v;
  if (blockIdx.x == 0) reinterpret_cast<int32_t*>(s + nslots)[slot] = nblocks;
}
__device__ __forceinline__ void put_partial(lomo_state* st, int slot, double v, int nblocks) {
  put_partial(st, slot, v, nblocks, st->nslots);
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// fixed-order CTA reduction; result valid in thread 0
__device__ __forceinline__ double block_sum(double v, double* sm) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sm[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r += sm[i];
  }
  __syncthreads();
  return r;
}

__device__ __forceinline__ bool is_fin(float x) { return fabsf(x) <= 3.402823466e38f; }
__device__ __forceinline__ bool is_fin(double x) { return fabs(x) <= 1.7976931348623157e308; }

// per-vector partial: squares (exact for 16-bit storage) summed in the math
// type, then accumulated across vectors in f64.
template <typename T, typename M>
__device__ __forceinline__ double vec_sumsq(const uint4& gv, M inv_scale, bool use_scale,
                                            bool& bad) {
  Vec16<T> G;
  G.u = gv;
  M acc = 0;
#pragma unroll
  for (int k = 0; k < (int)(16 / sizeof(T)); ++k) {
    M x = to_m<M>(G.e[k]);
    bad |= !is_fin(x);
    if (use_scale) x = x * inv_scale;
    acc = fma(x, x, acc);
  }
  return (double)acc;
}

// Hot-loop form (M = float): no per-element finiteness test.  A non-finite
// element makes its square inf/NaN, so the thread's running sum is
// non-finite; only then does the thread re-scan its elements to tell a
// non-finite gradient (probe_hook's overflow) from squares that merely
// overflowed fp32 (which stay an inf partial, as before).  Same arithmetic as
// vec_sumsq -- (g*inv_scale)^2 by FMA in fp32 per 16-byte vector -- at about
// half the instructions per element: at 5+ TB/s K2 is issue-bound otherwise.
template <typename T>
__device__ __forceinline__ double vec_sumsq_nocheck(const uint4& gv, float inv_scale,
                                                    bool use_scale) {
  Vec16<T> G;
  G.u = gv;
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < (int)(16 / sizeof(T)); ++k) {
    float x = to_m<float>(G.e[k]);
    if (use_scale) x = x * inv_scale;
    acc = fmaf(x, x, acc);
  }
  return (double)acc;
}

template <typename T>
__device__ __forceinline__ bool vec_has_nonfinite(const uint4& gv) {
  Vec16<T> G;
  G.u = gv;
  bool bad = false;
#pragma unroll
  for (int k = 0; k < (int)(16 / sizeof(T)); ++k) bad |= !is_fin(to_m<float>(G.e[k]));
  return bad;
}

template <typename T, typename M>
__device__ __forceinline__ double tile_sumsq(const uint4& gv, M inv_scale, bool use_scale,
                                             bool& bad) {
  if constexpr (std::is_same<M, float>::value) {
    return vec_sumsq_nocheck<T>(gv, inv_scale, use_scale);
  } else {
    return vec_sumsq<T, M>(gv, inv_scale, use_scale, bad);
  }
}

// Fixed-order CTA sum for a CTA that reduces once: one barrier (block_sum's
// second barrier only protects `sm` for reuse).  Result valid in thread 0.
__device__ __forceinline__ double block_sum_once(double v, double* sm) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < kThreads / 32; ++i) r += sm[i];
  }
  return r;
}

// K2's cold paths, kept out of line so the hot kernel carries none of their
// registers or instructions (each cost 1-3 % of the probe pass inline,
// tools/k1_state_ab.cu "k2p -..." ablations).  Both return NaN when they see
// a non-finite gradient element (probe_hook's overflow, stabilize.py:196-197).
//
// The scalar head (before the first aligned vector) and tail (CTA 0).
template <typename T, typename M>
__device__ __noinline__ double k2_head_tail(const T* g, int64_t n, int head, int64_t nvec) {
  constexpr int V = 16 / sizeof(T);
  const int64_t tail0 = head + nvec * V;
  const int64_t ntail = n - tail0;
  double acc = 0.0;
  bool bad = false;
  for (int64_t i = threadIdx.x; i < head + ntail; i += blockDim.x) {
    const int64_t e = i < head ? i : tail0 + (i - head);
    M x = to_m<M>(g[e]);
    bad |= !is_fin(x);
    acc += (double)x * (double)x;
  }
  return bad ? __longlong_as_double(0x7ff8000000000000ll) : acc;
}
// A thread whose fp32 running sum came out non-finite: a non-finite element
// (NaN result), or finite elements whose fp32 squares overflowed (the sum
// redone in f64 from `acc0`).
template <typename T>
__device__ __noinline__ double k2_rescan(const uint4* gv, int64_t beg, int64_t end, double acc0) {
  constexpr int V = 16 / sizeof(T);
  for (int64_t i = beg + threadIdx.x; i < end; i += kThreads)
    if (vec_has_nonfinite<T>(ld_stream_ro(gv + i))) return __longlong_as_double(0x7ff8000000000000ll);
  double acc = acc0;
  for (int64_t i = beg + threadIdx.x; i < end; i += kThreads) {
    Vec16<T> G;
    G.u = ld_stream_ro(gv + i);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const double x = (double)to_m<float>(G.e[k]);
      acc += x * x;
    }
  }
  return acc;
}

// One tile of K2: kUnroll 16-byte vectors per thread, all loads issued
// before the first square.
template <typename T, typename M>
__device__ __forceinline__ double k2_tile(const uint4* __restrict__ gv, int64_t base, int64_t end,
                                          bool& bad) {
  uint4 G[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const int64_t i = base + (int64_t)u * kThreads;
    if (i < end) G[u] = ld_stream_ro(gv + i);
  }
  double acc = 0.0;
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const int64_t i = base + (int64_t)u * kThreads;
    if (i < end) acc += tile_sumsq<T, M>(G[u], (M)1, false, bad);
  }
  return acc;
}

// CHAIN (LOMO_CHAINED): the previous launch is a K2 on another gradient and
// slot, so the CTA runs entirely before griddepcontrol.wait (its tile's loads
// need no L2 prefetch) and waits at its end, as chained K1 does.
template <typename T, typename M, bool CHAIN>
__global__ void __launch_bounds__(kThreads, 6)
    k2_probe(const T* __restrict__ g, int64_t n, int head, int64_t nvec, int64_t per_cta,
             int slot, unsigned flags, void* state) {
  __shared__ double sm[kThreads / 32];
  const int64_t beg = (int64_t)blockIdx.x * per_cta;
  const int64_t end = min(beg + per_cta, nvec);
  const uint4* gv = reinterpret_cast<const uint4*>(g + head);
  if (CHAIN) {
    pdl_launch_dependents();
  } else {
    if (threadIdx.x == 0 && end > beg)  // this CTA's tile into L2 while the previous grid drains
      prefetch_l2(gv + beg, (uint32_t)((end - beg) * 16));
    pdl_wait();
    pdl_launch_dependents();
  }
  lomo_state* st = hdr(state);
  // 1/scale and nslots for the CTA's partial, loaded now (after the wait: an
  // earlier step's K3 may have changed the scale) and consumed at the end, so
  // the L2 round trip hides behind the tile's loads instead of extending the
  // CTA's life (tools/k1_state_ab.cu: 2.20 vs 2.24 ms per pass read at the end)
  double sc = 1.0;
  int nslots = 0;
  if (threadIdx.x == 0) {
    if (flags & LOMO_USE_SCALE)
      asm volatile("ld.global.f64 %0, [%1];" : "=d"(sc) : "l"(&st->inv_scale));
    asm volatile("ld.global.s32 %0, [%1];" : "=r"(nslots) : "l"(&st->nslots));
  }

  // small fixed tiles (>= 1024 vectors = 16 KB, <= LOMO_PROBE_BLOCKS_PER_SLOT
  // CTAs): the block scheduler balances them across SMs like K1's tiles.
  //
  // The squares are summed UNSCALED and the CTA's sum is multiplied by
  // inv_scale^2 once, at the end: inv_scale is a power of two (the loss
  // scale; with a data-parallel divisor that is a power of two too), so every
  // term, every partial sum and the result scale exactly -- the same bits as
  // summing (g * inv_scale)^2 (stabilize.py:199) -- but no load of the loop
  // depends on the state.  (Any other divisor: within f64 rounding.)
  bool bad = false;
  double acc = 0.0;
  if (blockIdx.x == 0) {
    acc = k2_head_tail<T, M>(g, n, head, nvec);
    bad = acc != acc;  // (the NaN then flows into the partial, as before)
  }
  const double acc_ht = acc;
  // One 16 KB tile per CTA (every launch but the largest tensors'): straight
  // -line code, all of the tile's loads in flight before the first square.
  // Larger per-CTA ranges loop over tiles (no outer unroll: the compiler
  // otherwise software-pipelines the loop so a tile's loads are no longer all
  // in flight at once -- 5.37 vs 6.1 TB/s).
  if (per_cta == (int64_t)kThreads * kUnroll) {
    acc += k2_tile<T, M>(gv, beg + threadIdx.x, end, bad);
  } else {
#pragma unroll 1
    for (int64_t base = beg + threadIdx.x; base < end; base += (int64_t)kThreads * kUnroll)
      acc += k2_tile<T, M>(gv, base, end, bad);
  }
  if constexpr (std::is_same<M, float>::value) {
    if (!is_fin(acc)) {  // rare
      acc = k2_rescan<T>(gv, beg, end, acc_ht);
      if (acc != acc) bad = true;
    }
  }
  // any thread that saw a non-finite element raises the flag (all store 1:
  // no barrier needed, K3 reads it after this grid completes)
  if (bad) st->overflow = 1;

  // per-CTA partial into this slot's partial row; K3 reduces the row in CTA
  // order (deterministic, no atomics on the hot path)
  double bsum = block_sum_once(acc, sm);
  if (threadIdx.x == 0) {
    if (flags & LOMO_USE_SCALE) bsum *= sc * sc;  // exact: a power of two
    put_partial(st, slot, bsum, (int)gridDim.x, nslots);
  }
  if (CHAIN) pdl_wait();
}

// Multi-tensor probe: one CTA per (small) tensor, which writes its slot
// directly (fixed-order CTA reduction; no cross-CTA finish needed).
template <typename T, typename M>
__global__ void __launch_bounds__(kThreads)
    k2_probe_multi(const __grid_constant__ MultiTable tab, unsigned flags, void* state) {
  constexpr int V = 16 / sizeof(T);
  __shared__ double sm[kThreads / 32];
  pdl_wait();
  pdl_launch_dependents();
  lomo_state* st = hdr(state);
  const bool use_scale = (flags & LOMO_USE_SCALE) != 0;
  const M inv_scale = use_scale ? (M)st->inv_scale : (M)1;
  const T* g = static_cast<const T*>(tab.g[blockIdx.x]);
  const int64_t n = tab.n[blockIdx.x];
  const int64_t nvec = (((uintptr_t)g) & 15) == 0 ? n / V : 0;
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  double acc = 0.0;
  bool bad = false;
  for (int64_t i = threadIdx.x; i < nvec; i += kThreads)
    acc += vec_sumsq<T, M>(ld_stream_ro(gv + i), inv_scale, use_scale, bad);
  for (int64_t i = nvec * V + threadIdx.x; i < n; i += kThreads) {
    M x = to_m<M>(g[i]);
    bad |= !is_fin(x);
    if (use_scale) x = x * inv_scale;
    acc += (double)x * (double)x;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) st->overflow = 1;
  const double r = block_sum(acc, sm);
  if (threadIdx.x == 0) {
    const int slot = tab.slot[blockIdx.x];
    if ((unsigned)slot >= (unsigned)st->nslots) {
      st->error = 1;
    } else {
      slots_of(st)[slot] = r;
      nblocks_of(st)[slot] = 0;  // reduced in place
    }
  }
}

// K6 second stage: row r of the [rows, ld] fp32 partial matrix (K6's per
// tile-row column sums) -> partial r of the slot, in fixed order; a NaN
// partial marks a non-finite gradient element (lomo_gemm_probe.cu).
__global__ void __launch_bounds__(kThreads)
    k6_rows(const float* __restrict__ part, int64_t ld, int64_t cols, int slot, void* state) {
  __shared__ double sm[kThreads / 32];
  pdl_wait();
  pdl_launch_dependents();
  lomo_state* st = hdr(state);
  const float* row = part + (int64_t)blockIdx.x * ld;
  double acc = 0.0;
  bool bad = false;
  for (int64_t c = threadIdx.x; c < cols; c += kThreads) {
    const float v = row[c];
    bad |= isnan(v);
    acc += (double)v;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) st->overflow = 1;
  const double bsum = block_sum(acc, sm);
  if (threadIdx.x == 0) {
    put_partial(st, slot, bsum, (int)gridDim.x);
  }
}

// Many K6 partial matrices in one launch (deferred mode): blockIdx.y picks
// the entry, blockIdx.x its row; the table travels by value.
struct RowsTable {
  const float* part[kMulti];
  int64_t rows[kMulti];
  int64_t ld[kMulti];
  int64_t cols[kMulti];
  int32_t slot[kMulti];
};

__global__ void __launch_bounds__(kThreads) k6_rows_multi(const __grid_constant__ RowsTable tab,
                                                          void* state) {
  __shared__ double sm[kThreads / 32];
  pdl_wait();
  pdl_launch_dependents();
  const int e = blockIdx.y;
  if ((int64_t)blockIdx.x >= tab.rows[e]) return;  // CTA-uniform
  lomo_state* st = hdr(state);
  const float* row = tab.part[e] + (int64_t)blockIdx.x * tab.ld[e];
  const int64_t cols = tab.cols[e];
  double acc = 0.0;
  bool bad = false;
  int64_t c = threadIdx.x;
  for (; c + 3 * kThreads < cols; c += 4 * kThreads) {  // four loads in flight
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = row[c + u * kThreads];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      bad |= isnan(v[u]);
      acc += (double)v[u];
    }
  }
  for (; c < cols; c += kThreads) {
    const float v = row[c];
    bad |= isnan(v);
    acc += (double)v;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) st->overflow = 1;
  const double bsum = block_sum(acc, sm);
  if (threadIdx.x == 0) {
    put_partial(st, tab.slot[e], bsum, (int)tab.rows[e]);
  }
}

// --------------------------------------------------------------------------
// K4: reduce-scatter fused with the update / probe over peer memory
// --------------------------------------------------------------------------
// Sharded mode: every rank's flat bucket gradient lives in symmetric memory
// (peer-mapped over NVLink).  Rank r owns [off, off+n) of the bucket; K4 loads
// that slice from all `world` peers' buffers (P2P loads through NVSwitch),
// sums in the math type in rank order (deterministic), and feeds the sum
// straight into the update (K1 arithmetic) or the sum of squares (K2): the
// reduced gradient is never written to HBM.  Requires 16-byte aligned slices
// (ShardedLOMO pads buckets to 8*world elements).
constexpr int kMaxPeers = 16;
// Peers are read in chunks of kPeerChunk: a chunk's loads are all in flight
// before its adds, and only one chunk is live in registers.  A fully
// unrolled 16-peer array held 64 registers of loads (92 / 138 registers per
// thread for update / probe, 2 / 1 CTAs per SM); tools/k4_local.py.
constexpr int kPeerChunk = 4;

// acc[k] = sum over ranks r = 0..world-1, in rank order, of peer r's vector idx
template <typename T, typename M>
__device__ __forceinline__ void peer_sum_vec(const T* const* __restrict__ peers, int world,
                                             int64_t idx, M (&acc)[16 / sizeof(T)]) {
  constexpr int V = 16 / sizeof(T);
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = (M)0;
  for (int r0 = 0; r0 < world; r0 += kPeerChunk) {
    uint4 buf[kPeerChunk];
#pragma unroll
    for (int j = 0; j < kPeerChunk; ++j)  // the chunk's loads in flight before the adds
      if (r0 + j < world) buf[j] = ld_stream_ro(reinterpret_cast<const uint4*>(peers[r0 + j]) + idx);
#pragma unroll
    for (int j = 0; j < kPeerChunk; ++j) {
      if (r0 + j < world) {
        Vec16<T> G;
        G.u = buf[j];
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] += to_m<M>(G.e[k]);
      }
    }
  }
}

template <typename T, typename M>
__global__ void __launch_bounds__(kThreads)
    k4_rs_update(T* __restrict__ p, const T* const* __restrict__ peers_dev, int world, int64_t off,
                 int64_t nvec, UpdArgs<M> a, unsigned flags, const lomo_state* st) {
  constexpr int V = 16 / sizeof(T);
  pdl_enter();
  __shared__ const T* peers[kMaxPeers];
  if (threadIdx.x < kMaxPeers)
    peers[threadIdx.x] = threadIdx.x < world ? peers_dev[threadIdx.x] + off : nullptr;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (i >= nvec) return;
  uint4* pv = reinterpret_cast<uint4*>(p);
  Vec16<T> P, O;
  P.u = ld_stream_rw(pv + i);  // in flight with the first chunk of peer loads
  M g[V];
  peer_sum_vec<T, M>(peers, world, i, g);
  if (!resolve_args(a, flags, st)) return;
#pragma unroll
  for (int k = 0; k < V; ++k) O.e[k] = from_m<T, M>(upd_elem(to_m<M>(P.e[k]), g[k], a));
  st_stream(pv + i, O.u);
}

// The peer table is written once when the ring is set up (never by a kernel
// of the step), so it is read before the PDL wait; each peer's slice of the
// CTA's tile is bulk-prefetched into L2 while the previous grid drains (as
// K2 does).
// KEEP (lomo_fused_rs_probe_keep): the reduced slice, rounded to the storage
// dtype as a reduce-scatter output is, is also written to `out` and the
// squares are taken of those rounded values -- the gradient pass 2 then
// applies (ShardedLOMO keep_grads over K4).
template <typename T, typename M, bool KEEP>
__global__ void __launch_bounds__(kThreads, 5)
    k4_rs_probe(const T* const* __restrict__ peers_dev, int world, int64_t off, int64_t nvec,
                int64_t per_cta, int slot, unsigned flags, void* state, T* __restrict__ out) {
  constexpr int V = 16 / sizeof(T);
  __shared__ double sm[kThreads / 32];
  __shared__ const T* peers[kMaxPeers];
  const int64_t beg = (int64_t)blockIdx.x * per_cta;
  const int64_t end = min(beg + per_cta, nvec);
  if (threadIdx.x < kMaxPeers) {
    const T* q = threadIdx.x < world ? peers_dev[threadIdx.x] + off : nullptr;
    peers[threadIdx.x] = q;
    if (q != nullptr && end > beg)
      prefetch_l2(reinterpret_cast<const uint4*>(q) + beg, (uint32_t)((end - beg) * 16));
  }
  pdl_wait();
  pdl_launch_dependents();
  lomo_state* st = hdr(state);
  __syncthreads();
  const bool use_scale = (flags & LOMO_USE_SCALE) != 0;
  const M inv_scale = use_scale ? (M)st->inv_scale : (M)1;
  double acc = 0.0;
  bool bad = false;
  for (int64_t i = beg + threadIdx.x; i < end; i += kThreads) {
    M g[V];
    peer_sum_vec<T, M>(peers, world, i, g);
    if (KEEP) {
      Vec16<T> O;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        O.e[k] = from_m<T, M>(g[k]);
        g[k] = to_m<M>(O.e[k]);
      }
      reinterpret_cast<uint4*>(out)[i] = O.u;
    }
    M part = 0;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      M x = g[k];
      bad |= !is_fin(x);
      if (use_scale) x = x * inv_scale;
      part = fma(x, x, part);
    }
    acc += (double)part;
  }
  if (bad) st->overflow = 1;  // any thread (all store 1)
  const double bsum = block_sum_once(acc, sm);
  if (threadIdx.x == 0) {
    put_partial(st, slot, bsum, (int)gridDim.x);
  }
}

// NVLS form: one multimem.ld_reduce per 16-byte vector at the multicast
// address -- the switch fetches the vector from every rank's copy and returns
// the sum (fp32 accumulation for 16-bit storage, one rounding to storage, as
// an NCCL reduce-scatter output would be), so each GPU's inbound NVLink
// traffic is its slice once instead of once per peer.
template <typename T>
__device__ __forceinline__ uint4 mc_ld_reduce(const void* mc) {
  uint4 r;
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(mc) : "memory");
  } else if constexpr (std::is_same<T, __half>::value) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(mc) : "memory");
  } else {
    static_assert(std::is_same<T, float>::value, "NVLS K4: f32, f16 or bf16 storage");
    float x, y, z, w;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "l"(mc) : "memory");
    r = make_uint4(__float_as_uint(x), __float_as_uint(y), __float_as_uint(z), __float_as_uint(w));
  }
  return r;
}

template <typename T, typename M>
__global__ void __launch_bounds__(kThreads)
    k4_mc_update(T* __restrict__ p, const T* __restrict__ mc, int64_t nvec, UpdArgs<M> a,
                 unsigned flags, const lomo_state* st) {
  pdl_enter();
  const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (i >= nvec) return;
  const uint4 gv = mc_ld_reduce<T>(reinterpret_cast<const uint4*>(mc) + i);
  uint4* pv = reinterpret_cast<uint4*>(p);
  const uint4 P = ld_stream_rw(pv + i);
  if (!resolve_args(a, flags, st)) return;  // overlaps the loads above
  st_stream(pv + i, upd_vec<T, M>(P, gv, a));
}

template <typename T, typename M>
__global__ void __launch_bounds__(kThreads)
    k4_mc_probe(const T* __restrict__ mc, int64_t nvec, int64_t per_cta, int slot,
                unsigned flags, void* state, T* __restrict__ out) {
  __shared__ double sm[kThreads / 32];
  pdl_wait();
  pdl_launch_dependents();
  lomo_state* st = hdr(state);
  const bool use_scale = (flags & LOMO_USE_SCALE) != 0;
  const M inv_scale = use_scale ? (M)st->inv_scale : (M)1;
  double acc = 0.0;
  bool bad = false;
  const int64_t beg = (int64_t)blockIdx.x * per_cta;
  const int64_t end = min(beg + per_cta, nvec);
  const uint4* gv = reinterpret_cast<const uint4*>(mc);
  for (int64_t i = beg + threadIdx.x; i < end; i += kThreads) {
    const uint4 r = mc_ld_reduce<T>(gv + i);  // the switch's sum, rounded to T
    if (out != nullptr) reinterpret_cast<uint4*>(out)[i] = r;  // keep: the reduced slice
    acc += vec_sumsq<T, M>(r, inv_scale, use_scale, bad);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) st->overflow = 1;
  const double bsum = block_sum(acc, sm);
  if (threadIdx.x == 0) {
    put_partial(st, slot, bsum, (int)gridDim.x);
  }
}

// --------------------------------------------------------------------------
// K3 + bookkeeping kernels (single CTA)
// --------------------------------------------------------------------------
__device__ void scaler_on_overflow(lomo_state* st) {
  // stabilize.py:115-121
  if (!st->has_scaler) return;
  if (st->scale / 2.0 < st->min_scale) {
    st->underflow = 1;
    return;
  }
  st->scale = st->scale / 2.0;
  st->inv_scale = 1.0 / (st->scale * st->grad_div);
  st->scale_f32 = (float)st->scale;
  st->clean_steps = 0;
}

__device__ void decide(lomo_state* st, double total) {
  // stabilize.py:201-213
  st->sumsq_total = total;
  const double N = sqrt(total);
  st->total_norm = N;
  const bool norm_clip = st->max_norm > 0.0;
  bool skip = st->overflow != 0;
  double coef = 1.0;
  if (!skip && norm_clip) {
    if (!isfinite(N)) {
      skip = true;
    } else if (N > 0.0) {
      coef = fmin(1.0, st->max_norm / N);
    }
  }
  st->clip_coef = coef;
  st->skip = skip ? 1 : 0;
  if (skip) {
    st->steps_skipped += 1;
    scaler_on_overflow(st);  // _skip, stabilize.py:155-159
  }
  publish_rec(st);
}

// K3a: CTA c reduces slots c, c+grid, ... (each slot's K2 partials in CTA
// order); the
// last CTA to finish (ticket) sums the slots in slot (= delivery) order and
// either decides (mode 0: finalize) or exports {sum, overflow} (mode 1:
// the sharded-mode local partial).
__global__ void __launch_bounds__(kThreads) k3_reduce(void* state, int mode, double* out2) {
  __shared__ double sm[kThreads / 32];
  __shared__ bool am_last;
  pdl_wait();
  lomo_state* st = hdr(state);
  for (int s = blockIdx.x; s < st->nslots; s += gridDim.x) {  // CTA-uniform loop
    const int nb = nblocks_of(st)[s];
    if (nb > 0) {
      const double* part = partials_of(st, s);
      double r = 0.0;
      for (int i = threadIdx.x; i < nb; i += kThreads) r += part[i];
      r = block_sum(r, sm);
      if (threadIdx.x == 0) slots_of(st)[s] = r;
    }
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atomicAdd(&st->ticket, 1u);
    am_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last || threadIdx.x != 0) return;
  __threadfence();
  const volatile double* sq = slots_of(st);
  double total = 0.0;
  for (int i = 0; i < st->nslots; ++i) total += sq[i];  // delivery (slot) order
  st->ticket = 0;
  if (mode == 0) {
    decide(st, total);
  } else {
    out2[0] = total;
    out2[1] = st->overflow ? 1.0 : 0.0;
  }
}

__global__ void k3_finalize_ranks(void* state, const double* parts, int world) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  lomo_state* st = hdr(state);
  double total = 0.0;
  int ovf = st->overflow;
  for (int r = 0; r < world; ++r) {  // rank order: identical on every rank
    total += parts[2 * r];
    ovf |= parts[2 * r + 1] != 0.0;
  }
  st->overflow = ovf;
  decide(st, total);
}

__global__ void k3_on_clean(void* state) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  lomo_state* st = hdr(state);
  if (st->skip) return;
  st->steps_applied += 1;
  if (!st->has_scaler) return;
  // stabilize.py:123-127
  st->clean_steps += 1;
  if (st->clean_steps >= st->growth_interval) {
    st->scale = fmin(st->scale * 2.0, st->max_scale);
    st->inv_scale = 1.0 / (st->scale * st->grad_div);
    st->scale_f32 = (float)st->scale;
    st->clean_steps = 0;
    publish_rec(st);
  }
}

__global__ void k_state_init(void* state, int nslots, double scale, int growth_interval,
                             double min_scale, double max_scale, double max_norm,
                             double grad_div) {
  lomo_state* st = hdr(state);
  if (threadIdx.x == 0) {
    const bool has = scale > 0.0;
    st->grad_div = grad_div > 0.0 ? grad_div : 1.0;
    st->has_scaler = has ? 1 : 0;
    st->scale = has ? scale : 1.0;
    st->inv_scale = 1.0 / (st->scale * st->grad_div);
    st->scale_f32 = (float)st->scale;
    st->min_scale = min_scale;
    st->max_scale = max_scale;
    st->clip_coef = 1.0;
    st->total_norm = 0.0;
    st->sumsq_total = 0.0;
    st->max_norm = max_norm;
    st->growth_interval = growth_interval;
    st->clean_steps = 0;
    st->overflow = 0;
    st->skip = 0;
    st->underflow = 0;
    st->nslots = nslots;
    st->steps_applied = 0;
    st->steps_skipped = 0;
    st->ticket = 0;
    st->error = 0;
    st->lr = 0.0;
  }
  if (threadIdx.x == 0) publish_rec(st);
  double* s = slots_of(st);
  const size_t words = (size_t)nslots + nblocks_words(nslots);  // partials need no init
  for (size_t i = threadIdx.x; i < words; i += blockDim.x) s[i] = 0.0;
}

__global__ void k_set_lr(void* state, double lr) {
  pdl_wait();
  if (threadIdx.x == 0) {
    hdr(state)->lr = lr;
    publish_rec(hdr(state));
  }
}

// LossScaler state restored from a checkpoint (stabilize.py:94-127's live
// fields): scale, its reciprocal and fp32 copy, the clean-step counter and
// the applied/skipped step counts; the pass-2 record is republished.
__global__ void k_set_scaler(void* state, double scale, int clean_steps, int applied,
                             int skipped) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  lomo_state* st = hdr(state);
  if (st->has_scaler) {
    st->scale = scale;
    st->inv_scale = 1.0 / (scale * st->grad_div);
    st->scale_f32 = (float)scale;
    st->clean_steps = clean_steps;
  }
  st->steps_applied = applied;
  st->steps_skipped = skipped;
  publish_rec(st);
}

__global__ void k_update_coefs(const void* state, double wd, unsigned flags, float* out) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  const lomo_state* st = reinterpret_cast<const lomo_state*>(state);
  if ((flags & LOMO_USE_SKIP) && st->skip) {
    out[0] = 0.0f;
    out[1] = 1.0f;
    return;
  }
  double a = -st->lr;
  if (flags & LOMO_USE_COEF) a *= st->clip_coef;
  if (flags & LOMO_USE_SCALE) a *= st->inv_scale;
  out[0] = (float)a;
  out[1] = (float)(1.0 - st->lr * wd);
}

__device__ __forceinline__ bool loss_finite(const void* loss, int dt) {
  switch (dt) {
    case LOMO_F32: return isfinite(*(const float*)loss);
    case LOMO_F64: return isfinite(*(const double*)loss);
    case LOMO_F16: return isfinite(__half2float(*(const __half*)loss));
    case LOMO_BF16: return isfinite(__bfloat162float(*(const __nv_bfloat16*)loss));
  }
  return true;
}

__global__ void k_begin_step(void* state, const void* loss, int loss_dtype) {
  pdl_wait();
  lomo_state* st = hdr(state);
  const int ns = st->nslots;
  double* s = slots_of(st);
  int32_t* nb = nblocks_of(st);
  for (int i = threadIdx.x; i < ns; i += blockDim.x) {
    s[i] = 0.0;
    nb[i] = 0;
  }
  if (threadIdx.x == 0) {
    st->overflow = 0;
    st->skip = 0;
    st->underflow = 0;
    st->clip_coef = 1.0;
    st->ticket = 0;
    if (loss != nullptr && !loss_finite(loss, loss_dtype)) {
      st->overflow = 1;  // optim.py:63-65 / stabilize.py:188-189
      st->skip = 1;
    }
    publish_rec(st);
  }
}

// --------------------------------------------------------------------------
// host-side launch helpers
// --------------------------------------------------------------------------
inline int dtype_size(int dt) {
  switch (dt) {
    case LOMO_F32: return 4;
    case LOMO_F16: return 2;
    case LOMO_BF16: return 2;
    case LOMO_F64: return 8;
  }
  return 0;
}

// resident CTAs per SM for one kernel instantiation (queried once)
template <typename K>
int occupancy(K kernel) {
  static int occ = 0;
  if (occ == 0) {
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, kThreads, 0) != cudaSuccess ||
        o < 1) {
      cudaGetLastError();
      o = 1;
    }
    occ = o;
  }
  return occ;
}

inline int grid_for(int64_t nvec_per_thread_units, int occ) {
  const DevInfo& di = dev_info();
  const int64_t cap = (int64_t)di.sms * occ;
  int64_t want = (nvec_per_thread_units + kThreads - 1) / kThreads;
  if (want < 1) want = 1;
  return (int)(want < cap ? want : cap);
}

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LOMO_PDL");
    v = (e == nullptr || e[0] != '0') ? 1 : 0;
  }
  return v == 1;
}

// cudaLaunchKernelEx with programmatic stream serialisation (PDL)
template <typename... KArgs, typename... Args>
int launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

template <typename M>
UpdArgs<M> make_args(double lr, double clip_value, double weight_decay, unsigned flags) {
  UpdArgs<M> a;
  a.lr = (M)lr;
  a.clip = (M)(clip_value > 0 ? clip_value : 0);
  a.decay = (M)(1.0 - lr * weight_decay);
  a.wd = (M)weight_decay;
  a.inv_scale = (M)1;
  a.coef = (M)1;
  a.use_scale = (flags & LOMO_USE_SCALE) != 0;
  a.use_coef = (flags & LOMO_USE_COEF) != 0;
  a.use_clip = clip_value > 0;
  a.has_wd = weight_decay != 0.0;
  return a;
}

template <typename T, typename M>
int launch_update(void* p_, const void* g_, int64_t n, double lr, double clip, double wd,
                  unsigned flags, const void* state, cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  T* p = static_cast<T*>(p_);
  const T* g = static_cast<const T*>(g_);
  const lomo_state* st = static_cast<const lomo_state*>(state);
  UpdArgs<M> a = make_args<M>(lr, clip, wd, flags);
  const uintptr_t pa = (uintptr_t)p, ga = (uintptr_t)g;
  if ((pa & 15) == (ga & 15) && (pa % sizeof(T)) == 0) {
    int head = (int)(((16 - (pa & 15)) & 15) / sizeof(T));
    if (head > n) head = (int)n;
    const int64_t nvec = (n - head) / V;
    const int64_t tiles = (nvec + kThreads * kK1Vec - 1) / (kThreads * kK1Vec);
    const unsigned grid = (unsigned)(tiles > 0 ? tiles : 1);
    if (flags & LOMO_CHAINED)
      return launch(k1_update<T, M, true>, dim3(grid), dim3(kThreads), s, p, g, n, head, nvec, a,
                    flags, st);
    return launch(k1_update<T, M, false>, dim3(grid), dim3(kThreads), s, p, g, n, head, nvec, a,
                  flags, st);
  }
  const int grid = grid_for((n + 3) / 4, occupancy(k1_update_scalar<T, M>));
  return launch(k1_update_scalar<T, M>, dim3(grid), dim3(kThreads), s, p, g, n, a, flags, st);
}

template <typename T, typename M>
int launch_update_multi(void* const* pl, const void* const* gl, const int64_t* nl, int count,
                        double lr, double clip, double wd, unsigned flags, const void* state,
                        cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  UpdArgs<M> a = make_args<M>(lr, clip, wd, flags);
  for (int base = 0; base < count; base += kMulti) {
    MultiTable tab;
    tab.count = count - base < kMulti ? count - base : kMulti;
    int64_t max_n = 0;
    for (int i = 0; i < tab.count; ++i) {
      tab.p[i] = pl[base + i];
      tab.g[i] = gl[base + i];
      tab.n[i] = nl[base + i];
      tab.slot[i] = 0;
      if (nl[base + i] > max_n) max_n = nl[base + i];
    }
    if (max_n == 0) continue;
    int gx = (int)(((max_n + V - 1) / V + kThreads - 1) / kThreads);
    if (gx < 1) gx = 1;
    if (gx > 64) gx = 64;
    int rc = launch(k1_update_multi<T, M>, dim3(gx, tab.count), dim3(kThreads), s, tab, a, flags,
                    static_cast<const lomo_state*>(state));
    if (rc) return rc;
  }
  return 0;
}

template <typename T, typename M>
int launch_probe_multi(const void* const* gl, const int64_t* nl, const int* slots, int count,
                       unsigned flags, void* state, cudaStream_t s) {
  for (int base = 0; base < count; base += kMulti) {
    MultiTable tab;
    tab.count = count - base < kMulti ? count - base : kMulti;
    for (int i = 0; i < tab.count; ++i) {
      tab.p[i] = nullptr;
      tab.g[i] = gl[base + i];
      tab.n[i] = nl[base + i];
      tab.slot[i] = slots[base + i];
    }
    int rc = launch(k2_probe_multi<T, M>, dim3(tab.count), dim3(kThreads), s, tab, flags, state);
    if (rc) return rc;
  }
  return 0;
}

template <typename T, typename M>
int launch_probe(const void* g_, int64_t n, int slot, unsigned flags, void* state,
                 cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  const T* g = static_cast<const T*>(g_);
  const uintptr_t ga = (uintptr_t)g;
  if ((ga % sizeof(T)) != 0) return LOMO_E_ARG;
  int head = (int)(((16 - (ga & 15)) & 15) / sizeof(T));
  if (head > n) head = (int)n;
  const int64_t nvec = (n - head) / V;
  const int64_t tile = kThreads * kUnroll;
  int64_t per_cta = (nvec + LOMO_PROBE_BLOCKS_PER_SLOT - 1) / LOMO_PROBE_BLOCKS_PER_SLOT;
  per_cta = (per_cta + tile - 1) / tile * tile;
  if (per_cta < tile) per_cta = tile;
  int64_t grid = (nvec + per_cta - 1) / per_cta;
  if (grid < 1) grid = 1;
  if (flags & LOMO_CHAINED)
    return launch(k2_probe<T, M, true>, dim3((unsigned)grid), dim3(kThreads), s, g, n, head, nvec,
                  per_cta, slot, flags, state);
  return launch(k2_probe<T, M, false>, dim3((unsigned)grid), dim3(kThreads), s, g, n, head, nvec,
                per_cta, slot, flags, state);
}

template <typename T, typename M>
int launch_rs_update(void* p, const void* const* peers, int world, int64_t off, int64_t n,
                     double lr, double clip, double wd, unsigned flags, const void* state,
                     cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  if (n % V != 0 || (off * (int64_t)sizeof(T)) % 16 != 0 || ((uintptr_t)p & 15) != 0)
    return LOMO_E_ARG;
  const int64_t nvec = n / V;
  UpdArgs<M> a = make_args<M>(lr, clip, wd, flags);
  const unsigned grid = (unsigned)((nvec + kThreads - 1) / kThreads);
  return launch(k4_rs_update<T, M>, dim3(grid > 0 ? grid : 1), dim3(kThreads), s,
                static_cast<T*>(p), reinterpret_cast<const T* const*>(peers), world, off, nvec, a,
                flags, static_cast<const lomo_state*>(state));
}

template <typename T, typename M>
int launch_rs_probe(const void* const* peers, int world, int64_t off, int64_t n, int slot,
                    unsigned flags, void* state, cudaStream_t s, void* out = nullptr) {
  constexpr int V = 16 / sizeof(T);
  if (n % V != 0 || (off * (int64_t)sizeof(T)) % 16 != 0) return LOMO_E_ARG;
  const int64_t nvec = n / V;
  int64_t per_cta = (nvec + LOMO_PROBE_BLOCKS_PER_SLOT - 1) / LOMO_PROBE_BLOCKS_PER_SLOT;
  per_cta = (per_cta + kThreads - 1) / kThreads * kThreads;
  if (per_cta < kThreads) per_cta = kThreads;  // one vector per thread where the slot allows (tools/k4_local.py)
  int64_t grid = (nvec + per_cta - 1) / per_cta;
  if (grid < 1) grid = 1;
  if (out != nullptr) {
    if (((uintptr_t)out & 15) != 0) return LOMO_E_ARG;
    return launch(k4_rs_probe<T, M, true>, dim3((unsigned)grid), dim3(kThreads), s,
                  reinterpret_cast<const T* const*>(peers), world, off, nvec, per_cta, slot, flags,
                  state, static_cast<T*>(out));
  }
  return launch(k4_rs_probe<T, M, false>, dim3((unsigned)grid), dim3(kThreads), s,
                reinterpret_cast<const T* const*>(peers), world, off, nvec, per_cta, slot, flags,
                state, static_cast<T*>(nullptr));
}

template <typename T, typename M>
int launch_mc_update(void* p, const void* mc, int64_t n, double lr, double clip, double wd,
                     unsigned flags, const void* state, cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  if (n % V != 0 || ((uintptr_t)mc & 15) != 0 || ((uintptr_t)p & 15) != 0) return LOMO_E_ARG;
  const int64_t nvec = n / V;
  const unsigned grid = (unsigned)((nvec + kThreads - 1) / kThreads);
  return launch(k4_mc_update<T, M>, dim3(grid > 0 ? grid : 1), dim3(kThreads), s,
                static_cast<T*>(p), static_cast<const T*>(mc), nvec,
                make_args<M>(lr, clip, wd, flags), flags, static_cast<const lomo_state*>(state));
}

template <typename T, typename M>
int launch_mc_probe(const void* mc, int64_t n, int slot, unsigned flags, void* state,
                    cudaStream_t s, void* out = nullptr) {
  constexpr int V = 16 / sizeof(T);
  if (n % V != 0 || ((uintptr_t)mc & 15) != 0 || ((uintptr_t)out & 15) != 0) return LOMO_E_ARG;
  const int64_t nvec = n / V;
  int64_t per_cta = (nvec + LOMO_PROBE_BLOCKS_PER_SLOT - 1) / LOMO_PROBE_BLOCKS_PER_SLOT;
  per_cta = (per_cta + kThreads - 1) / kThreads * kThreads;
  if (per_cta < 4 * kThreads) per_cta = 4 * kThreads;
  int64_t grid = (nvec + per_cta - 1) / per_cta;
  if (grid < 1) grid = 1;
  return launch(k4_mc_probe<T, M>, dim3((unsigned)grid), dim3(kThreads), s,
                static_cast<const T*>(mc), nvec, per_cta, slot, flags, state, static_cast<T*>(out));
}

}  // namespace lomo_k
using namespace lomo_k;

// ==========================================================================
// C ABI
// ==========================================================================
extern "C" {

int lomo_abi_version(void) { return LOMO_ABI_VERSION; }

size_t lomo_state_bytes(int nslots) {
  if (nslots < 0) nslots = 0;
  return LOMO_STATE_SLOTS_OFFSET +
         sizeof(double) * ((size_t)nslots + nblocks_words(nslots) +
                           (size_t)nslots * LOMO_PROBE_BLOCKS_PER_SLOT);
}

int lomo_num_sms(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return 0;
  }
  return dev_info().sms;
}

int lomo_state_init(void* state, int nslots, double scale, int growth_interval,
                    double min_scale, double max_scale, double max_norm, double grad_div,
                    void* stream) {
  if (state == nullptr || nslots < 0 || growth_interval < 1) return LOMO_E_ARG;
  k_state_init<<<1, 256, 0, (cudaStream_t)stream>>>(state, nslots, scale, growth_interval,
                                                     min_scale, max_scale, max_norm, grad_div);
  return (int)cudaGetLastError();
}

int lomo_begin_step(void* state, const void* loss, int loss_dtype, void* stream) {
  if (state == nullptr) return LOMO_E_ARG;
  if (loss != nullptr && dtype_size(loss_dtype) == 0) return LOMO_E_ARG;
  k_begin_step<<<1, 256, 0, (cudaStream_t)stream>>>(state, loss, loss_dtype);
  return (int)cudaGetLastError();
}

int lomo_read_status(const void* state, lomo_status* out, void* stream) {
  if (state == nullptr || out == nullptr) return LOMO_E_ARG;
  return (int)cudaMemcpyAsync(out, state, sizeof(lomo_status), cudaMemcpyDeviceToHost,
                              (cudaStream_t)stream);
}

int lomo_fused_update(void* p, const void* g, int64_t n, int dtype, int math, double lr,
                      double clip_value, double weight_decay, unsigned flags,
                      const void* state, void* stream) {
  if (n < 0) return LOMO_E_ARG;
  if (n == 0) return 0;
  if (p == nullptr || g == nullptr) return LOMO_E_ARG;
  if ((flags & (LOMO_USE_SCALE | LOMO_USE_COEF | LOMO_USE_SKIP | LOMO_LR_FROM_STATE)) &&
      state == nullptr)
    return LOMO_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const bool f64 = math == LOMO_MATH_F64;
  if (math != LOMO_MATH_F32 && math != LOMO_MATH_F64) return LOMO_E_ARG;
  switch (dtype) {
    case LOMO_F16:
      return f64 ? launch_update<__half, double>(p, g, n, lr, clip_value, weight_decay, flags, state, s)
                 : launch_update<__half, float>(p, g, n, lr, clip_value, weight_decay, flags, state, s);
    case LOMO_BF16:
      return f64 ? launch_update<__nv_bfloat16, double>(p, g, n, lr, clip_value, weight_decay, flags, state, s)
                 : launch_update<__nv_bfloat16, float>(p, g, n, lr, clip_value, weight_decay, flags, state, s);
    case LOMO_F32:
      return f64 ? launch_update<float, double>(p, g, n, lr, clip_value, weight_decay, flags, state, s)
                 : launch_update<float, float>(p, g, n, lr, clip_value, weight_decay, flags, state, s);
    case LOMO_F64:
      // f64 storage always computes in f64
      return launch_update<double, double>(p, g, n, lr, clip_value, weight_decay, flags, state, s);
  }
  return LOMO_E_ARG;
}

int lomo_fused_update_multi(void* const* p_list, const void* const* g_list,
                            const int64_t* n_list, int count, int dtype, int math, double lr,
                            double clip_value, double weight_decay, unsigned flags,
                            const void* state, void* stream) {
  if (count < 0) return LOMO_E_ARG;
  if (count == 0) return 0;
  if (p_list == nullptr || g_list == nullptr || n_list == nullptr) return LOMO_E_ARG;
  for (int i = 0; i < count; ++i) {
    if (n_list[i] < 0) return LOMO_E_ARG;
    if (n_list[i] > 0 && (p_list[i] == nullptr || g_list[i] == nullptr)) return LOMO_E_ARG;
  }
  if ((flags & (LOMO_USE_SCALE | LOMO_USE_COEF | LOMO_USE_SKIP | LOMO_LR_FROM_STATE)) &&
      state == nullptr)
    return LOMO_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const bool f64 = math == LOMO_MATH_F64;
  if (math != LOMO_MATH_F32 && math != LOMO_MATH_F64) return LOMO_E_ARG;
#define LOMO_MULTI(T, M) \
  launch_update_multi<T, M>(p_list, g_list, n_list, count, lr, clip_value, weight_decay, flags, state, s)
  switch (dtype) {
    case LOMO_F16: return f64 ? LOMO_MULTI(__half, double) : LOMO_MULTI(__half, float);
    case LOMO_BF16: return f64 ? LOMO_MULTI(__nv_bfloat16, double) : LOMO_MULTI(__nv_bfloat16, float);
    case LOMO_F32: return f64 ? LOMO_MULTI(float, double) : LOMO_MULTI(float, float);
    case LOMO_F64: return LOMO_MULTI(double, double);
  }
#undef LOMO_MULTI
  return LOMO_E_ARG;
}

int lomo_rows_aggregate(const int64_t* sorted_ids, const int64_t* perm, const void* dy,
                        int64_t ntok, int64_t h, int dtype, void* rows, int64_t* row_ids,
                        void* stream) {
  if (ntok < 0 || h <= 0) return LOMO_E_ARG;
  if (ntok == 0) return 0;
  if (!sorted_ids || !perm || !dy || !rows || !row_ids) return LOMO_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned g = (unsigned)ntok;
  switch (dtype) {
    case LOMO_F16: return launch(k_rows_aggregate<__half>, dim3(g), dim3(kThreads), s, sorted_ids, perm, static_cast<const __half*>(dy), ntok, h, static_cast<__half*>(rows), row_ids);
    case LOMO_BF16: return launch(k_rows_aggregate<__nv_bfloat16>, dim3(g), dim3(kThreads), s, sorted_ids, perm, static_cast<const __nv_bfloat16*>(dy), ntok, h, static_cast<__nv_bfloat16*>(rows), row_ids);
    case LOMO_F32: return launch(k_rows_aggregate<float>, dim3(g), dim3(kThreads), s, sorted_ids, perm, static_cast<const float*>(dy), ntok, h, static_cast<float*>(rows), row_ids);
  }
  return LOMO_E_ARG;
}

int lomo_fused_update_rows(void* p, const void* rows, const int64_t* row_ids, int64_t nrows,
                           int64_t h, int dtype, int math, double lr, double clip_value,
                           double weight_decay, unsigned flags, const void* state,
                           void* stream) {
  if (nrows < 0 || h <= 0) return LOMO_E_ARG;
  if (nrows == 0) return 0;
  if (!p || !rows || !row_ids) return LOMO_E_ARG;
  if (weight_decay != 0.0) return LOMO_E_ARG;  // decay touches every row: use the dense K1
  if ((flags & (LOMO_USE_SCALE | LOMO_USE_COEF | LOMO_USE_SKIP | LOMO_LR_FROM_STATE)) &&
      state == nullptr)
    return LOMO_E_ARG;
  if (math != LOMO_MATH_F32 && math != LOMO_MATH_F64) return LOMO_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t ycta = (h / 8 + kThreads - 1) / kThreads;  // one 16-byte vector per thread
  const dim3 grid((unsigned)nrows, (unsigned)(ycta < 1 ? 1 : (ycta > 8 ? 8 : ycta)));
  const lomo_state* st = static_cast<const lomo_state*>(state);
  const bool f64 = math == LOMO_MATH_F64;
#define LOMO_ROWS(T, M)                                                                       \
  launch(k1_rows<T, M>, grid, dim3(kThreads), s, static_cast<T*>(p),                          \
         static_cast<const T*>(rows), row_ids, h, make_args<M>(lr, clip_value, 0.0, flags),   \
         flags, st)
  switch (dtype) {
    case LOMO_F16: return f64 ? LOMO_ROWS(__half, double) : LOMO_ROWS(__half, float);
    case LOMO_BF16: return f64 ? LOMO_ROWS(__nv_bfloat16, double) : LOMO_ROWS(__nv_bfloat16, float);
    case LOMO_F32: return f64 ? LOMO_ROWS(float, double) : LOMO_ROWS(float, float);
  }
#undef LOMO_ROWS
  return LOMO_E_ARG;
}

int lomo_probe_multi(const void* const* g_list, const int64_t* n_list, const int* slot_list,
                     int count, int dtype, unsigned flags, void* state, void* stream) {
  if (state == nullptr || count < 0) return LOMO_E_ARG;
  if (count == 0) return 0;
  if (g_list == nullptr || n_list == nullptr || slot_list == nullptr) return LOMO_E_ARG;
  for (int i = 0; i < count; ++i) {
    if (n_list[i] < 0) return LOMO_E_ARG;
    if (n_list[i] > 0 && g_list[i] == nullptr) return LOMO_E_ARG;
    if (slot_list[i] < 0) return LOMO_E_SLOT;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const bool f64 = (flags & LOMO_ACCUM_F64) != 0;
  switch (dtype) {
    case LOMO_F16:
      return f64 ? launch_probe_multi<__half, double>(g_list, n_list, slot_list, count, flags, state, s)
                 : launch_probe_multi<__half, float>(g_list, n_list, slot_list, count, flags, state, s);
    case LOMO_BF16:
      return f64 ? launch_probe_multi<__nv_bfloat16, double>(g_list, n_list, slot_list, count, flags, state, s)
                 : launch_probe_multi<__nv_bfloat16, float>(g_list, n_list, slot_list, count, flags, state, s);
    case LOMO_F32: return launch_probe_multi<float, double>(g_list, n_list, slot_list, count, flags, state, s);
    case LOMO_F64: return launch_probe_multi<double, double>(g_list, n_list, slot_list, count, flags, state, s);
  }
  return LOMO_E_ARG;
}

int lomo_probe(const void* g, int64_t n, int dtype, int slot, unsigned flags, void* state,
               void* stream) {
  if (state == nullptr || n < 0) return LOMO_E_ARG;
  if (slot < 0) return LOMO_E_SLOT;
  if (n > 0 && g == nullptr) return LOMO_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) return 0;
  const bool f64 = (flags & LOMO_ACCUM_F64) != 0;
  switch (dtype) {
    case LOMO_F16:
      return f64 ? launch_probe<__half, double>(g, n, slot, flags, state, s)
                 : launch_probe<__half, float>(g, n, slot, flags, state, s);
    case LOMO_BF16:
      return f64 ? launch_probe<__nv_bfloat16, double>(g, n, slot, flags, state, s)
                 : launch_probe<__nv_bfloat16, float>(g, n, slot, flags, state, s);
    case LOMO_F32: return launch_probe<float, double>(g, n, slot, flags, state, s);
    case LOMO_F64: return launch_probe<double, double>(g, n, slot, flags, state, s);
  }
  return LOMO_E_ARG;
}

int lomo_set_lr(void* state, double lr, void* stream) {
  if (state == nullptr) return LOMO_E_ARG;
  k_set_lr<<<1, 32, 0, (cudaStream_t)stream>>>(state, lr);
  return (int)cudaGetLastError();
}

int lomo_set_scaler_state(void* state, double scale, int clean_steps, int steps_applied,
                          int steps_skipped, void* stream) {
  if (state == nullptr || !(scale > 0.0) || clean_steps < 0 || steps_applied < 0 ||
      steps_skipped < 0)
    return LOMO_E_ARG;
  k_set_scaler<<<1, 32, 0, (cudaStream_t)stream>>>(state, scale, clean_steps, steps_applied,
                                                   steps_skipped);
  return (int)cudaGetLastError();
}

int lomo_update_coefs(const void* state, double weight_decay, unsigned flags, float* coefs_dev,
                      void* stream) {
  if (state == nullptr || coefs_dev == nullptr) return LOMO_E_ARG;
  k_update_coefs<<<1, 32, 0, (cudaStream_t)stream>>>(state, weight_decay, flags, coefs_dev);
  return (int)cudaGetLastError();
}

int lomo_fused_rs_update(void* p_shard, const void* const* peer_bufs_dev, int world,
                         int64_t offset, int64_t n, int dtype, int math, double lr,
                         double clip_value, double weight_decay, unsigned flags,
                         const void* state, void* stream) {
  if (n < 0 || offset < 0 || world < 1 || world > kMaxPeers) return LOMO_E_ARG;
  if (n == 0) return 0;
  if (p_shard == nullptr || peer_bufs_dev == nullptr) return LOMO_E_ARG;
  if ((flags & (LOMO_USE_SCALE | LOMO_USE_COEF | LOMO_USE_SKIP | LOMO_LR_FROM_STATE)) &&
      state == nullptr)
    return LOMO_E_ARG;
  if (math != LOMO_MATH_F32 && math != LOMO_MATH_F64) return LOMO_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const bool f64 = math == LOMO_MATH_F64;
#define LOMO_RSU(T, M) \
  launch_rs_update<T, M>(p_shard, peer_bufs_dev, world, offset, n, lr, clip_value, weight_decay, flags, state, s)
  switch (dtype) {
    case LOMO_F16: return f64 ? LOMO_RSU(__half, double) : LOMO_RSU(__half, float);
    case LOMO_BF16: return f64 ? LOMO_RSU(__nv_bfloat16, double) : LOMO_RSU(__nv_bfloat16, float);
    case LOMO_F32: return f64 ? LOMO_RSU(float, double) : LOMO_RSU(float, float);
    case LOMO_F64: return LOMO_RSU(double, double);
  }
#undef LOMO_RSU
  return LOMO_E_ARG;
}

static int rs_probe_impl(const void* const* peers, int world, int64_t offset, int64_t n, int dtype,
                         int slot, unsigned flags, void* state, void* out, void* stream) {
  if (state == nullptr || n < 0 || offset < 0 || world < 1 || world > kMaxPeers) return LOMO_E_ARG;
  if (slot < 0) return LOMO_E_SLOT;
  if (n == 0) return 0;
  if (peers == nullptr) return LOMO_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const bool f64 = (flags & LOMO_ACCUM_F64) != 0;
#define LOMO_RSP(T, M) launch_rs_probe<T, M>(peers, world, offset, n, slot, flags, state, s, out)
  switch (dtype) {
    case LOMO_F16: return f64 ? LOMO_RSP(__half, double) : LOMO_RSP(__half, float);
    case LOMO_BF16: return f64 ? LOMO_RSP(__nv_bfloat16, double) : LOMO_RSP(__nv_bfloat16, float);
    case LOMO_F32: return LOMO_RSP(float, double);
    case LOMO_F64: return LOMO_RSP(double, double);
  }
#undef LOMO_RSP
  return LOMO_E_ARG;
}

int lomo_fused_rs_probe(const void* const* peer_bufs_dev, int world, int64_t offset, int64_t n,
                        int dtype, int slot, unsigned flags, void* state, void* stream) {
  return rs_probe_impl(peer_bufs_dev, world, offset, n, dtype, slot, flags, state, nullptr,
                       stream);
}

int lomo_fused_rs_probe_keep(const void* const* peer_bufs_dev, int world, int64_t offset,
                             int64_t n, int dtype, int slot, unsigned flags, void* state,
                             void* out, void* stream) {
  if (out == nullptr && n > 0) return LOMO_E_ARG;
  return rs_probe_impl(peer_bufs_dev, world, offset, n, dtype, slot, flags, state, out, stream);
}

int lomo_fused_mc_update(void* p_shard, const void* mc, int64_t n, int dtype, int math, double lr,
                         double clip_value, double weight_decay, unsigned flags,
                         const void* state, void* stream) {
  if (n < 0) return LOMO_E_ARG;
  if (n == 0) return 0;
  if (p_shard == nullptr || mc == nullptr) return LOMO_E_ARG;
  if ((flags & (LOMO_USE_SCALE | LOMO_USE_COEF | LOMO_USE_SKIP | LOMO_LR_FROM_STATE)) &&
      state == nullptr)
    return LOMO_E_ARG;
  if (math != LOMO_MATH_F32 && math != LOMO_MATH_F64) return LOMO_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const bool f64 = math == LOMO_MATH_F64;
#define LOMO_MCU(T, M) \
  launch_mc_update<T, M>(p_shard, mc, n, lr, clip_value, weight_decay, flags, state, s)
  switch (dtype) {
    case LOMO_F16: return f64 ? LOMO_MCU(__half, double) : LOMO_MCU(__half, float);
    case LOMO_BF16: return f64 ? LOMO_MCU(__nv_bfloat16, double) : LOMO_MCU(__nv_bfloat16, float);
    case LOMO_F32: return f64 ? LOMO_MCU(float, double) : LOMO_MCU(float, float);
  }
#undef LOMO_MCU
  return LOMO_E_ARG;  // f64 storage: no multimem f64 vector reduction; use the IPC form
}

static int mc_probe_impl(const void* mc, int64_t n, int dtype, int slot, unsigned flags,
                         void* state, void* out, void* stream) {
  if (state == nullptr || n < 0) return LOMO_E_ARG;
  if (slot < 0) return LOMO_E_SLOT;
  if (n == 0) return 0;
  if (mc == nullptr) return LOMO_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const bool f64 = (flags & LOMO_ACCUM_F64) != 0;
#define LOMO_MCP(T, M) launch_mc_probe<T, M>(mc, n, slot, flags, state, s, out)
  switch (dtype) {
    case LOMO_F16: return f64 ? LOMO_MCP(__half, double) : LOMO_MCP(__half, float);
    case LOMO_BF16: return f64 ? LOMO_MCP(__nv_bfloat16, double) : LOMO_MCP(__nv_bfloat16, float);
    case LOMO_F32: return LOMO_MCP(float, double);
  }
#undef LOMO_MCP
  return LOMO_E_ARG;
}

int lomo_fused_mc_probe(const void* mc, int64_t n, int dtype, int slot, unsigned flags,
                        void* state, void* stream) {
  return mc_probe_impl(mc, n, dtype, slot, flags, state, nullptr, stream);
}

int lomo_fused_mc_probe_keep(const void* mc, int64_t n, int dtype, int slot, unsigned flags,
                             void* state, void* out, void* stream) {
  if (out == nullptr && n > 0) return LOMO_E_ARG;
  return mc_probe_impl(mc, n, dtype, slot, flags, state, out, stream);
}

int lomo_probe_rows(const float* partials_dev, int64_t rows, int64_t ld, int64_t cols, int slot,
                    void* state, void* stream) {
  if (state == nullptr || partials_dev == nullptr) return LOMO_E_ARG;
  if (rows < 1 || rows > LOMO_PROBE_BLOCKS_PER_SLOT || cols < 1 || ld < cols) return LOMO_E_ARG;
  if (slot < 0) return LOMO_E_SLOT;
  return launch(k6_rows, dim3((unsigned)rows), dim3(kThreads), (cudaStream_t)stream, partials_dev,
                ld, cols, slot, state);
}

int lomo_probe_rows_multi(const float* const* partials_dev, const int64_t* rows,
                          const int64_t* ld, const int64_t* cols, const int* slots, int count,
                          void* state, void* stream) {
  if (state == nullptr || count < 0) return LOMO_E_ARG;
  if (count == 0) return 0;
  if (partials_dev == nullptr || rows == nullptr || ld == nullptr || cols == nullptr ||
      slots == nullptr)
    return LOMO_E_ARG;
  for (int i = 0; i < count; ++i) {
    if (partials_dev[i] == nullptr || rows[i] < 1 || rows[i] > LOMO_PROBE_BLOCKS_PER_SLOT ||
        cols[i] < 1 || ld[i] < cols[i])
      return LOMO_E_ARG;
    if (slots[i] < 0) return LOMO_E_SLOT;
  }
  for (int base = 0; base < count; base += kMulti) {
    RowsTable tab;
    const int k = count - base < kMulti ? count - base : kMulti;
    int64_t max_rows = 1;
    for (int i = 0; i < k; ++i) {
      tab.part[i] = partials_dev[base + i];
      tab.rows[i] = rows[base + i];
      tab.ld[i] = ld[base + i];
      tab.cols[i] = cols[base + i];
      tab.slot[i] = slots[base + i];
      if (rows[base + i] > max_rows) max_rows = rows[base + i];
    }
    const int rc = launch(k6_rows_multi, dim3((unsigned)max_rows, (unsigned)k), dim3(kThreads),
                          (cudaStream_t)stream, tab, state);
    if (rc) return rc;
  }
  return 0;
}

int lomo_finalize_norm(void* state, void* stream) {
  if (state == nullptr) return LOMO_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  k3_reduce<<<dev_info().sms, kThreads, 0, s>>>(state, 0, nullptr);
  return (int)cudaGetLastError();
}

int lomo_scaler_on_clean(void* state, void* stream) {
  if (state == nullptr) return LOMO_E_ARG;
  k3_on_clean<<<1, 32, 0, (cudaStream_t)stream>>>(state);
  return (int)cudaGetLastError();
}

int lomo_local_norm_partial(const void* state, double* out2_dev, void* stream) {
  if (state == nullptr || out2_dev == nullptr) return LOMO_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  k3_reduce<<<dev_info().sms, kThreads, 0, s>>>(const_cast<void*>(state), 1, out2_dev);
  return (int)cudaGetLastError();
}

int lomo_finalize_norm_ranks(void* state, const double* parts_dev, int world, void* stream) {
  if (state == nullptr || parts_dev == nullptr || world < 1) return LOMO_E_ARG;
  k3_finalize_ranks<<<1, 32, 0, (cudaStream_t)stream>>>(state, parts_dev, world);
  return (int)cudaGetLastError();
}

}  // extern "C"
