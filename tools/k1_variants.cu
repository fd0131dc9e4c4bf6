// k1_variants.cu -- design-space probe for the K1 streaming update on B200.
// Not part of the product: a standalone harness that times variants of the
// bf16 / fp32-math update over the LLaMA-7B tensor list (one launch per
// tensor, the hook pattern) and over one flat buffer (one launch), so the
// per-launch boundary cost and the in-kernel efficiency can be separated.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -o tools/k1_variants tools/k1_variants.cu && ./tools/k1_variants
#include "../paper_2306_09782_b200/csrc/lomo_kernels.cu"

#include <cstdio>
#include <vector>

using namespace lomo_k;

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

typedef __nv_bfloat16 bf;

// ---- variant: grid-stride interleaved (CTA-consecutive 16B vectors) --------
template <int UNROLL>
__global__ void __launch_bounds__(256) v_interleaved(bf* __restrict__ p, const bf* __restrict__ g,
                                                     int64_t nvec, UpdArgs<float> a) {
  pdl_wait();
  pdl_launch_dependents();
  uint4* pv = reinterpret_cast<uint4*>(p);
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  const int64_t stride = (int64_t)gridDim.x * 256 * UNROLL;
  for (int64_t base = (int64_t)blockIdx.x * 256 * UNROLL + threadIdx.x; base < nvec;
       base += stride) {
    uint4 P[UNROLL], G[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t i = base + u * 256;
      if (i < nvec) {
        G[u] = ld_stream_ro(gv + i);
        P[u] = ld_stream_rw(pv + i);
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t i = base + u * 256;
      if (i < nvec) st_stream(pv + i, upd_vec<bf, float>(P[u], G[u], a));
    }
  }
}

// ---- variant: contiguous chunk per CTA with configurable unroll / threads ---
template <int UNROLL, int THREADS>
__global__ void __launch_bounds__(THREADS) v_chunked(bf* __restrict__ p, const bf* __restrict__ g,
                                                     int64_t nvec, UpdArgs<float> a) {
  pdl_wait();
  pdl_launch_dependents();
  const int64_t chunk = (nvec + gridDim.x - 1) / gridDim.x;
  const int64_t beg = (int64_t)blockIdx.x * chunk;
  const int64_t end = min(beg + chunk, nvec);
  uint4* pv = reinterpret_cast<uint4*>(p);
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  for (int64_t base = beg + threadIdx.x; base < end; base += (int64_t)THREADS * UNROLL) {
    uint4 P[UNROLL], G[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t i = base + (int64_t)u * THREADS;
      if (i < end) {
        G[u] = ld_stream_ro(gv + i);
        P[u] = ld_stream_rw(pv + i);
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t i = base + (int64_t)u * THREADS;
      if (i < end) st_stream(pv + i, upd_vec<bf, float>(P[u], G[u], a));
    }
  }
}

// ---- variant: one tile per CTA (non-persistent; the block scheduler balances)
template <int UNROLL>
__global__ void __launch_bounds__(256) v_tile(bf* __restrict__ p, const bf* __restrict__ g,
                                              int64_t nvec, UpdArgs<float> a) {
  pdl_wait();
  pdl_launch_dependents();
  uint4* pv = reinterpret_cast<uint4*>(p);
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  const int64_t base = (int64_t)blockIdx.x * 256 * UNROLL + threadIdx.x;
  uint4 P[UNROLL], G[UNROLL];
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    const int64_t i = base + u * 256;
    if (i < nvec) {
      G[u] = ld_stream_ro(gv + i);
      P[u] = ld_stream_rw(pv + i);
    }
  }
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    const int64_t i = base + u * 256;
    if (i < nvec) st_stream(pv + i, upd_vec<bf, float>(P[u], G[u], a));
  }
}

// ---- K2 variant: probe with per-CTA tile of PER vectors, U loads in flight --
template <int U>
__global__ void __launch_bounds__(256) v_probe(const bf* __restrict__ g, int64_t nvec,
                                               int64_t per, double* __restrict__ part) {
  __shared__ double sm[8];
  pdl_wait();
  pdl_launch_dependents();
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  const int64_t beg = (int64_t)blockIdx.x * per, end = min(beg + per, nvec);
  double acc = 0.0;
  bool bad = false;
  for (int64_t base = beg + threadIdx.x; base < end; base += 256 * U) {
    uint4 G[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 256;
      if (i < end) G[u] = ld_stream_ro(gv + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 256;
      if (i < end) acc += vec_sumsq<bf, float>(G[u], 1.0f, false, bad);
    }
  }
  const double r = block_sum(acc, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = r + (bad ? 1.0 : 0.0);
}

// ---- K2 variant: the product's structure minus one feature at a time -------
// MODE 0: product-like (state partial row, nblocks, __syncthreads_or flag)
// MODE 1: flag folded into the partial as NaN (no extra barrier)
// MODE 2: MODE 1 + no nblocks write
template <int MODE>
__global__ void __launch_bounds__(256, 5) v_probe2(const bf* __restrict__ g, int64_t nvec,
                                                   int64_t per, void* state, int slot) {
  __shared__ double sm[8];
  pdl_wait();
  pdl_launch_dependents();
  lomo_state* st = hdr(state);
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  const int64_t beg = (int64_t)blockIdx.x * per, end = min(beg + per, nvec);
  double acc = 0.0;
  bool bad = false;
  for (int64_t base = beg + threadIdx.x; base < end; base += 256 * 8) {
    uint4 G[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = base + u * 256;
      if (i < end) G[u] = ld_stream_ro(gv + i);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = base + u * 256;
      if (i < end) acc += vec_sumsq<bf, float>(G[u], 1.0f, false, bad);
    }
  }
  if (MODE == 0) {
    if (__syncthreads_or(bad) && threadIdx.x == 0) st->overflow = 1;
  } else if (bad) {
    acc = __longlong_as_double(0x7ff8000000000000ll);
  }
  const double r = block_sum(acc, sm);
  if (threadIdx.x == 0) {
    partials_of(st, slot)[blockIdx.x] = r;
    if (MODE < 2 && blockIdx.x == 0) nblocks_of(st)[slot] = (int32_t)gridDim.x;
  }
}

// ---- K2 variant with the L2 prefetch: PF tiles ahead (0 = own tile only) ----
template <int U, int AHEAD>
__global__ void __launch_bounds__(256, 5) v_probe_pf(const bf* __restrict__ g, int64_t nvec,
                                                     int64_t per, double* __restrict__ part) {
  __shared__ double sm[8];
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  const int64_t beg = (int64_t)blockIdx.x * per, end = min(beg + per, nvec);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int a = 0; a <= AHEAD; ++a) {
      const int64_t b0 = beg + a * per * gridDim.x / gridDim.x * 0 + a * per;
      const int64_t nt = min(per, nvec - b0);
      if (nt > 0 && (a == 0 || blockIdx.x < 148 * 5))
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gv + b0),
                     "r"((uint32_t)(nt * 16)) : "memory");
    }
  }
  pdl_wait();
  pdl_launch_dependents();
  double acc = 0.0;
  bool bad = false;
  for (int64_t base = beg + threadIdx.x; base < end; base += 256 * U) {
    uint4 G[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 256;
      if (i < end) G[u] = ld_stream_ro(gv + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 256;
      if (i < end) acc += vec_sumsq<bf, float>(G[u], 1.0f, false, bad);
    }
  }
  const double r = block_sum(acc, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = r + (bad ? 1.0 : 0.0);
}

// ---- K2: the product kernel with one feature switched at a time (MASK bits) --
// 1: non-finite flag folded into the partial as NaN (no __syncthreads_or)
// 2: no CTA-0 head/tail branch     4: no inv_scale branch in the loop
// 8: per-element finiteness test (vec_sumsq) instead of the rescan
template <int MASK>
__global__ void __launch_bounds__(256, 5) v_k2(const bf* __restrict__ g, int64_t n, int head,
                                                int64_t nvec, int64_t per_cta, int slot,
                                                unsigned flags, void* state) {
  constexpr int V = 8;
  __shared__ double sm[8];
  int nsl = 0;
  if (threadIdx.x == 0) {
    const int64_t b0 = (int64_t)blockIdx.x * per_cta;
    const int64_t nt = min(per_cta, nvec - b0);
    if (nt > 0) prefetch_l2(reinterpret_cast<const uint4*>(g + head) + b0, (uint32_t)(nt * 16));
    // (the round-1 product read nslots before the wait with ld.global.nc;
    // the round-2 kernel loads it after the wait)
    asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(nsl) : "l"(&hdr(state)->nslots));
  }
  pdl_wait();
  pdl_launch_dependents();
  lomo_state* st = hdr(state);
  const bool use_scale = (flags & LOMO_USE_SCALE) != 0;
  double acc = 0.0;
  bool bad = false;
  const int64_t beg = (int64_t)blockIdx.x * per_cta;
  const int64_t end = min(beg + per_cta, nvec);
  const uint4* gv = reinterpret_cast<const uint4*>(g + head);
  float inv_scale = 1.f;
  bool have_scale = !use_scale || (MASK & 4) || (MASK & 32);
  if (!(MASK & 2) && blockIdx.x == 0) {
    if (!have_scale) {
      inv_scale = (float)st->inv_scale;
      have_scale = true;
    }
    const int64_t tail0 = head + nvec * V;
    const int64_t ntail = n - tail0;
    for (int64_t i = threadIdx.x; i < head + ntail; i += blockDim.x) {
      const int64_t e = i < head ? i : tail0 + (i - head);
      float x = to_m<float>(g[e]);
      bad |= !is_fin(x);
      if (use_scale) x = x * inv_scale;
      acc += (double)x * (double)x;
    }
  }
  if ((MASK & 16) && !have_scale) {  // peeled form: the scale read outside the loop
    double sc;
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(sc) : "l"(&st->inv_scale));
    inv_scale = (float)sc;
    have_scale = true;
  }
  for (int64_t base = beg + threadIdx.x; base < end; base += 256 * 8) {
    uint4 G[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = base + (int64_t)u * 256;
      if (i < end) G[u] = ld_stream_ro(gv + i);
    }
    if (!(MASK & 16) && !have_scale) {
      double sc;
      asm volatile("ld.global.f64 %0, [%1];" : "=d"(sc) : "l"(&st->inv_scale));
      inv_scale = (float)sc;
      have_scale = true;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = base + (int64_t)u * 256;
      if (i < end) {
        if (MASK & 8) acc += vec_sumsq<bf, float>(G[u], inv_scale, use_scale, bad);
        else acc += vec_sumsq_nocheck<bf>(G[u], inv_scale, use_scale);
      }
    }
  }
  if (!(MASK & 8) && !is_fin(acc)) {
    for (int64_t i = beg + threadIdx.x; i < end && !bad; i += 256)
      bad = vec_has_nonfinite<bf>(ld_stream_ro(gv + i));
  }
  if ((MASK & 32) && use_scale) {  // unscaled sums, scaled once at the end (exact: power of 2)
    double sc;
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(sc) : "l"(&st->inv_scale));
    acc *= sc * sc;
  }
  if (MASK & 1) {
    if (bad) acc = __longlong_as_double(0x7ff8000000000000ll);
  } else if (__syncthreads_or(bad) && threadIdx.x == 0) {
    st->overflow = 1;
  }
  const double bsum = block_sum(acc, sm);
  if (threadIdx.x == 0) put_partial(st, slot, bsum, (int)gridDim.x, nsl);
}

// ---- variant: TMA bulk copies through a 4-stage shared-memory ring ---------
constexpr int kTileElems = 8192;  // 16 KB per operand per stage
constexpr int kStages = 4;
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, int phase) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(m)),
      "r"(phase));
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(m))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(256) v_tma(bf* __restrict__ p, const bf* __restrict__ g,
                                             int64_t n, UpdArgs<float> a) {
  extern __shared__ __align__(128) unsigned char smem[];
  bf* sp = reinterpret_cast<bf*>(smem);
  bf* sg = sp + kStages * kTileElems;
  uint64_t* full = reinterpret_cast<uint64_t*>(sg + kStages * kTileElems);
  pdl_wait();
  pdl_launch_dependents();
  const int64_t ntiles = n / kTileElems;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // tiles handled by this CTA: blockIdx.x, +gridDim.x, ...
  auto issue = [&](int64_t t, int s) {
    mbar_expect_tx(&full[s], 2 * kTileElems * sizeof(bf));
    bulk_load(sp + s * kTileElems, p + t * kTileElems, kTileElems * sizeof(bf), &full[s]);
    bulk_load(sg + s * kTileElems, g + t * kTileElems, kTileElems * sizeof(bf), &full[s]);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
      if (t < ntiles) issue(t, s);
    }
  }
  int k = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % kStages;
    mbar_wait(&full[s], (k / kStages) & 1);
    uint4* P = reinterpret_cast<uint4*>(sp + s * kTileElems);
    const uint4* G = reinterpret_cast<const uint4*>(sg + s * kTileElems);
#pragma unroll
    for (int j = 0; j < kTileElems * 2 / 16 / 256; ++j) {
      const int i = threadIdx.x + j * 256;
      P[i] = upd_vec<bf, float>(P[i], G[i], a);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_store(p + t * kTileElems, sp + s * kTileElems, kTileElems * sizeof(bf));
      const int64_t nt = t + (int64_t)kStages * gridDim.x;
      if (nt < ntiles) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        issue(nt, s);
      }
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------------------
struct Tensor {
  bf* p;
  bf* g;
  int64_t n;
};

__global__ void fill(bf* x, int64_t n, float lo, float hi, uint32_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    x[i] = __float2bfloat16(lo + (hi - lo) * (h & 0xffffff) / 16777216.0f);
  }
}

template <typename F>
float time_passes(F&& one_pass, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int i = 0; i < 3; ++i) one_pass();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) one_pass();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

template <typename K>
int occ_of(K k, int threads, size_t smem = 0) {
  int o = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, threads, smem));
  return o;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  // LLaMA-7B tensors (bytes identical to the bench), norms excluded
  std::vector<int64_t> sizes;
  sizes.push_back(32000LL * 4096);
  for (int l = 0; l < 32; ++l) {
    for (int k = 0; k < 4; ++k) sizes.push_back(4096LL * 4096);
    for (int k = 0; k < 3; ++k) sizes.push_back(4096LL * 11008);
  }
  sizes.push_back(32000LL * 4096);
  std::vector<Tensor> ts;
  int64_t total = 0;
  for (auto n : sizes) {
    Tensor t;
    t.n = n;
    CK(cudaMalloc(&t.p, n * 2));
    CK(cudaMalloc(&t.g, n * 2));
    fill<<<1184, 256>>>(t.p, n, -0.08f, 0.08f, 1);
    fill<<<1184, 256>>>(t.g, n, -1e-3f, 1e-3f, 2);
    ts.push_back(t);
    total += n;
  }
  CK(cudaDeviceSynchronize());
  UpdArgs<float> a = make_args<float>(0.05, 0.0, 0.0, 0);
  const double gb = 6.0 * total / 1e9;
  printf("sms %d, %zu tensors, %.3f G elements, %.2f GB algorithmic per pass\n", sms, ts.size(),
         total / 1e9, gb);

  auto report = [&](const char* name, float ms) {
    printf("%-44s %8.3f ms  %7.1f GB/s\n", name, ms, gb / (ms * 1e-3));
  };

  // product kernel through the C-ABI (PDL on)
  report("product lomo_fused_update (per tensor)", time_passes([&] {
           for (int i = (int)ts.size() - 1; i >= 0; --i)
             lomo_fused_update(ts[i].p, ts[i].g, ts[i].n, LOMO_BF16, LOMO_MATH_F32, 0.05, 0, 0, 0,
                               nullptr, nullptr);
         }, 10));

  auto per_tensor = [&](auto kern, int threads, int grid_per_sm, size_t smem, const char* name,
                        bool pdl, bool vec_units) {
    float ms = time_passes([&] {
      for (int i = (int)ts.size() - 1; i >= 0; --i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(sms * grid_per_sm);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const int64_t units = vec_units ? ts[i].n / 8 : ts[i].n;
        CK(cudaLaunchKernelEx(&cfg, kern, ts[i].p, (const bf*)ts[i].g, units, a));
      }
    }, 10);
    report(name, ms);
  };

  char buf[128];
  auto tiled = [&](auto kern, int unroll, const char* name) {
    float ms = time_passes([&] {
      for (int i = (int)ts.size() - 1; i >= 0; --i) {
        cudaLaunchConfig_t cfg = {};
        const int64_t nvec = ts[i].n / 8;
        cfg.gridDim = dim3((unsigned)((nvec + 256 * unroll - 1) / (256 * unroll)));
        cfg.blockDim = dim3(256);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, kern, ts[i].p, (const bf*)ts[i].g, nvec, a));
      }
    }, 10);
    report(name, ms);
  };
  tiled(v_tile<1>, 1, "tile 256 vec/CTA (u1)");
  tiled(v_tile<2>, 2, "tile 512 vec/CTA (u2)");
  tiled(v_tile<4>, 4, "tile 1024 vec/CTA (u4)");
  tiled(v_tile<8>, 8, "tile 2048 vec/CTA (u8)");
  tiled(v_tile<16>, 16, "tile 4096 vec/CTA (u16)");
  {
    auto k = v_chunked<4, 256>;
    int o = occ_of(k, 256);
    for (int gps : {o, 2 * o, 4 * o, 8 * o, 16 * o}) {
      snprintf(buf, sizeof buf, "chunked u4 t256 grid=%dx%d pdl", sms, gps);
      per_tensor(k, 256, gps, 0, buf, true, true);
    }
    snprintf(buf, sizeof buf, "chunked u4 t256 grid=%dx%d nopdl", sms, o);
    per_tensor(k, 256, o, 0, buf, false, true);
  }
  {
    auto k = v_chunked<8, 256>;
    int o = occ_of(k, 256);
    for (int gps : {o, 4 * o, 8 * o}) {
      snprintf(buf, sizeof buf, "chunked u8 t256 grid=%dx%d pdl", sms, gps);
      per_tensor(k, 256, gps, 0, buf, true, true);
    }
  }
  {
    auto k = v_chunked<2, 256>;
    int o = occ_of(k, 256);
    for (int gps : {4 * o, 8 * o, 16 * o}) {
      snprintf(buf, sizeof buf, "chunked u2 t256 grid=%dx%d pdl", sms, gps);
      per_tensor(k, 256, gps, 0, buf, true, true);
    }
  }
  {
    auto k = v_chunked<2, 512>;
    int o = occ_of(k, 512);
    snprintf(buf, sizeof buf, "chunked u2 t512 grid=%dx%d pdl", sms, o);
    per_tensor(k, 512, o, 0, buf, true, true);
  }
  {
    auto k = v_chunked<4, 128>;
    int o = occ_of(k, 128);
    snprintf(buf, sizeof buf, "chunked u4 t128 grid=%dx%d pdl", sms, o);
    per_tensor(k, 128, o, 0, buf, true, true);
  }
  for (int u : {2, 4, 8}) {
    auto k = u == 2 ? v_interleaved<2> : (u == 4 ? v_interleaved<4> : v_interleaved<8>);
    int o = occ_of(k, 256);
    for (int m : {1, 4}) {
      snprintf(buf, sizeof buf, "interleaved u%d t256 grid=%dx%d pdl", u, sms, o * m);
      per_tensor(k, 256, o * m, 0, buf, true, true);
    }
  }
  {
    size_t smem = kStages * kTileElems * 2 * 2 + 64;
    CK(cudaFuncSetAttribute(v_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int o = occ_of(v_tma, 256, smem);
    snprintf(buf, sizeof buf, "tma 4x16KB ring grid=%dx%d pdl", sms, o);
    per_tensor(v_tma, 256, o, smem, buf, true, false);
  }

  // K2 probe variants (read g only, 2 B/elem)
  {
    double* part;
    CK(cudaMalloc(&part, sizeof(double) * (1 << 20)));
    const double gbp = 2.0 * total / 1e9;
    auto probe_pass = [&](auto kern, int64_t min_per, int64_t max_ctas, const char* name) {
      float ms = time_passes([&] {
        for (int i = (int)ts.size() - 1; i >= 0; --i) {
          const int64_t nvec = ts[i].n / 8;
          int64_t per = (nvec + max_ctas - 1) / max_ctas;
          per = (per + min_per - 1) / min_per * min_per;
          if (per < min_per) per = min_per;
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3((unsigned)((nvec + per - 1) / per));
          cfg.blockDim = dim3(256);
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          CK(cudaLaunchKernelEx(&cfg, kern, (const bf*)ts[i].g, nvec, per, part));
        }
      }, 10);
      printf("%-44s %8.3f ms  %7.1f GB/s\n", name, ms, gbp / (ms * 1e-3));
    };
    {  // the product K2 through the C-ABI, with and without the scale read
      void* st;
      const int ns = (int)ts.size();
      CK(cudaMalloc(&st, lomo_state_bytes(ns)));
      CK((cudaError_t)lomo_state_init(st, ns, 1024.0, 16, 1.0, 16777216.0, 1.0, 1.0, nullptr));
      for (unsigned fl : {0u, (unsigned)LOMO_USE_SCALE}) {
        float ms = time_passes([&] {
          for (int i = ns - 1; i >= 0; --i)
            lomo_probe(ts[i].g, ts[i].n, LOMO_BF16, ns - 1 - i, fl, st, nullptr);
        }, 10);
        printf("%-44s %8.3f ms  %7.1f GB/s\n",
               fl ? "product lomo_probe (per tensor, USE_SCALE)" : "product lomo_probe (per tensor)",
               ms, gbp / (ms * 1e-3));
      }
      auto p2 = [&](auto kern, const char* name) {
        float ms = time_passes([&] {
          for (int i = ns - 1; i >= 0; --i) {
            const int64_t nvec = ts[i].n / 8;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)((nvec + 2047) / 2048));
            cfg.blockDim = dim3(256);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            CK(cudaLaunchKernelEx(&cfg, kern, (const bf*)ts[i].g, nvec, (int64_t)2048, st,
                                  ns - 1 - i));
          }
        }, 10);
        printf("%-44s %8.3f ms  %7.1f GB/s\n", name, ms, gbp / (ms * 1e-3));
      };
      auto pk = [&](auto kern, unsigned fl, const char* name) {
        float ms = time_passes([&] {
          for (int i = ns - 1; i >= 0; --i) {
            const int64_t nvec = ts[i].n / 8;
            int64_t per = (nvec + LOMO_PROBE_BLOCKS_PER_SLOT - 1) / LOMO_PROBE_BLOCKS_PER_SLOT;
            per = (per + 2047) / 2048 * 2048;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)((nvec + per - 1) / per));
            cfg.blockDim = dim3(256);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            CK(cudaLaunchKernelEx(&cfg, kern, (const bf*)ts[i].g, ts[i].n, 0, nvec, per, ns - 1 - i,
                                  fl, st));
          }
        }, 10);
        printf("%-44s %8.3f ms  %7.1f GB/s\n", name, ms, gbp / (ms * 1e-3));
      };
      for (int rep = 0; rep < 2; ++rep) {
        pk(v_k2<0>, 0u, "k2 clone (product)");
        pk(v_k2<1>, 0u, "k2 clone: NaN-folded flag");
        pk(v_k2<2>, 0u, "k2 clone: no head/tail branch");
        pk(v_k2<8>, 0u, "k2 clone: per-element check");
        pk(v_k2<3>, 0u, "k2 clone: NaN + no head/tail");
        pk(v_k2<0>, (unsigned)LOMO_USE_SCALE, "k2 clone (product) USE_SCALE");
        pk(v_k2<1>, (unsigned)LOMO_USE_SCALE, "k2 clone NaN-folded USE_SCALE");
        pk(v_k2<4>, (unsigned)LOMO_USE_SCALE, "k2 clone USE_SCALE, no scale read");
        pk(v_k2<16>, (unsigned)LOMO_USE_SCALE, "k2 clone USE_SCALE, scale read pre-loop");
        pk(v_k2<32>, (unsigned)LOMO_USE_SCALE, "k2 clone USE_SCALE, scaled at the end");
        pk(v_k2<33>, (unsigned)LOMO_USE_SCALE, "k2 clone USE_SCALE, end-scaled + NaN flag");
        float ms = time_passes([&] {
          for (int i = ns - 1; i >= 0; --i)
            lomo_probe(ts[i].g, ts[i].n, LOMO_BF16, ns - 1 - i, LOMO_USE_SCALE, st, nullptr);
        }, 10);
        printf("%-44s %8.3f ms  %7.1f GB/s\n", "product (peeled) USE_SCALE", ms, gbp / (ms * 1e-3));
        ms = time_passes([&] {
          for (int i = ns - 1; i >= 0; --i)
            lomo_probe(ts[i].g, ts[i].n, LOMO_BF16, ns - 1 - i, 0u, st, nullptr);
        }, 10);
        printf("%-44s %8.3f ms  %7.1f GB/s\n", "product (peeled)", ms, gbp / (ms * 1e-3));
      }
      p2(v_probe2<0>, "k2-like: state row + syncthreads_or");
      p2(v_probe2<1>, "k2-like: NaN-folded flag");
      p2(v_probe2<2>, "k2-like: NaN flag, no nblocks");
      CK(cudaFree(st));
    }
    probe_pass(v_probe<1>, 256, 1 << 20, "probe 256 vec/CTA u1");
    probe_pass(v_probe<2>, 512, 1 << 20, "probe 512 vec/CTA u2");
    probe_pass(v_probe<4>, 1024, 1 << 20, "probe 1024 vec/CTA u4");
    probe_pass(v_probe<4>, 1024, 4096, "probe >=1024 vec/CTA u4, <=4096 CTAs");
    probe_pass(v_probe<4>, 2048, 1 << 20, "probe 2048 vec/CTA u4");
    probe_pass(v_probe<8>, 2048, 1 << 20, "probe 2048 vec/CTA u8");
    probe_pass(v_probe_pf<8, 0>, 2048, 1 << 20, "probe 2048 u8 + L2 prefetch own tile");
    probe_pass(v_probe_pf<4, 0>, 1024, 1 << 20, "probe 1024 u4 + L2 prefetch own tile");
    probe_pass(v_probe_pf<8, 0>, 4096, 1 << 20, "probe 4096 u8 + L2 prefetch own tile");
    probe_pass(v_probe_pf<8, 1>, 2048, 1 << 20, "probe 2048 u8 + prefetch own + next");
    probe_pass(v_probe_pf<16, 0>, 4096, 1 << 20, "probe 4096 u16 + L2 prefetch own tile");
    probe_pass(v_probe<8>, 4096, 1 << 20, "probe 4096 vec/CTA u8");
    probe_pass(v_probe<8>, 8192, 1 << 20, "probe 8192 vec/CTA u8");
    probe_pass(v_probe<16>, 8192, 1 << 20, "probe 8192 vec/CTA u16");
    // K1-like geometry: tiles of >= nvec/8192 vectors (the partial-row limit),
    // as small as one vector per thread, own tile prefetched into L2
    probe_pass(v_probe_pf<1, 0>, 256, 8192, "probe >=256 u1 (<=8192 CTAs) + prefetch");
    probe_pass(v_probe_pf<2, 0>, 512, 8192, "probe >=512 u2 (<=8192 CTAs) + prefetch");
    probe_pass(v_probe_pf<4, 0>, 1024, 8192, "probe >=1024 u4 (<=8192 CTAs) + prefetch");
    // read ceiling: the same kernels over ONE flat 2.4 GB buffer (one launch)
    {
      const int64_t nflat = 3 * (int64_t)ts[0].n;  // the largest tensor, x3 (padding)
      bf* flat;
      CK(cudaMalloc(&flat, nflat * 2));
      CK(cudaMemset(flat, 0, nflat * 2));
      for (int64_t per : {(int64_t)2048, (int64_t)8192}) {
        const int64_t nvec = nflat / 8;
        float ms = time_passes([&] {
          v_probe<8><<<(unsigned)((nvec + per - 1) / per), 256>>>(flat, nvec, per, part);
        }, 10);
        printf("flat one launch %5lld vec/CTA u8 (%.2f GB)     %8.3f ms  %7.1f GB/s\n",
               (long long)per, 2.0 * nflat / 1e9, ms, 2.0 * nflat / 1e9 / (ms * 1e-3));
      }
      CK(cudaFree(flat));
    }
  }

  // one flat launch over the biggest tensor only (in-kernel efficiency)
  {
    auto k = v_chunked<4, 256>;
    int o = occ_of(k, 256);
    Tensor& t = ts[0];
    float ms = time_passes([&] {
      k<<<sms * o, 256>>>(t.p, t.g, t.n / 8, a);
    }, 20);
    printf("%-44s %8.3f ms  %7.1f GB/s\n", "single 32000x4096 chunked u4", ms,
           6.0 * t.n / 1e9 / (ms * 1e-3));
    Tensor& t2 = ts[1];
    ms = time_passes([&] {
      k<<<sms * o, 256>>>(t2.p, t2.g, t2.n / 8, a);
    }, 50);
    printf("%-44s %8.3f ms  %7.1f GB/s\n", "single 4096x4096 chunked u4 (L2-warm)", ms,
           6.0 * t2.n / 1e9 / (ms * 1e-3));
  }
  // plain copy for reference (cudaMemcpy D2D of the biggest tensor)
  {
    Tensor& t = ts[0];
    float ms = time_passes([&] { CK(cudaMemcpyAsync(t.p, t.g, t.n * 2, cudaMemcpyDeviceToDevice)); }, 20);
    printf("%-44s %8.3f ms  %7.1f GB/s (read+write)\n", "cudaMemcpy D2D 262MB", ms,
           4.0 * t.n / 1e9 / (ms * 1e-3));
  }
  return 0;
}
