// k1_state_ab.cu -- A/B of the ways K1 can read the step state (skip, 1/scale,
// clip coefficient, lr) in the two-pass protocol's update pass, against the
// flag-free K1.  Not part of the product: it includes the product source and
// times one LLaMA-7B update pass (226 large bf16 tensors, one PDL launch per
// tensor, delivery order) per variant, alternating the variants 4 times.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -o tools/k1_state_ab tools/k1_state_ab.cu -lcuda && ./tools/k1_state_ab
#include "../paper_2306_09782_b200/csrc/lomo_kernels.cu"

#include <cstdio>
#include <functional>
#include <string>
#include <vector>

using namespace lomo_k;

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

typedef __nv_bfloat16 bf;

struct Rec {  // the compact pass-2 record (f32 math)
  int32_t skip;
  float inv_scale, coef, lr;
};

__device__ __forceinline__ uint4 ld_bcast(const void* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// MODE 1: every lane loads the 16-byte record (broadcast), after the wait
// MODE 2: lane 0 loads it, 4 x 32-bit shuffles
// MODE 3: every lane loads it BEFORE the PDL wait (unsafe bound)
// MODE 4: MODE 2 with the tile's data loads issued BEFORE the PDL wait
// MODE 5: data + record loads first, trigger dependents at entry, the PDL
//         wait only after the stores (the grid still completes after its
//         predecessor)
// MODE 6: no PDL wait at all (unsafe bound)
template <int MODE>
__global__ void __launch_bounds__(kThreads)
    k1_rec(bf* __restrict__ p, const bf* __restrict__ g, int64_t nvec, UpdArgs<float> a,
           const Rec* rec) {
  uint4* pv = reinterpret_cast<uint4*>(p);
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  uint4 r;
  uint4 P, G;
  if (MODE == 3) r = ld_bcast(rec);
  if (MODE >= 4 && i < nvec) {
    G = ld_stream_ro(gv + i);
    P = ld_stream_rw(pv + i);
  }
  if (MODE >= 5) {
    pdl_launch_dependents();
  } else {
    pdl_enter();
  }
  if (MODE <= 3 && i < nvec) {
    G = ld_stream_ro(gv + i);
    P = ld_stream_rw(pv + i);
  }
  if (MODE == 1) r = ld_bcast(rec);
  if (MODE == 2 || MODE >= 4) {
    if ((threadIdx.x & 31) == 0) r = ld_bcast(rec);
    r.x = __shfl_sync(0xffffffffu, r.x, 0);
    r.y = __shfl_sync(0xffffffffu, r.y, 0);
    r.z = __shfl_sync(0xffffffffu, r.z, 0);
    r.w = __shfl_sync(0xffffffffu, r.w, 0);
  }
  if (!r.x) {
    a.inv_scale = __uint_as_float(r.y);
    a.coef = __uint_as_float(r.z);
    a.lr = __uint_as_float(r.w);
    if (i < nvec) st_stream(pv + i, upd_vec<bf, float>(P, G, a));
  }
  if (MODE == 5) pdl_wait();
}

// K2 variants: tile = UNROLL x 256 vectors per CTA (one pass over the tile),
// MINB CTAs per SM, PF: L2 prefetch of the tile before the PDL wait, MATH:
// 0 = XOR only (load-path ceiling), 1 = fp32 squares
template <int UNROLL, int MINB, bool PF, int MATH, int SC = 0>
__global__ void __launch_bounds__(256, MINB)
    k2v(const bf* __restrict__ g, int64_t nvec, int64_t per_cta, double* part,
        const double* scale = nullptr) {
  __shared__ double sm[8];
  const int64_t beg = (int64_t)blockIdx.x * per_cta;
  const int64_t end = min(beg + per_cta, nvec);
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  if (PF && threadIdx.x == 0 && end > beg) prefetch_l2(gv + beg, (uint32_t)((end - beg) * 16));
  pdl_wait();
  pdl_launch_dependents();
  double sc = 1.0;
  if (SC == 2 && threadIdx.x == 0) asm volatile("ld.global.f64 %0, [%1];" : "=d"(sc) : "l"(scale));
  double acc = 0.0;
  uint32_t x = 0;
  for (int64_t base = beg + threadIdx.x; base < end; base += 256LL * UNROLL) {
    uint4 G[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t i = base + (int64_t)u * 256;
      if (i < end) G[u] = ld_stream_ro(gv + i);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t i = base + (int64_t)u * 256;
      if (i < end) {
        if (MATH == 0) x ^= G[u].x ^ G[u].y ^ G[u].z ^ G[u].w;
        else acc += vec_sumsq_nocheck<bf>(G[u], 1.0f, false);
      }
    }
  }
  if (MATH == 0) acc = (double)x;
  double b = block_sum(acc, sm);
  if (SC == 1 && threadIdx.x == 0) sc = *scale;
  if (threadIdx.x == 0) part[blockIdx.x] = b * sc * sc;
}

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

struct Tensor {
  bf *p, *g;
  int64_t n;
};

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

int main(int argc, char** argv) {
  const bool ncu_mode = argc > 1 && std::string(argv[1]) == "ncu";
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
  void* state;
  CK(cudaMalloc(&state, lomo_state_bytes((int)ts.size())));
  CK((cudaError_t)lomo_state_init(state, (int)ts.size(), 1024.0, 16, 1.0, 16777216.0, 1.0, 1.0,
                                  nullptr));
  CK((cudaError_t)lomo_set_lr(state, 0.05, nullptr));
  Rec h{0, 1.0f / 1024, 1.0f, 0.05f};
  Rec* rec;
  CK(cudaMalloc(&rec, 64));
  CK(cudaMemcpy(rec, &h, sizeof h, cudaMemcpyHostToDevice));
  CK(cudaDeviceSynchronize());
  const double gb = 6.0 * total / 1e9;
  const unsigned FL = LOMO_USE_SKIP | LOMO_USE_SCALE | LOMO_USE_COEF | LOMO_LR_FROM_STATE;

  auto product = [&](bool st) {
    return time_passes([&] {
      for (int i = (int)ts.size() - 1; i >= 0; --i)
        lomo_fused_update(ts[i].p, ts[i].g, ts[i].n, LOMO_BF16, LOMO_MATH_F32, 0.05, 0, 0,
                          st ? FL : 0, st ? state : nullptr, nullptr);
    }, 10);
  };
  auto variant = [&](auto kern) {
    UpdArgs<float> a = make_args<float>(0.05, 0.0, 0.0, LOMO_USE_SCALE | LOMO_USE_COEF);
    return time_passes([&] {
      for (int i = (int)ts.size() - 1; i >= 0; --i) {
        const int64_t nvec = ts[i].n / 8;
        launch(kern, dim3((unsigned)((nvec + 255) / 256)), dim3(256), (cudaStream_t)0, ts[i].p,
               (const bf*)ts[i].g, nvec, a, (const Rec*)rec);
      }
    }, 10);
  };
  if (ncu_mode) {  // a few launches of each probe form, for ncu --set full
    double* part;
    CK(cudaMalloc(&part, sizeof(double) * 65536));
    for (int i = (int)ts.size() - 2; i >= (int)ts.size() - 4; --i) {
      const int64_t nvec = ts[i].n / 8;
      lomo_probe(ts[i].g, ts[i].n, LOMO_BF16, i, LOMO_USE_SCALE, state, nullptr);
      launch(k2v<4, 5, true, 1, 2>, dim3((unsigned)((nvec + 1023) / 1024)), dim3(256),
             (cudaStream_t)0, (const bf*)ts[i].g, nvec, (int64_t)1024, part,
             (const double*)((char*)state + 8));
    }
    CK(cudaDeviceSynchronize());
    return 0;
  }
  const char* names[] = {"plain (no state)", "product state (record)",
                         "rec: lane0 ld.v4 + 4 shfl", "rec + data loads before wait",
                         "loads first, trigger at entry, wait at end", "no wait (unsafe)"};
  constexpr int NV = 6;
  double sum[NV] = {0};
  const int rounds = 4;
  for (int r = 0; r < rounds; ++r) {
    float ms[NV] = {product(false), product(true), variant(k1_rec<2>), variant(k1_rec<4>),
                    variant(k1_rec<5>), variant(k1_rec<6>)};
    for (int v = 0; v < NV; ++v) {
      printf("round %d %-42s %7.3f ms %7.1f GB/s\n", r, names[v], ms[v], gb / (ms[v] * 1e-3));
      sum[v] += ms[v];
    }
  }
  for (int v = 0; v < NV; ++v)
    printf("mean  %-42s %7.3f ms %7.1f GB/s\n", names[v], sum[v] / rounds,
           gb / (sum[v] / rounds * 1e-3));
  if (argc < 2 || std::string(argv[1]) != "k2") return 0;

  // ---- K2 probe pass (2 B/elem) ----
  const double gbp = 2.0 * total / 1e9;
  double* part;
  CK(cudaMalloc(&part, sizeof(double) * 65536));
  auto probe_product = [&] {
    return time_passes([&] {
      for (int i = (int)ts.size() - 1; i >= 0; --i)
        lomo_probe(ts[i].g, ts[i].n, LOMO_BF16, (int)ts.size() - 1 - i, LOMO_USE_SCALE, state,
                   nullptr);
    }, 10);
  };
  auto probe_v = [&](auto kern, int tile_vec) {
    return time_passes([&] {
      for (int i = (int)ts.size() - 1; i >= 0; --i) {
        const int64_t nvec = ts[i].n / 8;
        launch(kern, dim3((unsigned)((nvec + tile_vec - 1) / tile_vec)), dim3(256),
               (cudaStream_t)0, (const bf*)ts[i].g, nvec, (int64_t)tile_vec, part,
               (const double*)((char*)state + 8));
      }
    }, 10);
  };
  struct PV {
    const char* name;
    std::function<float()> f;
  };
  std::vector<PV> pv = {
      {"K2 product (USE_SCALE)", probe_product},
      {"k2v u4 t1024 5/SM pf scale early", [&] { return probe_v(k2v<4, 5, true, 1, 2>, 1024); }},
      {"k2v u8 t2048 5/SM pf scale early", [&] { return probe_v(k2v<8, 5, true, 1, 2>, 2048); }},
  };






  std::vector<double> psum(pv.size(), 0.0);
  const int prounds = 4;
  for (int r = 0; r < prounds; ++r)
    for (size_t vi = 0; vi < pv.size(); ++vi) {
      const size_t v = (r & 1) ? pv.size() - 1 - vi : vi;
      const float ms = pv[v].f();
      psum[v] += ms;
      printf("round %d %-44s %7.3f ms %7.1f GB/s\n", r, pv[v].name, ms, gbp / (ms * 1e-3));
    }
  for (size_t v = 0; v < pv.size(); ++v)
    printf("mean  %-44s %7.3f ms %7.1f GB/s\n", pv[v].name, psum[v] / prounds,
           gbp / (psum[v] / prounds * 1e-3));
  // flat read ceiling: one launch over the 32000x4096 head (262 MB)
  {
    const int64_t nvec = ts[0].n / 8;
    float ms = time_passes([&] {
      launch(k2v<8, 5, false, 0>, dim3((unsigned)((nvec + 2047) / 2048)), dim3(256),
             (cudaStream_t)0, (const bf*)ts[0].g, nvec, (int64_t)2048, part,
             (const double*)nullptr);
    }, 50);
    printf("single 32000x4096 read XOR: %7.3f ms %7.1f GB/s\n", ms, 2.0 * ts[0].n / 1e9 / (ms * 1e-3));
  }
  return 0;
}
