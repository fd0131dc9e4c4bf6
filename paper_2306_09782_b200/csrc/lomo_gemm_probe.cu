// lomo_gemm_probe.cu -- K6: the pass-1 probe fused into the weight-gradient GEMM.
//
// Pass 1 of the two-pass protocol (stabilize.py:180-213) needs each weight
// gradient only for two things: whether any element is non-finite
// (probe_hook, :192-194) and its unscaled sum of squares (:195-197).  For a
// linear layer y = x W^T the gradient is dW = dy^T x (M = out, N = in,
// K = tokens).  K6 computes dW tile by tile on the tensor cores (the same
// tcgen05 2-SM mainloop as K5, so pass 2 re-derives bit-identical
// accumulators) and its epilogue turns each accumulator element into
//
//     v = float(round_storage(acc))          -- the gradient as autograd would
//                                               store it (fp16/bf16 RNE,
//                                               overflow -> inf)
//     s = isfinite(v) ? (v * inv_scale)^2 : NaN
//
// and reduces s along the N axis of the CTA tile (in registers: each epilogue
// thread owns one TMEM accumulator row; CUTLASS Sm90ColReduction in its
// non-final, atomic-free form).  The per-(row, N-tile) sums land in a
// [ceil(N/256), M] fp32 scratch matrix; k6_rows (lomo_kernels.cu,
// lomo_probe_rows) sums it in fixed order into the parameter's norm slot and
// raises the overflow flag if a sum is NaN.  No K2 launch re-reads the
// gradient, and none is written to HBM (ClippedStore below).
//
// Semantics vs the materialised path (cuBLAS dW -> K2):
//  * overflow: an element whose storage rounding is +-inf or NaN makes its
//    column sum NaN -> overflow flag, exactly probe_hook's any-non-finite rule;
//  * sum of squares: the squares of the storage-rounded gradient, scaled by
//    the device inv_scale; fp32 within a 128-row tile column, f64 across.
//    The summation order differs from K2's, so N agrees to fp32 rounding
//    (tests/test_gpu_gemm_update.py: relative 1e-6), and decisions are equal
//    on well-separated fixtures.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdlib.h>

#include "cute/tensor.hpp"
#include "cutlass/cutlass.h"
#include "cutlass/epilogue/collective/collective_builder.hpp"
#include "cutlass/epilogue/fusion/operations.hpp"
#include "cutlass/epilogue/fusion/sm90_callbacks_tma_warpspecialized.hpp"
#include "cutlass/gemm/collective/collective_builder.hpp"
#include "cutlass/gemm/device/gemm_universal_adapter.h"
#include "cutlass/gemm/kernel/gemm_universal.hpp"
#include "cutlass/util/packed_stride.hpp"

#include "lomo_b200.h"

inline bool lomo_gemm_pdl() {  // as in lomo_gemm_update.cu
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LOMO_GEMM_PDL");
    v = (e != nullptr && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

namespace lomo_probe_gemm {

using namespace cute;

// storage rounding of one fp32 accumulator value
template <typename Element>
CUTLASS_DEVICE float round_storage(float v);
template <>
CUTLASS_DEVICE float round_storage<cutlass::half_t>(float v) {
  return __half2float(__float2half_rn(v));
}
template <>
CUTLASS_DEVICE float round_storage<cutlass::bfloat16_t>(float v) {
  return __bfloat162float(__float2bfloat16_rn(v));
}

// (acc, inv_scale) -> squared unscaled storage-rounded gradient, NaN marks a
// non-finite element
template <typename Element>
struct ProbeSq {
  template <class T>
  struct Fn {
    CUTLASS_HOST_DEVICE T operator()(T const& acc, T const& s) const { return acc * s; }
  };
  template <int N>
  struct Fn<cutlass::Array<float, N>> {
    CUTLASS_DEVICE cutlass::Array<float, N> operator()(cutlass::Array<float, N> const& acc,
                                                       cutlass::Array<float, N> const& s) const {
      cutlass::Array<float, N> out;
      CUTLASS_PRAGMA_UNROLL
      for (int i = 0; i < N; ++i) {
        const float v = round_storage<Element>(acc[i]);
        const float u = v * s[i];
        out[i] = fabsf(v) <= 3.402823466e38f ? u * u : __int_as_float(0x7fffffff);
      }
      return out;
    }
  };
};

// root of the tree: pass the accumulator through (the reduction child's
// value is only there for its side effect)
template <class T>
struct First {
  struct Fn {
    CUTLASS_HOST_DEVICE T operator()(T const& a, T const&) const { return a; }
  };
};

// The by-product store without its HBM traffic.  CUTLASS 4.5's sm100 TMA
// epilogue has no void-D form, so the non-KeepGrad kernel keeps the store
// but its TMA descriptor describes only the first kClipN elements of row 0
// of D: every TMA store box outside that corner is clipped by the TMA unit
// and writes nothing (the smem staging still runs).  The caller's grad_out
// then needs only kClipN elements.  Everything else (tiles, EVT, schedule)
// is the builder's epilogue unchanged.
constexpr int kClipN = 32;
template <class Base>
struct ClippedStore : Base {
  using Base::Base;
  template <class ProblemShape>
  static typename Base::Params to_underlying_arguments(ProblemShape const& problem_shape,
                                                       typename Base::Arguments const& args,
                                                       void* workspace) {
    typename Base::Params p = Base::to_underlying_arguments(problem_shape, args, workspace);
    ProblemShape corner{1, kClipN, cute::get<2>(problem_shape), cute::get<3>(problem_shape)};
    p.tma_store_d = Base::to_underlying_arguments(corner, args, workspace).tma_store_d;
    return p;
  }
};

// EpiN: epilogue sub-tile 128 x EpiN, 0 = CUTLASS's choice (measured equal
// to 128 x 32 and better than 128 x 16 here, profiles/r01_gemm_shapes.md)
// KeepGrad: the epilogue stores dW in the storage dtype (GroupedLOMO keeps it
// as the retained gradient); otherwise the store is a by-product nobody reads
// back, staged as fp4 (e2m1, the fewest smem bytes) and clipped (ClippedStore);
// per 7B pass 10.8 ms with an fp16 store, 10.3 fp8, 9.80 fp4, 9.5 clipped
template <typename Element, bool KeepGrad = false, int ClusterN = 1, int EpiN = 0>
struct ProbeGemm {
  using ElementA = Element;  // dy [T, out] row-major == A (M=out, K=T), M-major
  using LayoutA = cutlass::layout::ColumnMajor;
  using ElementB = Element;  // x  [T, in]  row-major == B (K=T, N=in), N-major
  using LayoutB = cutlass::layout::RowMajor;
  using ElementAcc = float;
  static constexpr int kAlign = 128 / cutlass::sizeof_bits<Element>::value;
  using ElementD = cute::conditional_t<KeepGrad, Element, cutlass::float_e2m1_t>;
  static constexpr int kAlignD = 128 / cutlass::sizeof_bits<ElementD>::value;

  // identical mainloop configuration to K5 (lomo_gemm_update.cu)
  using MmaTileShape = Shape<_256, _256, _64>;
  using ClusterShape = Shape<_2, Int<ClusterN>, _1>;
  using CtaTileShape = Shape<_128, _256, _64>;  // one SM's half of the 2-SM tile
  static constexpr int kCtaM = 128;
  static constexpr int kCtaN = 256;

  template <class T>
  using ProbeFn = typename ProbeSq<Element>::template Fn<T>;
  template <class T>
  using FirstFn = typename First<T>::Fn;

  // D = round(acc) (the gradient, written to the caller's scratch by the
  // epilogue's TMA store, overlapped with the next tile's mainloop);
  // the row reduction consumes the squares and its output is dropped
  // reduce along N (each epilogue thread owns one accumulator row of the
  // TMEM tile, so the sum stays in its registers until one final shuffle)
  using RowReduce = cutlass::epilogue::fusion::Sm90ColReduction<
      cutlass::plus, cutlass::plus, cutlass::plus, 0, CtaTileShape, float, float,
      cutlass::FloatRoundStyle::round_to_nearest, Stride<_1, _0, _0>, 4,
      /*EnableNullptr=*/false, /*FinalReduction=*/false, /*VisitCheckOOB=*/true>;
  using Square = cutlass::epilogue::fusion::Sm90EVT<
      cutlass::epilogue::fusion::Sm90Compute<ProbeFn, float, float,
                                             cutlass::FloatRoundStyle::round_to_nearest>,
      cutlass::epilogue::fusion::Sm90AccFetch,
      cutlass::epilogue::fusion::Sm90ScalarBroadcast<double>>;
  using Reduced = cutlass::epilogue::fusion::Sm90EVT<RowReduce, Square>;
  using EVT = cutlass::epilogue::fusion::Sm90EVT<
      cutlass::epilogue::fusion::Sm90Compute<FirstFn, ElementD, float,
                                             cutlass::FloatRoundStyle::round_to_nearest>,
      cutlass::epilogue::fusion::Sm90AccFetch, Reduced>;

  using BuiltEpilogue = typename cutlass::epilogue::collective::CollectiveBuilder<
      cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, MmaTileShape, ClusterShape,
      cute::conditional_t<EpiN == 0, cutlass::epilogue::collective::EpilogueTileAuto,
                          Shape<_128, Int<(EpiN > 0 ? EpiN : 1)>>>,
      ElementAcc, float, void,
      cutlass::layout::RowMajor, kAlignD, ElementD, cutlass::layout::RowMajor, kAlignD,
      cute::conditional_t<EpiN == 0, cutlass::epilogue::collective::EpilogueScheduleAuto,
                          cutlass::epilogue::TmaWarpSpecialized2Sm>,
      EVT>::CollectiveOp;
  using CollectiveEpilogue =
      cute::conditional_t<KeepGrad, BuiltEpilogue, ClippedStore<BuiltEpilogue>>;

  using CollectiveMainloop = typename cutlass::gemm::collective::CollectiveBuilder<
      cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, ElementA, LayoutA, kAlign, ElementB,
      LayoutB, kAlign, ElementAcc, MmaTileShape, ClusterShape,
      cutlass::gemm::collective::StageCountAutoCarveout<static_cast<int>(
          sizeof(typename CollectiveEpilogue::SharedStorage))>,
      cutlass::gemm::collective::KernelScheduleAuto>::CollectiveOp;

  using GemmKernel = cutlass::gemm::kernel::GemmUniversal<Shape<int, int, int, int>,
                                                          CollectiveMainloop, CollectiveEpilogue>;
  using Gemm = cutlass::gemm::device::GemmUniversalAdapter<GemmKernel>;

  // partial sums: one per (row m, N-tile), m-major: [ceil(N/256)][round(M,128)]
  static int64_t rows(int N) { return (N + kCtaN - 1) / kCtaN; }
  static int64_t ld(int M) { return (M + kCtaM - 1) / kCtaM * kCtaM; }
  static size_t part_bytes(int M, int N) {
    return ((size_t)rows(N) * ld(M) * sizeof(float) + 255) / 256 * 256;
  }

  static typename Gemm::Arguments make_args(const void* dy, const void* x, void* grad, int M,
                                            int N, int K, const double* inv_scale_dev,
                                            float* partials) {
    using StrideA = typename Gemm::GemmKernel::StrideA;
    using StrideB = typename Gemm::GemmKernel::StrideB;
    using StrideC = typename Gemm::GemmKernel::StrideC;
    using StrideD = typename Gemm::GemmKernel::StrideD;
    StrideA sA = cutlass::make_cute_packed_stride(StrideA{}, make_shape(M, K, 1));
    StrideB sB = cutlass::make_cute_packed_stride(StrideB{}, make_shape(N, K, 1));
    StrideC sC = cutlass::make_cute_packed_stride(StrideC{}, make_shape(M, N, 1));
    StrideD sD = cutlass::make_cute_packed_stride(StrideD{}, make_shape(M, N, 1));
    typename Gemm::Arguments args{
        cutlass::gemm::GemmUniversalMode::kGemm,
        {M, N, K, 1},
        {static_cast<const ElementA*>(dy), sA, static_cast<const ElementB*>(x), sB},
        {{}, nullptr, sC, static_cast<ElementD*>(grad), sD}};
    // tree arguments are stored children first, node last
    typename cutlass::epilogue::fusion::Sm90ScalarBroadcast<double>::Arguments sb{};
    sb.scalars[0] = 1.0;
    sb.scalar_ptrs[0] = inv_scale_dev;  // nullptr: the host scalar 1.0
    typename Square::Arguments sa{{}, sb, {}};
    typename RowReduce::Arguments ra{};
    ra.ptr_col = partials;
    ra.reduction_identity = 0.f;
    typename Reduced::Arguments rd{sa, ra};
    args.epilogue.thread = typename EVT::Arguments{{}, rd, {}};
    args.hw_info = hw_info();
    return args;
  }

  static int run(const void* dy, const void* x, void* grad, int M, int N, int K,
                 const double* inv_scale_dev, void* workspace, size_t workspace_bytes,
                 cudaStream_t stream) {
    const size_t off = part_bytes(M, N);
    if (workspace_bytes < off) return LOMO_E_ARG;
    auto args = make_args(dy, x, grad, M, N, K, inv_scale_dev, static_cast<float*>(workspace));
    Gemm gemm;
    if (gemm.can_implement(args) != cutlass::Status::kSuccess) return LOMO_E_ARG;
    const size_t need = Gemm::get_workspace_size(args);
    if (off + need > workspace_bytes) return LOMO_E_ARG;
    if (gemm.initialize(args, static_cast<char*>(workspace) + off, stream) !=
        cutlass::Status::kSuccess)
      return LOMO_E_ARG;
    if (gemm.run(stream, nullptr, lomo_gemm_pdl()) != cutlass::Status::kSuccess) return (int)cudaGetLastError();
    return (int)cudaGetLastError();
  }

  static size_t workspace(int M, int N, int K) {
    auto args = make_args(nullptr, nullptr, nullptr, M, N, K, nullptr, nullptr);
    return part_bytes(M, N) + Gemm::get_workspace_size(args);
  }

  static cutlass::KernelHardwareInfo hw_info() {
    static int dev = -1, sms = 0;
    int d = 0;
    cudaGetDevice(&d);
    if (d != dev) {
      sms = cutlass::KernelHardwareInfo::query_device_multiprocessor_count(d);
      dev = d;
    }
    cutlass::KernelHardwareInfo hw;
    hw.device_id = d;
    hw.sm_count = sms;
    return hw;
  }
};

}  // namespace lomo_probe_gemm

extern "C" {

int lomo_gemm_probe(const void* dy, const void* x, void* grad_out, int64_t out_features,
                    int64_t in_features, int64_t tokens, int dtype, int slot, unsigned flags,
                    void* state, void* workspace, size_t workspace_bytes, void* stream) {
  if (dy == nullptr || x == nullptr || grad_out == nullptr || state == nullptr ||
      workspace == nullptr)
    return LOMO_E_ARG;
  if (out_features <= 0 || in_features <= 0 || tokens <= 0) return LOMO_E_ARG;
  if (out_features > INT32_MAX || in_features > INT32_MAX || tokens > INT32_MAX) return LOMO_E_ARG;
  if (flags & LOMO_ACCUM_F64) return LOMO_E_ARG;  // the exactness mode keeps GEMM + K2
  if (slot < 0) return LOMO_E_SLOT;
  const int M = (int)out_features, N = (int)in_features, K = (int)tokens;
  cudaStream_t s = (cudaStream_t)stream;
  const double* inv =
      (flags & LOMO_USE_SCALE) ? &static_cast<const lomo_state*>(state)->inv_scale : nullptr;
  int rc = LOMO_E_ARG;
  int64_t rows = 0, ld = 0;
  const bool keep = (flags & LOMO_PROBE_KEEP_GRAD) != 0;
  switch (dtype) {
    case LOMO_BF16: {
      using G = lomo_probe_gemm::ProbeGemm<cutlass::bfloat16_t>;
      if (G::rows(N) > LOMO_PROBE_BLOCKS_PER_SLOT) return LOMO_E_ARG;
      rc = keep ? lomo_probe_gemm::ProbeGemm<cutlass::bfloat16_t, true>::run(
                      dy, x, grad_out, M, N, K, inv, workspace, workspace_bytes, s)
                : G::run(dy, x, grad_out, M, N, K, inv, workspace, workspace_bytes, s);
      rows = G::rows(N);
      ld = G::ld(M);
      break;
    }
    case LOMO_F16: {
      using G = lomo_probe_gemm::ProbeGemm<cutlass::half_t>;
      if (G::rows(N) > LOMO_PROBE_BLOCKS_PER_SLOT) return LOMO_E_ARG;
      rc = keep ? lomo_probe_gemm::ProbeGemm<cutlass::half_t, true>::run(
                      dy, x, grad_out, M, N, K, inv, workspace, workspace_bytes, s)
                : G::run(dy, x, grad_out, M, N, K, inv, workspace, workspace_bytes, s);
      rows = G::rows(N);
      ld = G::ld(M);
      break;
    }
  }
  if (rc) return rc;
  if (flags & LOMO_DEFER_ROWS) return 0;  // lomo_gemm_probe_finish reduces it later
  return lomo_probe_rows(static_cast<const float*>(workspace), rows, ld, out_features, slot, state,
                         stream);
}

int lomo_gemm_probe_finish(void* const* workspaces, const int64_t* out_features,
                           const int64_t* in_features, const int* slots, int count, int dtype,
                           void* state, void* stream) {
  if (count < 0 || state == nullptr) return LOMO_E_ARG;
  if (count == 0) return 0;
  if (workspaces == nullptr || out_features == nullptr || in_features == nullptr ||
      slots == nullptr)
    return LOMO_E_ARG;
  if (dtype != LOMO_BF16 && dtype != LOMO_F16) return LOMO_E_ARG;
  using G = lomo_probe_gemm::ProbeGemm<cutlass::half_t>;  // same tiling for both dtypes
  static_assert(G::kCtaM == lomo_probe_gemm::ProbeGemm<cutlass::bfloat16_t>::kCtaM &&
                    G::kCtaN == lomo_probe_gemm::ProbeGemm<cutlass::bfloat16_t>::kCtaN,
                "tiling");
  constexpr int kChunk = 256;
  const float* parts[kChunk];
  int64_t rows[kChunk], ld[kChunk], cols[kChunk];
  for (int base = 0; base < count; base += kChunk) {
    const int k = count - base < kChunk ? count - base : kChunk;
    for (int i = 0; i < k; ++i) {
      const int64_t M = out_features[base + i], N = in_features[base + i];
      if (M <= 0 || N <= 0 || M > INT32_MAX || N > INT32_MAX) return LOMO_E_ARG;
      parts[i] = static_cast<const float*>(workspaces[base + i]);
      rows[i] = G::rows((int)N);
      ld[i] = G::ld((int)M);
      cols[i] = M;
    }
    const int rc = lomo_probe_rows_multi(parts, rows, ld, cols, slots + base, k, state, stream);
    if (rc) return rc;
  }
  return 0;
}

size_t lomo_gemm_probe_workspace(int64_t out_features, int64_t in_features, int64_t tokens,
                                 int dtype) {
  if (out_features <= 0 || in_features <= 0 || tokens <= 0) return 0;
  if (out_features > INT32_MAX || in_features > INT32_MAX || tokens > INT32_MAX) return 0;
  const int M = (int)out_features, N = (int)in_features, K = (int)tokens;
  size_t a = 0, b = 0;  // the larger of the two store variants
  if (dtype == LOMO_BF16) {
    a = lomo_probe_gemm::ProbeGemm<cutlass::bfloat16_t>::workspace(M, N, K);
    b = lomo_probe_gemm::ProbeGemm<cutlass::bfloat16_t, true>::workspace(M, N, K);
  } else if (dtype == LOMO_F16) {
    a = lomo_probe_gemm::ProbeGemm<cutlass::half_t>::workspace(M, N, K);
    b = lomo_probe_gemm::ProbeGemm<cutlass::half_t, true>::workspace(M, N, K);
  }
  return a > b ? a : b;
}

}  // extern "C"
