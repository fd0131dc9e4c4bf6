// lomo_gemm_update.cu -- the LOMO update fused into the weight-gradient GEMM.
//
// For a linear layer y = x W^T (W: [out, in], x: [T, in], dy: [T, out]) the
// weight gradient is dW = dy^T x (M = out, N = in, K = T).  LOMO consumes dW
// only to apply p <- p - lr * coef * dW / scale (optim.py:52-54 with the
// update_hook stages, stabilize.py:217-224).  Here that update is the GEMM's
// epilogue: the tcgen05 tensor-core GEMM accumulates dW tile by tile in TMEM
// and the epilogue writes  p <- alpha * round(acc) + beta * p  (round = to the
// storage dtype, the gradient autograd / the reference tape would deliver) with
// alpha = -lr * coef / scale and beta = 1 - lr * wd, so the gradient is never
// materialised in HBM (K1 would have read it and p, and written p: 6 B/elem;
// the fused epilogue moves 4 B/elem and needs no separate launch).
//
// Built with the CUTLASS 4.x sm100 collective builders (tcgen05.mma issued by
// one thread, TMA loads, TMEM accumulators, 2-SM CTA pairs), instantiated
// inside this library; see DESIGN.md.  Value clipping is not linear in the
// accumulator and stays on the K1 path.
#include <cuda_runtime.h>
#include <stdlib.h>

#include "cute/tensor.hpp"
#include "cutlass/cutlass.h"
#include "cutlass/epilogue/collective/collective_builder.hpp"
#include "cutlass/epilogue/fusion/operations.hpp"
#include "cutlass/gemm/collective/collective_builder.hpp"
#include "cutlass/gemm/device/gemm_universal_adapter.h"
#include "cutlass/gemm/kernel/gemm_universal.hpp"
#include "cutlass/util/packed_stride.hpp"

#include "lomo_b200.h"

// PDL for the CUTLASS launches (built with CUTLASS_ENABLE_GDC_FOR_SM100: the
// kernels run griddepcontrol.wait before touching global memory), so a K5/K6
// prologue -- TMEM allocation, barrier init, descriptor prefetch -- overlaps the
// previous kernel's tail.  Opt-in (LOMO_GEMM_PDL=1): back to back it saves
// 3 % per 7B pass (tools/gemm_shapes.py), but inside the training step it
// measured 0.4-1.3 ms slower per step (profiles/r01_gemm_shapes.md).
inline bool lomo_gemm_pdl() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LOMO_GEMM_PDL");
    v = (e != nullptr && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

namespace lomo_gemm {

using namespace cute;

// fp32 accumulator -> the storage dtype's value (round to nearest even),
// kept in fp32 for the update arithmetic
template <typename Element>
struct RoundToStorage {
  template <class T>
  struct Fn {
    CUTLASS_HOST_DEVICE T operator()(T const& v) const { return v; }
  };
  template <int N>
  struct Fn<cutlass::Array<float, N>> {
    CUTLASS_DEVICE cutlass::Array<float, N> operator()(cutlass::Array<float, N> const& v) const {
      cutlass::Array<float, N> out;
      CUTLASS_PRAGMA_UNROLL
      for (int i = 0; i < N; ++i) {
        if constexpr (std::is_same<Element, cutlass::half_t>::value)
          out[i] = __half2float(__float2half_rn(v[i]));
        else
          out[i] = __bfloat162float(__float2bfloat16_rn(v[i]));
      }
      return out;
    }
  };
};

// EpiN: epilogue sub-tile 128 x EpiN (0 = CUTLASS's choice).  128 x 32 keeps
// more C-load / D-store stages in flight than the automatic 128 x 64: 4 %
// faster over a 7B pass (profiles/r01_gemm_shapes.md)
template <typename Element, int ClusterN = 1, int EpiN = 32>
struct FusedUpdateGemm {
  using ElementA = Element;                      // dy  [T, out] row-major == A (M=out, K=T), M-major
  using LayoutA = cutlass::layout::ColumnMajor;
  using ElementB = Element;                      // x   [T, in]  row-major == B (K=T, N=in), N-major
  using LayoutB = cutlass::layout::RowMajor;
  using ElementC = Element;                      // p   [out, in] row-major (source and destination)
  using LayoutC = cutlass::layout::RowMajor;
  using ElementAcc = float;
  using ElementCompute = float;
  static constexpr int kAlign = 128 / cutlass::sizeof_bits<Element>::value;

  using MmaTileShape = Shape<_256, _256, _64>;
  // one CTA pair per 256x256 tile; a 2x2 cluster (TMA multicast of the
  // A/B panels, cuBLAS's choice for 4096x4096) measured 1-5% slower here
  // (profiles/r01_gemm_shapes.md)
  using ClusterShape = Shape<_2, Int<ClusterN>, _1>;

  // D = fma(alpha, round_storage(acc), beta * C): the accumulator is first
  // rounded to the storage dtype -- the gradient the reference's tape would
  // deliver (tape.py:377, grad = self._round(grad)) and K1 would read --
  // then the update of optim.py:52-54 with one rounding (beta == 1 exactly
  // when there is no weight decay).
  template <class T>
  using RoundFn = typename RoundToStorage<Element>::template Fn<T>;
  using Scalar = cutlass::epilogue::fusion::Sm90ScalarBroadcast<float, Stride<_0, _0, int64_t>>;
  using RoundAcc = cutlass::epilogue::fusion::Sm90EVT<
      cutlass::epilogue::fusion::Sm90Compute<RoundFn, float, float,
                                             cutlass::FloatRoundStyle::round_to_nearest>,
      cutlass::epilogue::fusion::Sm90AccFetch>;
  using BetaC = cutlass::epilogue::fusion::Sm90EVT<
      cutlass::epilogue::fusion::Sm90Compute<cutlass::multiplies, float, float,
                                             cutlass::FloatRoundStyle::round_to_nearest>,
      Scalar, cutlass::epilogue::fusion::Sm90SrcFetch<ElementC>>;
  using Fusion = cutlass::epilogue::fusion::Sm90EVT<
      cutlass::epilogue::fusion::Sm90Compute<cutlass::homogeneous_multiply_add, ElementC, float,
                                             cutlass::FloatRoundStyle::round_to_nearest>,
      Scalar, RoundAcc, BetaC>;

  using CollectiveEpilogue = typename cutlass::epilogue::collective::CollectiveBuilder<
      cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, MmaTileShape, ClusterShape,
      cute::conditional_t<EpiN == 0, cutlass::epilogue::collective::EpilogueTileAuto,
                          Shape<_128, Int<(EpiN > 0 ? EpiN : 1)>>>,
      ElementAcc, ElementCompute, ElementC,
      LayoutC, kAlign, ElementC, LayoutC, kAlign,
      cute::conditional_t<EpiN == 0, cutlass::epilogue::collective::EpilogueScheduleAuto,
                          cutlass::epilogue::TmaWarpSpecialized2Sm>,
      Fusion>::CollectiveOp;

  using CollectiveMainloop = typename cutlass::gemm::collective::CollectiveBuilder<
      cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, ElementA, LayoutA, kAlign, ElementB,
      LayoutB, kAlign, ElementAcc, MmaTileShape, ClusterShape,
      cutlass::gemm::collective::StageCountAutoCarveout<static_cast<int>(
          sizeof(typename CollectiveEpilogue::SharedStorage))>,
      cutlass::gemm::collective::KernelScheduleAuto>::CollectiveOp;

  using GemmKernel = cutlass::gemm::kernel::GemmUniversal<Shape<int, int, int, int>,
                                                          CollectiveMainloop, CollectiveEpilogue>;
  using Gemm = cutlass::gemm::device::GemmUniversalAdapter<GemmKernel>;

  static int run(void* p, const void* dy, const void* x, int M, int N, int K, float alpha,
                 float beta, const float* coefs_dev, void* workspace, size_t workspace_bytes,
                 cudaStream_t stream) {
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
        {{}, static_cast<const ElementC*>(p), sC, static_cast<ElementC*>(p), sD}};
    // tree arguments: children first, node last; alpha/beta from device
    // memory at run time when coefs_dev is given (graph-capturable)
    typename Scalar::Arguments a{}, b{};
    a.scalars[0] = alpha;
    b.scalars[0] = beta;
    if (coefs_dev != nullptr) {
      a.scalar_ptrs[0] = coefs_dev;
      b.scalar_ptrs[0] = coefs_dev + 1;
    }
    args.epilogue.thread = typename Fusion::Arguments{
        a, typename RoundAcc::Arguments{{}, {}}, typename BetaC::Arguments{b, {}, {}}, {}};
    // persistent tile scheduler sized to the device (epilogue of tile i overlaps
    // the mainloop of tile i+1 through the double-buffered TMEM accumulator)
    args.hw_info = hw_info();
    Gemm gemm;
    if (gemm.can_implement(args) != cutlass::Status::kSuccess) return LOMO_E_ARG;
    const size_t need = Gemm::get_workspace_size(args);
    if (need > workspace_bytes) return LOMO_E_ARG;
    if (gemm.initialize(args, workspace, stream) != cutlass::Status::kSuccess) return LOMO_E_ARG;
    if (gemm.run(stream, nullptr, lomo_gemm_pdl()) != cutlass::Status::kSuccess) return (int)cudaGetLastError();
    return (int)cudaGetLastError();
  }

  static size_t workspace(int M, int N, int K) {
    typename Gemm::Arguments args{cutlass::gemm::GemmUniversalMode::kGemm, {M, N, K, 1}, {}, {}};
    args.hw_info = hw_info();
    return Gemm::get_workspace_size(args);
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

}  // namespace lomo_gemm

extern "C" {
int lomo_gemm_update(void* p, const void* dy, const void* x, int64_t out_features,
                     int64_t in_features, int64_t tokens, int dtype, double alpha, double beta,
                     void* workspace, size_t workspace_bytes, void* stream);

static int gemm_update(void* p, const void* dy, const void* x, int64_t out_features,
                       int64_t in_features, int64_t tokens, int dtype, double alpha, double beta,
                       const float* coefs_dev, void* workspace, size_t workspace_bytes,
                       void* stream) {
  if (p == nullptr || dy == nullptr || x == nullptr) return LOMO_E_ARG;
  if (out_features <= 0 || in_features <= 0 || tokens <= 0) return LOMO_E_ARG;
  if (out_features > INT32_MAX || in_features > INT32_MAX || tokens > INT32_MAX) return LOMO_E_ARG;
  const int M = (int)out_features, N = (int)in_features, K = (int)tokens;
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case LOMO_BF16:
      return lomo_gemm::FusedUpdateGemm<cutlass::bfloat16_t>::run(
          p, dy, x, M, N, K, (float)alpha, (float)beta, coefs_dev, workspace, workspace_bytes, s);
    case LOMO_F16:
      return lomo_gemm::FusedUpdateGemm<cutlass::half_t>::run(
          p, dy, x, M, N, K, (float)alpha, (float)beta, coefs_dev, workspace, workspace_bytes, s);
  }
  return LOMO_E_ARG;
}

int lomo_gemm_update(void* p, const void* dy, const void* x, int64_t out_features,
                     int64_t in_features, int64_t tokens, int dtype, double alpha, double beta,
                     void* workspace, size_t workspace_bytes, void* stream) {
  return gemm_update(p, dy, x, out_features, in_features, tokens, dtype, alpha, beta, nullptr,
                     workspace, workspace_bytes, stream);
}

int lomo_gemm_update_dev(void* p, const void* dy, const void* x, int64_t out_features,
                         int64_t in_features, int64_t tokens, int dtype, const float* coefs_dev,
                         void* workspace, size_t workspace_bytes, void* stream) {
  if (coefs_dev == nullptr) return LOMO_E_ARG;
  return gemm_update(p, dy, x, out_features, in_features, tokens, dtype, 0.0, 1.0, coefs_dev,
                     workspace, workspace_bytes, stream);
}

size_t lomo_gemm_update_workspace(int64_t out_features, int64_t in_features, int64_t tokens,
                                  int dtype) {
  if (out_features <= 0 || in_features <= 0 || tokens <= 0) return 0;
  if (dtype == LOMO_BF16)
    return lomo_gemm::FusedUpdateGemm<cutlass::bfloat16_t>::workspace(
        (int)out_features, (int)in_features, (int)tokens);
  if (dtype == LOMO_F16)
    return lomo_gemm::FusedUpdateGemm<cutlass::half_t>::workspace(
        (int)out_features, (int)in_features, (int)tokens);
  return 0;
}

}  // extern "C"
