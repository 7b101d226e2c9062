// pipeline_variant.cu — one pipeline-kernel family per compilation: build.py compiles
// this file once per (RS_VARIANT_T, RS_VARIANT_STRICT, RS_VARIANT_REFL) so the eight
// fully unrolled kernel families (each with its resident / host-streaming and right /
// left-side variants) build in parallel. The launcher opts the kernel in to the device's full dynamic shared
// memory once per device and launches it (cooperative: all CTAs co-resident).
#include "rotseq_device.cuh"

#if !defined(RS_VARIANT_T) || !defined(RS_VARIANT_STRICT) || !defined(RS_VARIANT_REFL)
#error "compile with -DRS_VARIANT_T=double|float -DRS_VARIANT_STRICT=0|1 -DRS_VARIANT_REFL=0|1"
#endif

namespace rsk {

template <typename T, bool STRICT, bool REFL, bool HS, bool LEFT, int K, int MW>
cudaError_t launch_pipeline(const cudaLaunchConfig_t& cfg, const PipeParams& P) {
  auto kern = rs_pipeline_kernel<T, K, rows_for(sizeof(T)), STRICT, REFL, HS, LEFT, MW>;
  static std::atomic<int> configured{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const int bit = 1 << (dev & 31);
  if (!(configured.load(std::memory_order_relaxed) & bit)) {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit, std::memory_order_relaxed);
  }
  return cudaLaunchKernelEx(&cfg, kern, P);
}

#define RS_INST(HS, LEFT, K, MW)                                                                              \
  template cudaError_t launch_pipeline<RS_VARIANT_T, RS_VARIANT_STRICT != 0, RS_VARIANT_REFL != 0, HS, LEFT, K, MW>( \
      const cudaLaunchConfig_t&, const PipeParams&);
RS_INST(false, false, 8, max_warps_for(sizeof(RS_VARIANT_T), false, 8))
RS_INST(true, false, 8, max_warps_for(sizeof(RS_VARIANT_T), false, 8))
RS_INST(false, true, 8, max_warps_for(sizeof(RS_VARIANT_T), true, 8))
RS_INST(true, true, 8, max_warps_for(sizeof(RS_VARIANT_T), true, 8))
// fp64 right side: the 168-register build for plans of <= 12 warps per CTA
#if !RS_VARIANT_F32
RS_INST(false, false, 8, kSmallCtaWarps)
RS_INST(true, false, 8, kSmallCtaWarps)
#endif
// the wide windows (right side, off by default): 16 sweeps for fp32, 12 for fp64
#if RS_VARIANT_F32 && RS_F32_WIDE
RS_INST(false, false, 16, max_warps_for(4, false, 16))
RS_INST(true, false, 16, max_warps_for(4, false, 16))
#endif
#if !RS_VARIANT_F32 && RS_F64_WIDE
RS_INST(false, false, 12, max_warps_for(8, false, 12))
RS_INST(true, false, 12, max_warps_for(8, false, 12))
#endif

}  // namespace rsk
