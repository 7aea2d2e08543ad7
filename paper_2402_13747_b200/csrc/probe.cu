// probe.cu — in-run peak probe for the FP64 pipe without FMA contraction.
//
// MEASURED_PEAKS.json carries HBM and bf16 figures only; the refinement kernel is
// bounded by separate DMUL/DADD issue (the parity contract forbids FMA), so its
// roofline denominator is measured here with the same flags (--fmad=false): every
// thread runs 8 independent mul+add chains; 2 flops per pair.
#include "common.cuh"
#include "../../include/pcray_b200.h"
#include "device_state.cuh"
#include "geom.cuh"

namespace pcr {
namespace {

__global__ void __launch_bounds__(256) fp64_probe_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = 1.0 + 1e-3 * (threadIdx.x + k);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = x[k] * a + b;  // DMUL + DADD (no fusion)
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

__global__ void libm_exp_kernel(const double* __restrict__ x, double* __restrict__ y, uint64_t n) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) y[i] = glibc_exp(x[i]);
}

}  // namespace
}  // namespace pcr

#include "handles.cuh"

extern "C" int pcr_fp64_probe(pcr_ctx* ctx, double* tflops) {
  if (!ctx || !tflops) return PCR_ERR_INVALID;
  try {
    PCR_CUDA(cudaSetDevice(ctx->c.device));
    cudaStream_t s = ctx->c.stream;
    pcr::DBuf<double> out(1, s);
    const int blocks = ctx->c.sm_count * 8, threads = 256, iters = 4096;
    cudaEvent_t a, b;
    PCR_CUDA(cudaEventCreate(&a));
    PCR_CUDA(cudaEventCreate(&b));
    pcr::fp64_probe_kernel<<<blocks, threads, 0, s>>>(out.get(), 64, 0.999999, 1e-7);  // warm-up
    PCR_CUDA(cudaEventRecord(a, s));
    pcr::fp64_probe_kernel<<<blocks, threads, 0, s>>>(out.get(), iters, 0.999999, 1e-7);
    PCR_CUDA(cudaEventRecord(b, s));
    PCR_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    PCR_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double flops = 2.0 * 8.0 * iters * static_cast<double>(blocks) * threads;
    *tflops = flops / (ms * 1e-3) / 1e12;
    return PCR_OK;
  } catch (const std::exception& e) {
    ctx->c.last_error = e.what();
    return PCR_ERR_CUDA;
  }
}

// The device exp() of the non-planar SDF on host arrays (parity hook: the tests compare
// it with the host libm bit for bit).
extern "C" int pcr_libm_exp_batch(pcr_ctx* ctx, const double* x, double* y, uint64_t n) {
  if (!ctx || (n && (!x || !y))) return PCR_ERR_INVALID;
  try {
    PCR_CUDA(cudaSetDevice(ctx->c.device));
    cudaStream_t s = ctx->c.stream;
    pcr::DBuf<double> dx(n ? n : 1, s), dy(n ? n : 1, s);
    pcr::h2d(dx.get(), x, n, s);
    if (n) {
      pcr::count_launch();
      pcr::libm_exp_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(dx.get(), dy.get(), n);
      PCR_LAUNCH_CHECK();
    }
    pcr::d2h(y, dy.get(), n, s);
    pcr::stream_wait(s);
    return PCR_OK;
  } catch (const std::exception& e) {
    ctx->c.last_error = e.what();
    return PCR_ERR_CUDA;
  }
}
