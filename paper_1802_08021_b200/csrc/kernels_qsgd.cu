// kernels_qsgd.cu — stand-alone QSGD encode/decode (§6) for the
// C-ABI calls sparcml_quantize / sparcml_dequantize.  The DSAR path uses the
// same device code fused into the owner window kernel (encode) and the
// allgather pull (decode).
#include <algorithm>

#include "kernels.h"

namespace sparcml {

// one block per kThreads*4 = 1024 consecutive values
__global__ void __launch_bounds__(kThreads) quantize_kernel(const float* __restrict__ x, uint64_t n, int bits,
                                                            uint32_t bucket, uint32_t k0, uint32_t k1,
                                                            uint64_t ctr_base, uint8_t* __restrict__ codes,
                                                            float* __restrict__ scales, int norm) {
  __shared__ uint32_t bmax[kWin / 8];
  const uint64_t nwin = (n + kWin - 1) / kWin;
  for (uint64_t w = blockIdx.x; w < nwin; w += gridDim.x) {
    const uint64_t e = w * kWin + (uint64_t)threadIdx.x * 4;
    const int valid = (int)std::min<uint64_t>(4, e < n ? n - e : 0);
    float r[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    if (valid == 4 && ((reinterpret_cast<uintptr_t>(x + e) & 15u) == 0)) {
      const float4 a = ld_stream_f4(reinterpret_cast<const float4*>(x + e));
      r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w;
    } else {
      for (int i = 0; i < valid; ++i) r[i] = x[e + i];
    }
    qsgd_block_encode(r, valid, e, ctr_base + e, bits, bucket, k0, k1, codes, scales, bmax, norm);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kThreads) dequantize_kernel(const uint8_t* __restrict__ codes,
                                                              const float* __restrict__ scales, uint64_t n,
                                                              int bits, uint32_t bucket, float* __restrict__ out) {
  const uint32_t s = (1u << (bits - 1)) - 1u;
  const uint32_t mask = (1u << bits) - 1u;
  const uint64_t groups = (n + 7) / 8;
  for (uint64_t g = (uint64_t)blockIdx.x * kThreads + threadIdx.x; g < groups; g += (uint64_t)gridDim.x * kThreads) {
    const uint64_t e = g * 8;
    const int cnt = (int)std::min<uint64_t>(8, n - e);
    const uint8_t* cp = codes + (e * bits) / 8;
    uint64_t word = 0;
    if (cnt == 8 && bits == 4) word = *reinterpret_cast<const uint32_t*>(cp);
    else if (cnt == 8 && bits == 8) word = *reinterpret_cast<const unsigned long long*>(cp);
    else if (cnt == 8 && bits == 2) word = *reinterpret_cast<const uint16_t*>(cp);
    else
      for (int b = 0; b < (cnt * bits + 7) / 8; ++b) word |= (uint64_t)cp[b] << (8 * b);
    const float scale = scales[e / bucket];
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = qsgd_decode((uint32_t)(word >> (i * bits)) & mask, scale, s, bits);
    float* d = out + e;
    if (cnt == 8 && ((reinterpret_cast<uintptr_t>(d) & 15u) == 0)) {
      reinterpret_cast<float4*>(d)[0] = make_float4(v[0], v[1], v[2], v[3]);
      reinterpret_cast<float4*>(d)[1] = make_float4(v[4], v[5], v[6], v[7]);
    } else {
      for (int i = 0; i < cnt; ++i) d[i] = v[i];
    }
  }
}

cudaError_t launch_quantize(const float* x, uint64_t n, int bits, uint32_t bucket, uint64_t seed, uint64_t ctr_base,
                            uint8_t* codes, float* scales, cudaStream_t s, int norm) {
  const uint64_t nwin = (n + kWin - 1) / kWin;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(nwin, (uint64_t)device_sm_count() * 8));
  SPARCML_PROF("quantize", s);
  quantize_kernel<<<grid, kThreads, 0, s>>>(x, n, bits, bucket, (uint32_t)seed, (uint32_t)(seed >> 32), ctr_base,
                                            codes, scales, norm);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_dequantize(const uint8_t* codes, const float* scales, uint64_t n, int bits, uint32_t bucket,
                              float* out, cudaStream_t s) {
  const uint64_t groups = (n + 7) / 8;
  const unsigned grid =
      (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((groups + kThreads - 1) / kThreads, (uint64_t)device_sm_count() * 8));
  SPARCML_PROF("dequantize", s);
  dequantize_kernel<<<grid, kThreads, 0, s>>>(codes, scales, n, bits, bucket, out);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace sparcml
