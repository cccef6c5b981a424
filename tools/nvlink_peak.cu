// nvlink_peak.cu — measured NVLink 5 peer bandwidth on this box, the
// denominator of the exchange roofline ("measure on the box").
//
// For every ordered GPU pair (i, j), i != j, with peer access enabled:
//   pull:  a kernel on GPU i reads GPU j's buffer with 16-byte loads (what the
//          library's concat / owner kernels do) and writes it locally;
//   push:  a kernel on GPU i writes GPU j's buffer with 16-byte stores (the
//          split push);
//   ce:    cudaMemcpyPeerAsync (copy engines);
//   bidir: GPU i and GPU j pull from each other at the same time (sum of both).
// Sizes 256 MiB and 1 GiB; CUDA events, best of 5.  Prints one JSON object.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_peak tools/nvlink_peak.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

__global__ void copy16(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u * stride < n) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u * stride < n) dst[i + u * stride] = v[u];
  }
}

static float time_kernel(int dev, const void* src, void* dst, size_t bytes, int sms) {
  CK(cudaSetDevice(dev));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    CK(cudaEventRecord(a));
    copy16<<<sms * 4, 512>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst), bytes / 16);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (rep > 0 && ms < best) best = ms;
  }
  CK(cudaEventDestroy(a));
  CK(cudaEventDestroy(b));
  return best;
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("{\"error\": \"needs >= 2 GPUs\", \"gpus\": %d}\n", n);
    return 0;
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t sizes[2] = {256ull << 20, 1024ull << 20};
  std::vector<void*> buf(n), loc(n);
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaMalloc(&buf[d], sizes[1]));
    CK(cudaMalloc(&loc[d], sizes[1]));
    CK(cudaMemset(buf[d], d + 1, sizes[1]));
    for (int e = 0; e < n; ++e)
      if (e != d) {
        int can = 0;
        CK(cudaDeviceCanAccessPeer(&can, d, e));
        if (can) {
          cudaError_t r = cudaDeviceEnablePeerAccess(e, 0);
          if (r != cudaSuccess && r != cudaErrorPeerAccessAlreadyEnabled) CK(r);
          cudaGetLastError();
        }
      }
  }
  printf("{\"gpus\": %d, \"sms\": %d, \"pairs\": [", n, sms);
  double best_pull = 0, best_push = 0, best_ce = 0, best_bi = 0;
  bool first = true;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      if (i == j) continue;
      if (!(i == 0 || j == 0)) continue;   // pairs with GPU 0 (NVSwitch: every pair is one hop)
      for (size_t bytes : sizes) {
        const float pull = time_kernel(i, buf[j], loc[i], bytes, sms);   // i reads j
        const float push = time_kernel(i, loc[i], buf[j], bytes, sms);   // i writes j
        // copy engine
        CK(cudaSetDevice(i));
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        float ce = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
          CK(cudaEventRecord(a));
          CK(cudaMemcpyPeerAsync(loc[i], i, buf[j], j, bytes));
          CK(cudaEventRecord(b));
          CK(cudaEventSynchronize(b));
          float ms;
          CK(cudaEventElapsedTime(&ms, a, b));
          if (rep > 0 && ms < ce) ce = ms;
        }
        // bidirectional: i pulls from j while j pulls from i (two streams, one per device)
        float bi = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
          CK(cudaSetDevice(i));
          CK(cudaDeviceSynchronize());
          CK(cudaSetDevice(j));
          CK(cudaDeviceSynchronize());
          CK(cudaSetDevice(i));
          CK(cudaEventRecord(a));
          copy16<<<sms * 4, 512>>>(static_cast<const uint4*>(buf[j]), static_cast<uint4*>(loc[i]), bytes / 16);
          CK(cudaSetDevice(j));
          copy16<<<sms * 4, 512>>>(static_cast<const uint4*>(buf[i]), static_cast<uint4*>(loc[j]), bytes / 16);
          CK(cudaDeviceSynchronize());
          CK(cudaSetDevice(i));
          CK(cudaEventRecord(b));
          CK(cudaEventSynchronize(b));
          float ms;
          CK(cudaEventElapsedTime(&ms, a, b));
          if (rep > 0 && ms < bi) bi = ms;
        }
        CK(cudaEventDestroy(a));
        CK(cudaEventDestroy(b));
        const double gb = (double)bytes / 1e9;
        const double gpull = gb / (pull * 1e-3), gpush = gb / (push * 1e-3), gce = gb / (ce * 1e-3),
                     gbi = 2 * gb / (bi * 1e-3);
        if (gpull > best_pull) best_pull = gpull;
        if (gpush > best_push) best_push = gpush;
        if (gce > best_ce) best_ce = gce;
        if (gbi > best_bi) best_bi = gbi;
        printf("%s{\"src\": %d, \"dst\": %d, \"bytes\": %zu, \"pull_gbs\": %.1f, \"push_gbs\": %.1f, \"ce_gbs\": %.1f, "
               "\"bidir_sum_gbs\": %.1f}",
               first ? "" : ", ", j, i, bytes, gpull, gpush, gce, gbi);
        first = false;
      }
    }
  printf("], \"best_pull_gbs\": %.1f, \"best_push_gbs\": %.1f, \"best_ce_gbs\": %.1f, \"best_bidir_sum_gbs\": %.1f, "
         "\"nominal_per_direction_gbs\": 900}\n",
         best_pull, best_push, best_ce, best_bi);
  return 0;
}
