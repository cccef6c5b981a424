// microbench_sync.cu — diagnostics for the top-k kernel's synchronisation
// costs on B200 (one CTA of 512 threads per SM, cooperative launch):
//   1. grid barrier (arrival counter + release flag), with and without fences
//   2. __syncthreads after global stores / reductions vs after none
//   3. a 4096-bin block scan (find_desc's shape)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbs tools/microbench_sync.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_release(uint32_t* p, uint32_t v) {
  uint32_t r;
  asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}

struct Ctl {
  uint32_t arrive, flag;
  uint32_t pad[30];
  uint64_t t[64];
};

template <int MODE>
__device__ __forceinline__ void gbar(Ctl* c, uint32_t target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t old;
    if (MODE == 0) {   // fence + atomic + release flag + acquire + fence
      __threadfence();
      old = atomicAdd(&c->arrive, 1u);
    } else {           // release RMW, no separate fences
      old = atom_add_release(&c->arrive, 1u);
    }
    if (old == gridDim.x * target - 1) {
      st_release(&c->flag, target);
    } else {
      while ((int)(ld_relaxed(&c->flag) - target) < 0) {
      }
      (void)ld_acquire(&c->flag);
    }
    if (MODE == 0) __threadfence();
  }
  __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k_barrier(Ctl* c, int iters) {
  const uint64_t t0 = gtime();
  for (int i = 1; i <= iters; ++i) gbar<MODE>(c, i);
  if (blockIdx.x == 0 && threadIdx.x == 0) c->t[MODE] = gtime() - t0;
}

// __syncthreads cost after each thread issued `nst` global stores (STG) or reductions (RED)
template <int KIND>
__global__ void __launch_bounds__(512, 1) k_sync(Ctl* c, uint32_t* buf, int iters, int nst) {
  uint64_t tot = 0;
  for (int i = 0; i < iters; ++i) {
    for (int j = 0; j < nst; ++j) {
      uint32_t* p = buf + ((size_t)blockIdx.x * 512 * 16 + (size_t)j * 512 + threadIdx.x);
      if (KIND == 1) *p = i;
      if (KIND == 2) atomicAdd(p, 1u);
    }
    const uint64_t t0 = gtime();
    __syncthreads();
    tot += gtime() - t0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) c->t[8 + KIND * 4 + (nst > 1)] = tot / iters;
}

// 4096-bin descending scan (find_desc shape) x iters
__global__ void __launch_bounds__(512, 1) k_scan(Ctl* c, int iters) {
  __shared__ uint32_t h[4096];
  __shared__ uint64_t sc[17];
  for (int i = threadIdx.x; i < 4096; i += 512) h[i] = i & 7;
  __syncthreads();
  const uint64_t t0 = gtime();
  uint64_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int base = 4096 - 8 * (tid + 1);
    const uint4 lo4 = *reinterpret_cast<const uint4*>(h + base);
    const uint4 hi4 = *reinterpret_cast<const uint4*>(h + base + 4);
    uint64_t x = (uint64_t)lo4.x + lo4.y + lo4.z + lo4.w + hi4.x + hi4.y + hi4.z + hi4.w;
    uint64_t inc = x;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) sc[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      uint64_t w = lane < 16 ? sc[lane] : 0, wi = w;
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      if (lane < 16) sc[lane] = wi - w;
    }
    __syncthreads();
    acc += sc[warp] + inc - x;
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) c->t[20] = (gtime() - t0) / iters + (acc == 12345 ? 1 : 0);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  Ctl* c;
  uint32_t* buf;
  cudaMalloc(&c, sizeof(Ctl));
  cudaMalloc(&buf, (size_t)sms * 512 * 16 * 4);
  const int iters = 200;
  Ctl h;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(c, 0, sizeof(Ctl));
    void* a0[] = {&c, (void*)&iters};
    cudaLaunchCooperativeKernel((void*)k_barrier<0>, sms, 512, a0, 0, 0);
    cudaDeviceSynchronize();
    cudaMemset(c, 0, 8);
    cudaLaunchCooperativeKernel((void*)k_barrier<1>, sms, 512, a0, 0, 0);
    cudaDeviceSynchronize();
    for (int nst : {0, 1, 8}) {
      void* a1[] = {&c, &buf, (void*)&iters, &nst};
      cudaLaunchCooperativeKernel((void*)k_sync<1>, sms, 512, a1, 0, 0);
      cudaLaunchCooperativeKernel((void*)k_sync<2>, sms, 512, a1, 0, 0);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, c, sizeof(Ctl), cudaMemcpyDeviceToHost);
      if (rep) printf("syncthreads after %d STG/thread: %.0f ns; after %d RED/thread: %.0f ns\n", nst,
                      (double)h.t[8 + 4 + (nst > 1)], nst, (double)h.t[8 + 8 + (nst > 1)]);
    }
    void* a2[] = {&c, (void*)&iters};
    cudaLaunchCooperativeKernel((void*)k_scan, sms, 512, a2, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, sizeof(Ctl), cudaMemcpyDeviceToHost);
    if (rep) {
      printf("grid barrier (fence+atomic+flag): %.0f ns\n", (double)h.t[0] / iters);
      printf("grid barrier (release RMW + flag): %.0f ns\n", (double)h.t[1] / iters);
      printf("4096-bin block scan: %.0f ns\n", (double)h.t[20]);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
