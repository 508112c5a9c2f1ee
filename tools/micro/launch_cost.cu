// Launch-cost probe (one B200): device time of ONE launch of an almost empty
// kernel, 148 CTAs x 32 threads, as a function of the kernel-parameter size
// and the dynamic shared memory per CTA. The stream is held by a spin kernel
// while the host enqueues, so the numbers are device-side (event to event).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_cost launch_cost.cu && ./launch_cost
#include <cuda_runtime.h>
#include <stdio.h>
#include <algorithm>
#include <vector>

template <int N>
struct Blob { int v[N]; };

template <int N>
__global__ void k_param(const __grid_constant__ Blob<N> b, int* out) {
  extern __shared__ int sm[];
  if (threadIdx.x == 0 && b.v[blockIdx.x % N] == 12345) out[0] = sm[0];
}

__global__ void spin(long long ns) {
  long long t0 = clock64();
  while (clock64() - t0 < ns) {}
}

#include <chrono>
// host time of the launch call itself (median of 2000, stream kept busy)
template <int N>
float host_one(cudaStream_t st, int* out) {
  Blob<N> b{};
  std::vector<float> ts;
  for (int r = 0; r < 2000; ++r) {
    if (r % 100 == 0) {
      cudaStreamSynchronize(st);
      spin<<<1, 1, 0, st>>>(2000000);
    }
    auto t0 = std::chrono::steady_clock::now();
    k_param<N><<<148, 32, 0, st>>>(b, out);
    auto t1 = std::chrono::steady_clock::now();
    ts.push_back(std::chrono::duration<float, std::micro>(t1 - t0).count());
  }
  cudaStreamSynchronize(st);
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

template <int N>
float time_one(int smem, cudaStream_t st, int* out) {
  Blob<N> b{};
  cudaFuncSetAttribute(k_param<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> ts;
  for (int r = 0; r < 205; ++r) {
    spin<<<1, 1, 0, st>>>(400000);
    cudaEventRecord(e0, st);
    k_param<N><<<148, 32, smem, st>>>(b, out);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 5) ts.push_back(ms * 1e3f);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  int* out;
  cudaMalloc(&out, 4);
  const int smems[] = {0, 98304, 196608};
  for (int s : smems) {
    printf("{\"smem\": %d, \"param_64B_us\": %.2f, \"param_1KB_us\": %.2f, \"param_4KB_us\": %.2f, "
           "\"param_6KB_us\": %.2f, \"param_16KB_us\": %.2f}\n",
           s, time_one<16>(s, st, out), time_one<256>(s, st, out), time_one<1000>(s, st, out),
           time_one<1536>(s, st, out), time_one<4000>(s, st, out));
  }
  printf("{\"host_launch_us\": {\"64B\": %.2f, \"1KB\": %.2f, \"4KB\": %.2f, \"6KB\": %.2f, "
         "\"16KB\": %.2f}}\n",
         host_one<16>(st, out), host_one<256>(st, out), host_one<1000>(st, out),
         host_one<1536>(st, out), host_one<4000>(st, out));
  return 0;
}
