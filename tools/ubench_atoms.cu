// Microbenchmark: shared-memory scatter-add throughput on B200 (design
// probe for a symmetric-storage hop).  One CTA per SM, 1024
// threads, each thread adds into a random slot of a shared table.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_atoms tools/ubench_atoms.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kSlots = 8192 * 4;    // 32-bit tables: F = 4 x 8192 columns (128 KB)
constexpr int kSlots64 = 8192 * 2;  // 64-bit tables: F = 2 x 8192 columns (128 KB)

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_scatter(int iters, float v, unsigned long long* out) {
  extern __shared__ unsigned char smem[];
  unsigned x = 2463534242u ^ (threadIdx.x * 747796405u + blockIdx.x * 2891336453u);
  constexpr int slots = (MODE == 0 || MODE == 3) ? kSlots64 : kSlots;
  if (MODE == 0 || MODE == 3) {
    unsigned long long* t = reinterpret_cast<unsigned long long*>(smem);
    for (int i = threadIdx.x; i < slots; i += blockDim.x) t[i] = 0;
  } else {
    unsigned* t = reinterpret_cast<unsigned*>(smem);
    for (int i = threadIdx.x; i < slots; i += blockDim.x) t[i] = 0;
  }
  __syncthreads();
  float acc = v;
  for (int it = 0; it < iters; ++it) {
    x ^= x << 13; x ^= x >> 17; x ^= x << 5;
    const int slot = x & (slots - 1);
    acc = acc * 1.0000001f + 0.5f;
    if (MODE == 0) {  // int64 fixed point: float -> int64 conversion + 64-bit shared atomic
      atomicAdd(reinterpret_cast<unsigned long long*>(smem) + slot, (unsigned long long)__float2ll_rn(acc * 4096.f));
    } else if (MODE == 1) {  // fp32 shared atomic (non-deterministic order)
      atomicAdd(reinterpret_cast<float*>(smem) + slot, acc);
    } else if (MODE == 2) {  // int32 shared atomic, magic-number conversion (FADD + IADD)
      const float f = acc + 12582912.0f;
      atomicAdd(reinterpret_cast<unsigned*>(smem) + slot, (unsigned)(__float_as_int(f) - 0x4B400000));
    } else {  // int64 shared atomic, magic-number conversion
      const float f = acc + 12582912.0f;
      atomicAdd(reinterpret_cast<unsigned long long*>(smem) + slot,
                (unsigned long long)(long long)(__float_as_int(f) - 0x4B400000));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = reinterpret_cast<unsigned long long*>(smem)[5];
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* out;
  cudaMalloc(&out, sms * sizeof(unsigned long long));
  const int iters = 4096;
  const char* names[4] = {"int64 atomics + F2I.S64", "fp32 atomics", "int32 atomics + magic", "int64 atomics + magic"};
  for (int mode = 0; mode < 4; ++mode) {
    const size_t smem = (mode == 0 || mode == 3) ? kSlots64 * 8 : kSlots * 4;
    void (*k)(int, float, unsigned long long*) =
        mode == 0 ? k_scatter<0> : mode == 1 ? k_scatter<1> : mode == 2 ? k_scatter<2> : k_scatter<3>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<sms, 1024, smem>>>(iters, 1.f, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<<<sms, 1024, smem>>>(iters, 1.f, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = 5.0 * sms * 1024.0 * iters;
    printf("%-26s %8.3f ms  %7.2f Gatomic/s  %6.2f lane-atomics/clk/SM @1.9GHz  (%s)\n", names[mode], ms,
           ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.9e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
