// Primitive-rate microbenchmarks on the B200 (one binary, JSON lines out):
//   lop3     : dependent-free LOP3 throughput (INT/bitwise roofline R_int)
//   atoms    : shared-memory atomicXor, random addresses
//   atoms_cf : shared-memory atomicXor, bank-conflict-free addresses
//   rmw_cf   : plain LDS + XOR + STS, bank-conflict-free (lane-owned words)
//   rmw_rand : plain LDS + XOR + STS, random addresses
//   philox   : Philox4x32-10 blocks per second
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/microbench.cu -o build/microbench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void k_lop3(uint32_t* out, uint32_t seed) {
  uint32_t a = seed ^ threadIdx.x, b = a * 3, c = a * 5, d = a * 7, e = a * 11, f = a * 13, g = a * 17, h = a * 19;
#pragma unroll 16
  for (int i = 0; i < kIters; ++i) {
    a = a ^ b ^ c; b = b ^ c ^ d; c = c ^ d ^ e; d = d ^ e ^ f;
    e = e ^ f ^ g; f = f ^ g ^ h; g = g ^ h ^ a; h = h ^ a ^ b;
  }
  if ((a ^ b ^ c ^ d ^ e ^ f ^ g ^ h) == 0x12345678u) out[0] = 1;
}

template <int kMode>
__global__ void k_smem(uint32_t* out, uint32_t seed) {
  __shared__ uint32_t buf[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  uint32_t x = seed * 2654435761u + threadIdx.x * 40503u;
  for (int i = 0; i < kIters; ++i) {
    x = x * 1664525u + 1013904223u;
    uint32_t addr;
    if (kMode == 0 || kMode == 3) addr = (x >> 19) & 8191;           // random
    else addr = (((x >> 20) & 255) << 5) | lane;                    // lane-owned bank
    if (kMode <= 1) atomicXor(&buf[addr], x);
    else buf[addr] ^= x;
  }
  __syncthreads();
  if (buf[threadIdx.x] == 0x12345678u) out[0] = 1;
}

__device__ __forceinline__ uint4 philox10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

__global__ void k_philox(uint32_t* out, uint32_t seed) {
  uint32_t acc = 0;
  for (int i = 0; i < kIters / 8; ++i) {
    uint4 r = philox10(make_uint4(threadIdx.x, i, blockIdx.x, 0), seed, 77);
    acc ^= r.x ^ r.y ^ r.z ^ r.w;
  }
  if (acc == 0x12345678u) out[0] = 1;
}

template <class F>
double time_ms(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  uint32_t* out;
  cudaMalloc(&out, 16);
  const int blocks = sms * 4, threads = 512;
  const double n_threads = double(blocks) * threads;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double ms = time_ms([&] { k_lop3<<<blocks, threads>>>(out, 1); });
  double ops = n_threads * kIters * 8;  // 8 LOP3 per iteration (3-input XOR each)
  printf("{\"bench\": \"lop3\", \"ms\": %.4f, \"ops_per_s\": %.4e, \"per_sm_per_clk\": %.2f}\n", ms,
         ops / ms * 1e3, ops / (ms * 1e-3) / sms / (clk * 1e3));
  const char* names[4] = {"atoms_rand", "atoms_cf", "rmw_cf", "rmw_rand"};
  for (int m = 0; m < 4; ++m) {
    auto run = [&] {
      if (m == 0) k_smem<0><<<blocks, threads>>>(out, 3);
      if (m == 1) k_smem<1><<<blocks, threads>>>(out, 3);
      if (m == 2) k_smem<2><<<blocks, threads>>>(out, 3);
      if (m == 3) k_smem<3><<<blocks, threads>>>(out, 3);
    };
    ms = time_ms(run);
    double n = n_threads * kIters;
    printf("{\"bench\": \"%s\", \"ms\": %.4f, \"lane_ops_per_s\": %.4e, \"lane_ops_per_sm_per_clk\": %.3f}\n",
           names[m], ms, n / ms * 1e3, n / (ms * 1e-3) / sms / (clk * 1e3));
  }
  ms = time_ms([&] { k_philox<<<blocks, threads>>>(out, 5); });
  double calls = n_threads * (kIters / 8);
  printf("{\"bench\": \"philox4x32_10\", \"ms\": %.4f, \"blocks_per_s\": %.4e, \"per_sm_per_clk\": %.3f}\n",
         ms, calls / ms * 1e3, calls / (ms * 1e-3) / sms / (clk * 1e3));
  printf("{\"bench\": \"device\", \"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  return 0;
}
