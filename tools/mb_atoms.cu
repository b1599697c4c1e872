// Shared-atomic XOR throughput vs active lanes (is the ATOMS cost per
// instruction or per lane?) and vs bank conflicts. JSON lines out.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/mb_atoms.cu -o build/mb_atoms
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

// kActive lanes of each warp issue the XOR (the rest branch around it);
// kRand: random word addresses, else lane-owned banks.
template <int kActive, bool kRand>
__global__ void k_atoms(uint32_t* out, uint32_t seed) {
  __shared__ uint32_t buf[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  uint32_t x = seed * 2654435761u + threadIdx.x * 40503u;
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
#pragma unroll 4
  for (int i = 0; i < kIters; ++i) {
    x = x * 1664525u + 1013904223u;
    const uint32_t addr = kRand ? ((x >> 19) & 8191) : ((((x >> 20) & 255) << 5) | lane);
    if (lane < kActive)
      asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(s + addr * 4), "r"(x) : "memory");
  }
  __syncthreads();
  if (buf[threadIdx.x] == 0x12345678u) out[0] = 1;
}

// Same loop, no atomics (the ALU cost of the loop itself).
__global__ void k_none(uint32_t* out, uint32_t seed) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t x = seed * 2654435761u + threadIdx.x * 40503u, acc = 0;
#pragma unroll 4
  for (int i = 0; i < kIters; ++i) {
    x = x * 1664525u + 1013904223u;
    acc ^= ((((x >> 20) & 255) << 5) | lane);
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
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 4, threads = 512;
  const double warps = double(blocks) * threads / 32;
  auto report = [&](const char* name, int active, double ms) {
    const double inst = warps * kIters;
    const double sm_clk = (ms * 1e-3) * sms * (clk * 1e3);
    printf("{\"bench\": \"%s\", \"active\": %d, \"ms\": %.4f, \"warp_inst_per_sm_clk\": %.4f, "
           "\"lane_ops_per_sm_clk\": %.3f}\n",
           name, active, ms, inst / sm_clk, inst * active / sm_clk);
  };
  report("none", 0, time_ms([&] { k_none<<<blocks, threads>>>(out, 1); }));
  report("atoms_cf", 32, time_ms([&] { k_atoms<32, false><<<blocks, threads>>>(out, 1); }));
  report("atoms_cf", 16, time_ms([&] { k_atoms<16, false><<<blocks, threads>>>(out, 1); }));
  report("atoms_cf", 8, time_ms([&] { k_atoms<8, false><<<blocks, threads>>>(out, 1); }));
  report("atoms_cf", 4, time_ms([&] { k_atoms<4, false><<<blocks, threads>>>(out, 1); }));
  report("atoms_cf", 1, time_ms([&] { k_atoms<1, false><<<blocks, threads>>>(out, 1); }));
  report("atoms_rand", 32, time_ms([&] { k_atoms<32, true><<<blocks, threads>>>(out, 1); }));
  report("atoms_rand", 16, time_ms([&] { k_atoms<16, true><<<blocks, threads>>>(out, 1); }));
  report("atoms_rand", 8, time_ms([&] { k_atoms<8, true><<<blocks, threads>>>(out, 1); }));
  return 0;
}
