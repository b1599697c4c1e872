// Device phase store for the host symbolic pass (frontend.cpp).
//
// The one-pass symbolic tableau (tableau.cpp:17-198) keeps, per stabilizer
// row, a phase bit-vector over all symbols. For large circuits (the paper's
// Fig. 3 dense families at n = 1,000: 1,000 rows x 2*10^6 symbols) almost all
// of the pass is the row XORs of those vectors at measurements: a random
// outcome XORs the pivot's phase into every anticommuting stabilizer, a
// determined one XORs the selected stabilizers' phases into the outcome.
// Here the phase matrix lives in HBM and those two operations are kernels
// (the north star's "row-XOR of phase bit-vector columns ... in a simple
// kernel"); the Clifford x/z part and all bookkeeping stay on the host.
// Single-bit phase flips (noise symbols, constant terms) are queued on the
// host and applied in one launch before the next row operation, so every
// operation sees them in program order. Everything is XOR: bit-exact.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "frontend_dev.hpp"

namespace symphase {
namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

__global__ void k_flips(uint64_t* ph, uint64_t ws, const uint64_t* flips, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint64_t f = flips[i];
    const uint64_t row = f >> 32, sym = f & 0xFFFFFFFFull;
    atomicXor(reinterpret_cast<unsigned long long*>(ph + row * ws + sym / 64),
              1ull << (sym & 63));
  }
}

// Row lists of up to kParamRows rows travel in the kernel parameters (no
// host->device copy per operation; CUDA 12.1+ takes 32 KB of parameters).
constexpr uint32_t kParamRows = 2048;
struct RowList {
  uint32_t r[kParamRows];
};

// ph[t] ^= ph[src] over words [0, words) for every target t (blockIdx.y).
__device__ __forceinline__ void xor_row(uint64_t* ph, uint64_t ws, uint32_t src, uint32_t dst,
                                        uint32_t words) {
  const uint64_t* s = ph + static_cast<uint64_t>(src) * ws;
  uint64_t* d = ph + static_cast<uint64_t>(dst) * ws;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x)
    d[w] ^= s[w];
}
__global__ void k_xor_rows(uint64_t* ph, uint64_t ws, uint32_t src, const uint32_t* targets,
                           uint32_t words) {
  xor_row(ph, ws, src, targets[blockIdx.y], words);
}
__global__ void k_xor_rows_p(uint64_t* ph, uint64_t ws, uint32_t src, const __grid_constant__ RowList t,
                             uint32_t words) {
  xor_row(ph, ws, src, t.r[blockIdx.y], words);
}

// out[w] = XOR over the listed rows of ph[row][w], words [0, words).
__global__ void k_reduce_rows_p(const uint64_t* ph, uint64_t ws, const __grid_constant__ RowList rows,
                                uint32_t n_rows, uint32_t words, uint64_t* out) {
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
    uint64_t a = 0;
    for (uint32_t r = 0; r < n_rows; ++r) a ^= ph[static_cast<uint64_t>(rows.r[r]) * ws + w];
    out[w] = a;
  }
}

// out[w] = XOR over rows of ph[row][w], words [0, words).
__global__ void k_reduce_rows(const uint64_t* ph, uint64_t ws, const uint32_t* rows, uint32_t n_rows,
                              uint32_t words, uint64_t* out) {
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
    uint64_t a = 0;
    for (uint32_t r = 0; r < n_rows; ++r) a ^= ph[static_cast<uint64_t>(rows[r]) * ws + w];
    out[w] = a;
  }
}

}  // namespace

struct PhaseDev {
  uint64_t ws = 0;
  size_t n_rows = 0;
  uint64_t* ph = nullptr;
  uint64_t* d_flips = nullptr;
  size_t flips_cap = 0;
  uint32_t* d_rows = nullptr;
  size_t rows_cap = 0;
  uint64_t* d_out = nullptr;
  uint64_t* h_out = nullptr;  // pinned
  cudaStream_t stream = nullptr;
};

bool phase_dev_available() {
  int n = 0;
  return cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
}

PhaseDev* phase_dev_create(size_t n_rows, uint64_t ws) {
  auto* p = new PhaseDev;
  p->ws = ws;
  p->n_rows = n_rows;
  try {
    ck(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaMalloc(&p->ph, n_rows * ws * 8), "cudaMalloc (phase matrix)");
    ck(cudaMemsetAsync(p->ph, 0, n_rows * ws * 8, p->stream), "cudaMemset");
    ck(cudaMalloc(&p->d_out, ws * 8), "cudaMalloc");
    ck(cudaMallocHost(&p->h_out, ws * 8), "cudaMallocHost");
  } catch (...) {
    phase_dev_destroy(p);
    throw;
  }
  return p;
}

void phase_dev_destroy(PhaseDev* p) {
  if (!p) return;
  if (p->stream) cudaStreamSynchronize(p->stream);
  cudaFree(p->ph);
  cudaFree(p->d_flips);
  cudaFree(p->d_rows);
  cudaFree(p->d_out);
  cudaFreeHost(p->h_out);
  if (p->stream) cudaStreamDestroy(p->stream);
  delete p;
}

namespace {
template <class T>
void stage(PhaseDev* p, T*& buf, size_t& cap, const T* host, size_t n) {
  if (n > cap) {
    ck(cudaStreamSynchronize(p->stream), "sync");
    cudaFree(buf);
    cap = std::max<size_t>(n, 2 * cap);
    ck(cudaMalloc(&buf, cap * sizeof(T)), "cudaMalloc");
  }
  // pageable source: the copy is staged before cudaMemcpyAsync returns
  ck(cudaMemcpyAsync(buf, host, n * sizeof(T), cudaMemcpyHostToDevice, p->stream), "H2D");
}
}  // namespace

void phase_dev_flips(PhaseDev* p, const uint64_t* flips, size_t n) {
  if (n == 0) return;
  stage(p, p->d_flips, p->flips_cap, flips, n);
  const int grid = static_cast<int>(std::min<size_t>((n + 255) / 256, 1024));
  k_flips<<<grid, 256, 0, p->stream>>>(p->ph, p->ws, p->d_flips, n);
  ck(cudaGetLastError(), "flips launch");
}

void phase_dev_xor_rows(PhaseDev* p, uint32_t src, const uint32_t* targets, size_t n_t,
                        uint32_t words) {
  if (n_t == 0 || words == 0) return;
  const unsigned gx = std::max(1u, std::min(64u, (words + 255) / 256));
  if (n_t <= kParamRows) {
    RowList t;
    std::copy(targets, targets + n_t, t.r);
    k_xor_rows_p<<<dim3(gx, static_cast<unsigned>(n_t)), 256, 0, p->stream>>>(p->ph, p->ws, src, t, words);
    ck(cudaGetLastError(), "xor launch");
    return;
  }
  stage(p, p->d_rows, p->rows_cap, targets, n_t);
  for (size_t t0 = 0; t0 < n_t; t0 += 65535) {
    const unsigned gy = static_cast<unsigned>(std::min<size_t>(65535, n_t - t0));
    k_xor_rows<<<dim3(gx, gy), 256, 0, p->stream>>>(p->ph, p->ws, src, p->d_rows + t0, words);
  }
  ck(cudaGetLastError(), "xor launch");
}

void phase_dev_upload(PhaseDev* p, const uint64_t* host) {
  ck(cudaMemcpyAsync(p->ph, host, p->n_rows * p->ws * 8, cudaMemcpyHostToDevice, p->stream), "H2D");
  ck(cudaStreamSynchronize(p->stream), "sync");
}

void phase_dev_clear_row(PhaseDev* p, uint32_t row, uint32_t words) {
  if (words == 0) return;
  ck(cudaMemsetAsync(p->ph + static_cast<uint64_t>(row) * p->ws, 0, words * 8ull, p->stream),
     "cudaMemset");
}

const uint64_t* phase_dev_reduce(PhaseDev* p, const uint32_t* rows, size_t n_r, uint32_t words) {
  if (words == 0) return p->h_out;
  if (n_r == 0) {
    std::fill(p->h_out, p->h_out + words, 0ull);
    return p->h_out;
  }
  const int grid = static_cast<int>(std::min<uint32_t>((words + 255) / 256, 1024));
  if (n_r <= kParamRows) {
    RowList t;
    std::copy(rows, rows + n_r, t.r);
    k_reduce_rows_p<<<grid, 256, 0, p->stream>>>(p->ph, p->ws, t, static_cast<uint32_t>(n_r), words,
                                                 p->d_out);
  } else {
    stage(p, p->d_rows, p->rows_cap, rows, n_r);
    k_reduce_rows<<<grid, 256, 0, p->stream>>>(p->ph, p->ws, p->d_rows, static_cast<uint32_t>(n_r),
                                               words, p->d_out);
  }
  ck(cudaGetLastError(), "reduce launch");
  ck(cudaMemcpyAsync(p->h_out, p->d_out, words * 8ull, cudaMemcpyDeviceToHost, p->stream), "D2H");
  ck(cudaStreamSynchronize(p->stream), "sync");
  return p->h_out;
}

}  // namespace symphase
