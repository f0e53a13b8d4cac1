// peaks.cu -- libdts_peaks.so: pipe-throughput microbenchmarks for the
// "% of FP32/SFU issue roofline" denominators (SURVEY.md 8(d.2), step 0 of the
// build plan).  MEASURED_PEAKS.json carries HBM and bf16 tensor peaks only; the
// DARTS path is bound by plain ALU issue, so its denominators are measured here:
// FFMA (register and immediate forms), the MUFU ops the path uses (EX2, LG2,
// RSQRT, RCP, SIN), integer IMAD.WIDE / LOP3, an FFMA+LOP3 dual-pipe mix (the
// issue ceiling), and global RED.F32 / shared-memory atomic throughput.
//
// Every kernel runs a fixed number of independent dependency chains per thread
// written in inline PTX (so nothing is folded), on a persistent grid of
// blocks_per_sm x #SM CTAs; each CTA records its clock64() span so the rate is
// reported per SM clock (clock-independent) as well as per second.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

namespace {

constexpr int kChains = 8;

template <int OP>
__device__ __forceinline__ void step(float (&a)[kChains], uint32_t (&u)[kChains], float b, float c) {
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
    if (OP == 1) asm volatile("fma.rn.f32 %0, %0, 0f3F800347, 0f3EFFF000;" : "+f"(a[i]));
    if (OP == 2) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
    if (OP == 3) asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
    if (OP == 4) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
    if (OP == 5) asm volatile("rcp.approx.ftz.f32 %0, %0;\n\tadd.ftz.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(c));  // + FADD: ptxas folds rcp(rcp(x))
    if (OP == 6) asm volatile("sin.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
    if (OP == 7) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[i]) : "r"(__float_as_uint(b)), "r"(__float_as_uint(c)));
    if (OP == 8) {
      uint64_t v;
      asm volatile("mul.wide.u32 %0, %1, 0xD2511F53;" : "=l"(v) : "r"(u[i]));
      u[i] = (uint32_t)(v >> 32) ^ (uint32_t)v;
    }
    if (OP == 9) {  // dual-pipe: one FFMA (fma pipe) + one LOP3 (alu pipe) per chain
      asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[i]) : "r"(__float_as_uint(b)), "r"(__float_as_uint(c)));
    }
  }
}

template <int OP>
__global__ void pipe_kernel(int iters, float b, float c, float* sink, long long* cycles) {
  float a[kChains];
  uint32_t u[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    a[i] = 0.5f + 1e-3f * (threadIdx.x + i);
    u[i] = threadIdx.x * 2654435761u + i;
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) step<OP>(a, u, b, c);
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += a[i] + (float)(u[i] & 1u);
  if (s == 12345.678f) sink[threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// global fp32 RED throughput: each thread issues `iters` REDs to addresses
// spread over n_cells (random-ish, like per-path splats) or to a hot window.
__global__ void red_kernel(float* hist, uint32_t n_cells, uint32_t hot_mask, int iters, long long* cycles) {
  uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    const uint32_t cell = hot_mask ? (x >> 8) & hot_mask : (uint32_t)(((uint64_t)x * n_cells) >> 32);
    atomicAdd(hist + cell, 1.0f);
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// shared-memory fp32 atomics into a 4096-cell private tile, flushed once
__global__ void smem_atomic_kernel(float* out, int iters, long long* cycles) {
  __shared__ float tile[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) tile[i] = 0.0f;
  uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 777u;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    atomicAdd(tile + (x >> 20), 1.0f);
  }
  __syncthreads();
  const long long t1 = clock64();
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) atomicAdd(out + i, tile[i]);
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

}  // namespace

extern "C" {

// Result of one microbenchmark: thread-level operations executed, kernel
// time (CUDA events), and the mean per-CTA clock64 span.
typedef struct {
  double ops;
  double ms;
  double mean_cycles;
  int32_t grid, block;
} dts_peak_result;

// op: 0 FFMA reg, 1 FFMA imm, 2 EX2, 3 LG2, 4 RSQRT, 5 RCP, 6 SIN, 7 LOP3,
// 8 IMAD.WIDE(+LOP3), 9 FFMA+LOP3 pair, 10 global RED random (n_cells),
// 11 global RED hot (4096 cells), 12 shared-memory atomics.
// Returns 0 on success, a cudaError_t otherwise.  Synchronous.
int dts_peak_run(int op, int iters, int blocks_per_sm, int block, uint32_t n_cells, dts_peak_result* res) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = sms * blocks_per_sm;
  float* sink = nullptr;
  long long* cyc = nullptr;
  float* hist = nullptr;
  cudaError_t e;
  if ((e = cudaMalloc(&sink, 4096 * sizeof(float))) != cudaSuccess) return (int)e;
  if ((e = cudaMalloc(&cyc, grid * sizeof(long long))) != cudaSuccess) return (int)e;
  const size_t ncell = op == 10 ? n_cells : 4096;
  if (op >= 10 && (e = cudaMalloc(&hist, ncell * sizeof(float))) != cudaSuccess) return (int)e;
  if (hist) cudaMemset(hist, 0, ncell * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto launch = [&]() {
    switch (op) {
      case 0: pipe_kernel<0><<<grid, block>>>(iters, 1.0001f, 0.5f, sink, cyc); break;
      case 1: pipe_kernel<1><<<grid, block>>>(iters, 1.0001f, 0.5f, sink, cyc); break;
      case 2: pipe_kernel<2><<<grid, block>>>(iters, 1.0001f, 0.5f, sink, cyc); break;
      case 3: pipe_kernel<3><<<grid, block>>>(iters, 1.0001f, 0.5f, sink, cyc); break;
      case 4: pipe_kernel<4><<<grid, block>>>(iters, 1.0001f, 0.5f, sink, cyc); break;
      case 5: pipe_kernel<5><<<grid, block>>>(iters, 1.0001f, 0.5f, sink, cyc); break;
      case 6: pipe_kernel<6><<<grid, block>>>(iters, 1.0001f, 0.5f, sink, cyc); break;
      case 7: pipe_kernel<7><<<grid, block>>>(iters, 1.0001f, 0.5f, sink, cyc); break;
      case 8: pipe_kernel<8><<<grid, block>>>(iters, 1.0001f, 0.5f, sink, cyc); break;
      case 9: pipe_kernel<9><<<grid, block>>>(iters, 1.0001f, 0.5f, sink, cyc); break;
      case 10: red_kernel<<<grid, block>>>(hist, n_cells, 0u, iters, cyc); break;
      case 11: red_kernel<<<grid, block>>>(hist, 4096u, 4095u, iters, cyc); break;
      case 12: smem_atomic_kernel<<<grid, block>>>(hist, iters, cyc); break;
      default: break;
    }
  };
  launch();  // warm-up
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  e = cudaEventSynchronize(e1);
  if (e == cudaSuccess) e = cudaGetLastError();
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[grid];
  cudaMemcpy(h, cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  double mc = 0.0;
  for (int i = 0; i < grid; ++i) mc += (double)h[i];
  delete[] h;
  const double per_thread = op == 9 ? 2.0 * kChains : (op == 8 ? 2.0 * kChains : (op >= 10 ? 1.0 : (double)kChains));
  res->ops = (double)grid * block * (double)iters * per_thread;
  res->ms = ms;
  res->mean_cycles = mc / grid;
  res->grid = grid;
  res->block = block;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  cudaFree(cyc);
  cudaFree(hist);
  return (int)e;
}

}  // extern "C"
