// Microbenchmark (tooling, not product): random 4-byte reads from a 32 MB
// table (2^23 floats: the size of a full normal_icdf table over the
// sampler's 2^23 uniforms) at full occupancy, to decide whether a table
// lookup can replace the in-register Acklam rational on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbt tools/microbench_table.cu && /tmp/mbt
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  return x;
}

template <int MODE, int ILP>
__global__ void __launch_bounds__(256) probe(const float* __restrict__ tab, cudaTextureObject_t tex, int iters,
                                             float* out) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0.f;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int j = 0; j < ILP; ++j) {
      s = mix(s + 0x9E3779B9u * (j + 1));
      const uint32_t idx = s >> 9;
      float v;
      if (MODE == 0) v = __ldg(tab + idx);
      else if (MODE == 1) v = tex1Dfetch<float>(tex, (int)idx);
      else v = __ldg(tab + (idx & 0xFFF));  // 16 KB footprint: L1-resident reference
      acc += v;
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

template <int MODE, int ILP>
void run(const char* name, const float* tab, cudaTextureObject_t tex, float* out, int blocks_per_sm) {
  const int blocks = 148 * blocks_per_sm, threads = 256, iters = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  probe<MODE, ILP><<<blocks, threads>>>(tab, tex, 4, out);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    probe<MODE, ILP><<<blocks, threads>>>(tab, tex, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double loads = (double)blocks * threads * iters * ILP;
  printf("%-28s blocks/SM %d ILP %d: %.3f ms  %.1f G loads/s  (%.1f TB/s of 32B sectors)\n", name, blocks_per_sm, ILP,
         best, loads / (best * 1e-3) / 1e9, loads * 32 / (best * 1e-3) / 1e12);
}

int main() {
  const size_t n = 1u << 23;
  float* tab;
  float* out;
  cudaMalloc(&tab, n * sizeof(float));
  cudaMemset(tab, 0, n * sizeof(float));
  cudaMalloc(&out, 4);
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = tab;
  rd.res.linear.desc = cudaCreateChannelDesc<float>();
  rd.res.linear.sizeInBytes = n * sizeof(float);
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex;
  cudaCreateTextureObject(&tex, &rd, &td, nullptr);
  for (int bps : {4, 8}) {
    run<0, 1>("ldg 32MB", tab, tex, out, bps);
    run<0, 4>("ldg 32MB", tab, tex, out, bps);
    run<1, 1>("tex 32MB", tab, tex, out, bps);
    run<1, 4>("tex 32MB", tab, tex, out, bps);
    run<2, 4>("ldg 16KB (L1)", tab, tex, out, bps);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
