// Microbenchmark of the device scans (ow_scan.cuh) on synthetic flag arrays
// (GPU box helper):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//     -I paper_2502_16310_b200/csrc tools/scan_bench.cu -L paper_2502_16310_b200 -lowb200 \
//     -Xlinker -rpath=$PWD/paper_2502_16310_b200 -o gpurun_out/scan_bench && gpurun_out/scan_bench
#include <cstdio>
#include <vector>

#include "ow_scan.cuh"

struct Flag01 {
  const uint8_t* f;
  __device__ int64_t operator()(int64_t i) const { return f[i] != 0; }
};
struct Compact {
  int32_t* out;
  __device__ void operator()(int64_t i, int64_t e, int64_t v) const {
    if (v) out[e] = (int32_t)i;
  }
};

int main() {
  ow_ctx* ctx;
  if (ow_ctx_create(0, &ctx)) return 1;
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int64_t n : {131072ll, 1ll << 20, 4ll << 20, 8ll << 20, 32ll << 20}) {
    std::vector<uint8_t> h(n);
    for (int64_t i = 0; i < n; ++i) h[i] = (i * 2654435761u >> 7) % 17 == 0;
    uint8_t* f;
    int32_t* out;
    int64_t* tot;
    cudaMalloc(&f, n);
    cudaMalloc(&out, 4 * n);
    cudaMalloc(&tot, 8);
    cudaMemcpy(f, h.data(), n, cudaMemcpyHostToDevice);
    for (int kind = 0; kind < 2; ++kind) {
      for (int w = 0; w < 3; ++w)
        kind ? ow::scan01(ctx, Flag01{f}, Compact{out}, n, tot, s) : ow::scan(ctx, Flag01{f}, Compact{out}, n, tot, s);
      const int it = 20;
      cudaEventRecord(e0, s);
      for (int r = 0; r < it; ++r)
        kind ? ow::scan01(ctx, Flag01{f}, Compact{out}, n, tot, s) : ow::scan(ctx, Flag01{f}, Compact{out}, n, tot, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      int64_t t;
      cudaMemcpy(&t, tot, 8, cudaMemcpyDeviceToHost);
      int64_t ref = 0;
      for (int64_t i = 0; i < n; ++i) ref += h[i];
      printf("n=%10lld %-7s %8.2f us/scan  total %lld %s\n", (long long)n, kind ? "scan01" : "scan", 1000.0f * ms / it,
             (long long)t, t == ref ? "ok" : "MISMATCH");
    }
    cudaFree(f);
    cudaFree(out);
    cudaFree(tot);
  }
  return 0;
}
