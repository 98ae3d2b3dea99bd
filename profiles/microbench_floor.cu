// Microbenchmark: the fixed cost of one event-timed step after the bench's
// L2 flush -- events around nothing, around a 1-warp no-op, around a no-op on
// every SM with ~200 KB of dynamic shared memory (the system kernel's
// carveout), stream launch vs CUDA-graph replay, with and without the flush.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -o profiles/mb_floor profiles/microbench_floor.cu && profiles/mb_floor
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void k_noop(int* p) {
  if (p != nullptr && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1;
}
__global__ void k_noop_smem(int* p) {
  extern __shared__ int sm[];
  if (threadIdx.x == 0) sm[0] = blockIdx.x;
  __syncthreads();
  if (p != nullptr && threadIdx.x == 0 && blockIdx.x == 0) p[0] = sm[0];
}
__global__ void k_write(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(0, 0, 0, 0);
}
__global__ void k_read(const uint4* p, size_t n, int* sink) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = p[i];
    acc ^= v.x ^ v.w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t nb = 256u << 20;
  uint4 *wbuf, *rbuf;
  int* sink;
  cudaMalloc(&wbuf, nb);
  cudaMalloc(&rbuf, nb);
  cudaMalloc(&sink, 64);
  cudaMemset(rbuf, 1, nb);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_noop_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t st;
  cudaStreamCreate(&st);
  auto flush = [&]() {
    k_write<<<sms * 4, 512, 0, st>>>(wbuf, nb / 16);
    k_read<<<sms * 4, 512, 0, st>>>(rbuf, nb / 16, sink);
  };
  auto rflush = [&]() { k_read<<<sms * 4, 512, 0, st>>>(rbuf, nb / 16, sink); };
  auto none = [&]() {};
  struct Case {
    const char* name;
    int what;  // 0 nothing, 1 noop 1 warp, 2 noop smem all SMs, 3 both kernels
  };
  const Case cases[] = {{"events only", 0}, {"noop <<<1,32>>>", 1},
                        {"noop <<<148,384,200KB>>>", 2}, {"smem noop then noop", 3}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int fl = 0; fl < 3; ++fl) {
    for (const Case& c : cases) {
      for (int graph = 0; graph < 2; ++graph) {
        auto body = [&]() {
          if (c.what == 1 || c.what == 3) {
            if (c.what == 3) k_noop_smem<<<sms, 384, smem, st>>>(nullptr);
            k_noop<<<1, 32, 0, st>>>(nullptr);
          } else if (c.what == 2) {
            k_noop_smem<<<sms, 384, smem, st>>>(nullptr);
          }
        };
        cudaGraphExec_t ge = nullptr;
        if (graph && c.what != 0) {
          cudaGraph_t g;
          cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
          body();
          cudaStreamEndCapture(st, &g);
          cudaGraphInstantiate(&ge, g, 0);
        }
        std::vector<float> ts;
        for (int it = 0; it < 40; ++it) {
          if (fl == 0) flush();
          else if (fl == 1) rflush();
          else none();
          cudaEventRecord(e0, st);
          if (ge) cudaGraphLaunch(ge, st);
          else body();
          cudaEventRecord(e1, st);
          cudaStreamSynchronize(st);
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          if (it >= 5) ts.push_back(ms * 1000.f);
        }
        std::sort(ts.begin(), ts.end());
        printf("%-12s %-28s %-6s median %6.2f us  min %6.2f\n",
               fl == 0 ? "flush(w+r)" : fl == 1 ? "flush(r)" : "no flush", c.name,
               graph ? "graph" : "stream", ts[ts.size() / 2], ts[0]);
      }
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
