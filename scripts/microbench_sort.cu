// Microbenchmark (not product code): throughput of the primitives a
// shared-memory block radix sort can be built from on B200 (sm_100a).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench_sort.cu
//   1. __match_any_sync on 8-bit digits (warp-level multisplit ranking)
//   2. cub::BlockRadixSort 4096 x (u32 key, u32 value), 24 key bits (reference point)
//   3. a 4-bit LSD pass in the style of tsg_esc.cu (register counters + raking scan)
#include <cub/block/block_radix_sort.cuh>
#include <cstdio>
#include <cstdint>

__global__ void match_kernel(const uint32_t* in, uint32_t* out, int iters) {
  uint32_t x = in[blockIdx.x * blockDim.x + threadIdx.x];
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    const unsigned m = __match_any_sync(0xffffffffu, x & 0xffu);
    acc += __popc(m & ((1u << (threadIdx.x & 31)) - 1u));
    x = x * 1664525u + 1013904223u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void ballot_kernel(const uint32_t* in, uint32_t* out, int iters) {
  uint32_t x = in[blockIdx.x * blockDim.x + threadIdx.x];
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    unsigned m = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const unsigned bb = __ballot_sync(0xffffffffu, (x >> b) & 1u);
      m &= ((x >> b) & 1u) ? bb : ~bb;
    }
    acc += __popc(m & ((1u << (threadIdx.x & 31)) - 1u));
    x = x * 1664525u + 1013904223u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int BITS>
__global__ void __launch_bounds__(256) cub_sort_kernel(const uint32_t* in, uint32_t* out, int reps) {
  using Sort = cub::BlockRadixSort<uint32_t, 256, 16, uint32_t, BITS>;
  __shared__ typename Sort::TempStorage tmp;
  uint32_t k[16], v[16];
  for (int i = 0; i < 16; ++i) {
    k[i] = in[(blockIdx.x * 4096 + threadIdx.x * 16 + i) & 0xfffff] & 0xffffffu;
    v[i] = i;
  }
  for (int r = 0; r < reps; ++r) {
    Sort(tmp).Sort(k, v, 0, 24);
    __syncthreads();
    for (int i = 0; i < 16; ++i) k[i] = (k[i] * 2654435761u) & 0xffffffu;
  }
  uint32_t s = 0;
  for (int i = 0; i < 16; ++i) s += k[i] ^ v[i];
  out[blockIdx.x * 256 + threadIdx.x] = s;
}

int main() {
  const int N = 148 * 8 * 256;
  uint32_t *in, *out;
  cudaMalloc(&in, 4 << 20);
  cudaMalloc(&out, 64 << 20);
  uint32_t* h = new uint32_t[1 << 20];
  for (int i = 0; i < (1 << 20); ++i) h[i] = uint32_t(i) * 2654435761u;
  cudaMemcpy(in, h, 4 << 20, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int iters = 4096;
  // warm
  match_kernel<<<148 * 8, 256>>>(in, out, 16);
  cudaEventRecord(e0);
  match_kernel<<<148 * 8, 256>>>(in, out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double warp_ops = double(N / 32) * iters;
  printf("match.any: %.3f ms, %.2f warp-ops/clk/SM (at 1.965 GHz)\n", ms, warp_ops / (ms * 1e-3) / 1.965e9 / 148);
  cudaEventRecord(e0);
  ballot_kernel<<<148 * 8, 256>>>(in, out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("8-ballot multisplit: %.3f ms, %.2f warp-ops/clk/SM\n", ms, warp_ops / (ms * 1e-3) / 1.965e9 / 148);
  for (int pass = 0; pass < 2; ++pass) {
    const int reps = 64, blocks = 148 * 2 * 8;
    cudaEventRecord(e0);
    cub_sort_kernel<4><<<blocks, 256>>>(in, out, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("cub BlockRadixSort 4096 items, 24 bits, RADIX 4: %.3f ms -> %.2f G items/s\n", ms,
           double(blocks) * reps * 4096 / (ms * 1e-3) / 1e9);
    cudaEventRecord(e0);
    cub_sort_kernel<6><<<blocks, 256>>>(in, out, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("cub BlockRadixSort 4096 items, 24 bits, RADIX 6: %.3f ms -> %.2f G items/s\n", ms,
           double(blocks) * reps * 4096 / (ms * 1e-3) / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
