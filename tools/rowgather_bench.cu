// Micro-benchmark: what DRAM bandwidth can a B200 sustain for RANDOM gathers of whole rows (the access pattern of
// the GEMPE gather), as opposed to the streaming copy that MEASURED_PEAKS.json's hbm_gbs was taken with?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/rowgather_bench.cu -o /tmp/rowgather && /tmp/rowgather
// One warp per row-batch, UNROLL independent 16-byte-per-lane row loads in flight, ids from a seeded LCG, the table
// (rows x row_bytes) far larger than L2.  Prints GB/s per (row_bytes, warps/SM, unroll).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int LPR, int UNROLL>
__global__ void gather_rows(const float4* __restrict__ table, std::uint32_t rows, std::uint64_t per_warp, float* out) {
  const int lane = threadIdx.x & 31, grp = lane / LPR, r = lane % LPR;
  constexpr int G = 32 / LPR;
  const std::uint64_t warp = (static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  std::uint32_t s = static_cast<std::uint32_t>(warp * 2654435761u + 12345u);
  float4 acc = make_float4(0, 0, 0, 0);
  for (std::uint64_t i = 0; i < per_warp; i += UNROLL * G) {
    float4 v[UNROLL];
#pragma unroll
    for (int q = 0; q < UNROLL; ++q) {
      s = s * 1103515245u + 12345u;
      std::uint32_t id = __shfl_sync(0xffffffffu, s, 0) + 977u * (q * G + grp);
      id = static_cast<std::uint32_t>((static_cast<std::uint64_t>(id) * rows) >> 32);
      v[q] = __ldg(table + static_cast<std::size_t>(id) * LPR + r);
    }
#pragma unroll
    for (int q = 0; q < UNROLL; ++q) {
      acc.x += v[q].x; acc.y += v[q].y; acc.z += v[q].z; acc.w += v[q].w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 123.456f) out[0] = acc.x;
}

template <int LPR, int UNROLL>
void run(const float4* table, std::uint32_t rows, float* out, int blocks_per_sm, int threads) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * blocks_per_sm;
  const std::uint64_t total_rows = 48ull << 20;  // 48 Mi rows per launch
  const std::uint64_t warps = static_cast<std::uint64_t>(blocks) * threads / 32;
  const std::uint64_t per_warp = total_rows / warps / (UNROLL * (32 / LPR)) * (UNROLL * (32 / LPR));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  gather_rows<LPR, UNROLL><<<blocks, threads>>>(table, rows, per_warp, out);
  cudaEventRecord(e0);
  for (int it = 0; it < 3; ++it) gather_rows<LPR, UNROLL><<<blocks, threads>>>(table, rows, per_warp, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = 3.0 * per_warp * warps * LPR * 16.0;
  printf("row_bytes=%4d warps/SM=%2d unroll=%2d : %7.1f GB/s\n", LPR * 16, blocks_per_sm * threads / 32, UNROLL,
         bytes / (ms * 1e-3) / 1e9);
}

int main() {
  const std::size_t table_bytes = 4ull << 30;  // 4 GiB >> 126 MB L2
  float4* table;
  float* out;
  cudaMalloc(&table, table_bytes);
  cudaMalloc(&out, 4);
  cudaMemset(table, 0, table_bytes);
  printf("random whole-row gather, table 4 GiB (uniform ids):\n");
  run<32, 4>(table, table_bytes / 512, out, 8, 256);
  run<32, 8>(table, table_bytes / 512, out, 8, 256);
  run<32, 16>(table, table_bytes / 512, out, 4, 256);
  run<32, 16>(table, table_bytes / 512, out, 8, 256);
  run<32, 8>(table, table_bytes / 512, out, 4, 128);
  run<32, 16>(table, table_bytes / 512, out, 4, 128);
  run<16, 8>(table, table_bytes / 256, out, 8, 256);
  run<16, 16>(table, table_bytes / 256, out, 8, 256);
  run<8, 16>(table, table_bytes / 128, out, 8, 256);
  run<2, 16>(table, table_bytes / 32, out, 8, 256);
  // same ids, table that fits L2 (64 MiB): the L2-resident ceiling of the same code
  printf("same kernel, table 64 MiB (L2 resident):\n");
  run<32, 16>(table, (64u << 20) / 512, out, 8, 256);
  run<16, 16>(table, (64u << 20) / 256, out, 8, 256);
  return 0;
}
