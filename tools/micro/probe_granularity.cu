// Microbenchmark: DRAM bytes fetched per random 4-byte read of a table far larger than L2, for the load flavours PTX
// offers.  Run under ncu (--metrics dram__bytes_read.sum,gpu__time_duration.sum); kernel names carry the flavour.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_granularity probe_granularity.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ std::uint32_t rnd(std::uint64_t t) {
  t += 0x9e3779b97f4a7c15ull;
  t = (t ^ (t >> 30)) * 0xbf58476d1ce4e5b9ull;
  t = (t ^ (t >> 27)) * 0x94d049bb133111ebull;
  return static_cast<std::uint32_t>((t ^ (t >> 31)) >> 16);
}

#define KERNEL(NAME, ASM)                                                                                         \
  __global__ void NAME(const std::uint32_t* __restrict__ words, std::uint32_t mask, std::uint64_t count,           \
                       unsigned long long* out) {                                                                  \
    const std::uint64_t t = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;                     \
    if (t >= count) return;                                                                                        \
    const std::uint32_t* p = words + (rnd(t) & mask);                                                              \
    std::uint32_t v;                                                                                               \
    asm volatile(ASM : "=r"(v) : "l"(p));                                                                          \
    if (v == 0xdeadbeefu) atomicAdd(out, 1ull);                                                                    \
  }

KERNEL(ld_plain, "ld.global.b32 %0, [%1];")
KERNEL(ld_nc, "ld.global.nc.b32 %0, [%1];")
KERNEL(ld_nc_l2_64, "ld.global.nc.L2::64B.b32 %0, [%1];")
KERNEL(ld_nc_l2_128, "ld.global.nc.L2::128B.b32 %0, [%1];")
KERNEL(ld_nc_l2_256, "ld.global.nc.L2::256B.b32 %0, [%1];")
KERNEL(ld_cg, "ld.global.cg.b32 %0, [%1];")
KERNEL(ld_cs, "ld.global.cs.b32 %0, [%1];")
KERNEL(ld_lu, "ld.global.lu.b32 %0, [%1];")
KERNEL(ld_cv, "ld.global.cv.b32 %0, [%1];")
KERNEL(ld_nc_noalloc, "ld.global.nc.L1::no_allocate.b32 %0, [%1];")

int main() {
  const std::uint64_t words = 1ull << 28;  // 1 GiB table
  const std::uint64_t count = 1ull << 26;  // 64 M probes
  std::uint32_t* tab;
  unsigned long long* out;
  cudaMalloc(&tab, words * 4);
  cudaMalloc(&out, 8);
  cudaMemset(tab, 0, words * 4);
  cudaMemset(out, 0, 8);
  const unsigned blocks = static_cast<unsigned>(count / 256);
  const std::uint32_t mask = static_cast<std::uint32_t>(words - 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
#define RUN(NAME)                                                          \
  for (int rep = 0; rep < 2; ++rep) {                                      \
    cudaEventRecord(e0);                                                   \
    NAME<<<blocks, 256>>>(tab, mask, count, out);                          \
    cudaEventRecord(e1);                                                   \
    cudaEventSynchronize(e1);                                              \
    float ms;                                                              \
    cudaEventElapsedTime(&ms, e0, e1);                                     \
    if (rep) std::printf("%-22s %.3f ms  %.1f G probes/s\n", #NAME, ms, count / ms * 1e-6); \
  }
  RUN(ld_plain) RUN(ld_nc) RUN(ld_nc_l2_64) RUN(ld_nc_l2_128) RUN(ld_nc_l2_256) RUN(ld_cg) RUN(ld_cs) RUN(ld_lu) RUN(ld_cv)
  std::printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
