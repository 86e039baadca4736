// Exhaustive check of K1's div_by_sb (paper_2108_05818_b200/csrc/adam_tma.cu):
// RN_f32(x * RN_f64(1/c)) == __fdiv_rn(x, c) for EVERY non-negative float x
// (all 2^31 bit patterns: zero, subnormals, normals, inf, nan) and each
// divisor c given on the command line (as float bit patterns, hex).
// Prints, per c, the mismatch counts for x >= 2^-75 or x in {0, inf, nan}
// (the operands K1 sees: x = sqrt(v)) and for the remaining tiny x.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>

__global__ void check(float c, double rc, unsigned long long* bad) {
  unsigned long long dom = 0, rest = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < 0x80000000u; i += stride) {
    const float x = __uint_as_float(i);
    const float a = __fdiv_rn(x, c);
    const float b = __double2float_rn(__dmul_rn((double)x, rc));
    const bool same = (__float_as_uint(a) == __float_as_uint(b)) || (a != a && b != b);
    if (!same) {
      if (i >= 0x1a000000u || i == 0u) ++dom;   // 0x1a000000 = 2^-75
      else ++rest;
    }
  }
  if (dom) atomicAdd(&bad[0], dom);
  if (rest) atomicAdd(&bad[1], rest);
}

int main(int argc, char** argv) {
  unsigned long long* bad;
  cudaMalloc(&bad, 2 * sizeof(unsigned long long));
  unsigned long long total_dom = 0;
  for (int k = 1; k < argc; ++k) {
    const uint32_t bits = (uint32_t)strtoul(argv[k], nullptr, 16);
    float c;
    std::memcpy(&c, &bits, 4);
    cudaMemset(bad, 0, 2 * sizeof(unsigned long long));
    check<<<148 * 8, 256>>>(c, 1.0 / (double)c, bad);
    unsigned long long h[2];
    cudaMemcpy(h, bad, sizeof(h), cudaMemcpyDeviceToHost);
    if (cudaGetLastError() != cudaSuccess) { printf("cuda error\n"); return 2; }
    printf("%08x %.9g %llu %llu\n", bits, c, h[0], h[1]);
    total_dom += h[0];
  }
  return total_dom ? 1 : 0;
}
