// div_guard_by(guard, y) (stencil.cuh) against the IEEE quotient guard / y, bitwise, over random
// operands of the ranges logequi_pair uses it for.   nvcc -arch=sm_100a -fmad=false ...
#include <cstdio>
#include <cstdint>
#include "../paper_2006_14602_b200/csrc/stencil.cuh"
using namespace ddpma::dev;
__device__ unsigned long long rng(unsigned long long& s) {
  s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s;
}
__global__ void k(unsigned long long* bad, unsigned long long* first, int iters) {
  unsigned long long s = 0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  unsigned long long nb = 0;
  for (int i = 0; i < iters; ++i) {
    const unsigned long long a = rng(s), b = rng(s), c = rng(s);
    // guard: mantissa random, exponent in [-300, 300] (half of the samples in [-20, 20])
    const int eg = (c & 1) ? (int)((c >> 8) % 41) - 20 : (int)((c >> 8) % 601) - 300;
    const double guard = __longlong_as_double((long long)(((unsigned long long)(1023 + eg) << 52) | (a >> 12)));
    // y in [1, 2^100]: mantissa random, exponent in [0, 100) (half of the samples in [0, 2))
    const int ey = (c & 2) ? (int)((c >> 24) % 2) : (int)((c >> 24) % 100);
    double y = __longlong_as_double((long long)(((unsigned long long)(1023 + ey) << 52) | (b >> 12)));
    if ((c & 12) == 0) y = 2.0 - __longlong_as_double((long long)((1022ull << 52) | (b >> 12))) * ((c & 16) ? 1.0 : -1.0);
    if (!(y >= 1.0 && y <= 0x1p100)) continue;
    const double q = div_guard_by(guard, y), ref = guard / y;
    if (__double_as_longlong(q) != __double_as_longlong(ref)) {
      if (nb == 0) { first[0] = __double_as_longlong(guard); first[1] = __double_as_longlong(y); }
      ++nb;
    }
  }
  atomicAdd(bad, nb);
}
int main() {
  unsigned long long *bad, *first;
  cudaMallocManaged(&bad, 8); cudaMallocManaged(&first, 16);
  *bad = 0; first[0] = first[1] = 0;
  const int iters = 4000;
  k<<<1184, 256>>>(bad, first, iters);
  cudaDeviceSynchronize();
  printf("samples=%llu mismatches=%llu first=(%a, %a) err=%s\n", 1184ull * 256 * iters, *bad,
         *(double*)&first[0], *(double*)&first[1], cudaGetErrorString(cudaGetLastError()));
  return *bad ? 1 : 0;
}
