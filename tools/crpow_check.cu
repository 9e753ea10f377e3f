// Device check of crpow.cuh: pow_m13_rn on the GPU vs the same code on the
// host and vs glibc pow(x, -1.0/3.0) (the reference's Python float power).
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include "../paper_2006_14602_b200/csrc/crpow.cuh"

__global__ void k(const double* x, double* cr, double* cu, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    cr[i] = ddpma::dev::pow_m13_rn(x[i]);
    cu[i] = pow(x[i], -1.0 / 3.0);
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1 << 22;
  std::vector<double> x(n), cr(n), cu(n);
  std::mt19937_64 rng(3);
  std::uniform_real_distribution<double> u(-40.0, 6.0);
  for (auto& v : x) v = std::exp2(u(rng));
  x[0] = 0.17039558108204853;
  x[1] = 0.045791081266422486;
  double *dx, *dcr, *dcu;
  cudaMalloc(&dx, n * 8); cudaMalloc(&dcr, n * 8); cudaMalloc(&dcu, n * 8);
  cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice);
  k<<<(n + 255) / 256, 256>>>(dx, dcr, dcu, n);
  cudaMemcpy(cr.data(), dcr, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(cu.data(), dcu, n * 8, cudaMemcpyDeviceToHost);
  long dev_vs_host = 0, dev_vs_glibc = 0, cuda_vs_glibc = 0;
  for (int i = 0; i < n; ++i) {
    const double h = ddpma::dev::pow_m13_rn(x[i]), g = std::pow(x[i], -1.0 / 3.0);
    if (i < 2) printf("x=%.17g dev=%.17g host=%.17g glibc=%.17g cuda=%.17g\n", x[i], cr[i], h, g, cu[i]);
    dev_vs_host += cr[i] != h;
    dev_vs_glibc += cr[i] != g;
    cuda_vs_glibc += cu[i] != g;
  }
  printf("n=%d device-vs-host %ld device-vs-glibc %ld cuda-pow-vs-glibc %ld\n", n, dev_vs_host,
         dev_vs_glibc, cuda_vs_glibc);
  return dev_vs_host != 0;
}
