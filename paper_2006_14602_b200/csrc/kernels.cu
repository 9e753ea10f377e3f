// Device kernels of the DDPMA hot path (sm_100a, fp64).
//
// Every arithmetic expression restates the reference's numpy expression in
// the same evaluation order; the library is compiled with -fmad=false so no
// multiply-add contraction changes the rounding.  Divisions by grid-derived
// constants (h*h, 2*h) become multiplications by the exact reciprocal when
// every spacing is a power of two (the BASELINE grids: n-1 = 2^k), which is
// bitwise identical; otherwise a true IEEE division is used.
//
// Layout: every field is one arena; local subdomain boxes are stored
// back-to-back, C order, last axis fastest, rows padded to `pitch` elements.
// A launch covers a list of Entries (one per participating subdomain); CTA b
// belongs to the entry whose tile range contains b.  Tiles are TX x TY nodes
// on the two fastest axes (one plane per CTA in 3D).

#include <cuda_runtime.h>

#include <cmath>

#include "ddpma_internal.h"

namespace ddpma {

namespace {

template <bool P2>
__device__ __forceinline__ double dv(double x, double d, double inv) {
  if constexpr (P2) {
    return x * inv;
  } else {
    return x / d;
  }
}

template <int DIM>
__device__ __forceinline__ long long lin(const SubGeo& g, int i0, int i1, int i2) {
  if constexpr (DIM == 2) {
    return g.off + (long long)i0 * g.pitch + i1;
  } else {
    return g.off + ((long long)i0 * g.n[1] + i1) * g.pitch + i2;
  }
}

enum YMode { YM_PLAIN = 0, YM_ADD = 1, YM_SCALED = 2, YM_SEED = 3 };

// Stage input Y at absolute box indices.
//   PLAIN : y                       SCALED: y + c*a   (a = f0 or v)
//   ADD   : y + a  (a = d_{j-1})    SEED  : y + (+-c)  (checkerboard, integrate.py:127-129)
template <int DIM, int YM>
struct YAcc {
  const SubGeo* g;
  const double* __restrict__ y;
  const double* __restrict__ a;
  double c;
  __device__ __forceinline__ double operator()(int i0, int i1, int i2) const {
    const long long k = lin<DIM>(*g, i0, i1, i2);
    const double yv = __ldg(y + k);
    if constexpr (YM == YM_PLAIN) {
      return yv;
    } else if constexpr (YM == YM_ADD) {
      return yv + __ldg(a + k);
    } else if constexpr (YM == YM_SCALED) {
      return yv + c * __ldg(a + k);
    } else {
      const int par = (i0 + i1 + (DIM == 3 ? i2 : 0)) & 1;
      return yv + (par ? -c : c);
    }
  }
};

// _second_diff (pma.py:87-115) at index i of an axis with n nodes.
template <bool P2, class F1>
__device__ __forceinline__ double d2ax(const AxisC& A, int n, int i, int plo, int phi,
                                       double halo, double hahi, const F1& f) {
  if (i >= 1 && i <= n - 2) return dv<P2>((f(1) - 2.0 * f(0)) + f(-1), A.hh, A.ihh);
  if (i == 0) {
    if (plo) return dv<P2>(2.0 * ((f(1) - f(0)) - halo), A.hh, A.ihh);
    if (n >= 4) return dv<P2>(((2.0 * f(0) - 5.0 * f(1)) + 4.0 * f(2)) - f(3), A.hh, A.ihh);
    return dv<P2>((f(2) - 2.0 * f(1)) + f(0), A.hh, A.ihh);
  }
  if (phi) return dv<P2>(2.0 * ((f(-1) - f(0)) + hahi), A.hh, A.ihh);
  if (n >= 4) return dv<P2>(((2.0 * f(0) - 5.0 * f(-1)) + 4.0 * f(-2)) - f(-3), A.hh, A.ihh);
  return dv<P2>((f(0) - 2.0 * f(-1)) + f(-2), A.hh, A.ihh);
}

// np.gradient(edge_order=2, uniform spacing) at index i
// (numpy/lib/_function_base_impl.py:1305 interior, :1343-1372 edges).
template <bool P2, class F1>
__device__ __forceinline__ double grad1(const AxisC& A, int n, int i, const F1& f) {
  if (i >= 1 && i <= n - 2) return dv<P2>(f(1) - f(-1), A.twoh, A.itwoh);
  if (i == 0) return (A.ea * f(0) + A.eb * f(1)) + A.ec * f(2);
  return (A.fa * f(-2) + A.fb * f(-1)) + A.fc * f(0);
}

// _cross_diff (pma.py:118-130): gradient along l, then along k, zero on the
// physical faces of either axis.  f(a, b) = Y at offsets (a along k, b along l).
template <bool P2, class F2>
__device__ __forceinline__ double cross(const AxisC& K, const AxisC& L, int nk, int nl, int i,
                                        int j, int plk, int phk, int pll, int phl, const F2& f) {
  if ((i == 0 && plk) || (i == nk - 1 && phk) || (j == 0 && pll) || (j == nl - 1 && phl))
    return 0.0;
  auto G = [&](int a) { return grad1<P2>(L, nl, j, [&](int b) { return f(a, b); }); };
  return grad1<P2>(K, nk, i, G);
}

// hessian_det_fd (pma.py:133-149) at one node.
template <int DIM, bool P2, class YF>
__device__ __forceinline__ double hdet(const Prob& P, const SubGeo& g, int i0, int i1, int i2,
                                       const YF& Y) {
  const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];
  if constexpr (DIM == 2) {
    if (i0 >= 1 && i0 <= n0 - 2 && i1 >= 1 && i1 <= n1 - 2) {
      const double c = Y(i0, i1, 0);
      const double h00 = dv<P2>((Y(i0 + 1, i1, 0) - 2.0 * c) + Y(i0 - 1, i1, 0), P.ax[0].hh, P.ax[0].ihh);
      const double h11 = dv<P2>((Y(i0, i1 + 1, 0) - 2.0 * c) + Y(i0, i1 - 1, 0), P.ax[1].hh, P.ax[1].ihh);
      const double gp = dv<P2>(Y(i0 + 1, i1 + 1, 0) - Y(i0 + 1, i1 - 1, 0), P.ax[1].twoh, P.ax[1].itwoh);
      const double gm = dv<P2>(Y(i0 - 1, i1 + 1, 0) - Y(i0 - 1, i1 - 1, 0), P.ax[1].twoh, P.ax[1].itwoh);
      const double h01 = dv<P2>(gp - gm, P.ax[0].twoh, P.ax[0].itwoh);
      return h00 * h11 - h01 * h01;
    }
    const double h00 = d2ax<P2>(P.ax[0], n0, i0, g.plo[0], g.phi[0], g.halo[0], g.hahi[0],
                                [&](int o) { return Y(i0 + o, i1, 0); });
    const double h11 = d2ax<P2>(P.ax[1], n1, i1, g.plo[1], g.phi[1], g.halo[1], g.hahi[1],
                                [&](int o) { return Y(i0, i1 + o, 0); });
    const double h01 = cross<P2>(P.ax[0], P.ax[1], n0, n1, i0, i1, g.plo[0], g.phi[0], g.plo[1],
                                 g.phi[1], [&](int a, int b) { return Y(i0 + a, i1 + b, 0); });
    return h00 * h11 - h01 * h01;
  } else {
    double h00, h11, h22, h01, h02, h12;
    if (i0 >= 1 && i0 <= n0 - 2 && i1 >= 1 && i1 <= n1 - 2 && i2 >= 1 && i2 <= n2 - 2) {
      const double c = Y(i0, i1, i2);
      h00 = dv<P2>((Y(i0 + 1, i1, i2) - 2.0 * c) + Y(i0 - 1, i1, i2), P.ax[0].hh, P.ax[0].ihh);
      h11 = dv<P2>((Y(i0, i1 + 1, i2) - 2.0 * c) + Y(i0, i1 - 1, i2), P.ax[1].hh, P.ax[1].ihh);
      h22 = dv<P2>((Y(i0, i1, i2 + 1) - 2.0 * c) + Y(i0, i1, i2 - 1), P.ax[2].hh, P.ax[2].ihh);
      double gp = dv<P2>(Y(i0 + 1, i1 + 1, i2) - Y(i0 + 1, i1 - 1, i2), P.ax[1].twoh, P.ax[1].itwoh);
      double gm = dv<P2>(Y(i0 - 1, i1 + 1, i2) - Y(i0 - 1, i1 - 1, i2), P.ax[1].twoh, P.ax[1].itwoh);
      h01 = dv<P2>(gp - gm, P.ax[0].twoh, P.ax[0].itwoh);
      gp = dv<P2>(Y(i0 + 1, i1, i2 + 1) - Y(i0 + 1, i1, i2 - 1), P.ax[2].twoh, P.ax[2].itwoh);
      gm = dv<P2>(Y(i0 - 1, i1, i2 + 1) - Y(i0 - 1, i1, i2 - 1), P.ax[2].twoh, P.ax[2].itwoh);
      h02 = dv<P2>(gp - gm, P.ax[0].twoh, P.ax[0].itwoh);
      gp = dv<P2>(Y(i0, i1 + 1, i2 + 1) - Y(i0, i1 + 1, i2 - 1), P.ax[2].twoh, P.ax[2].itwoh);
      gm = dv<P2>(Y(i0, i1 - 1, i2 + 1) - Y(i0, i1 - 1, i2 - 1), P.ax[2].twoh, P.ax[2].itwoh);
      h12 = dv<P2>(gp - gm, P.ax[1].twoh, P.ax[1].itwoh);
    } else {
      h00 = d2ax<P2>(P.ax[0], n0, i0, g.plo[0], g.phi[0], g.halo[0], g.hahi[0],
                     [&](int o) { return Y(i0 + o, i1, i2); });
      h11 = d2ax<P2>(P.ax[1], n1, i1, g.plo[1], g.phi[1], g.halo[1], g.hahi[1],
                     [&](int o) { return Y(i0, i1 + o, i2); });
      h22 = d2ax<P2>(P.ax[2], n2, i2, g.plo[2], g.phi[2], g.halo[2], g.hahi[2],
                     [&](int o) { return Y(i0, i1, i2 + o); });
      h01 = cross<P2>(P.ax[0], P.ax[1], n0, n1, i0, i1, g.plo[0], g.phi[0], g.plo[1], g.phi[1],
                      [&](int a, int b) { return Y(i0 + a, i1 + b, i2); });
      h02 = cross<P2>(P.ax[0], P.ax[2], n0, n2, i0, i2, g.plo[0], g.phi[0], g.plo[2], g.phi[2],
                      [&](int a, int b) { return Y(i0 + a, i1, i2 + b); });
      h12 = cross<P2>(P.ax[1], P.ax[2], n1, n2, i1, i2, g.plo[1], g.phi[1], g.plo[2], g.phi[2],
                      [&](int a, int b) { return Y(i0, i1 + a, i2 + b); });
    }
    return (h00 * (h11 * h22 - h12 * h12) - h01 * (h01 * h22 - h12 * h02)) +
           h02 * (h01 * h12 - h11 * h02);
  }
}

// gradient_fd (pma.py:67-84) component k at a node: np.gradient, with the
// exact face coordinate on the physical faces of axis k.
template <int DIM, bool P2, class YF>
__device__ __forceinline__ double coord(const Prob& P, const SubGeo& g, int k, int i0, int i1,
                                        int i2, const YF& Y) {
  const int i = k == 0 ? i0 : (k == 1 ? i1 : i2);
  if (i == 0 && g.plo[k]) return g.alo[k];
  if (i == g.n[k] - 1 && g.phi[k]) return g.ahi[k];
  if (k == 0) return grad1<P2>(P.ax[0], g.n[0], i0, [&](int o) { return Y(i0 + o, i1, i2); });
  if (k == 1) return grad1<P2>(P.ax[1], g.n[1], i1, [&](int o) { return Y(i0, i1 + o, i2); });
  return grad1<P2>(P.ax[2], g.n[2], i2, [&](int o) { return Y(i0, i1, i2 + o); });
}

// _log_equidistribution (pma.py:186-192) with the host-computed guard.
__device__ __forceinline__ double logequi(double mr, double det, double guard, double floor) {
  const double eff = (det >= guard) ? det : guard / (2.0 - det / guard);
  const double m = (eff >= floor || isnan(eff)) ? eff : floor;   // np.maximum (NaN-propagating)
  return log(mr * m);
}

template <int DIM>
__device__ __forceinline__ bool dirichlet(const SubGeo& g, int i0, int i1, int i2) {
  bool d = (i0 == 0 && !g.plo[0]) || (i0 == g.n[0] - 1 && !g.phi[0]) ||
           (i1 == 0 && !g.plo[1]) || (i1 == g.n[1] - 1 && !g.phi[1]);
  if constexpr (DIM == 3) d = d || (i2 == 0 && !g.plo[2]) || (i2 == g.n[2] - 1 && !g.phi[2]);
  return d;
}

__device__ __forceinline__ double clampv(double p, double lo, double hi) {
  return p < lo ? lo : (p > hi ? hi : p);   // np.clip, NaN passes through
}

// MonitorField.raw of the native descriptors (monitor.py:100-104 callers).
template <int DIM>
__device__ double mon_raw(const MonitorD& M, const double* x) {
  double p[3];
#pragma unroll
  for (int k = 0; k < DIM; ++k) p[k] = clampv(x[k], M.lo[k], M.hi[k]);
  if (M.kind == 0) return M.constant;
  if (M.kind == 1) {
    double t = p[0] - M.center[0];
    double acc = t * t;
#pragma unroll
    for (int k = 1; k < DIM; ++k) {
      t = p[k] - M.center[k];
      acc = acc + t * t;
    }
    return 1.0 + M.amp * exp(M.nsharp * fabs(acc - M.r2));
  }
  double tot = 0.0;
  for (int b = 0; b < M.nb; ++b) {
    double t = p[0] - M.c[b * 3 + 0];
    double d2 = t * t;
#pragma unroll
    for (int k = 1; k < DIM; ++k) {
      t = p[k] - M.c[b * 3 + k];
      d2 = d2 + t * t;
    }
    tot = tot + M.a[b] * exp((-d2) / M.den[b]);
  }
  return 1.0 + tot;
}

__device__ __forceinline__ unsigned long long okey(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ int find_entry(const Entry* ent, int nent, int b) {
  int lo = 0, hi = nent - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (ent[mid].tile_begin <= b) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

template <int DIM>
__device__ __forceinline__ bool tile_node(const SubGeo& g, int t, int& i0, int& i1, int& i2) {
  const int tx = t % g.tiles_x;
  const int r = t / g.tiles_x;
  const int ty = r % g.tiles_y;
  const int tz = r / g.tiles_y;
  if constexpr (DIM == 2) {
    i1 = tx * TX + threadIdx.x;
    i0 = ty * TY + threadIdx.y;
    i2 = 0;
    return i0 < g.n[0] && i1 < g.n[1];
  } else {
    i2 = tx * TX + threadIdx.x;
    i1 = ty * TY + threadIdx.y;
    i0 = tz;
    return i1 < g.n[1] && i2 < g.n[2];
  }
}

// Fixed-order CTA sum (warp tree, then warps in order): deterministic.
__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  const int lane = threadIdx.x, warp = threadIdx.y;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double tot = 0.0;
  if (lane == 0 && warp == 0) {
    tot = sh[0];
    for (int w = 1; w < NT / 32; ++w) tot += sh[w];
  }
  __syncthreads();
  return tot;
}

__device__ __forceinline__ unsigned long long block_max_u64(unsigned long long v,
                                                            unsigned long long* sh) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_down_sync(0xffffffffu, v, off);
    v = o > v ? o : v;
  }
  const int lane = threadIdx.x, warp = threadIdx.y;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  unsigned long long m = 0;
  if (lane == 0 && warp == 0) {
    m = sh[0];
    for (int w = 1; w < NT / 32; ++w) m = sh[w] > m ? sh[w] : m;
  }
  __syncthreads();
  return m;
}

__device__ __forceinline__ unsigned long long block_min_u64(unsigned long long v,
                                                            unsigned long long* sh) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_down_sync(0xffffffffu, v, off);
    v = o < v ? o : v;
  }
  const int lane = threadIdx.x, warp = threadIdx.y;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  unsigned long long m = ~0ull;
  if (lane == 0 && warp == 0) {
    m = sh[0];
    for (int w = 1; w < NT / 32; ++w) m = sh[w] < m ? sh[w] : m;
  }
  __syncthreads();
  return m;
}

// ------------------------------------------------------------- eval kernel --
// One frozen-density RHS evaluation (pma_rhs_frozen, pma.py:195-219) per node,
// fused with what consumes it in the integrator (integrate.py:163-208).
template <int DIM, bool P2, int MODE>
__global__ void __launch_bounds__(NT) k_eval(const KArgs a) {
  __shared__ double sh_sum[NT / 32];
  __shared__ unsigned long long sh_max[NT / 32];
  const int b = blockIdx.x;
  const Entry e = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[e.sub];
  int i0, i1, i2;
  const bool valid = tile_node<DIM>(g, b - e.tile_begin, i0, i1, i2);
  unsigned flag = 0, nonfin = 0;
  double ratio = 0.0, psum = 0.0;
  if (valid) {
    const long long k = lin<DIM>(g, i0, i1, i2);
    const bool dir = dirichlet<DIM>(g, i0, i1, i2);
    const double* __restrict__ yb = a.F.y[e.yi];
    double det;
    if constexpr (MODE == M_F0 || MODE == M_EULER) {
      det = hdet<DIM, P2>(a.P, g, i0, i1, i2, YAcc<DIM, YM_PLAIN>{&g, yb, nullptr, 0.0});
    } else if constexpr (MODE == M_STAGE2) {
      det = hdet<DIM, P2>(a.P, g, i0, i1, i2, YAcc<DIM, YM_SCALED>{&g, yb, a.F.f[e.fi], e.c});
    } else if constexpr (MODE == M_STAGE3 || MODE == M_STAGEN) {
      det = hdet<DIM, P2>(a.P, g, i0, i1, i2, YAcc<DIM, YM_ADD>{&g, yb, a.F.d[(a.j - 1) % 3], 0.0});
    } else if constexpr (MODE == M_FINAL) {
      det = hdet<DIM, P2>(a.P, g, i0, i1, i2, YAcc<DIM, YM_ADD>{&g, yb, a.F.d[e.s % 3], 0.0});
    } else if constexpr (MODE == M_POWER) {
      det = hdet<DIM, P2>(a.P, g, i0, i1, i2, YAcc<DIM, YM_SCALED>{&g, yb, a.F.d[e.vin], e.c});
    } else {
      det = hdet<DIM, P2>(a.P, g, i0, i1, i2, YAcc<DIM, YM_SEED>{&g, yb, nullptr, e.c});
    }
    const double F = dir ? 0.0 : logequi(__ldg(a.F.mr + k), det, a.P.guard, a.P.floor);
    flag = (det <= a.P.floor && !dir) ? 1u : 0u;
    if constexpr (MODE == M_F0) {
      a.F.f[e.fi][k] = F;
    } else if constexpr (MODE == M_EULER) {
      a.F.y[1 - e.yi][k] = yb[k] + e.c * F;
    } else if constexpr (MODE == M_STAGE2 || MODE == M_STAGE3 || MODE == M_STAGEN) {
      const Coef q = a.coef[e.coef + a.j];
      const double f0 = __ldg(a.F.f[e.fi] + k);
      const double d1 = e.c * f0;
      double dp, dp2;
      if constexpr (MODE == M_STAGE2) {
        dp = d1;
        dp2 = 0.0;
      } else if constexpr (MODE == M_STAGE3) {
        dp = __ldg(a.F.d[2] + k);
        dp2 = d1;
      } else {
        dp = __ldg(a.F.d[(a.j - 1) % 3] + k);
        dp2 = __ldg(a.F.d[(a.j - 2) % 3] + k);
      }
      a.F.d[a.j % 3][k] = ((q.mu * dp + q.nu * dp2) + q.hmut * F) + q.hgt * f0;
    } else if constexpr (MODE == M_FINAL) {
      const double ds = __ldg(a.F.d[e.s % 3] + k);
      const double yv = yb[k];
      const double yn = yv + ds;
      const double f0 = __ldg(a.F.f[e.fi] + k);
      a.F.f[1 - e.fi][k] = F;
      a.F.y[1 - e.yi][k] = yn;
      const double err = -0.8 * ds + e.h04 * (f0 + F);
      const double ay = fabs(yv), an = fabs(yn);
      const double mx = (ay >= an || isnan(ay)) ? ay : an;     // np.maximum
      const double r = fabs(err) / (a.P.atol + a.P.rtol * mx);
      if (isfinite(r)) ratio = r;
      else nonfin = 1;
    } else {   // power iteration: diff = F(y + c v) - f0
      const double diff = F - __ldg(a.F.f[e.fi] + k);
      a.F.d[e.vout][k] = diff;
      psum = diff * diff;
    }
  }
  const int any = __syncthreads_or(flag);
  if constexpr (MODE == M_FINAL) {
    const int anynf = __syncthreads_or(nonfin);
    const unsigned long long m =
        block_max_u64((unsigned long long)__double_as_longlong(ratio), sh_max);
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      unsigned bits = (any ? 2u : 0u) | (anynf ? 4u : 0u);
      if (bits) atomicOr(&a.res[e.sub].flags, bits);
      atomicMax(&a.res[e.sub].emax, m);
    }
  } else {
    if (any && threadIdx.x == 0 && threadIdx.y == 0) atomicOr(&a.res[e.sub].flags, 1u);
  }
  if constexpr (MODE == M_POWER || MODE == M_POWER_SEED) {
    const double s = block_sum(psum, sh_sum);
    if (threadIdx.x == 0 && threadIdx.y == 0) a.part[b] = s;
  }
}

// sum of y^2 per CTA (np.linalg.norm(y), integrate.py:133).
template <int DIM>
__global__ void __launch_bounds__(NT) k_sumsq(const KArgs a) {
  __shared__ double sh[NT / 32];
  const int b = blockIdx.x;
  const Entry e = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[e.sub];
  int i0, i1, i2;
  double v = 0.0;
  if (tile_node<DIM>(g, b - e.tile_begin, i0, i1, i2)) {
    const double y = a.F.y[e.yi][lin<DIM>(g, i0, i1, i2)];
    v = y * y;
  }
  const double s = block_sum(v, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0) a.part[b] = s;
}

__global__ void __launch_bounds__(256) k_finalize(const Entry* ent, const double* part,
                                                  SubRes* res, int which) {
  __shared__ double sh[256];
  const Entry e = ent[blockIdx.x];
  double v = 0.0;
  for (int i = threadIdx.x; i < e.ntiles; i += 256) v += part[e.tile_begin + i];
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (which == 0) res[e.sub].sum = sh[0];
    else res[e.sub].sum2 = sh[0];
  }
}

// ----------------------------------------------------------- mesh kernel --
// physical_mesh (pma.py:222-225) + mesh_density (monitor.py:151-180) + the
// owned-node transport partial w*raw*J (schwarz.py:182-186) + the window
// residual (psi - psi_level_n)^2 * w_box (schwarz.py:111-115) + J min/max.
template <int DIM, bool P2>
__global__ void __launch_bounds__(NT) k_mesh(const KArgs a, int with_res) {
  __shared__ double sh_sum[NT / 32];
  __shared__ unsigned long long sh_u[NT / 32];
  const int b = blockIdx.x;
  const Entry e = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[e.sub];
  int i0, i1, i2;
  const bool valid = tile_node<DIM>(g, b - e.tile_begin, i0, i1, i2);
  double zp = 0.0, rp = 0.0;
  unsigned long long kmin = ~0ull, kmax = 0ull, rmax = 0ull;
  unsigned jn = 0;
  if (valid) {
    const long long k = lin<DIM>(g, i0, i1, i2);
    const double* __restrict__ yb = a.F.y[e.yi];
    const YAcc<DIM, YM_PLAIN> Y{&g, yb, nullptr, 0.0};
    double x[3];
#pragma unroll
    for (int q = 0; q < DIM; ++q) x[q] = coord<DIM, P2>(a.P, g, q, i0, i1, i2, Y);
    const double det = hdet<DIM, P2>(a.P, g, i0, i1, i2, Y);
    const double raw = mon_raw<DIM>(*a.mon, x);
    a.F.raw[k] = raw;
    const int idx[3] = {i0, i1, i2};
    bool owned = true;
#pragma unroll
    for (int q = 0; q < DIM; ++q) owned = owned && idx[q] >= g.olo[q] && idx[q] <= g.ohi[q];
    if (owned) {
      double w = 1.0;
#pragma unroll
      for (int q = 0; q < DIM; ++q) {
        const int gi = g.glo[q] + idx[q];
        const double wq = (gi == 0 || gi == a.P.ax[q].n - 1) ? a.P.ax[q].w_end : a.P.ax[q].w_in;
        w = q == 0 ? wq : w * wq;
      }
      zp = (w * raw) * det;
    }
    if (with_res) {
      double w = 1.0;
#pragma unroll
      for (int q = 0; q < DIM; ++q) {
        const double wq = (idx[q] == 0 || idx[q] == g.n[q] - 1) ? a.P.ax[q].w_end : a.P.ax[q].w_in;
        w = q == 0 ? wq : w * wq;
      }
      const double v = yb[k] - a.F.old[k];
      rp = (v * v) * w;
    }
    if (isnan(det)) jn = 1;
    kmin = kmax = okey(det);
    rmax = okey(raw);
  }
  const double zs = block_sum(zp, sh_sum);
  if (threadIdx.x == 0 && threadIdx.y == 0) a.part[b] = zs;
  const double rs = block_sum(rp, sh_sum);
  if (threadIdx.x == 0 && threadIdx.y == 0) a.part2[b] = rs;
  const unsigned long long mn = block_min_u64(kmin, sh_u);
  const unsigned long long mx = block_max_u64(kmax, sh_u);
  const unsigned long long rm = block_max_u64(rmax, sh_u);
  const int anyn = __syncthreads_or(jn);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    SubRes* r = a.res + e.sub;
    atomicMin(&r->jmin, mn);
    atomicMax(&r->jmax, mx);
    atomicMax(&r->rawmax, rm);
    if (anyn) atomicOr(&r->jnan, 1u);
  }
}

// Window prologue: psi_level_n snapshot + measure*(raw/z) (schwarz.py:190,251).
template <int DIM>
__global__ void __launch_bounds__(NT) k_prologue(const KArgs a, double z) {
  const int b = blockIdx.x;
  const Entry e = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[e.sub];
  int i0, i1, i2;
  if (!tile_node<DIM>(g, b - e.tile_begin, i0, i1, i2)) return;
  const long long k = lin<DIM>(g, i0, i1, i2);
  a.F.old[k] = a.F.y[e.yi][k];
  a.F.mr[k] = a.P.measure * (a.F.raw[k] / z);
}

// psi0 = 0.5*sum_k xi_k^2 on the global grid, sliced (pma.py:61-64).
template <int DIM>
__global__ void __launch_bounds__(NT) k_psi0(const KArgs a) {
  const int b = blockIdx.x;
  const Entry e = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[e.sub];
  int i0, i1, i2;
  if (!tile_node<DIM>(g, b - e.tile_begin, i0, i1, i2)) return;
  const int idx[3] = {i0, i1, i2};
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < DIM; ++q) {
    const double x = a.P.a0[q] + (double)(g.glo[q] + idx[q]) * a.P.ax[q].h;
    s = q == 0 ? x * x : s + x * x;
  }
  a.F.y[e.yi][lin<DIM>(g, i0, i1, i2)] = 0.5 * s;
}

template <int DIM>
__device__ __forceinline__ long long glin(const Prob& P, const SubGeo& g, int i0, int i1, int i2) {
  if constexpr (DIM == 2) {
    return (long long)(g.glo[0] + i0) * P.ax[1].n + (g.glo[1] + i1);
  } else {
    return ((long long)(g.glo[0] + i0) * P.ax[1].n + (g.glo[1] + i1)) * P.ax[2].n + (g.glo[2] + i2);
  }
}

// Warm start: slice a global field into the boxes (schwarz.py:128).
template <int DIM>
__global__ void __launch_bounds__(NT) k_scatter(const KArgs a, const double* __restrict__ gsrc) {
  const int b = blockIdx.x;
  const Entry e = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[e.sub];
  int i0, i1, i2;
  if (!tile_node<DIM>(g, b - e.tile_begin, i0, i1, i2)) return;
  a.F.y[e.yi][lin<DIM>(g, i0, i1, i2)] = gsrc[glin<DIM>(a.P, g, i0, i1, i2)];
}

// _assemble (schwarz.py:271-282): owned blocks into global psi/coords/jac.
template <int DIM, bool P2>
__global__ void __launch_bounds__(NT) k_assemble(const KArgs a, double* psi, double* coords,
                                                 double* jac) {
  const int b = blockIdx.x;
  const Entry e = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[e.sub];
  int i0, i1, i2;
  if (!tile_node<DIM>(g, b - e.tile_begin, i0, i1, i2)) return;
  const int idx[3] = {i0, i1, i2};
#pragma unroll
  for (int q = 0; q < DIM; ++q)
    if (idx[q] < g.olo[q] || idx[q] > g.ohi[q]) return;
  const long long gk = glin<DIM>(a.P, g, i0, i1, i2);
  const double* yb = a.F.y[e.yi];
  const YAcc<DIM, YM_PLAIN> Y{&g, yb, nullptr, 0.0};
  if (psi) psi[gk] = yb[lin<DIM>(g, i0, i1, i2)];
  if (coords) {
#pragma unroll
    for (int q = 0; q < DIM; ++q) coords[gk * DIM + q] = coord<DIM, P2>(a.P, g, q, i0, i1, i2, Y);
  }
  if (jac) jac[gk] = hdet<DIM, P2>(a.P, g, i0, i1, i2, Y);
}

// Dense box outputs of gradient_fd / hessian_det_fd / mesh_density for the
// operator-level API (pma.py:67-84,133-149; monitor.py:151-180).
template <int DIM, bool P2>
__global__ void __launch_bounds__(NT) k_box_mesh(const KArgs a, double* coords, double* jac,
                                                 double* raw) {
  const int b = blockIdx.x;
  const Entry e = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[e.sub];
  int i0, i1, i2;
  if (!tile_node<DIM>(g, b - e.tile_begin, i0, i1, i2)) return;
  const long long dk = DIM == 2 ? (long long)i0 * g.n[1] + i1
                                : ((long long)i0 * g.n[1] + i1) * g.n[2] + i2;
  const YAcc<DIM, YM_PLAIN> Y{&g, a.F.y[e.yi], nullptr, 0.0};
  double x[3];
#pragma unroll
  for (int q = 0; q < DIM; ++q) x[q] = coord<DIM, P2>(a.P, g, q, i0, i1, i2, Y);
  if (coords) {
#pragma unroll
    for (int q = 0; q < DIM; ++q) coords[dk * DIM + q] = x[q];
  }
  if (jac) jac[dk] = hdet<DIM, P2>(a.P, g, i0, i1, i2, Y);
  if (raw) raw[dk] = mon_raw<DIM>(*a.mon, x);
}

// Box <-> dense copies (operator-level API, sub_psi).
template <int DIM>
__global__ void __launch_bounds__(NT) k_box_copy(const KArgs a, const double* src, double* dst,
                                                 int to_arena) {
  const int b = blockIdx.x;
  const Entry e = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[e.sub];
  int i0, i1, i2;
  if (!tile_node<DIM>(g, b - e.tile_begin, i0, i1, i2)) return;
  const long long k = lin<DIM>(g, i0, i1, i2);
  const long long dk = DIM == 2 ? (long long)i0 * g.n[1] + i1
                                : ((long long)i0 * g.n[1] + i1) * g.n[2] + i2;
  if (to_arena) dst[k] = src[dk];
  else dst[dk] = src[k];
}

// Error ratio mask of the last step of a failed subdomain (nodes of the
// StiffnessError, integrate.py:246).  Writes 1.0 where ratio > 1 (dense box).
template <int DIM>
__global__ void __launch_bounds__(NT) k_ratio_mask(const KArgs a, double* out) {
  const int b = blockIdx.x;
  const Entry e = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[e.sub];
  int i0, i1, i2;
  if (!tile_node<DIM>(g, b - e.tile_begin, i0, i1, i2)) return;
  const long long k = lin<DIM>(g, i0, i1, i2);
  const double ds = a.F.d[e.s % 3][k];
  const double yv = a.F.y[e.yi][k];
  const double yn = a.F.y[1 - e.yi][k];
  const double err = -0.8 * ds + e.h04 * (a.F.f[e.fi][k] + a.F.f[1 - e.fi][k]);
  const double ay = fabs(yv), an = fabs(yn);
  const double mx = (ay >= an || isnan(ay)) ? ay : an;
  const double r = fabs(err) / (a.P.atol + a.P.rtol * mx);
  const long long dk = DIM == 2 ? (long long)i0 * g.n[1] + i1
                                : ((long long)i0 * g.n[1] + i1) * g.n[2] + i2;
  out[dk] = r > 1.0 ? 1.0 : 0.0;
}

__global__ void k_res_init(SubRes* r, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  r[i].emax = 0ull;
  r[i].jmin = ~0ull;
  r[i].jmax = 0ull;
  r[i].rawmax = 0ull;
  r[i].flags = 0u;
  r[i].jnan = 0u;
  r[i].sum = 0.0;
  r[i].sum2 = 0.0;
}

// Face trace copies (_apply_traces, schwarz.py:137-159) and trace packing.
__global__ void k_faces(const FaceJob* jobs, int njobs, int nnodes) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= nnodes) return;
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].node_begin <= gid) lo = mid;
    else hi = mid - 1;
  }
  const FaceJob& J = jobs[lo];
  const int local = gid - J.node_begin;
  const int t0 = local % J.ext[0];
  const int t1 = local / J.ext[0];
  if ((t0 == 0 && J.skip_lo[0]) || (t0 == J.ext[0] - 1 && J.skip_hi[0]) ||
      (t1 == 0 && J.skip_lo[1]) || (t1 == J.ext[1] - 1 && J.skip_hi[1]))
    return;
  J.dst[t0 * J.dstr[0] + t1 * J.dstr[1]] = J.src[t0 * J.sstr[0] + t1 * J.sstr[1]];
}

// max |psi_i - psi_j| over a box intersection (_overlap_gap, schwarz.py:285-304).
__global__ void k_gap(const GapJob* jobs, int njobs, int nnodes, unsigned long long* out) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (gid < nnodes) {
    int lo = 0, hi = njobs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (jobs[mid].node_begin <= gid) lo = mid;
      else hi = mid - 1;
    }
    const GapJob& J = jobs[lo];
    int l = gid - J.node_begin;
    const int t2 = l % J.ext[2];
    l /= J.ext[2];
    const int t1 = l % J.ext[1];
    const int t0 = l / J.ext[1];
    const double x = J.a[t0 * J.astr[0] + t1 * J.astr[1] + t2 * J.astr[2]];
    const double y = J.b[t0 * J.bstr[0] + t1 * J.bstr[1] + t2 * J.bstr[2]];
    v = fabs(x - y);
    if (!(v == v)) v = 0.0;
  }
  unsigned long long u = (unsigned long long)__double_as_longlong(v);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_down_sync(0xffffffffu, u, off);
    u = o > u ? o : u;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, u);
}

template <int DIM, bool P2>
void eval_dispatch(int mode, const KArgs& a, int nb, cudaStream_t st) {
  const dim3 blk(TX, TY);
  switch (mode) {
    case M_F0: k_eval<DIM, P2, M_F0><<<nb, blk, 0, st>>>(a); break;
    case M_STAGE2: k_eval<DIM, P2, M_STAGE2><<<nb, blk, 0, st>>>(a); break;
    case M_STAGE3: k_eval<DIM, P2, M_STAGE3><<<nb, blk, 0, st>>>(a); break;
    case M_STAGEN: k_eval<DIM, P2, M_STAGEN><<<nb, blk, 0, st>>>(a); break;
    case M_FINAL: k_eval<DIM, P2, M_FINAL><<<nb, blk, 0, st>>>(a); break;
    case M_POWER: k_eval<DIM, P2, M_POWER><<<nb, blk, 0, st>>>(a); break;
    case M_POWER_SEED: k_eval<DIM, P2, M_POWER_SEED><<<nb, blk, 0, st>>>(a); break;
    case M_EULER: k_eval<DIM, P2, M_EULER><<<nb, blk, 0, st>>>(a); break;
    default: break;
  }
}

}  // namespace

void launch_eval(int mode, const KArgs& a, int nb, void* stream) {
  if (nb <= 0) return;
  cudaStream_t st = (cudaStream_t)stream;
  if (a.P.dim == 2) {
    if (a.P.pow2) eval_dispatch<2, true>(mode, a, nb, st);
    else eval_dispatch<2, false>(mode, a, nb, st);
  } else {
    if (a.P.pow2) eval_dispatch<3, true>(mode, a, nb, st);
    else eval_dispatch<3, false>(mode, a, nb, st);
  }
}

void launch_sumsq(const KArgs& a, int nb, void* stream) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  if (a.P.dim == 2) k_sumsq<2><<<nb, blk, 0, (cudaStream_t)stream>>>(a);
  else k_sumsq<3><<<nb, blk, 0, (cudaStream_t)stream>>>(a);
}

void launch_finalize(const Entry* ent, int nent, const double* part, SubRes* res, int which,
                     void* stream) {
  if (nent <= 0) return;
  k_finalize<<<nent, 256, 0, (cudaStream_t)stream>>>(ent, part, res, which);
}

void launch_mesh(const KArgs& a, int nb, int with_res, void* stream) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  cudaStream_t st = (cudaStream_t)stream;
  if (a.P.dim == 2) {
    if (a.P.pow2) k_mesh<2, true><<<nb, blk, 0, st>>>(a, with_res);
    else k_mesh<2, false><<<nb, blk, 0, st>>>(a, with_res);
  } else {
    if (a.P.pow2) k_mesh<3, true><<<nb, blk, 0, st>>>(a, with_res);
    else k_mesh<3, false><<<nb, blk, 0, st>>>(a, with_res);
  }
}

void launch_prologue(const KArgs& a, int nb, double z, void* stream) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  if (a.P.dim == 2) k_prologue<2><<<nb, blk, 0, (cudaStream_t)stream>>>(a, z);
  else k_prologue<3><<<nb, blk, 0, (cudaStream_t)stream>>>(a, z);
}

void launch_res_init(SubRes* res, int n, void* stream) {
  if (n <= 0) return;
  k_res_init<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(res, n);
}

void launch_faces(const FaceJob* jobs, int njobs, int nnodes, void* stream) {
  if (njobs <= 0 || nnodes <= 0) return;
  k_faces<<<(nnodes + 255) / 256, 256, 0, (cudaStream_t)stream>>>(jobs, njobs, nnodes);
}

void launch_gap(const GapJob* jobs, int njobs, int nnodes, unsigned long long* out,
                void* stream) {
  if (njobs <= 0 || nnodes <= 0) return;
  k_gap<<<(nnodes + 255) / 256, 256, 0, (cudaStream_t)stream>>>(jobs, njobs, nnodes, out);
}

void launch_psi0(const KArgs& a, int nb, void* stream) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  if (a.P.dim == 2) k_psi0<2><<<nb, blk, 0, (cudaStream_t)stream>>>(a);
  else k_psi0<3><<<nb, blk, 0, (cudaStream_t)stream>>>(a);
}

void launch_scatter(const KArgs& a, int nb, const double* global, void* stream) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  if (a.P.dim == 2) k_scatter<2><<<nb, blk, 0, (cudaStream_t)stream>>>(a, global);
  else k_scatter<3><<<nb, blk, 0, (cudaStream_t)stream>>>(a, global);
}

void launch_assemble(const KArgs& a, int nb, double* psi, double* coords, double* jac,
                     void* stream) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  cudaStream_t st = (cudaStream_t)stream;
  if (a.P.dim == 2) {
    if (a.P.pow2) k_assemble<2, true><<<nb, blk, 0, st>>>(a, psi, coords, jac);
    else k_assemble<2, false><<<nb, blk, 0, st>>>(a, psi, coords, jac);
  } else {
    if (a.P.pow2) k_assemble<3, true><<<nb, blk, 0, st>>>(a, psi, coords, jac);
    else k_assemble<3, false><<<nb, blk, 0, st>>>(a, psi, coords, jac);
  }
}

void launch_ratio_mask(const KArgs& a, int nb, double* out, void* stream) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  if (a.P.dim == 2) k_ratio_mask<2><<<nb, blk, 0, (cudaStream_t)stream>>>(a, out);
  else k_ratio_mask<3><<<nb, blk, 0, (cudaStream_t)stream>>>(a, out);
}

void launch_box_mesh(const KArgs& a, int nb, double* coords, double* jac, double* raw,
                     void* stream) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  cudaStream_t st = (cudaStream_t)stream;
  if (a.P.dim == 2) {
    if (a.P.pow2) k_box_mesh<2, true><<<nb, blk, 0, st>>>(a, coords, jac, raw);
    else k_box_mesh<2, false><<<nb, blk, 0, st>>>(a, coords, jac, raw);
  } else {
    if (a.P.pow2) k_box_mesh<3, true><<<nb, blk, 0, st>>>(a, coords, jac, raw);
    else k_box_mesh<3, false><<<nb, blk, 0, st>>>(a, coords, jac, raw);
  }
}

void launch_box_copy(const KArgs& a, int nb, const double* src, double* dst, int to_arena,
                     void* stream) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  if (a.P.dim == 2) k_box_copy<2><<<nb, blk, 0, (cudaStream_t)stream>>>(a, src, dst, to_arena);
  else k_box_copy<3><<<nb, blk, 0, (cudaStream_t)stream>>>(a, src, dst, to_arena);
}

}  // namespace ddpma
