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
#include "stencil.cuh"

namespace ddpma {

namespace {

using namespace ddpma::dev;

// ------------------------------------------------------------- eval kernel --
// One frozen-density RHS evaluation (pma_rhs_frozen, pma.py:195-219) per node,
// fused with what consumes it in the integrator (integrate.py:163-208).  A
// launch mixes entries in different modes / stages (one subdomain each); the
// mode is uniform per CTA, so the dispatch below never diverges in a warp.
// Results go to the launch's own result slot `a.res` (per local subdomain).
template <int DIM, bool P2, int MODE>
__device__ __forceinline__ void eval_cta(const KArgs& a, const Entry& e, int b) {
  __shared__ double sh_sum[NT / 32];
  __shared__ unsigned long long sh_max[NT / 32];
  const SubGeo& g = a.geo[e.sub];
  int i0, i1, i2;
  const bool valid = tile_node<DIM>(g, b - e.tile_begin, i0, i1, i2);
  unsigned flag = 0, nonfin = 0;
  double ratio = 0.0, psum = 0.0;
  if (valid) {
    const long long k = lin<DIM>(g, i0, i1, i2);
    const double* __restrict__ yb = a.F.y[e.yi];
    if constexpr (MODE == M_NORM) {
      const double y = yb[k];
      psum = y * y;
    } else {
      const bool dir = dirichlet<DIM>(g, i0, i1, i2);
      double det;
      if constexpr (MODE == M_F0 || MODE == M_EULER) {
        det = hdet<DIM, P2>(a.P, g, i0, i1, i2, YAcc<DIM, YM_PLAIN>{&g, yb, nullptr, 0.0});
      } else if constexpr (MODE == M_STAGE2) {
        det = hdet<DIM, P2>(a.P, g, i0, i1, i2, YAcc<DIM, YM_SCALED>{&g, yb, a.F.f[e.fi], e.c});
      } else if constexpr (MODE == M_STAGE3 || MODE == M_STAGEN) {
        det = hdet<DIM, P2>(a.P, g, i0, i1, i2, YAcc<DIM, YM_ADD>{&g, yb, a.F.d[(e.j - 1) % 3], 0.0});
      } else if constexpr (MODE == M_FINAL) {
        det = hdet<DIM, P2>(a.P, g, i0, i1, i2, YAcc<DIM, YM_ADD>{&g, yb, a.F.d[e.s % 3], 0.0});
      } else if constexpr (MODE == M_POWER) {
        det = hdet<DIM, P2>(a.P, g, i0, i1, i2, YAcc<DIM, YM_SCALED>{&g, yb, a.F.d[e.vin], e.c});
      } else {
        det = hdet<DIM, P2>(a.P, g, i0, i1, i2, YAcc<DIM, YM_SEED>{&g, yb, nullptr, e.c});
      }
      const double F = dir ? 0.0 : logequi(__ldg(a.F.mr + k), det, a.P.guard, a.P.floor, a.P.rguard);
      flag = (det <= a.P.floor && !dir) ? 1u : 0u;
      if constexpr (MODE == M_F0) {
        a.F.f[e.fi][k] = F;
      } else if constexpr (MODE == M_EULER) {
        a.F.y[1 - e.yi][k] = yb[k] + e.c * F;
      } else if constexpr (MODE == M_STAGE2 || MODE == M_STAGE3 || MODE == M_STAGEN) {
        // d_j = mu_j d_{j-1} + nu_j d_{j-2} + (h mu~_j) F_j + (h gamma~_j) f0 (integrate.py:174-175)
        const double f0 = __ldg(a.F.f[e.fi] + k);
        const double d1 = e.c * f0;                 // d_1 = (h mu~_1) f0 (integrate.py:170)
        double dp, dp2;
        if constexpr (MODE == M_STAGE2) {
          dp = d1;
          dp2 = 0.0;
        } else if constexpr (MODE == M_STAGE3) {
          dp = __ldg(a.F.d[2] + k);
          dp2 = d1;
        } else {
          dp = __ldg(a.F.d[(e.j - 1) % 3] + k);
          dp2 = __ldg(a.F.d[(e.j - 2) % 3] + k);
        }
        a.F.d[e.j % 3][k] = ((e.mu * dp + e.nu * dp2) + e.hmut * F) + e.hgt * f0;
      } else if constexpr (MODE == M_FINAL) {
        const double ds = __ldg(a.F.d[e.s % 3] + k);
        const double yv = yb[k];
        const double yn = yv + ds;
        const double f0 = __ldg(a.F.f[e.fi] + k);
        a.F.f[1 - e.fi][k] = F;
        a.F.y[1 - e.yi][k] = yn;
        const double err = -0.8 * ds + e.h04 * (f0 + F);            // integrate.py:205
        const double ay = fabs(yv), an = fabs(yn);
        const double mx = (ay >= an || isnan(ay)) ? ay : an;        // np.maximum
        const double r = fabs(err) / (a.P.atol + a.P.rtol * mx);    // :206-207
        if (isfinite(r)) ratio = r;
        else nonfin = 1;
      } else {   // power iteration: diff = F(y + c v) - f0 (integrate.py:139-140)
        const double diff = F - __ldg(a.F.f[e.fi] + k);
        a.F.d[e.vout][k] = diff;
        psum = diff * diff;
      }
    }
  }
  if constexpr (MODE != M_NORM) {
    const int any = __syncthreads_or(flag);
    if constexpr (MODE == M_FINAL) {
      const int anynf = __syncthreads_or(nonfin);
      const unsigned long long m =
          block_max_u64((unsigned long long)__double_as_longlong(ratio), sh_max);
      if (threadIdx.x == 0 && threadIdx.y == 0) {
        const unsigned bits = (any ? 2u : 0u) | (anynf ? 4u : 0u);
        if (bits) atomicOr(&a.res[e.sub].flags, bits);
        atomicMax(&a.res[e.sub].emax, m);
      }
    } else {
      if (any && threadIdx.x == 0 && threadIdx.y == 0) atomicOr(&a.res[e.sub].flags, 1u);
    }
  }
  if constexpr (MODE == M_POWER || MODE == M_POWER_SEED || MODE == M_NORM) {
    const double s = block_sum(psum, sh_sum);
    if (threadIdx.x == 0 && threadIdx.y == 0) a.part[b] = s;
  }
}

template <int DIM, bool P2>
__global__ void __launch_bounds__(NT) k_eval(const KArgs a) {
  const int b = blockIdx.x;
  const Entry e = a.ent[find_entry(a.ent, a.nent, b)];
  switch (e.mode) {
    case M_F0: eval_cta<DIM, P2, M_F0>(a, e, b); break;
    case M_STAGE2: eval_cta<DIM, P2, M_STAGE2>(a, e, b); break;
    case M_STAGE3: eval_cta<DIM, P2, M_STAGE3>(a, e, b); break;
    case M_STAGEN: eval_cta<DIM, P2, M_STAGEN>(a, e, b); break;
    case M_FINAL: eval_cta<DIM, P2, M_FINAL>(a, e, b); break;
    case M_POWER: eval_cta<DIM, P2, M_POWER>(a, e, b); break;
    case M_POWER_SEED: eval_cta<DIM, P2, M_POWER_SEED>(a, e, b); break;
    case M_EULER: eval_cta<DIM, P2, M_EULER>(a, e, b); break;
    case M_NORM: eval_cta<DIM, P2, M_NORM>(a, e, b); break;
    default: break;
  }
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

// ------------------------------------------------ u-backed mesh density --
// Scratch fields of the pull-back (free between windows: the RKC ring and
// f_new are rebuilt by every window, integrate.py:184).
__device__ __forceinline__ void upull_fields(const Fields& F, double** S) {
  S[0] = F.d[0];
  S[1] = F.d[1];
  S[2] = F.d[2];
  S[3] = F.f[1];
}

// Pre-pass of mesh_density's u branch (monitor.py:170-172): the mesh
// coordinates (gradient_fd, pma.py:67-84) and u at the clamped coordinates.
template <int DIM, bool P2>
__global__ void __launch_bounds__(NT) k_upre(const KArgs a) {
  const int b = blockIdx.x;
  const Entry e = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[e.sub];
  int i0, i1, i2;
  if (!tile_node<DIM>(g, b - e.tile_begin, i0, i1, i2)) return;
  const long long k = lin<DIM>(g, i0, i1, i2);
  const YAcc<DIM, YM_PLAIN> Y{&g, a.F.y[e.yi], nullptr, 0.0};
  double* S[4];
  upull_fields(a.F, S);
  const MonitorD& M = *a.mon;
  double x[3], p[3];
#pragma unroll
  for (int q = 0; q < DIM; ++q) {
    x[q] = coord<DIM, P2>(a.P, g, q, i0, i1, i2, Y);
    S[q][k] = x[q];
    p[q] = clampv(x[q], M.lo[q], M.hi[q]);
  }
  S[DIM][k] = tf_u<DIM>(M, p);
}

// Nodal raw density: the analytic monitor at x, or the pull-back.
template <int DIM, bool P2>
__device__ __forceinline__ double node_raw(const KArgs& a, const SubGeo& g, int i0, int i1,
                                           int i2, const double* x) {
  if (a.upull) {
    double* S[4];
    upull_fields(a.F, S);
    return pull_raw<DIM, P2>(a.P, g, S, i0, i1, i2);
  }
  return mon_raw<DIM>(*a.mon, x);
}

// ----------------------------------------------------------- mesh kernel --
// physical_mesh (pma.py:222-225) + mesh_density (monitor.py:151-180) + the
// owned-node transport partial w*raw*J (schwarz.py:182-186) + the window
// residual (psi - psi_level_n)^2 * w_box (schwarz.py:111-115) + J min/max.
// Smoothing / relaxation buffers (free between windows: mr is rebuilt by the
// prologue, y[1-yi] is the integrator's candidate slot).
__device__ __forceinline__ double* dens_buf(const KArgs& a, const Entry& e, int sel) {
  return sel == 1 ? a.F.mr : a.F.y[1 - e.yi];
}

// Nodal raw density into a smoothing buffer (mesh_density before _smooth).
template <int DIM, bool P2>
__global__ void __launch_bounds__(NT) k_rawfill(const KArgs a, int dst) {
  const int b = blockIdx.x;
  const Entry e = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[e.sub];
  int i0, i1, i2;
  if (!tile_node<DIM>(g, b - e.tile_begin, i0, i1, i2)) return;
  const YAcc<DIM, YM_PLAIN> Y{&g, a.F.y[e.yi], nullptr, 0.0};
  double x[3];
#pragma unroll
  for (int q = 0; q < DIM; ++q) x[q] = coord<DIM, P2>(a.P, g, q, i0, i1, i2, Y);
  dens_buf(a, e, dst)[lin<DIM>(g, i0, i1, i2)] = node_raw<DIM, P2>(a, g, i0, i1, i2, x);
}

// One axis of monitor._smooth (monitor.py:395-409): reflected edges
// (out[1] before index 0, out[-2] after n-1), 0.25*left + 0.5*mid + 0.25*right.
template <int DIM>
__global__ void __launch_bounds__(NT) k_smooth(const KArgs a, int axis, int src, int dst) {
  const int b = blockIdx.x;
  const Entry e = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[e.sub];
  int i0, i1, i2;
  if (!tile_node<DIM>(g, b - e.tile_begin, i0, i1, i2)) return;
  const double* __restrict__ s = dens_buf(a, e, src);
  int idx[3] = {i0, i1, i2};
  const int n = g.n[axis], i = idx[axis];
  const int il = i == 0 ? 1 : i - 1, ir = i == n - 1 ? n - 2 : i + 1;
  idx[axis] = il;
  const double left = s[lin<DIM>(g, idx[0], idx[1], idx[2])];
  idx[axis] = ir;
  const double right = s[lin<DIM>(g, idx[0], idx[1], idx[2])];
  const long long k = lin<DIM>(g, i0, i1, i2);
  dens_buf(a, e, dst)[k] = (0.25 * left + 0.5 * s[k]) + 0.25 * right;
}

// src: 0 = evaluate the density here, else the smoothing buffer holding it;
// blend: (1-relax)*raw + relax*previous raw (schwarz.py:176-179).
template <int DIM, bool P2>
__global__ void __launch_bounds__(NT) k_mesh(const KArgs a, int with_res, int src, double relax,
                                             int blend) {
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
    double raw = src ? dens_buf(a, e, src)[k] : node_raw<DIM, P2>(a, g, i0, i1, i2, x);
    if (blend) raw = (1.0 - relax) * raw + relax * a.F.raw[k];
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

// Owned blocks of the local subdomains, packed for the multi-GPU gather
// (SURVEY §8(e)): subdomain l occupies out[offs[l] ..) as [psi | coords
// (interleaved) | jac] over its owned range in C order, the same values
// k_assemble writes into the global arrays (schwarz.py:271-282).
template <int DIM, bool P2>
__global__ void __launch_bounds__(NT) k_pack_owned(const KArgs a, double* out,
                                                   const long long* offs) {
  const int b = blockIdx.x;
  const Entry e = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[e.sub];
  int i0, i1, i2;
  if (!tile_node<DIM>(g, b - e.tile_begin, i0, i1, i2)) return;
  const int idx[3] = {i0, i1, i2};
  long long o = 0, on = 1;
#pragma unroll
  for (int q = 0; q < DIM; ++q) {
    if (idx[q] < g.olo[q] || idx[q] > g.ohi[q]) return;
    const long long n = g.ohi[q] - g.olo[q] + 1;
    o = o * n + (idx[q] - g.olo[q]);
    on *= n;
  }
  double* base = out + offs[e.sub];
  const double* yb = a.F.y[e.yi];
  const YAcc<DIM, YM_PLAIN> Y{&g, yb, nullptr, 0.0};
  base[o] = yb[lin<DIM>(g, i0, i1, i2)];
#pragma unroll
  for (int q = 0; q < DIM; ++q) base[on + o * DIM + q] = coord<DIM, P2>(a.P, g, q, i0, i1, i2, Y);
  base[on * (1 + DIM) + o] = hdet<DIM, P2>(a.P, g, i0, i1, i2, Y);
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
  if (raw) raw[dk] = node_raw<DIM, P2>(a, g, i0, i1, i2, x);
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

}  // namespace

void launch_eval(const KArgs& a, int nb, void* stream) {
  if (nb <= 0) return;
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 blk(TX, TY);
  if (a.P.dim == 2) {
    if (a.P.pow2) k_eval<2, true><<<nb, blk, 0, st>>>(a);
    else k_eval<2, false><<<nb, blk, 0, st>>>(a);
  } else {
    if (a.P.pow2) k_eval<3, true><<<nb, blk, 0, st>>>(a);
    else k_eval<3, false><<<nb, blk, 0, st>>>(a);
  }
}

void launch_finalize(const Entry* ent, int nent, const double* part, SubRes* res, int which,
                     void* stream) {
  if (nent <= 0) return;
  k_finalize<<<nent, 256, 0, (cudaStream_t)stream>>>(ent, part, res, which);
}

void launch_mesh(const KArgs& a, int nb, int with_res, void* stream) {
  launch_mesh_ex(a, nb, with_res, 0, 0.0, 0, stream);
}

void launch_mesh_ex(const KArgs& a, int nb, int with_res, int src, double relax, int blend,
                    void* stream) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  cudaStream_t st = (cudaStream_t)stream;
  if (a.P.dim == 2) {
    if (a.P.pow2) k_mesh<2, true><<<nb, blk, 0, st>>>(a, with_res, src, relax, blend);
    else k_mesh<2, false><<<nb, blk, 0, st>>>(a, with_res, src, relax, blend);
  } else {
    if (a.P.pow2) k_mesh<3, true><<<nb, blk, 0, st>>>(a, with_res, src, relax, blend);
    else k_mesh<3, false><<<nb, blk, 0, st>>>(a, with_res, src, relax, blend);
  }
}

void launch_rawfill(const KArgs& a, int nb, int dst, void* stream) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  cudaStream_t st = (cudaStream_t)stream;
  if (a.P.dim == 2) {
    if (a.P.pow2) k_rawfill<2, true><<<nb, blk, 0, st>>>(a, dst);
    else k_rawfill<2, false><<<nb, blk, 0, st>>>(a, dst);
  } else {
    if (a.P.pow2) k_rawfill<3, true><<<nb, blk, 0, st>>>(a, dst);
    else k_rawfill<3, false><<<nb, blk, 0, st>>>(a, dst);
  }
}

void launch_smooth(const KArgs& a, int nb, int axis, int src, int dst, void* stream) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  cudaStream_t st = (cudaStream_t)stream;
  if (a.P.dim == 2) k_smooth<2><<<nb, blk, 0, st>>>(a, axis, src, dst);
  else k_smooth<3><<<nb, blk, 0, st>>>(a, axis, src, dst);
}

void launch_upre(const KArgs& a, int nb, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 blk(TX, TY);
  if (a.P.dim == 2) {
    if (a.P.pow2) k_upre<2, true><<<nb, blk, 0, st>>>(a);
    else k_upre<2, false><<<nb, blk, 0, st>>>(a);
  } else {
    if (a.P.pow2) k_upre<3, true><<<nb, blk, 0, st>>>(a);
    else k_upre<3, false><<<nb, blk, 0, st>>>(a);
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

void launch_pack_owned(const KArgs& a, int nb, double* out, const long long* offs, void* stream) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  cudaStream_t st = (cudaStream_t)stream;
  if (a.P.dim == 2) {
    if (a.P.pow2) k_pack_owned<2, true><<<nb, blk, 0, st>>>(a, out, offs);
    else k_pack_owned<2, false><<<nb, blk, 0, st>>>(a, out, offs);
  } else {
    if (a.P.pow2) k_pack_owned<3, true><<<nb, blk, 0, st>>>(a, out, offs);
    else k_pack_owned<3, false><<<nb, blk, 0, st>>>(a, out, offs);
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

// ------------------------------------------------------------- metrics ---
// metrics.quality_measure (metrics.py:57-85) and relative_errors
// (metrics.py:100-118) on one box (the plan's single box = the whole grid).
// Per CTA fixed-order partials: QP_N doubles per block, reduced by one CTA in
// block order (deterministic).

// trapezoid weight of box node (i0,i1,i2): quadrature.weights (quadrature.py:16-21)
template <int DIM>
__device__ __forceinline__ double box_weight(const Prob& P, const SubGeo& g, int i0, int i1,
                                             int i2) {
  const int idx[3] = {i0, i1, i2};
  double w = 1.0;
#pragma unroll
  for (int q = 0; q < DIM; ++q) {
    const double wq = (idx[q] == 0 || idx[q] == g.n[q] - 1) ? P.ax[q].w_end : P.ax[q].w_in;
    w = q == 0 ? wq : w * wq;
  }
  return w;
}

constexpr int QP_N = 6;

// mode 0: z = sum (w*raw)*jac (sample_on_mesh normaliser, metrics.py:75-77)
// mode 1: e = (|Omega| * (raw / norm)) * jac; partials
//         {sum (w*e)*e, sum w, max|e| key, sum e, nonpositive jac count, NaN seen}
template <int DIM, bool P2>
__global__ void __launch_bounds__(NT) k_quality(const KArgs a, int mode, double norm,
                                                double* e_out, double* part, int src) {
  __shared__ double sh_sum[NT / 32];
  __shared__ unsigned long long sh_u[NT / 32];
  const int b = blockIdx.x;
  const Entry en = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[en.sub];
  int i0, i1, i2;
  const bool valid = tile_node<DIM>(g, b - en.tile_begin, i0, i1, i2);
  double s0 = 0.0, s1 = 0.0, s3 = 0.0, tang = 0.0, nan = 0.0;
  unsigned long long mk = 0ull;
  if (valid) {
    const YAcc<DIM, YM_PLAIN> Y{&g, a.F.y[en.yi], nullptr, 0.0};
    double x[3];
#pragma unroll
    for (int q = 0; q < DIM; ++q) x[q] = coord<DIM, P2>(a.P, g, q, i0, i1, i2, Y);
    const double jac = hdet<DIM, P2>(a.P, g, i0, i1, i2, Y);
    const double raw = src ? dens_buf(a, en, src)[lin<DIM>(g, i0, i1, i2)]
                           : node_raw<DIM, P2>(a, g, i0, i1, i2, x);
    const double w = box_weight<DIM>(a.P, g, i0, i1, i2);
    if (mode == 0) {
      s0 = (w * raw) * jac;
    } else {
      const double e = (a.P.measure * (raw / norm)) * jac;
      const long long dk = DIM == 2 ? (long long)i0 * g.n[1] + i1
                                    : ((long long)i0 * g.n[1] + i1) * g.n[2] + i2;
      e_out[dk] = e;
      s0 = (w * e) * e;
      s1 = w;
      s3 = e;
      tang = jac <= 0.0 ? 1.0 : 0.0;
      nan = isnan(e) ? 1.0 : 0.0;
      mk = okey(fabs(e));
    }
  }
  double v[5] = {s0, s1, s3, tang, nan};
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const double r = block_sum(v[q], sh_sum);
    if (threadIdx.x == 0 && threadIdx.y == 0) part[(long long)b * QP_N + q] = r;
  }
  const unsigned long long m = block_max_u64(mk, sh_u);
  if (threadIdx.x == 0 && threadIdx.y == 0)
    part[(long long)b * QP_N + 5] = __longlong_as_double((long long)m);
}

// relative_errors partials on dense box arrays: {sum w*diff, sum w*ref,
// sum (w*diff)*diff, sum (w*ref)*ref, max diff key, max ref key}
template <int DIM>
__global__ void __launch_bounds__(NT) k_relerr(const KArgs a, const double* dd, const double* sd,
                                               double* part) {
  __shared__ double sh_sum[NT / 32];
  __shared__ unsigned long long sh_u[NT / 32];
  const int b = blockIdx.x;
  const Entry en = a.ent[find_entry(a.ent, a.nent, b)];
  const SubGeo& g = a.geo[en.sub];
  int i0, i1, i2;
  const bool valid = tile_node<DIM>(g, b - en.tile_begin, i0, i1, i2);
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  unsigned long long kd = 0ull, kr = 0ull;
  if (valid) {
    const long long dk = DIM == 2 ? (long long)i0 * g.n[1] + i1
                                  : ((long long)i0 * g.n[1] + i1) * g.n[2] + i2;
    const double diff = fabs(sd[dk] - dd[dk]);   // np.abs(psi_sd - psi_dd)
    const double ref = fabs(sd[dk]);
    const double w = box_weight<DIM>(a.P, g, i0, i1, i2);
    v[0] = w * diff;
    v[1] = w * ref;
    v[2] = (w * diff) * diff;
    v[3] = (w * ref) * ref;
    kd = okey(diff);
    kr = okey(ref);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double r = block_sum(v[q], sh_sum);
    if (threadIdx.x == 0 && threadIdx.y == 0) part[(long long)b * QP_N + q] = r;
  }
  const unsigned long long m1 = block_max_u64(kd, sh_u);
  const unsigned long long m2 = block_max_u64(kr, sh_u);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    part[(long long)b * QP_N + 4] = __longlong_as_double((long long)m1);
    part[(long long)b * QP_N + 5] = __longlong_as_double((long long)m2);
  }
}

__device__ __forceinline__ double unkey(unsigned long long k) {
  const unsigned long long u = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// One CTA: columns 0..nsum-1 summed in block order, the rest max-reduced
// (ordered keys), results in out[0..QP_N-1].
__global__ void __launch_bounds__(32) k_qfinal(const double* part, int nb, int nsum, double* out) {
  const int q = threadIdx.x;
  if (q >= QP_N) return;
  if (q < nsum) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[(long long)b * QP_N + q];
    out[q] = s;
  } else {
    unsigned long long m = 0ull;
    for (int b = 0; b < nb; ++b) {
      const unsigned long long k = (unsigned long long)__double_as_longlong(part[(long long)b * QP_N + q]);
      m = k > m ? k : m;
    }
    out[q] = unkey(m);
  }
}

// normalize's probe quadrature (_trapezoid_mass monitor.py:112-120,
// quadrature.integrate :24-26): values = raw(lattice) UNclamped (the
// descriptor's clamp box is opened to +-inf by the host), w = tensor product
// of the 1D trapezoid weights in axis order; partials {sum raw*w, #bad, -, -,
// -, max raw key}.
template <int DIM>
__global__ void __launch_bounds__(NT) k_mass(const MonitorD* __restrict__ mon, const MassArgs m,
                                             double* part) {
  __shared__ double sh_sum[NT / 32];
  __shared__ unsigned long long sh_u[NT / 32];
  const long long q = (long long)blockIdx.x * NT + threadIdx.y * TX + threadIdx.x;
  double v = 0.0, bad = 0.0;
  unsigned long long mk = 0ull;
  if (q < m.nodes) {
    int idx[3];
    long long r = q;
#pragma unroll
    for (int k = DIM - 1; k >= 0; --k) {
      idx[k] = (int)(r % m.n[k]);
      r /= m.n[k];
    }
    double x[3], w = 1.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      x[k] = m.a[k] + (double)idx[k] * m.step[k];                // probe_axes (:107-109)
      const double wk = (idx[k] == 0 || idx[k] == m.n[k] - 1) ? m.w_end[k] : m.w_in[k];
      w = k == 0 ? wk : w * wk;                                    // np.multiply.outer order
    }
    const double raw = mon_raw<DIM>(*mon, x);
    v = raw * w;
    bad = (!isfinite(raw) || raw <= 0.0) ? 1.0 : 0.0;
    mk = okey(raw);
  }
  const double vs = block_sum(v, sh_sum);
  const double bs = block_sum(bad, sh_sum);
  const unsigned long long mx = block_max_u64(mk, sh_u);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    double* o = part + (long long)blockIdx.x * QP_N;
    o[0] = vs;
    o[1] = bs;
    o[2] = o[3] = o[4] = 0.0;
    o[5] = __longlong_as_double((long long)mx);
  }
}

void launch_mass(const MonitorD* mon, const MassArgs& m, int nb, double* part, double* out,
                 void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 blk(TX, TY);
  if (m.dim == 2) k_mass<2><<<nb, blk, 0, st>>>(mon, m, part);
  else k_mass<3><<<nb, blk, 0, st>>>(mon, m, part);
  k_qfinal<<<1, 32, 0, st>>>(part, nb, 5, out);
}

void launch_quality(const KArgs& a, int nb, int mode, double norm, double* e_out, double* part,
                    double* out, void* stream, int src) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  cudaStream_t st = (cudaStream_t)stream;
  if (a.P.dim == 2) {
    if (a.P.pow2) k_quality<2, true><<<nb, blk, 0, st>>>(a, mode, norm, e_out, part, src);
    else k_quality<2, false><<<nb, blk, 0, st>>>(a, mode, norm, e_out, part, src);
  } else {
    if (a.P.pow2) k_quality<3, true><<<nb, blk, 0, st>>>(a, mode, norm, e_out, part, src);
    else k_quality<3, false><<<nb, blk, 0, st>>>(a, mode, norm, e_out, part, src);
  }
  k_qfinal<<<1, 32, 0, st>>>(part, nb, 5, out);
}

void launch_relerr(const KArgs& a, int nb, const double* dd, const double* sd, double* part,
                   double* out, void* stream) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  cudaStream_t st = (cudaStream_t)stream;
  if (a.P.dim == 2) k_relerr<2><<<nb, blk, 0, st>>>(a, dd, sd, part);
  else k_relerr<3><<<nb, blk, 0, st>>>(a, dd, sd, part);
  k_qfinal<<<1, 32, 0, st>>>(part, nb, 4, out);
}

void launch_box_copy(const KArgs& a, int nb, const double* src, double* dst, int to_arena,
                     void* stream) {
  if (nb <= 0) return;
  const dim3 blk(TX, TY);
  if (a.P.dim == 2) k_box_copy<2><<<nb, blk, 0, (cudaStream_t)stream>>>(a, src, dst, to_arena);
  else k_box_copy<3><<<nb, blk, 0, (cudaStream_t)stream>>>(a, src, dst, to_arena);
}

}  // namespace ddpma
