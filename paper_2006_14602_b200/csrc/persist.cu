// Persistent, device-resident window kernel (sm_100a).
//
// One cooperative launch integrates one pseudo-time window for every active
// local subdomain.  Each subdomain runs its own Rkc2Integrator/Euler state
// machine (integrate.py:109-250) ON THE DEVICE: its current *action* (f0
// evaluation, a power-iteration evaluation, RKC2 stage j, the final
// evaluation with the error ratio, an Euler substep, ||y||) is a pass over
// all work items (tiles) of its box.  CTAs pull items from any subdomain
// whose action has unclaimed items (work conserving: a subdomain that needs
// thousands of stages keeps the whole GPU busy while others are done); the
// CTA that completes an action's last item reduces its partial sums in a
// fixed order (deterministic), runs the controller decision on one thread
// and publishes the next action.
//
// Memory ordering: item stores -> __threadfence -> atomicAdd(done); the
// completing CTA fences before reading partials / controller state (all via
// L1-bypassing loads).  Publishing writes the action, fences, then swaps the
// (sequence, cursor) word; a claimer's atomicAdd on that word + fence makes
// the action and all data of the previous action visible.  Mutable fields are
// therefore never read through the non-coherent (__ldg) path in this kernel.

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cmath>
#include <type_traits>

#include "ddpma_internal.h"
#include "stencil.cuh"

#ifndef DDPMA_MINB2
#define DDPMA_MINB2 4   // resident CTAs per SM of the 2D window kernel (register cap)
#endif

namespace ddpma {

namespace {

using namespace ddpma::dev;

// Phases of the device controller (same meaning as the host Ctl in plan.cu).
enum { P_IDLE = 0, P_F0, P_SIG_NORM, P_SIG_ITER, P_STEP, P_EULER, P_DONE, P_FAILED };
enum { R_START = 0, R_ACCEPT, R_REJECT };

constexpr double kSqrtEps = 1.4901161193847656e-08;   // np.sqrt(np.finfo(float).eps)
constexpr double kStab = 0.653;                       // integrate.py:36
constexpr double kMinStep = 1e-14;                    // integrate.py:37
// Low half of a finished subdomain's synchronisation word.  Far from 2^32 so
// that stray claim increments (a claimer that scanned the word before the
// publish) can never carry into the sequence half and make it claimable.
constexpr unsigned long long kDoneLow = 0x80000000ull;

// Shared-memory copy of the log table (filled at the start of k_windowP;
// the table lookups are the fp64 log's only memory accesses).
__shared__ double s_logtab[97][3];

// coherent (L2) loads of mutable data
__device__ __forceinline__ double ldc(const double* p) { return __ldcg(p); }

// ------------------------------------------------------------- accessors --

template <int DIM, int YM>
struct GAcc {   // Y from global memory (boundary nodes), coherent loads
  const SubGeo* g;
  const double* y;
  const double* a;
  double c;
  __device__ __forceinline__ double operator()(int i0, int i1, int i2) const {
    const long long k = lin<DIM>(*g, i0, i1, i2);
    const double yv = ldc(y + k);
    if constexpr (YM == YM_PLAIN) {
      return yv;
    } else if constexpr (YM == YM_ADD) {
      return yv + ldc(a + k);
    } else if constexpr (YM == YM_SCALED) {
      return yv + c * ldc(a + k);
    } else {
      const int par = (i0 + i1 + (DIM == 3 ? i2 : 0)) & 1;
      return yv + (par ? -c : c);
    }
  }
};

struct SAcc2 {   // 2D smem tile with a 1-node halo
  const double* s;
  int r0, c0;
  __device__ __forceinline__ double operator()(int i0, int i1, int) const {
    return s[(i0 - r0 + 1) * (TX + 2) + (i1 - c0 + 1)];
  }
};

struct SAcc3 {   // 3D smem tile with a 1-node halo
  const double* s;
  int z0, r0, c0;
  __device__ __forceinline__ double operator()(int i0, int i1, int i2) const {
    return s[((i0 - z0 + 1) * (TY + 2) + (i1 - r0 + 1)) * (TX + 2) + (i2 - c0 + 1)];
  }
};

struct Act {      // the action of the claimed item (broadcast through smem)
  int mode, j, s, yi, fi, vin, vout, sub;
  double c, h04, mu, nu, hmut, hgt;
};

struct Acc {      // per-thread accumulators over the thread's nodes
  unsigned flag, nonfin;
  double ratio, psum;
};

template <int YM>
__device__ __forceinline__ double ymake(double yv, double av, double c, int par) {
  if constexpr (YM == YM_PLAIN) {
    return yv;
  } else if constexpr (YM == YM_ADD) {
    return yv + av;
  } else if constexpr (YM == YM_SCALED) {
    return yv + c * av;
  } else {
    return yv + (par ? -c : c);
  }
}

// One node: RHS (pma_rhs_frozen) + the consuming epilogue of the action.
template <int DIM, bool P2, int MODE, int YM, class SA>
__device__ __forceinline__ void node(const WinArgs& A, const SubGeo& g, const Act& t, int i0,
                                     int i1, int i2, const SA& S, const double* aptr, Acc& acc) {
  const long long k = lin<DIM>(g, i0, i1, i2);
  const double* yb = A.F.y[t.yi];
  if constexpr (MODE == M_NORM) {
    const double y = ldc(yb + k);
    acc.psum += y * y;
    return;
  } else {
    const bool dir = dirichlet<DIM>(g, i0, i1, i2);
    bool interior = i0 >= 1 && i0 <= g.n[0] - 2 && i1 >= 1 && i1 <= g.n[1] - 2;
    if constexpr (DIM == 3) interior = interior && i2 >= 1 && i2 <= g.n[2] - 2;
    double det;
    if (interior) det = hdet<DIM, P2>(A.P, g, i0, i1, i2, S);
    else det = hdet<DIM, P2>(A.P, g, i0, i1, i2, GAcc<DIM, YM>{&g, yb, aptr, t.c});
    const double F = dir ? 0.0 : logequi(ldc(A.F.mr + k), det, A.P.guard, A.P.floor, A.P.rguard);
    acc.flag |= (det <= A.P.floor && !dir) ? 1u : 0u;
    if constexpr (MODE == M_F0) {
      A.F.f[t.fi][k] = F;
    } else if constexpr (MODE == M_EULER) {
      A.F.y[1 - t.yi][k] = ldc(yb + k) + t.c * F;
    } else if constexpr (MODE == M_STAGE2 || MODE == M_STAGE3 || MODE == M_STAGEN) {
      const double f0 = ldc(A.F.f[t.fi] + k);
      const double d1 = t.c * f0;
      double dp, dp2;
      if constexpr (MODE == M_STAGE2) {
        dp = d1;
        dp2 = 0.0;
      } else if constexpr (MODE == M_STAGE3) {
        dp = ldc(A.F.d[2] + k);
        dp2 = d1;
      } else {
        dp = ldc(A.F.d[(t.j - 1) % 3] + k);
        dp2 = ldc(A.F.d[(t.j - 2) % 3] + k);
      }
      A.F.d[t.j % 3][k] = ((t.mu * dp + t.nu * dp2) + t.hmut * F) + t.hgt * f0;
    } else if constexpr (MODE == M_FINAL) {
      const double ds = ldc(A.F.d[t.s % 3] + k);
      const double yv = ldc(yb + k);
      const double yn = yv + ds;
      const double f0 = ldc(A.F.f[t.fi] + k);
      A.F.f[1 - t.fi][k] = F;
      A.F.y[1 - t.yi][k] = yn;
      const double err = -0.8 * ds + t.h04 * (f0 + F);
      const double ay = fabs(yv), an = fabs(yn);
      const double mx = (ay >= an || isnan(ay)) ? ay : an;
      const double r = fabs(err) / (A.P.atol + A.P.rtol * mx);
      if (isfinite(r)) acc.ratio = r > acc.ratio ? r : acc.ratio;
      else acc.nonfin = 1;
    } else {
      const double diff = F - ldc(A.F.f[t.fi] + k);
      A.F.d[t.vout][k] = diff;
      acc.psum += diff * diff;
    }
  }
}

// Interior 2D Hessian determinant straight from the smem tile: the interior
// formulas of hessian_det_fd (pma.py:87-140, np.gradient interior) in the
// same evaluation order as hdet's interior branch (bitwise identical).
template <bool P2>
__device__ __forceinline__ double hdet2_fast(const Prob& P, const double* p) {
  constexpr int W = TX + 2;
  const double c = p[0];
  const double h00 = dv<P2>((p[W] - 2.0 * c) + p[-W], P.ax[0].hh, P.ax[0].ihh);
  const double h11 = dv<P2>((p[1] - 2.0 * c) + p[-1], P.ax[1].hh, P.ax[1].ihh);
  const double gp = dv<P2>(p[W + 1] - p[W - 1], P.ax[1].twoh, P.ax[1].itwoh);
  const double gm = dv<P2>(p[-W + 1] - p[-W - 1], P.ax[1].twoh, P.ax[1].itwoh);
  const double h01 = dv<P2>(gp - gm, P.ax[0].twoh, P.ax[0].itwoh);
  return h00 * h11 - h01 * h01;
}

// One 2D work item: TX x IR2 nodes, each thread IR2/TY rows.  Center values
// are prefetched first, then the tile + halo of Y is staged in smem, then the
// nodes are evaluated (interior: smem stencil; box faces: generic path).
template <bool P2, int MODE, int YM>
__device__ void item2(const WinArgs& A, const SubGeo& g, const Act& t, int item, double* sY,
                      Acc& acc) {
  constexpr int W = TX + 2, H = IR2 + 2, R = IR2 / TY;
  const int ix = item % g.items_x, iy = item / g.items_x;
  const int c0 = ix * TX, r0 = iy * IR2;
  const int n0 = g.n[0], n1 = g.n[1];
  const double* yb = A.F.y[t.yi];
  const double* ap = nullptr;
  if constexpr (MODE == M_STAGE2) ap = A.F.f[t.fi];
  if constexpr (MODE == M_STAGE3 || MODE == M_STAGEN) ap = A.F.d[(t.j - 1) % 3];
  if constexpr (MODE == M_FINAL) ap = A.F.d[t.s % 3];
  if constexpr (MODE == M_POWER) ap = A.F.d[t.vin];
  constexpr bool NEED_F0 = MODE == M_STAGE2 || MODE == M_STAGE3 || MODE == M_STAGEN ||
                           MODE == M_FINAL || MODE == M_POWER || MODE == M_POWER_SEED;
  constexpr bool NEED_Y = MODE == M_FINAL || MODE == M_EULER || MODE == M_NORM;
  const int tid = threadIdx.y * TX + threadIdx.x;
  const int i1 = c0 + threadIdx.x;
  double cm[R], cf[R], cd[R], cd2[R], cy[R];
  bool ok[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int i0 = r0 + threadIdx.y + q * TY;
    ok[q] = i1 < n1 && i0 < n0;
    cm[q] = cf[q] = cd[q] = cd2[q] = cy[q] = 0.0;
    if (ok[q]) {
      const long long k = g.off + (long long)i0 * g.pitch + i1;
      if constexpr (MODE != M_NORM) cm[q] = ldc(A.F.mr + k);
      if constexpr (NEED_F0) cf[q] = ldc(A.F.f[t.fi] + k);
      if constexpr (MODE == M_STAGE3) cd[q] = ldc(A.F.d[2] + k);
      if constexpr (MODE == M_STAGEN) {
        cd[q] = ldc(A.F.d[(t.j - 1) % 3] + k);
        cd2[q] = ldc(A.F.d[(t.j - 2) % 3] + k);
      }
      if constexpr (MODE == M_FINAL) cd[q] = ldc(A.F.d[t.s % 3] + k);
      if constexpr (NEED_Y) cy[q] = ldc(yb + k);
    }
  }
  if constexpr (MODE != M_NORM) {
#pragma unroll
    for (int it = 0; it < (W * H + NT - 1) / NT; ++it) {
      const int e = tid + it * NT;
      if (e < W * H) {
        const int rr = e / W, cc = e - rr * W;
        const int i0 = r0 - 1 + rr, j1 = c0 - 1 + cc;
        double v = 0.0;
        if (i0 >= 0 && i0 < n0 && j1 >= 0 && j1 < n1) {
          const long long k = g.off + (long long)i0 * g.pitch + j1;
          const double av = (YM == YM_ADD || YM == YM_SCALED) ? ldc(ap + k) : 0.0;
          v = ymake<YM>(ldc(yb + k), av, t.c, (i0 + j1) & 1);
        }
        sY[e] = v;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < R; ++q) {
    if (!ok[q]) continue;
    const int i0 = r0 + threadIdx.y + q * TY;
    const long long k = g.off + (long long)i0 * g.pitch + i1;
    if constexpr (MODE == M_NORM) {
      acc.psum += cy[q] * cy[q];
    } else {
      const bool dir = dirichlet<2>(g, i0, i1, 0);
      const bool interior = i0 >= 1 && i0 <= n0 - 2 && i1 >= 1 && i1 <= n1 - 2;
      double det;
      if (interior) det = hdet2_fast<P2>(A.P, sY + (threadIdx.y + q * TY + 1) * W + threadIdx.x + 1);
      else det = hdet<2, P2>(A.P, g, i0, i1, 0, GAcc<2, YM>{&g, yb, ap, t.c});
      const double F = dir ? 0.0 : logequi(cm[q], det, A.P.guard, A.P.floor, A.P.rguard);
      acc.flag |= (det <= A.P.floor && !dir) ? 1u : 0u;
      if constexpr (MODE == M_F0) {
        A.F.f[t.fi][k] = F;
      } else if constexpr (MODE == M_EULER) {
        A.F.y[1 - t.yi][k] = cy[q] + t.c * F;
      } else if constexpr (MODE == M_STAGE2 || MODE == M_STAGE3 || MODE == M_STAGEN) {
        const double f0 = cf[q];
        const double d1 = t.c * f0;
        double dp, dp2;
        if constexpr (MODE == M_STAGE2) {
          dp = d1;
          dp2 = 0.0;
        } else if constexpr (MODE == M_STAGE3) {
          dp = cd[q];
          dp2 = d1;
        } else {
          dp = cd[q];
          dp2 = cd2[q];
        }
        A.F.d[t.j % 3][k] = ((t.mu * dp + t.nu * dp2) + t.hmut * F) + t.hgt * f0;
      } else if constexpr (MODE == M_FINAL) {
        const double ds = cd[q], yv = cy[q], f0 = cf[q];
        const double yn = yv + ds;
        A.F.f[1 - t.fi][k] = F;
        A.F.y[1 - t.yi][k] = yn;
        const double err = -0.8 * ds + t.h04 * (f0 + F);
        const double ay = fabs(yv), an = fabs(yn);
        const double mx = (ay >= an || isnan(ay)) ? ay : an;
        const double r = fabs(err) / (A.P.atol + A.P.rtol * mx);
        if (isfinite(r)) acc.ratio = r > acc.ratio ? r : acc.ratio;
        else acc.nonfin = 1;
      } else {
        const double diff = F - cf[q];
        A.F.d[t.vout][k] = diff;
        acc.psum += diff * diff;
      }
    }
  }
}

// One 3D work item: TX x TY x IZ3 nodes; tile + halo staged in smem.
template <bool P2, int MODE, int YM>
__device__ void item3(const WinArgs& A, const SubGeo& g, const Act& t, int item, double* sY,
                      Acc& acc) {
  const int ix = item % g.items_x;
  const int r = item / g.items_x;
  const int iy = r % g.items_y, iz = r / g.items_y;
  const int c0 = ix * TX, r0 = iy * TY, z0 = iz * IZ3;
  const double* yb = A.F.y[t.yi];
  const double* ap = nullptr;
  if constexpr (MODE == M_STAGE2) ap = A.F.f[t.fi];
  if constexpr (MODE == M_STAGE3 || MODE == M_STAGEN) ap = A.F.d[(t.j - 1) % 3];
  if constexpr (MODE == M_FINAL) ap = A.F.d[t.s % 3];
  if constexpr (MODE == M_POWER) ap = A.F.d[t.vin];
  const int tid = threadIdx.y * TX + threadIdx.x;
  if constexpr (MODE != M_NORM) {
    constexpr int W = TX + 2, H = TY + 2, D = IZ3 + 2;
    for (int e = tid; e < W * H * D; e += NT) {
      const int cc = e % W, rr = (e / W) % H, zz = e / (W * H);
      const int i0 = z0 - 1 + zz, i1 = r0 - 1 + rr, i2 = c0 - 1 + cc;
      double v = 0.0;
      if (i0 >= 0 && i0 < g.n[0] && i1 >= 0 && i1 < g.n[1] && i2 >= 0 && i2 < g.n[2]) {
        const long long k = g.off + ((long long)i0 * g.n[1] + i1) * g.pitch + i2;
        const double av = (YM == YM_ADD || YM == YM_SCALED) ? ldc(ap + k) : 0.0;
        v = ymake<YM>(ldc(yb + k), av, t.c, (i0 + i1 + i2) & 1);
      }
      sY[e] = v;
    }
    __syncthreads();
  }
  const SAcc3 S{sY, z0, r0, c0};
  const int i2 = c0 + threadIdx.x, i1 = r0 + threadIdx.y;
  if (i1 < g.n[1] && i2 < g.n[2]) {
    for (int q = 0; q < IZ3; ++q) {
      const int i0 = z0 + q;
      if (i0 < g.n[0]) node<3, P2, MODE, YM>(A, g, t, i0, i1, i2, S, ap, acc);
    }
  }
}

template <int DIM, bool P2, int MODE, int YM>
__device__ __forceinline__ void run_item(const WinArgs& A, const SubGeo& g, const Act& t, int item,
                                         double* sY, Acc& acc) {
  if constexpr (DIM == 2) item2<P2, MODE, YM>(A, g, t, item, sY, acc);
  else item3<P2, MODE, YM>(A, g, t, item, sY, acc);
}

template <int DIM, bool P2>
__device__ void dispatch_item(const WinArgs& A, const SubGeo& g, const Act& t, int item,
                              double* sY, Acc& acc) {
  switch (t.mode) {
    case M_F0: run_item<DIM, P2, M_F0, YM_PLAIN>(A, g, t, item, sY, acc); break;
    case M_EULER: run_item<DIM, P2, M_EULER, YM_PLAIN>(A, g, t, item, sY, acc); break;
    case M_STAGE2: run_item<DIM, P2, M_STAGE2, YM_SCALED>(A, g, t, item, sY, acc); break;
    case M_STAGE3: run_item<DIM, P2, M_STAGE3, YM_ADD>(A, g, t, item, sY, acc); break;
    case M_STAGEN: run_item<DIM, P2, M_STAGEN, YM_ADD>(A, g, t, item, sY, acc); break;
    case M_FINAL: run_item<DIM, P2, M_FINAL, YM_ADD>(A, g, t, item, sY, acc); break;
    case M_POWER: run_item<DIM, P2, M_POWER, YM_SCALED>(A, g, t, item, sY, acc); break;
    case M_POWER_SEED: run_item<DIM, P2, M_POWER_SEED, YM_SEED>(A, g, t, item, sY, acc); break;
    case M_NORM: run_item<DIM, P2, M_NORM, YM_PLAIN>(A, g, t, item, sY, acc); break;
    default: break;
  }
}

__device__ __forceinline__ double mode_bytes_d(int mode) {
  switch (mode) {
    case M_F0: return 24.0;
    case M_STAGE2: return 32.0;
    case M_STAGE3: return 40.0;
    case M_STAGEN: return 48.0;
    case M_FINAL: return 48.0;
    case M_POWER: return 40.0;
    case M_POWER_SEED: return 32.0;
    case M_EULER: return 24.0;
    case M_NORM: return 8.0;
    default: return 0.0;
  }
}

// ------------------------------------------------- device controller --------
// Runs on ONE thread (thread 0 of the CTA completing an action) on a private
// copy of the subdomain's DevCtl.  Statement for statement the host Ctl logic
// of plan.cu, i.e. integrate.py:180-250.

__device__ void trace_rec(const WinArgs& A, int gid, int kind, double h, int s, double v, int fl,
                          int acc) {
  if (A.trace == nullptr) return;
  const unsigned i = atomicAdd(A.trace_n, 1u);
  if ((int)i < A.trace_cap) A.trace[i] = TraceRec{gid, kind, s, fl, acc, 0, h, v};
}

__device__ void d_loop_check(const WinArgs& A, DevCtl& c);

__device__ void d_fail(DevCtl& c, int status) {
  c.phase = P_FAILED;
  c.fail_status = status;
  c.fail_t = c.t;
  c.fail_h = c.h;
  c.fail_s = c.s;
  c.fail_yi = c.yi;
  c.fail_fi = c.fi;
  c.fail_h04 = 0.4 * c.h;
}

__device__ void d_prepare_step(const WinArgs& A, DevCtl& c) {   // integrate.py:198-202
  const double total = A.dtau;
  const int ms = A.max_stages;
  const double rem = total - c.t;
  c.h = rem < c.h ? rem : c.h;
  const double cap = kStab * (double)((long long)ms * ms);
  if (c.sigma > 0.0 && c.h * c.sigma > cap) c.h = cap / c.sigma;
  const double hs = c.h * c.sigma;
  long long s;
  if (hs <= 0.0) {
    s = 2;
  } else {
    const double v = ceil(sqrt(1.05 * hs / kStab));
    if (isnan(v)) {
      d_fail(c, DDPMA_ERR_VALUE_D);
      return;
    }
    if (isinf(v)) {
      d_fail(c, DDPMA_ERR_OVERFLOW_D);
      return;
    }
    s = v > 1e9 ? 1000000000LL : (long long)v;
    s = s < 2 ? 2 : s;
  }
  c.s = (int)(s < ms ? s : ms);
  c.j = 0;
  c.phase = P_STEP;
}

__device__ void d_after_start(const WinArgs& A, DevCtl& c) {    // integrate.py:187-196
  const double total = A.dtau;
  double h;
  if (c.sigma <= 0.0) {
    h = total;
  } else {
    const double lo = 10.0 * kMinStep * total, q = 0.25 / c.sigma;
    const double mx = lo < q ? q : lo;           // max(lo, q)
    h = mx < total ? mx : total;                 // min(total, .)
  }
  if (c.has_h) h = c.h_last < total ? c.h_last : total;
  c.h = h;
  c.t = 0.0;
  c.state_flag = c.start_flag;
  c.rej_row = 0;
  c.flag_rej = 0;
  d_loop_check(A, c);
}

__device__ void d_loop_check(const WinArgs& A, DevCtl& c) {     // integrate.py:197
  if (c.t < A.dtau * (1.0 - 1e-13)) d_prepare_step(A, c);
  else c.phase = P_DONE;
}

__device__ void d_finish_sigma(const WinArgs& A, DevCtl& c, int gid) {   // :147-153
  c.since = 0;
  if (c.has_sigma && c.sig <= 1.05 * c.sigma / 1.2) c.interval = 2 * c.interval < 500 ? 2 * c.interval : 500;
  else c.interval = 25;
  c.sigma = 1.2 * c.sig;
  c.has_sigma = 1;
  trace_rec(A, gid, 1, 0.0, 0, c.sigma, 0, 0);
  if (c.ret == R_START) d_after_start(A, c);
  else d_loop_check(A, c);
}

__device__ void d_start_sigma(DevCtl& c, int ret) {
  c.ret = ret;
  c.phase = P_SIG_NORM;
}

// The action `a_mode` of this subdomain has completed; decide.
__device__ void d_complete(const WinArgs& A, DevCtl& c, int l, double sum, long long nodes) {
  const double total = A.dtau;
  const int gid = A.geo[l].gid;
  const int mode = c.a_mode;
  c.bytes += mode_bytes_d(mode) * (double)nodes;
  if (mode != M_NORM) c.evals += 1;
  switch (mode) {
    case M_STAGE2:
    case M_STAGE3:
    case M_STAGEN:
      c.step_flag |= (c.acc_flags & 1u) ? 1 : 0;
      c.j += 1;
      break;
    case M_F0:
      c.start_flag = (c.acc_flags & 1u) ? 1 : 0;
      if (!c.has_sigma || c.since >= c.interval) d_start_sigma(c, R_START);
      else d_after_start(A, c);
      break;
    case M_NORM: {                              // integrate.py:132-133
      c.delta = kSqrtEps * (1.0 + sqrt(sum));
      c.sig = 0.0;
      c.sig_k = 0;
      c.vin = -1;
      c.vnorm = sqrt((double)nodes);
      if (c.vnorm == 0.0) d_finish_sigma(A, c, gid);
      else c.phase = P_SIG_ITER;
      break;
    }
    case M_POWER:
    case M_POWER_SEED: {                        // integrate.py:135-146
      const double nrm = sqrt(sum);
      const double ns = nrm / c.delta;
      c.vin = c.vout;
      c.sig_k += 1;
      if (c.sig > 0.0 && fabs(ns - c.sig) <= 0.01 * ns) {
        c.sig = ns;
        d_finish_sigma(A, c, gid);
        break;
      }
      c.sig = ns;
      if (c.sig_k >= 20) {
        d_finish_sigma(A, c, gid);
        break;
      }
      c.vnorm = nrm;
      if (c.vnorm == 0.0) d_finish_sigma(A, c, gid);
      break;
    }
    case M_FINAL: {                             // integrate.py:203-249
      const bool nonfin = (c.acc_flags & 4u) != 0;
      const bool flagged = c.step_flag || (c.acc_flags & 3u) != 0;
      const bool end_flag = (c.acc_flags & 2u) != 0;
      const double emax = __longlong_as_double((long long)c.acc_emax);
      const bool flag_fail = flagged && !c.state_flag && c.flag_rej < 8;
      const bool bad = flag_fail || nonfin;
      const bool ok = !bad && emax <= 1.0;
      trace_rec(A, gid, 0, c.h, c.s, nonfin ? __longlong_as_double(0x7ff8000000000000LL) : emax,
                flagged ? 1 : 0, ok ? 1 : 0);
      c.j = 0;
      if (ok) {
        c.t += c.h;
        c.yi ^= 1;
        c.fi ^= 1;
        c.state_flag = end_flag ? 1 : 0;
        c.since += 1;
        c.rej_row = 0;
        const bool need = c.since >= c.interval && c.t < total;
        double grow = 5.0;
        if (emax != 0.0) {
          const double gg = 0.8 * pow(emax, -1.0 / 3.0);
          grow = gg < 5.0 ? gg : 5.0;
        }
        c.h = c.h * (0.1 < grow ? grow : 0.1);
        c.h_last = c.h;
        c.has_h = 1;
        if (need) d_start_sigma(c, R_ACCEPT);
        else d_loop_check(A, c);
      } else {
        if (flag_fail) {
          c.flag_rej += 1;
          c.h *= 0.5;
        } else if (nonfin) {
          c.h *= 0.5;
          c.rej_row += 1;
        } else {
          const double gg = 0.8 * pow(emax, -1.0 / 3.0);
          c.h *= (0.1 < gg ? gg : 0.1);
          c.rej_row += 1;
        }
        const bool need = c.rej_row >= 2;
        if (need) c.rej_row = 0;
        if (c.h < kMinStep * total || c.flag_rej + c.rej_row > 60) {
          d_fail(c, DDPMA_ERR_STIFFNESS_D);
          c.fail_nonfin = nonfin ? 1 : 0;
          break;
        }
        if (need) d_start_sigma(c, R_REJECT);
        else d_loop_check(A, c);
      }
      break;
    }
    case M_EULER:                               // integrate.py:69-74
      c.yi ^= 1;
      if (--c.euler_left == 0) c.phase = P_DONE;
      break;
    default:
      break;
  }
}

// Fill the action fields from the phase (the next action of the subdomain).
// Returns false when the subdomain has finished (DONE / FAILED).
__device__ bool d_next_action(const WinArgs& A, DevCtl& c) {
  c.a_yi = c.yi;
  c.a_fi = c.fi;
  c.a_s = c.s;
  switch (c.phase) {
    case P_F0:
      c.a_mode = M_F0;
      return true;
    case P_SIG_NORM:
      c.a_mode = M_NORM;
      return true;
    case P_SIG_ITER:
      c.a_mode = c.vin < 0 ? M_POWER_SEED : M_POWER;
      c.a_vin = c.vin;
      c.vout = c.vin < 0 ? 0 : 1 - c.vin;
      c.a_vout = c.vout;
      c.a_c = c.delta / c.vnorm;
      return true;
    case P_STEP: {
      if (c.j == 0) {
        c.j = 2;
        c.step_flag = 0;
      }
      const int base = A.coef_off[c.s];
      c.a_c = c.h * A.coef[4 * base + 0];      // h * mu1_t
      if (c.j <= c.s) {
        const int j = c.j;
        c.a_mode = j == 2 ? M_STAGE2 : (j == 3 ? M_STAGE3 : M_STAGEN);
        c.a_j = j;
        c.a_mu = A.coef[4 * (base + j) + 0];
        c.a_nu = A.coef[4 * (base + j) + 1];
        c.a_hmut = c.h * A.coef[4 * (base + j) + 2];
        c.a_hgt = c.h * A.coef[4 * (base + j) + 3];
      } else {
        c.a_mode = M_FINAL;
        c.a_h04 = 0.4 * c.h;
      }
      return true;
    }
    case P_EULER:
      c.a_mode = M_EULER;
      c.a_c = A.dtau / (double)A.substeps;
      return true;
    default:
      return false;
  }
}

__device__ __forceinline__ void ctl_load(DevCtl& dst, const DevCtl* src) {
  long long* d = reinterpret_cast<long long*>(&dst);
  const long long* s = reinterpret_cast<const long long*>(src);
#pragma unroll 4
  for (int i = 0; i < (int)(sizeof(DevCtl) / 8); ++i) d[i] = __ldcg(s + i);
}

__device__ __forceinline__ void ctl_store(DevCtl* dst, const DevCtl& src) {
  long long* d = reinterpret_cast<long long*>(dst);
  const long long* s = reinterpret_cast<const long long*>(&src);
  // never overwrite the synchronisation word here (published separately)
  const int wi = (int)(offsetof(DevCtl, word) / 8);
#pragma unroll 4
  for (int i = 0; i < (int)(sizeof(DevCtl) / 8); ++i)
    if (i != wi) __stcg(d + i, s[i]);
}

// Publish the next action of subdomain l from the private copy c (thread 0).
__device__ void d_publish(const WinArgs& A, DevCtl& c, DevCtl* gc) {
  const unsigned long long seq = (c.word >> 32) + 1;
  const bool more = d_next_action(A, c);
  c.acc_flags = 0;
  c.acc_emax = 0ull;
  c.done = 0;
  ctl_store(gc, c);
  __threadfence();
  if (more) {
    atomicExch(&gc->word, seq << 32);
  } else {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    __stcg(reinterpret_cast<long long*>(&gc->t_done), (long long)now);
    atomicExch(&gc->word, (seq << 32) | kDoneLow);
    atomicAdd(A.n_done, 1u);
  }
}

__device__ __forceinline__ double block_sum2(double v, double* sh) {
  return block_sum(v, sh);
}

template <int DIM, bool P2>
__global__ void __launch_bounds__(NT, DIM == 2 ? 4 : 2) k_window(const WinArgs A) {
  constexpr int SM_ELEMS = DIM == 2 ? (TX + 2) * (IR2 + 2) : (TX + 2) * (TY + 2) * (IZ3 + 2);
  __shared__ double sY[SM_ELEMS];
  __shared__ double sh_sum[NT / 32];
  __shared__ unsigned long long sh_max[NT / 32];
  __shared__ Act s_act;
  __shared__ DevCtl s_ctl;
  __shared__ int s_sub, s_item, s_exit, s_last;
  const int tid = threadIdx.y * TX + threadIdx.x;
  unsigned backoff = 32;
  while (true) {
    // Warp 0 claims the next item: subdomains are scanned in PRIORITY order
    // (A.act is sorted by the previous window's work, the straggler first),
    // 32 candidates per round in parallel; the first claimable one wins.
    if (threadIdx.y == 0) {
      const int lane = threadIdx.x;
      int got = -1, item = 0;
      for (int base = 0; base < A.nact && got < 0; base += 32) {
        const int q = base + lane;
        int l = -1;
        bool claimable = false;
        if (q < A.nact) {
          l = A.act[q];
          const unsigned long long w = *(volatile unsigned long long*)&A.ctl[l].word;
          claimable = (unsigned)(w & 0xffffffffull) < (unsigned)A.geo[l].nitems;
        }
        unsigned mask = __ballot_sync(0xffffffffu, claimable);
        while (mask != 0u && got < 0) {
          const int src = __ffs(mask) - 1;
          mask &= mask - 1u;
          int it = -1;
          if (lane == src) {
            const unsigned long long w2 = atomicAdd(&A.ctl[l].word, 1ull);
            const unsigned u = (unsigned)(w2 & 0xffffffffull);
            if (u < (unsigned)A.geo[l].nitems) it = (int)u;
          }
          it = __shfl_sync(0xffffffffu, it, src);
          if (it >= 0) {
            got = __shfl_sync(0xffffffffu, l, src);
            item = it;
          }
        }
      }
      if (lane == 0) {
        s_sub = got;
        s_item = item;
        s_exit = 0;
        if (got < 0) {
          s_exit = *(volatile unsigned*)A.n_done >= (unsigned)A.nact;
        } else {
          __threadfence();   // acquire: the action and the previous action's data
          const DevCtl* gc = A.ctl + got;
          Act t;
          t.mode = __ldcg(&gc->a_mode);
          t.j = __ldcg(&gc->a_j);
          t.s = __ldcg(&gc->a_s);
          t.yi = __ldcg(&gc->a_yi);
          t.fi = __ldcg(&gc->a_fi);
          t.vin = __ldcg(&gc->a_vin);
          t.vout = __ldcg(&gc->a_vout);
          t.sub = got;
          t.c = __ldcg(&gc->a_c);
          t.h04 = __ldcg(&gc->a_h04);
          t.mu = __ldcg(&gc->a_mu);
          t.nu = __ldcg(&gc->a_nu);
          t.hmut = __ldcg(&gc->a_hmut);
          t.hgt = __ldcg(&gc->a_hgt);
          s_act = t;
        }
      }
    }
    __syncthreads();
    if (s_sub < 0) {
      if (s_exit) break;
      if (tid == 0) __nanosleep(backoff);
      backoff = backoff < 256 ? backoff * 2 : 256;
      __syncthreads();
      continue;
    }
    backoff = 32;
    const Act t = s_act;
    const int l = t.sub;
    const SubGeo& g = A.geo[l];
    Acc acc{0u, 0u, 0.0, 0.0};
    dispatch_item<DIM, P2>(A, g, t, s_item, sY, acc);
    // CTA reductions of the item
    const int any = __syncthreads_or(acc.flag);
    const int anynf = __syncthreads_or(acc.nonfin);
    unsigned long long emax = 0ull;
    if (t.mode == M_FINAL)
      emax = block_max_u64((unsigned long long)__double_as_longlong(acc.ratio), sh_max);
    double psum = 0.0;
    const bool sums = t.mode == M_POWER || t.mode == M_POWER_SEED || t.mode == M_NORM;
    if (sums) psum = block_sum2(acc.psum, sh_sum);
    if (tid == 0) {
      DevCtl* gc = A.ctl + l;
      if (sums) __stcg(A.part + A.poff[l] + s_item, psum);
      unsigned bits = 0;
      if (any) bits |= t.mode == M_FINAL ? 2u : 1u;
      if (anynf) bits |= 4u;
      if (bits) atomicOr(&gc->acc_flags, bits);
      if (t.mode == M_FINAL) atomicMax(&gc->acc_emax, emax);
      __threadfence();
      const unsigned d = atomicAdd(&gc->done, 1u);
      s_last = d == (unsigned)g.nitems - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      double sum = 0.0;
      if (sums) {   // fixed-order reduction of the item partials (deterministic)
        double v = 0.0;
        for (int i = tid; i < g.nitems; i += NT) v += __ldcg(A.part + A.poff[l] + i);
        sum = block_sum2(v, sh_sum);
      }
      if (threadIdx.y == 0) {   // warp 0: controller state in/out in parallel
        DevCtl* gc = A.ctl + l;
        constexpr int NW = (int)(sizeof(DevCtl) / 8);
        constexpr int WI = (int)(offsetof(DevCtl, word) / 8);
        long long* sc = reinterpret_cast<long long*>(&s_ctl);
        const long long* gsrc = reinterpret_cast<const long long*>(gc);
        for (int i = threadIdx.x; i < NW; i += 32) sc[i] = __ldcg(gsrc + i);
        __syncwarp();
        bool more = false;
        unsigned long long seq = 0;
        if (threadIdx.x == 0) {
          d_complete(A, s_ctl, l, sum, g.nodes);
          seq = (s_ctl.word >> 32) + 1;
          more = d_next_action(A, s_ctl);
          s_ctl.acc_flags = 0;
          s_ctl.acc_emax = 0ull;
          s_ctl.done = 0;
          if (!more) {
            unsigned long long now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            s_ctl.t_done = now;
          }
        }
        __syncwarp();
        long long* gdst = reinterpret_cast<long long*>(gc);
        for (int i = threadIdx.x; i < NW; i += 32)
          if (i != WI) __stcg(gdst + i, sc[i]);
        __syncwarp();
        if (threadIdx.x == 0) {
          __threadfence();
          if (more) {
            atomicExch(&gc->word, seq << 32);
          } else {
            atomicExch(&gc->word, (seq << 32) | kDoneLow);
            atomicAdd(A.n_done, 1u);
          }
        }
      }
    }
    __syncthreads();
  }
}

// ============================================================================
// 2D window kernel with a chunked, double-buffered cp.async item pipeline.
//
// A CTA claims a CHUNK of consecutive work items of one subdomain action
// (A.chunk_bulk = 8 items while many subdomains are active, A.chunk_tail = 2 on the tail's critical path),
// then streams each item's sources into shared memory with 16-byte cp.async
// (no register staging): the Y halo sources (y and the stage increment / f0 /
// v tile, 34 x 36 each) and the centre fields the epilogue needs (|Omega|rho,
// f0, d_{j-2}).  Item i+1's copies are in flight while item i is computed.
// The arithmetic per node is exactly node()/hdet's (bitwise identical).
// ============================================================================

constexpr int TW2 = TX + 4;    // 36 doubles: columns c0-2 .. c0+33 (16-B aligned chunks)
constexpr int TH2 = IR2 + 2;   // 34 rows
constexpr int HALO2 = (TH2 * TW2 + 15) / 16 * 16;   // 128-B multiple (TMA destinations)
struct Stage2 {
  double ys[HALO2];
  double as[HALO2];
  double cm[IR2 * TX];
  double cf[IR2 * TX];
  double cd[IR2 * TX];
};
constexpr int STAGE2_BYTES = (int)sizeof(Stage2);

__device__ __forceinline__ void cpa16(double* sdst, const double* gsrc, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gsrc), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int MODE, int YM>
__device__ __forceinline__ void issue2(const WinArgs& A, const SubGeo& g, const Act& t, int c0,
                                       int r0, Stage2& st) {
  const double* yb = A.F.y[t.yi];
  const double* ap = nullptr;
  if constexpr (MODE == M_STAGE2) ap = A.F.f[t.fi];
  if constexpr (MODE == M_STAGE3 || MODE == M_STAGEN) ap = A.F.d[(t.j - 1) % 3];
  if constexpr (MODE == M_FINAL) ap = A.F.d[t.s % 3];
  if constexpr (MODE == M_POWER) ap = A.F.d[t.vin];
  constexpr bool HAS_A = YM == YM_ADD || YM == YM_SCALED;
  constexpr bool NEED_F0 = MODE == M_STAGE3 || MODE == M_STAGEN || MODE == M_FINAL ||
                           MODE == M_POWER || MODE == M_POWER_SEED;
  const int tid = threadIdx.y * TX + threadIdx.x;
  constexpr int CH = TW2 / 2;   // 18 chunks per halo row
  for (int e = tid; e < TH2 * CH; e += NT) {
    const int rr = e / CH, cc = e - rr * CH;
    const int i0 = r0 - 1 + rr, col = c0 - 2 + 2 * cc;
    const bool ok = i0 >= 0 && i0 < g.n[0] && col >= 0 && col < g.pitch;
    const long long k = ok ? g.off + (long long)i0 * g.pitch + col : g.off;
    cpa16(&st.ys[rr * TW2 + 2 * cc], yb + k, ok ? 16 : 0);
    if constexpr (HAS_A) cpa16(&st.as[rr * TW2 + 2 * cc], ap + k, ok ? 16 : 0);
  }
  if constexpr (MODE != M_NORM) {
    constexpr int CC = TX / 2;  // 16 chunks per centre row
    for (int e = tid; e < IR2 * CC; e += NT) {
      const int rr = e / CC, cc = e - rr * CC;
      const int i0 = r0 + rr, col = c0 + 2 * cc;
      const bool ok = i0 < g.n[0] && col < g.pitch;
      const long long k = ok ? g.off + (long long)i0 * g.pitch + col : g.off;
      cpa16(&st.cm[rr * TX + 2 * cc], A.F.mr + k, ok ? 16 : 0);
      if constexpr (NEED_F0) cpa16(&st.cf[rr * TX + 2 * cc], A.F.f[t.fi] + k, ok ? 16 : 0);
      if constexpr (MODE == M_STAGEN)
        cpa16(&st.cd[rr * TX + 2 * cc], A.F.d[(t.j - 2) % 3] + k, ok ? 16 : 0);
    }
  }
  cpa_commit();
}

// ---- TMA (cp.async.bulk.tensor) tile loads, completion on an mbarrier ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* m) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void mbar_init_n(unsigned long long* m, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(m)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(m)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(m)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma2(void* dst, const void* tmap, int x, int y,
                                     unsigned long long* m) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(m))
      : "memory");
}

// One thread: the TMA copies of one 2D item into stage `st` (zero fill outside the box).
template <int MODE, int YM>
__device__ __forceinline__ void issue2_tma(const WinArgs& A, int l, const Act& t, int c0, int r0,
                                           Stage2& st, unsigned long long* mbar) {
  constexpr bool HAS_A = YM == YM_ADD || YM == YM_SCALED;
  constexpr bool NEED_F0 = MODE == M_STAGE3 || MODE == M_STAGEN || MODE == M_FINAL ||
                           MODE == M_POWER || MODE == M_POWER_SEED;
  int fa = 0;
  if constexpr (MODE == M_STAGE2) fa = TF_F0 + t.fi;
  if constexpr (MODE == M_STAGE3 || MODE == M_STAGEN) fa = TF_D0 + (t.j - 1) % 3;
  if constexpr (MODE == M_FINAL) fa = TF_D0 + t.s % 3;
  if constexpr (MODE == M_POWER) fa = TF_D0 + t.vin;
  const char* tm = reinterpret_cast<const char*>(A.tmap) + (size_t)l * TF_N * 2 * 128;
  auto map = [&](int f, int kind) { return tm + (f * 2 + kind) * 128; };
  unsigned bytes = TH2 * TW2 * 8;
  if constexpr (HAS_A) bytes += TH2 * TW2 * 8;
  if constexpr (MODE != M_NORM) {
    bytes += IR2 * TX * 8;
    if constexpr (NEED_F0) bytes += IR2 * TX * 8;
    if constexpr (MODE == M_STAGEN) bytes += IR2 * TX * 8;
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  mbar_expect(mbar, bytes);
  tma2(st.ys, map(TF_Y0 + t.yi, 0), c0 - 2, r0 - 1, mbar);
  if constexpr (HAS_A) tma2(st.as, map(fa, 0), c0 - 2, r0 - 1, mbar);
  if constexpr (MODE != M_NORM) {
    tma2(st.cm, map(TF_MR, 1), c0, r0, mbar);
    if constexpr (NEED_F0) tma2(st.cf, map(TF_F0 + t.fi, 1), c0, r0, mbar);
    if constexpr (MODE == M_STAGEN) tma2(st.cd, map(TF_D0 + (t.j - 2) % 3, 1), c0, r0, mbar);
  }
}

template <int YM>
__device__ __forceinline__ double yat(const Stage2& st, int p, double c, int par) {
  if constexpr (YM == YM_PLAIN) {
    return st.ys[p];
  } else if constexpr (YM == YM_ADD) {
    return st.ys[p] + st.as[p];
  } else if constexpr (YM == YM_SCALED) {
    return st.ys[p] + c * st.as[p];
  } else {
    return st.ys[p] + (par ? -c : c);
  }
}

// Y for the generic (box-face) formulas: from the smem tile when the point
// lies inside it (always, except for 1-3 row/column slivers at a box end),
// else from global memory.
template <int YM, int YMG = YM>
struct TileAcc2 {
  const Stage2* st;
  int r0, c0;
  GAcc<2, YMG> g;
  __device__ __forceinline__ double operator()(int i0, int i1, int) const {
    const int rr = i0 - r0 + 1, cc = i1 - c0 + 2;
    if (rr >= 0 && rr < TH2 && cc >= 0 && cc < TW2) {
      const int p = rr * TW2 + cc;
      if constexpr (YM == YM_PLAIN) {
        return st->ys[p];
      } else if constexpr (YM == YM_ADD) {
        return st->ys[p] + st->as[p];
      } else if constexpr (YM == YM_SCALED) {
        return st->ys[p] + g.c * st->as[p];
      } else {
        return st->ys[p] + (((i0 + i1) & 1) ? -g.c : g.c);
      }
    }
    return g(i0, i1, 0);
  }
};

template <bool P2, int MODE, int YM>
__device__ __forceinline__ void compute2(const WinArgs& A, const SubGeo& g, const Act& t, int c0,
                                         int r0, const Stage2& st, Acc& acc, double* psum_item) {
  constexpr int R = IR2 / TY;
  // how Y is formed from global memory (outside the tile) for this mode
  constexpr int YMG = MODE == M_STAGE2 ? YM_SCALED
                      : (MODE == M_STAGE3 || MODE == M_STAGEN) ? YM_ADD : YM;
  const int n0 = g.n[0], n1 = g.n[1];
  const int i1 = c0 + threadIdx.x;
  const double* yb = A.F.y[t.yi];
  const double* ap = nullptr;
  if constexpr (MODE == M_STAGE2) ap = A.F.f[t.fi];
  if constexpr (MODE == M_STAGE3 || MODE == M_STAGEN) ap = A.F.d[(t.j - 1) % 3];
  if constexpr (MODE == M_FINAL) ap = A.F.d[t.s % 3];
  if constexpr (MODE == M_POWER) ap = A.F.d[t.vin];
  if constexpr (MODE == M_NORM) {
    double ps = 0.0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int lr = threadIdx.y + q * TY;
      if (r0 + lr < n0 && i1 < n1) {
        const double y = st.ys[(lr + 1) * TW2 + threadIdx.x + 2];
        ps += y * y;
      }
    }
    *psum_item = ps;
    return;
  } else {
    // phase 1: determinants of all R rows, branch-free interior formula
    // (independent chains -> ILP); box-face rows patched in phase 2
    double det[R];
    unsigned edge = 0u;   // bit q: node q is on a box face
    unsigned valid = 0u;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int lr = threadIdx.y + q * TY;
      const int i0 = r0 + lr;
      const bool ok = i0 < n0 && i1 < n1;
      valid |= ok ? (1u << q) : 0u;
      const bool interior = i0 >= 1 && i0 <= n0 - 2 && i1 >= 1 && i1 <= n1 - 2;
      edge |= (ok && !interior) ? (1u << q) : 0u;
      const int p = (lr + 1) * TW2 + threadIdx.x + 2;
      const int par = (i0 + i1) & 1;
      const double yc = yat<YM>(st, p, t.c, par);
      const double yn = yat<YM>(st, p - TW2, t.c, par ^ 1);
      const double ys_ = yat<YM>(st, p + TW2, t.c, par ^ 1);
      const double yw = yat<YM>(st, p - 1, t.c, par ^ 1);
      const double ye = yat<YM>(st, p + 1, t.c, par ^ 1);
      const double yne = yat<YM>(st, p - TW2 + 1, t.c, par);
      const double ynw = yat<YM>(st, p - TW2 - 1, t.c, par);
      const double yse = yat<YM>(st, p + TW2 + 1, t.c, par);
      const double ysw = yat<YM>(st, p + TW2 - 1, t.c, par);
      const double h00 = dv<P2>((ys_ - 2.0 * yc) + yn, A.P.ax[0].hh, A.P.ax[0].ihh);
      const double h11 = dv<P2>((ye - 2.0 * yc) + yw, A.P.ax[1].hh, A.P.ax[1].ihh);
      const double gp = dv<P2>(yse - ysw, A.P.ax[1].twoh, A.P.ax[1].itwoh);
      const double gm = dv<P2>(yne - ynw, A.P.ax[1].twoh, A.P.ax[1].itwoh);
      const double h01 = dv<P2>(gp - gm, A.P.ax[0].twoh, A.P.ax[0].itwoh);
      det[q] = h00 * h11 - h01 * h01;
    }
    // phase 2: generic face formulas (rare).  Dirichlet (interface-face)
    // nodes need no determinant: F = 0 there and they never raise the flag.
    unsigned dirm = 0u;
    if (edge) {
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (edge & (1u << q)) {
          const int i0 = r0 + threadIdx.y + q * TY;
          if (dirichlet<2>(g, i0, i1, 0)) {
            dirm |= 1u << q;
          } else {
            det[q] = hdet<2, P2>(A.P, g, i0, i1, 0,
                                 TileAcc2<YM, YMG>{&st, r0, c0, GAcc<2, YMG>{&g, yb, ap, t.c}});
          }
        }
      }
    }
    // phase 3: log-equidistribution for all rows (independent chains)
    double F[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int lr = threadIdx.y + q * TY;
      const bool dir = (dirm >> q) & 1u;
      const int pc = lr * TX + threadIdx.x;
      F[q] = dir ? 0.0 : logequi(st.cm[pc], det[q], A.P.guard, A.P.floor, A.P.rguard, s_logtab);
      acc.flag |= ((valid >> q) & 1u) && det[q] <= A.P.floor && !dir ? 1u : 0u;
    }
    // phase 4: epilogues
    double ps = 0.0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      if (!((valid >> q) & 1u)) continue;
      const int lr = threadIdx.y + q * TY;
      const int i0 = r0 + lr;
      const int p = (lr + 1) * TW2 + threadIdx.x + 2;
      const int pc = lr * TX + threadIdx.x;
      const long long k = g.off + (long long)i0 * g.pitch + i1;
      if constexpr (MODE == M_F0) {
        A.F.f[t.fi][k] = F[q];
      } else if constexpr (MODE == M_EULER) {
        A.F.y[1 - t.yi][k] = st.ys[p] + t.c * F[q];
      } else if constexpr (MODE == M_STAGE2) {
        const double f0 = st.as[p];             // the a tile of stage 2 is f0
        const double d1 = t.c * f0;
        A.F.d[2][k] = ((t.mu * d1 + t.nu * 0.0) + t.hmut * F[q]) + t.hgt * f0;
      } else if constexpr (MODE == M_STAGE3) {
        const double f0 = st.cf[pc];
        const double d1 = t.c * f0;
        A.F.d[0][k] = ((t.mu * st.as[p] + t.nu * d1) + t.hmut * F[q]) + t.hgt * f0;
      } else if constexpr (MODE == M_STAGEN) {
        const double f0 = st.cf[pc];
        A.F.d[t.j % 3][k] = ((t.mu * st.as[p] + t.nu * st.cd[pc]) + t.hmut * F[q]) + t.hgt * f0;
      } else if constexpr (MODE == M_FINAL) {
        const double ds = st.as[p], yv = st.ys[p], f0 = st.cf[pc];
        const double yn = yv + ds;
        A.F.f[1 - t.fi][k] = F[q];
        A.F.y[1 - t.yi][k] = yn;
        const double err = -0.8 * ds + t.h04 * (f0 + F[q]);
        const double ay = fabs(yv), an = fabs(yn);
        const double mx = (ay >= an || isnan(ay)) ? ay : an;
        const double r = fabs(err) / (A.P.atol + A.P.rtol * mx);
        if (isfinite(r)) acc.ratio = r > acc.ratio ? r : acc.ratio;
        else acc.nonfin = 1;
      } else {
        const double diff = F[q] - st.cf[pc];
        A.F.d[t.vout][k] = diff;
        ps += diff * diff;
      }
    }
    *psum_item = ps;
  }
}

// Face-node determinant (generic one-sided formulas, hdet<2>).
template <bool P2, int YM>
__device__ __forceinline__ double hdet_face(const WinArgs& A, const SubGeo& g, const Act& t, int i0,
                                         int i1, int r0, int c0, const Stage2& st,
                                         const double* yb, const double* ap) {
  return hdet<2, P2>(A.P, g, i0, i1, 0,
                     TileAcc2<YM, YM>{&st, r0, c0, GAcc<2, YM>{&g, yb, ap, t.c}});
}

// Fused RHS + epilogue of one 2D item for the modes without partial sums
// (F0, EULER, STAGE2/3/N, FINAL).  Thread (tx, ty) owns the two consecutive
// rows 2ty and 2ty+1 of column tx, so the 3x4 Y neighbourhood is loaded once
// for both nodes.  Every node first takes compute2's branch-free interior
// formula (same expressions, same order: bitwise identical); with EDGE (the
// item touches a box face or extends past the box) face nodes are then
// patched exactly as compute2 does: Dirichlet (interface) nodes get F = 0 and
// no determinant, physical-face nodes the one-sided formulas of hdet<2>, and
// nodes past the box are skipped.
template <bool P2, int MODE, int YM, bool EDGE>
__device__ __forceinline__ void compute2_int(const WinArgs& A, const SubGeo& g, const Act& t,
                                             long long kb, long long pitch, int r0, int c0,
                                             int n0, int n1, const Stage2& st, Acc& acc) {
  const int tx = threadIdx.x, lr = 2 * threadIdx.y;
  const int p = (lr + 1) * TW2 + tx + 2;       // tile index of node (lr, tx)
  const int par = (r0 + c0 + lr + tx) & 1;     // (i0 + i1) & 1 of node (lr, tx)
  double w[4], c[4], e[4];                     // tile rows lr-1 .. lr+2, columns tx-1..tx+1
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int b = p + (r - 1) * TW2;
    const int pr = par ^ ((r + 1) & 1);        // parity of (lr + r - 1, tx)
    w[r] = yat<YM>(st, b - 1, t.c, pr ^ 1);
    c[r] = yat<YM>(st, b, t.c, pr);
    e[r] = yat<YM>(st, b + 1, t.c, pr ^ 1);
  }
  const double ihh0 = A.P.ax[0].ihh, hh0 = A.P.ax[0].hh, ihh1 = A.P.ax[1].ihh, hh1 = A.P.ax[1].hh;
  const double it0 = A.P.ax[0].itwoh, tw0 = A.P.ax[0].twoh, it1 = A.P.ax[1].itwoh,
               tw1 = A.P.ax[1].twoh;
  double gd[4];                                // (e - w)/2h1 per row: gm of row r+1, gp of r-1
#pragma unroll
  for (int r = 0; r < 4; ++r) gd[r] = dv<P2>(e[r] - w[r], tw1, it1);
  double F[2], det[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const double yc = c[q + 1];
    const double h00 = dv<P2>((c[q + 2] - 2.0 * yc) + c[q], hh0, ihh0);
    const double h11 = dv<P2>((e[q + 1] - 2.0 * yc) + w[q + 1], hh1, ihh1);
    const double h01 = dv<P2>(gd[q + 2] - gd[q], tw0, it0);
    det[q] = h00 * h11 - h01 * h01;
  }
  unsigned valid = 3u, dirm = 0u;
  if constexpr (EDGE) {
    const double* yb = A.F.y[t.yi];
    const double* ap = nullptr;
    if constexpr (MODE == M_STAGE2) ap = A.F.f[t.fi];
    if constexpr (MODE == M_STAGE3 || MODE == M_STAGEN) ap = A.F.d[(t.j - 1) % 3];
    if constexpr (MODE == M_FINAL) ap = A.F.d[t.s % 3];
    const int i1 = c0 + tx;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int i0 = r0 + lr + q;
      if (!(i0 < n0 && i1 < n1)) {
        valid &= ~(1u << q);
      } else if (i0 == 0 || i0 == n0 - 1 || i1 == 0 || i1 == n1 - 1) {
        if (dirichlet<2>(g, i0, i1, 0)) dirm |= 1u << q;
        else det[q] = hdet_face<P2, YM>(A, g, t, i0, i1, r0, c0, st, yb, ap);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int pc = (lr + q) * TX + tx;
    const bool dir = (dirm >> q) & 1u;
    F[q] = dir ? 0.0 : logequi(st.cm[pc], det[q], A.P.guard, A.P.floor, A.P.rguard, s_logtab);
    acc.flag |= ((valid >> q) & 1u) && !dir && det[q] <= A.P.floor ? 1u : 0u;
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    if (EDGE && !((valid >> q) & 1u)) continue;
    const int pq = p + q * TW2;
    const int pc = (lr + q) * TX + tx;
    const long long k = kb + (long long)(lr + q) * pitch;
    if constexpr (MODE == M_F0) {
      A.F.f[t.fi][k] = F[q];
    } else if constexpr (MODE == M_EULER) {
      A.F.y[1 - t.yi][k] = st.ys[pq] + t.c * F[q];
    } else if constexpr (MODE == M_STAGE2) {
      const double f0 = st.as[pq];
      const double d1 = t.c * f0;
      A.F.d[2][k] = ((t.mu * d1 + t.nu * 0.0) + t.hmut * F[q]) + t.hgt * f0;
    } else if constexpr (MODE == M_STAGE3) {
      const double f0 = st.cf[pc];
      const double d1 = t.c * f0;
      A.F.d[0][k] = ((t.mu * st.as[pq] + t.nu * d1) + t.hmut * F[q]) + t.hgt * f0;
    } else if constexpr (MODE == M_STAGEN) {
      const double f0 = st.cf[pc];
      A.F.d[t.j % 3][k] = ((t.mu * st.as[pq] + t.nu * st.cd[pc]) + t.hmut * F[q]) + t.hgt * f0;
    } else if constexpr (MODE == M_FINAL) {
      const double ds = st.as[pq], yv = st.ys[pq], f0 = st.cf[pc];
      const double yn = yv + ds;
      A.F.f[1 - t.fi][k] = F[q];
      A.F.y[1 - t.yi][k] = yn;
      const double err = -0.8 * ds + t.h04 * (f0 + F[q]);
      const double ay = fabs(yv), an = fabs(yn);
      const double mx = (ay >= an || isnan(ay)) ? ay : an;
      const double r = fabs(err) / (A.P.atol + A.P.rtol * mx);
      if (isfinite(r)) acc.ratio = r > acc.ratio ? r : acc.ratio;
      else acc.nonfin = 1;
    }
  }
}

// Claim (warp 0): scan active subdomains in priority order, 32 at a time, and
// grab up to `chunk` consecutive items of the first claimable action.
__device__ __forceinline__ void claim(const WinArgs& A, int chunk, int& got, int& it0, int& nit) {
  const int lane = threadIdx.x;
  got = -1;
  it0 = 0;
  nit = 0;
  for (int base = 0; base < A.nact && got < 0; base += 32) {
    const int q = base + lane;
    int l = -1;
    bool claimable = false;
    if (q < A.nact) {
      l = A.act[q];
      const unsigned long long w = *(volatile unsigned long long*)&A.ctl[l].word;
      claimable = (unsigned)(w & 0xffffffffull) < (unsigned)A.geo[l].nitems;
    }
    unsigned mask = __ballot_sync(0xffffffffu, claimable);
    while (mask != 0u && got < 0) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1u;
      int it = -1, n = 0;
      if (lane == src) {
        const unsigned long long w2 = atomicAdd(&A.ctl[l].word, (unsigned long long)chunk);
        const unsigned u = (unsigned)(w2 & 0xffffffffull);
        const unsigned ni = (unsigned)A.geo[l].nitems;
        if (u < ni) {
          it = (int)u;
          n = (int)(ni - u < (unsigned)chunk ? ni - u : (unsigned)chunk);
        }
      }
      it = __shfl_sync(0xffffffffu, it, src);
      n = __shfl_sync(0xffffffffu, n, src);
      if (it >= 0) {
        got = __shfl_sync(0xffffffffu, l, src);
        it0 = it;
        nit = n;
      }
    }
  }
}

__device__ __forceinline__ Act load_act(const WinArgs& A, int l) {
  const DevCtl* gc = A.ctl + l;
  Act t;
  t.mode = __ldcg(&gc->a_mode);
  t.j = __ldcg(&gc->a_j);
  t.s = __ldcg(&gc->a_s);
  t.yi = __ldcg(&gc->a_yi);
  t.fi = __ldcg(&gc->a_fi);
  t.vin = __ldcg(&gc->a_vin);
  t.vout = __ldcg(&gc->a_vout);
  t.sub = l;
  t.c = __ldcg(&gc->a_c);
  t.h04 = __ldcg(&gc->a_h04);
  t.mu = __ldcg(&gc->a_mu);
  t.nu = __ldcg(&gc->a_nu);
  t.hmut = __ldcg(&gc->a_hmut);
  t.hgt = __ldcg(&gc->a_hgt);
  return t;
}

// Decision by warp 0 of the CTA that completed an action (see k_window).
__device__ void decide(const WinArgs& A, int l, const SubGeo& g, double sum, DevCtl& s_ctl) {
  DevCtl* gc = A.ctl + l;
  constexpr int NW = (int)(sizeof(DevCtl) / 8);
  constexpr int WI = (int)(offsetof(DevCtl, word) / 8);
  long long* sc = reinterpret_cast<long long*>(&s_ctl);
  const long long* gsrc = reinterpret_cast<const long long*>(gc);
  for (int i = threadIdx.x; i < NW; i += 32) sc[i] = __ldcg(gsrc + i);
  __syncwarp();
  bool more = false;
  unsigned long long seq = 0;
  if (threadIdx.x == 0) {
    d_complete(A, s_ctl, l, sum, g.nodes);
    seq = (s_ctl.word >> 32) + 1;
    more = d_next_action(A, s_ctl);
    s_ctl.acc_flags = 0;
    s_ctl.acc_emax = 0ull;
    s_ctl.done = 0;
    if (!more) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      s_ctl.t_done = now;
    }
  }
  __syncwarp();
  long long* gdst = reinterpret_cast<long long*>(gc);
  for (int i = threadIdx.x; i < NW; i += 32)
    if (i != WI) __stcg(gdst + i, sc[i]);
  __syncwarp();
  if (threadIdx.x == 0) {
    __threadfence();
    if (A.probe && l == A.probe_sub) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      const unsigned long long sq = (seq - 1) % (unsigned long long)A.probe_cap;
      A.probe[sq * 4 + 3] = now;
      A.probe[(seq % (unsigned long long)A.probe_cap) * 4 + 0] = now;
    }
    if (more) {
      atomicExch(&gc->word, seq << 32);
    } else {
      atomicExch(&gc->word, (seq << 32) | kDoneLow);
      atomicAdd(A.n_done, 1u);
    }
  }
}

template <bool P2, int MODE, int YM>
__device__ void chunk2(const WinArgs& A, const SubGeo& g, const Act& t, int it0, int nit,
                       Stage2* stage, Acc& acc, double* sh_sum, unsigned long long* mbar,
                       unsigned& phases) {
  constexpr bool SUMS = MODE == M_POWER || MODE == M_POWER_SEED || MODE == M_NORM;
  // box geometry in registers (the geo table is immutable during the kernel)
  const int n0 = __ldg(&g.n[0]), n1 = __ldg(&g.n[1]), items_x = __ldg(&g.items_x);
  const long long pitch = __ldg(&g.pitch), goff = __ldg(&g.off);
  // item -> (column, row) tile origin, decoded once per chunk then stepped
  int ix = it0 % items_x, iy = it0 / items_x;
  int nx = ix + 1, ny = iy;
  if (nx == items_x) {
    nx = 0;
    ++ny;
  }
  const bool tma = A.tmap != nullptr;
  const bool lead = threadIdx.x == 0 && threadIdx.y == 0;
  // TMA pipeline: mbar[b] = "buffer b full" (1 arrival + tx bytes), mbar[2+b]
  // = "buffer b consumed" (one arrival per warp).  phases: bits 0-1 full
  // parity, 2-3 consumed parity, 4-5 buffer used before.  The issuing thread
  // waits for the previous use of a buffer to be consumed by every warp, so
  // warps never meet at a CTA barrier between items.
  auto issue = [&](int b, int cx, int cy) {
    if ((phases >> (4 + b)) & 1u) {
      mbar_wait(&mbar[2 + b], (phases >> (2 + b)) & 1u);
      phases ^= 1u << (2 + b);
    }
    phases |= 1u << (4 + b);
    issue2_tma<MODE, YM>(A, t.sub, t, cx * TX, cy * IR2, stage[b], &mbar[b]);
  };
  if (tma) {
    if (lead) issue(0, ix, iy);
  } else {
    issue2<MODE, YM>(A, g, t, ix * TX, iy * IR2, stage[0]);
  }
  for (int i = 0; i < nit; ++i) {
    const int s = i & 1;
    if (tma) {
      if (i + 1 < nit && lead) issue(s ^ 1, nx, ny);
      mbar_wait(&mbar[s], (phases >> s) & 1u);
      phases ^= 1u << s;
    } else {
      if (i + 1 < nit) {
        issue2<MODE, YM>(A, g, t, nx * TX, ny * IR2, stage[s ^ 1]);
        cpa_wait<1>();
      } else {
        cpa_wait<0>();
      }
      __syncthreads();
    }
    double ps = 0.0;
    const int c0 = ix * TX, r0 = iy * IR2;
    const long long kb = goff + (long long)r0 * pitch + c0 + threadIdx.x;
    if constexpr (SUMS) {
      compute2<P2, MODE, YM>(A, g, t, c0, r0, stage[s], acc, &ps);
    } else if (r0 >= 1 && r0 + IR2 <= n0 - 1 && c0 >= 1 && c0 + TX <= n1 - 1) {
      compute2_int<P2, MODE, YM, false>(A, g, t, kb, pitch, r0, c0, n0, n1, stage[s], acc);
    } else {
      compute2_int<P2, MODE, YM, true>(A, g, t, kb, pitch, r0, c0, n0, n1, stage[s], acc);
    }
    ix = nx;
    iy = ny;
    if (++nx == items_x) {
      nx = 0;
      ++ny;
    }
    if (tma) {
      __syncwarp();
      if (threadIdx.x == 0) mbar_arrive(&mbar[2 + s]);   // this warp is done with buffer s
    }
    if constexpr (SUMS) {
      const double s = block_sum(ps, sh_sum);   // per-item partial: deterministic
      if (threadIdx.x == 0 && threadIdx.y == 0) __stcg(A.part + A.poff[t.sub] + it0 + i, s);
    } else {
      if (!tma) __syncthreads();   // the stage buffer is refilled by the next iteration's issue
    }
  }
}

template <bool P2>
__device__ void dispatch_chunk2(const WinArgs& A, const SubGeo& g, const Act& t, int it0, int nit,
                                Stage2* st, Acc& acc, double* sh, unsigned long long* mb,
                                unsigned& ph) {
  switch (t.mode) {
    case M_F0: chunk2<P2, M_F0, YM_PLAIN>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    case M_EULER: chunk2<P2, M_EULER, YM_PLAIN>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    case M_STAGE2: chunk2<P2, M_STAGE2, YM_SCALED>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    case M_STAGE3: chunk2<P2, M_STAGE3, YM_ADD>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    case M_STAGEN: chunk2<P2, M_STAGEN, YM_ADD>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    case M_FINAL: chunk2<P2, M_FINAL, YM_ADD>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    case M_POWER: chunk2<P2, M_POWER, YM_SCALED>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    case M_POWER_SEED:
      chunk2<P2, M_POWER_SEED, YM_SEED>(A, g, t, it0, nit, st, acc, sh, mb, ph);
      break;
    case M_NORM: chunk2<P2, M_NORM, YM_PLAIN>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    default: break;
  }
}

// ----------------------------------------------------------------- 3D ----
// Same pipeline for 3D boxes: items of TX x TY x IZ3 nodes (32 x 8 x 2); the
// stage holds the (IZ3+2) x (TY+2) x 36 halo tiles of y and a plus the centre
// fields.  The interior Hessian is the 19-point formula of hdet<3>.
constexpr int TH3 = TY + 2, TD3 = IZ3 + 2;
constexpr int SY3 = TW2, SZ3 = TH3 * TW2;
struct Stage3 {
  double ys[TD3 * TH3 * TW2];
  double as[TD3 * TH3 * TW2];
  double cm[IZ3 * TY * TX];
  double cf[IZ3 * TY * TX];
  double cd[IZ3 * TY * TX];
};

template <int MODE, int YM>
__device__ __forceinline__ void issue3(const WinArgs& A, const SubGeo& g, const Act& t, int c0,
                                       int r0, int z0, Stage3& st) {
  const double* yb = A.F.y[t.yi];
  const double* ap = nullptr;
  if constexpr (MODE == M_STAGE2) ap = A.F.f[t.fi];
  if constexpr (MODE == M_STAGE3 || MODE == M_STAGEN) ap = A.F.d[(t.j - 1) % 3];
  if constexpr (MODE == M_FINAL) ap = A.F.d[t.s % 3];
  if constexpr (MODE == M_POWER) ap = A.F.d[t.vin];
  constexpr bool HAS_A = YM == YM_ADD || YM == YM_SCALED;
  constexpr bool NEED_F0 = MODE == M_STAGE3 || MODE == M_STAGEN || MODE == M_FINAL ||
                           MODE == M_POWER || MODE == M_POWER_SEED;
  const int tid = threadIdx.y * TX + threadIdx.x;
  constexpr int CH = TW2 / 2;
  const long long plane = (long long)g.n[1] * g.pitch;
  for (int e = tid; e < TD3 * TH3 * CH; e += NT) {
    const int cc = e % CH, rr = (e / CH) % TH3, zz = e / (CH * TH3);
    const int i0 = z0 - 1 + zz, i1 = r0 - 1 + rr, col = c0 - 2 + 2 * cc;
    const bool ok = i0 >= 0 && i0 < g.n[0] && i1 >= 0 && i1 < g.n[1] && col >= 0 && col < g.pitch;
    const long long k = ok ? g.off + i0 * plane + (long long)i1 * g.pitch + col : g.off;
    const int sidx = (zz * TH3 + rr) * TW2 + 2 * cc;
    cpa16(&st.ys[sidx], yb + k, ok ? 16 : 0);
    if constexpr (HAS_A) cpa16(&st.as[sidx], ap + k, ok ? 16 : 0);
  }
  if constexpr (MODE != M_NORM) {
    constexpr int CC = TX / 2;
    for (int e = tid; e < IZ3 * TY * CC; e += NT) {
      const int cc = e % CC, rr = (e / CC) % TY, zz = e / (CC * TY);
      const int i0 = z0 + zz, i1 = r0 + rr, col = c0 + 2 * cc;
      const bool ok = i0 < g.n[0] && i1 < g.n[1] && col < g.pitch;
      const long long k = ok ? g.off + i0 * plane + (long long)i1 * g.pitch + col : g.off;
      const int cidx = (zz * TY + rr) * TX + 2 * cc;
      cpa16(&st.cm[cidx], A.F.mr + k, ok ? 16 : 0);
      if constexpr (NEED_F0) cpa16(&st.cf[cidx], A.F.f[t.fi] + k, ok ? 16 : 0);
      if constexpr (MODE == M_STAGEN) cpa16(&st.cd[cidx], A.F.d[(t.j - 2) % 3] + k, ok ? 16 : 0);
    }
  }
  cpa_commit();
}

template <int YM, int YMG = YM>
struct TileAcc3 {
  const Stage3* st;
  int z0, r0, c0;
  GAcc<3, YMG> g;
  __device__ __forceinline__ double operator()(int i0, int i1, int i2) const {
    const int zz = i0 - z0 + 1, rr = i1 - r0 + 1, cc = i2 - c0 + 2;
    if (zz >= 0 && zz < TD3 && rr >= 0 && rr < TH3 && cc >= 0 && cc < TW2) {
      const int p = (zz * TH3 + rr) * TW2 + cc;
      if constexpr (YM == YM_PLAIN) {
        return st->ys[p];
      } else if constexpr (YM == YM_ADD) {
        return st->ys[p] + st->as[p];
      } else if constexpr (YM == YM_SCALED) {
        return st->ys[p] + g.c * st->as[p];
      } else {
        return st->ys[p] + (((i0 + i1 + i2) & 1) ? -g.c : g.c);
      }
    }
    return g(i0, i1, i2);
  }
};

template <int YM>
__device__ __forceinline__ double yat3(const Stage3& st, int p, double c, int par) {
  if constexpr (YM == YM_PLAIN) {
    return st.ys[p];
  } else if constexpr (YM == YM_ADD) {
    return st.ys[p] + st.as[p];
  } else if constexpr (YM == YM_SCALED) {
    return st.ys[p] + c * st.as[p];
  } else {
    return st.ys[p] + (par ? -c : c);
  }
}

template <bool P2, int MODE, int YM>
__device__ __forceinline__ void compute3(const WinArgs& A, const SubGeo& g, const Act& t, int c0,
                                         int r0, int z0, const Stage3& st, Acc& acc,
                                         double* psum_item) {
  constexpr int YMG = MODE == M_STAGE2 ? YM_SCALED
                      : (MODE == M_STAGE3 || MODE == M_STAGEN) ? YM_ADD : YM;
  const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];
  const int i1 = r0 + threadIdx.y, i2 = c0 + threadIdx.x;
  const double* yb = A.F.y[t.yi];
  const double* ap = nullptr;
  if constexpr (MODE == M_STAGE2) ap = A.F.f[t.fi];
  if constexpr (MODE == M_STAGE3 || MODE == M_STAGEN) ap = A.F.d[(t.j - 1) % 3];
  if constexpr (MODE == M_FINAL) ap = A.F.d[t.s % 3];
  if constexpr (MODE == M_POWER) ap = A.F.d[t.vin];
  const long long plane = (long long)n1 * g.pitch;
  double ps = 0.0;
#pragma unroll
  for (int q = 0; q < IZ3; ++q) {
    const int i0 = z0 + q;
    if (i0 >= n0 || i1 >= n1 || i2 >= n2) continue;
    const int p = ((q + 1) * TH3 + threadIdx.y + 1) * TW2 + threadIdx.x + 2;
    const int pc = (q * TY + threadIdx.y) * TX + threadIdx.x;
    const long long k = g.off + i0 * plane + (long long)i1 * g.pitch + i2;
    if constexpr (MODE == M_NORM) {
      const double y = st.ys[p];
      ps += y * y;
      continue;
    } else {
      const bool interior = i0 >= 1 && i0 <= n0 - 2 && i1 >= 1 && i1 <= n1 - 2 && i2 >= 1 &&
                            i2 <= n2 - 2;
      double det;
      if (interior) {
        const int par = (i0 + i1 + i2) & 1;
        const double c = yat3<YM>(st, p, t.c, par);
        const double h00 = dv<P2>((yat3<YM>(st, p + SZ3, t.c, par ^ 1) - 2.0 * c) +
                                      yat3<YM>(st, p - SZ3, t.c, par ^ 1),
                                  A.P.ax[0].hh, A.P.ax[0].ihh);
        const double h11 = dv<P2>((yat3<YM>(st, p + SY3, t.c, par ^ 1) - 2.0 * c) +
                                      yat3<YM>(st, p - SY3, t.c, par ^ 1),
                                  A.P.ax[1].hh, A.P.ax[1].ihh);
        const double h22 = dv<P2>((yat3<YM>(st, p + 1, t.c, par ^ 1) - 2.0 * c) +
                                      yat3<YM>(st, p - 1, t.c, par ^ 1),
                                  A.P.ax[2].hh, A.P.ax[2].ihh);
        double gp = dv<P2>(yat3<YM>(st, p + SZ3 + SY3, t.c, par) -
                               yat3<YM>(st, p + SZ3 - SY3, t.c, par),
                           A.P.ax[1].twoh, A.P.ax[1].itwoh);
        double gm = dv<P2>(yat3<YM>(st, p - SZ3 + SY3, t.c, par) -
                               yat3<YM>(st, p - SZ3 - SY3, t.c, par),
                           A.P.ax[1].twoh, A.P.ax[1].itwoh);
        const double h01 = dv<P2>(gp - gm, A.P.ax[0].twoh, A.P.ax[0].itwoh);
        gp = dv<P2>(yat3<YM>(st, p + SZ3 + 1, t.c, par) - yat3<YM>(st, p + SZ3 - 1, t.c, par),
                    A.P.ax[2].twoh, A.P.ax[2].itwoh);
        gm = dv<P2>(yat3<YM>(st, p - SZ3 + 1, t.c, par) - yat3<YM>(st, p - SZ3 - 1, t.c, par),
                    A.P.ax[2].twoh, A.P.ax[2].itwoh);
        const double h02 = dv<P2>(gp - gm, A.P.ax[0].twoh, A.P.ax[0].itwoh);
        gp = dv<P2>(yat3<YM>(st, p + SY3 + 1, t.c, par) - yat3<YM>(st, p + SY3 - 1, t.c, par),
                    A.P.ax[2].twoh, A.P.ax[2].itwoh);
        gm = dv<P2>(yat3<YM>(st, p - SY3 + 1, t.c, par) - yat3<YM>(st, p - SY3 - 1, t.c, par),
                    A.P.ax[2].twoh, A.P.ax[2].itwoh);
        const double h12 = dv<P2>(gp - gm, A.P.ax[1].twoh, A.P.ax[1].itwoh);
        det = (h00 * (h11 * h22 - h12 * h12) - h01 * (h01 * h22 - h12 * h02)) +
              h02 * (h01 * h12 - h11 * h02);
      } else {
        det = hdet<3, P2>(A.P, g, i0, i1, i2,
                          TileAcc3<YM, YMG>{&st, z0, r0, c0, GAcc<3, YMG>{&g, yb, ap, t.c}});
      }
      const bool dir = !interior && dirichlet<3>(g, i0, i1, i2);
      const double F = dir ? 0.0 : logequi(st.cm[pc], det, A.P.guard, A.P.floor, A.P.rguard, s_logtab);
      acc.flag |= (det <= A.P.floor && !dir) ? 1u : 0u;
      if constexpr (MODE == M_F0) {
        A.F.f[t.fi][k] = F;
      } else if constexpr (MODE == M_EULER) {
        A.F.y[1 - t.yi][k] = st.ys[p] + t.c * F;
      } else if constexpr (MODE == M_STAGE2) {
        const double f0 = st.as[p];
        const double d1 = t.c * f0;
        A.F.d[2][k] = ((t.mu * d1 + t.nu * 0.0) + t.hmut * F) + t.hgt * f0;
      } else if constexpr (MODE == M_STAGE3) {
        const double f0 = st.cf[pc];
        const double d1 = t.c * f0;
        A.F.d[0][k] = ((t.mu * st.as[p] + t.nu * d1) + t.hmut * F) + t.hgt * f0;
      } else if constexpr (MODE == M_STAGEN) {
        const double f0 = st.cf[pc];
        A.F.d[t.j % 3][k] = ((t.mu * st.as[p] + t.nu * st.cd[pc]) + t.hmut * F) + t.hgt * f0;
      } else if constexpr (MODE == M_FINAL) {
        const double ds = st.as[p], yv = st.ys[p], f0 = st.cf[pc];
        const double yn = yv + ds;
        A.F.f[1 - t.fi][k] = F;
        A.F.y[1 - t.yi][k] = yn;
        const double err = -0.8 * ds + t.h04 * (f0 + F);
        const double ay = fabs(yv), an = fabs(yn);
        const double mx = (ay >= an || isnan(ay)) ? ay : an;
        const double r = fabs(err) / (A.P.atol + A.P.rtol * mx);
        if (isfinite(r)) acc.ratio = r > acc.ratio ? r : acc.ratio;
        else acc.nonfin = 1;
      } else {
        const double diff = F - st.cf[pc];
        A.F.d[t.vout][k] = diff;
        ps += diff * diff;
      }
    }
  }
  *psum_item = ps;
}

template <bool P2, int MODE, int YM>
__device__ void chunk3(const WinArgs& A, const SubGeo& g, const Act& t, int it0, int nit,
                       Stage3* stage, Acc& acc, double* sh_sum) {
  constexpr bool SUMS = MODE == M_POWER || MODE == M_POWER_SEED || MODE == M_NORM;
  auto origin = [&](int item, int& c0, int& r0, int& z0) {
    const int ix = item % g.items_x;
    const int rest = item / g.items_x;
    c0 = ix * TX;
    r0 = (rest % g.items_y) * TY;
    z0 = (rest / g.items_y) * IZ3;
  };
  int c0, r0, z0, nc0 = 0, nr0 = 0, nz0 = 0;
  origin(it0, c0, r0, z0);
  issue3<MODE, YM>(A, g, t, c0, r0, z0, stage[0]);
  for (int i = 0; i < nit; ++i) {
    if (i + 1 < nit) {
      origin(it0 + i + 1, nc0, nr0, nz0);
      issue3<MODE, YM>(A, g, t, nc0, nr0, nz0, stage[(i + 1) & 1]);
      cpa_wait<1>();
    } else {
      cpa_wait<0>();
    }
    __syncthreads();
    constexpr bool COMBINED = MODE == M_STAGE2 || MODE == M_STAGE3 || MODE == M_STAGEN;
    if constexpr (COMBINED) {
      Stage3& sg = stage[i & 1];
      const int tid = threadIdx.y * TX + threadIdx.x;
      for (int e = tid; e < TD3 * TH3 * TW2; e += NT) {
        if constexpr (YM == YM_ADD) sg.ys[e] = sg.ys[e] + sg.as[e];
        else sg.ys[e] = sg.ys[e] + t.c * sg.as[e];
      }
      __syncthreads();
    }
    double ps = 0.0;
    compute3<P2, MODE, COMBINED ? YM_PLAIN : YM>(A, g, t, c0, r0, z0, stage[i & 1], acc, &ps);
    if constexpr (SUMS) {
      const double s = block_sum(ps, sh_sum);
      if (threadIdx.x == 0 && threadIdx.y == 0) __stcg(A.part + A.poff[t.sub] + it0 + i, s);
    } else {
      __syncthreads();
    }
    c0 = nc0;
    r0 = nr0;
    z0 = nz0;
  }
}

template <bool P2>
__device__ void dispatch_chunk3(const WinArgs& A, const SubGeo& g, const Act& t, int it0, int nit,
                                Stage3* st, Acc& acc, double* sh) {
  switch (t.mode) {
    case M_F0: chunk3<P2, M_F0, YM_PLAIN>(A, g, t, it0, nit, st, acc, sh); break;
    case M_EULER: chunk3<P2, M_EULER, YM_PLAIN>(A, g, t, it0, nit, st, acc, sh); break;
    case M_STAGE2: chunk3<P2, M_STAGE2, YM_SCALED>(A, g, t, it0, nit, st, acc, sh); break;
    case M_STAGE3: chunk3<P2, M_STAGE3, YM_ADD>(A, g, t, it0, nit, st, acc, sh); break;
    case M_STAGEN: chunk3<P2, M_STAGEN, YM_ADD>(A, g, t, it0, nit, st, acc, sh); break;
    case M_FINAL: chunk3<P2, M_FINAL, YM_ADD>(A, g, t, it0, nit, st, acc, sh); break;
    case M_POWER: chunk3<P2, M_POWER, YM_SCALED>(A, g, t, it0, nit, st, acc, sh); break;
    case M_POWER_SEED: chunk3<P2, M_POWER_SEED, YM_SEED>(A, g, t, it0, nit, st, acc, sh); break;
    case M_NORM: chunk3<P2, M_NORM, YM_PLAIN>(A, g, t, it0, nit, st, acc, sh); break;
    default: break;
  }
}

template <int DIM, bool P2>
__global__ void __launch_bounds__(NT, DIM == 2 ? DDPMA_MINB2 : 3) k_windowP(const WinArgs A) {
  using Stage = typename std::conditional<DIM == 2, Stage2, Stage3>::type;
  extern __shared__ __align__(128) unsigned char dsm[];
  Stage* stage = reinterpret_cast<Stage*>(
      dsm + ((128 - ((unsigned)__cvta_generic_to_shared(dsm) & 127u)) & 127u));
  __shared__ __align__(8) unsigned long long s_mbar[4];
  unsigned phases = 0u;
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    mbar_init(&s_mbar[0]);
    mbar_init(&s_mbar[1]);
    mbar_init_n(&s_mbar[2], NT / 32);
    mbar_init_n(&s_mbar[3], NT / 32);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int i = threadIdx.y * TX + threadIdx.x; i < 97 * 3; i += NT)
    (&s_logtab[0][0])[i] = (&kLogTabD[0][0])[i];
  __syncthreads();
  __shared__ double sh_sum[NT / 32];
  __shared__ unsigned long long sh_max[NT / 32];
  __shared__ Act s_act;
  __shared__ DevCtl s_ctl;
  __shared__ int s_sub, s_it0, s_nit, s_exit, s_last;
  const int tid = threadIdx.y * TX + threadIdx.x;
  unsigned backoff = 32;
  while (true) {
    if (threadIdx.y == 0) {
      // chunk of A.chunk_bulk items while many subdomains are active, A.chunk_tail on the tail
      const unsigned nd = *(volatile unsigned*)A.n_done;
      const int chunk = (A.nact - (int)nd) >= A.tail_n ? A.chunk_bulk : A.chunk_tail;
      int got, it0, nit;
      claim(A, chunk, got, it0, nit);
      if (threadIdx.x == 0) {
        s_sub = got;
        s_it0 = it0;
        s_nit = nit;
        s_exit = 0;
        if (got < 0) {
          s_exit = *(volatile unsigned*)A.n_done >= (unsigned)A.nact;
        } else {
          __threadfence();   // acquire
          // the previous action's data was written by other CTAs through the
          // generic proxy; the TMA loads of this chunk read it through the
          // async proxy (this thread issues them)
          asm volatile("fence.proxy.async.global;\n" ::: "memory");
          s_act = load_act(A, got);
          if (A.probe && got == A.probe_sub && it0 + nit == A.geo[got].nitems) {
            unsigned long long now;   // LAST chunk of the action claimed
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            const unsigned long long sq = (*(volatile unsigned long long*)&A.ctl[got].word) >> 32;
            A.probe[(sq % (unsigned long long)A.probe_cap) * 4 + 1] = now;
          }
        }
      }
    }
    __syncthreads();
    if (s_sub < 0) {
      if (s_exit) break;
      if (tid == 0) __nanosleep(backoff);
      backoff = backoff < 256 ? backoff * 2 : 256;
      __syncthreads();
      continue;
    }
    backoff = 32;
    const Act t = s_act;
    const int l = t.sub;
    const int it0 = s_it0, nit = s_nit;
    const SubGeo& g = A.geo[l];
    Acc acc{0u, 0u, 0.0, 0.0};
    if constexpr (DIM == 2)
      dispatch_chunk2<P2>(A, g, t, it0, nit, stage, acc, sh_sum, s_mbar, phases);
    else dispatch_chunk3<P2>(A, g, t, it0, nit, stage, acc, sh_sum);
    const int any = __syncthreads_or(acc.flag);
    const int anynf = __syncthreads_or(acc.nonfin);
    unsigned long long emax = 0ull;
    if (t.mode == M_FINAL)
      emax = block_max_u64((unsigned long long)__double_as_longlong(acc.ratio), sh_max);
    const bool sums = t.mode == M_POWER || t.mode == M_POWER_SEED || t.mode == M_NORM;
    if (tid == 0) {
      DevCtl* gc = A.ctl + l;
      unsigned bits = 0;
      if (any) bits |= t.mode == M_FINAL ? 2u : 1u;
      if (anynf) bits |= 4u;
      if (bits) atomicOr(&gc->acc_flags, bits);
      if (t.mode == M_FINAL) atomicMax(&gc->acc_emax, emax);
      __threadfence();
      const unsigned d = atomicAdd(&gc->done, (unsigned)nit);
      s_last = d + (unsigned)nit == (unsigned)g.nitems;
      if (s_last && A.probe && l == A.probe_sub) {
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        const unsigned long long sq = (*(volatile unsigned long long*)&gc->word) >> 32;
        A.probe[(sq % (unsigned long long)A.probe_cap) * 4 + 2] = now;
      }
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      double sum = 0.0;
      if (sums) {
        double v = 0.0;
        for (int i = tid; i < g.nitems; i += NT) v += __ldcg(A.part + A.poff[l] + i);
        sum = block_sum(v, sh_sum);
      }
      if (threadIdx.y == 0) decide(A, l, g, sum, s_ctl);
    }
    __syncthreads();
  }
}

// Window start for the active subdomains (one thread each): phase F0 /
// EULER, first action published.
__global__ void k_window_begin(const WinArgs A) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= A.nact) return;
  const int l = A.act[q];
  DevCtl* gc = A.ctl + l;
  DevCtl c;
  ctl_load(c, gc);
  c.fail_status = 0;
  c.j = 0;
  if (A.scheme == DDPMA_SCHEME_EULER_D) {
    c.phase = P_EULER;
    c.euler_left = A.substeps;
  } else {
    c.phase = P_F0;
  }
  c.word = (c.word & 0xffffffff00000000ull);
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(c.t_begin));
  d_publish(A, c, gc);
}

// ============================================================================
// Warp-specialised 2D window kernel (k_windowW): 8 consumer warps + 1
// producer warp per CTA.
//
// The producer warp claims chunks (claim-ahead: the next chunk is claimed
// while the consumers still work on the current one), publishes each chunk's
// action through a 2-slot mailbox (mbarriers cfull / cempty) and streams every
// item's tiles into an NS-deep ring of shared-memory stages with TMA (full[b]:
// transaction bytes; empty[b]: one arrival per consumer warp).  Consumers
// never meet the producer at a barrier; among themselves they synchronise
// only at chunk ends (named barrier 1) for the flag / error-ratio reductions
// and the completion accounting.  The per-item arithmetic is compute2_int /
// compute2 (bitwise identical to the other window kernels).
// ============================================================================

constexpr int NS2 = 3;                 // ring depth (stages) of k_windowW
constexpr int NTW = NT + 32;           // threads per CTA of k_windowW

__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }
__device__ __forceinline__ int cbar_or(int p) {
  int r;
  asm volatile(
      "{\n .reg .pred pi, po;\n setp.ne.s32 pi, %1, 0;\n"
      " bar.red.or.pred po, 1, 256, pi;\n selp.s32 %0, 1, 0, po;\n}\n"
      : "=r"(r)
      : "r"(p)
      : "memory");
  return r;
}
__device__ __forceinline__ double csum(double v, double* sh) {   // block_sum over consumers
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  if (threadIdx.x == 0) sh[threadIdx.y] = v;
  cbar();
  double tot = 0.0;
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    tot = sh[0];
    for (int w = 1; w < NT / 32; ++w) tot += sh[w];
  }
  cbar();
  return tot;
}
__device__ __forceinline__ unsigned long long cmax(unsigned long long v, unsigned long long* sh) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_down_sync(0xffffffffu, v, off);
    v = o > v ? o : v;
  }
  if (threadIdx.x == 0) sh[threadIdx.y] = v;
  cbar();
  unsigned long long m = 0;
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    m = sh[0];
    for (int w = 1; w < NT / 32; ++w) m = sh[w] > m ? sh[w] : m;
  }
  cbar();
  return m;
}

// Producer side: the TMA copies of one item for a runtime mode.
__device__ __forceinline__ void issue_any2(const WinArgs& A, const Act& t, int c0, int r0,
                                           Stage2& st, unsigned long long* mb) {
  switch (t.mode) {
    case M_F0: issue2_tma<M_F0, YM_PLAIN>(A, t.sub, t, c0, r0, st, mb); break;
    case M_EULER: issue2_tma<M_EULER, YM_PLAIN>(A, t.sub, t, c0, r0, st, mb); break;
    case M_STAGE2: issue2_tma<M_STAGE2, YM_SCALED>(A, t.sub, t, c0, r0, st, mb); break;
    case M_STAGE3: issue2_tma<M_STAGE3, YM_ADD>(A, t.sub, t, c0, r0, st, mb); break;
    case M_STAGEN: issue2_tma<M_STAGEN, YM_ADD>(A, t.sub, t, c0, r0, st, mb); break;
    case M_FINAL: issue2_tma<M_FINAL, YM_ADD>(A, t.sub, t, c0, r0, st, mb); break;
    case M_POWER: issue2_tma<M_POWER, YM_SCALED>(A, t.sub, t, c0, r0, st, mb); break;
    case M_POWER_SEED: issue2_tma<M_POWER_SEED, YM_SEED>(A, t.sub, t, c0, r0, st, mb); break;
    default: issue2_tma<M_NORM, YM_PLAIN>(A, t.sub, t, c0, r0, st, mb); break;
  }
}

// Consumer side of one chunk: n = ring position (items consumed so far).
template <bool P2, int MODE, int YM>
__device__ void cchunk2(const WinArgs& A, const SubGeo& g, const Act& t, int it0, int nit,
                        Stage2* stage, Acc& acc, double* sh_sum, unsigned long long* full,
                        unsigned long long* empty, unsigned& n) {
  constexpr bool SUMS = MODE == M_POWER || MODE == M_POWER_SEED || MODE == M_NORM;
  const int n0 = __ldg(&g.n[0]), n1 = __ldg(&g.n[1]), items_x = __ldg(&g.items_x);
  const long long pitch = __ldg(&g.pitch), goff = __ldg(&g.off);
  int ix = it0 % items_x, iy = it0 / items_x;
  for (int i = 0; i < nit; ++i, ++n) {
    const unsigned b = n % NS2, u = n / NS2;
    mbar_wait(&full[b], u & 1u);
    double ps = 0.0;
    const int c0 = ix * TX, r0 = iy * IR2;
    const long long kb = goff + (long long)r0 * pitch + c0 + threadIdx.x;
    if constexpr (SUMS) {
      compute2<P2, MODE, YM>(A, g, t, c0, r0, stage[b], acc, &ps);
    } else if (r0 >= 1 && r0 + IR2 <= n0 - 1 && c0 >= 1 && c0 + TX <= n1 - 1) {
      compute2_int<P2, MODE, YM, false>(A, g, t, kb, pitch, r0, c0, n0, n1, stage[b], acc);
    } else {
      compute2_int<P2, MODE, YM, true>(A, g, t, kb, pitch, r0, c0, n0, n1, stage[b], acc);
    }
    __syncwarp();
    if (threadIdx.x == 0) mbar_arrive(&empty[b]);   // this warp is done with stage b
    if (++ix == items_x) {
      ix = 0;
      ++iy;
    }
    if constexpr (SUMS) {
      const double sv = csum(ps, sh_sum);   // per-item partial: deterministic
      if (threadIdx.x == 0 && threadIdx.y == 0) __stcg(A.part + A.poff[t.sub] + it0 + i, sv);
    }
  }
}

template <bool P2>
__device__ void dispatch_cchunk2(const WinArgs& A, const SubGeo& g, const Act& t, int it0,
                                 int nit, Stage2* st, Acc& acc, double* sh,
                                 unsigned long long* fu, unsigned long long* em, unsigned& n) {
  switch (t.mode) {
    case M_F0: cchunk2<P2, M_F0, YM_PLAIN>(A, g, t, it0, nit, st, acc, sh, fu, em, n); break;
    case M_EULER: cchunk2<P2, M_EULER, YM_PLAIN>(A, g, t, it0, nit, st, acc, sh, fu, em, n); break;
    case M_STAGE2: cchunk2<P2, M_STAGE2, YM_SCALED>(A, g, t, it0, nit, st, acc, sh, fu, em, n); break;
    case M_STAGE3: cchunk2<P2, M_STAGE3, YM_ADD>(A, g, t, it0, nit, st, acc, sh, fu, em, n); break;
    case M_STAGEN: cchunk2<P2, M_STAGEN, YM_ADD>(A, g, t, it0, nit, st, acc, sh, fu, em, n); break;
    case M_FINAL: cchunk2<P2, M_FINAL, YM_ADD>(A, g, t, it0, nit, st, acc, sh, fu, em, n); break;
    case M_POWER: cchunk2<P2, M_POWER, YM_SCALED>(A, g, t, it0, nit, st, acc, sh, fu, em, n); break;
    case M_POWER_SEED:
      cchunk2<P2, M_POWER_SEED, YM_SEED>(A, g, t, it0, nit, st, acc, sh, fu, em, n);
      break;
    case M_NORM: cchunk2<P2, M_NORM, YM_PLAIN>(A, g, t, it0, nit, st, acc, sh, fu, em, n); break;
    default: break;
  }
}

struct ChunkSlot {
  Act t;
  int it0, nit, exit, pad;
};

template <bool P2>
__global__ void __launch_bounds__(NTW, 3) k_windowW(const WinArgs A) {
  extern __shared__ __align__(128) unsigned char dsm[];
  Stage2* stage = reinterpret_cast<Stage2*>(
      dsm + ((128 - ((unsigned)__cvta_generic_to_shared(dsm) & 127u)) & 127u));
  __shared__ __align__(8) unsigned long long s_full[NS2], s_empty[NS2], s_cfull[2], s_cempty[2];
  __shared__ ChunkSlot s_cs[2];
  __shared__ double sh_sum[NT / 32];
  __shared__ unsigned long long sh_max[NT / 32];
  __shared__ DevCtl s_ctl;
  __shared__ int s_last;
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    for (int b = 0; b < NS2; ++b) {
      mbar_init(&s_full[b]);
      mbar_init_n(&s_empty[b], NT / 32);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&s_cfull[k]);
      mbar_init(&s_cempty[k]);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int i = threadIdx.y * TX + threadIdx.x; i < 97 * 3; i += NTW)
    (&s_logtab[0][0])[i] = (&kLogTabD[0][0])[i];
  __syncthreads();

  if (threadIdx.y == TY) {
    // ---------------------------------------------------------- producer
    const int lane = threadIdx.x;
    unsigned n = 0;       // items issued
    int k = 0;            // chunks published
    unsigned backoff = 32;
    while (true) {
      const int slot = k & 1;
      if (k >= 2) mbar_wait(&s_cempty[slot], ((k >> 1) - 1) & 1);
      const unsigned nd = *(volatile unsigned*)A.n_done;
      const int chunk = (A.nact - (int)nd) >= A.tail_n ? A.chunk_bulk : A.chunk_tail;
      int got, it0, nit;
      claim(A, chunk, got, it0, nit);
      if (got < 0) {
        if (*(volatile unsigned*)A.n_done >= (unsigned)A.nact) {
          if (lane == 0) {
            s_cs[slot].exit = 1;
            mbar_arrive(&s_cfull[slot]);
          }
          break;
        }
        __nanosleep(backoff);
        backoff = backoff < 256 ? backoff * 2 : 256;
        continue;
      }
      backoff = 32;
      if (lane == 0) {
        __threadfence();   // acquire: the action and the data of the previous action
        asm volatile("fence.proxy.async.global;\n" ::: "memory");   // generic writes -> TMA reads
        const Act t = load_act(A, got);
        s_cs[slot].t = t;
        s_cs[slot].it0 = it0;
        s_cs[slot].nit = nit;
        s_cs[slot].exit = 0;
        mbar_arrive(&s_cfull[slot]);
        const int items_x = __ldg(&A.geo[got].items_x);
        int ix = it0 % items_x, iy = it0 / items_x;
        for (int i = 0; i < nit; ++i, ++n) {
          const unsigned b = n % NS2, u = n / NS2;
          if (u >= 1) mbar_wait(&s_empty[b], (u - 1) & 1u);
          issue_any2(A, t, ix * TX, iy * IR2, stage[b], &s_full[b]);
          if (++ix == items_x) {
            ix = 0;
            ++iy;
          }
        }
      }
      __syncwarp();
      ++k;
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const int tid = threadIdx.y * TX + threadIdx.x;
  unsigned n = 0;
  int k = 0;
  while (true) {
    const int slot = k & 1;
    mbar_wait(&s_cfull[slot], (k >> 1) & 1);
    const int ex = s_cs[slot].exit;
    // the action stays in the mailbox slot (read from shared memory where
    // used) until the chunk is complete; the slot is released at chunk end
    const Act& t = s_cs[slot].t;
    const int it0 = s_cs[slot].it0, nit = s_cs[slot].nit;
    ++k;
    if (ex) break;
    const int l = t.sub;
    const SubGeo& g = A.geo[l];
    Acc acc{0u, 0u, 0.0, 0.0};
    dispatch_cchunk2<P2>(A, g, t, it0, nit, stage, acc, sh_sum, s_full, s_empty, n);
    const int any = cbar_or(acc.flag);
    const int anynf = cbar_or(acc.nonfin);
    unsigned long long emax = 0ull;
    if (t.mode == M_FINAL)
      emax = cmax((unsigned long long)__double_as_longlong(acc.ratio), sh_max);
    const bool sums = t.mode == M_POWER || t.mode == M_POWER_SEED || t.mode == M_NORM;
    if (tid == 0) {
      DevCtl* gc = A.ctl + l;
      unsigned bits = 0;
      if (any) bits |= t.mode == M_FINAL ? 2u : 1u;
      if (anynf) bits |= 4u;
      if (bits) atomicOr(&gc->acc_flags, bits);
      if (t.mode == M_FINAL) atomicMax(&gc->acc_emax, emax);
      __threadfence();
      const unsigned d = atomicAdd(&gc->done, (unsigned)nit);
      s_last = d + (unsigned)nit == (unsigned)g.nitems;
    }
    cbar();
    if (s_last) {
      __threadfence();
      double sum = 0.0;
      if (sums) {
        double v = 0.0;
        for (int i = tid; i < g.nitems; i += NT) v += __ldcg(A.part + A.poff[l] + i);
        sum = csum(v, sh_sum);
      }
      if (threadIdx.y == 0) decide(A, l, g, sum, s_ctl);
    }
    cbar();
    if (tid == 0) mbar_arrive(&s_cempty[slot]);   // mailbox slot free
  }
}

}  // namespace

// DDPMA_WS=1 selects the warp-specialised 2D kernel k_windowW (default: the
// single-role k_windowP, measured faster on C3: 4 vs 3 resident CTAs per SM).
static bool window_ws() {
  static const int ws = getenv("DDPMA_WS") ? atoi(getenv("DDPMA_WS")) : 0;
  return ws != 0;
}

int window_blocks(int dim, int pow2) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (dim == 2 && window_ws()) {
    const int smem = NS2 * STAGE2_BYTES + 128;
    cudaFuncSetAttribute(k_windowW<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_windowW<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (pow2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_windowW<true>, NTW, smem);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_windowW<false>, NTW, smem);
  } else if (dim == 2) {
    const int smem = 2 * STAGE2_BYTES + 128;
    cudaFuncSetAttribute(k_windowP<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_windowP<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (pow2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_windowP<2, true>, NT, smem);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_windowP<2, false>, NT, smem);
  } else {
    const int smem = 2 * (int)sizeof(Stage3) + 128;
    cudaFuncSetAttribute(k_windowP<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_windowP<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (pow2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_windowP<3, true>, NT, smem);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_windowP<3, false>, NT, smem);
  }
  return sms * (per > 0 ? per : 1);
}

void launch_window_begin(const WinArgs& a, void* stream) {
  if (a.nact <= 0) return;
  k_window_begin<<<(a.nact + 63) / 64, 64, 0, (cudaStream_t)stream>>>(a);
}

void launch_window(const WinArgs& a, int nb, void* stream) {
  if (a.nact <= 0) return;
  const dim3 blk(TX, TY);
  void* args[] = {(void*)&a};
  void* fn;
  size_t smem = 0;
  if (a.P.dim == 2 && window_ws() && a.tmap != nullptr) {
    fn = a.P.pow2 ? (void*)k_windowW<true> : (void*)k_windowW<false>;
    smem = NS2 * STAGE2_BYTES + 128;
    cudaLaunchCooperativeKernel(fn, dim3(nb), dim3(TX, TY + 1), args, smem, (cudaStream_t)stream);
    return;
  } else if (a.P.dim == 2) {
    fn = a.P.pow2 ? (void*)k_windowP<2, true> : (void*)k_windowP<2, false>;
    smem = 2 * STAGE2_BYTES + 128;
  } else {
    fn = a.P.pow2 ? (void*)k_windowP<3, true> : (void*)k_windowP<3, false>;
    smem = 2 * sizeof(Stage3) + 128;
  }
  cudaLaunchCooperativeKernel(fn, dim3(nb), blk, args, smem, (cudaStream_t)stream);
}

}  // namespace ddpma
