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
#include "crpow.cuh"

#ifndef DDPMA_MINB2
#define DDPMA_MINB2 3   // resident CTAs per SM of the 2D window kernels (register cap 80)
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
__device__ __forceinline__ unsigned w_cursor(unsigned long long w) {
  return (unsigned)(w & kWordCurMask);
}
__device__ __forceinline__ unsigned w_ntasks(unsigned long long w) {
  return (unsigned)((w >> kWordCurBits) & kWordCurMask);
}
__device__ __forceinline__ unsigned long long w_seq(unsigned long long w) { return w >> 48; }
__device__ __forceinline__ unsigned long long w_make(unsigned long long seq, unsigned ntasks) {
  return (seq << 48) | ((unsigned long long)ntasks << kWordCurBits);
}

// Shared-memory copy of the log table (filled at the start of k_windowP;
// the table lookups are the fp64 log's only memory accesses).
__shared__ double s_logtab[97][3];

// coherent (L2) loads of mutable data
__device__ __forceinline__ double ldc(const double* p) { return __ldcg(p); }

// ------------------------------------------------------------- accessors --

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
  int mode = c.a_mode;
  if (mode == M_SWEEP) {   // stages 2..s and the final evaluation of one step
    const int s = c.a_s;
    c.bytes += (32.0 + (s >= 3 ? 40.0 : 0.0) + 48.0 * (double)(s - 3 > 0 ? s - 3 : 0) + 48.0) *
               (double)nodes;
    c.evals += s;
    c.sbase += (unsigned long long)s * (unsigned long long)A.geo[l].ipr;
    c.step_flag = (c.acc_flags & 1u) ? 1 : 0;
    mode = M_FINAL;
  } else {
    c.bytes += mode_bytes_d(mode) * (double)nodes;
    if (mode != M_NORM) c.evals += 1;
  }
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
          const double gg = 0.8 * pow_m13_rn(emax);   // crpow.cuh: glibc-faithful pow
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
          const double gg = 0.8 * pow_m13_rn(emax);   // crpow.cuh: glibc-faithful pow
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
__device__ bool d_next_action(const WinArgs& A, DevCtl& c, int nitems) {
  c.a_yi = c.yi;
  c.a_fi = c.fi;
  c.a_s = c.s;
  c.a_ntasks = nitems;
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
      if (A.sweep) {   // the whole step (stages 2..s, final) as one dataflow action
        c.a_mode = M_SWEEP;
        c.a_h = c.h;
        c.a_h04 = 0.4 * c.h;
        c.a_sbase = c.sbase;
        c.a_ntasks = c.s * nitems;
        return true;
      }
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
__device__ void d_publish(const WinArgs& A, DevCtl& c, DevCtl* gc, int nitems) {
  const unsigned long long seq = w_seq(c.word) + 1;
  const bool more = d_next_action(A, c, nitems);
  c.acc_flags = 0;
  c.acc_emax = 0ull;
  c.done = 0;
  ctl_store(gc, c);
  __threadfence();
  if (more) {
    atomicExch(&gc->word, w_make(seq, (unsigned)c.a_ntasks));
  } else {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    __stcg(reinterpret_cast<long long*>(&gc->t_done), (long long)now);
    atomicExch(&gc->word, w_make(seq, 0u));
    atomicAdd(A.n_done, 1u);
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
#ifndef DDPMA_RING2
#define DDPMA_RING2 2
#endif
constexpr int RD2 = DDPMA_RING2;   // depth of k_windowP<2>'s TMA tile ring

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

// Determinant at a box-face node that is NOT Dirichlet.  Inside the window
// kernels every non-physical box face is an interface (Dirichlet) face, so such
// a node lies on physical faces only: per axis the second difference is the
// interior formula or the Neumann-ghost formula of _second_diff
// (pma.py:87-115, d2ax), the cross term is zero on a physical face
// (pma.py:118-130, cross) -- every Y it needs is within one node, i.e. inside
// the staged tile.  Same expressions, same order as hdet<2>'s generic branch
// (bitwise identical); the one-sided 4-point formulas of hdet<> can never be
// reached here and are not instantiated (they were most of the kernel's code).
template <bool P2, int YM>
__device__ __forceinline__ double hdet2_face(const Prob& P, const SubGeo& g, int i0, int i1,
                                             const Stage2& st, int p, double c, int par) {
  const int n0 = g.n[0], n1 = g.n[1];
  const double yc = yat<YM>(st, p, c, par);
  double h00, h11, h01 = 0.0;
  if (i0 == 0)
    h00 = dv<P2>(2.0 * ((yat<YM>(st, p + TW2, c, par ^ 1) - yc) - g.halo[0]), P.ax[0].hh, P.ax[0].ihh);
  else if (i0 == n0 - 1)
    h00 = dv<P2>(2.0 * ((yat<YM>(st, p - TW2, c, par ^ 1) - yc) + g.hahi[0]), P.ax[0].hh, P.ax[0].ihh);
  else
    h00 = dv<P2>((yat<YM>(st, p + TW2, c, par ^ 1) - 2.0 * yc) + yat<YM>(st, p - TW2, c, par ^ 1),
                 P.ax[0].hh, P.ax[0].ihh);
  if (i1 == 0)
    h11 = dv<P2>(2.0 * ((yat<YM>(st, p + 1, c, par ^ 1) - yc) - g.halo[1]), P.ax[1].hh, P.ax[1].ihh);
  else if (i1 == n1 - 1)
    h11 = dv<P2>(2.0 * ((yat<YM>(st, p - 1, c, par ^ 1) - yc) + g.hahi[1]), P.ax[1].hh, P.ax[1].ihh);
  else
    h11 = dv<P2>((yat<YM>(st, p + 1, c, par ^ 1) - 2.0 * yc) + yat<YM>(st, p - 1, c, par ^ 1),
                 P.ax[1].hh, P.ax[1].ihh);
  if (!(i0 == 0 || i0 == n0 - 1 || i1 == 0 || i1 == n1 - 1)) {
    const double gp = dv<P2>(yat<YM>(st, p + TW2 + 1, c, par) - yat<YM>(st, p + TW2 - 1, c, par),
                             P.ax[1].twoh, P.ax[1].itwoh);
    const double gm = dv<P2>(yat<YM>(st, p - TW2 + 1, c, par) - yat<YM>(st, p - TW2 - 1, c, par),
                             P.ax[1].twoh, P.ax[1].itwoh);
    h01 = dv<P2>(gp - gm, P.ax[0].twoh, P.ax[0].itwoh);
  }
  return h00 * h11 - h01 * h01;
}

template <bool P2, int MODE, int YM>
__device__ __forceinline__ void compute2(const WinArgs& A, const SubGeo& g, const Act& t, int c0,
                                         int r0, const Stage2& st, Acc& acc, double* psum_item) {
  constexpr int R = IR2 / TY;
  const int n0 = g.n[0], n1 = g.n[1];
  const int i1 = c0 + threadIdx.x;
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
            const int lr = threadIdx.y + q * TY;
            det[q] = hdet2_face<P2, YM>(A.P, g, i0, i1, st, (lr + 1) * TW2 + threadIdx.x + 2, t.c,
                                        (i0 + i1) & 1);
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
    const int i1 = c0 + tx;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int i0 = r0 + lr + q;
      if (!(i0 < n0 && i1 < n1)) {
        valid &= ~(1u << q);
      } else if (i0 == 0 || i0 == n0 - 1 || i1 == 0 || i1 == n1 - 1) {
        if (dirichlet<2>(g, i0, i1, 0)) dirm |= 1u << q;
        else det[q] = hdet2_face<P2, YM>(A.P, g, i0, i1, st, p + q * TW2, t.c, par ^ q);
      }
    }
  }
  {
    // nodes past the box (EDGE) carry zero-filled tiles: no F needed either
    const unsigned skip = dirm | (~valid & 3u);
    const double mrv[2] = {st.cm[lr * TX + tx], st.cm[(lr + 1) * TX + tx]};
    const double g_ = A.P.guard;
    logequi_pair(mrv, det, skip, g_, A.P.floor, A.P.rguard, g_ >= 0x1p-900 && g_ < 0x1p900, s_logtab, F);
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const bool dir = (dirm >> q) & 1u;
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
    int mychunk = chunk;
    if (q < A.nact) {
      l = A.act[q];
      const unsigned long long w = *(volatile unsigned long long*)&A.ctl[l].word;
      claimable = w_cursor(w) < w_ntasks(w);
      // bulk phase: the subdomain's own chunk size (small for the subdomains
      // whose sequential chain of actions would otherwise outlast the window)
      if (A.chunk_q != nullptr && chunk == A.chunk_bulk) mychunk = __ldg(A.chunk_q + q);
    }
    unsigned mask = __ballot_sync(0xffffffffu, claimable);
    while (mask != 0u && got < 0) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1u;
      int it = -1, n = 0;
      if (lane == src) {
        const int chunk = mychunk;
        const unsigned long long w2 = atomicAdd(&A.ctl[l].word, (unsigned long long)chunk);
        const unsigned u = w_cursor(w2);
        const unsigned ni = w_ntasks(w2);
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
    seq = w_seq(s_ctl.word) + 1;
    more = d_next_action(A, s_ctl, g.nitems);
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
      atomicExch(&gc->word, w_make(seq, (unsigned)s_ctl.a_ntasks));
    } else {
      atomicExch(&gc->word, w_make(seq, 0u));
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
  const bool tma = A.tmap != nullptr;
  const bool lead = threadIdx.x == 0 && threadIdx.y == 0;
  // TMA pipeline, RD2 stages deep: mbar[b] = "buffer b full" (1 arrival + tx
  // bytes), mbar[RD2+b] = "buffer b consumed" (one arrival per warp).  phases:
  // bits [0,RD2) full parity, [RD2,2RD2) consumed parity, [2RD2,3RD2) buffer
  // used before.  The issuing thread waits for the previous use of a buffer
  // to be consumed by every warp, so warps never meet at a CTA barrier
  // between items; item i+RD2-1 is in flight while item i is computed.
  auto issue = [&](int b, int item) {
    if ((phases >> (2 * RD2 + b)) & 1u) {
      mbar_wait(&mbar[RD2 + b], (phases >> (RD2 + b)) & 1u);
      phases ^= 1u << (RD2 + b);
    }
    phases |= 1u << (2 * RD2 + b);
    const int cy = item / items_x, cx = item - cy * items_x;
    issue2_tma<MODE, YM>(A, t.sub, t, cx * TX, cy * IR2, stage[b], &mbar[b]);
  };
  // item -> (column, row) tile origin, decoded once per chunk then stepped
  int ix = it0 % items_x, iy = it0 / items_x;
  int nx = ix + 1, ny = iy;
  if (nx == items_x) {
    nx = 0;
    ++ny;
  }
  if (tma) {
    if (lead)
      for (int k = 0; k < RD2 - 1 && k < nit; ++k) issue(k, it0 + k);
  } else {
    issue2<MODE, YM>(A, g, t, ix * TX, iy * IR2, stage[0]);
  }
  for (int i = 0; i < nit; ++i) {
    const int s = tma ? i % RD2 : (i & 1);
    if (tma) {
      if (i + RD2 - 1 < nit && lead) issue((i + RD2 - 1) % RD2, it0 + i + RD2 - 1);
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
      if (threadIdx.x == 0) mbar_arrive(&mbar[RD2 + s]);   // this warp is done with buffer s
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

__device__ __forceinline__ void tma3(void* dst, const void* tmap, int x, int y, int z,
                                     unsigned long long* m) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(m))
      : "memory");
}

// One thread: the TMA copies of one 3D item into stage `st` (the halo boxes
// of y and the a field, 36 x (TY+2) x (IZ3+2) at (c0-2, r0-1, z0-1), and the
// TX x TY x IZ3 centre boxes; zero fill outside the box), completion on `mbar`.
template <int MODE, int YM>
__device__ __forceinline__ void issue3_tma(const WinArgs& A, int l, const Act& t, int c0, int r0,
                                           int z0, Stage3& st, unsigned long long* mbar) {
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
  constexpr unsigned HALO = TD3 * TH3 * TW2 * 8, CEN = IZ3 * TY * TX * 8;
  unsigned bytes = HALO;
  if constexpr (HAS_A) bytes += HALO;
  if constexpr (MODE != M_NORM) {
    bytes += CEN;
    if constexpr (NEED_F0) bytes += CEN;
    if constexpr (MODE == M_STAGEN) bytes += CEN;
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  mbar_expect(mbar, bytes);
  tma3(st.ys, map(TF_Y0 + t.yi, 0), c0 - 2, r0 - 1, z0 - 1, mbar);
  if constexpr (HAS_A) tma3(st.as, map(fa, 0), c0 - 2, r0 - 1, z0 - 1, mbar);
  if constexpr (MODE != M_NORM) {
    tma3(st.cm, map(TF_MR, 1), c0, r0, z0, mbar);
    if constexpr (NEED_F0) tma3(st.cf, map(TF_F0 + t.fi, 1), c0, r0, z0, mbar);
    if constexpr (MODE == M_STAGEN) tma3(st.cd, map(TF_D0 + (t.j - 2) % 3, 1), c0, r0, z0, mbar);
  }
}

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

// 3D twin of hdet2_face: the determinant at a non-Dirichlet box-face node
// (physical faces only), every Y from the staged tile; hdet<3>'s generic
// branch restricted to the formulas reachable here, same expressions and
// order (bitwise identical).
template <bool P2, int YM>
__device__ __forceinline__ double hdet3_face(const Prob& P, const SubGeo& g, int i0, int i1,
                                             int i2, const Stage3& st, int p, double c, int par) {
  const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];
  const double yc = yat3<YM>(st, p, c, par);
  auto Y1 = [&](int off) { return yat3<YM>(st, p + off, c, par ^ 1); };   // one axis step
  auto Y2 = [&](int off) { return yat3<YM>(st, p + off, c, par); };       // two axis steps
  auto d2 = [&](int ax, int i, int n, int off) {
    if (i == 0) return dv<P2>(2.0 * ((Y1(off) - yc) - g.halo[ax]), P.ax[ax].hh, P.ax[ax].ihh);
    if (i == n - 1) return dv<P2>(2.0 * ((Y1(-off) - yc) + g.hahi[ax]), P.ax[ax].hh, P.ax[ax].ihh);
    return dv<P2>((Y1(off) - 2.0 * yc) + Y1(-off), P.ax[ax].hh, P.ax[ax].ihh);
  };
  const double h00 = d2(0, i0, n0, SZ3);
  const double h11 = d2(1, i1, n1, SY3);
  const double h22 = d2(2, i2, n2, 1);
  const bool on0 = i0 == 0 || i0 == n0 - 1, on1 = i1 == 0 || i1 == n1 - 1,
             on2 = i2 == 0 || i2 == n2 - 1;
  auto cr = [&](bool onface, int k, int l, int offk, int offl) {   // d/dk of d/dl
    if (onface) return 0.0;
    const double gp = dv<P2>(Y2(offk + offl) - Y2(offk - offl), P.ax[l].twoh, P.ax[l].itwoh);
    const double gm = dv<P2>(Y2(-offk + offl) - Y2(-offk - offl), P.ax[l].twoh, P.ax[l].itwoh);
    return dv<P2>(gp - gm, P.ax[k].twoh, P.ax[k].itwoh);
  };
  const double h01 = cr(on0 || on1, 0, 1, SZ3, SY3);
  const double h02 = cr(on0 || on2, 0, 2, SZ3, 1);
  const double h12 = cr(on1 || on2, 1, 2, SY3, 1);
  return (h00 * (h11 * h22 - h12 * h12) - h01 * (h01 * h22 - h12 * h02)) +
         h02 * (h01 * h12 - h11 * h02);
}

template <bool P2, int MODE, int YM>
__device__ __forceinline__ void compute3(const WinArgs& A, const SubGeo& g, const Act& t, int c0,
                                         int r0, int z0, const Stage3& st, Acc& acc,
                                         double* psum_item) {
  const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];
  const int i1 = r0 + threadIdx.y, i2 = c0 + threadIdx.x;
  const long long plane = (long long)n1 * g.pitch;
  static_assert(IZ3 == 2, "logequi_pair handles the two nodes of a thread");
  double ps = 0.0;
  double detq[IZ3] = {1.0, 1.0}, Fq[IZ3] = {0.0, 0.0};
  unsigned validm = 0u, dirm = 0u;   // bit q: node q inside the box / on an interface face
  // phase 1: determinants of both nodes
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
      }
      // box-face nodes: interface (Dirichlet) faces need no determinant (F = 0,
      // never flagged); physical faces take the Neumann-ghost formulas
      const bool dir = !interior && dirichlet<3>(g, i0, i1, i2);
      // box-face nodes: interface (Dirichlet) faces need no determinant (F = 0,
      // never flagged); physical faces take the Neumann-ghost formulas
      if (!interior)
        det = dir ? 0.0
                  : hdet3_face<P2, YM>(A.P, g, i0, i1, i2, st, p, t.c, (i0 + i1 + i2) & 1);
      detq[q] = det;
      validm |= 1u << q;
      dirm |= dir ? (1u << q) : 0u;
    }
  }
  if constexpr (MODE != M_NORM) {
    // phase 2: log-equidistribution of both nodes, interleaved (logequi_pair)
    const double mrv[2] = {st.cm[threadIdx.y * TX + threadIdx.x],
                           st.cm[(TY + threadIdx.y) * TX + threadIdx.x]};
    const double g_ = A.P.guard;
    logequi_pair(mrv, detq, dirm | (~validm & 3u), g_, A.P.floor, A.P.rguard,
                 g_ >= 0x1p-900 && g_ < 0x1p900, s_logtab, Fq);
    // phase 3: epilogues
#pragma unroll
    for (int q = 0; q < IZ3; ++q) {
      if (!((validm >> q) & 1u)) continue;
      const int i0 = z0 + q;
      const int p = ((q + 1) * TH3 + threadIdx.y + 1) * TW2 + threadIdx.x + 2;
      const int pc = (q * TY + threadIdx.y) * TX + threadIdx.x;
      const long long k = g.off + i0 * plane + (long long)i1 * g.pitch + i2;
      const bool dir = (dirm >> q) & 1u;
      const double F = Fq[q];
      acc.flag |= (detq[q] <= A.P.floor && !dir) ? 1u : 0u;
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
                       Stage3* stage, Acc& acc, double* sh_sum, unsigned long long* mbar,
                       unsigned& phases) {
  constexpr bool SUMS = MODE == M_POWER || MODE == M_POWER_SEED || MODE == M_NORM;
  auto origin = [&](int item, int& c0, int& r0, int& z0) {
    const int ix = item % g.items_x;
    const int rest = item / g.items_x;
    c0 = ix * TX;
    r0 = (rest % g.items_y) * TY;
    z0 = (rest / g.items_y) * IZ3;
  };
  // TMA (cp.async.bulk.tensor.3d) with mbarrier completion when the plan has
  // 3D tensor maps; cp.async otherwise.  TMA pipeline as in chunk2: mbar[b] =
  // "buffer b full", mbar[2+b] = "buffer b consumed" (one arrival per warp);
  // the issuing thread waits for the previous use of a buffer to be consumed,
  // so no CTA barrier ends an item.
  const bool tma = A.tmap != nullptr;
  const bool lead = threadIdx.x == 0 && threadIdx.y == 0;
  int c0, r0, z0, nc0 = 0, nr0 = 0, nz0 = 0;
  origin(it0, c0, r0, z0);
  auto issue = [&](int b, int x, int y, int z) {
    if ((phases >> (4 + b)) & 1u) {
      mbar_wait(&mbar[2 + b], (phases >> (2 + b)) & 1u);
      phases ^= 1u << (2 + b);
    }
    phases |= 1u << (4 + b);
    issue3_tma<MODE, YM>(A, t.sub, t, x, y, z, stage[b], &mbar[b]);
  };
  if (tma) {
    if (lead) issue(0, c0, r0, z0);
  } else {
    issue3<MODE, YM>(A, g, t, c0, r0, z0, stage[0]);
  }
  for (int i = 0; i < nit; ++i) {
    const int sb = i & 1;
    if (i + 1 < nit) {
      origin(it0 + i + 1, nc0, nr0, nz0);
      if (tma) {
        if (lead) issue(sb ^ 1, nc0, nr0, nz0);
      } else {
        issue3<MODE, YM>(A, g, t, nc0, nr0, nz0, stage[sb ^ 1]);
        cpa_wait<1>();
      }
    } else if (!tma) {
      cpa_wait<0>();
    }
    if (tma) {
      mbar_wait(&mbar[sb], (phases >> sb) & 1u);
      phases ^= 1u << sb;
    } else {
      __syncthreads();
    }
#ifndef DDPMA_3D_COMBINED
#define DDPMA_3D_COMBINED 1
#endif
    // COMBINED: Y = y + a (stage increments) formed once per tile element in
    // shared memory instead of once per stencil read
    constexpr bool COMBINED = DDPMA_3D_COMBINED && (MODE == M_STAGE2 || MODE == M_STAGE3 || MODE == M_STAGEN);
    if constexpr (COMBINED) {
      Stage3& sg = stage[sb];
      const int tid = threadIdx.y * TX + threadIdx.x;
      for (int e = tid; e < TD3 * TH3 * TW2; e += NT) {
        if constexpr (YM == YM_ADD) sg.ys[e] = sg.ys[e] + sg.as[e];
        else sg.ys[e] = sg.ys[e] + t.c * sg.as[e];
      }
      __syncthreads();
    }
    double ps = 0.0;
    compute3<P2, MODE, COMBINED ? YM_PLAIN : YM>(A, g, t, c0, r0, z0, stage[sb], acc, &ps);
    if (tma) {
      __syncwarp();
      if (threadIdx.x == 0) mbar_arrive(&mbar[2 + sb]);   // this warp is done with buffer sb
    }
    if constexpr (SUMS) {
      const double s = block_sum(ps, sh_sum);
      if (threadIdx.x == 0 && threadIdx.y == 0) __stcg(A.part + A.poff[t.sub] + it0 + i, s);
    } else {
      if (!tma) __syncthreads();   // the stage buffer is refilled by the next iteration's issue
    }
    c0 = nc0;
    r0 = nr0;
    z0 = nz0;
  }
}

template <bool P2>
__device__ void dispatch_chunk3(const WinArgs& A, const SubGeo& g, const Act& t, int it0, int nit,
                                Stage3* st, Acc& acc, double* sh, unsigned long long* mb,
                                unsigned& ph) {
  switch (t.mode) {
    case M_F0: chunk3<P2, M_F0, YM_PLAIN>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    case M_EULER: chunk3<P2, M_EULER, YM_PLAIN>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    case M_STAGE2: chunk3<P2, M_STAGE2, YM_SCALED>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    case M_STAGE3: chunk3<P2, M_STAGE3, YM_ADD>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    case M_STAGEN: chunk3<P2, M_STAGEN, YM_ADD>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    case M_FINAL: chunk3<P2, M_FINAL, YM_ADD>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    case M_POWER: chunk3<P2, M_POWER, YM_SCALED>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    case M_POWER_SEED:
      chunk3<P2, M_POWER_SEED, YM_SEED>(A, g, t, it0, nit, st, acc, sh, mb, ph);
      break;
    case M_NORM: chunk3<P2, M_NORM, YM_PLAIN>(A, g, t, it0, nit, st, acc, sh, mb, ph); break;
    default: break;
  }
}

template <int DIM, bool P2>
__global__ void __launch_bounds__(NT, DIM == 2 ? DDPMA_MINB2 : 3) k_windowP(const __grid_constant__ WinArgs A) {
  using Stage = typename std::conditional<DIM == 2, Stage2, Stage3>::type;
  extern __shared__ __align__(128) unsigned char dsm[];
  Stage* stage = reinterpret_cast<Stage*>(
      dsm + ((128 - ((unsigned)__cvta_generic_to_shared(dsm) & 127u)) & 127u));
  constexpr int RD = DIM == 2 ? RD2 : 2;   // ring depth: full barriers [0,RD), consumed [RD,2RD)
  __shared__ __align__(8) unsigned long long s_mbar[2 * RD];
  unsigned phases = 0u;
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    for (int b = 0; b < RD; ++b) {
      mbar_init(&s_mbar[b]);
      mbar_init_n(&s_mbar[RD + b], NT / 32);
    }
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
  __shared__ unsigned s_bits;
  __shared__ unsigned long long s_emax;
  const int tid = threadIdx.y * TX + threadIdx.x;
  if (tid == 0) {
    s_bits = 0u;
    s_emax = 0ull;
  }
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
          if (A.proxy_fence) asm volatile("fence.proxy.async.global;\n" ::: "memory");
          s_act = load_act(A, got);
          if (A.probe && got == A.probe_sub && it0 + nit == A.geo[got].nitems) {
            unsigned long long now;   // LAST chunk of the action claimed
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            const unsigned long long sq = w_seq(*(volatile unsigned long long*)&A.ctl[got].word);
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
    else dispatch_chunk3<P2>(A, g, t, it0, nit, stage, acc, sh_sum, s_mbar, phases);
    // chunk completion: flags / error ratio folded per warp (shuffles), then
    // through shared accumulators -- one CTA barrier, not one per quantity
    {
      const unsigned wb = __reduce_or_sync(0xffffffffu, (acc.flag ? 1u : 0u) | (acc.nonfin ? 4u : 0u));
      unsigned long long em = (unsigned long long)__double_as_longlong(acc.ratio);
      if (t.mode == M_FINAL) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const unsigned long long o = __shfl_down_sync(0xffffffffu, em, off);
          em = o > em ? o : em;
        }
      }
      if (threadIdx.x == 0) {
        if (wb) atomicOr(&s_bits, wb);
        if (t.mode == M_FINAL && em) atomicMax(&s_emax, em);
      }
    }
    __syncthreads();
    // Completion bookkeeping (global atomics, ~1.5 us of round trips) runs on
    // warp 1 while warp 0 already claims the next chunk: the two latencies
    // overlap instead of adding up at every chunk boundary.  The actions with
    // a partial sum (norm / power iteration: rare) need every thread for the
    // fixed-order reduction and keep the serial form.
    const bool sums = t.mode == M_POWER || t.mode == M_POWER_SEED || t.mode == M_NORM;
    auto complete = [&]() -> int {   // one thread: publish this chunk's results
      DevCtl* gc = A.ctl + l;
      const unsigned wb = s_bits;
      const unsigned long long emax = s_emax;
      s_bits = 0u;
      s_emax = 0ull;
      unsigned bits = 0;
      if (wb & 1u) bits |= t.mode == M_FINAL ? 2u : 1u;
      if (wb & 4u) bits |= 4u;
      if (bits) atomicOr(&gc->acc_flags, bits);
      if (t.mode == M_FINAL) atomicMax(&gc->acc_emax, emax);
      __threadfence();
      const unsigned d = atomicAdd(&gc->done, (unsigned)nit);
      const int last = d + (unsigned)nit == (unsigned)g.nitems;
      if (last && A.probe && l == A.probe_sub) {
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        const unsigned long long sq = w_seq(*(volatile unsigned long long*)&gc->word);
        A.probe[(sq % (unsigned long long)A.probe_cap) * 4 + 2] = now;
      }
      return last;
    };
    if (!sums) {
      if (threadIdx.y == 1) {
        int last = 0;
        if (threadIdx.x == 0) last = complete();
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          __threadfence();
          decide(A, l, g, 0.0, s_ctl);
        }
      }
    } else {
      if (tid == 0) s_last = complete();
      __syncthreads();
      if (s_last) {
        __threadfence();
        double v = 0.0;
        for (int i = tid; i < g.nitems; i += NT) v += __ldcg(A.part + A.poff[l] + i);
        const double sum = block_sum(v, sh_sum);
        if (threadIdx.y == 0) decide(A, l, g, sum, s_ctl);
      }
    }
    // no barrier here: the other warps wait for warp 0's next claim at the top
    // of the loop; nothing they still read is written before that barrier
  }
}

// ============================================================================
// Dataflow 2D window kernel (k_windowD).
//
// An RKC2 step of a subdomain (stages 2..s and the final evaluation,
// integrate.py:163-178) is published as ONE action, M_SWEEP, of s * nitems
// tasks (level, item), level = j - 2.  Stage j at an item reads the stage
// j-1 increments only in the item and its 8 neighbours (the 9-point stencil
// of pma.py:87-149), so no stage needs a barrier over the whole box: a task
// of level L in item row r is ready once rows r-1..r+1 completed level L-1,
// which the per-row counters rowprog[] record (every completed sweep task
// adds 1 to its row).  The 3-slot d ring of the stage recurrence stays safe
// under that rule: the task that overwrites d_{j-2} at an item runs after
// level j-1 completed in its rows and level j-2 completed two rows around.
// The controller (accept/reject, error norm, sigma) still runs once per step,
// when the last task of the sweep completes.  Levels of one subdomain thus
// pipeline like a wavefront, and a single straggling subdomain keeps the
// whole GPU busy (its tail used to run stage by stage on a few CTAs).
//
// Inside a CTA nothing waits on a CTA-wide barrier: warp 0 lane 0 claims
// tasks and streams their tiles with TMA into a 2-deep ring of stages, each
// slot carrying its task descriptor; every warp computes its rows of the
// item, folds its flags / error ratio / partial sum into the slot and counts
// itself done with a CTA-scope acquire-release atomic; the warp that
// completes an item publishes it (row counter, action completion) and, when
// it completes an action, runs the controller (decide) on its own -- the
// other warps keep streaming.  Warp 0 only blocks waiting for work when it
// has consumed every item it issued, so a task it waits for can never be one
// its own CTA still has to compute.
//
// Per-node arithmetic (compute2_int / compute2) and every reduction order are
// those of k_windowP, so both kernels give bitwise identical results.
// ============================================================================

#ifndef DDPMA_NBD
#define DDPMA_NBD 2
#endif
constexpr int NBD = DDPMA_NBD;        // ring depth of k_windowD
constexpr int NWD = NT / 32;          // warps per CTA
constexpr int M_EXIT = 99;            // ring-slot marker: no more work

struct SlotD {                        // the task whose tiles occupy stage[b]
  Act t;
  int item, batch;
  unsigned cnt;                       // warps done with the item (CTA-scope atomic)
  unsigned wflag[NWD];                // per warp: bit0 flag, bit2 non-finite ratio
  unsigned long long wemax[NWD];      // per warp: max error ratio (FINAL)
  double wpsum[NWD];                  // per warp: partial sum (NORM / POWER)
};

// Completion accounting is batched: consecutive tasks of one claimed chunk
// that share an item row (same cell of a sweep) form a batch; the warp that
// completes a batch's last item publishes the whole batch with one fence and
// one atomic per counter (row progress, action completion).
constexpr int NBB = NBD + 2;          // batch records (>= NBD + 2: see fill_ring_d)
struct BatchD {
  int sub, row, sweep, ntasks;
  int size, final_, pad0, pad1;
  unsigned done;                      // items completed (CTA-scope atomic)
  unsigned flags;                     // ctl acc_flags bits of the batch's items
  unsigned long long emax;            // max error ratio (FINAL items)
  volatile int busy;                  // open: set by the issuer, cleared by the flusher
};

struct QueueD {                       // issuer state (warp 0 lane 0)
  int sub, next, end, issued;         // claimed tasks [next, end) of subdomain sub
  int bleft, bcur, nbatch, fence;     // open batch: items still to issue, record, count;
                                      // fence: acquire + proxy fence due before the next TMA
  int lock;                           // the ring filler's lock (one warp at a time)
  int nfold;                          // items completed and published by their last warp
  int mode, ntasks, nitems, ipr, nrows;
  int kr_sub, kr_row, kr_lev;         // known: levels < kr_lev complete around kr_row
  unsigned long long sbase, kr_base;
  double h;
  Act base;                           // the claimed action (yi, fi, s, c, h04, ...)
};

__device__ __forceinline__ unsigned atom_add_acqrel_cta(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;"
               : "=r"(old)
               : "r"(smem_u32(p)), "r"(v)
               : "memory");
  return old;
}

__device__ __forceinline__ bool mbar_test(unsigned long long* m, unsigned phase) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(m)), "r"(phase)
      : "memory");
  return ok != 0;
}

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

// Sweep tasks are enumerated level-major (task = level * nitems + item):
// with readiness-aware claiming, level L+1 starts in the first item rows as
// soon as their neighbourhood completed level L, so consecutive levels of one
// subdomain overlap by most of a level.
// Readiness of sweep task tau of subdomain l (rows row-1..row+1 completed
// level lev-1); returns the number of levels completed around the row.
__device__ __forceinline__ long long sweep_levels_done(const WinArgs& A, const SubGeo& g, int row,
                                                       unsigned long long sbase) {
  const int r0 = row > 0 ? row - 1 : 0;
  const int r1 = row + 1 < g.nrows ? row + 1 : g.nrows - 1;
  const unsigned long long* rp = A.rowprog + g.rowoff;
  unsigned long long m = ~0ull;
  for (int r = r0; r <= r1; ++r) {
    const unsigned long long v = *(volatile const unsigned long long*)(rp + r);
    m = v < m ? v : m;
  }
  return m >= sbase ? (long long)((m - sbase) / (unsigned long long)g.ipr) : 0;
}

// Claim (warp 0, k_windowD): like claim(), but a sweep is only claimed when
// the task at its cursor is ready, so CTAs spread over the subdomains'
// ready wavefronts instead of queueing behind one.  The readiness test is a
// heuristic (the cursor may move before the atomic): the claimed task may
// still have to wait, briefly.
__device__ __forceinline__ void claim_d(const WinArgs& A, int chunk, int& got, int& it0, int& nit) {
  const int lane = threadIdx.x;
  got = -1;
  it0 = 0;
  nit = 0;
  for (int base = 0; base < A.nact && got < 0; base += 32) {
    const int q = base + lane;
    int l = -1;
    bool ready = false;
    if (q < A.nact) {
      l = A.act[q];
      const unsigned long long w = *(volatile unsigned long long*)&A.ctl[l].word;
      const unsigned cur = w_cursor(w);
      ready = cur < w_ntasks(w);
      const DevCtl* gc = A.ctl + l;
      if (ready && *(volatile const int*)&gc->a_mode == M_SWEEP) {
        const SubGeo& g = A.geo[l];
        const int S = *(volatile const int*)&gc->a_s;
        const unsigned long long sb = *(volatile const unsigned long long*)&gc->a_sbase;
        const int ipr = __ldg(&g.ipr), R = __ldg(&g.nrows);
        const int ni = __ldg(&g.nitems);
        const int lev = (int)(cur / (unsigned)ni);
        const int row = (int)(cur - (unsigned)lev * (unsigned)ni) / ipr;
        (void)S;
        (void)R;
        if (lev >= 1) ready = sweep_levels_done(A, g, row, sb) >= lev;
      }
    }
    unsigned mask = __ballot_sync(0xffffffffu, ready);
    while (mask != 0u && got < 0) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1u;
      int it = -1, n = 0;
      if (lane == src) {
        const unsigned long long w2 = atomicAdd(&A.ctl[l].word, (unsigned long long)chunk);
        const unsigned u = w_cursor(w2);
        const unsigned ni = w_ntasks(w2);
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

// Fill the ring (one warp; called by whichever warp completed an item, so the
// issuing latency -- claims, readiness polls, fences -- lands on a warp that
// has a whole item of slack).  Issues in order while the next slot is free
// and the front task is ready.  It may WAIT (for work, for readiness) only
// when every issued item of this CTA has been completed and published
// (nfold == issued): a task can then never depend on work this CTA still
// holds, and the waiting cannot deadlock (tasks are claimed in cursor order
// and a CTA's queue holds one subdomain's chunk).  Otherwise it returns and
// the warp completing the next pending item tries again.
__device__ void fill_ring_d(const WinArgs& A, QueueD& q, SlotD* slot, BatchD* bat, Stage2* stage,
                            unsigned long long* full, unsigned long long* empty) {
  const int lane = threadIdx.x;
  {
    // Lock-free early out: the next slot is still being read by some warp.
    // That warp calls fill_ring_d after it arrives on the slot's empty
    // barrier, so nothing is lost by returning.  (q.issued can only grow
    // while we look; a slot issued meanwhile reads as free: we then take the
    // lock and look again.)
    int go = 1;
    if (lane == 0) {
      const int n = *(volatile int*)&q.issued;
      const unsigned u = (unsigned)(n / NBD);
      if (u >= 1 && !mbar_test(&empty[n % NBD], (u - 1) & 1u)) go = 0;
    }
    if (!__shfl_sync(0xffffffffu, go, 0)) return;
  }
  if (lane == 0) {
    while (atomicCAS(&q.lock, 0, 1) != 0) __nanosleep(32);
    __threadfence_block();   // acquire: the queue state left by the previous holder
  }
  __syncwarp();
  unsigned backoff = 64;
  while (true) {
    const int n = __shfl_sync(0xffffffffu, lane == 0 ? q.issued : 0, 0);
    const int b = n % NBD;
    const unsigned u = (unsigned)(n / NBD);
    int idle = 0;   // nothing of this CTA pending: waiting is allowed
    if (lane == 0) idle = *(volatile int*)&q.nfold == n;
    idle = __shfl_sync(0xffffffffu, idle, 0);
    // ---- the slot: its previous item consumed by every warp
    if (u >= 1) {
      int ok = 0;
      if (lane == 0) ok = mbar_test(&empty[b], (u - 1) & 1u) ? 1 : 0;
      if (!__shfl_sync(0xffffffffu, ok, 0)) break;   // that item's completion retries
    }
    // ---- a claimed task
    int have = __shfl_sync(0xffffffffu, (q.sub >= 0 && q.next < q.end) ? 1 : 0, 0);
    if (!have) {
      const unsigned nd = *(volatile unsigned*)A.n_done;
      const int chunk = (A.nact - (int)nd) >= A.tail_n ? A.chunk_bulk : A.chunk_tail;
      int got, it0, nit;
      claim_d(A, chunk, got, it0, nit);
      if (got < 0) {
        if (!idle) break;
        int ex = 0;
        if (lane == 0) ex = *(volatile unsigned*)A.n_done >= (unsigned)A.nact;
        ex = __shfl_sync(0xffffffffu, ex, 0);
        if (ex) {   // every subdomain finished its window: the exit marker
          if (lane == 0) {
            slot[b].t.mode = M_EXIT;
            mbar_arrive(&full[b]);   // release: the marker
            ++q.issued;
          }
          break;
        }
        if (lane == 0) __nanosleep(backoff);
        backoff = backoff < 1024 ? 2 * backoff : 1024;
        __syncwarp();
        continue;
      }
      if (lane == 0) {
        __threadfence();   // acquire: the action and the data of the previous action
        const DevCtl* gc = A.ctl + got;
        q.base = load_act(A, got);
        q.mode = q.base.mode;
        q.ntasks = __ldcg(&gc->a_ntasks);
        q.h = __ldcg(&gc->a_h);
        q.sbase = (unsigned long long)__ldcg(reinterpret_cast<const long long*>(&gc->a_sbase));
        const SubGeo& g = A.geo[got];
        q.nitems = g.nitems;
        q.ipr = g.ipr;
        q.nrows = g.nrows;
        q.sub = got;
        q.next = it0;
        q.end = it0 + nit;
        q.fence = 1;
      }
      __syncwarp();
    }
    // ---- the front task: readiness, then issue (lane 0)
    int state = 0;   // 1 issued, 0 not ready
    if (lane == 0) {
      const int tau = q.next;
      int lev = 0, item = tau;
      if (q.mode == M_SWEEP) {
        lev = tau / q.nitems;
        item = tau - lev * q.nitems;
      }
      const int row = item / q.ipr;
      bool ready = true;
      if (q.mode == M_SWEEP && lev >= 1) {
        const bool known = q.kr_sub == q.sub && q.kr_row == row && q.kr_base == q.sbase &&
                           lev <= q.kr_lev;
        if (!known) {
          q.fence = 1;   // new counter values observed: acquire before the TMA reads
          const long long L = sweep_levels_done(A, A.geo[q.sub], row, q.sbase);
          q.kr_sub = q.sub;
          q.kr_row = row;
          q.kr_base = q.sbase;
          q.kr_lev = (int)(L < (1 << 30) ? L : (1 << 30));
          ready = lev <= q.kr_lev;
        }
      }
      if (ready) {
        Act t = q.base;
        if (q.mode == M_SWEEP) {
          const int j = lev + 2;
          const int s = t.s;
          if (j <= s) {
            const int base = A.coef_off[s];
            t.mode = j == 2 ? M_STAGE2 : (j == 3 ? M_STAGE3 : M_STAGEN);
            t.j = j;
            t.mu = A.coef[4 * (base + j) + 0];
            t.nu = A.coef[4 * (base + j) + 1];
            t.hmut = q.h * A.coef[4 * (base + j) + 2];
            t.hgt = q.h * A.coef[4 * (base + j) + 3];
          } else {
            t.mode = M_FINAL;
          }
        }
        if (q.bleft == 0) {   // open a batch: the rest of this item row / chunk
          const int nb = q.nbatch % NBB;
          while (bat[nb].busy) __nanosleep(32);   // its flusher needs nothing from us
          __threadfence_block();
          BatchD& bt = bat[nb];
          int size = q.end - tau;
          if (q.mode == M_SWEEP) size = min(size, (row + 1) * q.ipr - item);
          bt.sub = q.sub;
          bt.row = row;
          bt.sweep = q.mode == M_SWEEP ? 1 : 0;
          bt.ntasks = q.ntasks;
          bt.size = size;
          bt.final_ = t.mode == M_FINAL ? 1 : 0;
          bt.done = 0u;
          bt.flags = 0u;
          bt.emax = 0ull;
          bt.busy = 1;
          q.bleft = size;
          q.bcur = nb;
          ++q.nbatch;
        }
        --q.bleft;
        SlotD& sd = slot[b];
        sd.t = t;
        sd.item = item;
        sd.batch = q.bcur;
        if (q.fence) {   // once per claim / fresh readiness observation
          __threadfence();   // acquire side of the readiness counters
          if (A.proxy_fence) asm volatile("fence.proxy.async.global;\n" ::: "memory");   // generic writes -> TMA reads
          q.fence = 0;
        }
        const SubGeo& g = A.geo[q.sub];
        const int ix = item % g.items_x, iy = item / g.items_x;
        issue_any2(A, t, ix * TX, iy * IR2, stage[b], &full[b]);
        ++q.issued;
        ++q.next;
        state = 1;
      }
    }
    state = __shfl_sync(0xffffffffu, state, 0);
    if (state == 1) continue;
    if (!idle) break;
    if (lane == 0) __nanosleep(backoff);
    backoff = backoff < 1024 ? 2 * backoff : 1024;
    __syncwarp();
  }
  __syncwarp();
  if (lane == 0) {
    __threadfence_block();   // release: the queue state
    atomicExch(&q.lock, 0);
  }
}

// Fixed-order sum of the per-item partials of an action by one warp, in
// exactly block_sum's order over NT threads (k_windowP): thread t sums items
// t, t+NT, ..., each warp reduces its 32 values by the shuffle tree, the
// warp totals are added in warp order.
__device__ double warp_items_sum(const double* part, int n) {
  double tot = 0.0;
#pragma unroll 1
  for (int w = 0; w < NWD; ++w) {
    double v = 0.0;
    for (int i = w * 32 + (int)threadIdx.x; i < n; i += NT) v += __ldcg(part + i);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    tot = w == 0 ? v : tot + v;
  }
  return __shfl_sync(0xffffffffu, tot, 0);
}

template <bool P2, int MODE, int YM>
__device__ __forceinline__ void item_d(const WinArgs& A, const SubGeo& g, const Act& t, int item,
                                       const Stage2& st, Acc& acc, double& ps) {
  constexpr bool SUMS = MODE == M_POWER || MODE == M_POWER_SEED || MODE == M_NORM;
  const int n0 = g.n[0], n1 = g.n[1], items_x = g.items_x;
  const long long pitch = g.pitch;
  const int ix = item % items_x, iy = item / items_x;
  const int c0 = ix * TX, r0 = iy * IR2;
  const long long kb = g.off + (long long)r0 * pitch + c0 + threadIdx.x;
  if constexpr (SUMS) {
    compute2<P2, MODE, YM>(A, g, t, c0, r0, st, acc, &ps);
  } else if (r0 >= 1 && r0 + IR2 <= n0 - 1 && c0 >= 1 && c0 + TX <= n1 - 1) {
    compute2_int<P2, MODE, YM, false>(A, g, t, kb, pitch, r0, c0, n0, n1, st, acc);
  } else {
    compute2_int<P2, MODE, YM, true>(A, g, t, kb, pitch, r0, c0, n0, n1, st, acc);
  }
}

template <bool P2>
__device__ __forceinline__ void dispatch_item_d(const WinArgs& A, const SubGeo& g, const Act& t,
                                                int item, const Stage2& st, Acc& acc, double& ps) {
  switch (t.mode) {
    case M_F0: item_d<P2, M_F0, YM_PLAIN>(A, g, t, item, st, acc, ps); break;
    case M_EULER: item_d<P2, M_EULER, YM_PLAIN>(A, g, t, item, st, acc, ps); break;
    case M_STAGE2: item_d<P2, M_STAGE2, YM_SCALED>(A, g, t, item, st, acc, ps); break;
    case M_STAGE3: item_d<P2, M_STAGE3, YM_ADD>(A, g, t, item, st, acc, ps); break;
    case M_STAGEN: item_d<P2, M_STAGEN, YM_ADD>(A, g, t, item, st, acc, ps); break;
    case M_FINAL: item_d<P2, M_FINAL, YM_ADD>(A, g, t, item, st, acc, ps); break;
    case M_POWER: item_d<P2, M_POWER, YM_SCALED>(A, g, t, item, st, acc, ps); break;
    case M_POWER_SEED: item_d<P2, M_POWER_SEED, YM_SEED>(A, g, t, item, st, acc, ps); break;
    case M_NORM: item_d<P2, M_NORM, YM_PLAIN>(A, g, t, item, st, acc, ps); break;
    default: break;
  }
}

// Batch completion (one warp): publish its items with one fence and one atomic
// per counter; the warp completing an action runs its controller (decide).
template <bool P2>
__device__ __noinline__ void publish_batch_d(const WinArgs& A, BatchD* s_bat, int bi, const Act& t,
                                             int l, const SubGeo& g, DevCtl& ctlw) {
    const int lane = threadIdx.x;
    int done_act = 0;
    if (lane == 0) {
      BatchD& bt = s_bat[bi];
      const int size = bt.size, row = bt.row, sweep = bt.sweep, ntasks = bt.ntasks;
      const unsigned gb = bt.flags;
      const unsigned long long emax = bt.emax;
      const bool final_ = bt.final_ != 0;
      __threadfence_block();
      bt.busy = 0;   // the record is free again
      DevCtl* gc = A.ctl + l;
      if (gb) atomicOr(&gc->acc_flags, gb);
      if (final_) atomicMax(&gc->acc_emax, emax);
      __threadfence();   // release: the batch's outputs before its counters
      if (sweep) atomicAdd(A.rowprog + g.rowoff + row, (unsigned long long)size);
      const unsigned d = atomicAdd(&gc->done, (unsigned)size);
      done_act = d + (unsigned)size == (unsigned)ntasks;
    }
    done_act = __shfl_sync(0xffffffffu, done_act, 0);
    if (done_act) {
      __threadfence();   // acquire: every task's partials / accumulators
      double sum = 0.0;
      if (t.mode == M_POWER || t.mode == M_POWER_SEED || t.mode == M_NORM)
        sum = warp_items_sum(A.part + A.poff[l], g.nitems);
      decide(A, l, g, sum, ctlw);
    }
}

template <bool P2>
__global__ void __launch_bounds__(NT, DDPMA_MINB2) k_windowD(const __grid_constant__ WinArgs A) {
  extern __shared__ __align__(128) unsigned char dsm[];
  Stage2* stage = reinterpret_cast<Stage2*>(
      dsm + ((128 - ((unsigned)__cvta_generic_to_shared(dsm) & 127u)) & 127u));
  __shared__ __align__(8) unsigned long long s_full[NBD], s_empty[NBD];
  __shared__ SlotD s_slot[NBD];
  __shared__ BatchD s_bat[NBB];
  __shared__ QueueD s_q;
  __shared__ DevCtl s_ctlw[NWD];      // per-warp controller scratch (decide)
  const int lane = threadIdx.x, warp = threadIdx.y;
  if (lane == 0 && warp == 0) {
    for (int b = 0; b < NBD; ++b) {
      mbar_init(&s_full[b]);
      mbar_init_n(&s_empty[b], NWD);
      s_slot[b].cnt = 0;
    }
    for (int b = 0; b < NBB; ++b) s_bat[b].busy = 0;
    s_q.sub = -1;
    s_q.next = s_q.end = 0;
    s_q.issued = 0;
    s_q.bleft = 0;
    s_q.nbatch = 0;
    s_q.kr_sub = -1;
    s_q.fence = 1;
    s_q.lock = 0;
    s_q.nfold = 0;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int i = warp * TX + lane; i < 97 * 3; i += NT) (&s_logtab[0][0])[i] = (&kLogTabD[0][0])[i];
  __syncthreads();

  if (warp == 0) fill_ring_d(A, s_q, s_slot, s_bat, stage, s_full, s_empty);
  int k = 0;   // items consumed by this warp
  while (true) {
    const int b = k % NBD;
    mbar_wait(&s_full[b], (unsigned)(k / NBD) & 1u);
    SlotD& sd = s_slot[b];
    const Act t = sd.t;
    if (t.mode == M_EXIT) break;
    const int item = sd.item;
    const int l = t.sub;
    const SubGeo& g = A.geo[l];
    Acc acc{0u, 0u, 0.0, 0.0};
    double ps = 0.0;
    dispatch_item_d<P2>(A, g, t, item, stage[b], acc, ps);
    // per-warp fold of the item's flags / error ratio / partial sum
    const unsigned fl = __any_sync(0xffffffffu, acc.flag != 0u) ? 1u : 0u;
    const unsigned nf = __any_sync(0xffffffffu, acc.nonfin != 0u) ? 4u : 0u;
    unsigned long long em = (unsigned long long)__double_as_longlong(acc.ratio);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_down_sync(0xffffffffu, em, off);
      em = o > em ? o : em;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ps += __shfl_down_sync(0xffffffffu, ps, off);
    int last = 0;
    if (lane == 0) {
      sd.wflag[warp] = fl | nf;
      sd.wemax[warp] = em;
      sd.wpsum[warp] = ps;
    }
    __syncwarp();   // every lane's global stores of the item precede lane 0's release
    if (lane == 0) last = atom_add_acqrel_cta(&sd.cnt, 1u) == (unsigned)(NWD - 1);
    last = __shfl_sync(0xffffffffu, last, 0);
    // the warp completing the item folds it into its batch, then frees the slot
    int flush = 0, bi = 0;
    if (last && lane == 0) {
      unsigned bits = 0;
      unsigned long long emax = 0ull;
      double psum = 0.0;
      for (int w = 0; w < NWD; ++w) {
        bits |= sd.wflag[w];
        emax = sd.wemax[w] > emax ? sd.wemax[w] : emax;
        psum = w == 0 ? sd.wpsum[0] : psum + sd.wpsum[w];   // block_sum's order
      }
      bi = sd.batch;
      sd.cnt = 0;
      BatchD& bt = s_bat[bi];
      const bool final_ = t.mode == M_FINAL;
      unsigned gb = 0;
      if (bits & 1u) gb |= final_ ? 2u : 1u;
      if (bits & 4u) gb |= 4u;
      if (gb) atomicOr(&bt.flags, gb);
      if (final_) atomicMax(&bt.emax, emax);
      if (t.mode == M_POWER || t.mode == M_POWER_SEED || t.mode == M_NORM)
        __stcg(A.part + A.poff[l] + item, psum);
      flush = atom_add_acqrel_cta(&bt.done, 1u) + 1u == (unsigned)bt.size;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&s_empty[b]);   // this warp is done with stage b
    ++k;
    flush = __shfl_sync(0xffffffffu, flush, 0);
    if (flush) publish_batch_d<P2>(A, s_bat, bi, t, l, g, s_ctlw[warp]);
    // the item is completed and published (by its last warp: one count per
    // item, fill_ring_d compares it with the items issued); every warp then
    // tries to refill the ring
    if (last && lane == 0) atomicAdd(&s_q.nfold, 1);
    __syncwarp();
    fill_ring_d(A, s_q, s_slot, s_bat, stage, s_full, s_empty);
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
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(c.t_begin));
  d_publish(A, c, gc, A.geo[l].nitems);
}

}  // namespace


// 2D windows run the stage-by-stage kernel k_windowP<2> or the dataflow kernel
// k_windowD (bitwise identical results); DDPMA_KERNEL=P / D overrides the
// built-in default below.  3D windows run k_windowP<3>.
#ifndef DDPMA_DEFAULT_DATAFLOW
#define DDPMA_DEFAULT_DATAFLOW 0
#endif
bool window_dataflow(int dim) {
  static const int sel = [] {
    const char* e = getenv("DDPMA_KERNEL");
    if (e && e[0] == 'P') return 0;
    if (e && e[0] == 'D') return 1;
    return DDPMA_DEFAULT_DATAFLOW;
  }();
  return dim == 2 && sel != 0;
}

static int smem_bytes(int dim, bool dataflow) {
  if (dim == 2) return (dataflow ? NBD : RD2) * STAGE2_BYTES + 128;
  return 2 * (int)sizeof(Stage3) + 128;
}

int window_blocks(int dim, int pow2) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = smem_bytes(dim, window_dataflow(dim));
  const void* fn;
  if (dim == 2 && window_dataflow(2)) fn = pow2 ? (const void*)k_windowD<true> : (const void*)k_windowD<false>;
  else if (dim == 2) fn = pow2 ? (const void*)k_windowP<2, true> : (const void*)k_windowP<2, false>;
  else fn = pow2 ? (const void*)k_windowP<3, true> : (const void*)k_windowP<3, false>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, NT, smem);
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
  const void* fn;
  if (a.P.dim == 2 && a.sweep) fn = a.P.pow2 ? (const void*)k_windowD<true> : (const void*)k_windowD<false>;
  else if (a.P.dim == 2) fn = a.P.pow2 ? (const void*)k_windowP<2, true> : (const void*)k_windowP<2, false>;
  else fn = a.P.pow2 ? (const void*)k_windowP<3, true> : (const void*)k_windowP<3, false>;
  cudaLaunchCooperativeKernel(fn, dim3(nb), blk, args, smem_bytes(a.P.dim, a.sweep != 0),
                              (cudaStream_t)stream);
}

}  // namespace ddpma
