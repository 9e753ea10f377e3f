// Host runtime of libddpma.so: plan (device arena), the batched RKC2/Euler
// controller, the window loop of solve(), and the C ABI (include/ddpma.h).
//
// The controller is a statement-for-statement restatement of
// Rkc2Integrator.advance / _estimate_sigma / _stages_for
// (ddmesh/integrate.py:109-250) as a per-subdomain state machine.  All local
// subdomains advance together in "rounds": each round launches, per phase,
// ONE batched kernel sequence over every subdomain in that phase (their own
// h, s, coefficients), then reads back one small result record per
// subdomain.  Host scalar arithmetic is compiled with -ffp-contract=off so it
// rounds exactly like the reference's Python floats.

#include <cuda.h>   // CUtensorMap / cuTensorMapEncodeTiled types (entry point fetched at run time)
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ddpma.h"
#include "ddpma_internal.h"

using namespace ddpma;

namespace {

constexpr double kSqrtEps = 1.4901161193847656e-08;   // np.sqrt(np.finfo(float).eps)
constexpr double kStab = 0.653;                       // integrate.py:36
constexpr double kMinStep = 1e-14;                    // integrate.py:37
constexpr int kSigmaRefresh = 25;                     // integrate.py:38
// DDPMA_TRACE=1 prints every controller decision (debugging parity).
const bool g_trace = getenv("DDPMA_TRACE") != nullptr;

enum Phase { PH_IDLE, PH_F0, PH_SIG_NORM, PH_SIG_ITER, PH_STEP, PH_EULER, PH_DONE, PH_FAILED };
enum SigRet { RET_START, RET_ACCEPT, RET_REJECT };

// Per-subdomain integrator state (Rkc2Integrator fields + advance() locals).
struct Ctl {
  // persistent caches (integrate.py:118-123)
  bool has_sigma = false;
  double sigma = 0.0;
  int since = 0;
  int interval = kSigmaRefresh;
  bool has_h = false;
  double h_last = 0.0;
  // window locals
  Phase phase = PH_IDLE;
  double t = 0.0, h = 0.0;
  bool start_flag = false, state_flag = false;
  int rej_row = 0, flag_rej = 0;
  int s = 2;
  int yi = 0, fi = 0;
  // sigma estimation
  SigRet ret = RET_START;
  double delta = 0.0, vnorm = 0.0, sig = 0.0;
  int sig_k = 0, vin = -1, vout = 0;
  // euler
  int euler_left = 0;
  // pipeline
  bool waiting = false;   // an issued action needs its result before the next one
  int j_next = 0;         // next stage of the current step (0 = step not started)
  bool step_flag = false; // OR of the stage positivity flags of the current step
};

struct Failure {
  bool set = false;
  int gid = -1;
  ddpma_status status = DDPMA_OK;
  std::string msg;
  double t = 0.0, h = 0.0;
  int64_t nnodes = -1;
  int local = -1;
  int s = 0, yi = 0, fi = 0;
  double h04 = 0.0;
};

struct ProfRec {
  cudaEvent_t a, b;
  int klass;
  double bytes;
  long long nodes;
};

inline long long round_up(long long x, long long m) { return (x + m - 1) / m * m; }

inline double okey_dec(unsigned long long k) {
  unsigned long long u = (k & 0x8000000000000000ull) ? (k & ~0x8000000000000000ull) : ~k;
  double d;
  memcpy(&d, &u, 8);
  return d;
}

inline double bits_dec(unsigned long long u) {
  double d;
  memcpy(&d, &u, 8);
  return d;
}

bool is_pow2(double h) {
  int e;
  const double m = frexp(h, &e);
  return m == 0.5;
}

}  // namespace

struct ddpma_plan {
  int device = 0;
  cudaStream_t st = nullptr;
  ddpma_grid grid{};
  ddpma_solver_cfg cfg{};
  int dim = 2;
  std::vector<ddpma_subdomain> subs;
  int nsub = 0;
  std::vector<int> local;       // global ids, ascending
  std::vector<int> local_of;    // gid -> local index or -1
  // alternating transmission: wavefront levels of the id-ordered sweep (local
  // indices, ascending inside a level); only for plans owning every subdomain
  std::vector<std::vector<int>> alt_levels;
  std::vector<SubGeo> geo;
  SubGeo* d_geo = nullptr;
  Prob P{};
  MonitorD mon{};
  MonitorD* d_mon = nullptr;
  bool u_backed = false;   // arc-length monitor carrying u (pull-back density)
  std::vector<void*> lat_allocs;   // sampled-field lattice copies
  long long arena = 0;
  double* d_arena = nullptr;
  Fields F{};
  double* d_scratch = nullptr;  // dense box scratch (operator API, error nodes)
  long long scratch_elems = 0;
  std::vector<Ctl> ctl;
  SubRes* d_res = nullptr;
  SubRes* h_res = nullptr;
  double* d_part = nullptr;
  double* d_part2 = nullptr;
  int total_tiles = 0;
  // staging of launch descriptors
  char* h_stage = nullptr;
  char* d_stage = nullptr;
  size_t stage_cap = 0, stage_used = 0;
  // window state
  bool state_set = false;
  bool density_ready = false;
  bool have_old = false;
  bool raw_valid = false;   // F.raw holds the previous window's density (monitor_relax)
  double z = 0.0, rho_max = 0.0;
  std::vector<double> zpart, rawmax, resid, jmin, jmax;
  // errors
  std::string err;
  Failure fail;
  // counters
  long long node_updates = 0, rhs_evals = 0, launches = 0;
  double algo_bytes = 0.0;
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<ProfRec> prof_pending;
  double prof_ms[NCLASS] = {0}, prof_bytes[NCLASS] = {0};
  long long prof_launches[NCLASS] = {0}, prof_nodes[NCLASS] = {0};
  // sharded trace exchange
  std::vector<int> rank_of;
  int my_rank = 0, nranks = 1;
  bool exch_ready = false;
  struct Seg { int recv_gid, axis, side, donor_gid; long long off; int ext0, ext1; };
  std::vector<Seg> send_segs, recv_segs;   // send_segs: offsets into the send buffer
  // asynchronous launch pipeline (advance_set): per-slot entries/results
  static constexpr int R = 4;
  Entry* h_ent[R] = {};
  Entry* d_ent[R] = {};
  SubRes* d_ring = nullptr;
  SubRes* h_ring = nullptr;
  double* d_partring = nullptr;
  cudaEvent_t ring_ev[R] = {};
  long long kissue = 0;
  std::vector<RkcCoeffs> coeff_cache;       // index s (lru_cache of _rkc_coeffs)
  // device-resident controller (persist.cu)
  DevCtl* d_ctl = nullptr;
  DevCtl* h_ctl = nullptr;
  std::vector<DevCtl> ctl_prev;            // counters at the previous read-back
  double* d_coef = nullptr;
  int* d_coef_off = nullptr;
  double* d_part_items = nullptr;
  long long* d_poff = nullptr;
  int* d_act = nullptr;       // [0, nl): priority order; [nl, 2nl): per-position chunk sizes
  int* h_act = nullptr;
  unsigned int* d_ndone = nullptr;
  TraceRec* d_trace = nullptr;
  unsigned int* d_trace_n = nullptr;
  int trace_cap = 0;
  int win_blocks = 0;
  int chunk_bulk = 8, chunk_tail = 2, tail_n = 16;   // window scheduler knobs (parsed once)
  bool chunk_adapt = true;   // per-subdomain bulk chunk sizes from the last window's tallies
  unsigned long long* d_probe = nullptr;             // DDPMA_PROBE timestamps (debug)
  unsigned long long* d_rowprog = nullptr;           // k_windowD per-row task counters
  long long total_rows = 0;
  bool host_ctl = false;
  bool integ_ready = false;                // ddpma_integrate_window: integrators initialised
  void* d_tmap = nullptr;                  // 2D TMA tensor maps (persist.cu issue2_tma)
  std::vector<long long> last_evals;       // per local subdomain, previous window
  std::vector<long long> sub_evals;        // per local subdomain, RHS evaluations since set_state
  long long mode_nodes[9] = {0};
};

namespace {

// ------------------------------------------------------------ utilities --

ddpma_status cuda_fail(ddpma_plan* p, cudaError_t e, const char* where) {
  p->err = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
  return DDPMA_ERR_CUDA;
}

#define CK(p, call)                                     \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(p, e_, #call); \
  } while (0)

ddpma_status check_launch(ddpma_plan* p, const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(p, e, where);
  return DDPMA_OK;
}

// Bump allocator over pinned host + device staging; H2D per segment.
ddpma_status stage_reset(ddpma_plan* p) {
  p->stage_used = 0;
  return DDPMA_OK;
}

// Make sure `bytes` more can be staged without an intervening reset (a group
// of launches whose descriptors must all stay live).
ddpma_status stage_reserve(ddpma_plan* p, size_t bytes) {
  if (p->stage_used + bytes <= p->stage_cap) return DDPMA_OK;
  CK(p, cudaStreamSynchronize(p->st));
  p->stage_used = 0;
  if (bytes > p->stage_cap) {
    size_t cap = std::max(bytes, p->stage_cap * 2);
    if (p->h_stage) cudaFreeHost(p->h_stage);
    if (p->d_stage) cudaFree(p->d_stage);
    p->h_stage = nullptr;
    p->d_stage = nullptr;
    CK(p, cudaMallocHost((void**)&p->h_stage, cap));
    CK(p, cudaMalloc((void**)&p->d_stage, cap));
    p->stage_cap = cap;
  }
  return DDPMA_OK;
}

ddpma_status stage_put(ddpma_plan* p, const void* data, size_t bytes, void** dev_out) {
  size_t need = round_up((long long)bytes, 256);
  if (p->stage_used + need > p->stage_cap) {
    CK(p, cudaStreamSynchronize(p->st));
    p->stage_used = 0;
    if (need > p->stage_cap) {
      size_t cap = std::max(need, p->stage_cap * 2);
      if (p->h_stage) cudaFreeHost(p->h_stage);
      if (p->d_stage) cudaFree(p->d_stage);
      p->h_stage = nullptr;
      p->d_stage = nullptr;
      CK(p, cudaMallocHost((void**)&p->h_stage, cap));
      CK(p, cudaMalloc((void**)&p->d_stage, cap));
      p->stage_cap = cap;
    }
  }
  memcpy(p->h_stage + p->stage_used, data, bytes);
  CK(p, cudaMemcpyAsync(p->d_stage + p->stage_used, p->h_stage + p->stage_used, bytes,
                        cudaMemcpyHostToDevice, p->st));
  *dev_out = p->d_stage + p->stage_used;
  p->stage_used += need;
  return DDPMA_OK;
}

// Fill tile prefix of entries (in order); returns total CTAs.
int prefix_tiles(ddpma_plan* p, std::vector<Entry>& ents) {
  int acc = 0;
  for (auto& e : ents) {
    e.tile_begin = acc;
    e.ntiles = p->geo[e.sub].ntiles;
    acc += e.ntiles;
  }
  return acc;
}

KArgs base_args(ddpma_plan* p) {
  KArgs a{};
  a.P = p->P;
  a.geo = p->d_geo;
  a.F = p->F;
  a.res = p->d_res;
  a.part = p->d_part;
  a.part2 = p->d_part2;
  a.mon = p->d_mon;
  return a;
}

// ddpma_monitor -> device descriptor.
void fill_monitor(const ddpma_monitor* monitor, int dim, MonitorD& M) {
  memset(&M, 0, sizeof M);
  M.kind = monitor->kind;
  M.dim = dim;
  for (int k = 0; k < 3; ++k) {
    M.lo[k] = monitor->domain[k][0];
    M.hi[k] = monitor->domain[k][1];
    M.center[k] = monitor->center[k];
  }
  M.constant = monitor->constant;
  M.amp = monitor->amp;
  M.nsharp = -monitor->sharp;
  M.r2 = monitor->r2;
  M.eps = monitor->eps;
  M.nb = monitor->kind == DDPMA_MON_MIXTURE ? monitor->nbumps : 0;
  for (int b = 0; b < M.nb; ++b) {
    for (int k = 0; k < dim; ++k) M.c[b * 3 + k] = monitor->c[b * dim + k];
    M.den[b] = 2.0 * monitor->s[b] * monitor->s[b];
    M.a[b] = monitor->a[b];
  }
}

// Device copies of a sampled field's lattice (axes, values, gradients).
cudaError_t upload_lattice(const ddpma_monitor* m, int dim, MonitorD& M,
                           std::vector<void*>& owned) {
  if (m->kind != DDPMA_MON_SAMPLED) return cudaSuccess;
  size_t nv = 1;
  for (int k = 0; k < dim; ++k) {
    M.sm[k] = m->lat[k];
    nv *= (size_t)m->lat[k];
  }
  auto up = [&](const double* src, size_t n, const double** dst) -> cudaError_t {
    double* d = nullptr;
    cudaError_t e = cudaMalloc((void**)&d, sizeof(double) * n);
    if (e != cudaSuccess) return e;
    owned.push_back(d);
    *dst = d;
    return cudaMemcpy(d, src, sizeof(double) * n, cudaMemcpyHostToDevice);
  };
  cudaError_t e;
  for (int k = 0; k < dim; ++k) {
    if ((e = up(m->axes[k], (size_t)m->lat[k], &M.sax[k])) != cudaSuccess) return e;
    if ((e = up(m->grads[k], nv, &M.sg[k])) != cudaSuccess) return e;
  }
  return up(m->values, nv, &M.sv);
}

bool sampled_ok(const ddpma_monitor* m, int dim) {
  if (m->kind != DDPMA_MON_SAMPLED) return true;
  if (!m->values) return false;
  for (int k = 0; k < dim; ++k)
    if (m->lat[k] < 2 || !m->axes[k] || !m->grads[k]) return false;
  return true;
}

// u-backed monitors (arc-length of a test function): mesh_density is the
// mesh pull-back of u (monitor.py:170-180); run its pre-pass and let the
// following raw-density pass read it.
void upull_prepass(ddpma_plan* p, KArgs& a, int nb) {
  if (p->u_backed) {
    launch_upre(a, nb, p->st);
    a.upull = 1;
  }
}

Entry make_entry(ddpma_plan* p, int l) {
  Entry e{};
  e.sub = l;
  e.yi = p->ctl[l].yi;
  e.fi = p->ctl[l].fi;
  e.vin = -1;
  e.s = 2;
  return e;
}

cudaEvent_t take_event(ddpma_plan* p) {
  if (p->ev_used == p->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    p->ev_pool.push_back(e);
  }
  return p->ev_pool[p->ev_used++];
}

// kernel class / algorithmic bytes per node (SURVEY §8(d) byte model)
void account(ddpma_plan* p, int klass, long long nodes, double bpn, bool rhs) {
  p->launches += 1;
  p->algo_bytes += bpn * (double)nodes;
  if (rhs) {
    p->node_updates += nodes;
  }
  p->prof_launches[klass] += 1;
  p->prof_bytes[klass] += bpn * (double)nodes;
  p->prof_nodes[klass] += nodes;
}

long long entries_nodes(ddpma_plan* p, const Entry* ents, int n) {
  long long s = 0;
  for (int i = 0; i < n; ++i) s += p->geo[ents[i].sub].nodes;
  return s;
}

ddpma_status sync(ddpma_plan* p);

// SURVEY §8(d) algorithmic bytes per node-update of each action.
double mode_bytes(int mode) {
  switch (mode) {
    case M_F0: return 24.0;        // y, mr -> f0
    case M_STAGE2: return 32.0;    // y, f0, mr -> d2
    case M_STAGE3: return 40.0;    // y, d2, f0, mr -> d3
    case M_STAGEN: return 48.0;    // y, d_{j-1}, d_{j-2}, f0, mr -> d_j
    case M_FINAL: return 48.0;     // y, d_s, f0, mr -> f_new, y_new
    case M_POWER: return 40.0;     // y, v, f0, mr -> v'
    case M_POWER_SEED: return 32.0;
    case M_EULER: return 24.0;     // y, mr -> y_new
    case M_NORM: return 8.0;
    default: return 0.0;
  }
}

const RkcCoeffs& coeffs(ddpma_plan* p, int s) {
  if ((int)p->coeff_cache.size() <= s) p->coeff_cache.resize(s + 1);
  RkcCoeffs& c = p->coeff_cache[s];
  if (c.mu.empty()) rkc_coeffs(s, c);
  return c;
}

// Enqueue one mixed eval launch over `ents` into result slot `slot`:
// reset slot, copy entries, kernel, (finalize sums), D2H results, event.
ddpma_status issue(ddpma_plan* p, std::vector<Entry>& ents, int slot) {
  const int n = (int)p->local.size();
  const int nb = prefix_tiles(p, ents);
  memcpy(p->h_ent[slot], ents.data(), sizeof(Entry) * ents.size());
  SubRes* res = p->d_ring + (size_t)slot * n;
  double* part = p->d_partring + (size_t)slot * std::max(p->total_tiles, 1);
  CK(p, cudaMemsetAsync(res, 0, sizeof(SubRes) * n, p->st));
  CK(p, cudaMemcpyAsync(p->d_ent[slot], p->h_ent[slot], sizeof(Entry) * ents.size(),
                        cudaMemcpyHostToDevice, p->st));
  KArgs a = base_args(p);
  a.ent = p->d_ent[slot];
  a.nent = (int)ents.size();
  a.res = res;
  a.part = part;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (p->prof) {
    e0 = take_event(p);
    e1 = take_event(p);
    cudaEventRecord(e0, p->st);
  }
  launch_eval(a, nb, p->st);
  double bytes = 0.0;
  long long nodes = 0;
  bool sums = false;
  for (auto& e : ents) {
    const long long nn = p->geo[e.sub].nodes;
    bytes += mode_bytes(e.mode) * (double)nn;
    p->mode_nodes[e.mode] += nn;
    if (e.mode != M_NORM) {
      nodes += nn;
      p->rhs_evals += 1;
      p->sub_evals[e.sub] += 1;
    }
    sums |= e.mode == M_POWER || e.mode == M_POWER_SEED || e.mode == M_NORM;
  }
  if (p->prof) {
    cudaEventRecord(e1, p->st);
    p->prof_pending.push_back({e0, e1, 0, bytes, nodes});
  }
  p->launches += 1;
  p->algo_bytes += bytes;
  p->node_updates += nodes;
  p->prof_launches[0] += 1;
  p->prof_bytes[0] += bytes;
  p->prof_nodes[0] += nodes;
  if (sums) launch_finalize(p->d_ent[slot], (int)ents.size(), part, res, 0, p->st);
  CK(p, cudaMemcpyAsync(p->h_ring + (size_t)slot * n, res, sizeof(SubRes) * n,
                        cudaMemcpyDeviceToHost, p->st));
  CK(p, cudaEventRecord(p->ring_ev[slot], p->st));
  return check_launch(p, "eval kernel");
}

// Synchronous single launch (operator-level exports): results in h_ring slot 0.
ddpma_status issue_sync(ddpma_plan* p, std::vector<Entry>& ents) {
  ddpma_status s = issue(p, ents, 0);
  if (s != DDPMA_OK) return s;
  return sync(p);
}

void prof_collect(ddpma_plan* p) {
  for (auto& r : p->prof_pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) p->prof_ms[r.klass] += ms;
  }
  p->prof_pending.clear();
  p->ev_used = 0;
}

ddpma_status sync(ddpma_plan* p) {
  CK(p, cudaStreamSynchronize(p->st));
  if (p->prof) prof_collect(p);
  stage_reset(p);
  return DDPMA_OK;
}

void set_fail(ddpma_plan* p, int l, ddpma_status st, const std::string& msg) {
  Ctl& c = p->ctl[l];
  c.phase = PH_FAILED;
  const int gid = p->local[l];
  if (!p->fail.set || gid < p->fail.gid) {
    p->fail = Failure{};
    p->fail.set = true;
    p->fail.gid = gid;
    p->fail.status = st;
    p->fail.msg = msg;
    p->fail.t = c.t;
    p->fail.h = c.h;
    p->fail.local = l;
    p->fail.s = c.s;
    p->fail.yi = c.yi;
    p->fail.fi = c.fi;
    p->fail.h04 = 0.4 * c.h;
  }
}

// ------------------------------------------------------- state machine --

void loop_check(ddpma_plan* p, int l);

void prepare_step(ddpma_plan* p, int l) {
  Ctl& c = p->ctl[l];
  const double total = p->cfg.dtau;
  const int ms = p->cfg.max_stages;
  c.h = std::min(c.h, total - c.t);                         // integrate.py:198
  const double cap = kStab * (double)((long long)ms * ms);   // :199
  if (c.sigma > 0.0 && c.h * c.sigma > cap) c.h = cap / c.sigma;
  const double hs = c.h * c.sigma;                           // _stages_for :157-161
  long long s;
  if (hs <= 0.0) {
    s = 2;
  } else {
    const double v = std::ceil(std::sqrt(1.05 * hs / kStab));
    if (std::isnan(v)) {
      set_fail(p, l, DDPMA_ERR_VALUE, "cannot convert float NaN to integer");
      return;
    }
    if (std::isinf(v)) {
      set_fail(p, l, DDPMA_ERR_OVERFLOW, "cannot convert float infinity to integer");
      return;
    }
    s = v > 1e9 ? (long long)1e9 : (long long)v;
    s = std::max(2LL, s);
  }
  c.s = (int)std::min((long long)ms, s);
  c.phase = PH_STEP;
}

void start_sigma(ddpma_plan* p, int l, SigRet ret) {
  Ctl& c = p->ctl[l];
  c.ret = ret;
  c.phase = PH_SIG_NORM;
}

void after_start(ddpma_plan* p, int l) {       // integrate.py:187-196
  Ctl& c = p->ctl[l];
  const double total = p->cfg.dtau;
  double h;
  if (c.sigma <= 0.0) h = total;
  else h = std::min(total, std::max(10.0 * kMinStep * total, 0.25 / c.sigma));
  if (c.has_h) h = std::min(total, c.h_last);
  c.h = h;
  c.t = 0.0;
  c.state_flag = c.start_flag;
  c.rej_row = 0;
  c.flag_rej = 0;
  loop_check(p, l);
}

void finish_sigma(ddpma_plan* p, int l) {      // integrate.py:147-153
  Ctl& c = p->ctl[l];
  c.since = 0;
  if (c.has_sigma && c.sig <= 1.05 * c.sigma / 1.2) c.interval = std::min(500, 2 * c.interval);
  else c.interval = kSigmaRefresh;
  c.sigma = 1.2 * c.sig;
  c.has_sigma = true;
  if (g_trace) fprintf(stderr, "TRACE %d sigma %.17g\n", p->local[l], c.sigma);
  if (c.ret == RET_START) after_start(p, l);
  else loop_check(p, l);
}

void loop_check(ddpma_plan* p, int l) {        // integrate.py:197
  Ctl& c = p->ctl[l];
  const double total = p->cfg.dtau;
  if (c.t < total * (1.0 - 1e-13)) prepare_step(p, l);
  else c.phase = PH_DONE;
}

void begin_window_ctl(ddpma_plan* p, int l) {
  Ctl& c = p->ctl[l];
  if (p->cfg.scheme == DDPMA_SCHEME_EULER) {
    c.phase = PH_EULER;
    c.euler_left = p->cfg.substeps;
  } else {
    c.phase = PH_F0;
  }
}

// Decision after an action's result (integrate.py:180-250 restated).
void on_result(ddpma_plan* p, int l, Phase ph, const SubRes& r) {
  Ctl& c = p->ctl[l];
  const double total = p->cfg.dtau;
  c.waiting = false;
  switch (ph) {
    case PH_F0:
      c.start_flag = (r.flags & 1u) != 0;
      if (!c.has_sigma || c.since >= c.interval) start_sigma(p, l, RET_START);
      else after_start(p, l);
      break;
    case PH_SIG_NORM: {                         // integrate.py:132-133
      const double ny = std::sqrt(r.sum);
      c.delta = kSqrtEps * (1.0 + ny);
      c.sig = 0.0;
      c.sig_k = 0;
      c.vin = -1;
      c.vnorm = std::sqrt((double)p->geo[l].nodes);   // |checkerboard| = sqrt(N), exact
      if (c.vnorm == 0.0) finish_sigma(p, l);
      else c.phase = PH_SIG_ITER;
      break;
    }
    case PH_SIG_ITER: {                         // integrate.py:135-146
      const double nrm = std::sqrt(r.sum);
      const double ns = nrm / c.delta;
      c.vin = c.vout;
      c.sig_k += 1;
      if (c.sig > 0.0 && std::fabs(ns - c.sig) <= 0.01 * ns) {
        c.sig = ns;
        finish_sigma(p, l);
        break;
      }
      c.sig = ns;
      if (c.sig_k >= 20) {
        finish_sigma(p, l);
        break;
      }
      c.vnorm = nrm;
      if (c.vnorm == 0.0) finish_sigma(p, l);
      break;
    }
    case PH_STEP: {                             // integrate.py:203-249
      const bool nonfin = (r.flags & 4u) != 0;
      const bool flagged = c.step_flag || (r.flags & 3u) != 0;
      const bool end_flag = (r.flags & 2u) != 0;
      const double emax = bits_dec(r.emax);
      const bool flag_fail = flagged && !c.state_flag && c.flag_rej < 8;
      const bool bad = flag_fail || nonfin;
      c.j_next = 0;
      if (g_trace)
        fprintf(stderr, "TRACE %d step %.17g %d %.17g %d %d\n", p->local[l], c.h, c.s,
                nonfin ? NAN : emax, flagged ? 1 : 0, (!bad && emax <= 1.0) ? 1 : 0);
      if (!bad && emax <= 1.0) {
        c.t += c.h;
        c.yi ^= 1;
        c.fi ^= 1;
        c.state_flag = end_flag;
        c.since += 1;
        c.rej_row = 0;
        const bool need = c.since >= c.interval && c.t < total;
        const double grow = emax == 0.0 ? 5.0 : std::min(5.0, 0.8 * std::pow(emax, -1.0 / 3.0));
        c.h = c.h * std::max(0.1, grow);
        c.h_last = c.h;
        c.has_h = true;
        if (need) start_sigma(p, l, RET_ACCEPT);
        else loop_check(p, l);
      } else {
        if (flag_fail) {
          c.flag_rej += 1;
          c.h *= 0.5;
        } else if (nonfin) {
          c.h *= 0.5;
          c.rej_row += 1;
        } else {
          c.h *= std::max(0.1, 0.8 * std::pow(emax, -1.0 / 3.0));
          c.rej_row += 1;
        }
        const bool need = c.rej_row >= 2;
        if (need) c.rej_row = 0;
        if (c.h < kMinStep * total || c.flag_rej + c.rej_row > 60) {
          set_fail(p, l, DDPMA_ERR_STIFFNESS, "internal step underflow");
          if (p->fail.local == l) p->fail.nnodes = nonfin ? -1 : -2;   // -2: count lazily
          break;
        }
        if (need) start_sigma(p, l, RET_REJECT);
        else loop_check(p, l);
      }
      break;
    }
    default:
      break;
  }
}

// The next action of subdomain l as a launch entry; updates the host-side
// bookkeeping of actions that need no decision (stages, Euler substeps).
Entry next_action(ddpma_plan* p, int l) {
  Ctl& c = p->ctl[l];
  Entry e = make_entry(p, l);
  switch (c.phase) {
    case PH_F0:
      e.mode = M_F0;
      c.waiting = true;
      break;
    case PH_SIG_NORM:
      e.mode = M_NORM;
      c.waiting = true;
      break;
    case PH_SIG_ITER:
      e.mode = c.vin < 0 ? M_POWER_SEED : M_POWER;
      e.vin = c.vin;
      c.vout = c.vin < 0 ? 0 : 1 - c.vin;
      e.vout = c.vout;
      e.c = c.delta / c.vnorm;
      c.waiting = true;
      break;
    case PH_STEP: {
      const RkcCoeffs& rc = coeffs(p, c.s);
      if (c.j_next == 0) {
        c.j_next = 2;
        c.step_flag = false;
      }
      e.s = c.s;
      e.c = c.h * rc.mu1t;
      if (c.j_next <= c.s) {
        const int j = c.j_next++;
        e.mode = j == 2 ? M_STAGE2 : (j == 3 ? M_STAGE3 : M_STAGEN);
        e.j = j;
        e.mu = rc.mu[j];
        e.nu = rc.nu[j];
        e.hmut = c.h * rc.mut[j];
        e.hgt = c.h * rc.gt[j];
      } else {
        e.mode = M_FINAL;
        e.h04 = 0.4 * c.h;
        c.waiting = true;
      }
      break;
    }
    case PH_EULER:
      e.mode = M_EULER;
      e.c = p->cfg.dtau / (double)p->cfg.substeps;
      c.yi ^= 1;
      if (--c.euler_left == 0) c.phase = PH_DONE;
      break;
    default:
      e.mode = -1;
      break;
  }
  return e;
}

struct Inflight {
  int slot;
  std::vector<std::pair<int, int>> who;   // (local sub, mode)
  std::vector<Phase> phase;                // phase at issue
};

// Process one completed launch: accumulate stage flags, run decisions.
ddpma_status process(ddpma_plan* p, const Inflight& f) {
  CK(p, cudaEventSynchronize(p->ring_ev[f.slot]));
  const int n = (int)p->local.size();
  const SubRes* res = p->h_ring + (size_t)f.slot * n;
  for (size_t i = 0; i < f.who.size(); ++i) {
    const int l = f.who[i].first, mode = f.who[i].second;
    Ctl& c = p->ctl[l];
    if (c.phase == PH_FAILED) continue;
    const SubRes& r = res[l];
    if (mode == M_STAGE2 || mode == M_STAGE3 || mode == M_STAGEN) {
      c.step_flag = c.step_flag || (r.flags & 1u) != 0;
    } else if (mode == M_EULER) {
      // no decision (EulerIntegrator ignores the flag, integrate.py:72)
    } else {
      on_result(p, l, f.phase[i], r);
    }
  }
  return DDPMA_OK;
}

// One window of integration for the local subdomains `act`: an asynchronous
// pipeline.  Every launch carries one action for each subdomain that is not
// waiting on a host decision (stages of different steps, power iterations,
// f0 evaluations mix freely); the result of launch k is processed while
// launch k+1 runs, so a decision costs a subdomain one skipped launch.
ddpma_status advance_set_host(ddpma_plan* p, const std::vector<int>& act) {
  for (int l : act) {
    begin_window_ctl(p, l);
    p->ctl[l].waiting = false;
    p->ctl[l].j_next = 0;
  }
  std::vector<Inflight> q;   // FIFO (front = oldest)
  size_t head = 0;
  ddpma_status s;
  while (true) {
    std::vector<Entry> ents;
    Inflight f;
    for (int l : act) {
      Ctl& c = p->ctl[l];
      if (c.waiting) continue;
      if (c.phase != PH_F0 && c.phase != PH_SIG_NORM && c.phase != PH_SIG_ITER &&
          c.phase != PH_STEP && c.phase != PH_EULER)
        continue;
      const Phase ph = c.phase;
      Entry e = next_action(p, l);
      f.who.push_back({l, e.mode});
      f.phase.push_back(ph);
      ents.push_back(e);
    }
    if (!ents.empty()) {
      f.slot = (int)(p->kissue % ddpma_plan::R);
      if ((s = issue(p, ents, f.slot)) != DDPMA_OK) return s;
      p->kissue++;
      q.push_back(std::move(f));
    }
    const size_t inflight = q.size() - head;
    if (inflight == 0) break;
    if (ents.empty() || inflight >= 2) {
      if ((s = process(p, q[head])) != DDPMA_OK) return s;
      ++head;
    }
  }
  return sync(p);
}

// One window on the device-resident controller: window-begin kernel + one
// cooperative persistent kernel (persist.cu), then one read-back of the
// controller states.  This is the production path.
ddpma_status advance_set(ddpma_plan* p, const std::vector<int>& act) {
  if (p->host_ctl) return advance_set_host(p, act);
  const int nl = (int)p->local.size();
  // priority: most RHS evaluations in the previous window first (the
  // straggler's critical path is served before filler work)
  std::vector<int> order(act);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
    return p->last_evals[x] * p->geo[x].nodes > p->last_evals[y] * p->geo[y].nodes;
  });
  for (size_t q = 0; q < order.size(); ++q) p->h_act[q] = order[q];
  // Per-subdomain chunk size.  A subdomain's actions are a sequential chain: an
  // action claimed in chunks of c items takes ~(c + o) item-times (o ~ 2: claim,
  // first tile, completion, controller), so a subdomain with n actions cannot
  // finish before n (c + o).  The window as a whole needs ~T = (all items) /
  // (CTAs) item-times.  Subdomains whose chain at the bulk chunk size would
  // reach 0.6 T (from the previous window's action counts) get smaller chunks,
  // so the heaviest subdomains finish early instead of leaving a serial tail.
  {
    int* hq = p->h_act + nl;
    double items_tot = 0.0;
    for (int l : act) items_tot += (double)p->last_evals[l] * (double)p->geo[l].nitems;
    const double T = items_tot / (double)std::max(1, p->win_blocks);
    for (size_t q = 0; q < order.size(); ++q) {
      const long long n = p->last_evals[order[q]];
      int c = p->chunk_bulk;
      if (p->chunk_adapt && n > 0 && T > 0.0) {
        const double cmax = 0.6 * T / (double)n - 2.0;
        c = cmax >= (double)p->chunk_bulk ? p->chunk_bulk : (cmax < 2.0 ? 2 : (int)cmax);
      }
      hq[q] = c;
    }
    for (size_t q = order.size(); q < (size_t)nl; ++q) hq[q] = p->chunk_bulk;
  }
  CK(p, cudaMemcpyAsync(p->d_act, p->h_act, sizeof(int) * 2 * nl, cudaMemcpyHostToDevice, p->st));
  CK(p, cudaMemsetAsync(p->d_ndone, 0, sizeof(unsigned int) * 2, p->st));
  WinArgs A{};
  A.P = p->P;
  A.geo = p->d_geo;
  A.F = p->F;
  A.ctl = p->d_ctl;
  A.act = p->d_act;
  A.nact = (int)act.size();
  A.scheme = p->cfg.scheme;
  A.substeps = p->cfg.substeps;
  A.max_stages = p->cfg.max_stages;
  A.dtau = p->cfg.dtau;
  A.coef = p->d_coef;
  A.coef_off = p->d_coef_off;
  A.part = p->d_part_items;
  A.poff = p->d_poff;
  A.n_done = p->d_ndone;
  A.trace = p->d_trace;
  A.trace_n = p->d_trace_n;
  A.trace_cap = p->trace_cap;
  A.chunk_bulk = p->chunk_bulk;
  A.chunk_q = p->d_act + nl;
  A.chunk_tail = p->chunk_tail;
  A.tail_n = p->tail_n;
  A.tmap = p->d_tmap;
  A.sweep = (window_dataflow(p->dim) && p->d_tmap != nullptr) ? 1 : 0;
  A.rowprog = p->d_rowprog;
  A.proxy_fence = getenv("DDPMA_NO_PROXY_FENCE") ? 0 : 1;   // measurement knob only
  unsigned long long* d_probe = p->d_probe;
  const bool pe = d_probe != nullptr;
  if (pe) {
    A.probe_cap = 1 << 16;
    CK(p, cudaMemsetAsync(d_probe, 0, sizeof(unsigned long long) * 4 * A.probe_cap, p->st));
    A.probe = d_probe;
    A.probe_sub = order[0];
  }
  launch_window_begin(A, p->st);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (p->prof) {
    e0 = take_event(p);
    e1 = take_event(p);
    cudaEventRecord(e0, p->st);
  }
  launch_window(A, p->win_blocks, p->st);
  if (p->prof) cudaEventRecord(e1, p->st);
  ddpma_status s = check_launch(p, "window kernel");
  if (s != DDPMA_OK) return s;
  CK(p, cudaMemcpyAsync(p->h_ctl, p->d_ctl, sizeof(DevCtl) * nl, cudaMemcpyDeviceToHost, p->st));
  unsigned int ntr = 0;
  if (p->d_trace) CK(p, cudaMemcpyAsync(&ntr, p->d_trace_n, sizeof(unsigned), cudaMemcpyDeviceToHost, p->st));
  CK(p, cudaStreamSynchronize(p->st));
  double bytes = 0.0;
  long long nodes = 0;
  for (int l : act) {
    const DevCtl& c = p->h_ctl[l];
    DevCtl& prev = p->ctl_prev[l];
    const long long de = c.evals - prev.evals;
    p->last_evals[l] = de;
    bytes += c.bytes - prev.bytes;
    nodes += de * p->geo[l].nodes;
    p->rhs_evals += de;
    p->sub_evals[l] += de;
    prev.evals = c.evals;
    prev.bytes = c.bytes;
    p->ctl[l].yi = c.yi;
    p->ctl[l].fi = c.fi;
    if (c.fail_status != 0) {
      const int gid = p->local[l];
      if (!p->fail.set || gid < p->fail.gid) {
        p->fail = Failure{};
        p->fail.set = true;
        p->fail.gid = gid;
        p->fail.status = (ddpma_status)c.fail_status;
        p->fail.msg = c.fail_status == DDPMA_ERR_VALUE ? "cannot convert float NaN to integer"
                      : c.fail_status == DDPMA_ERR_OVERFLOW ? "cannot convert float infinity to integer"
                                                            : "internal step underflow";
        p->fail.t = c.fail_t;
        p->fail.h = c.fail_h;
        p->fail.local = l;
        p->fail.s = c.fail_s;
        p->fail.yi = c.fail_yi;
        p->fail.fi = c.fail_fi;
        p->fail.h04 = c.fail_h04;
        p->fail.nnodes = c.fail_nonfin ? -1 : -2;
      }
    }
  }
  if (pe) {
    std::vector<unsigned long long> pr(4 * (size_t)A.probe_cap);
    CK(p, cudaMemcpy(pr.data(), d_probe, sizeof(unsigned long long) * pr.size(), cudaMemcpyDeviceToHost));
    double s_wait = 0, s_proc = 0, s_dec = 0;
    long n = 0;
    for (int i = 0; i < A.probe_cap; ++i) {
      const unsigned long long* r = &pr[4 * (size_t)i];
      if (r[0] && r[1] && r[2] && r[3] && r[1] >= r[0] && r[2] >= r[1] && r[3] >= r[2]) {
        s_wait += (r[1] - r[0]) * 1e-3;
        s_proc += (r[2] - r[1]) * 1e-3;
        s_dec += (r[3] - r[2]) * 1e-3;
        ++n;
      }
    }
    fprintf(stderr, "PROBE sub %d actions %ld: avg publish->claim %.2f us, claim->done %.2f us, done->published %.2f us\n",
            p->local[A.probe_sub], n, n ? s_wait / n : 0.0, n ? s_proc / n : 0.0, n ? s_dec / n : 0.0);
  }
  if (getenv("DDPMA_TIMELINE")) {
    unsigned long long t0 = ~0ull;
    for (int l : act) t0 = std::min(t0, p->h_ctl[l].t_begin);
    fprintf(stderr, "TIMELINE");
    for (int l : act)
      fprintf(stderr, " %d:%.2fms/%lld", p->local[l], (p->h_ctl[l].t_done - t0) * 1e-6,
              p->h_ctl[l].evals);
    fprintf(stderr, "\n");
  }
  p->node_updates += nodes;
  p->algo_bytes += bytes;
  p->launches += 2;
  p->prof_launches[0] += 1;
  p->prof_bytes[0] += bytes;
  p->prof_nodes[0] += nodes;
  if (p->prof) p->prof_pending.push_back({e0, e1, 0, 0.0, 0});
  if (ntr > 0 && p->d_trace) {
    std::vector<TraceRec> tr(std::min<unsigned>(ntr, (unsigned)p->trace_cap));
    CK(p, cudaMemcpy(tr.data(), p->d_trace, sizeof(TraceRec) * tr.size(), cudaMemcpyDeviceToHost));
    for (auto& r : tr) {
      if (r.kind == 1) fprintf(stderr, "TRACE %d sigma %.17g\n", r.sub, r.val);
      else
        fprintf(stderr, "TRACE %d step %.17g %d %.17g %d %d\n", r.sub, r.h, r.s, r.val, r.flagged,
                r.accepted);
    }
  }
  return sync(p);
}

// Entries for every local subdomain (current buffers).
std::vector<Entry> all_entries(ddpma_plan* p, int* nb) {
  std::vector<Entry> ents;
  for (int l = 0; l < (int)p->local.size(); ++l) ents.push_back(make_entry(p, l));
  *nb = prefix_tiles(p, ents);
  return ents;
}

// Mesh/density/residual pass over local subdomains.
ddpma_status mesh_pass(ddpma_plan* p, bool with_res) {
  int nb;
  std::vector<Entry> ents = all_entries(p, &nb);
  void* d;
  ddpma_status s;
  if ((s = stage_put(p, ents.data(), ents.size() * sizeof(Entry), &d)) != DDPMA_OK) return s;
  launch_res_init(p->d_res, (int)p->local.size(), p->st);
  KArgs a = base_args(p);
  a.ent = (Entry*)d;
  a.nent = (int)ents.size();
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (p->prof) {
    e0 = take_event(p);
    e1 = take_event(p);
    cudaEventRecord(e0, p->st);
  }
  // _window_densities (schwarz.py:162-192): density, smoothing, relaxation
  int src = 0;
  upull_prepass(p, a, nb);
  if (p->cfg.monitor_smooth_passes > 0) {
    launch_rawfill(a, nb, 1, p->st);
    src = 1;
    for (int pass = 0; pass < p->cfg.monitor_smooth_passes; ++pass)
      for (int ax = 0; ax < p->dim; ++ax) {
        launch_smooth(a, nb, ax, src, 3 - src, p->st);
        src = 3 - src;
      }
  }
  const int blend = p->cfg.monitor_relax > 0.0 && p->raw_valid ? 1 : 0;
  launch_mesh_ex(a, nb, with_res ? 1 : 0, src, p->cfg.monitor_relax, blend, p->st);
  p->raw_valid = true;
  const long long nodes = entries_nodes(p, ents.data(), (int)ents.size());
  if (p->prof) {
    cudaEventRecord(e1, p->st);
    p->prof_pending.push_back({e0, e1, 1, 24.0 * nodes, nodes});
  }
  account(p, 1, nodes, with_res ? 24.0 : 16.0, false);
  launch_finalize((Entry*)d, (int)ents.size(), p->d_part, p->d_res, 0, p->st);
  launch_finalize((Entry*)d, (int)ents.size(), p->d_part2, p->d_res, 1, p->st);
  if ((s = check_launch(p, "mesh")) != DDPMA_OK) return s;
  CK(p, cudaMemcpyAsync(p->h_res, p->d_res, sizeof(SubRes) * p->local.size(),
                        cudaMemcpyDeviceToHost, p->st));
  if ((s = sync(p)) != DDPMA_OK) return s;
  const int n = (int)p->local.size();
  p->zpart.assign(n, 0.0);
  p->rawmax.assign(n, 0.0);
  p->resid.assign(n, 0.0);
  p->jmin.assign(n, 0.0);
  p->jmax.assign(n, 0.0);
  for (int l = 0; l < n; ++l) {
    const SubRes& r = p->h_res[l];
    p->zpart[l] = r.sum;
    p->resid[l] = std::sqrt(r.sum2);
    p->rawmax[l] = okey_dec(r.rawmax);
    if (r.jnan) {
      p->jmin[l] = p->jmax[l] = NAN;
    } else {
      p->jmin[l] = okey_dec(r.jmin);
      p->jmax[l] = okey_dec(r.jmax);
    }
  }
  p->density_ready = true;
  return DDPMA_OK;
}

void set_guard(ddpma_plan* p, double rho_max) {     // pma.py:188-190
  double guard = p->cfg.det_floor;
  if (rho_max != 0.0) guard = std::max(p->cfg.det_floor, 0.1 / (p->P.measure * rho_max));
  p->P.guard = guard;
  p->P.rguard = 1.0 / guard;
}

// snapshot + measure*rho for the listed local subdomains
ddpma_status prologue(ddpma_plan* p, const std::vector<int>& act, double z) {
  std::vector<Entry> ents;
  for (int l : act) ents.push_back(make_entry(p, l));
  const int nb = prefix_tiles(p, ents);
  void* d;
  ddpma_status s;
  if ((s = stage_put(p, ents.data(), ents.size() * sizeof(Entry), &d)) != DDPMA_OK) return s;
  KArgs a = base_args(p);
  a.ent = (Entry*)d;
  a.nent = (int)ents.size();
  launch_prologue(a, nb, z, p->st);
  account(p, 2, entries_nodes(p, ents.data(), (int)ents.size()), 32.0, false);
  p->have_old = true;
  return check_launch(p, "prologue");
}

long long axis_stride(const SubGeo& g, int dim, int axis) {
  if (dim == 2) return axis == 0 ? g.pitch : 1;
  if (axis == 0) return (long long)g.n[1] * g.pitch;
  return axis == 1 ? g.pitch : 1;
}

// tangential axes of a face normal to `axis`: t0 = highest remaining axis
void tang_axes(int dim, int axis, int* t0, int* t1) {
  int ax[2], m = 0;
  for (int q = dim - 1; q >= 0; --q)
    if (q != axis) ax[m++] = q;
  *t0 = ax[0];
  *t1 = dim == 3 ? ax[1] : -1;
}

// Faces of receiver `l` (local) from donors.  src_mode 0: donor snapshot
// (old), 1: donor current y.  Remote donors read from recv_dev segments.
void add_apply_jobs(ddpma_plan* p, int l, int src_mode, const double* recv_dev,
                    std::vector<FaceJob>& jobs, int& nnodes) {
  const ddpma_subdomain& R = p->subs[p->local[l]];
  const SubGeo& gr = p->geo[l];
  for (int k = 0; k < p->dim; ++k) {
    for (int side = 0; side < 2; ++side) {
      const int d = R.donor[k][side];
      if (d < 0) continue;
      int t0, t1;
      tang_axes(p->dim, k, &t0, &t1);
      FaceJob J{};
      J.dst = p->F.y[p->ctl[l].yi] + gr.off + (side ? (long long)(gr.n[k] - 1) * axis_stride(gr, p->dim, k) : 0);
      J.dstr[0] = axis_stride(gr, p->dim, t0);
      J.dstr[1] = t1 >= 0 ? axis_stride(gr, p->dim, t1) : 0;
      J.ext[0] = gr.n[t0];
      J.ext[1] = t1 >= 0 ? gr.n[t1] : 1;
      // lowest donor id wins at shared edge nodes (schwarz.py:141-147)
      for (int q = 0; q < 2; ++q) {
        const int ta = q == 0 ? t0 : t1;
        if (ta < 0) continue;
        const int dlo = R.donor[ta][0], dhi = R.donor[ta][1];
        J.skip_lo[q] = (dlo >= 0 && dlo < d) ? 1 : 0;
        J.skip_hi[q] = (dhi >= 0 && dhi < d) ? 1 : 0;
      }
      const int dl = p->local_of[d];
      if (dl >= 0) {
        const ddpma_subdomain& D = p->subs[d];
        const SubGeo& gd = p->geo[dl];
        const double* base = src_mode == 0 ? p->F.old : p->F.y[p->ctl[dl].yi];
        long long off = gd.off + (long long)(R.box[k][side] - D.box[k][0]) * axis_stride(gd, p->dim, k);
        off += (long long)(R.box[t0][0] - D.box[t0][0]) * axis_stride(gd, p->dim, t0);
        if (t1 >= 0) off += (long long)(R.box[t1][0] - D.box[t1][0]) * axis_stride(gd, p->dim, t1);
        J.src = base + off;
        J.sstr[0] = axis_stride(gd, p->dim, t0);
        J.sstr[1] = t1 >= 0 ? axis_stride(gd, p->dim, t1) : 0;
      } else {
        long long off = -1;
        for (auto& sg : p->recv_segs)
          if (sg.recv_gid == R.id && sg.axis == k && sg.side == side) off = sg.off;
        if (off < 0 || recv_dev == nullptr) continue;   // validated by caller
        J.src = recv_dev + off;
        J.sstr[0] = 1;
        J.sstr[1] = J.ext[0];
      }
      J.node_begin = nnodes;
      nnodes += J.ext[0] * J.ext[1];
      jobs.push_back(J);
    }
  }
}

ddpma_status run_faces(ddpma_plan* p, std::vector<FaceJob>& jobs, int nnodes) {
  if (jobs.empty()) return DDPMA_OK;
  void* d;
  ddpma_status s;
  if ((s = stage_put(p, jobs.data(), jobs.size() * sizeof(FaceJob), &d)) != DDPMA_OK) return s;
  launch_faces((FaceJob*)d, (int)jobs.size(), nnodes, p->st);
  account(p, 2, nnodes, 16.0, false);
  return check_launch(p, "faces");
}

ddpma_status check_z(ddpma_plan* p, double z) {   // schwarz.py:187-189
  if (!std::isfinite(z) || z <= 0.0) {
    char buf[128];
    snprintf(buf, sizeof buf, "%.17g", z);
    p->err = std::string("transport quadrature of the mesh density is ") + buf;
    p->fail = Failure{};
    p->fail.set = true;
    p->fail.status = DDPMA_ERR_INVALID_MONITOR;
    p->fail.t = z;   // the value, for the host mirror's message
    return DDPMA_ERR_INVALID_MONITOR;
  }
  return DDPMA_OK;
}

ddpma_status report_failure(ddpma_plan* p) {
  char buf[256];
  if (p->fail.status == DDPMA_ERR_STIFFNESS) {
    snprintf(buf, sizeof buf, "internal step underflow at tau offset %.3e (h = %.3e, window = %.3e)",
             p->fail.t, p->fail.h, p->cfg.dtau);
    p->err = buf;
  } else {
    p->err = p->fail.msg;
  }
  return p->fail.status;
}

ddpma_status begin_window_all(ddpma_plan* p, double z, double rho_max) {
  p->z = z;
  p->rho_max = rho_max;
  set_guard(p, rho_max);
  std::vector<int> all(p->local.size());
  for (int l = 0; l < (int)all.size(); ++l) all[l] = l;
  return prologue(p, all, z);
}

double window_z(ddpma_plan* p) {      // z = 0.0; z += partial (id order), schwarz.py:182-186
  double z = 0.0;
  for (int l = 0; l < (int)p->local.size(); ++l) z += p->zpart[l];
  return z;
}

double window_rho_max(ddpma_plan* p, double z) {   // schwarz.py:190-191
  double m = p->rawmax[0] / z;
  for (int l = 1; l < (int)p->local.size(); ++l) {
    const double v = p->rawmax[l] / z;
    if (v > m) m = v;
  }
  return m;
}

ddpma_status do_box_entry(ddpma_plan* p, int l, void** d_ent, int* nb) {
  std::vector<Entry> ents{make_entry(p, l)};
  *nb = prefix_tiles(p, ents);
  return stage_put(p, ents.data(), sizeof(Entry), d_ent);
}

ddpma_status ensure_scratch(ddpma_plan* p, long long elems) {
  if (elems <= p->scratch_elems) return DDPMA_OK;
  if (p->d_scratch) cudaFree(p->d_scratch);
  p->d_scratch = nullptr;
  CK(p, cudaMalloc((void**)&p->d_scratch, sizeof(double) * elems));
  p->scratch_elems = elems;
  return DDPMA_OK;
}

ddpma_status h2d_box(ddpma_plan* p, int l, const double* host, double* field) {
  const SubGeo& g = p->geo[l];
  ddpma_status s;
  if ((s = ensure_scratch(p, g.nodes)) != DDPMA_OK) return s;
  CK(p, cudaMemcpyAsync(p->d_scratch, host, sizeof(double) * g.nodes, cudaMemcpyHostToDevice, p->st));
  void* d;
  int nb;
  if ((s = do_box_entry(p, l, &d, &nb)) != DDPMA_OK) return s;
  KArgs a = base_args(p);
  a.ent = (Entry*)d;
  a.nent = 1;
  launch_box_copy(a, nb, p->d_scratch, field, 1, p->st);
  return sync(p);
}

ddpma_status d2h_box(ddpma_plan* p, int l, const double* field, double* host) {
  const SubGeo& g = p->geo[l];
  ddpma_status s;
  if ((s = ensure_scratch(p, g.nodes)) != DDPMA_OK) return s;
  void* d;
  int nb;
  if ((s = do_box_entry(p, l, &d, &nb)) != DDPMA_OK) return s;
  KArgs a = base_args(p);
  a.ent = (Entry*)d;
  a.nent = 1;
  launch_box_copy(a, nb, field, p->d_scratch, 0, p->st);
  CK(p, cudaMemcpyAsync(host, p->d_scratch, sizeof(double) * g.nodes, cudaMemcpyDeviceToHost, p->st));
  return sync(p);
}

int local_of_checked(ddpma_plan* p, int gid) {
  if (gid < 0 || gid >= p->nsub) return -1;
  return p->local_of[gid];
}

}  // namespace

// ================================================================= C ABI ==

extern "C" const char* ddpma_last_error(const ddpma_plan* p) {
  return p ? p->err.c_str() : global_error();
}

extern "C" void* ddpma_stream(const ddpma_plan* p) { return p ? (void*)p->st : nullptr; }

extern "C" const char* ddpma_window_kernel(const ddpma_plan* p) {
  if (!p) return "";
  if (p->dim == 3) return "k_windowP<3>";
  return (window_dataflow(2) && p->d_tmap != nullptr) ? "k_windowD" : "k_windowP<2>";
}

extern "C" void ddpma_plan_destroy(ddpma_plan* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  if (p->st) cudaStreamSynchronize(p->st);
  for (auto e : p->ev_pool) cudaEventDestroy(e);
  cudaFree(p->d_arena);
  cudaFree(p->d_geo);
  cudaFree(p->d_mon);
  for (void* q : p->lat_allocs) cudaFree(q);
  cudaFree(p->d_res);
  cudaFree(p->d_part);
  cudaFree(p->d_part2);
  cudaFree(p->d_stage);
  cudaFree(p->d_scratch);
  if (p->h_res) cudaFreeHost(p->h_res);
  for (int r = 0; r < ddpma_plan::R; ++r) {
    if (p->h_ent[r]) cudaFreeHost(p->h_ent[r]);
    cudaFree(p->d_ent[r]);
    if (p->ring_ev[r]) cudaEventDestroy(p->ring_ev[r]);
  }
  cudaFree(p->d_ring);
  if (p->h_ring) cudaFreeHost(p->h_ring);
  cudaFree(p->d_partring);
  cudaFree(p->d_ctl);
  if (p->h_ctl) cudaFreeHost(p->h_ctl);
  cudaFree(p->d_coef);
  cudaFree(p->d_coef_off);
  cudaFree(p->d_part_items);
  cudaFree(p->d_poff);
  cudaFree(p->d_act);
  if (p->h_act) cudaFreeHost(p->h_act);
  cudaFree(p->d_ndone);
  cudaFree(p->d_trace);
  cudaFree(p->d_tmap);
  cudaFree(p->d_probe);
  cudaFree(p->d_rowprog);
  if (p->h_stage) cudaFreeHost(p->h_stage);
  if (p->st) cudaStreamDestroy(p->st);
  delete p;
}

extern "C" ddpma_status ddpma_plan_create(const ddpma_grid* grid, const ddpma_subdomain* subs,
                                          int nsub, const int* local_ids, int nlocal,
                                          const ddpma_monitor* monitor,
                                          const ddpma_solver_cfg* cfg, int device,
                                          ddpma_plan** out) {
  *out = nullptr;
  if (!grid || !subs || nsub < 1 || !monitor || !cfg) {
    set_global_error("ddpma_plan_create: null argument");
    return DDPMA_ERR_STATE;
  }
  if (grid->dim != 2 && grid->dim != 3) {
    set_global_error("dim must be 2 or 3");
    return DDPMA_ERR_CONFIG;
  }
  if (cfg->dtau <= 0.0) {
    set_global_error("window length must be > 0");
    return DDPMA_ERR_CONFIG;
  }
  if (cfg->scheme == DDPMA_SCHEME_ADAPTIVE && cfg->max_stages < 2) {
    set_global_error("max_stages must be >= 2 for the adaptive RKC2 scheme");
    return DDPMA_ERR_CONFIG;
  }
  if (cfg->scheme == DDPMA_SCHEME_EULER && cfg->substeps < 1) {
    set_global_error("euler mode needs at least 1 substep");
    return DDPMA_ERR_CONFIG;
  }
  // window scheduler knobs (profiling sweeps): parsed once, validated
  int knob[3] = {8, 2, 16};   // DDPMA_CHUNK, DDPMA_CHUNK_TAIL (r1 sweeps: 2 beats 1 by ~1.2 %), DDPMA_TAIL_N
  {
    const char* names[3] = {"DDPMA_CHUNK", "DDPMA_CHUNK_TAIL", "DDPMA_TAIL_N"};
    const int hi[3] = {64, 64, 1 << 20};
    for (int i = 0; i < 3; ++i) {
      const char* v = getenv(names[i]);
      if (!v) continue;
      char* end = nullptr;
      const long x = strtol(v, &end, 10);
      if (end == v || *end != '\0' || x < 1 || x > hi[i]) {
        set_global_error(std::string(names[i]) + " must be an integer in [1, " +
                         std::to_string(hi[i]) + "], got '" + v + "'");
        return DDPMA_ERR_CONFIG;
      }
      knob[i] = (int)x;
    }
  }
  if (monitor->kind == DDPMA_MON_MIXTURE && (monitor->nbumps < 0 || monitor->nbumps > MAXB)) {
    set_global_error("mixture monitor supports at most 64 bumps");
    return DDPMA_ERR_CONFIG;
  }
  if (monitor->kind < DDPMA_MON_UNIFORM || monitor->kind > DDPMA_MON_SAMPLED) {
    set_global_error("unknown monitor kind");
    return DDPMA_ERR_CONFIG;
  }
  if (!sampled_ok(monitor, grid->dim)) {
    set_global_error("sampled field needs >= 2 lattice nodes per axis and its arrays");
    return DDPMA_ERR_CONFIG;
  }
  if (monitor->kind >= DDPMA_MON_BURGERS2D && monitor->kind != DDPMA_MON_SAMPLED) {   // test-function domains (monitor.py:223-345)
    const bool three = monitor->kind == DDPMA_MON_SPHERE3D || monitor->kind == DDPMA_MON_NINE_SPHERES3D;
    if (grid->dim != (three ? 3 : 2)) {
      set_global_error("grid dimension does not match monitor domain");
      return DDPMA_ERR_CONFIG;
    }
    if (monitor->kind == DDPMA_MON_BURGERS2D && !(monitor->eps > 0.0)) {
      set_global_error("burgers2d needs eps > 0");
      return DDPMA_ERR_CONFIG;
    }
  }
  auto* p = new ddpma_plan();
  p->chunk_bulk = knob[0];
  p->chunk_tail = knob[1];
  p->tail_n = knob[2];
  if (const char* e = getenv("DDPMA_CHUNK_ADAPT")) p->chunk_adapt = e[0] != '0';   // A/B knob
  p->device = device;
  p->grid = *grid;
  p->cfg = *cfg;
  p->dim = grid->dim;
  p->subs.assign(subs, subs + nsub);
  p->nsub = nsub;
  p->local_of.assign(nsub, -1);
  if (local_ids) {
    std::vector<int> ids(local_ids, local_ids + nlocal);
    std::sort(ids.begin(), ids.end());
    p->local = ids;
  } else {
    for (int i = 0; i < nsub; ++i) p->local.push_back(i);
  }
  for (int l = 0; l < (int)p->local.size(); ++l) {
    if (p->local[l] < 0 || p->local[l] >= nsub) {
      set_global_error("local subdomain id out of range");
      delete p;
      return DDPMA_ERR_CONFIG;
    }
    p->local_of[p->local[l]] = l;
  }
  if ((int)p->local.size() == nsub) {
    // level(l) = 1 + max level over the face donors / receivers of lower id
    // (schwarz.py:216-233 visits ids in order; see ddpma_run).
    // DDPMA_ALT_SERIAL=1 keeps one subdomain per launch (A/B comparisons).
    const bool serial = getenv("DDPMA_ALT_SERIAL") != nullptr;
    std::vector<int> level(nsub, 0);
    if (serial)
      for (int i = 0; i < nsub; ++i) level[i] = i;
    else
      ddpma_alternating_levels(p->dim, p->subs.data(), nsub, level.data());
    for (int i = 0; i < nsub; ++i) {
      if ((int)p->alt_levels.size() <= level[i]) p->alt_levels.resize(level[i] + 1);
      p->alt_levels[level[i]].push_back(p->local_of[i]);
    }
  }
  cudaError_t ce = cudaSetDevice(device);
  if (ce != cudaSuccess) {
    set_global_error(std::string("cudaSetDevice: ") + cudaGetErrorString(ce));
    delete p;
    return DDPMA_ERR_CUDA;
  }
  // problem constants
  Prob& P = p->P;
  P.dim = p->dim;
  P.pow2 = 1;
  double measure = 1.0;
  for (int k = 0; k < p->dim; ++k) {
    const double a = grid->extents[k][0], b = grid->extents[k][1];
    const int n = grid->counts[k];
    AxisC& A = P.ax[k];
    A.h = grid->explicit_geom ? grid->spacing[k] : (b - a) / (double)(n - 1);
    A.n = n;
    A.hh = A.h * A.h;
    A.twoh = 2. * A.h;
    A.ea = -1.5 / A.h;
    A.eb = 2. / A.h;
    A.ec = -0.5 / A.h;
    A.fa = 0.5 / A.h;
    A.fb = -2. / A.h;
    A.fc = 1.5 / A.h;
    A.w_in = A.h;
    A.w_end = 0.5 * A.h;
    if (!is_pow2(A.h)) P.pow2 = 0;
    P.a0[k] = a;
    measure *= b - a;
  }
  for (int k = 0; k < p->dim; ++k) {
    P.ax[k].ihh = 1.0 / P.ax[k].hh;
    P.ax[k].itwoh = 1.0 / P.ax[k].twoh;
  }
  P.measure = grid->explicit_geom ? grid->measure : measure;
  P.floor = cfg->det_floor;
  P.guard = cfg->det_floor;
  P.rguard = 1.0 / cfg->det_floor;
  P.atol = cfg->atol;
  P.rtol = cfg->rtol;
  // monitor
  fill_monitor(monitor, p->dim, p->mon);
  p->u_backed = monitor->kind >= DDPMA_MON_BURGERS2D && monitor->u_backed;
  // geometry + arena
  long long off = 0;
  int tiles = 0;
  long long nrows_total = 0;
  for (int l = 0; l < (int)p->local.size(); ++l) {
    const ddpma_subdomain& S = p->subs[p->local[l]];
    SubGeo g{};
    g.gid = S.id;
    g.n[2] = 1;
    for (int k = 0; k < p->dim; ++k) {
      g.n[k] = S.box[k][1] - S.box[k][0] + 1;
      g.plo[k] = S.face[k][0] == DDPMA_FACE_PHYSICAL;
      g.phi[k] = S.face[k][1] == DDPMA_FACE_PHYSICAL;
      const double a = grid->extents[k][0], h = P.ax[k].h;
      g.alo[k] = a + (double)S.box[k][0] * h;          // a + np.arange(n)*h (grid.py:51)
      g.ahi[k] = a + (double)S.box[k][1] * h;
      if (grid->explicit_geom) {
        g.alo[k] = grid->face_coord[k][0];
        g.ahi[k] = grid->face_coord[k][1];
      }
      g.halo[k] = h * g.alo[k];
      g.hahi[k] = h * g.ahi[k];
      g.glo[k] = S.box[k][0];
      g.olo[k] = S.owned[k][0] - S.box[k][0];
      g.ohi[k] = S.owned[k][1] - S.box[k][0];
    }
    const int last = p->dim - 1;
    g.pitch = (int)round_up(g.n[last], 8);
    const long long rows = p->dim == 2 ? g.n[0] : (long long)g.n[0] * g.n[1];
    g.off = off;
    off += round_up(rows * g.pitch, 32);
    g.nodes = (long long)g.n[0] * g.n[1] * (p->dim == 3 ? g.n[2] : 1);
    if (p->dim == 2) {
      g.tiles_x = (g.n[1] + TX - 1) / TX;
      g.tiles_y = (g.n[0] + TY - 1) / TY;
      g.tiles_z = 1;
    } else {
      g.tiles_x = (g.n[2] + TX - 1) / TX;
      g.tiles_y = (g.n[1] + TY - 1) / TY;
      g.tiles_z = g.n[0];
    }
    g.ntiles = g.tiles_x * g.tiles_y * g.tiles_z;
    if (p->dim == 2) {
      g.items_x = (g.n[1] + TX - 1) / TX;
      g.items_y = (g.n[0] + IR2 - 1) / IR2;
      g.items_z = 1;
    } else {
      g.items_x = (g.n[2] + TX - 1) / TX;
      g.items_y = (g.n[1] + TY - 1) / TY;
      g.items_z = (g.n[0] + IZ3 - 1) / IZ3;
    }
    g.nitems = g.items_x * g.items_y * g.items_z;
    g.ipr = p->dim == 2 ? g.items_x : g.items_x * g.items_y;   // a row of items / a plane
    g.nrows = g.nitems / g.ipr;
    g.rowoff = nrows_total;
    nrows_total += g.nrows;
    tiles += g.ntiles;
    p->geo.push_back(g);
  }
  p->arena = off;
  p->total_tiles = tiles;
  p->total_rows = nrows_total;
  p->ctl.assign(p->local.size(), Ctl{});
  p->sub_evals.assign(p->local.size(), 0);
  p->last_evals.assign(p->local.size(), 0);
  p->ctl_prev.assign(p->local.size(), DevCtl{});
  ddpma_status s = DDPMA_OK;
  auto fail = [&](cudaError_t e, const char* w) {
    set_global_error(std::string("CUDA error in ") + w + ": " + cudaGetErrorString(e));
    ddpma_plan_destroy(p);
    return DDPMA_ERR_CUDA;
  };
  if ((ce = cudaStreamCreateWithFlags(&p->st, cudaStreamNonBlocking)) != cudaSuccess)
    return fail(ce, "stream");
  const size_t fbytes = sizeof(double) * (size_t)p->arena;
  if ((ce = cudaMalloc((void**)&p->d_arena, fbytes * 10)) != cudaSuccess) return fail(ce, "arena");
  if ((ce = cudaMemsetAsync(p->d_arena, 0, fbytes * 10, p->st)) != cudaSuccess) return fail(ce, "memset");
  double* base = p->d_arena;
  p->F.y[0] = base + 0 * p->arena;
  p->F.y[1] = base + 1 * p->arena;
  p->F.f[0] = base + 2 * p->arena;
  p->F.f[1] = base + 3 * p->arena;
  p->F.d[0] = base + 4 * p->arena;
  p->F.d[1] = base + 5 * p->arena;
  p->F.d[2] = base + 6 * p->arena;
  p->F.mr = base + 7 * p->arena;
  p->F.raw = base + 8 * p->arena;
  p->F.old = base + 9 * p->arena;
  if ((ce = cudaMalloc((void**)&p->d_geo, sizeof(SubGeo) * p->geo.size())) != cudaSuccess)
    return fail(ce, "geo");
  if ((ce = cudaMemcpy(p->d_geo, p->geo.data(), sizeof(SubGeo) * p->geo.size(),
                       cudaMemcpyHostToDevice)) != cudaSuccess)
    return fail(ce, "geo copy");
  if ((ce = upload_lattice(monitor, p->dim, p->mon, p->lat_allocs)) != cudaSuccess)
    return fail(ce, "sampled lattice");
  if ((ce = cudaMalloc((void**)&p->d_mon, sizeof(MonitorD))) != cudaSuccess) return fail(ce, "mon");
  if ((ce = cudaMemcpy(p->d_mon, &p->mon, sizeof(MonitorD), cudaMemcpyHostToDevice)) != cudaSuccess)
    return fail(ce, "mon copy");
  if ((ce = cudaMalloc((void**)&p->d_res, sizeof(SubRes) * p->local.size())) != cudaSuccess)
    return fail(ce, "res");
  if ((ce = cudaMallocHost((void**)&p->h_res, sizeof(SubRes) * p->local.size())) != cudaSuccess)
    return fail(ce, "res host");
  if ((ce = cudaMalloc((void**)&p->d_part, sizeof(double) * std::max(tiles, 1))) != cudaSuccess)
    return fail(ce, "part");
  if ((ce = cudaMalloc((void**)&p->d_part2, sizeof(double) * std::max(tiles, 1))) != cudaSuccess)
    return fail(ce, "part2");
  for (int r = 0; r < ddpma_plan::R; ++r) {
    if ((ce = cudaMallocHost((void**)&p->h_ent[r], sizeof(Entry) * p->local.size())) != cudaSuccess)
      return fail(ce, "ent host");
    if ((ce = cudaMalloc((void**)&p->d_ent[r], sizeof(Entry) * p->local.size())) != cudaSuccess)
      return fail(ce, "ent dev");
    if ((ce = cudaEventCreateWithFlags(&p->ring_ev[r], cudaEventDisableTiming)) != cudaSuccess)
      return fail(ce, "ring event");
  }
  if ((ce = cudaMalloc((void**)&p->d_ring, sizeof(SubRes) * p->local.size() * ddpma_plan::R)) !=
      cudaSuccess)
    return fail(ce, "ring");
  if ((ce = cudaMallocHost((void**)&p->h_ring, sizeof(SubRes) * p->local.size() * ddpma_plan::R)) !=
      cudaSuccess)
    return fail(ce, "ring host");
  if ((ce = cudaMalloc((void**)&p->d_partring,
                       sizeof(double) * std::max(tiles, 1) * ddpma_plan::R)) != cudaSuccess)
    return fail(ce, "part ring");
  {   // device controller: state, RKC2 tables, item partials, trace
    const int nl = (int)p->local.size();
    if ((ce = cudaMalloc((void**)&p->d_ctl, sizeof(DevCtl) * nl)) != cudaSuccess) return fail(ce, "ctl");
    if ((ce = cudaMallocHost((void**)&p->h_ctl, sizeof(DevCtl) * nl)) != cudaSuccess) return fail(ce, "ctl host");
    memset(p->h_ctl, 0, sizeof(DevCtl) * nl);
    const int ms = std::max(2, cfg->max_stages);
    std::vector<int> off(ms + 1, 0);
    std::vector<double> tab;
    for (int sst = 2; sst <= ms && cfg->scheme == DDPMA_SCHEME_ADAPTIVE; ++sst) {
      off[sst] = (int)(tab.size() / 4);
      const RkcCoeffs& rc = coeffs(p, sst);
      for (int j = 0; j <= sst; ++j) {
        if (j == 0) {
          tab.insert(tab.end(), {rc.mu1t, rc.w0, rc.w1, 0.0});
        } else {
          tab.insert(tab.end(), {rc.mu[j], rc.nu[j], rc.mut[j], rc.gt[j]});
        }
      }
    }
    p->coeff_cache.clear();
    p->coeff_cache.shrink_to_fit();
    if (tab.empty()) tab.assign(4, 0.0);
    if ((ce = cudaMalloc((void**)&p->d_coef, sizeof(double) * tab.size())) != cudaSuccess) return fail(ce, "coef");
    if ((ce = cudaMemcpy(p->d_coef, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
      return fail(ce, "coef copy");
    if ((ce = cudaMalloc((void**)&p->d_coef_off, sizeof(int) * off.size())) != cudaSuccess) return fail(ce, "coef off");
    if ((ce = cudaMemcpy(p->d_coef_off, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
      return fail(ce, "coef off copy");
    std::vector<long long> poff(nl);
    long long acc = 0;
    for (int l = 0; l < nl; ++l) {
      poff[l] = acc;
      acc += p->geo[l].nitems;
    }
    if ((ce = cudaMalloc((void**)&p->d_part_items, sizeof(double) * std::max(acc, 1LL))) != cudaSuccess)
      return fail(ce, "part items");
    if ((ce = cudaMalloc((void**)&p->d_poff, sizeof(long long) * nl)) != cudaSuccess) return fail(ce, "poff");
    if ((ce = cudaMemcpy(p->d_poff, poff.data(), sizeof(long long) * nl, cudaMemcpyHostToDevice)) != cudaSuccess)
      return fail(ce, "poff copy");
    if ((ce = cudaMalloc((void**)&p->d_act, sizeof(int) * 2 * nl)) != cudaSuccess) return fail(ce, "act");
    if ((ce = cudaMallocHost((void**)&p->h_act, sizeof(int) * 2 * nl)) != cudaSuccess) return fail(ce, "act host");
    if ((ce = cudaMalloc((void**)&p->d_ndone, sizeof(unsigned int) * 2)) != cudaSuccess) return fail(ce, "ndone");
    p->d_trace_n = p->d_ndone + 1;
    if (g_trace) {
      p->trace_cap = 1 << 22;
      if ((ce = cudaMalloc((void**)&p->d_trace, sizeof(TraceRec) * p->trace_cap)) != cudaSuccess)
        return fail(ce, "trace");
    }
    p->win_blocks = window_blocks(p->dim, P.pow2);
    if ((ce = cudaMalloc((void**)&p->d_rowprog, sizeof(unsigned long long) * std::max(1LL, p->total_rows))) != cudaSuccess)
      return fail(ce, "rowprog");
    if ((ce = cudaMemsetAsync(p->d_rowprog, 0, sizeof(unsigned long long) * std::max(1LL, p->total_rows), p->st)) != cudaSuccess)
      return fail(ce, "rowprog memset");
    if (getenv("DDPMA_PROBE")) {
      if ((ce = cudaMalloc((void**)&p->d_probe, sizeof(unsigned long long) * 4 * (1 << 16))) != cudaSuccess)
        return fail(ce, "probe");
    }
    if (getenv("DDPMA_NO_TMA") == nullptr) {
      // one tensor map per (subdomain, field, box).  2D: halo box 36 x (IR2+2)
      // at (c0-2, r0-1), centre box 32 x IR2.  3D: halo box 36 x (TY+2) x
      // (IZ3+2) at (c0-2, r0-1, z0-1), centre box 32 x TY x IZ3.  Out-of-box
      // elements are zero-filled.
      typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
      void* fnp = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q) ==
              cudaSuccess && fnp) {
        EncodeFn enc = (EncodeFn)fnp;
        double* fields[TF_N] = {p->F.y[0], p->F.y[1], p->F.f[0], p->F.f[1],
                                p->F.d[0], p->F.d[1], p->F.d[2], p->F.mr};
        std::vector<CUtensorMap> maps((size_t)nl * TF_N * 2);
        bool ok = true;
        for (int l = 0; l < nl && ok; ++l) {
          const SubGeo& g = p->geo[l];
          const bool d3 = p->dim == 3;
          const cuuint32_t rank = d3 ? 3 : 2;
          const cuuint64_t gdim[3] = {(cuuint64_t)(d3 ? g.n[2] : g.n[1]),
                                      (cuuint64_t)(d3 ? g.n[1] : g.n[0]), (cuuint64_t)g.n[0]};
          const cuuint64_t gstr[2] = {(cuuint64_t)g.pitch * 8,
                                      (cuuint64_t)g.pitch * 8 * (cuuint64_t)g.n[1]};
          const cuuint32_t estr[3] = {1, 1, 1};
          for (int f = 0; f < TF_N && ok; ++f) {
            for (int kind = 0; kind < 2; ++kind) {
              cuuint32_t box[3];
              if (!d3) {
                box[0] = kind == 0 ? TX + 4 : TX;
                box[1] = kind == 0 ? IR2 + 2 : IR2;
                box[2] = 1;
              } else {
                box[0] = kind == 0 ? TX + 4 : TX;
                box[1] = kind == 0 ? TY + 2 : TY;
                box[2] = kind == 0 ? IZ3 + 2 : IZ3;
              }
              CUresult r = enc(&maps[((size_t)l * TF_N + f) * 2 + kind], CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                               rank, fields[f] + g.off, gdim, gstr, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
              if (r != CUDA_SUCCESS) ok = false;
            }
          }
        }
        if (ok) {
          if ((ce = cudaMalloc(&p->d_tmap, sizeof(CUtensorMap) * maps.size())) != cudaSuccess)
            return fail(ce, "tmap");
          if ((ce = cudaMemcpy(p->d_tmap, maps.data(), sizeof(CUtensorMap) * maps.size(),
                               cudaMemcpyHostToDevice)) != cudaSuccess)
            return fail(ce, "tmap copy");
        }
      }
    }
    p->host_ctl = getenv("DDPMA_HOST_CONTROLLER") != nullptr;
  }
  p->stage_cap = 1 << 20;
  if ((ce = cudaMallocHost((void**)&p->h_stage, p->stage_cap)) != cudaSuccess) return fail(ce, "stage");
  if ((ce = cudaMalloc((void**)&p->d_stage, p->stage_cap)) != cudaSuccess) return fail(ce, "stage dev");
  if ((ce = cudaStreamSynchronize(p->st)) != cudaSuccess) return fail(ce, "init sync");
  (void)s;
  *out = p;
  return DDPMA_OK;
}

// Fresh integrators for every local subdomain (schwarz.py:133,
// integrate.py:118-123: no sigma / step caches yet).
ddpma_status reset_integrators(ddpma_plan* p) {
  for (auto& c : p->ctl) c = Ctl{};
  const int nl = (int)p->local.size();
  memset(p->h_ctl, 0, sizeof(DevCtl) * nl);
  for (int l = 0; l < nl; ++l) p->h_ctl[l].interval = 25;   // _SIGMA_REFRESH
  CK(p, cudaMemcpyAsync(p->d_ctl, p->h_ctl, sizeof(DevCtl) * nl, cudaMemcpyHostToDevice, p->st));
  // the sweep row counters start with the controllers (DevCtl::sbase = 0)
  if (p->d_rowprog)
    CK(p, cudaMemsetAsync(p->d_rowprog, 0, sizeof(unsigned long long) * std::max(1LL, p->total_rows), p->st));
  p->ctl_prev.assign(nl, DevCtl{});
  p->last_evals.assign(nl, 0);
  p->sub_evals.assign(nl, 0);
  return DDPMA_OK;
}

extern "C" ddpma_status ddpma_set_state(ddpma_plan* p, const double* psi_global_host) {
  CK(p, cudaSetDevice(p->device));
  ddpma_status s0 = reset_integrators(p);
  if (s0 != DDPMA_OK) return s0;
  int nb;
  std::vector<Entry> ents = all_entries(p, &nb);
  void* d;
  ddpma_status s;
  if ((s = stage_put(p, ents.data(), ents.size() * sizeof(Entry), &d)) != DDPMA_OK) return s;
  KArgs a = base_args(p);
  a.ent = (Entry*)d;
  a.nent = (int)ents.size();
  if (psi_global_host == nullptr) {
    launch_psi0(a, nb, p->st);
  } else {
    long long n = 1;
    for (int k = 0; k < p->dim; ++k) n *= p->grid.counts[k];
    double* tmp = nullptr;
    CK(p, cudaMalloc((void**)&tmp, sizeof(double) * n));
    CK(p, cudaMemcpyAsync(tmp, psi_global_host, sizeof(double) * n, cudaMemcpyHostToDevice, p->st));
    launch_scatter(a, nb, tmp, p->st);
    CK(p, cudaStreamSynchronize(p->st));
    cudaFree(tmp);
  }
  if ((s = check_launch(p, "set_state")) != DDPMA_OK) return s;
  p->state_set = true;
  p->density_ready = false;
  p->have_old = false;
  p->raw_valid = false;
  p->fail = Failure{};
  return sync(p);
}

extern "C" ddpma_status ddpma_density(ddpma_plan* p, double* z_part, double* raw_max, double* res,
                                      double* jac_min, double* jac_max) {
  if (!p->state_set) {
    p->err = "state not set";
    return DDPMA_ERR_STATE;
  }
  CK(p, cudaSetDevice(p->device));
  ddpma_status s = mesh_pass(p, p->have_old);
  if (s != DDPMA_OK) return s;
  for (int i = 0; i < p->nsub; ++i) {
    const int l = p->local_of[i];
    if (z_part) z_part[i] = l >= 0 ? p->zpart[l] : 0.0;
    if (raw_max) raw_max[i] = l >= 0 ? p->rawmax[l] : 0.0;
    if (res) res[i] = l >= 0 ? p->resid[l] : 0.0;
    if (jac_min) jac_min[i] = l >= 0 ? p->jmin[l] : 0.0;
    if (jac_max) jac_max[i] = l >= 0 ? p->jmax[l] : 0.0;
  }
  return DDPMA_OK;
}

extern "C" ddpma_status ddpma_begin_window(ddpma_plan* p, double z, double rho_max) {
  CK(p, cudaSetDevice(p->device));
  if (!p->density_ready) {
    p->err = "ddpma_density must run before ddpma_begin_window";
    return DDPMA_ERR_STATE;
  }
  ddpma_status s = check_z(p, z);
  if (s != DDPMA_OK) return s;
  if ((s = begin_window_all(p, z, rho_max)) != DDPMA_OK) return s;
  return sync(p);
}

extern "C" ddpma_status ddpma_trace_counts(ddpma_plan* p, const int* rank_of, int nranks,
                                           int my_rank, int64_t* send_counts,
                                           int64_t* recv_counts) {
  p->rank_of.assign(rank_of, rank_of + p->nsub);
  p->nranks = nranks;
  p->my_rank = my_rank;
  p->send_segs.clear();
  p->recv_segs.clear();
  for (int r = 0; r < nranks; ++r) {
    send_counts[r] = 0;
    recv_counts[r] = 0;
  }
  // canonical order: receiver id, axis, side; per peer contiguous, peers in rank order
  std::vector<std::vector<ddpma_plan::Seg>> sendp(nranks), recvp(nranks);
  for (int R = 0; R < p->nsub; ++R) {
    const ddpma_subdomain& S = p->subs[R];
    for (int k = 0; k < p->dim; ++k) {
      for (int side = 0; side < 2; ++side) {
        const int d = S.donor[k][side];
        if (d < 0) continue;
        const int rr = rank_of[R], rd = rank_of[d];
        if (rr == rd) continue;
        int t0, t1;
        tang_axes(p->dim, k, &t0, &t1);
        ddpma_plan::Seg sg{R, k, side, d, 0, S.box[t0][1] - S.box[t0][0] + 1,
                           t1 >= 0 ? S.box[t1][1] - S.box[t1][0] + 1 : 1};
        if (rd == my_rank) sendp[rr].push_back(sg);
        if (rr == my_rank) recvp[rd].push_back(sg);
      }
    }
  }
  long long so = 0, ro = 0;
  for (int r = 0; r < nranks; ++r) {
    for (auto sg : sendp[r]) {
      sg.off = so;
      so += (long long)sg.ext0 * sg.ext1;
      send_counts[r] += (long long)sg.ext0 * sg.ext1;
      p->send_segs.push_back(sg);
    }
    for (auto sg : recvp[r]) {
      sg.off = ro;
      ro += (long long)sg.ext0 * sg.ext1;
      recv_counts[r] += (long long)sg.ext0 * sg.ext1;
      p->recv_segs.push_back(sg);
    }
  }
  p->exch_ready = true;
  return DDPMA_OK;
}

extern "C" ddpma_status ddpma_pack_traces(ddpma_plan* p, double* send_dev) {
  CK(p, cudaSetDevice(p->device));
  std::vector<FaceJob> jobs;
  int nnodes = 0;
  for (auto& sg : p->send_segs) {
    const int dl = p->local_of[sg.donor_gid];
    if (dl < 0) continue;
    const ddpma_subdomain& R = p->subs[sg.recv_gid];
    const ddpma_subdomain& D = p->subs[sg.donor_gid];
    const SubGeo& gd = p->geo[dl];
    int t0, t1;
    tang_axes(p->dim, sg.axis, &t0, &t1);
    FaceJob J{};
    long long off = gd.off + (long long)(R.box[sg.axis][sg.side] - D.box[sg.axis][0]) * axis_stride(gd, p->dim, sg.axis);
    off += (long long)(R.box[t0][0] - D.box[t0][0]) * axis_stride(gd, p->dim, t0);
    if (t1 >= 0) off += (long long)(R.box[t1][0] - D.box[t1][0]) * axis_stride(gd, p->dim, t1);
    J.src = p->F.old + off;   // level-n snapshot (schwarz.py:251)
    J.sstr[0] = axis_stride(gd, p->dim, t0);
    J.sstr[1] = t1 >= 0 ? axis_stride(gd, p->dim, t1) : 0;
    J.dst = send_dev + sg.off;
    J.dstr[0] = 1;
    J.dstr[1] = sg.ext0;
    J.ext[0] = sg.ext0;
    J.ext[1] = sg.ext1;
    J.node_begin = nnodes;
    nnodes += sg.ext0 * sg.ext1;
    jobs.push_back(J);
  }
  ddpma_status s = run_faces(p, jobs, nnodes);
  if (s != DDPMA_OK) return s;
  return sync(p);
}

extern "C" ddpma_status ddpma_apply_traces(ddpma_plan* p, const double* recv_dev) {
  CK(p, cudaSetDevice(p->device));
  if (!p->recv_segs.empty() && recv_dev == nullptr) {
    p->err = "remote traces expected but recv buffer is NULL";
    return DDPMA_ERR_STATE;
  }
  std::vector<FaceJob> jobs;
  int nnodes = 0;
  for (int l = 0; l < (int)p->local.size(); ++l) add_apply_jobs(p, l, 0, recv_dev, jobs, nnodes);
  ddpma_status s = run_faces(p, jobs, nnodes);
  if (s != DDPMA_OK) return s;
  return sync(p);
}

extern "C" ddpma_status ddpma_advance(ddpma_plan* p) {
  CK(p, cudaSetDevice(p->device));
  std::vector<int> all(p->local.size());
  for (int l = 0; l < (int)all.size(); ++l) all[l] = l;
  p->fail = Failure{};
  ddpma_status s = advance_set(p, all);
  if (s != DDPMA_OK) return s;
  if (p->fail.set) return report_failure(p);
  return DDPMA_OK;
}

extern "C" ddpma_status ddpma_run(ddpma_plan* p, int max_windows, double tol, double* hist_res,
                                  double* hist_stats, int* windows, int* converged,
                                  double* final_residual) {
  if (!p->state_set) {
    p->err = "state not set";
    return DDPMA_ERR_STATE;
  }
  if ((int)p->local.size() != p->nsub) {
    p->err = "ddpma_run needs a plan that owns every subdomain";
    return DDPMA_ERR_STATE;
  }
  CK(p, cudaSetDevice(p->device));
  p->fail = Failure{};
  *windows = 0;
  *converged = 0;
  *final_residual = INFINITY;
  ddpma_status s;
  if (!p->density_ready) {
    if ((s = mesh_pass(p, false)) != DDPMA_OK) return s;   // init_states mesh (schwarz.py:131)
  }
  const int n = p->nsub;
  std::vector<int> all(n);
  for (int l = 0; l < n; ++l) all[l] = l;
  for (int w = 0; w < max_windows; ++w) {
    const auto t0 = std::chrono::steady_clock::now();
    const double z = window_z(p);
    if ((s = check_z(p, z)) != DDPMA_OK) return s;
    const double rmax = window_rho_max(p, z);
    if (p->cfg.transmission == DDPMA_PARALLEL) {
      if ((s = begin_window_all(p, z, rmax)) != DDPMA_OK) return s;
      std::vector<FaceJob> jobs;
      int nnodes = 0;
      for (int l = 0; l < n; ++l) add_apply_jobs(p, l, 0, nullptr, jobs, nnodes);
      if ((s = run_faces(p, jobs, nnodes)) != DDPMA_OK) return s;
      if (getenv("DDPMA_SERIAL_ADVANCE")) {
        for (int l = 0; l < n; ++l) {
          std::vector<int> one{l};
          if ((s = advance_set(p, one)) != DDPMA_OK) return s;
        }
      } else if ((s = advance_set(p, all)) != DDPMA_OK) {
        return s;
      }
      if (p->fail.set) return report_failure(p);
    } else {                       // alternating_sweep (schwarz.py:216-233)
      p->z = z;
      p->rho_max = rmax;
      set_guard(p, rmax);
      // The sequential sweep only orders a subdomain after its face donors of
      // lower id (it reads their advanced state) and before those of higher id
      // (it reads their previous state): subdomains of one wavefront level
      // (anti-diagonals of the lattice) are independent and share one window
      // kernel launch.  Results are those of the id-ordered loop.
      int cap = -1;   // a failure at id f: only ids < f can still change the report
      for (const std::vector<int>& lev : p->alt_levels) {
        std::vector<int> set;
        for (int l : lev)
          if (cap < 0 || p->local[l] < cap) set.push_back(l);
        if (set.empty()) continue;
        if ((s = prologue(p, set, z)) != DDPMA_OK) return s;
        std::vector<FaceJob> jobs;
        int nnodes = 0;
        for (int l : set) add_apply_jobs(p, l, 1, nullptr, jobs, nnodes);
        if ((s = run_faces(p, jobs, nnodes)) != DDPMA_OK) return s;
        if ((s = advance_set(p, set)) != DDPMA_OK) return s;
        if (p->fail.set) cap = p->fail.gid;
      }
      if (p->fail.set) return report_failure(p);
    }
    if ((s = mesh_pass(p, true)) != DDPMA_OK) return s;
    double stop = p->resid[0];
    double jmn = p->jmin[0], jmx = p->jmax[0];
    for (int l = 1; l < n; ++l) {
      if (p->cfg.stop_rule == DDPMA_STOP_MIN) {
        if (p->resid[l] < stop) stop = p->resid[l];
      } else if (p->resid[l] > stop) {
        stop = p->resid[l];
      }
      if (p->jmin[l] < jmn) jmn = p->jmin[l];
      if (p->jmax[l] > jmx) jmx = p->jmax[l];
    }
    const double secs =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (hist_res)
      for (int l = 0; l < n; ++l) hist_res[(size_t)w * n + l] = p->resid[l];
    if (hist_stats) {
      hist_stats[w * 4 + 0] = stop;
      hist_stats[w * 4 + 1] = jmn;
      hist_stats[w * 4 + 2] = jmx;
      hist_stats[w * 4 + 3] = secs;
    }
    *windows = w + 1;
    *final_residual = stop;
    if (stop <= tol) {
      *converged = 1;
      break;
    }
  }
  return DDPMA_OK;
}

extern "C" ddpma_status ddpma_error_info(const ddpma_plan* p, int* subdomain, double* tau_offset,
                                         double* h, int64_t* nnodes) {
  if (!p->fail.set) return DDPMA_ERR_STATE;
  if (subdomain) *subdomain = p->fail.gid;
  if (tau_offset) *tau_offset = p->fail.t;
  if (h) *h = p->fail.h;
  if (nnodes) *nnodes = p->fail.nnodes;   // -1: emax not finite (nodes=None); else call error_nodes
  return DDPMA_OK;
}

extern "C" ddpma_status ddpma_error_nodes(ddpma_plan* p, int64_t* out, int64_t cap) {
  if (!p->fail.set || p->fail.status != DDPMA_ERR_STIFFNESS || p->fail.local < 0) {
    p->err = "no stiffness failure recorded";
    return DDPMA_ERR_STATE;
  }
  CK(p, cudaSetDevice(p->device));
  const int l = p->fail.local;
  const SubGeo& g = p->geo[l];
  ddpma_status s;
  if ((s = ensure_scratch(p, g.nodes)) != DDPMA_OK) return s;
  std::vector<Entry> ents{make_entry(p, l)};
  ents[0].s = p->fail.s;
  ents[0].yi = p->fail.yi;
  ents[0].fi = p->fail.fi;
  ents[0].h04 = p->fail.h04;
  const int nb = prefix_tiles(p, ents);
  void* d;
  if ((s = stage_put(p, ents.data(), sizeof(Entry), &d)) != DDPMA_OK) return s;
  KArgs a = base_args(p);
  a.ent = (Entry*)d;
  a.nent = 1;
  launch_ratio_mask(a, nb, p->d_scratch, p->st);
  std::vector<double> mask(g.nodes);
  CK(p, cudaMemcpyAsync(mask.data(), p->d_scratch, sizeof(double) * g.nodes,
                        cudaMemcpyDeviceToHost, p->st));
  if ((s = sync(p)) != DDPMA_OK) return s;
  int64_t cnt = 0;
  for (int64_t i = 0; i < g.nodes; ++i) {
    if (mask[i] != 0.0) {
      if (out && cnt < cap) out[cnt] = i;
      ++cnt;
    }
  }
  p->fail.nnodes = cnt;
  return cnt <= cap || out == nullptr ? DDPMA_OK : DDPMA_ERR_STATE;
}

extern "C" ddpma_status ddpma_assemble_dev(ddpma_plan* p, double* psi, double* coords,
                                           double* jac) {
  CK(p, cudaSetDevice(p->device));
  int nb;
  std::vector<Entry> ents = all_entries(p, &nb);
  void* d;
  ddpma_status s;
  if ((s = stage_put(p, ents.data(), ents.size() * sizeof(Entry), &d)) != DDPMA_OK) return s;
  KArgs a = base_args(p);
  a.ent = (Entry*)d;
  a.nent = (int)ents.size();
  launch_assemble(a, nb, psi, coords, jac, p->st);
  if ((s = check_launch(p, "assemble")) != DDPMA_OK) return s;
  return sync(p);
}

extern "C" ddpma_status ddpma_pack_owned(ddpma_plan* p, double* out_dev, int64_t* size) {
  CK(p, cudaSetDevice(p->device));
  const int nl = (int)p->local.size();
  std::vector<long long> offs(nl);
  long long tot = 0;
  for (int l = 0; l < nl; ++l) {
    const SubGeo& g = p->geo[l];
    long long on = 1;
    for (int q = 0; q < p->dim; ++q) on *= (long long)(g.ohi[q] - g.olo[q] + 1);
    offs[l] = tot;
    tot += on * (2 + p->dim);
  }
  if (size) *size = tot;
  if (!out_dev) return DDPMA_OK;
  int nb;
  std::vector<Entry> ents = all_entries(p, &nb);
  void *d, *d_offs;
  ddpma_status s;
  if ((s = stage_put(p, ents.data(), ents.size() * sizeof(Entry), &d)) != DDPMA_OK) return s;
  if ((s = stage_put(p, offs.data(), offs.size() * sizeof(long long), &d_offs)) != DDPMA_OK) return s;
  KArgs a = base_args(p);
  a.ent = (Entry*)d;
  a.nent = (int)ents.size();
  launch_pack_owned(a, nb, out_dev, (const long long*)d_offs, p->st);
  if ((s = check_launch(p, "pack_owned")) != DDPMA_OK) return s;
  return sync(p);
}

extern "C" ddpma_status ddpma_assemble_host(ddpma_plan* p, double* psi, double* coords,
                                            double* jac) {
  CK(p, cudaSetDevice(p->device));
  long long n = 1;
  for (int k = 0; k < p->dim; ++k) n *= p->grid.counts[k];
  double *dp = nullptr, *dc = nullptr, *dj = nullptr;
  if (psi) CK(p, cudaMalloc((void**)&dp, sizeof(double) * n));
  if (coords) CK(p, cudaMalloc((void**)&dc, sizeof(double) * n * p->dim));
  if (jac) CK(p, cudaMalloc((void**)&dj, sizeof(double) * n));
  ddpma_status s = ddpma_assemble_dev(p, dp, dc, dj);
  if (s == DDPMA_OK) {
    if (psi) CK(p, cudaMemcpy(psi, dp, sizeof(double) * n, cudaMemcpyDeviceToHost));
    if (coords) CK(p, cudaMemcpy(coords, dc, sizeof(double) * n * p->dim, cudaMemcpyDeviceToHost));
    if (jac) CK(p, cudaMemcpy(jac, dj, sizeof(double) * n, cudaMemcpyDeviceToHost));
  }
  cudaFree(dp);
  cudaFree(dc);
  cudaFree(dj);
  return s;
}

extern "C" ddpma_status ddpma_get_sub_psi(ddpma_plan* p, int sub_id, double* out_host) {
  const int l = local_of_checked(p, sub_id);
  if (l < 0) {
    p->err = "subdomain is not local to this plan";
    return DDPMA_ERR_STATE;
  }
  CK(p, cudaSetDevice(p->device));
  return d2h_box(p, l, p->F.y[p->ctl[l].yi], out_host);
}

extern "C" ddpma_status ddpma_overlap_gap(ddpma_plan* p, double* gap) {
  CK(p, cudaSetDevice(p->device));
  std::vector<GapJob> jobs;
  int nnodes = 0;
  const int n = (int)p->local.size();
  for (int i = 0; i < n; ++i) {
    for (int j = i + 1; j < n; ++j) {
      const ddpma_subdomain& A = p->subs[p->local[i]];
      const ddpma_subdomain& B = p->subs[p->local[j]];
      int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
      bool empty = false;
      for (int k = 0; k < p->dim; ++k) {
        lo[k] = std::max(A.box[k][0], B.box[k][0]);
        hi[k] = std::min(A.box[k][1], B.box[k][1]);
        if (lo[k] > hi[k]) empty = true;
      }
      if (empty) continue;
      const SubGeo& ga = p->geo[i];
      const SubGeo& gb = p->geo[j];
      GapJob J{};
      long long oa = ga.off, ob = gb.off;
      for (int k = 0; k < p->dim; ++k) {
        oa += (long long)(lo[k] - A.box[k][0]) * axis_stride(ga, p->dim, k);
        ob += (long long)(lo[k] - B.box[k][0]) * axis_stride(gb, p->dim, k);
      }
      J.a = p->F.y[p->ctl[i].yi] + oa;
      J.b = p->F.y[p->ctl[j].yi] + ob;
      const int q0 = 3 - p->dim;   // pad 2D to 3 axes with a unit leading axis
      for (int k = 0; k < 3; ++k) {
        if (k < q0) {
          J.ext[k] = 1;
          J.astr[k] = J.bstr[k] = 0;
        } else {
          const int ax = k - q0;
          J.ext[k] = hi[ax] - lo[ax] + 1;
          J.astr[k] = axis_stride(ga, p->dim, ax);
          J.bstr[k] = axis_stride(gb, p->dim, ax);
        }
      }
      J.node_begin = nnodes;
      nnodes += J.ext[0] * J.ext[1] * J.ext[2];
      jobs.push_back(J);
    }
  }
  *gap = 0.0;
  if (jobs.empty()) return DDPMA_OK;
  ddpma_status s;
  if ((s = ensure_scratch(p, 1)) != DDPMA_OK) return s;
  CK(p, cudaMemsetAsync(p->d_scratch, 0, sizeof(double), p->st));
  void* d;
  if ((s = stage_put(p, jobs.data(), jobs.size() * sizeof(GapJob), &d)) != DDPMA_OK) return s;
  launch_gap((GapJob*)d, (int)jobs.size(), nnodes, (unsigned long long*)p->d_scratch, p->st);
  if ((s = check_launch(p, "gap")) != DDPMA_OK) return s;
  CK(p, cudaMemcpyAsync(gap, p->d_scratch, sizeof(double), cudaMemcpyDeviceToHost, p->st));
  return sync(p);
}

// ------------------------------------------------ operator-level exports --

extern "C" ddpma_status ddpma_rhs_frozen(ddpma_plan* p, int sub_id, const double* psi,
                                         const double* rho, double rho_max, double* F_out,
                                         int* flag) {
  const int l = local_of_checked(p, sub_id);
  if (l < 0) {
    p->err = "subdomain is not local to this plan";
    return DDPMA_ERR_STATE;
  }
  CK(p, cudaSetDevice(p->device));
  Ctl& c = p->ctl[l];
  c.yi = 0;
  c.fi = 0;
  ddpma_status s;
  if ((s = h2d_box(p, l, psi, p->F.y[0])) != DDPMA_OK) return s;
  if ((s = h2d_box(p, l, rho, p->F.raw)) != DDPMA_OK) return s;
  set_guard(p, rho_max);
  std::vector<int> one{l};
  if ((s = prologue(p, one, 1.0)) != DDPMA_OK) return s;   // mr = measure*(rho/1.0)
  std::vector<Entry> ents{make_entry(p, l)};
  ents[0].mode = M_F0;
  if ((s = issue_sync(p, ents)) != DDPMA_OK) return s;
  *flag = (p->h_ring[l].flags & 1u) ? 1 : 0;
  return d2h_box(p, l, p->F.f[0], F_out);
}

extern "C" ddpma_status ddpma_integrate_window(ddpma_plan* p, int sub_id, double* y,
                                               const double* rho, double rho_max) {
  const int l = local_of_checked(p, sub_id);
  if (l < 0) {
    p->err = "subdomain is not local to this plan";
    return DDPMA_ERR_STATE;
  }
  CK(p, cudaSetDevice(p->device));
  ddpma_status s;
  if (!p->integ_ready) {   // first advance() of this integrator: no caches
    if ((s = reset_integrators(p)) != DDPMA_OK) return s;
    p->integ_ready = true;
  }
  // y into the subdomain's current buffer (the device controller's yi),
  // the frozen density into raw, measure*rho and the guard (pma.py:186-219)
  if ((s = h2d_box(p, l, y, p->F.y[p->ctl[l].yi])) != DDPMA_OK) return s;
  if ((s = h2d_box(p, l, rho, p->F.raw)) != DDPMA_OK) return s;
  set_guard(p, rho_max);
  std::vector<int> one{l};
  if ((s = prologue(p, one, 1.0)) != DDPMA_OK) return s;   // mr = measure*(rho/1.0)
  p->fail = Failure{};
  if ((s = advance_set(p, one)) != DDPMA_OK) return s;
  if (p->fail.set) return report_failure(p);
  return d2h_box(p, l, p->F.y[p->ctl[l].yi], y);
}

extern "C" ddpma_status ddpma_mesh(ddpma_plan* p, int sub_id, const double* psi, double* coords,
                                   double* jac) {
  const int l = local_of_checked(p, sub_id);
  if (l < 0) {
    p->err = "subdomain is not local to this plan";
    return DDPMA_ERR_STATE;
  }
  CK(p, cudaSetDevice(p->device));
  p->ctl[l].yi = 0;
  ddpma_status s;
  if ((s = h2d_box(p, l, psi, p->F.y[0])) != DDPMA_OK) return s;
  const SubGeo& g = p->geo[l];
  double *dc = nullptr, *dj = nullptr;
  CK(p, cudaMalloc((void**)&dc, sizeof(double) * g.nodes * p->dim));
  CK(p, cudaMalloc((void**)&dj, sizeof(double) * g.nodes));
  void* d;
  int nb;
  if ((s = do_box_entry(p, l, &d, &nb)) == DDPMA_OK) {
    KArgs a = base_args(p);
    a.ent = (Entry*)d;
    a.nent = 1;
    launch_box_mesh(a, nb, dc, dj, nullptr, p->st);
    s = check_launch(p, "box_mesh");
  }
  if (s == DDPMA_OK && coords)
    if (cudaMemcpyAsync(coords, dc, sizeof(double) * g.nodes * p->dim, cudaMemcpyDeviceToHost, p->st) != cudaSuccess) s = DDPMA_ERR_CUDA;
  if (s == DDPMA_OK && jac)
    if (cudaMemcpyAsync(jac, dj, sizeof(double) * g.nodes, cudaMemcpyDeviceToHost, p->st) != cudaSuccess) s = DDPMA_ERR_CUDA;
  if (s == DDPMA_OK) s = sync(p);
  cudaFree(dc);
  cudaFree(dj);
  return s;
}

extern "C" ddpma_status ddpma_raw_density(ddpma_plan* p, int sub_id, const double* psi,
                                          double* raw) {
  const int l = local_of_checked(p, sub_id);
  if (l < 0) {
    p->err = "subdomain is not local to this plan";
    return DDPMA_ERR_STATE;
  }
  CK(p, cudaSetDevice(p->device));
  p->ctl[l].yi = 0;
  ddpma_status s;
  if ((s = h2d_box(p, l, psi, p->F.y[0])) != DDPMA_OK) return s;
  if ((s = ensure_scratch(p, p->geo[l].nodes)) != DDPMA_OK) return s;
  void* d;
  int nb;
  if ((s = do_box_entry(p, l, &d, &nb)) != DDPMA_OK) return s;
  KArgs a = base_args(p);
  a.ent = (Entry*)d;
  a.nent = 1;
  upull_prepass(p, a, nb);
  launch_box_mesh(a, nb, nullptr, nullptr, p->d_scratch, p->st);
  if ((s = check_launch(p, "box_mesh raw")) != DDPMA_OK) return s;
  CK(p, cudaMemcpyAsync(raw, p->d_scratch, sizeof(double) * p->geo[l].nodes,
                        cudaMemcpyDeviceToHost, p->st));
  return sync(p);
}

extern "C" ddpma_status ddpma_residual(ddpma_plan* p, int sub_id, const double* a_host,
                                       const double* b_host, double* out) {
  const int l = local_of_checked(p, sub_id);
  if (l < 0) {
    p->err = "subdomain is not local to this plan";
    return DDPMA_ERR_STATE;
  }
  CK(p, cudaSetDevice(p->device));
  p->ctl[l].yi = 0;
  ddpma_status s;
  if ((s = h2d_box(p, l, a_host, p->F.y[0])) != DDPMA_OK) return s;
  if ((s = h2d_box(p, l, b_host, p->F.old)) != DDPMA_OK) return s;
  std::vector<Entry> ents{make_entry(p, l)};
  const int nb = prefix_tiles(p, ents);
  void* d;
  if ((s = stage_put(p, ents.data(), sizeof(Entry), &d)) != DDPMA_OK) return s;
  launch_res_init(p->d_res, (int)p->local.size(), p->st);
  KArgs a = base_args(p);
  a.ent = (Entry*)d;
  a.nent = 1;
  launch_mesh(a, nb, 1, p->st);
  launch_finalize((Entry*)d, 1, p->d_part2, p->d_res, 1, p->st);
  if ((s = check_launch(p, "residual")) != DDPMA_OK) return s;
  CK(p, cudaMemcpyAsync(p->h_res, p->d_res, sizeof(SubRes) * p->local.size(),
                        cudaMemcpyDeviceToHost, p->st));
  if ((s = sync(p)) != DDPMA_OK) return s;
  *out = std::sqrt(p->h_res[l].sum2);
  return DDPMA_OK;
}

// metrics kernels (kernels.cu)
namespace ddpma {
constexpr int QPN_MASS = 6;   // partial layout of k_mass / k_qfinal (kernels.cu QP_N)
void launch_quality(const KArgs& a, int nb, int mode, double norm, double* e_out, double* part,
                    double* out, void* stream, int src);
void launch_relerr(const KArgs& a, int nb, const double* dd, const double* sd, double* part,
                   double* out, void* stream);
}  // namespace ddpma

extern "C" ddpma_status ddpma_monitor_mass(const ddpma_monitor* monitor, const int* counts,
                                           int device, double* integral, double* peak,
                                           int* bad) {
  const int dim = monitor->dim;
  if (dim != 2 && dim != 3) {
    set_global_error("monitor dimension must be 2 or 3");
    return DDPMA_ERR_CONFIG;
  }
  MassArgs m{};
  m.dim = dim;
  m.nodes = 1;
  for (int k = 0; k < dim; ++k) {
    if (counts[k] < 2) {
      set_global_error("probe grid needs at least 2 nodes per axis");
      return DDPMA_ERR_CONFIG;
    }
    const double a = monitor->domain[k][0], b = monitor->domain[k][1];
    m.n[k] = counts[k];
    m.a[k] = a;
    m.step[k] = (b - a) / (double)(counts[k] - 1);   // probe_axes and the spacing (:109,119)
    m.w_in[k] = m.step[k];                           // axis_weights (quadrature.py:8-13)
    m.w_end[k] = 0.5 * m.step[k];
    m.nodes *= counts[k];
  }
  MonitorD M;
  fill_monitor(monitor, dim, M);
  for (int k = 0; k < 3; ++k) {   // fld.raw(mesh): no clamp
    M.lo[k] = -INFINITY;
    M.hi[k] = INFINITY;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    set_global_error("cudaSetDevice failed");
    return DDPMA_ERR_CUDA;
  }
  if (!sampled_ok(monitor, dim)) {
    set_global_error("sampled field needs >= 2 lattice nodes per axis and its arrays");
    return DDPMA_ERR_CONFIG;
  }
  const int nb = (int)((m.nodes + NT - 1) / NT);
  std::vector<void*> lat;
  if (upload_lattice(monitor, dim, M, lat) != cudaSuccess) {
    for (void* q : lat) cudaFree(q);
    set_global_error("CUDA error uploading the sampled lattice");
    return DDPMA_ERR_CUDA;
  }
  MonitorD* dm = nullptr;
  double *part = nullptr, *out = nullptr;
  ddpma_status s = DDPMA_OK;
  double h[6] = {0, 0, 0, 0, 0, 0};
  if (cudaMalloc((void**)&dm, sizeof(MonitorD)) != cudaSuccess ||
      cudaMalloc((void**)&part, sizeof(double) * QPN_MASS * (size_t)nb) != cudaSuccess ||
      cudaMalloc((void**)&out, sizeof(double) * 6) != cudaSuccess ||
      cudaMemcpy(dm, &M, sizeof(MonitorD), cudaMemcpyHostToDevice) != cudaSuccess) {
    s = DDPMA_ERR_CUDA;
  } else {
    launch_mass(dm, m, nb, part, out, nullptr);
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpy(h, out, sizeof(double) * 6, cudaMemcpyDeviceToHost) != cudaSuccess)
      s = DDPMA_ERR_CUDA;
  }
  cudaFree(dm);
  cudaFree(part);
  cudaFree(out);
  for (void* q : lat) cudaFree(q);
  if (s != DDPMA_OK) {
    set_global_error("CUDA error in ddpma_monitor_mass");
    return s;
  }
  *integral = h[0];
  *bad = h[1] > 0.0 ? 1 : 0;
  *peak = h[5];
  return DDPMA_OK;
}

extern "C" ddpma_status ddpma_quality(ddpma_plan* p, int sub_id, const double* psi_host,
                                      double normalizer, int sample_on_mesh, double* e_host,
                                      double* report) {
  const int l = local_of_checked(p, sub_id);
  if (l < 0) {
    p->err = "subdomain is not local to this plan";
    return DDPMA_ERR_STATE;
  }
  CK(p, cudaSetDevice(p->device));
  p->ctl[l].yi = 0;
  ddpma_status s;
  if ((s = h2d_box(p, l, psi_host, p->F.y[0])) != DDPMA_OK) return s;
  const SubGeo& g = p->geo[l];
  void* d;
  int nb;
  if ((s = do_box_entry(p, l, &d, &nb)) != DDPMA_OK) return s;
  double *de = nullptr, *dpart = nullptr, *dout = nullptr;
  CK(p, cudaMalloc((void**)&de, sizeof(double) * g.nodes));
  CK(p, cudaMalloc((void**)&dpart, sizeof(double) * 6 * (size_t)nb));
  CK(p, cudaMalloc((void**)&dout, sizeof(double) * 12));
  KArgs a = base_args(p);
  a.ent = (Entry*)d;
  a.nent = 1;
  double h[6] = {0, 0, 0, 0, 0, 0};
  double norm = normalizer;
  int qsrc = 0;
  if (sample_on_mesh) {   // rho = raw / sum(w * raw * jac) (metrics.py:75-77)
    upull_prepass(p, a, nb);  // mesh_density (metrics.py:75-76)
    if (p->cfg.monitor_smooth_passes > 0) {   // its smooth_passes (monitor.py:178-179)
      launch_rawfill(a, nb, 1, p->st);
      qsrc = 1;
      for (int pass = 0; pass < p->cfg.monitor_smooth_passes; ++pass)
        for (int ax = 0; ax < p->dim; ++ax) {
          launch_smooth(a, nb, ax, qsrc, 3 - qsrc, p->st);
          qsrc = 3 - qsrc;
        }
    }
    launch_quality(a, nb, 0, 1.0, de, dpart, dout + 6, p->st, qsrc);
    if ((s = check_launch(p, "quality z")) == DDPMA_OK &&
        cudaMemcpyAsync(h, dout + 6, sizeof(double) * 6, cudaMemcpyDeviceToHost, p->st) != cudaSuccess)
      s = DDPMA_ERR_CUDA;
    if (s == DDPMA_OK) s = sync(p);
    norm = h[0];
  }
  if (s == DDPMA_OK) {
    launch_quality(a, nb, 1, norm, de, dpart, dout, p->st, qsrc);
    s = check_launch(p, "quality");
  }
  if (s == DDPMA_OK && cudaMemcpyAsync(h, dout, sizeof(double) * 6, cudaMemcpyDeviceToHost, p->st) != cudaSuccess)
    s = DDPMA_ERR_CUDA;
  if (s == DDPMA_OK && e_host &&
      cudaMemcpyAsync(e_host, de, sizeof(double) * g.nodes, cudaMemcpyDeviceToHost, p->st) != cudaSuccess)
    s = DDPMA_ERR_CUDA;
  if (s == DDPMA_OK) s = sync(p);
  cudaFree(de);
  cudaFree(dpart);
  cudaFree(dout);
  if (s != DDPMA_OK) return s;
  // QualityReport (metrics.py:24-33): e2, emax, node_mean, tangled, normaliser used
  report[0] = std::sqrt(h[0] / h[1]);
  report[1] = h[5];
  report[2] = h[2] / (double)g.nodes;
  report[3] = h[3] > 0.0 ? 1.0 : 0.0;
  report[4] = norm;
  return DDPMA_OK;
}

extern "C" ddpma_status ddpma_relative_errors(ddpma_plan* p, int sub_id, const double* dd_host,
                                              const double* sd_host, double* out) {
  const int l = local_of_checked(p, sub_id);
  if (l < 0) {
    p->err = "subdomain is not local to this plan";
    return DDPMA_ERR_STATE;
  }
  CK(p, cudaSetDevice(p->device));
  const SubGeo& g = p->geo[l];
  void* d;
  int nb;
  ddpma_status s;
  if ((s = do_box_entry(p, l, &d, &nb)) != DDPMA_OK) return s;
  double *ddd = nullptr, *dsd = nullptr, *dpart = nullptr, *dout = nullptr;
  CK(p, cudaMalloc((void**)&ddd, sizeof(double) * g.nodes));
  CK(p, cudaMalloc((void**)&dsd, sizeof(double) * g.nodes));
  CK(p, cudaMalloc((void**)&dpart, sizeof(double) * 6 * (size_t)nb));
  CK(p, cudaMalloc((void**)&dout, sizeof(double) * 6));
  if (cudaMemcpyAsync(ddd, dd_host, sizeof(double) * g.nodes, cudaMemcpyHostToDevice, p->st) != cudaSuccess ||
      cudaMemcpyAsync(dsd, sd_host, sizeof(double) * g.nodes, cudaMemcpyHostToDevice, p->st) != cudaSuccess)
    s = DDPMA_ERR_CUDA;
  KArgs a = base_args(p);
  a.ent = (Entry*)d;
  a.nent = 1;
  double h[6] = {0, 0, 0, 0, 0, 0};
  if (s == DDPMA_OK) {
    launch_relerr(a, nb, ddd, dsd, dpart, dout, p->st);
    s = check_launch(p, "relative_errors");
  }
  if (s == DDPMA_OK && cudaMemcpyAsync(h, dout, sizeof(double) * 6, cudaMemcpyDeviceToHost, p->st) != cudaSuccess)
    s = DDPMA_ERR_CUDA;
  if (s == DDPMA_OK) s = sync(p);
  cudaFree(ddd);
  cudaFree(dsd);
  cudaFree(dpart);
  cudaFree(dout);
  if (s != DDPMA_OK) return s;
  // ErrorReport (metrics.py:114-117)
  out[0] = h[0] / h[1];
  out[1] = std::sqrt(h[2] / h[3]);
  out[2] = h[4] / h[5];
  return DDPMA_OK;
}

extern "C" ddpma_status ddpma_rkc_step(ddpma_plan* p, int sub_id, const double* y,
                                       const double* rho, double rho_max, double h, int s_stages,
                                       double* d_out, double* fnew_out, int* flagged,
                                       int* end_flagged) {
  if (s_stages < 2) {
    p->err = "s must be >= 2";
    return DDPMA_ERR_CONFIG;
  }
  if (local_of_checked(p, sub_id) < 0) {
    p->err = "subdomain is not local to this plan";
    return DDPMA_ERR_STATE;
  }
  int f0flag = 0;
  ddpma_status s;
  // f0 = F(y) into f[0]; y in y[0]; mr set
  std::vector<double> dummy(p->geo[p->local_of[sub_id]].nodes);
  if ((s = ddpma_rhs_frozen(p, sub_id, y, rho, rho_max, dummy.data(), &f0flag)) != DDPMA_OK) return s;
  const int l = p->local_of[sub_id];
  Ctl& c = p->ctl[l];
  c.yi = 0;
  c.fi = 0;
  c.h = h;
  c.s = s_stages;
  const RkcCoeffs& rc = coeffs(p, s_stages);
  bool stage_flag = false;
  for (int j = 2; j <= s_stages + 1; ++j) {   // integrate.py:169-177, one launch per stage
    Entry e = make_entry(p, l);
    e.s = s_stages;
    e.c = h * rc.mu1t;
    e.h04 = 0.4 * h;
    if (j <= s_stages) {
      e.mode = j == 2 ? M_STAGE2 : (j == 3 ? M_STAGE3 : M_STAGEN);
      e.j = j;
      e.mu = rc.mu[j];
      e.nu = rc.nu[j];
      e.hmut = h * rc.mut[j];
      e.hgt = h * rc.gt[j];
    } else {
      e.mode = M_FINAL;
    }
    std::vector<Entry> ents{e};
    if ((s = issue_sync(p, ents)) != DDPMA_OK) return s;
    if (j <= s_stages) stage_flag = stage_flag || (p->h_ring[l].flags & 1u);
  }
  *flagged = (stage_flag || (p->h_ring[l].flags & 3u)) ? 1 : 0;
  *end_flagged = (p->h_ring[l].flags & 2u) ? 1 : 0;
  if ((s = d2h_box(p, l, p->F.d[s_stages % 3], d_out)) != DDPMA_OK) return s;
  return d2h_box(p, l, p->F.f[1], fnew_out);
}

// ---------------------------------------------------------------- metrics --

extern "C" ddpma_status ddpma_counters(const ddpma_plan* p, int64_t* node_updates,
                                       int64_t* rhs_evals, int64_t* launches, double* algo_bytes) {
  if (node_updates) *node_updates = p->node_updates;
  if (rhs_evals) *rhs_evals = p->rhs_evals;
  if (launches) *launches = p->launches;
  if (algo_bytes) *algo_bytes = p->algo_bytes;
  return DDPMA_OK;
}

extern "C" ddpma_status ddpma_sub_evals(const ddpma_plan* p, int64_t* out, int n) {
  if (!p || (n > 0 && !out)) return DDPMA_ERR_STATE;
  const int nl = (int)p->local.size();
  for (int l = 0; l < n && l < nl; ++l) out[l] = l < (int)p->sub_evals.size() ? p->sub_evals[l] : 0;
  return DDPMA_OK;
}

extern "C" ddpma_status ddpma_set_profiling(ddpma_plan* p, int on) {
  p->prof = on != 0;
  for (int k = 0; k < NCLASS; ++k) {
    p->prof_ms[k] = 0.0;
    p->prof_bytes[k] = 0.0;
    p->prof_launches[k] = 0;
    p->prof_nodes[k] = 0;
  }
  return DDPMA_OK;
}

extern "C" ddpma_status ddpma_profile(const ddpma_plan* p, double* ms, double* bytes,
                                      int64_t* launches, int64_t* node_updates, int nclass) {
  for (int k = 0; k < nclass && k < NCLASS; ++k) {
    if (ms) ms[k] = p->prof_ms[k];
    if (bytes) bytes[k] = p->prof_bytes[k];
    if (launches) launches[k] = p->prof_launches[k];
    if (node_updates) node_updates[k] = p->prof_nodes[k];
  }
  return DDPMA_OK;
}
