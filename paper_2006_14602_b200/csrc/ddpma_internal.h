// Internal types shared by the host runtime (plan.cu) and the device kernels
// (kernels.cu).  Not part of the C ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace ddpma {

// ---------------------------------------------------------------- host ----
void set_global_error(const std::string& s);
const char* global_error();

struct RkcCoeffs {
  double w0, w1, mu1t;
  std::vector<double> mu, nu, mut, gt;
};
void rkc_coeffs(int s, RkcCoeffs& out);   // integrate.py:77-106

// -------------------------------------------------------------- device ----
constexpr int TX = 32;            // tile width along the contiguous axis
constexpr int TY = 8;             // tile height along the next axis
constexpr int NT = TX * TY;       // threads per CTA
constexpr int MAXB = 64;          // max Gaussian-mixture bumps
constexpr int NCLASS = 3;         // profiling kernel classes (ddpma.h): eval, mesh/density, other
// ddpma.h status / scheme values usable in device code
constexpr int DDPMA_ERR_STIFFNESS_D = 3;
constexpr int DDPMA_ERR_VALUE_D = 6;
constexpr int DDPMA_ERR_OVERFLOW_D = 7;
constexpr int DDPMA_SCHEME_EULER_D = 1;

// Per-axis constants of the uniform global grid (grid.py:37-39) in the exact
// forms the reference's numpy expressions use.
struct AxisC {
  double h;
  double hh, ihh;        // h*h (pma.py:96) and 1/(h*h) when h is a power of 2
  double twoh, itwoh;    // 2.*h (np.gradient interior) and its reciprocal
  double ea, eb, ec;     // -1.5/h, 2./h, -0.5/h  (np.gradient low edge)
  double fa, fb, fc;     // 0.5/h, -2./h, 1.5/h   (np.gradient high edge)
  double w_in, w_end;    // trapezoid weights h, 0.5*h (quadrature.py:8-13)
  int n;                 // global node count
};

struct Prob {
  int dim;
  int pow2;              // every spacing is a power of two -> exact reciprocals
  AxisC ax[3];
  double measure;        // global |Omega_c| (grid.py:41-47)
  double floor;          // det_floor
  double guard;          // max(floor, 0.1/(measure*rho_max)) (pma.py:188-190)
  double rguard;         // RN(1/guard) for the exact det/guard (stencil.cuh saturate)
  double atol, rtol;
  double a0[3];          // extents[k][0]
};

struct MonitorD {
  int kind, nb, dim, pad;
  double lo[3], hi[3];
  double constant;
  double center[3];
  double amp, nsharp, r2;   // nsharp = -sharp
  double eps;               // burgers2d
  // sampled field (kind 8): device copies of the lattice
  int sm[3];
  const double* sax[3];
  const double* sv;
  const double* sg[3];
  double c[MAXB * 3];
  double den[MAXB];         // (2.0*s)*s
  double a[MAXB];
};

// One local subdomain box in the arena (all fields share this layout).
struct SubGeo {
  int n[3];              // box extents (2D: n[2] = 1)
  int gid;               // global subdomain id
  long long off;         // element offset of the box in every field
  int pitch;             // elements per row of the contiguous axis
  int tiles_x, tiles_y, tiles_z, ntiles;
  int plo[3], phi[3];    // 1 = physical face
  double alo[3], ahi[3]; // axes[k][0], axes[k][-1] of the box
  double halo[3], hahi[3];  // h*axes[k][0], h*axes[k][-1] (pma.py:102,109)
  int glo[3];            // global index of the box origin
  int olo[3], ohi[3];    // owned range, box-local inclusive
  long long nodes;
  int items_x, items_y, items_z, nitems;   // persistent-kernel work items
  // dataflow sweeps (persist.cu k_windowD): items are grouped in rows of
  // `ipr` consecutive items (2D: one item row; 3D: one item plane); rowprog
  // [rowoff + r] counts the completed sweep tasks of row r
  long long rowoff;
  int ipr, nrows;
};

constexpr int IR2 = 16;   // 2D work item: TX x IR2 nodes (each thread IR2/TY rows)
constexpr int IZ3 = 2;    // 3D work item: TX x TY x IZ3 nodes

// One participant (local subdomain) of a batched launch: its action (mode),
// buffers and the scalars of that action.
struct Entry {
  int sub;               // local subdomain index
  int tile_begin;        // first CTA of this entry
  int ntiles;
  int mode;              // Mode
  int yi, fi;            // current y / f buffer
  int j, s;              // stage index / stages of the step
  int vin, vout;         // POWER: v buffers (-1 = checkerboard seed)
  int pad0, pad1;
  double c;              // STAGE: h*mu1t | POWER: delta/vnorm | EULER: dtau/m
  double h04;            // FINAL: 0.4*h
  double mu, nu, hmut, hgt;   // STAGE j: mu_j, nu_j, h*mut_j, h*gt_j
};

// Per-local-subdomain results of one round (zeroed / re-initialised each round).
struct SubRes {
  unsigned long long emax;     // max error ratio (bits of a non-negative double)
  unsigned long long jmin;     // ordered key of min jac
  unsigned long long jmax;     // ordered key of max jac
  unsigned long long rawmax;   // ordered key of max raw density
  unsigned int flags;          // bit0 eval flag, bit1 end flag, bit2 non-finite ratio
  unsigned int jnan;           // jac NaN seen
  double sum;                  // finalised sum 1 (norm^2 / z partial)
  double sum2;                 // finalised sum 2 (residual^2)
};

struct Fields {
  double* y[2];
  double* f[2];
  double* d[3];
  double* mr;     // measure * rho  (rho = raw / z), frozen per window
  double* raw;    // unnormalised nodal density of the level-n mesh
  double* old;    // psi_level_n (pre-trace snapshot)
};

enum Mode {
  M_F0 = 0,        // f0 = F(y)                          (integrate.py:184)
  M_STAGE2 = 1,    // stage j=2 (d1 = h*mu1t*f0 on the fly) (:170-175)
  M_STAGE3 = 2,    // stage j=3 (d_{j-2} = d1 on the fly)
  M_STAGEN = 3,    // stage j>=4
  M_FINAL = 4,     // f_new = F(y+d_s), y_new, error ratio max (:177, :204-208)
  M_POWER = 5,     // power-iteration eval (:139-141)
  M_POWER_SEED = 6,// first power-iteration eval from the checkerboard seed
  M_EULER = 7,     // y + (dtau/m)*F(y)                  (:69-74)
  M_NORM = 8,      // sum y^2 (np.linalg.norm(y), :133)
  M_SWEEP = 9      // one whole RKC2 step: stages 2..s + final as a dataflow
                   // of (level, item) tasks (persist.cu k_windowD)
};

struct KArgs {
  Prob P;
  const SubGeo* geo;
  const Entry* ent;
  int nent;
  int j;                 // stage index
  Fields F;
  SubRes* res;
  double* part;          // per-CTA partial sums
  double* part2;
  const MonitorD* mon;
  int upull;             // 1: raw = mesh pull-back from the k_upre fields (u-backed monitor)
};

// Device-resident controller of one local subdomain: the Rkc2Integrator /
// EulerIntegrator state (integrate.py:109-250) plus the action it currently
// publishes to the persistent window kernel (persist.cu).
struct DevCtl {
  // persistent caches (integrate.py:118-123)
  int has_sigma, since, interval, has_h;
  double sigma, h_last;
  // window state
  int phase, start_flag, state_flag, rej_row;
  int flag_rej, s, yi, fi;
  int ret, sig_k, vin, vout;
  int euler_left, j, step_flag, pad0;
  double t, h, delta, vnorm, sig;
  // failure
  int fail_status, fail_nonfin, fail_s, fail_yi;
  int fail_fi, pad1, pad2, pad3;
  double fail_t, fail_h, fail_h04;
  // current action (valid for sequence number word >> 48)
  int a_mode, a_j, a_s, a_yi;
  int a_fi, a_vin, a_vout, a_ntasks;
  double a_c, a_h04, a_mu, a_nu, a_hmut, a_hgt;
  double a_h;                    // SWEEP: step size (per-level h*mut_j, h*gt_j)
  unsigned long long a_sbase;    // SWEEP: rowprog value of every row at its start
  unsigned long long sbase;      // rowprog base of the next sweep
  // per-action accumulators and synchronisation words
  unsigned int acc_flags, done;
  unsigned long long acc_emax;
  unsigned long long word;       // (seq << 48) | (ntasks << 24) | claim cursor
  long long evals;               // RHS evaluations (node-updates / box nodes)
  double bytes;                  // algorithmic bytes moved
  unsigned long long t_begin, t_done;   // %globaltimer at window begin / subdomain done
};

struct TraceRec {
  int sub, kind, s, flagged, accepted, pad;
  double h, val;   // kind 0: step (val = emax), kind 1: sigma (val = sigma)
};

// Arguments of the persistent window kernel.
struct WinArgs {
  Prob P;
  const SubGeo* geo;
  Fields F;
  DevCtl* ctl;
  const int* act;            // active local subdomains
  int nact;
  int scheme, substeps, max_stages;
  double dtau;
  const double* coef;        // RKC2 tables: coef[4*(off[s]+j)+{0..3}] = mu, nu, mut, gt
  const int* coef_off;       //   and coef[4*off[s]+0] = mu1t
  double* part;              // per-item partial sums
  const long long* poff;     // per local subdomain offset into part
  unsigned int* n_done;
  TraceRec* trace;
  unsigned int* trace_n;
  int trace_cap;
  unsigned long long* probe;   // debug: [cap][4] = publish, first claim, last done, decided
  int probe_sub, probe_cap;
  int chunk_bulk;            // items per claim while >= tail_n subdomains are active
  const int* chunk_q;        // per priority position q (parallel to act[]): items per claim of
                             // that subdomain in the bulk phase (<= chunk_bulk), or nullptr
  int chunk_tail, tail_n;    // items per claim below that (the tail's critical path)
  const void* tmap;          // 2D: CUtensorMap[nlocal][8 fields][2 boxes] (TMA tile loads), or null
  int sweep;                 // 1: RKC2 steps run as M_SWEEP dataflow actions (k_windowD)
  int proxy_fence;           // fence.proxy.async.global before TMA reads of generic writes
  unsigned long long* rowprog;   // per-row completed sweep tasks (SubGeo::rowoff)
};

// Synchronisation word of a subdomain's current action: 16-bit sequence
// number, 24-bit task count, 24-bit claim cursor.  A finished subdomain
// publishes ntasks = 0, so it is never claimable, and stray claim
// increments (claimers that scanned before the publish) stay in the cursor
// field: 2^24 - ntasks of slack.
constexpr int kWordCurBits = 24;
constexpr unsigned long long kWordCurMask = (1ull << kWordCurBits) - 1ull;
constexpr unsigned kMaxTasks = 1u << 22;   // ntasks limit (leaves >= 12M of cursor slack)

// fields addressable by the window kernel's tensor maps
enum { TF_Y0 = 0, TF_Y1, TF_F0, TF_F1, TF_D0, TF_D1, TF_D2, TF_MR, TF_N };

void launch_window(const WinArgs& a, int nblocks, void* stream);
void launch_pack_owned(const KArgs& a, int nb, double* out, const long long* offs, void* stream);
int window_blocks(int dim, int pow2);   // co-resident CTAs for the cooperative launch
bool window_dataflow(int dim);           // k_windowD (M_SWEEP actions) runs this dimension
void launch_window_begin(const WinArgs& a, void* stream);

struct FaceJob {
  double* dst;
  const double* src;
  long long dstr[2], sstr[2];   // tangential strides
  int ext[2];                   // tangential extents (ext[1] = 1 in 2D)
  int skip_lo[2], skip_hi[2];   // lower-donor faces that win the edge nodes
  int node_begin;               // first flattened face node of this job
  int pad;
};

struct GapJob {
  const double* a;
  const double* b;
  long long astr[3], bstr[3];
  int ext[3];
  int node_begin;
};

// Launchers (kernels.cu).  All asynchronous on `stream`.
void launch_eval(const KArgs& a, int nblocks, void* stream);
void launch_finalize(const Entry* ent, int nent, const double* part, SubRes* res,
                     int which, void* stream);
void launch_mesh(const KArgs& a, int nblocks, int with_residual, void* stream);
// k_mesh with the density from smoothing buffer `src` (0: evaluate) and the
// relaxation blend (schwarz.py:162-192); buffers: 1 = mr, 2 = y[1-yi].
void launch_mesh_ex(const KArgs& a, int nblocks, int with_residual, int src, double relax,
                    int blend, void* stream);
void launch_rawfill(const KArgs& a, int nblocks, int dst, void* stream);
void launch_smooth(const KArgs& a, int nblocks, int axis, int src, int dst, void* stream);
// u-backed monitors: coordinates + u(clamp(coords)) into the scratch fields
// (d[0..2], f[1]) before a pass that reads raw with a.upull = 1.
void launch_upre(const KArgs& a, int nblocks, void* stream);

// normalize's probe lattice (monitor.py:107-120).
struct MassArgs {
  int dim;
  int n[3];
  double a[3], step[3];
  double w_in[3], w_end[3];
  long long nodes;
};
void launch_mass(const MonitorD* mon, const MassArgs& m, int nblocks, double* part, double* out,
                 void* stream);
void launch_prologue(const KArgs& a, int nblocks, double z, void* stream);
void launch_res_init(SubRes* res, int n, void* stream);
void launch_faces(const FaceJob* jobs, int njobs, int nnodes, void* stream);
void launch_gap(const GapJob* jobs, int njobs, int nnodes, unsigned long long* out,
                void* stream);
void launch_psi0(const KArgs& a, int nblocks, void* stream);
void launch_scatter(const KArgs& a, int nblocks, const double* global, void* stream);
void launch_assemble(const KArgs& a, int nblocks, double* psi, double* coords,
                     double* jac, void* stream);
void launch_ratio_mask(const KArgs& a, int nblocks, double* out, void* stream);
void launch_box_mesh(const KArgs& a, int nblocks, double* coords, double* jac, double* raw,
                     void* stream);
void launch_box_copy(const KArgs& a, int nblocks, const double* src_box, double* dst,
                     int to_arena, void* stream);

}  // namespace ddpma
