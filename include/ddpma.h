/*
 * ddpma.h — C ABI of libddpma.so, the B200-native DDPMA hot path.
 *
 * The reference (`ddmesh`, pure Python) has no FFI; the seams this library
 * sits behind are its Python entry points.  Each declaration below names the
 * reference interface it replaces (paths relative to
 * /root/reference/pkg/src/ddmesh/).  The Python host mirror
 * (paper_2006_14602_b200/) binds these through ctypes with the reference's
 * own names and argument meanings; INTEGRATION.md shows that binding.
 *
 * Conventions
 *   - fp64 everywhere; arrays are C-order with the last axis fastest, exactly
 *     as the reference's numpy arrays.
 *   - "host" pointers are plain CPU memory; "dev" pointers are CUDA device
 *     memory on the plan's device.  No torch types cross this boundary.
 *   - every call returns a ddpma_status; the message of the last failure is
 *     available from ddpma_last_error(plan) (or ddpma_global_error() for
 *     plan-less calls).  Status codes map 1:1 onto the reference exceptions
 *     (errors.py:8-49).
 *   - a plan is not re-entrant; one plan per host thread.
 */
#ifndef DDPMA_H
#define DDPMA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DDPMA_OK = 0,
  DDPMA_ERR_CONFIG = 1,           /* ConfigurationError   (errors.py:18) */
  DDPMA_ERR_INVALID_MONITOR = 2,  /* InvalidMonitorError  (errors.py:26) */
  DDPMA_ERR_STIFFNESS = 3,        /* StiffnessError       (errors.py:43) */
  DDPMA_ERR_CUDA = 4,             /* DdmeshError (device failure)        */
  DDPMA_ERR_STATE = 5,            /* DdmeshError (API misuse)            */
  /* The reference's integrator lets two plain Python errors escape when the
   * spectral radius estimate is NaN / inf: int(np.ceil(nan)) and
   * int(np.ceil(inf)) in _stages_for (integrate.py:160). */
  DDPMA_ERR_VALUE = 6,            /* ValueError    */
  DDPMA_ERR_OVERFLOW = 7,         /* OverflowError */
  DDPMA_ERR_IO = 8                /* OSError (file writers)             */
} ddpma_status;

enum { DDPMA_FACE_PHYSICAL = 0, DDPMA_FACE_INTERFACE = 1 };       /* grid.py:20-21 */
enum { DDPMA_ALTERNATING = 0, DDPMA_PARALLEL = 1 };                /* schwarz.py:41 */
enum { DDPMA_STOP_MIN = 0, DDPMA_STOP_MAX = 1 };                   /* schwarz.py:42 */
enum { DDPMA_SCHEME_ADAPTIVE = 0, DDPMA_SCHEME_EULER = 1 };        /* integrate.py:46 */
enum { DDPMA_MON_UNIFORM = 0, DDPMA_MON_RING = 1, DDPMA_MON_MIXTURE = 2,
       /* arc-length monitors of the analytic test functions
        * (arc_length_monitor monitor.py:88-97, registry :223-345): u-backed */
       DDPMA_MON_BURGERS2D = 3, DDPMA_MON_SPIRAL2D = 4, DDPMA_MON_SPHERE3D = 5,
       DDPMA_MON_NINE_SPHERES3D = 6, DDPMA_MON_QUASI1D_LINEAR = 7,
       /* arc-length monitor of a SampledField (monitor.py:361-391): u and
        * grad u by multilinear interpolation of the lattice arrays */
       DDPMA_MON_SAMPLED = 8 };

/* CompGrid (grid.py:24-55). extents[k] = {a_k, b_k}; counts[k] = N_k.
 * explicit_geom = 1 describes one BoxGeometry (grid.py:261-307) instead of a
 * grid: spacing, domain measure and the face coordinates axes[k][0] /
 * axes[k][-1] are then taken verbatim (operator-level plans). */
typedef struct {
  int dim;
  int counts[3];
  double extents[3][2];
  int explicit_geom;
  double spacing[3];
  double measure;
  double face_coord[3][2];
} ddpma_grid;

/* Subdomain (grid.py:78-110).  box/owned are inclusive global index ranges;
 * face[k][side] is DDPMA_FACE_*; donor[k][side] is the donor subdomain id of
 * an interface face (the `neighbors` dict), -1 on physical faces. */
typedef struct {
  int id;
  int pos[3];
  int box[3][2];
  int owned[3][2];
  int face[3][2];
  int donor[3][2];
} ddpma_subdomain;

/* Native density descriptor: the device-evaluable form of
 * MonitorField.raw (monitor.py:31-74, density_monitor :100-104).
 *   UNIFORM : raw = constant
 *   RING    : raw = 1 + amp*exp(-sharp*|sum_k (x_k-center_k)^2 - r2|)
 *             (BASELINE ring in 2D, spherical shell in 3D)
 *   MIXTURE : raw = 1 + sum_b a_b*exp(-|x-c_b|^2 / (2 s_b^2))
 *   BURGERS2D .. QUASI1D_LINEAR : arc-length monitors sqrt(1 + |grad u|^2)
 *             of the named test function (monitor.py:88-97,223-327; `eps`
 *             is burgers2d's parameter).  They carry u (MonitorField.u_fn),
 *             so the solver's nodal density is the mesh pull-back of
 *             mesh_density (monitor.py:151-180,183-216): u sampled on the
 *             clamped mesh, logical np.gradient of u and of the coordinates,
 *             |grad_x u|^2 through the adjugate of the map Jacobian.
 *             The analytic raw (eval_clamped, normalize) is the arc length
 *             of the analytic gradient.
 * Points are clamped into `domain` first (MonitorField.clamp, :70-74). */
typedef struct {
  int kind;
  int dim;
  double domain[3][2];
  double constant;
  double center[3];
  double amp, sharp, r2;
  int nbumps;
  const double* c;   /* host, nbumps*dim, row-major */
  const double* s;   /* host, nbumps */
  const double* a;   /* host, nbumps */
  double eps;        /* burgers2d eps (> 0) */
  int u_backed;      /* arc-length kinds: 1 = MonitorField.u_fn is set (the
                        solver's density is the pull-back of u); 0 = the
                        analytic raw at the clamped mesh points (e.g. after
                        normalize(), which drops u_fn, monitor.py:147-148) */
  /* SAMPLED: lattice of lat[k] nodes per axis (host arrays, copied by the
   * library): axes[k] (ascending), values (C order, already smoothed as the
   * SampledField constructor does) and grads[k] = np.gradient(values, h_k,
   * axis=k, edge_order=2) (monitor.py:372-380). */
  int lat[3];
  const double* axes[3];
  const double* values;
  const double* grads[3];
} ddpma_monitor;

/* normalize's probe quadrature (_trapezoid_mass, monitor.py:112-120) on the
 * device: raw (unclamped) at the nodes a_k + i*((b_k-a_k)/(n_k-1)) of the
 * monitor's domain, composite trapezoid integral (quadrature.py:24-26) and
 * max.  bad = 1 when any value is non-finite or <= 0 (InvalidMonitorError). */
ddpma_status ddpma_monitor_mass(const ddpma_monitor* monitor, const int* counts,
                                int device_ordinal, double* integral, double* peak,
                                int* bad);

/* SolverConfig (schwarz.py:35-67).  workers is meaningless on the device
 * (schedule independence is by construction) and is not carried. */
typedef struct {
  double dtau;
  double tol;
  int transmission;
  int stop_rule;
  int max_windows;
  int scheme;
  int substeps;
  double rtol;
  double atol;
  int max_stages;
  double det_floor;
  /* _window_densities (schwarz.py:162-192): per-axis [1,2,1]/4 smoothing
   * passes of each box's nodal density (monitor._smooth, monitor.py:395-409)
   * and the blend weight of the previous window's density. */
  int monitor_smooth_passes;
  double monitor_relax;
} ddpma_solver_cfg;

typedef struct ddpma_plan ddpma_plan;

/* ---------------------------------------------------------------- host --- */

/* Last error of plan-less calls (decomposition, plan creation). */
const char* ddpma_global_error(void);

/* build_decomposition (grid.py:176-237, incl. _partition_axis :125-135,
 * _extend_axis :138-173, _check_decomposition :240-258).  Pure host code; no
 * GPU needed.  `out` receives prod(layout) subdomains in id order
 * (itertools.product order, last axis fastest) when cap suffices; *nsub is
 * always set on success.  Errors are DDPMA_ERR_CONFIG with the reference's
 * message. */
ddpma_status ddpma_build_decomposition(int dim, const int* counts,
                                       const int* layout, int overlap,
                                       ddpma_subdomain* out, int cap, int* nsub);

/* Wavefront levels of alternating_sweep (schwarz.py:216-233).  The sweep
 * visits subdomains in id order; subdomain i only has to follow its face
 * donors / receivers of lower id, so level[i] = 1 + max level over those (0
 * without any): subdomains of one level are mutually independent and the
 * device advances them in one window-kernel launch, levels in ascending order
 * (bitwise the id-ordered result).  Pure host code.  Returns the number of
 * levels; level[] has nsub entries. */
int ddpma_alternating_levels(int dim, const ddpma_subdomain* subs, int nsub, int* level);

/* RKC2 recurrence coefficients (integrate.py:77-106) for s stages:
 * out arrays have s+1 entries (index j as in the reference). */
ddpma_status ddpma_rkc_coeffs(int s, double* w0, double* w1, double* mu1t,
                              double* mu, double* nu, double* mut, double* gt);

/* ---------------------------------------------------------------- plan --- */

/* Create a solver plan over the decomposition `subs` (all nsub subdomains of
 * the global problem, id order).  `local_ids` lists the subdomains this plan
 * (this GPU / rank) integrates; NULL = all.  Device memory for every local
 * box is allocated here (library-owned).  Replaces init_states
 * (schwarz.py:118-134) + the per-subdomain make_integrator (:133). */
ddpma_status ddpma_plan_create(const ddpma_grid* grid,
                               const ddpma_subdomain* subs, int nsub,
                               const int* local_ids, int nlocal,
                               const ddpma_monitor* monitor,
                               const ddpma_solver_cfg* cfg, int device,
                               ddpma_plan** out);
void ddpma_plan_destroy(ddpma_plan* plan);
const char* ddpma_last_error(const ddpma_plan* plan);

/* Initial / warm-start potential (schwarz.py:118-124).  psi_global_host is
 * the global counts-shaped field, or NULL for psi0 = |xi|^2/2
 * (pma.py:61-64), which is then formed on the device.  Resets integrator
 * caches (a fresh solve). */
ddpma_status ddpma_set_state(ddpma_plan* plan, const double* psi_global_host);

/* Full window loop of solve() (schwarz.py:307-350) for a plan owning ALL
 * subdomains.  Runs up to max_windows windows (alternating or parallel per
 * the config) until the stop rule meets tol.
 *   hist_res   [max_windows*nsub]  per-window per-subdomain residuals
 *   hist_stats [max_windows*4]     stop_residual, jac_min, jac_max, seconds
 * Either may be NULL.  *windows, *converged, *final_residual as in
 * SolveResult (:93-108).  Errors: STIFFNESS (see ddpma_error_info),
 * INVALID_MONITOR. */
ddpma_status ddpma_run(ddpma_plan* plan, int max_windows, double tol,
                       double* hist_res, double* hist_stats, int* windows,
                       int* converged, double* final_residual);

/* After a STIFFNESS status: failing subdomain id (first by id, schwarz.py
 * :262-268), tau offset and h of the failure (integrate.py:245-249), and
 * the number of nodes whose error ratio exceeded 1 (-1 when emax was not
 * finite, i.e. `nodes=None`). */
ddpma_status ddpma_error_info(const ddpma_plan* plan, int* subdomain,
                              double* tau_offset, double* h, int64_t* nnodes);
/* Flat box-local indices of those nodes (np.argwhere(ratio > 1), C order). */
ddpma_status ddpma_error_nodes(ddpma_plan* plan, int64_t* out, int64_t cap);

/* _assemble (schwarz.py:271-282): owned blocks of every local subdomain into
 * global device arrays psi[counts], coords[counts..., dim], jac[counts].
 * Any pointer may be NULL.  Only the local owned blocks are written. */
ddpma_status ddpma_assemble_dev(ddpma_plan* plan, double* psi_dev,
                                double* coords_dev, double* jac_dev);
/* Same into host arrays (device assembly + one D2H per array). */
ddpma_status ddpma_assemble_host(ddpma_plan* plan, double* psi_host,
                                 double* coords_host, double* jac_host);

/* Box-shaped Psi of local subdomain `sub_id` (SolveResult.sub_psi). */
ddpma_status ddpma_get_sub_psi(ddpma_plan* plan, int sub_id, double* out_host);

/* _overlap_gap (schwarz.py:285-304) over pairs of local subdomains. */
ddpma_status ddpma_overlap_gap(ddpma_plan* plan, double* gap);

/* ------------------------------------------- per-window phases (sharded) ---
 * The multi-GPU driver (paper_2006_14602_b200/distributed.py) runs one plan
 * per rank over its local subdomains and performs the per-window exchange
 * (face traces, the transport normaliser z, rho_max, residuals) with
 * torch.distributed/NCCL between these calls.  SURVEY §8(e). */

/* Mesh + density pass on the current local states (physical_mesh
 * pma.py:222-225, mesh_density monitor.py:151-180, the owned-node transport
 * partial of schwarz.py:182-186, raw max :191, window residual :213).
 * Outputs indexed by GLOBAL subdomain id (entries of non-local ids are
 * written as 0): z_part[nsub], raw_max[nsub], res[nsub], jac_min[nsub],
 * jac_max[nsub].  res is the trapezoid L2 norm of psi - psi_level_n
 * (meaningless before the first window). */
ddpma_status ddpma_density(ddpma_plan* plan, double* z_part, double* raw_max,
                           double* res, double* jac_min, double* jac_max);

/* Freeze the window density: rho = raw/z, rho_max, guard (schwarz.py:187-191);
 * snapshots psi_level_n and forms measure*rho on the device. */
ddpma_status ddpma_begin_window(ddpma_plan* plan, double z, double rho_max);

/* Remote trace traffic of this plan given the rank of every subdomain
 * (rank_of[nsub]) and this plan's rank: element counts per peer rank. */
ddpma_status ddpma_trace_counts(ddpma_plan* plan, const int* rank_of, int nranks,
                                int my_rank, int64_t* send_counts,
                                int64_t* recv_counts);
/* Pack the level-n face lines this rank donates to remote receivers into
 * send_dev (peers in rank order, canonical face order). */
ddpma_status ddpma_pack_traces(ddpma_plan* plan, double* send_dev);
/* Write every Dirichlet trace of the local receivers (_apply_traces,
 * schwarz.py:137-159; lowest donor id wins at corners) from local
 * snapshots and from recv_dev (remote donors, same canonical order). */
ddpma_status ddpma_apply_traces(ddpma_plan* plan, const double* recv_dev);

/* Integrate one window on every local subdomain (_advance_state
 * schwarz.py:195-213 → Rkc2Integrator.advance integrate.py:180-250 or
 * EulerIntegrator.advance :63-74). */
ddpma_status ddpma_advance(ddpma_plan* plan);

/* The integrator protocol (integrate.py:253-262, make_integrator(window)
 * .advance(y, rhs_fn)) for the frozen-density PMA right-hand side that
 * schwarz._advance_state builds (schwarz.py:201-208): advance the host box
 * field `y` (in/out) of subdomain `sub_id` by one window of cfg.dtau with
 * the plan's scheme, frozen nodal density `rho_host` and guard from
 * `rho_max` (0 = no guard, pma.py:188-190).  The integrator caches (sigma,
 * step size, refresh cadence; integrate.py:118-123) persist across calls on
 * the same plan, as they persist across advance() calls of one
 * Rkc2Integrator.  Errors: STIFFNESS (ddpma_error_info), VALUE/OVERFLOW. */
ddpma_status ddpma_integrate_window(ddpma_plan* plan, int sub_id, double* y_host,
                                   const double* rho_host, double rho_max);

/* ------------------------------------------------ operator-level exports ---
 * Box-level operators on host arrays for parity tests and the public
 * operator API (pma.py).  `sub_id` selects the box geometry (face kinds,
 * coordinates) of a subdomain of the plan; arrays are box-shaped. */

/* pma_rhs_frozen (pma.py:195-219): F and the positivity flag. */
ddpma_status ddpma_rhs_frozen(ddpma_plan* plan, int sub_id, const double* psi_host,
                              const double* rho_host, double rho_max,
                              double* F_host, int* flag);
/* hessian_det_fd (pma.py:133-149) and gradient_fd (pma.py:67-84). */
ddpma_status ddpma_mesh(ddpma_plan* plan, int sub_id, const double* psi_host,
                        double* coords_host, double* jac_host);
/* mesh_density (monitor.py:151-180) on the box mesh of psi. */
ddpma_status ddpma_raw_density(ddpma_plan* plan, int sub_id, const double* psi_host,
                               double* raw_host);
/* residual (schwarz.py:111-115): trapezoid L2 norm of a - b on the box. */
ddpma_status ddpma_residual(ddpma_plan* plan, int sub_id, const double* a_host,
                            const double* b_host, double* out);
/* One RKC2 step of s stages (integrate.py:163-178) from y with f0 = F(y):
 * d, f_new and flags.  rho frozen as given. */
ddpma_status ddpma_rkc_step(ddpma_plan* plan, int sub_id, const double* y_host,
                            const double* rho_host, double rho_max, double h,
                            int s, double* d_host, double* fnew_host,
                            int* flagged, int* end_flagged);

/* metrics.quality_measure (metrics.py:57-85) of a steady potential on the
 * plan's box (a single-box plan of the grid): e_adp = |Omega_c| rho J per
 * node into e_host (box-shaped, may be NULL) and report[0..4] = {e2, emax,
 * node_mean, tangled (0/1), normaliser used}.  rho = raw(clamp(x)) /
 * normalizer (MonitorField.eval_clamped), or with sample_on_mesh = 1 the
 * transport-normalised nodal density raw / sum(w*raw*J) (mesh_density
 * without smoothing). */
ddpma_status ddpma_quality(ddpma_plan* plan, int sub_id, const double* psi_host,
                           double normalizer, int sample_on_mesh, double* e_host,
                           double* report);
/* metrics.relative_errors (metrics.py:100-118): out = {e1, e2, einf} of two
 * box-shaped fields on the plan's box. */
ddpma_status ddpma_relative_errors(ddpma_plan* plan, int sub_id, const double* psi_dd_host,
                                   const double* psi_sd_host, double* out);

/* -------------------------------------------------------------- metrics --- */

/* Counters since plan creation: node-updates (box nodes x RHS evaluations,
 * SURVEY §8(d)), RHS evaluations, kernel launches, and algorithmic bytes
 * moved by the evaluation kernels. */
ddpma_status ddpma_counters(const ddpma_plan* plan, int64_t* node_updates,
                            int64_t* rhs_evals, int64_t* launches,
                            double* algo_bytes);
/* Owned blocks of the LOCAL subdomains (ascending id) packed into one device
 * buffer for the multi-GPU gather (replaces the reference's in-process
 * _assemble copies, schwarz.py:271-282): subdomain by subdomain, its owned
 * range in C order as [psi | coords (interleaved dim) | jac].  *size
 * receives the element count; out_dev may be NULL to query it. */
ddpma_status ddpma_pack_owned(ddpma_plan* plan, double* out_dev, int64_t* size);

/* RHS evaluations per LOCAL subdomain (ascending global id) since the last
 * ddpma_set_state: the device controller's tally of Rkc2Integrator /
 * EulerIntegrator right-hand-side calls (integrate.py:163-250), i.e. the
 * adaptive decision sequence of each subdomain.  Used by the parity tests
 * and by the multi-GPU load balancer.  Writes min(n, nlocal) entries. */
ddpma_status ddpma_sub_evals(const ddpma_plan* plan, int64_t* out, int n);
/* Per-kernel-class device time (ms, CUDA events on the plan stream) when
 * profiling is enabled: class 0 = evaluation kernels (the persistent window
 * kernel), 1 = mesh/density pass, 2 = other (prologue, traces).
 * bytes/launches per class likewise. */
ddpma_status ddpma_set_profiling(ddpma_plan* plan, int on);
ddpma_status ddpma_profile(const ddpma_plan* plan, double* ms, double* bytes,
                           int64_t* launches, int64_t* node_updates, int nclass);

/* The CUDA stream all plan work runs on (cudaStream_t as void*). */
void* ddpma_stream(const ddpma_plan* plan);
/* Name of the window kernel this plan's windows launch ("k_windowP<2>",
 * "k_windowP<3>" or "k_windowD"): benchmark / profile labelling only. */
const char* ddpma_window_kernel(const ddpma_plan* plan);

/* ------------------------------------------------------ output formats ---
 * write_mesh_vtk (fileio.py:45-68): legacy-VTK structured grid, x fastest,
 * 17 significant digits, byte-identical to the reference writer.  coords is
 * the C-order [..., dim] array of a SolveResult mesh (host), jac the
 * first point scalar (named `first_scalar`: "jacobian", or the field name of
 * write_scalar_field_vtk :71-80), e_adp optional (NULL).  Rows are formatted
 * on all host threads. */
ddpma_status ddpma_write_mesh_vtk(const char* path, int dim, const int* counts,
                                  const double* coords, const double* jac,
                                  const double* e_adp, const char* title,
                                  const char* first_scalar);
/* Message of the last failed file operation on this thread. */
const char* ddpma_io_error(void);

#ifdef __cplusplus
}
#endif

#endif /* DDPMA_H */
