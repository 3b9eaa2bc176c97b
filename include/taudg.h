/*
 * taudg.h — C-ABI of the B200 (sm_100a) DGSEM / RK3 / p-multigrid / tau hot path.
 *
 * The reference (/root/reference/pkg/src/taudg) is a pure-Python package with
 * no FFI; its hot-path boundary is the duck-typed operator object
 * `DGOperator` (operators.py:83-389) plus the transfer object `OrderTransfer`
 * (multigrid.py:101-143) and the step helpers in timestep.py.  Each entry
 * point below replaces one of those calls (cited per function); the Python
 * host package paper_1806_11456_b200 keeps the reference's class and method
 * names and binds these symbols through ctypes.
 *
 * Conventions
 *  - Plain C types only.  All field pointers are DEVICE pointers to float64
 *    arrays in the plan's layout: elements in slot order (buckets ascending by
 *    (N1,N2,N3) signature, element ids ascending inside a bucket — the
 *    reference's OrderField grouping, fields.py:34-43); per element a
 *    contiguous [nv][N3+1][N2+1][N1+1] block (xi fastest).
 *  - Every call is asynchronous on the given cudaStream_t (passed as void*),
 *    returns TDG_OK or a TDG_E_* code; tdg_last_error() gives a thread-local
 *    message.  No exception crosses the ABI.  A handle is not thread-safe.
 *  - Scalar device outputs that are maxima/minima of non-negative doubles
 *    (norms, tau, dt) are combined with integer atomics on the IEEE bit
 *    pattern, so results are independent of reduction order (bit-stable);
 *    callers must initialise them (0 for maxima, +inf for minima) — the
 *    functions with a `reset` argument do it themselves.
 */
#ifndef TAUDG_H
#define TAUDG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TDG_OK 0
#define TDG_E_CONFIG 1     /* -> ConfigError      */
#define TDG_E_MESH 2       /* -> MeshError        */
#define TDG_E_CUDA 3       /* -> DeviceError      */
#define TDG_E_ALLOC 4      /* -> DeviceError      */
#define TDG_E_ARG 5        /* -> ValueError       */

#define TDG_LAW_ADVDIFF 0  /* physics.py:49-69  AdvectionDiffusion, params a,b,c,mu      */
#define TDG_LAW_BURGERS 1  /* physics.py:72-88  ViscousBurgers,     params bx,by,bz,mu   */
#define TDG_LAW_NS 2       /* PAPER.md:744-816  Navier-Stokes, params gamma,Pr,M,Re      */

#define TDG_LG 0
#define TDG_LGL 1

#define TDG_BC_DIRICHLET 0 /* ghost = given state (operators.py:152-158) */
#define TDG_BC_FREESTREAM 1
#define TDG_BC_WALL 2      /* no-slip adiabatic */
#define TDG_BC_SYMMETRY 3

typedef struct tdg_plan tdg_plan;
typedef struct tdg_transfer tdg_transfer;

/* Host description of one operator level (one OrderField on one mesh);
 * built by paper_1806_11456_b200/operators.py (the _build_groups/_build_faces
 * of operators.py:104-171).  All arrays are HOST pointers, copied by
 * tdg_plan_create. */
typedef struct {
  int32_t law;                 /* TDG_LAW_* */
  double params[8];            /* law parameters (see TDG_LAW_*), params[7] = mu_cfl */
  int32_t family;              /* TDG_LG / TDG_LGL */
  const double* tables;        /* spectral tables, spectral.device_tables() layout */
  int64_t tables_len;

  int32_t nslots;              /* number of elements */
  const int32_t* orders;       /* [nslots*3] (N1,N2,N3) per slot */
  const int32_t* elem_id;      /* [nslots] element id of each slot */
  const int64_t* node_off;     /* [nslots+1] node offset of each slot (prefix sum) */
  const int64_t* metric_off;   /* [nslots] offset (doubles) into metrics */
  const int32_t* affine;       /* [nslots] 1: metrics are 10 doubles; 0: [10][n] */
  const double* metrics;       /* J, Ja^1(xyz), Ja^2(xyz), Ja^3(xyz) */
  int64_t metrics_len;
  const double* sizes;         /* [nslots*3] directional sizes h_d (mesh.py:161-163) */

  const int64_t* side_off;     /* [nslots*6] face-node offset of each element side */
  int64_t side_nodes;          /* total own-order face nodes over all sides */
  const double* side_geo;      /* [4][nf] per side at side_off*4: sigma, n_x, n_y, n_z */

  int32_t nfaces;              /* interior faces */
  const int32_t* face_info;    /* [nfaces*12] slotL,sideL,slotR,sideR,orient,L1,L2,R1,R2,M1,M2,0 */
  const int64_t* face_geo_off; /* [nfaces] offset (doubles) into face_geo */
  const double* face_geo;      /* [4][(M1+1)(M2+1)] mortar sigma, normal (left parametrisation) */
  int64_t face_geo_len;

  /* per element side (slot*6+side): x = nonconforming-interior | is_right<<1 | orient<<2,
   * y = M1 | M2<<8 (mortar orders in the left frame), z = face index or -1,
   * w = offset (nodes) of the side's mortar-order traces when nonconforming */
  const int32_t* side_info;    /* [nslots*6*4] */
  int64_t mtr_nodes;           /* total mortar-trace nodes of nonconforming sides */
  int32_t nbfaces;             /* boundary faces */
  const int32_t* bface_info;   /* [nbfaces*4] slot, side, bc kind, 0 */
  const int64_t* ghost_off;    /* [nbfaces] offset (doubles) into ghost, [nv][nf] */
  const double* ghost;
  int64_t ghost_len;
} tdg_plan_desc;

/* DGOperator.__init__ (operators.py:86-100): upload geometry + plan, size scratch. */
int tdg_plan_create(const tdg_plan_desc* desc, tdg_plan** out);
int tdg_plan_destroy(tdg_plan* plan);
/* Total nodes and unknowns per node of the plan. */
int tdg_plan_size(const tdg_plan* plan, int64_t* nodes, int32_t* nv);

/* DGOperator.apply(Q, isolated) (operators.py:269-335): F = F(Q). */
int tdg_apply(tdg_plan* plan, const double* Q, double* F, int isolated, void* stream);

/* DGOperator.m_inv_apply (operators.py:337-342): out = F(Q)/M [+ add].
 * `add` (nullable) fuses the FAS coarse source S_c = A_c(IQ) + I r
 * (multigrid.py:326-328). */
int tdg_m_inv_apply(tdg_plan* plan, const double* Q, const double* add, double* out,
                    int isolated, void* stream);

/* DGOperator.residual / residual_norm (operators.py:344-353): R = S - F(Q)/M.
 * S nullable (zero).  R nullable (norm only).  rnorm_dev (nullable) receives
 * max|R| (reset to 0 inside the call). */
int tdg_residual(tdg_plan* plan, const double* Q, const double* S, double* R,
                 double* rnorm_dev, void* stream);

/* DGOperator.residual (operators.py:344-353) on HOST buffers, for a batch of
 * independent states: R_host[b] = S - F(Q_host[b])/M, rnorm_host[b] = max|R|.
 * The reference's residual takes and returns host arrays; this is that call
 * for nbatch states at once.  Each state is copied in, evaluated and copied
 * out through two plan-owned device staging slots on two copy streams, so the
 * host->device copy of state b+1 and the device->host copy of state b-1 overlap
 * the evaluation of state b (use page-locked host buffers for the overlap).
 * S_dev is a device field (nullable, zero) shared by the batch; rnorm_host is
 * nullable.  Ordered after prior work on `stream`; returns when every R_host
 * and rnorm_host entry is written, with `stream` ordered after the copies. */
int tdg_residual_host(tdg_plan* plan, int32_t nbatch, const double* const* Q_host,
                      const double* S_dev, double* const* R_host, double* rnorm_host,
                      void* stream);

/* DGOperator.truncation / truncation_from_avalue (operators.py:355-364) and
 * tau.recorder_for (tau.py:173-183): tau[elem_id] = max |M S_pde - F(Q)|
 * over nodes and unknowns, with F isolated or coupled.  tau_dev has
 * nslots entries indexed by element id (reset inside the call). */
int tdg_tau(tdg_plan* plan, const double* Q, const double* S_pde, double* tau_dev,
            int isolated, void* stream);

/* DGOperator.truncation_from_avalue (operators.py:355-360), coupled tau of
 * tau.recorder_for (tau.py:178): tau_dev[elem_id] = max over nodes and
 * unknowns of |M (S_pde - A)| for a given A (device field).  S nullable
 * (zero).  Every element is written (no reset needed). */
int tdg_tau_from_avalue(tdg_plan* plan, const double* A, const double* S_pde, double* tau_dev,
                        void* stream);
/* timestep.element_dt / compute_dt (timestep.py:40-80):
 * dt_slot[slot] = min_d min(C_a h_d/(s_max max(N_d,1)^2), C_nu h_d^2/(mu max(N_d,1)^4));
 * dt_min_dev (nullable) = min over elements (reset inside). */
int tdg_element_dt(tdg_plan* plan, const double* Q, double cfl_adv, double cfl_visc,
                   double* dt_slot, double* dt_min_dev, void* stream);

/* One Williamson RK3 stage (timestep.py:83-113) fused into the residual:
 *   r = S - F(Q)/M;  W = (stage ? a_k W + r : r);  Q += b_k dt W
 * dt: device pointer, a scalar (local=0) or per-slot array (local=1).
 * rnorm_dev (nullable, stage 0): max|r| (NOT reset: caller zeroes).
 * nonfinite_dev (nullable): set to 1 if any updated Q is not finite. */
int tdg_rk3_stage(tdg_plan* plan, double* Q, double* W, const double* S, int stage,
                  const double* dt, int local, double* rnorm_dev, int32_t* nonfinite_dev,
                  void* stream);

/* tdg_rk3_stage with flags.  TDG_RK_TRACES_FRESH: the caller guarantees that
   Q has not been modified since the previous evaluation on this plan (the
   next stage of an RK step, or the next sweep of a smoothing run).  On LGL
   plans without nonconforming faces every RK stage writes the own-order side
   traces of its new state in its epilogue, and a fresh stage then skips the
   trace pass.  Results are identical with or without the flag. */
#define TDG_RK_TRACES_FRESH 1
int tdg_rk3_stage_ex(tdg_plan* plan, double* Q, double* W, const double* S, int stage,
                     const double* dt, int local, double* rnorm, int32_t* nonfinite, int flags,
                     void* stream);

/* NodalField.norm_inf / element_norms_inf (fields.py:144-152):
 * max_dev (nullable) = max|X| (reset inside); elem_dev (nullable, by element id). */
int tdg_norm_inf(tdg_plan* plan, const double* X, double* max_dev, double* elem_dev,
                 void* stream);

/* NodalField.all_finite (fields.py:154-162): flag_dev = 1 if any non-finite. */
int tdg_check_finite(tdg_plan* plan, const double* X, int32_t* flag_dev, void* stream);

/* OrderTransfer (multigrid.py:101-143) between two order fields: only the
 * slot layouts matter (orders, element ids, node offsets of both fields). */
typedef struct {
  int32_t nslots;
  int32_t nv;
  const double* tables;        /* spectral.device_tables(family) */
  int64_t tables_len;
  const int32_t* fine_orders;  /* [nslots*3] */
  const int32_t* fine_elem_id; /* [nslots] */
  const int64_t* fine_node_off;   /* [nslots+1] */
  const int32_t* coarse_orders;
  const int32_t* coarse_elem_id;
  const int64_t* coarse_node_off;
} tdg_transfer_desc;
int tdg_transfer_create(const tdg_transfer_desc* desc, tdg_transfer** out);
int tdg_transfer_destroy(tdg_transfer* t);
/* coarse = I fine (L2 projection per direction). */
int tdg_restrict(const tdg_transfer* t, const double* fine, double* coarse, void* stream);
/* fine = P coarse (interpolation). */
int tdg_prolong(const tdg_transfer* t, const double* coarse, double* fine, void* stream);
/* fine += P (Qc - Qc0) — the FAS correction (multigrid.py:333-335). */
int tdg_prolong_add(const tdg_transfer* t, const double* Qc, const double* Qc0, double* fine,
                    void* stream);

/* Element metrics on the device (mesh.py:132-164), invariant
 * curl form: for nel elements with control nodes ctrl (HOST, (nel, a1, a2,
 * a3, 3) C order, ctrl_shape = {a1, a2, a3} <= 4) and (n1p, n2p, n3p) = npts
 * solution nodes per direction, writes the HOST arrays jac (nel, n1p, n2p,
 * n3p), ja (nel, 3 [i], 3 [xyz], n1p, n2p, n3p), coords (nel, n1p, n2p, n3p,
 * 3) and sizes (nel, 3).  tables: interpolation L[3][8][4] (ctrl -> nodes),
 * collocation derivative D[3][64] and weights w[3][8] per direction.
 * Synchronous (a setup call). */
int tdg_volume_metrics(int32_t nel, const int32_t* ctrl_shape, const double* ctrl, const int32_t* npts,
                       const double* tables, double* jac, double* ja, double* coords, double* sizes);
/* Lifted BR1 gradient (operators.py:224-265; debug/parity): one trace + lift
 * pass over Q (coupled or isolated) that writes the per-node gradient,
 * [3][ngv][n] per element in slot order, to dst (device). */
int tdg_gradient(tdg_plan* plan, const double* Q, int isolated, double* dst, void* stream);
/* Plan facts for tests and the bench: element work items (blocks per
 * element-kernel launch), conforming and nonconforming (mortar) interior faces. */
int tdg_plan_info(const tdg_plan* plan, int32_t* nwork, int32_t* nconf_faces, int32_t* nmortar_faces);
/* Debug/parity: copy a face scratch buffer of the last evaluation to dst
 * (device): which = 0 Q traces [nv], 1 lift surface [3 ngv], 2 viscous
 * traces (scalar laws: gradient [3 ngv]; Navier-Stokes: the side's own
 * F_v.n sigma [4]), 3 flux surface [nv]; per element side at side_off*C as
 * [C][nf] with t1 fastest.  Returns the element count in *len_out. */
int tdg_debug_copy(tdg_plan* plan, int which, double* dst, int64_t* len_out, void* stream);

/* Device-resident tuned smoothing (multigrid.py:254-301):
 * a WHILE conditional node inside a CUDA-graph stream capture.
 * tdg_loop_begin, on a capturing `stream`, appends the node and starts
 * capturing its body on the caller's idle `body_stream` (issue the body's
 * work there); tdg_loop_test appends the end-of-batch test that
 * sets the loop condition: count += 1, floor = max(1e-13 max(1, *snorm),
 * *tolf); stop if *rnorm <= floor, or (mode 0, pre-smoothing) *rnorm <
 * eta * *cmp or *cmp == 0, or (mode 1, post-smoothing) *rnorm <= *cmp; the
 * body repeats while not stopped and count < max_iter (it always runs once).
 * tdg_loop_end closes the body capture and frees the handle object. */
typedef struct tdg_loop tdg_loop;
/* A private non-blocking stream for loop bodies (created outside any capture). */
int tdg_stream_create(void** stream_out);
int tdg_stream_destroy(void* stream);
int tdg_loop_begin(void* stream, void* body_stream, tdg_loop** out);
int tdg_loop_test(tdg_loop* loop, const double* rnorm, const double* snorm, const double* tolf,
                  const double* cmp, double eta, int mode, int32_t* count, int max_iter);
int tdg_loop_end(tdg_loop* loop);
/* Per-kernel timing (process-wide): when enabled, every kernel launch made
 * through this library is bracketed by CUDA events on its own stream.
 * tdg_timing_read synchronises the recorded events, writes the summed
 * milliseconds and launch counts per kernel class (TDG_K_*, up to k entries)
 * and clears the record. */
#define TDG_K_TRACE 0
#define TDG_K_SIDE_LIFT 1
#define TDG_K_FACE_LIFT 2
#define TDG_K_VOL_LIFT 3
#define TDG_K_SIDE_FLUX 4
#define TDG_K_FACE_FLUX 5
#define TDG_K_VOL_FLUX 6
#define TDG_K_DT 7
#define TDG_K_NORM 8
#define TDG_K_TRANSFER 9
#define TDG_K_DOWN 10
#define TDG_K_UP 11
#define TDG_K_COUNT 12
int tdg_timing_enable(int on);
int tdg_timing_read(double* ms, int64_t* counts, int k);
const char* tdg_kernel_name(int kind);

const char* tdg_last_error(void);
const char* tdg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TAUDG_H */
