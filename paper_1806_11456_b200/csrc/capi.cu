// capi.cu — C-ABI (include/taudg.h) over the sm_100a kernels.
//
// Plans own every device allocation they make; fields are caller-owned device
// buffers.  All launches go to the caller's stream; nothing here synchronises
// except tdg_plan_create / tdg_transfer_create (uploads).
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/taudg.h"
#include "common.cuh"
#include "faces.cuh"
#include "geometry.cuh"
#include "laws.cuh"
#include "transfer.cuh"
#include "volume.cuh"

using namespace tdg;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess)                                                          \
      return fail(TDG_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define LAUNCH_CHECK(what)                                                          \
  do {                                                                              \
    cudaError_t _e = cudaGetLastError();                                            \
    if (_e != cudaSuccess)                                                          \
      return fail(TDG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(_e));   \
  } while (0)

struct Allocs {
  std::vector<void*> ptrs;
  ~Allocs() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <class T>
  int upload(const T* h, size_t n, T** out) {
    *out = nullptr;
    if (n == 0) return TDG_OK;
    void* d = nullptr;
    if (cudaMalloc(&d, n * sizeof(T)) != cudaSuccess)
      return fail(TDG_E_ALLOC, "cudaMalloc failed (" + std::to_string(n * sizeof(T)) + " bytes)");
    ptrs.push_back(d);
    if (h && cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(TDG_E_CUDA, "cudaMemcpy upload failed");
    *out = static_cast<T*>(d);
    return TDG_OK;
  }
  template <class T>
  int zeros(size_t n, T** out) {
    int rc = upload<T>(nullptr, n, out);
    if (rc == TDG_OK && n) cudaMemset(*out, 0, n * sizeof(T));
    return rc;
  }
};

int law_nv(int law) { return law == TDG_LAW_NS ? 5 : 1; }
int law_ngv(int law) { return law == TDG_LAW_NS ? 4 : 1; }
// components of the viscous side traces (Law::NTR): the gradient for scalar
// laws, the side's own normal viscous flux for Navier-Stokes
int law_ntr(int law) { return law == TDG_LAW_NS ? 4 : 3; }

// ---- launch timing -------------------------------------------------------
struct TimedLaunch {
  int kind;
  cudaEvent_t a, b;
};
bool g_timing = false;
std::vector<TimedLaunch> g_launches;
std::vector<cudaEvent_t> g_event_pool;

cudaEvent_t take_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct KTimer {
  bool on;
  TimedLaunch t;
  cudaStream_t st;
  KTimer(int kind, cudaStream_t s) : on(g_timing), st(s) {
    if (on) {  // never record timing events into a CUDA-graph capture
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) on = false;
    }
    if (!on) return;
    t.kind = kind;
    t.a = take_event();
    t.b = take_event();
    cudaEventRecord(t.a, st);
  }
  ~KTimer() {
    if (!on) return;
    cudaEventRecord(t.b, st);
    g_launches.push_back(t);
  }
};

const char* const KNAMES[TDG_K_COUNT] = {"trace_q", "side_lift", "face_lift", "vol_lift", "side_flux",
                                         "face_flux", "vol_flux", "element_dt", "norm", "transfer", "mortar_face", "up_proj"};

// End-of-batch test of a tuned smoothing phase (multigrid.py:254-301), on the
// device: floor = max(1e-13 max(1, |S|), tol floor); pre-smoothing stops at
// |r| <= floor or |r| < eta |I r| (or |I r| = 0), post-smoothing at |r| <=
// floor or |r| <= the pre-smoothing norm; the loop also stops after max_iter
// batches.  Sets the enclosing WHILE node's condition.
__global__ void k_loop_test(cudaGraphConditionalHandle h, const double* rnorm, const double* snorm,
                            const double* tolf, const double* cmp, double eta, int mode, int* count,
                            int max_iter) {
  const int c = ++(*count);
  const double rn = *rnorm;
  const double fl = fmax(1e-13 * fmax(1.0, *snorm), *tolf);
  bool stop = rn <= fl;
  if (!stop) {
    const double cv = *cmp;
    stop = mode == 0 ? (rn < eta * cv || cv == 0.0) : (rn <= cv);
  }
  cudaGraphSetConditional(h, (!stop && c < max_iter) ? 1u : 0u);
}

__global__ void k_fill(double* p, double v, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

}  // namespace

struct tdg_plan {
  DevPlan d{};
  Allocs mem;
  int nv = 1, ngv = 1, ntr = 3;
  bool viscous = false;
  int64_t nodes = 0;
  std::vector<int> orders_h;      // per slot
  std::vector<int> elem_id_h;
  std::vector<long long> node_off_h;
  size_t smem_lift_own = 0;
  // Q buffer whose current contents the own-order trace array qtr holds
  // (set by evaluations; an RK stage leaves the traces of its new state only
  // when its epilogue wrote them)
  const double* traces_of = nullptr;
  bool rk_traces = false;   // LGL, no nonconforming face
  size_t smem_lift = 0, smem_flux = 0;
  int elem_threads = VOL_THREADS;   // block size of the lift / flux kernels
  int max_tot = MAXN;                // largest work item (nodes)
  int trace_threads = ELEM_THREADS;  // k_trace_q block size
  int64_t side_nodes = 0;
  int iso = -1;          // isotropic order of a single-bucket plan, else -1
  int nsm = 148;
  // host-buffer batch evaluation (tdg_residual_host): two device staging
  // slots, two copy streams, per-slot events; created on first use
  struct Staging {
    double* q[2] = {nullptr, nullptr};
    double* r[2] = {nullptr, nullptr};
    double* norm_dev = nullptr;
    double* norm_host = nullptr;   // page-locked
    int norm_cap = 0;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t in[2] = {}, done[2] = {}, out[2] = {}, start = nullptr, fin = nullptr;
    bool ready = false;
    ~Staging() {
      for (int s = 0; s < 2; ++s) {
        cudaFree(q[s]);
        cudaFree(r[s]);
        if (ready) {
          cudaEventDestroy(in[s]);
          cudaEventDestroy(done[s]);
          cudaEventDestroy(out[s]);
        }
      }
      cudaFree(norm_dev);
      cudaFreeHost(norm_host);
      if (ready) {
        cudaEventDestroy(start);
        cudaEventDestroy(fin);
        cudaStreamDestroy(h2d);
        cudaStreamDestroy(d2h);
      }
    }
  } stage;
};

// A WHILE conditional node being captured (tdg_loop_*): its body graph is
// captured on a private stream while the outer capture waits on the node.
struct tdg_loop {
  cudaGraphConditionalHandle handle{};
  cudaStream_t body = nullptr;
};

struct tdg_transfer {
  DevTransfer d{};
  Allocs mem;
  int nwork = 0;
  size_t smem = 0;
  int nv = 1;
  int iso_f = 0, iso_c = 0;   // points per direction when every element is isotropic and uniform
  bool lines = false;         // uniform pair, items contiguous on both levels: k_transfer_lines
};

namespace {

template <class K>
int allow_smem(K kernel, size_t bytes) {
  {  // dynamic + static must fit: always raise the dynamic limit to what we launch with
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(bytes));
    if (e != cudaSuccess) return fail(TDG_E_CUDA, std::string("smem attribute: ") + cudaGetErrorString(e));
  }
  return TDG_OK;
}

// compile-time isotropic order for single-bucket Navier-Stokes plans
template <int LAW, class F>
int with_nx(int iso, F&& f) {
  if (LAW == LAW_NS) {
    switch (iso) {
      case 1: return f(std::integral_constant<int, 1>());
      case 2: return f(std::integral_constant<int, 2>());
      case 3: return f(std::integral_constant<int, 3>());
      case 4: return f(std::integral_constant<int, 4>());
      case 5: return f(std::integral_constant<int, 5>());
      case 6: return f(std::integral_constant<int, 6>());
      case 7: return f(std::integral_constant<int, 7>());
      default: break;
    }
  }
  return f(std::integral_constant<int, -1>());
}

template <int LAW>
int setup_attrs(tdg_plan* p) {
  // The limit is a per-function, process-wide attribute shared by every
  // plan: set it to the MAXN-item bound, never to this plan's (smaller) need.
  const size_t ngv = p->ngv, ng = 3 * ngv, nv = p->nv, b = MAXN * sizeof(double);
  // k_vol_lift: [ngv + 9] per node, or [ngv] per node + [ntr] per face node (<= 1536 per item)
  const size_t lift = std::max<size_t>((ngv + std::max<size_t>(9, ng)) * b, ngv * b + ng * 1536 * sizeof(double)),
               own = (ngv + std::max<size_t>(9, nv)) * b + 16 + (ngv + 3) * (LIFT_FACE_NODES + 64 * 6) * sizeof(double),
               flux = 3 * nv * b;
  int rc = with_nx<LAW>(p->iso, [&](auto nx) -> int {
    constexpr int NX = decltype(nx)::value;
    int r;
    if ((r = allow_smem(k_vol_lift<LAW, NX>, lift))) return r;
    if ((r = allow_smem(k_vol_lift_own<LAW, NX>, own))) return r;
    if ((r = allow_smem(k_vol_lift_own_inl<LAW, NX>, own))) return r;
    if ((r = allow_smem(k_vol_flux<LAW, MODE_A, NX>, flux))) return r;
    if ((r = allow_smem(k_vol_flux<LAW, MODE_R, NX>, flux))) return r;
    if ((r = allow_smem(k_vol_flux<LAW, MODE_RK, NX>, flux))) return r;
    return TDG_OK;
  });
  if (rc) return rc;
  // cold modes use runtime orders only
  if ((rc = allow_smem(k_vol_flux<LAW, MODE_F, -1>, flux))) return rc;
  if ((rc = allow_smem(k_vol_flux<LAW, MODE_TAU, -1>, flux))) return rc;
  return TDG_OK;
}

// trace -> lift (if viscous) -> face fluxes; leaves fsurf ready for k_vol_flux.
// ``d`` is the plan's device view (tdg_gradient passes a copy that stores the
// per-node gradient); lift_only stops after the lift.
template <int LAW>
int run_surface(tdg_plan* p, const DevPlan& d, const double* Q, int isolated, cudaStream_t st,
                bool traces_fresh = false, bool lift_only = false) {
  using L = Law<LAW>;
  if (d.nwork == 0) return TDG_OK;
  const int coupled = isolated ? 0 : 1;
  if (!traces_fresh) {
    KTimer kt(TDG_K_TRACE, st);
    // mortar plans, coupled evaluation: the item's Q span is staged in shared memory
    const size_t smem_trace = (coupled && d.nmface != 0)
                                  ? (static_cast<size_t>(L::NV) * p->max_tot + 2) * sizeof(double) : 0;
    k_trace_q<L::NV><<<d.nwork, p->trace_threads, smem_trace, st>>>(d, Q, coupled);
    LAUNCH_CHECK("k_trace_q");
  }
  p->traces_of = Q;

  auto sides = [&](bool flux) -> int {
    const int4* items = isolated ? d.side_iso : d.side_bnd;
    const int n = isolated ? d.nside_iso : d.nside_bnd;
    if (n > 0) {
      const int grid = (n + SIDES_PER_BLOCK - 1) / SIDES_PER_BLOCK;
      KTimer kt(flux ? TDG_K_SIDE_FLUX : TDG_K_SIDE_LIFT, st);
      if (flux)
        k_side<LAW, true><<<grid, SIDE_THREADS, 0, st>>>(d, items, n);
      else
        k_side<LAW, false><<<grid, SIDE_THREADS, 0, st>>>(d, items, n);
      LAUNCH_CHECK("k_side");
    }
    if (!isolated && d.nfaces > 0) {
      if (d.ncface > 0) {
        KTimer kt(flux ? TDG_K_FACE_FLUX : TDG_K_FACE_LIFT, st);
        if (flux)
          k_face<LAW, true><<<(d.ncface + d.face_pack - 1) / d.face_pack, d.face_threads, 0, st>>>(d);
        else
          k_face<LAW, false><<<(d.ncface + d.face_pack - 1) / d.face_pack, d.face_threads, 0, st>>>(d);
        LAUNCH_CHECK("k_face");
      }
      if (d.nmface > 0) {
        // nonconforming faces: pointwise values and both down-projections in one warp
        // (timer class TDG_K_DOWN = "mortar_face")
        KTimer kd(TDG_K_DOWN, st);
        if (flux)
          k_mortar<LAW, true><<<(d.nmface + MORTAR_WARPS - 1) / MORTAR_WARPS, 32 * MORTAR_WARPS, 0, st>>>(d);
        else
          k_mortar<LAW, false><<<(d.nmface + MORTAR_WARPS - 1) / MORTAR_WARPS, 32 * MORTAR_WARPS, 0, st>>>(d);
        LAUNCH_CHECK("k_mortar");
      }
    }
    return TDG_OK;
  };
  int rc;
  if (p->viscous) {
    if ((rc = sides(false))) return rc;
    {
      KTimer kt(TDG_K_VOL_LIFT, st);
      // LGL and every evaluated side on own-order traces: direct trace writes
      const bool own = d.family == TDG_LGL && (isolated || d.nmface == 0);
      with_nx<LAW>(p->iso, [&](auto nx) -> int {
        constexpr int NX = decltype(nx)::value;
        if (own && d.lift_packed)
          k_vol_lift_own<LAW, NX><<<d.nwork, p->elem_threads, p->smem_lift_own, st>>>(d, Q, coupled);
        else if (own)
          k_vol_lift_own_inl<LAW, NX><<<d.nwork, p->elem_threads, p->smem_lift_own, st>>>(d, Q, coupled);
        else
          k_vol_lift<LAW, NX><<<d.nwork, p->elem_threads, p->smem_lift, st>>>(d, Q, coupled);
        return 0;
      });
    }
    LAUNCH_CHECK("k_vol_lift");
  }
  if (lift_only) return TDG_OK;
  return sides(true);
}

template <int LAW, int MODE>
int run_eval(tdg_plan* p, const double* Q, int isolated, const FluxArgs& a0, cudaStream_t st,
             bool traces_fresh = false) {
  int rc = run_surface<LAW>(p, p->d, Q, isolated, st, traces_fresh);
  if (rc) return rc;
  if (p->d.nwork == 0) return TDG_OK;
  FluxArgs a = a0;
  a.coupled = isolated ? 0 : 1;
  {
    KTimer kt(TDG_K_VOL_FLUX, st);
    constexpr bool hot = MODE == MODE_R || MODE == MODE_RK || MODE == MODE_A;
    if (hot) {
      with_nx<LAW>(p->iso, [&](auto nx) -> int {
        k_vol_flux<LAW, MODE, hot ? decltype(nx)::value : -1><<<p->d.nwork, p->elem_threads, p->smem_flux, st>>>(
            p->d, Q, a);
        return 0;
      });
    } else {
      k_vol_flux<LAW, MODE, -1><<<p->d.nwork, p->elem_threads, p->smem_flux, st>>>(p->d, Q, a);
    }
  }
  LAUNCH_CHECK("k_vol_flux");
  // an RK stage rewrote Q: qtr now holds its traces only if the epilogue wrote them
  if (MODE == MODE_RK) p->traces_of = a.traces ? Q : nullptr;
  return TDG_OK;
}

template <int MODE>
int dispatch_eval(tdg_plan* p, const double* Q, int isolated, const FluxArgs& a, cudaStream_t st,
                  bool traces_fresh = false) {
  switch (p->d.law) {
    case TDG_LAW_ADVDIFF: return run_eval<LAW_ADVDIFF, MODE>(p, Q, isolated, a, st, traces_fresh);
    case TDG_LAW_BURGERS: return run_eval<LAW_BURGERS, MODE>(p, Q, isolated, a, st, traces_fresh);
    case TDG_LAW_NS: return run_eval<LAW_NS, MODE>(p, Q, isolated, a, st, traces_fresh);
  }
  return fail(TDG_E_CONFIG, "unknown law");
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Transfer launch: compile-time sizes for the isotropic neighbour-order level
// pairs of a uniform p-multigrid (5 components), runtime sizes otherwise.
template <int MODE, int NS, int ND>
bool launch_transfer_iso(const tdg_transfer* t, int ns, int nd, const double* in, const double* in2,
                         double* out, cudaStream_t st) {
  if (ns != NS || nd != ND) return false;
  if (t->lines)
    k_transfer_lines<MODE, 5, NS, ND><<<t->nwork, transfer_lines_threads<NS, ND>(), t->smem, st>>>(t->d, in, in2,
                                                                                                  out);
  else
    k_transfer<MODE, 5, NS, ND><<<t->nwork, ELEM_THREADS, t->smem, st>>>(t->d, in, in2, out);
  return true;
}

template <int NS, int ND>
int allow_lines_pair(size_t b) {
  int rc;
  if ((rc = allow_smem(k_transfer_lines<TR_RESTRICT, 5, NS, ND>, b))) return rc;
  if ((rc = allow_smem(k_transfer_lines<TR_PROLONG, 5, NS, ND>, b))) return rc;
  return allow_smem(k_transfer_lines<TR_PROLONG_ADD, 5, NS, ND>, b);
}

int allow_lines_smem(size_t b) {
  int rc;
  if ((rc = allow_lines_pair<8, 7>(b)) || (rc = allow_lines_pair<7, 8>(b)) || (rc = allow_lines_pair<7, 6>(b)) ||
      (rc = allow_lines_pair<6, 7>(b)) || (rc = allow_lines_pair<6, 5>(b)) || (rc = allow_lines_pair<5, 6>(b)) ||
      (rc = allow_lines_pair<5, 4>(b)) || (rc = allow_lines_pair<4, 5>(b)) || (rc = allow_lines_pair<4, 3>(b)) ||
      (rc = allow_lines_pair<3, 4>(b)) || (rc = allow_lines_pair<3, 2>(b)) || (rc = allow_lines_pair<2, 3>(b)))
    return rc;
  return TDG_OK;
}

template <int MODE>
int launch_transfer(const tdg_transfer* t, const double* in, const double* in2, double* out,
                    cudaStream_t st) {
  const int ns = MODE == TR_RESTRICT ? t->iso_f : t->iso_c;
  const int nd = MODE == TR_RESTRICT ? t->iso_c : t->iso_f;
  bool done = false;
  if (t->nv == 5 && ns > 0 && nd > 0) {
    done = launch_transfer_iso<MODE, 8, 7>(t, ns, nd, in, in2, out, st) ||
           launch_transfer_iso<MODE, 7, 8>(t, ns, nd, in, in2, out, st) ||
           launch_transfer_iso<MODE, 7, 6>(t, ns, nd, in, in2, out, st) ||
           launch_transfer_iso<MODE, 6, 7>(t, ns, nd, in, in2, out, st) ||
           launch_transfer_iso<MODE, 6, 5>(t, ns, nd, in, in2, out, st) ||
           launch_transfer_iso<MODE, 5, 6>(t, ns, nd, in, in2, out, st) ||
           launch_transfer_iso<MODE, 5, 4>(t, ns, nd, in, in2, out, st) ||
           launch_transfer_iso<MODE, 4, 5>(t, ns, nd, in, in2, out, st) ||
           launch_transfer_iso<MODE, 4, 3>(t, ns, nd, in, in2, out, st) ||
           launch_transfer_iso<MODE, 3, 4>(t, ns, nd, in, in2, out, st) ||
           launch_transfer_iso<MODE, 3, 2>(t, ns, nd, in, in2, out, st) ||
           launch_transfer_iso<MODE, 2, 3>(t, ns, nd, in, in2, out, st);
  }
  if (!done) k_transfer<MODE><<<t->nwork, ELEM_THREADS, t->smem, st>>>(t->d, in, in2, out);
  return TDG_OK;
}

}  // namespace

extern "C" {

const char* tdg_last_error(void) { return g_err.c_str(); }

int tdg_timing_enable(int on) {
  g_timing = on != 0;
  return TDG_OK;
}

int tdg_timing_read(double* ms, int64_t* counts, int k) {
  std::vector<double> acc(TDG_K_COUNT, 0.0);
  std::vector<int64_t> cnt(TDG_K_COUNT, 0);
  for (auto& t : g_launches) {
    cudaError_t e = cudaEventSynchronize(t.b);
    if (e != cudaSuccess) return fail(TDG_E_CUDA, std::string("timing: ") + cudaGetErrorString(e));
    float x = 0.f;
    cudaEventElapsedTime(&x, t.a, t.b);
    acc[t.kind] += x;
    cnt[t.kind] += 1;
    g_event_pool.push_back(t.a);
    g_event_pool.push_back(t.b);
  }
  g_launches.clear();
  for (int i = 0; i < k && i < TDG_K_COUNT; ++i) {
    if (ms) ms[i] = acc[i];
    if (counts) counts[i] = cnt[i];
  }
  return TDG_OK;
}

const char* tdg_kernel_name(int kind) { return (kind >= 0 && kind < TDG_K_COUNT) ? KNAMES[kind] : "?"; }
const char* tdg_version(void) { return "taudg-b200 0.1.0 sm_100a"; }

int tdg_plan_create(const tdg_plan_desc* desc, tdg_plan** out) {
  if (!desc || !out) return fail(TDG_E_ARG, "null argument");
  *out = nullptr;
  if (desc->law < 0 || desc->law > 2) return fail(TDG_E_CONFIG, "unknown law id");
  if (desc->tables_len != TABLES_LEN) return fail(TDG_E_CONFIG, "spectral table length mismatch");
  if (desc->nslots < 0) return fail(TDG_E_ARG, "negative slot count");
  // packed face / down-projection descriptors hold node offsets as int32
  if (desc->side_nodes > INT32_MAX || desc->mtr_nodes > INT32_MAX ||
      desc->face_geo_len > INT32_MAX)
    return fail(TDG_E_CONFIG, "plan too large: side / mortar offsets exceed int32");
  auto* p = new tdg_plan();
  p->nv = law_nv(desc->law);
  p->ngv = law_ngv(desc->law);
  p->ntr = law_ntr(desc->law);
  p->viscous = desc->params[3] > 0.0;
  const int ns = desc->nslots;
  p->orders_h.assign(desc->orders, desc->orders + 3 * ns);
  p->elem_id_h.assign(desc->elem_id, desc->elem_id + ns);
  p->node_off_h.assign(desc->node_off, desc->node_off + ns + 1);
  p->nodes = p->node_off_h[ns];
  for (int s = 0; s < ns; ++s)
    for (int d = 0; d < 3; ++d) {
      const int o = p->orders_h[3 * s + d];
      if (o < 0 || o > 7) {
        delete p;
        return fail(TDG_E_CONFIG, "polynomial orders must lie in 0..7 on the device path");
      }
      if (desc->family == TDG_LGL && o < 1) {
        delete p;
        return fail(TDG_E_CONFIG, "Gauss-Lobatto nodes need orders >= 1");
      }
    }
  DevPlan& d = p->d;
  d.law = desc->law;
  d.family = desc->family;
  std::memcpy(d.prm, desc->params, sizeof(d.prm));
  if (desc->law == TDG_LAW_NS && d.prm[3] > 0.0) {
    // uniform constants of the viscous flux, formed once (laws.cuh visc_dir)
    d.prm[4] = 1.0 / d.prm[3];
    d.prm[5] = 1.0 / ((d.prm[0] - 1.0) * d.prm[1] * d.prm[2] * d.prm[2]);
  }
  d.nslots = ns;
  d.nfaces = desc->nfaces;
  d.nbfaces = desc->nbfaces;
  int rc = TDG_OK;
  double* tables;
  int *orders, *elem_id, *affine, *face_info, *bface_info;
  long long *node_off, *metric_off, *side_off, *face_geo_off, *ghost_off;
  double *metrics, *sizes, *side_geo, *face_geo, *ghost;
#define UP(ptr, src, n) if (!rc) rc = p->mem.upload(src, (size_t)(n), &ptr)
  UP(tables, desc->tables, desc->tables_len);
  UP(orders, desc->orders, 3 * ns);
  UP(elem_id, desc->elem_id, ns);
  UP(node_off, reinterpret_cast<const long long*>(desc->node_off), ns + 1);
  UP(metric_off, reinterpret_cast<const long long*>(desc->metric_off), ns);
  UP(affine, desc->affine, ns);
  UP(metrics, desc->metrics, desc->metrics_len);
  UP(sizes, desc->sizes, 3 * ns);
  UP(side_off, reinterpret_cast<const long long*>(desc->side_off), 6 * ns);
  UP(side_geo, desc->side_geo, 4 * desc->side_nodes);
  UP(face_info, desc->face_info, 12 * desc->nfaces);
  UP(face_geo_off, reinterpret_cast<const long long*>(desc->face_geo_off), desc->nfaces);
  UP(face_geo, desc->face_geo, desc->face_geo_len);
  int* side_info_i;
  UP(side_info_i, desc->side_info, 4 * 6 * ns);
  {
    // packed per-face descriptors and the conforming / nonconforming face lists
    // (nonconforming faces are projected in registers by k_mortar)
    std::vector<int4> fdv(2 * static_cast<size_t>(desc->nfaces));
    std::vector<int4> snb(6 * static_cast<size_t>(ns), make_int4(-1, 0, 0, 0));
    std::vector<int> cfv, mfv;
    for (int f = 0; f < desc->nfaces; ++f) {
      const int* fi = desc->face_info + 12 * f;
      const int M1 = fi[9], M2 = fi[10];
      const bool conf = fi[5] == M1 && fi[6] == M2 && fi[7] == M1 && fi[8] == M2;
      const int kl = 6 * fi[0] + fi[1], kr = 6 * fi[2] + fi[3];
      const long long tl = conf ? desc->side_off[kl] : desc->side_info[4 * kl + 3];
      const long long tr = conf ? desc->side_off[kr] : desc->side_info[4 * kr + 3];
      // uniform face geometry (every node's sigma and normal identical, e.g.
      // a face of an affine element): the kernels read node 0's values
      bool geo_const = true;
      {
        const int nmf = (M1 + 1) * (M2 + 1);
        const double* gg = desc->face_geo + desc->face_geo_off[f];
        for (int c = 0; c < 4 && geo_const; ++c)
          for (int k = 1; k < nmf && geo_const; ++k) geo_const = gg[c * nmf + k] == gg[c * nmf];
      }
      fdv[2 * f] = make_int4(static_cast<int>(tl), static_cast<int>(tr),
                             M1 | M2 << 3 | fi[4] << 6 | (conf ? 1 : 0) << 9 | (geo_const ? 1 : 0) << 10,
                             static_cast<int>(desc->face_geo_off[f]));
      fdv[2 * f + 1] = make_int4(0, static_cast<int>(desc->side_off[kl]), static_cast<int>(desc->side_off[kr]),
                                 fi[5] | fi[6] << 3 | fi[7] << 6 | fi[8] << 9);
      (conf ? cfv : mfv).push_back(f);
      if (conf) {
        const int code = M1 | M2 << 3 | fi[4] << 6;
        const int go = static_cast<int>(desc->face_geo_off[f]);
        snb[kl] = make_int4(static_cast<int>(tl), go, code | (geo_const ? 1 : 0) << 10, 0);
        snb[kr] = make_int4(static_cast<int>(tl), go, code | 1 << 9 | (geo_const ? 1 : 0) << 10, 0);
      }
    }
    int4* snb_d = nullptr;
    if (!rc && ns > 0) rc = p->mem.upload(snb.data(), snb.size(), &snb_d);
    d.side_nb = snb_d;
    int *cf_d = nullptr, *mf_d = nullptr;
    if (!rc && !cfv.empty()) rc = p->mem.upload(cfv.data(), cfv.size(), &cf_d);
    if (!rc && !mfv.empty()) rc = p->mem.upload(mfv.data(), mfv.size(), &mf_d);
    d.ncface = static_cast<int>(cfv.size());
    d.nmface = static_cast<int>(mfv.size());
    {
      // uniform small conforming faces: several per k_face block
      int nmu = -1;
      for (int f : cfv) {
        const int* fi = desc->face_info + 12 * f;
        const int nm = (fi[9] + 1) * (fi[10] + 1);
        if (nmu < 0) nmu = nm;
        if (nm != nmu) { nmu = 0; break; }
      }
      d.face_nm = nmu > 0 ? nmu : 0;
      // measured: 128-thread blocks pay off when they hold >= 3 faces (N <= 5);
      // 49- and 64-node faces run best one per 64-thread block
      d.face_pack = nmu > 0 ? (3 * nmu <= FACE_THREADS_MAX ? FACE_THREADS_MAX : FACE_THREADS) / nmu : 1;
      d.face_threads = nmu > 0 ? (d.face_pack * nmu + 31) / 32 * 32 : FACE_THREADS;
    }
    d.cface = cf_d;
    d.mface = mf_d;
    int4* fd_d = nullptr;
    if (!rc && !fdv.empty()) rc = p->mem.upload(fdv.data(), fdv.size(), &fd_d);
    d.fdesc = fd_d;
  }
  UP(bface_info, desc->bface_info, 4 * desc->nbfaces);
  UP(ghost_off, reinterpret_cast<const long long*>(desc->ghost_off), desc->nbfaces);
  UP(ghost, desc->ghost, desc->ghost_len);
#undef UP
  if (rc) {
    delete p;
    return rc;
  }
  d.tables = tables;
  d.orders = orders;
  d.elem_id = elem_id;
  d.node_off = node_off;
  d.metric_off = metric_off;
  d.affine = affine;
  d.metrics = metrics;
  d.sizes = sizes;
  d.side_off = side_off;
  d.side_geo = side_geo;
  d.face_info = face_info;
  d.face_geo_off = face_geo_off;
  d.face_geo = face_geo;
  d.bface_info = bface_info;
  d.ghost_off = ghost_off;
  d.ghost = ghost;
  d.side_info = reinterpret_cast<const int4*>(side_info_i);

  {
    int iso = ns > 0 ? p->orders_h[0] : -1;
    for (int s = 0; s < ns && iso >= 0; ++s)
      for (int dd = 0; dd < 3; ++dd)
        if (p->orders_h[3 * s + dd] != iso) iso = -1;
    p->iso = iso;
  }
  // element work items: runs of identical orders, <= MAXN nodes; small
  // plans get smaller items so that every SM receives work (>= 2 per SM)
  int nsm_attr = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&nsm_attr, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      nsm_attr = 148;
  }
  const long long item_nodes =
      std::max<long long>(1, std::min<long long>(MAXN, p->nodes / (2LL * nsm_attr)));
  // g* form of the conforming-face lift (plans served by k_vol_lift_own);
  // TDG_GSTAR=0 restores the per-side g*·n σ arrays
  {
    const char* gsv = getenv("TDG_GSTAR");
    d.gstar = (desc->family == TDG_LGL && p->viscous && d.ncface > 0 && d.nmface == 0 &&
               !(gsv && gsv[0] == '0')) ? 1 : 0;
  }
  // own-order lift variant: packed face-node passes on affine plans and on
  // curved plans of order >= 4 (measured: config 4 V-cycle 60.2 ms packed at
  // every level, 62.5 ms in-loop; config 5, curved N = 3: 26.2 ms in-loop,
  // 28.1 ms packed); TDG_LIFT_PACKED_MIN overrides the smallest order
  {
    bool any_curved = false;
    for (int s = 0; s < ns && !any_curved; ++s) any_curved = desc->affine[s] == 0;
    const char* pm = getenv("TDG_LIFT_PACKED_MIN");
    const int pmin = pm ? atoi(pm) : (any_curved ? 4 : 1);
    int omin = 99;
    for (int s = 0; s < ns; ++s)
      for (int dd = 0; dd < 3; ++dd) omin = std::min(omin, p->orders_h[3 * s + dd]);
    d.lift_packed = (ns > 0 && omin >= pmin) ? 1 : 0;
  }
  int lift_face_nodes = LIFT_FACE_NODES;
  if (const char* v = getenv("TDG_LIFT_FACE_NODES")) lift_face_nodes = std::min(LIFT_FACE_NODES, std::max(24, atoi(v)));
  std::vector<int2> work;
  for (int s = 0; s < ns;) {
    const int* o = &p->orders_h[3 * s];
    const int n = (o[0] + 1) * (o[1] + 1) * (o[2] + 1);
    // <= MAX_ITEM_ELEMS elements: per-element reductions (tau, dt, norms)
    // use fixed shared-memory arrays of that size
    int cap = std::min(MAX_ITEM_ELEMS, std::max(1, static_cast<int>(item_nodes / n)));
    // g* form: the lift stages g* and n sigma of the item's face nodes in
    // shared memory (k_vol_lift_own pass 1); small elements have more face
    // nodes than volume nodes, so the item is also capped by its face nodes
    if (d.gstar && d.lift_packed) {
      const int per_e = 2 * ((o[1] + 1) * (o[2] + 1) + (o[0] + 1) * (o[2] + 1) + (o[0] + 1) * (o[1] + 1));
      cap = std::max(1, std::min(cap, lift_face_nodes / per_e));
    }
    int e = s;
    while (e < ns && e - s < cap && p->orders_h[3 * e] == o[0] && p->orders_h[3 * e + 1] == o[1] &&
           p->orders_h[3 * e + 2] == o[2])
      ++e;
    work.push_back(make_int2(s, e - s));
    s = e;
  }
  // element-kernel block size: enough threads for the largest item at NPT
  // nodes per thread (a 343-node N=6 item runs 192 threads, not 256)
  long long max_tot = 1;
  for (const int2& w : work) {
    const int* o = &p->orders_h[3 * w.x];
    max_tot = std::max<long long>(max_tot, static_cast<long long>(w.y) * (o[0] + 1) * (o[1] + 1) * (o[2] + 1));
  }
  p->elem_threads = static_cast<int>(std::min<long long>(
      VOL_THREADS, std::max<long long>(128, (max_tot + NPT * 32 - 1) / (NPT * 32) * 32)));
  p->max_tot = static_cast<int>(max_tot);
  std::vector<int4> iso, bnd;
  iso.reserve(6 * ns);
  for (int s = 0; s < ns; ++s)
    for (int side = 0; side < 6; ++side) iso.push_back(make_int4(s, side, -1, -1));
  for (int f = 0; f < desc->nbfaces; ++f) {
    const int* b = desc->bface_info + 4 * f;
    const long long go = desc->ghost_off[f];
    bnd.push_back(make_int4(b[0], b[1], b[2], static_cast<int>(go)));
  }
  // per-side flags: boundary kind + 1 (bits 0-3), uniform own-order geometry (bit 4)
  std::vector<int> sflags(6 * static_cast<size_t>(ns), 0);
  for (int f = 0; f < desc->nbfaces; ++f) {
    const int* b = desc->bface_info + 4 * f;
    sflags[6 * static_cast<size_t>(b[0]) + b[1]] |= (b[2] + 1) & 15;
  }
  for (int s = 0; s < ns; ++s)
    for (int side = 0; side < 6; ++side) {
      const int dn = side >> 1, ta = dn == 0 ? 1 : 0, tb = dn == 2 ? 1 : 2;
      const int nf = (p->orders_h[3 * s + ta] + 1) * (p->orders_h[3 * s + tb] + 1);
      const double* gg = desc->side_geo + 4 * desc->side_off[6 * s + side];
      bool uni = true;
      for (int c = 0; c < 4 && uni; ++c)
        for (int k = 1; k < nf && uni; ++k) uni = gg[c * nf + k] == gg[c * nf];
      if (uni) sflags[6 * static_cast<size_t>(s) + side] |= 16;
    }
  int* sflags_d = nullptr;
  std::vector<int> work_aff(work.size());
  for (size_t k = 0; k < work.size(); ++k) {
    int a = 1;
    for (int e = 0; e < work[k].y; ++e) a &= desc->affine[work[k].x + e] != 0;
    work_aff[k] = a;
  }
  std::vector<int> work_ord(3 * work.size());
  for (size_t k = 0; k < work.size(); ++k)
    for (int dd = 0; dd < 3; ++dd) work_ord[3 * k + dd] = p->orders_h[3 * work[k].x + dd];
  std::vector<int> work_mul(8 * work.size(), 0);
  for (size_t k = 0; k < work.size(); ++k) {
    const int a = work_ord[3 * k] + 1, b = work_ord[3 * k + 1] + 1, c = work_ord[3 * k + 2] + 1;
    const int dv[5] = {a * b * c, a, b, a * b, 2 * (b * c + a * c + a * b)};
    for (int j = 0; j < 5; ++j) work_mul[8 * k + j] = mdiv_mul(dv[j]);
  }
  int* work_mul_d = nullptr;
  int2* work_d;
  int* work_aff_d = nullptr;
  int* work_ord_d = nullptr;
  int4 *iso_d, *bnd_d;
  rc = p->mem.upload(work.data(), work.size(), &work_d);
  if (!rc) rc = p->mem.upload(work_aff.data(), work_aff.size(), &work_aff_d);
  if (!rc && ns > 0) rc = p->mem.upload(sflags.data(), sflags.size(), &sflags_d);
  if (!rc) rc = p->mem.upload(work_ord.data(), work_ord.size(), &work_ord_d);
  if (!rc) rc = p->mem.upload(work_mul.data(), work_mul.size(), &work_mul_d);
  if (!rc) rc = p->mem.upload(iso.data(), iso.size(), &iso_d);
  if (!rc) rc = p->mem.upload(bnd.data(), bnd.size(), &bnd_d);
  const size_t sn = static_cast<size_t>(desc->side_nodes);
  p->side_nodes = desc->side_nodes;

  const int NG = 3 * p->ngv;
  const size_t tn = static_cast<size_t>(desc->mtr_nodes);
  double *qtr, *lsurf = nullptr, *gtr = nullptr, *fsurf, *grad = nullptr;
  double *qtrm = nullptr, *gtrm = nullptr, *gsf = nullptr;
  if (!rc) rc = p->mem.zeros(sn * p->nv, &qtr);
  if (!rc) rc = p->mem.zeros(tn * p->nv, &qtrm);
  if (!rc) rc = p->mem.zeros(sn * p->nv, &fsurf);
  if (p->viscous) {
    if (!rc) rc = p->mem.zeros(sn * NG, &lsurf);
    if (!rc) rc = p->mem.zeros(sn * p->ntr, &gtr);
    if (!rc) rc = p->mem.zeros(tn * p->ntr, &gtrm);
    if (!rc) rc = p->mem.zeros(sn * p->ngv, &gsf);
  }
  if (rc) {
    delete p;
    return rc;
  }
  d.nwork = static_cast<int>(work.size());
  d.nsm = nsm_attr;
  {
    auto knob = [](const char* name, int dflt) {
      const char* v = getenv(name);
      return v ? atoi(v) : dflt;
    };
    d.pf_trace = knob("TDG_PF_TRACE", 2);
    d.pf_face = knob("TDG_PF_FACE", 4);
    d.pf_down = knob("TDG_PF_DOWN", 5);
    d.pf_item = knob("TDG_PF_ITEM", 1);
    int coll = 0;
    for (int dd = 0; dd < 3; ++dd) {
      bool c = ns > 0;
      for (int s = 0; s < ns && c; ++s) c = p->orders_h[3 * s + dd] == 0;
      coll |= c ? 1 << dd : 0;
    }
    d.collapsed = coll;
    // own-order trace branch (no mortars): 128-thread blocks split an N=7
    // element's 384 face nodes into three full rounds (256: one full, one
    // half-empty); measured config 4 N=7 0.127 -> 0.097 ms.  Mortar plans
    // keep 256 (warp per side; 192 / 128 measured slower)
    // (items with many small elements, > 700 face nodes, keep 256: measured
    // on config-4 levels N = 1, 2)
    int tasks = 0;
    for (const int2& w : work) {
      const int* o = &p->orders_h[3 * w.x];
      tasks = std::max(tasks, w.y * 2 * ((o[1] + 1) * (o[2] + 1) + (o[0] + 1) * (o[2] + 1) + (o[0] + 1) * (o[1] + 1)));
    }
    p->trace_threads = knob("TDG_TRACE_THREADS", d.nmface == 0 && tasks <= 700 ? 128 : ELEM_THREADS);
  }
  d.work = work_d;
  d.work_aff = work_aff_d;
  d.side_flags = sflags_d;
  d.work_ord = work_ord_d;
  d.work_mul = work_mul_d;
  d.nside_iso = static_cast<int>(iso.size());
  d.side_iso = iso_d;
  d.nside_bnd = static_cast<int>(bnd.size());
  d.side_bnd = bnd_d;
  d.qtr = qtr;
  d.qtrm = qtrm;
  d.gtrm = gtrm;
  d.lsurf = lsurf;
  d.gtr = gtr;
  d.fsurf = fsurf;
  d.grad = nullptr;
  d.gsf = gsf;
  // dynamic shared memory sized by the largest work item (<= MAXN nodes)
  const size_t mt = static_cast<size_t>(p->max_tot);
  // (Navier-Stokes keeps the lifted variables beside G for the side traces)
  {
    // lifted variables + max(curved metric staging, the item's side values of
    // the packed viscous-trace pass ([ntr] per face node))
    size_t need = static_cast<size_t>(p->ngv + 9) * mt;
    for (const int2& w : work) {
      const int* o = &p->orders_h[3 * w.x];
      const size_t n = static_cast<size_t>(o[0] + 1) * (o[1] + 1) * (o[2] + 1);
      const size_t per_e = 2 * ((o[1] + 1) * (o[2] + 1) + (o[0] + 1) * (o[2] + 1) + (o[0] + 1) * (o[1] + 1));
      need = std::max(need, p->ngv * n * w.y + p->ntr * per_e * w.y);
    }
    p->smem_lift = need * sizeof(double);
  }
  {
    bool curved = false;
    for (int s = 0; s < ns && !curved; ++s) curved = desc->affine[s] == 0;
    // every item affine: the own-order lift receives the item's Q span by one
    // TMA bulk copy into the region the curved metrics would use (TDG_TMA_Q=0: LDG)
    const char* tq = getenv("TDG_TMA_Q");
    d.tma_q = (!curved && !(tq && tq[0] == '0')) ? 1 : 0;
    // largest staged g* span over the items ((ngv + 3) values per face node)
    size_t sfn = 0;
    if (d.gstar && d.lift_packed)
      for (const int2& w : work) {
        const int* o = &p->orders_h[3 * w.x];
        const size_t per_e = 2 * ((o[1] + 1) * (o[2] + 1) + (o[0] + 1) * (o[2] + 1) + (o[0] + 1) * (o[1] + 1));
        sfn = std::max(sfn, ((p->ngv + 3) * per_e * w.y + 1) & ~size_t(1));
      }
    const size_t base = static_cast<size_t>(p->ngv + (curved ? 9 : 0)) * mt + sfn;
    // the Q bulk copy is kept only while three blocks still fit on an SM
    if (d.tma_q && d.lift_packed && (base + p->nv * mt + 2) * sizeof(double) > LIFT_OWN_SMEM_3) d.tma_q = 0;
    p->smem_lift_own = (base + (d.tma_q ? static_cast<size_t>(p->nv) * mt + 2 : 0)) * sizeof(double);
  }
  p->smem_flux = static_cast<size_t>(3 * p->nv) * mt * sizeof(double);
  if (p->viscous) {
    if ((rc = p->mem.zeros(static_cast<size_t>(p->nodes) * NG, &grad))) {
      delete p;
      return rc;
    }
    d.grad = grad;
  }
  {
    p->rk_traces = desc->family == TDG_LGL && d.nmface == 0;
    int dev = 0, nsm = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && nsm > 0)
      p->nsm = nsm;
  }
  switch (d.law) {
    case TDG_LAW_ADVDIFF: rc = setup_attrs<LAW_ADVDIFF>(p); break;
    case TDG_LAW_BURGERS: rc = setup_attrs<LAW_BURGERS>(p); break;
    default: rc = setup_attrs<LAW_NS>(p); break;
  }
  if (rc) {
    delete p;
    return rc;
  }
  *out = p;
  return TDG_OK;
}

int tdg_plan_destroy(tdg_plan* plan) {
  delete plan;
  return TDG_OK;
}

int tdg_plan_size(const tdg_plan* plan, int64_t* nodes, int32_t* nv) {
  if (!plan) return fail(TDG_E_ARG, "null plan");
  if (nodes) *nodes = plan->nodes;
  if (nv) *nv = plan->nv;
  return TDG_OK;
}

int tdg_apply(tdg_plan* p, const double* Q, double* F, int isolated, void* stream) {
  if (!p || !Q || !F) return fail(TDG_E_ARG, "null argument");
  FluxArgs a{};
  a.out = F;
  return dispatch_eval<MODE_F>(p, Q, isolated, a, as_stream(stream));
}

int tdg_m_inv_apply(tdg_plan* p, const double* Q, const double* add, double* out, int isolated,
                    void* stream) {
  if (!p || !Q || !out) return fail(TDG_E_ARG, "null argument");
  FluxArgs a{};
  a.out = out;
  a.X = add;
  return dispatch_eval<MODE_A>(p, Q, isolated, a, as_stream(stream));
}

int tdg_residual(tdg_plan* p, const double* Q, const double* S, double* R, double* rnorm,
                 void* stream) {
  if (!p || !Q) return fail(TDG_E_ARG, "null argument");
  cudaStream_t st = as_stream(stream);
  if (rnorm) CUDA_TRY(cudaMemsetAsync(rnorm, 0, sizeof(double), st));
  FluxArgs a{};
  a.S = S;
  a.out = R;
  a.norm = rnorm;
  return dispatch_eval<MODE_R>(p, Q, 0, a, st);
}

int tdg_residual_host(tdg_plan* p, int32_t nbatch, const double* const* Qh, const double* S,
                      double* const* Rh, double* rnorm_host, void* stream) {
  if (!p || (nbatch > 0 && (!Qh || !Rh))) return fail(TDG_E_ARG, "null argument");
  if (nbatch < 0) return fail(TDG_E_ARG, "nbatch must be >= 0");
  for (int b = 0; b < nbatch; ++b)
    if (!Qh[b] || !Rh[b]) return fail(TDG_E_ARG, "null host buffer in batch");
  if (nbatch == 0) return TDG_OK;
  cudaStream_t st = as_stream(stream);
  auto& g = p->stage;
  const size_t bytes = static_cast<size_t>(p->nodes) * p->nv * sizeof(double);
  if (!g.ready) {
    for (int s = 0; s < 2; ++s) {
      CUDA_TRY(cudaMalloc(&g.q[s], bytes ? bytes : 8));
      CUDA_TRY(cudaMalloc(&g.r[s], bytes ? bytes : 8));
      CUDA_TRY(cudaEventCreateWithFlags(&g.in[s], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&g.done[s], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&g.out[s], cudaEventDisableTiming));
    }
    CUDA_TRY(cudaEventCreateWithFlags(&g.start, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&g.fin, cudaEventDisableTiming));
    CUDA_TRY(cudaStreamCreateWithFlags(&g.h2d, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&g.d2h, cudaStreamNonBlocking));
    g.ready = true;
  }
  if (g.norm_cap < nbatch) {
    cudaFree(g.norm_dev);
    cudaFreeHost(g.norm_host);
    g.norm_dev = nullptr;
    g.norm_host = nullptr;
    g.norm_cap = 0;
    CUDA_TRY(cudaMalloc(&g.norm_dev, sizeof(double) * nbatch));
    CUDA_TRY(cudaMallocHost(&g.norm_host, sizeof(double) * nbatch));
    g.norm_cap = nbatch;
  }
  // everything below is ordered after the caller's prior work on `stream`
  CUDA_TRY(cudaEventRecord(g.start, st));
  CUDA_TRY(cudaStreamWaitEvent(g.h2d, g.start, 0));
  CUDA_TRY(cudaStreamWaitEvent(g.d2h, g.start, 0));
  CUDA_TRY(cudaMemsetAsync(g.norm_dev, 0, sizeof(double) * nbatch, st));
  for (int b = 0; b < nbatch; ++b) {
    const int s = b & 1;
    // slot s is free for input once evaluation b-2 finished, for output once
    // its device->host copy finished
    if (b >= 2) CUDA_TRY(cudaStreamWaitEvent(g.h2d, g.done[s], 0));
    CUDA_TRY(cudaMemcpyAsync(g.q[s], Qh[b], bytes, cudaMemcpyHostToDevice, g.h2d));
    CUDA_TRY(cudaEventRecord(g.in[s], g.h2d));
    CUDA_TRY(cudaStreamWaitEvent(st, g.in[s], 0));
    if (b >= 2) CUDA_TRY(cudaStreamWaitEvent(st, g.out[s], 0));
    FluxArgs a{};
    a.S = S;
    a.out = g.r[s];
    a.norm = g.norm_dev + b;
    int rc = dispatch_eval<MODE_R>(p, g.q[s], 0, a, st);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(g.done[s], st));
    CUDA_TRY(cudaStreamWaitEvent(g.d2h, g.done[s], 0));
    CUDA_TRY(cudaMemcpyAsync(Rh[b], g.r[s], bytes, cudaMemcpyDeviceToHost, g.d2h));
    CUDA_TRY(cudaEventRecord(g.out[s], g.d2h));
  }
  CUDA_TRY(cudaMemcpyAsync(g.norm_host, g.norm_dev, sizeof(double) * nbatch, cudaMemcpyDeviceToHost,
                           g.d2h));
  CUDA_TRY(cudaEventRecord(g.fin, g.d2h));
  CUDA_TRY(cudaStreamWaitEvent(st, g.fin, 0));
  CUDA_TRY(cudaEventSynchronize(g.fin));
  if (rnorm_host) std::memcpy(rnorm_host, g.norm_host, sizeof(double) * nbatch);
  p->traces_of = nullptr;   // the staging slots are not caller buffers
  return TDG_OK;
}

int tdg_tau(tdg_plan* p, const double* Q, const double* S, double* tau, int isolated,
            void* stream) {
  if (!p || !Q || !tau) return fail(TDG_E_ARG, "null argument");
  cudaStream_t st = as_stream(stream);
  CUDA_TRY(cudaMemsetAsync(tau, 0, sizeof(double) * p->d.nslots, st));
  FluxArgs a{};
  a.S = S;
  a.out = tau;
  return dispatch_eval<MODE_TAU>(p, Q, isolated, a, st);
}

int tdg_tau_from_avalue(tdg_plan* p, const double* A, const double* S, double* tau, void* stream) {
  if (!p || !A || !tau) return fail(TDG_E_ARG, "null argument");
  cudaStream_t st = as_stream(stream);
  if (p->d.nwork == 0) return TDG_OK;
  KTimer kt(TDG_K_NORM, st);
  if (p->nv == 5)
    k_tau_avalue<5><<<p->d.nwork, ELEM_THREADS, 0, st>>>(p->d, A, S, tau);
  else
    k_tau_avalue<1><<<p->d.nwork, ELEM_THREADS, 0, st>>>(p->d, A, S, tau);
  LAUNCH_CHECK("k_tau_avalue");
  return TDG_OK;
}

int tdg_rk3_stage(tdg_plan* p, double* Q, double* W, const double* S, int stage, const double* dt,
                  int local, double* rnorm, int32_t* nonfinite, void* stream) {
  return tdg_rk3_stage_ex(p, Q, W, S, stage, dt, local, rnorm, nonfinite, 0, stream);
}

int tdg_rk3_stage_ex(tdg_plan* p, double* Q, double* W, const double* S, int stage, const double* dt,
                     int local, double* rnorm, int32_t* nonfinite, int flags, void* stream) {
  static const double RK_A[3] = {0.0, -5.0 / 9.0, -153.0 / 128.0};   // timestep.py:18-20
  static const double RK_B[3] = {1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0};
  if (!p || !Q || !W || !dt) return fail(TDG_E_ARG, "null argument");
  if (stage < 0 || stage > 2) return fail(TDG_E_ARG, "stage must be 0, 1 or 2");
  FluxArgs a{};
  a.S = S;
  a.W = W;
  a.Qout = Q;
  a.dt = dt;
  a.local = local;
  a.stage = stage;
  a.rk_a = RK_A[stage];
  a.rk_b = RK_B[stage];
  a.norm = rnorm;
  a.nonfinite = reinterpret_cast<int*>(nonfinite);
  a.traces = p->rk_traces ? 1 : 0;
  // the caller vouches that Q is unchanged since the previous call on this
  // plan; the traces are reused if that call left them for this buffer
  const bool fresh = (flags & TDG_RK_TRACES_FRESH) && p->rk_traces && p->traces_of == Q;
  return dispatch_eval<MODE_RK>(p, Q, 0, a, as_stream(stream), fresh);
}

int tdg_element_dt(tdg_plan* p, const double* Q, double cfl_a, double cfl_v, double* dt_slot,
                   double* dt_min, void* stream) {
  if (!p || !Q) return fail(TDG_E_ARG, "null argument");
  cudaStream_t st = as_stream(stream);
  if (dt_min) {
    k_fill<<<1, 32, 0, st>>>(dt_min, HUGE_VAL, 1);
    LAUNCH_CHECK("k_fill");
  }
  if (p->d.nwork == 0) return TDG_OK;
  KTimer kt(TDG_K_DT, st);
  switch (p->d.law) {
    case TDG_LAW_ADVDIFF:
      k_element_dt<LAW_ADVDIFF><<<p->d.nwork, ELEM_THREADS, 0, st>>>(p->d, Q, cfl_a, cfl_v, dt_slot, dt_min);
      break;
    case TDG_LAW_BURGERS:
      k_element_dt<LAW_BURGERS><<<p->d.nwork, ELEM_THREADS, 0, st>>>(p->d, Q, cfl_a, cfl_v, dt_slot, dt_min);
      break;
    default:
      k_element_dt<LAW_NS><<<p->d.nwork, ELEM_THREADS, 0, st>>>(p->d, Q, cfl_a, cfl_v, dt_slot, dt_min);
  }
  LAUNCH_CHECK("k_element_dt");
  return TDG_OK;
}

int tdg_norm_inf(tdg_plan* p, const double* X, double* gmax, double* emax, void* stream) {
  if (!p || !X) return fail(TDG_E_ARG, "null argument");
  cudaStream_t st = as_stream(stream);
  if (gmax) CUDA_TRY(cudaMemsetAsync(gmax, 0, sizeof(double), st));
  if (p->d.nwork == 0) return TDG_OK;
  KTimer kt(TDG_K_NORM, st);
  if (p->nv == 5)
    k_norm<5><<<p->d.nwork, ELEM_THREADS, 0, st>>>(p->d, X, gmax, emax, nullptr);
  else
    k_norm<1><<<p->d.nwork, ELEM_THREADS, 0, st>>>(p->d, X, gmax, emax, nullptr);
  LAUNCH_CHECK("k_norm");
  return TDG_OK;
}

int tdg_check_finite(tdg_plan* p, const double* X, int32_t* flag, void* stream) {
  if (!p || !X || !flag) return fail(TDG_E_ARG, "null argument");
  cudaStream_t st = as_stream(stream);
  if (p->d.nwork == 0) return TDG_OK;
  if (p->nv == 5)
    k_norm<5><<<p->d.nwork, ELEM_THREADS, 0, st>>>(p->d, X, nullptr, nullptr, reinterpret_cast<int*>(flag));
  else
    k_norm<1><<<p->d.nwork, ELEM_THREADS, 0, st>>>(p->d, X, nullptr, nullptr, reinterpret_cast<int*>(flag));
  LAUNCH_CHECK("k_norm");
  return TDG_OK;
}

int tdg_gradient(tdg_plan* p, const double* Q, int isolated, double* dst, void* stream) {
  if (!p || !Q || !dst) return fail(TDG_E_ARG, "null argument");
  if (!p->viscous) return fail(TDG_E_CONFIG, "inviscid plan has no gradient");
  // one trace + lift pass that stores the per-node gradient straight into dst
  DevPlan d = p->d;
  d.grad = dst;
  switch (p->d.law) {
    case TDG_LAW_ADVDIFF: return run_surface<LAW_ADVDIFF>(p, d, Q, isolated, as_stream(stream), false, true);
    case TDG_LAW_BURGERS: return run_surface<LAW_BURGERS>(p, d, Q, isolated, as_stream(stream), false, true);
    default: return run_surface<LAW_NS>(p, d, Q, isolated, as_stream(stream), false, true);
  }
}

int tdg_plan_info(const tdg_plan* p, int32_t* nwork, int32_t* nconf_faces, int32_t* nmortar_faces) {
  if (!p) return fail(TDG_E_ARG, "null plan");
  if (nwork) *nwork = p->d.nwork;
  if (nconf_faces) *nconf_faces = p->d.ncface;
  if (nmortar_faces) *nmortar_faces = p->d.nmface;
  return TDG_OK;
}

int tdg_debug_copy(tdg_plan* p, int which, double* dst, int64_t* len_out, void* stream) {
  if (!p) return fail(TDG_E_ARG, "null plan");
  const int NG = 3 * p->ngv;
  const double* src = nullptr;
  int64_t comps = 0;
  switch (which) {
    case 0: src = p->d.qtr; comps = p->nv; break;
    case 1: src = p->d.lsurf; comps = NG; break;
    case 2: src = p->d.gtr; comps = p->ntr; break;
    case 3: src = p->d.fsurf; comps = p->nv; break;
    default: return fail(TDG_E_ARG, "unknown buffer");
  }
  const int64_t n = comps * p->side_nodes;
  if (len_out) *len_out = n;
  if (!dst) return TDG_OK;
  if (!src) return fail(TDG_E_CONFIG, "buffer not allocated (inviscid plan)");
  CUDA_TRY(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, as_stream(stream)));
  return TDG_OK;
}

int tdg_loop_begin(void* stream, void* body_stream, tdg_loop** out) {
  if (!out || !body_stream) return fail(TDG_E_ARG, "null argument");
  cudaStream_t st = as_stream(stream);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CUDA_TRY(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
  if (cs != cudaStreamCaptureStatusActive) return fail(TDG_E_ARG, "tdg_loop_begin: stream is not capturing");
  auto* lp = new tdg_loop();
  cudaGraphNodeParams prm = {};
  cudaGraphNode_t node = nullptr;
  cudaError_t e = cudaGraphConditionalHandleCreate(&lp->handle, g, 1u, cudaGraphCondAssignDefault);
  if (e == cudaSuccess) {
    prm.type = cudaGraphNodeTypeConditional;
    prm.conditional.handle = lp->handle;
    prm.conditional.type = cudaGraphCondTypeWhile;
    prm.conditional.size = 1;
    e = cudaGraphAddNode(&node, g, deps, nd, &prm);
  }
  if (e == cudaSuccess) e = cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies);
  lp->body = as_stream(body_stream);
  if (e == cudaSuccess)
    e = cudaStreamBeginCaptureToGraph(lp->body, prm.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                      cudaStreamCaptureModeRelaxed);
  if (e != cudaSuccess) {
    delete lp;
    return fail(TDG_E_CUDA, std::string("tdg_loop_begin: ") + cudaGetErrorString(e));
  }
  *out = lp;
  return TDG_OK;
}

int tdg_volume_metrics(int32_t nel, const int32_t* ctrl_shape, const double* ctrl, const int32_t* npts,
                       const double* tables, double* jac, double* ja, double* coords, double* sizes) {
  if (!ctrl_shape || !npts || !tables || (nel > 0 && (!ctrl || !jac || !ja || !coords || !sizes)))
    return fail(TDG_E_ARG, "null argument");
  if (nel <= 0) return TDG_OK;
  const int a1 = ctrl_shape[0], a2 = ctrl_shape[1], a3 = ctrl_shape[2];
  const int n1p = npts[0], n2p = npts[1], n3p = npts[2];
  if (a1 < 1 || a2 < 1 || a3 < 1 || a1 > 4 || a2 > 4 || a3 > 4)
    return fail(TDG_E_CONFIG, "device metrics: mapping orders must lie in 0..3");
  if (n1p < 1 || n2p < 1 || n3p < 1 || n1p > 8 || n2p > 8 || n3p > 8)
    return fail(TDG_E_CONFIG, "device metrics: solution orders must lie in 0..7");
  const size_t n = static_cast<size_t>(n1p) * n2p * n3p, ne = static_cast<size_t>(nel);
  const size_t nc = ne * a1 * a2 * a3 * 3;
  Allocs mem;
  double *d_ctrl, *d_jac, *d_ja, *d_x, *d_h;
  GeoTables* d_tab;
  int rc = mem.upload(ctrl, nc, &d_ctrl);
  if (!rc) rc = mem.upload(reinterpret_cast<const GeoTables*>(tables), 1, &d_tab);
  if (!rc) rc = mem.zeros(ne * n, &d_jac);
  if (!rc) rc = mem.zeros(ne * n * 9, &d_ja);
  if (!rc) rc = mem.zeros(ne * n * 3, &d_x);
  if (!rc) rc = mem.zeros(ne * 3, &d_h);
  if (rc) return rc;
  const size_t smem = 15 * n * sizeof(double);
  if ((rc = allow_smem(k_volume_metrics, smem))) return rc;
  k_volume_metrics<<<nel, GEO_THREADS, smem>>>(d_ctrl, a1, a2, a3, n1p, n2p, n3p, d_tab, d_jac, d_ja, d_x, d_h);
  LAUNCH_CHECK("k_volume_metrics");
  CUDA_TRY(cudaMemcpy(jac, d_jac, ne * n * sizeof(double), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(ja, d_ja, ne * n * 9 * sizeof(double), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(coords, d_x, ne * n * 3 * sizeof(double), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(sizes, d_h, ne * 3 * sizeof(double), cudaMemcpyDeviceToHost));
  return TDG_OK;
}

int tdg_stream_create(void** out) {
  if (!out) return fail(TDG_E_ARG, "null argument");
  cudaStream_t s = nullptr;
  CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *out = s;
  return TDG_OK;
}

int tdg_stream_destroy(void* stream) {
  if (stream) CUDA_TRY(cudaStreamDestroy(as_stream(stream)));
  return TDG_OK;
}

int tdg_loop_test(tdg_loop* lp, const double* rnorm, const double* snorm, const double* tolf, const double* cmp,
                  double eta, int mode, int32_t* count, int max_iter) {
  if (!lp || !rnorm || !snorm || !tolf || !cmp || !count) return fail(TDG_E_ARG, "null argument");
  k_loop_test<<<1, 1, 0, lp->body>>>(lp->handle, rnorm, snorm, tolf, cmp, eta, mode, reinterpret_cast<int*>(count),
                                      max_iter);
  LAUNCH_CHECK("k_loop_test");
  return TDG_OK;
}

int tdg_loop_end(tdg_loop* lp) {
  if (!lp) return fail(TDG_E_ARG, "null loop");
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(lp->body, &g);
  delete lp;
  if (e != cudaSuccess) return fail(TDG_E_CUDA, std::string("tdg_loop_end: ") + cudaGetErrorString(e));
  return TDG_OK;
}

int tdg_transfer_create(const tdg_transfer_desc* desc, tdg_transfer** out) {
  if (!desc || !out) return fail(TDG_E_ARG, "null argument");
  *out = nullptr;
  if (desc->tables_len != TABLES_LEN) return fail(TDG_E_CONFIG, "spectral table length mismatch");
  const int ns = desc->nslots;
  std::vector<int> f_orders(desc->fine_orders, desc->fine_orders + 3 * ns);
  std::vector<int> c_orders(desc->coarse_orders, desc->coarse_orders + 3 * ns);
  for (int k = 0; k < 3 * ns; ++k)
    if (f_orders[k] < 0 || f_orders[k] > 7 || c_orders[k] < 0 || c_orders[k] > 7)
      return fail(TDG_E_CONFIG, "polynomial orders must lie in 0..7 on the device path");
  std::unordered_map<int, int> cslot;
  for (int s = 0; s < ns; ++s) cslot[desc->coarse_elem_id[s]] = s;
  std::vector<int> c_of_f(ns);
  for (int s = 0; s < ns; ++s) {
    auto it = cslot.find(desc->fine_elem_id[s]);
    if (it == cslot.end()) return fail(TDG_E_CONFIG, "element id missing in coarse field");
    c_of_f[s] = it->second;
  }
  auto* t = new tdg_transfer();
  t->nv = desc->nv;
  std::vector<int2> work;
  for (int s = 0; s < ns;) {
    const int* fo = &f_orders[3 * s];
    const int* co = &c_orders[3 * c_of_f[s]];
    int mx = 1;
    // largest staging footprint over both transfer directions
    for (int dir = 0; dir < 2; ++dir) {
      const int* a = dir ? co : fo;
      const int* b = dir ? fo : co;
      const int sizes[4] = {(a[0] + 1) * (a[1] + 1) * (a[2] + 1), (b[0] + 1) * (a[1] + 1) * (a[2] + 1),
                            (b[0] + 1) * (b[1] + 1) * (a[2] + 1), (b[0] + 1) * (b[1] + 1) * (b[2] + 1)};
      for (int k = 0; k < 4; ++k) mx = std::max(mx, sizes[k]);
    }
    const int cap = std::max(1, MAXN / mx);
    int e = s;
    while (e < ns && e - s < cap) {
      const int* fe = &f_orders[3 * e];
      const int* ce = &c_orders[3 * c_of_f[e]];
      if (fe[0] != fo[0] || fe[1] != fo[1] || fe[2] != fo[2] || ce[0] != co[0] || ce[1] != co[1] ||
          ce[2] != co[2])
        break;
      ++e;
    }
    work.push_back(make_int2(s, e - s));
    s = e;
  }
  int2* work_d;
  int *c_d, *fo_d, *co_d;
  long long *fno_d, *cno_d;
  double* tab_d;
  int rc = t->mem.upload(work.data(), work.size(), &work_d);
  if (!rc) rc = t->mem.upload(c_of_f.data(), c_of_f.size(), &c_d);
  if (!rc) rc = t->mem.upload(f_orders.data(), f_orders.size(), &fo_d);
  if (!rc) rc = t->mem.upload(c_orders.data(), c_orders.size(), &co_d);
  if (!rc) rc = t->mem.upload(reinterpret_cast<const long long*>(desc->fine_node_off), (size_t)ns + 1, &fno_d);
  if (!rc) rc = t->mem.upload(reinterpret_cast<const long long*>(desc->coarse_node_off), (size_t)ns + 1, &cno_d);
  if (!rc) rc = t->mem.upload(desc->tables, (size_t)desc->tables_len, &tab_d);
  if (rc) {
    delete t;
    return rc;
  }
  t->d.tables = tab_d;
  t->d.nv = desc->nv;
  t->d.f_orders = fo_d;
  t->d.f_node_off = fno_d;
  t->d.c_orders = co_d;
  t->d.c_node_off = cno_d;
  t->d.c_slot_of_f = c_d;
  t->d.work = work_d;
  t->nwork = static_cast<int>(work.size());
  t->smem = 2 * static_cast<size_t>(t->nv) * MAXN * sizeof(double);
  {
    auto iso_points = [](const std::vector<int>& o, int n) {
      if (n == 0) return 0;
      for (int k = 0; k < 3 * n; ++k)
        if (o[k] != o[0]) return 0;
      return o[0] + 1;
    };
    t->iso_f = iso_points(f_orders, ns);
    t->iso_c = iso_points(c_orders, static_cast<int>(c_orders.size() / 3));
    // line kernel: every item is a run of consecutive slots on both levels
    // (node offsets then advance by one element's points per slot)
    // (TDG_TRANSFER_LINES=0 keeps the one-output-per-thread kernel)
    const char* lenv = getenv("TDG_TRANSFER_LINES");
    bool contig = t->iso_f > 0 && t->iso_c > 0 && !(lenv && lenv[0] == '0');
    const long long pf = static_cast<long long>(t->iso_f) * t->iso_f * t->iso_f;
    const long long pc = static_cast<long long>(t->iso_c) * t->iso_c * t->iso_c;
    for (const int2& w : work) {
      for (int e = 1; e < w.y && contig; ++e) {
        const int s = w.x + e;
        contig = c_of_f[s] == c_of_f[w.x] + e &&
                 desc->fine_node_off[s] == desc->fine_node_off[w.x] + e * pf &&
                 desc->coarse_node_off[c_of_f[s]] == desc->coarse_node_off[c_of_f[w.x]] + e * pc;
      }
      if (!contig) break;
    }
    t->lines = contig;
  }
  if ((rc = allow_smem(k_transfer<TR_RESTRICT>, t->smem)) || (rc = allow_smem(k_transfer<TR_PROLONG>, t->smem)) ||
      (rc = allow_smem(k_transfer<TR_PROLONG_ADD>, t->smem)) || (rc = allow_lines_smem(t->smem))) {
    delete t;
    return rc;
  }
  *out = t;
  return TDG_OK;
}

int tdg_transfer_destroy(tdg_transfer* t) {
  delete t;
  return TDG_OK;
}

int tdg_restrict(const tdg_transfer* t, const double* fine, double* coarse, void* stream) {
  if (!t || !fine || !coarse) return fail(TDG_E_ARG, "null argument");
  if (!t->nwork) return TDG_OK;
  KTimer kt(TDG_K_TRANSFER, as_stream(stream));
  launch_transfer<TR_RESTRICT>(t, fine, nullptr, coarse, as_stream(stream));
  LAUNCH_CHECK("k_transfer(restrict)");
  return TDG_OK;
}

int tdg_prolong(const tdg_transfer* t, const double* coarse, double* fine, void* stream) {
  if (!t || !fine || !coarse) return fail(TDG_E_ARG, "null argument");
  if (!t->nwork) return TDG_OK;
  KTimer kt(TDG_K_TRANSFER, as_stream(stream));
  launch_transfer<TR_PROLONG>(t, coarse, nullptr, fine, as_stream(stream));
  LAUNCH_CHECK("k_transfer(prolong)");
  return TDG_OK;
}

int tdg_prolong_add(const tdg_transfer* t, const double* Qc, const double* Qc0, double* fine,
                    void* stream) {
  if (!t || !fine || !Qc) return fail(TDG_E_ARG, "null argument");
  if (!t->nwork) return TDG_OK;
  KTimer kt(TDG_K_TRANSFER, as_stream(stream));
  launch_transfer<TR_PROLONG_ADD>(t, Qc, Qc0, fine, as_stream(stream));
  LAUNCH_CHECK("k_transfer(prolong_add)");
  return TDG_OK;
}

}  // extern "C"

#ifdef TDG_PHASE_CLOCK
extern "C" int tdg_debug_phases(unsigned long long* out32, int reset) {
  if (out32) cudaMemcpyFromSymbol(out32, tdg::g_phase, sizeof(unsigned long long) * 32);
  if (reset) {
    unsigned long long z[32] = {};
    cudaMemcpyToSymbol(tdg::g_phase, z, sizeof(z));
  }
  return 0;
}
#endif
