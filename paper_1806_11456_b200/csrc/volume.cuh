// volume.cuh — element-parallel kernels over shape-uniform work items.
//
// A work item is a run of slots of ONE bucket (same (N1,N2,N3)), at most MAXN
// nodes in total; a 256-thread block owns one item, each thread up to NPT
// nodes.  Spectral tables of the bucket's three orders are staged in shared
// memory; contravariant fluxes are staged in shared memory and contracted
// direction by direction with the weighted derivative matrices (the weak
// divergence of operators.py:196-200).
#pragma once
#include "common.cuh"
#include "laws.cuh"

namespace tdg {

#ifdef TDG_PHASE_CLOCK
__device__ unsigned long long g_phase[32];
#define PHASE_T(k) do { if (threadIdx.x == 0) pt[k] = clock64(); } while (0)
#define PHASE_DECL long long pt[8] = {0,0,0,0,0,0,0,0}
#define PHASE_END(base, n) do { if (threadIdx.x == 0) { for (int z = 1; z < n; ++z) atomicAdd(&g_phase[base + z], (unsigned long long)(pt[z] - pt[z-1])); atomicAdd(&g_phase[base], 1ull);} } while (0)
#else
#define PHASE_T(k)
#define PHASE_DECL
#define PHASE_END(base, n)
#endif

struct ElemTables {
  double dh[3][64];   // Dhat[m*8+i] per direction
  double w[3][8];
  double bnd[3][16];  // l_i(-1) at [i], l_i(+1) at [8+i]
  double red[32];
  unsigned long long emax[MAX_ITEM_ELEMS];  // per-element max bits (tau / dt)
};

__device__ __forceinline__ void load_tables(const DevPlan& P, int N1, int N2, int N3,
                                            ElemTables& T) {
  for (int u = threadIdx.x; u < 3 * 64; u += blockDim.x) {
    const int d = u / 64, k = u % 64;
    T.dh[d][k] = P.tables[OFF_DHAT + sel3(d, N1, N2, N3) * 64 + k];
  }
  for (int u = threadIdx.x; u < 3 * 8; u += blockDim.x) {
    const int d = u / 8, k = u % 8;
    T.w[d][k] = P.tables[OFF_W + sel3(d, N1, N2, N3) * 8 + k];
  }
  for (int u = threadIdx.x; u < 3 * 16; u += blockDim.x) {
    const int d = u / 16, k = u % 16;
    T.bnd[d][k] = P.tables[OFF_BND + sel3(d, N1, N2, N3) * 16 + k];
  }
  for (int u = threadIdx.x; u < MAX_ITEM_ELEMS; u += blockDim.x) T.emax[u] = 0ull;
}

__device__ __forceinline__ const double* metric_ptr(const DevPlan& P, int slot, int node, int n,
                                                    int& stride) {
  const bool aff = P.affine[slot] != 0;
  stride = aff ? 1 : n;
  return P.metrics + P.metric_off[slot] + (aff ? 0 : node);
}

// ---------------------------------------------------------------------------
// Side traces (operators.py:73-80, 185-194).  One warp per element side: the
// own-order trace (LGL: gather of the face nodes; LG: boundary-row
// contraction) is written as is, or — for nonconforming interior sides of a
// coupled evaluation — interpolated onto the side's mortar (own frame)
// through warp_proj2, so the face kernels are pointwise.

__device__ __forceinline__ void side_mortar_dims(int4 si, int& ma, int& mb) {
  const int M1 = si.y & 255, M2 = (si.y >> 8) & 255;
  const bool swap_r = (si.x & 2) && (((si.x >> 2) & 7) & 4);
  ma = (swap_r ? M2 : M1) + 1;
  mb = (swap_r ? M1 : M2) + 1;
}

// Side traces of C components for every side of a work item, one warp per
// side.  Own-order sides: lanes over face nodes (coalesced) into ``own``.
// Nonconforming sides of a coupled evaluation: the own trace is interpolated
// onto the side's mortar (own frame) on the FP64 tensor cores (warp_proj_mma,
// reading the face layer through vol()) and written to ``mort`` at the side's
// mortar-trace offset, so the face kernels stay pointwise.
template <int C, class Vol>
__device__ __forceinline__ void item_side_traces(const DevPlan& P, int slot0, int E, int coupled,
                                                 const int np[3], const int strides[3],
                                                 const double (*bnd)[16], double* own, double* mort,
                                                 Vol vol) {
  const bool lgl = P.family == 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int task = warp; task < E * 6; task += blockDim.x >> 5) {
    const int e = task / 6, s = task % 6, slot = slot0 + e;
    int d, a, b;
    side_dirs(s, d, a, b);
    const int na = sel3(a, np[0], np[1], np[2]), nb = sel3(b, np[0], np[1], np[2]);
    const int nd = sel3(d, np[0], np[1], np[2]), nf = na * nb;
    const int sa = sel3(a, strides[0], strides[1], strides[2]);
    const int sb = sel3(b, strides[0], strides[1], strides[2]);
    const int sd = sel3(d, strides[0], strides[1], strides[2]);
    const int last = (s & 1) ? (nd - 1) * sd : 0;
    const double* row = bnd[d] + (s & 1) * 8;
    auto tr = [&](int c, int ia, int ib) -> double {
      const int off0 = ia * sa + ib * sb;
      if (lgl) return vol(e, c, off0 + last);
      double acc = 0.0;
      for (int m = 0; m < nd; ++m) acc += row[m] * vol(e, c, off0 + m * sd);
      return acc;
    };
    const int4 si = P.side_info[slot * 6 + s];
    if (coupled && (si.x & 1)) {
      const int M1 = si.y & 255, M2 = (si.y >> 8) & 255;
      const bool swap_r = (si.x & 2) && (((si.x >> 2) & 7) & 4);
      const int ma = (swap_r ? M2 : M1) + 1, mb = (swap_r ? M1 : M2) + 1, nm = ma * mb;
      const double* T1 = P.tables + OFF_T + ((na - 1) * 8 + (ma - 1)) * 64;
      const double* T2 = P.tables + OFF_T + ((nb - 1) * 8 + (mb - 1)) * 64;
      double* dst = mort + (long long)si.w * C;
      warp_proj_mma<C>(na, nb, T1, ma, T2, mb, tr, dst, nm, [&](int A, int B) { return A + ma * B; });
    } else {
      double* dst = own + P.side_off[slot * 6 + s] * C;
      for (int k = lane; k < nf; k += 32) {
        const int ib = k / na, ia = k - ib * na;
        for (int c = 0; c < C; ++c) dst[(long long)c * nf + k] = tr(c, ia, ib);
      }
    }
  }
}

// Own-order geometry of an element side at face node kf: sigma and the outward
// normal ([4][nf] per side; uniform sides read node 0).
__device__ __forceinline__ void side_geometry(const DevPlan& P, long long so, int nf, int kf, bool uni,
                                              double& sigma, double* nrm) {
  const double* geo = P.side_geo + so * 4 + (uni ? 0 : kf);
  sigma = geo[0];
  nrm[0] = geo[nf];
  nrm[1] = geo[2 * nf];
  nrm[2] = geo[3 * nf];
}

// L2 bulk prefetch of a work item's per-side surface span ([C][nf] per side,
// contiguous over the item's slots and sides), read late by the scatter.
template <int C>
__device__ __forceinline__ void prefetch_item_surface(const DevPlan& P, const double* surf, int2 wi,
                                                      int N1, int N2) {
  if (threadIdx.x != 0 || surf == nullptr) return;
  const long long s0 = P.side_off[wi.x * 6];
  const long long s1 = P.side_off[(wi.x + wi.y - 1) * 6 + 5] + (long long)(N1 + 1) * (N2 + 1);
  l2_prefetch_span(surf + s0 * C, static_cast<size_t>(s1 - s0) * C * sizeof(double));
}

// L2 bulk prefetch, one thread per element side, of the g* values and the
// face geometry of every conforming interior side of a work item (g* form).
template <int NGV>
__device__ __forceinline__ void prefetch_item_gstar(const DevPlan& P, int2 wi, int N1, int N2, int N3) {
  for (int u = threadIdx.x; u < wi.y * 6; u += blockDim.x) {
    const int4 sn = P.side_nb[wi.x * 6 + u];
    if (sn.x < 0) continue;
    const int d = (u % 6) >> 1;
    const int nf = d == 0 ? (N2 + 1) * (N3 + 1) : d == 1 ? (N1 + 1) * (N3 + 1) : (N1 + 1) * (N2 + 1);
    l2_prefetch_span(P.gsf + (long long)sn.x * NGV, sizeof(double) * nf * NGV);
    if (!((sn.z >> 10) & 1)) l2_prefetch_span(P.face_geo + sn.y, sizeof(double) * nf * 4);
  }
}

// L2 bulk prefetch of a work item's per-node span of a C-component field
// (the item's slots are contiguous), issued by thread ``who``.
template <int C>
__device__ __forceinline__ void prefetch_item_nodes(const DevPlan& P, const double* x, int2 wi,
                                                    int who) {
  if (threadIdx.x != who || x == nullptr) return;
  const long long n0 = P.node_off[wi.x], n1 = P.node_off[wi.x + wi.y];
  l2_prefetch_span(x + n0 * C, static_cast<size_t>(n1 - n0) * C * sizeof(double));
}

// L2 bulk prefetch of a curved work item's per-node metrics ([10][n] per
// slot, contiguous over the item's slots), issued by thread ``who``.
__device__ __forceinline__ void prefetch_item_metrics(const DevPlan& P, int2 wi, int n, int who) {
  if (threadIdx.x != who || P.work_aff[blockIdx.x]) return;
  const long long m0 = P.metric_off[wi.x], m1 = P.metric_off[wi.x + wi.y - 1] + 10LL * n;
  l2_prefetch_span(P.metrics + m0, static_cast<size_t>(m1 - m0) * sizeof(double));
}

// The work item per_sm * nsm blocks ahead of this block (blocks start in
// index order: with per_sm resident blocks per SM it runs about one wave
// later), or wi.y == 0 if none.
__device__ __forceinline__ int2 item_ahead(const DevPlan& P, int per_sm) {
  const int b = blockIdx.x + per_sm * P.nsm;
  return b < P.nwork ? P.work[b] : make_int2(0, 0);
}

template <int NV>
__global__ void __launch_bounds__(ELEM_THREADS) k_trace_q(DevPlan P, const double* __restrict__ Q,
                                                          int coupled) {
  __shared__ double sb[3][16];
  __shared__ unsigned long long qbar;
  extern __shared__ double qsm[];   // mortar plans: the item's Q span ([nv][n] x E)
  const int2 wi = P.work[blockIdx.x];
  {
    const int2 wn = item_ahead(P, P.pf_trace);
    if (wn.y > 0) prefetch_item_nodes<NV>(P, Q, wn, 0);
  }
  const int* od = P.work_ord + 3 * blockIdx.x;   // item orders: no hop through wi
  const int No[3] = {od[0], od[1], od[2]};
  const int np[3] = {No[0] + 1, No[1] + 1, No[2] + 1};
  const int n = np[0] * np[1] * np[2];
  // Mortar plans: the warp-per-side pass reads its face layers as strided
  // gathers (8.5 sectors moved per sector used when read from global memory);
  // the item's slots are contiguous in Q, so one TMA bulk copy stages them in
  // shared memory instead (16-byte aligned span, data `shift` doubles in).
  const bool staged = coupled && P.nmface != 0;
  int shift = 0;
  if (staged) {
    const double* src = Q + P.node_off[wi.x] * NV;
    shift = static_cast<int>((reinterpret_cast<unsigned long long>(src) & 15ull) >> 3);
    if (threadIdx.x == 0) {
      mbar_init(&qbar, 1);
      mbar_fence_init();
      const unsigned long long a = reinterpret_cast<unsigned long long>(src);
      const unsigned long long lo = a & ~15ull, hi = (a + 8ull * NV * n * wi.y + 15ull) & ~15ull;
      mbar_expect_tx(&qbar, static_cast<uint32_t>(hi - lo));
      bulk_g2s(qsm, reinterpret_cast<const void*>(lo), static_cast<uint32_t>(hi - lo), &qbar);
    }
  }
  for (int u = threadIdx.x; u < 48; u += blockDim.x)
    sb[u / 16][u % 16] = P.tables[OFF_BND + sel3(u / 16, No[0], No[1], No[2]) * 16 + (u % 16)];
  __syncthreads();   // tables staged; mbarrier initialised before anyone waits on it
  const int strides[3] = {1, np[0], np[0] * np[1]};
  if (!coupled || P.nmface == 0) {
    // every side on own-order traces: (element, side, face node) flattened
    // over the block, so small faces do not leave warps mostly idle
    const int nfs[3] = {np[1] * np[2], np[0] * np[2], np[0] * np[1]};
    const int per_e = 2 * (nfs[0] + nfs[1] + nfs[2]);
    const bool lgl = P.family == 1;
    for (int u = threadIdx.x; u < wi.y * per_e; u += blockDim.x) {
      const int e = u / per_e;
      int r = u - e * per_e, s = 0;
      while (r >= sel3(s >> 1, nfs[0], nfs[1], nfs[2])) {
        r -= sel3(s >> 1, nfs[0], nfs[1], nfs[2]);
        ++s;
      }
      int d, a, b;
      side_dirs(s, d, a, b);
      const int na = sel3(a, np[0], np[1], np[2]), nf = sel3(d, nfs[0], nfs[1], nfs[2]);
      const int nd = sel3(d, np[0], np[1], np[2]);
      const int ib = r / na, ia = r - ib * na;
      const int slot = wi.x + e;
      const double* q = Q + P.node_off[slot] * NV + ia * sel3(a, strides[0], strides[1], strides[2]) +
                        ib * sel3(b, strides[0], strides[1], strides[2]);
      double* dst = P.qtr + P.side_off[slot * 6 + s] * NV + r;
      const int sd = sel3(d, strides[0], strides[1], strides[2]);
      const double* row = sb[d] + (s & 1) * 8;
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        double acc;
        if (lgl) {
          acc = q[(long long)c * n + ((s & 1) ? (nd - 1) * sd : 0)];
        } else {
          acc = 0.0;
          for (int m = 0; m < nd; ++m) acc += row[m] * q[(long long)c * n + m * sd];
        }
        dst[(long long)c * nf] = acc;
      }
    }
    return;
  }
  mbar_wait(&qbar, 0);
  item_side_traces<NV>(P, wi.x, wi.y, coupled, np, strides, sb, P.qtr, P.qtrm,
                       [&](int e, int c, int off) { return qsm[shift + (e * NV + c) * n + off]; });
}

// Branch-free surface gather for LGL items with at least two nodes per
// direction: in a direction a node lies on at most one side, so each direction
// contributes ONE unconditional strided read of C values — from the side's
// surface array with weight l w_a w_b, or from a dummy address with weight 0
// and stride 0 (interior of that direction).  The three directions' loads are
// independent and issue together; the six-branch loop serialises a memory
// round trip per side a warp touches (config 3: lift 0.69 -> 0.63 ms, flux
// 0.35 -> 0.33 ms).  add(c, x) receives weight * value in direction order (the
// order of the loop form).
template <int C, class Add>
__device__ __forceinline__ void lgl_surface_gather(const DevPlan& P, const ElemTables& T,
                                                   const double* surf, int slot, int i, int j, int k,
                                                   int n1p, int n2p, int n3p, Add add) {
  const double* sp[3];
  double lw[3];
  int st[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int a = (d == 0) ? 1 : 0, b = (d == 2) ? 1 : 2;
    const int id = sel3(d, i, j, k), nd = sel3(d, n1p, n2p, n3p);
    const int ia = sel3(a, i, j, k), ib = sel3(b, i, j, k), na = sel3(a, n1p, n2p, n3p);
    const bool hi = id == nd - 1, on = hi || id == 0;
    const int nf = na * sel3(b, n1p, n2p, n3p);
    const double l = T.bnd[d][(hi ? 8 : 0) + id];
    lw[d] = on ? l * T.w[a][ia] * T.w[b][ib] : 0.0;
    st[d] = on ? nf : 0;
    sp[d] = on ? surf + P.side_off[slot * 6 + 2 * d + (hi ? 1 : 0)] * C + (ia + na * ib) : surf;
  }
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const double x0 = sp[0][(long long)c * st[0]], x1 = sp[1][(long long)c * st[1]],
                 x2 = sp[2][(long long)c * st[2]];
    add(c, lw[0] * x0);
    add(c, lw[1] * x1);
    add(c, lw[2] * x2);
  }
}

// BR1 lifted gradient at one node (operators.py:224-265): the volume part
// −Σ_i WD_i(g Ja^i) from the staged g (and Ja on curved items), plus the
// gathered surface contributions, times M⁻¹.  Shared by both lift kernels.
// Staged g* form of an item's conforming interior sides (k_vol_lift_own):
// sf[c][u], c < NGV: g*; c = NGV + d: n_d sigma (signed for this side), at
// u = e * per_e + (side prefix) + face node; on[e * 6 + side] != 0 marks the
// sides it serves.
struct SurfStage {
  const double* sf;
  const unsigned char* on;
  int nfi, per_e;
};

template <int LAW, int NX, int GSTAR = 0>
__device__ __forceinline__ void lift_node(const DevPlan& P, const ElemTables& T, const double* gs,
                                          const double* js, bool aff, int tot, int n, int n1p,
                                          int n2p, int n3p, int e, int node, int slot, int i, int j,
                                          int k, double* out /* [3 NGV] */,
                                          const SurfStage& SS = SurfStage{nullptr, nullptr, 0, 0}) {
  using L = Law<LAW>;
  constexpr int NGV = L::NGV, NG = 3 * NGV;
  const int eb = e * n;
  double acc[NG];
#pragma unroll
  for (int c = 0; c < NG; ++c) acc[c] = 0.0;
  if (aff) {
    // reference-space weak derivatives of g (the tangential weights wo_i are
    // applied with the constant metric transform), then that transform
    double W[3][NGV];
#pragma unroll
    for (int c = 0; c < 3 * NGV; ++c) W[c / NGV][c % NGV] = 0.0;
#pragma unroll
    for (int m = 0; m < (NX >= 0 ? NX + 1 : 8); ++m) {
      if (NX < 0 && m >= n1p) break;
      const int idx = eb + m + n1p * (j + n2p * k);
      const double dw = T.dh[0][m * 8 + i];
#pragma unroll
      for (int kk = 0; kk < NGV; ++kk) W[0][kk] += dw * gs[kk * tot + idx];
    }
#pragma unroll
    for (int m = 0; m < (NX >= 0 ? NX + 1 : 8); ++m) {
      if (NX < 0 && m >= n2p) break;
      const int idx = eb + i + n1p * (m + n2p * k);
      const double dw = T.dh[1][m * 8 + j];
#pragma unroll
      for (int kk = 0; kk < NGV; ++kk) W[1][kk] += dw * gs[kk * tot + idx];
    }
#pragma unroll
    for (int m = 0; m < (NX >= 0 ? NX + 1 : 8); ++m) {
      if (NX < 0 && m >= n3p) break;
      const int idx = eb + i + n1p * (j + n2p * m);
      const double dw = T.dh[2][m * 8 + k];
#pragma unroll
      for (int kk = 0; kk < NGV; ++kk) W[2][kk] += dw * gs[kk * tot + idx];
    }
    const double* mj = P.metrics + P.metric_off[slot] + 1;   // Ja^i_d at [3 i + d]
    const double wi_ = T.w[0][i], wj_ = T.w[1][j], wk_ = T.w[2][k];
    const double wo3[3] = {wj_ * wk_, wi_ * wk_, wi_ * wj_};
#pragma unroll
    for (int ii = 0; ii < 3; ++ii) {
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double ja = mj[3 * ii + d] * wo3[ii];
#pragma unroll
        for (int kk = 0; kk < NGV; ++kk) acc[d * NGV + kk] -= ja * W[ii][kk];
      }
    }
  } else {
    {
      const double wo = T.w[1][j] * T.w[2][k];
      for (int m = 0; m < n1p; ++m) {
        const int idx = eb + m + n1p * (j + n2p * k);
        const double dw = T.dh[0][m * 8 + i] * wo;
  #pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double ja = js[(0 * 3 + d) * tot + idx] * dw;
  #pragma unroll
          for (int kk = 0; kk < NGV; ++kk) acc[d * NGV + kk] -= ja * gs[kk * tot + idx];
        }
      }
    }
    {
      const double wo = T.w[0][i] * T.w[2][k];
      for (int m = 0; m < n2p; ++m) {
        const int idx = eb + i + n1p * (m + n2p * k);
        const double dw = T.dh[1][m * 8 + j] * wo;
  #pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double ja = js[(1 * 3 + d) * tot + idx] * dw;
  #pragma unroll
          for (int kk = 0; kk < NGV; ++kk) acc[d * NGV + kk] -= ja * gs[kk * tot + idx];
        }
      }
    }
    {
      const double wo = T.w[0][i] * T.w[1][j];
      for (int m = 0; m < n3p; ++m) {
        const int idx = eb + i + n1p * (j + n2p * m);
        const double dw = T.dh[2][m * 8 + k] * wo;
  #pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double ja = js[(2 * 3 + d) * tot + idx] * dw;
  #pragma unroll
          for (int kk = 0; kk < NGV; ++kk) acc[d * NGV + kk] -= ja * gs[kk * tot + idx];
        }
      }
    }
  }
  // surface scatter of the lift contributions
  const int ijk[3] = {i, j, k};
  const int np[3] = {n1p, n2p, n3p};
  const bool fast = GSTAR == 0 && NX < 0 && P.family == 1 && n1p > 1 && n2p > 1 && n3p > 1;
  if (fast)
    lgl_surface_gather<NG>(P, T, P.lsurf, slot, i, j, k, n1p, n2p, n3p,
                           [&](int c, double x) { acc[c] += x; });
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    if (fast) break;
    int d, a, b;
    side_dirs(s, d, a, b);
    const double l = T.bnd[d][(s & 1) * 8 + ijk[d]];
    if (l == 0.0) continue;
    const int nf = np[a] * np[b];
    const int kf = ijk[a] + np[a] * ijk[b];
    const double lw = l * T.w[a][ijk[a]] * T.w[b][ijk[b]];
    if (GSTAR == 2) {
      const int4 sn = P.side_nb[slot * 6 + s];
      if (sn.x >= 0) {
        // conforming interior side: g*·n σ from the face's g* (left frame)
        // and the left side's σ, n; negated on the right side (exactly the
        // values k_face<lift> would have stored for this side)
        int tl = kf;
        if ((sn.z >> 9) & 1) {
          const int M1 = sn.z & 7, M2 = (sn.z >> 3) & 7, orient = (sn.z >> 6) & 7;
          int ap, bp;
          if (orient & 4) {
            bp = kf % (M2 + 1);
            ap = kf / (M2 + 1);
          } else {
            ap = kf % (M1 + 1);
            bp = kf / (M1 + 1);
          }
          tl = ((orient & 1) ? M1 - ap : ap) + (M1 + 1) * ((orient & 2) ? M2 - bp : bp);
        }
        const double* gv = P.gsf + (long long)sn.x * NGV + tl;
        const double* geo = P.face_geo + sn.y + (((sn.z >> 10) & 1) ? 0 : tl);
        const double sg = ((sn.z >> 9) & 1) ? -geo[0] : geo[0];
        const double nrm[3] = {geo[nf], geo[2 * nf], geo[3 * nf]};
        double g[NGV];
#pragma unroll
        for (int kk = 0; kk < NGV; ++kk) g[kk] = gv[(long long)kk * nf];
#pragma unroll
        for (int d2 = 0; d2 < 3; ++d2)
#pragma unroll
          for (int kk = 0; kk < NGV; ++kk) acc[d2 * NGV + kk] += lw * (g[kk] * nrm[d2] * sg);
        continue;
      }
    }
    if (GSTAR == 1) {
      if (SS.on[e * 6 + s]) {
        // conforming interior side: g* and the side's signed n sigma, staged
        // per face node by the packed pass of k_vol_lift_own
        const int nf0 = n2p * n3p, nf1 = n1p * n3p;
        const int pre = s == 0 ? 0 : s == 1 ? nf0 : s == 2 ? 2 * nf0 : s == 3 ? 2 * nf0 + nf1
                      : s == 4 ? 2 * (nf0 + nf1) : 2 * (nf0 + nf1) + n1p * n2p;
        const double* sp = SS.sf + e * SS.per_e + pre + kf;
        double g[NGV], ns[3];
#pragma unroll
        for (int kk = 0; kk < NGV; ++kk) g[kk] = sp[kk * SS.nfi];
#pragma unroll
        for (int d2 = 0; d2 < 3; ++d2) ns[d2] = sp[(NGV + d2) * SS.nfi];
#pragma unroll
        for (int kk = 0; kk < NGV; ++kk) g[kk] *= lw;
#pragma unroll
        for (int d2 = 0; d2 < 3; ++d2)
#pragma unroll
          for (int kk = 0; kk < NGV; ++kk) acc[d2 * NGV + kk] += g[kk] * ns[d2];
        continue;
      }
    }
    const double* src = P.lsurf + P.side_off[slot * 6 + s] * NG + kf;
#pragma unroll
    for (int c = 0; c < NG; ++c) acc[c] += lw * src[(long long)c * nf];
  }
  int ms;
  const double* mp = metric_ptr(P, slot, node, n, ms);
  const double invm = 1.0 / (T.w[0][i] * T.w[1][j] * T.w[2][k] * mp[0]);
#pragma unroll
  for (int c = 0; c < NG; ++c) out[c] = acc[c] * invm;
}

// This thread's NPT nodes' state, loaded before the block's table barrier so
// that the loads are in flight while the spectral tables are staged.
template <int NV, class Div>
__device__ __forceinline__ void load_item_state(const DevPlan& P, const double* __restrict__ Q, int2 wi,
                                                int n, int tot, double (&q)[NPT][NV], const Div& dv) {
#pragma unroll
  for (int r = 0; r < NPT; ++r) {
    const int t = threadIdx.x + r * blockDim.x;
    if (t < tot) {
      const int e = dv.by_n(t), node = t - e * n;
      const long long base = P.node_off[wi.x + e] * NV;
#pragma unroll
      for (int v = 0; v < NV; ++v) q[r][v] = Q[base + (long long)v * n + node];
    }
  }
}

// Stage g(q) (and, on curved items, the 9 metric terms Ja) for the thread's
// nodes in shared memory.
template <int LAW, class Div>
__device__ __forceinline__ void stage_grad_vars(const DevPlan& P, int2 wi, int n, int tot, bool aff,
                                                const double (&q)[NPT][Law<LAW>::NV], double* gs,
                                                double* js, const Div& dv) {
  using L = Law<LAW>;
  constexpr int NGV = L::NGV;
#pragma unroll
  for (int r = 0; r < NPT; ++r) {
    const int t = threadIdx.x + r * blockDim.x;
    if (t < tot) {
      double g[NGV];
      L::grad_vars(P.prm, q[r], g);
#pragma unroll
      for (int k = 0; k < NGV; ++k) gs[k * tot + t] = g[k];
      if (!aff) {
        const int e = dv.by_n(t), node = t - e * n;
        int ms;
        const double* m = metric_ptr(P, wi.x + e, node, n, ms);
#pragma unroll
        for (int c = 0; c < 9; ++c) js[c * tot + t] = m[(1 + c) * ms];
      }
    }
  }
}

// Side and face node of the item-local face task u (u < E * per_e): tasks run
// element by element, side by side (0..5), face node by face node — the order
// of P.side_off, so u is also the node offset into the item's side arrays.
__device__ __forceinline__ void face_task(int u, int e, int per_e, int nf0, int nf1, int nf2, int& s,
                                          int& kf, int& nf) {
  int r = u - e * per_e;   // e = u / per_e, formed by the caller (ItemDiv)
  if (r < 2 * nf0) {
    s = r >= nf0;
    kf = r - s * nf0;
    nf = nf0;
  } else if (r < 2 * (nf0 + nf1)) {
    r -= 2 * nf0;
    s = 2 + (r >= nf1);
    kf = r - (s - 2) * nf1;
    nf = nf1;
  } else {
    r -= 2 * (nf0 + nf1);
    s = 4 + (r >= nf2);
    kf = r - (s - 4) * nf2;
    nf = nf2;
  }
}

// ---------------------------------------------------------------------------
// BR1 lift, volume part + scatter of the face contributions, times M^-1
// (operators.py:224-265); writes the gradient and its side traces.
//
// NX >= 0: compile-time isotropic order (the plan is one (NX,NX,NX) bucket),
// so index math folds and the contractions unroll; NX = -1: runtime orders.
// Work items whose elements are all affine take the reference-gradient path:
// -sum_i Ja^i_d WD_i(g) with the element's constant Ja (no per-node metrics).
template <int LAW, int NX>
__global__ void __launch_bounds__(VOL_THREADS, VOL_BLOCKS) k_vol_lift(DevPlan P, const double* __restrict__ Q,
                                                          int coupled) {
  using L = Law<LAW>;
  constexpr int NV = L::NV, NGV = L::NGV, NG = 3 * NGV;
  __shared__ ElemTables T;
  extern __shared__ double sm[];
  const int2 wi = P.work[blockIdx.x];
  const int* od = P.work_ord + 3 * blockIdx.x;   // item orders: no hop through wi
  const int N1 = NX >= 0 ? NX : od[0], N2 = NX >= 0 ? NX : od[1], N3 = NX >= 0 ? NX : od[2];
  const int n1p = N1 + 1, n2p = N2 + 1, n3p = N3 + 1;
  const int n = n1p * n2p * n3p, tot = wi.y * n;
  const ItemDiv<NX> dv(P.work_mul + 8 * blockIdx.x, n, n1p, n2p, n3p);
  double qa[NPT][NV];
  PHASE_DECL;
  PHASE_T(0);
  load_item_state<NV>(P, Q, wi, n, tot, qa, dv);
  prefetch_item_surface<NG>(P, P.lsurf, wi, N1, N2);
  if (P.pf_item) prefetch_item_metrics(P, wi, n, 32);
  load_tables(P, N1, N2, N3, T);
  const bool aff = P.work_aff[blockIdx.x] != 0;
  double* gs = sm;               // [NGV][tot]
  double* js = sm + NGV * tot;   // [9][tot]  (curved items only)
  // staging needs no table: one barrier covers both
  stage_grad_vars<LAW>(P, wi, n, tot, aff, qa, gs, js, dv);
  PHASE_T(1);
  __syncthreads();
  PHASE_T(2);
  // one node at a time: the gradient goes straight to P.grad (always stored
  // when the lift runs), so no value is held across a barrier
#pragma unroll 1
  for (int t = threadIdx.x; t < tot; t += blockDim.x) {
    const int e = dv.by_n(t), node = t - e * n, slot = wi.x + e;
    int i, j, k;
    dv.ijk(node, i, j, k);
    double x[NG];
    lift_node<LAW, NX>(P, T, gs, js, aff, tot, n, n1p, n2p, n3p, e, node, slot, i, j, k, x);
    const long long gb = P.node_off[slot] * NG;
#pragma unroll
    for (int c = 0; c < NG; ++c) P.grad[gb + (long long)c * n + node] = x[c];
  }
  PHASE_T(3);
  __syncthreads();   // the block's gradient stores are visible to the block
  PHASE_T(4);
  // viscous traces on the six sides (own order, or mortar order when
  // nonconforming), the gradient read back through L2
  const int np[3] = {n1p, n2p, n3p};
  const int strides[3] = {1, n1p, n1p * n2p};
  auto Gvol = [&](int e, int c, int off) {
    return __ldcg(P.grad + P.node_off[wi.x + e] * NG + (long long)c * n + off);
  };
  if constexpr (L::FVTR) {
    // (a) packed over the item's face nodes, one thread per (side, face node):
    // the side's own F_v.n sigma.  Sides on own-order traces store it; the
    // nonconforming sides of a coupled evaluation leave it in shared memory
    // (over the metric staging, dead by now) for (b).  A warp-per-side pass
    // would walk ~5 dependent memory round trips per side with most lanes idle.
    constexpr int NTR = L::NTR;
    const bool lgl = P.family == 1;
    const int nf0 = n2p * n3p, nf1 = n1p * n3p, nf2 = n1p * n2p;
    const int per_e = 2 * (nf0 + nf1 + nf2), nfi = wi.y * per_e;
    double* fvs = sm + NGV * tot;   // [NTR][nfi]
    const long long so0 = P.side_off[wi.x * 6];
    for (int u = threadIdx.x; u < nfi; u += blockDim.x) {
      int s, kf, nf;
      const int e = dv.by_per_e(u);
      face_task(u, e, per_e, nf0, nf1, nf2, s, kf, nf);
      const int slot = wi.x + e;
      int d, a, b;
      side_dirs(s, d, a, b);
      const int na = sel3(a, n1p, n2p, n3p), nd = sel3(d, n1p, n2p, n3p);
      const int sd = sel3(d, strides[0], strides[1], strides[2]);
      const int ib = d == 0 ? dv.by_n2p(kf) : dv.by_n1p(kf), ia = kf - ib * na;
      const int off0 = ia * sel3(a, strides[0], strides[1], strides[2]) +
                       ib * sel3(b, strides[0], strides[1], strides[2]);
      const int fl = P.side_flags[slot * 6 + s];
      const int4 si = P.side_info[slot * 6 + s];
      const long long so = so0 + u - kf;
      double gv[NGV], G3[3][NGV], fv[NTR], sigma, nrm[3];
      if (lgl) {
        const int off = off0 + ((s & 1) ? (nd - 1) * sd : 0);
#pragma unroll
        for (int c = 0; c < NG; ++c) G3[c / NGV][c % NGV] = Gvol(e, c, off);
#pragma unroll
        for (int kk = 0; kk < NGV; ++kk) gv[kk] = gs[kk * tot + e * n + off];
      } else {
        const double* row = T.bnd[d] + (s & 1) * 8;
#pragma unroll
        for (int kk = 0; kk < NGV; ++kk) gv[kk] = 0.0;
#pragma unroll
        for (int c = 0; c < NG; ++c) G3[c / NGV][c % NGV] = 0.0;
        for (int m = 0; m < nd; ++m) {
          const double r = row[m];
#pragma unroll
          for (int kk = 0; kk < NGV; ++kk) gv[kk] += r * gs[kk * tot + e * n + off0 + m * sd];
#pragma unroll
          for (int c = 0; c < NG; ++c) G3[c / NGV][c % NGV] += r * Gvol(e, c, off0 + m * sd);
        }
      }
      side_geometry(P, so, nf, kf, (fl >> 4) & 1, sigma, nrm);
      L::side_visc(P.prm, gv, G3, nrm, sigma, coupled ? (fl & 15) - 1 : -1, fv);
      if (coupled && (si.x & 1)) {
#pragma unroll
        for (int c = 0; c < NTR; ++c) fvs[c * nfi + u] = fv[c];
      } else {
        double* dst = P.gtr + so * NTR + kf;
#pragma unroll
        for (int c = 0; c < NTR; ++c) dst[(long long)c * nf] = fv[c];
      }
    }
    if (coupled && P.nmface > 0) {
      PHASE_T(5);
      __syncthreads();
      PHASE_T(6);
      // (b) one warp per nonconforming side: interpolate its values onto the
      // side's mortar (own frame) on the FP64 tensor cores
      const int warp = threadIdx.x >> 5;
      for (int task = warp; task < wi.y * 6; task += blockDim.x >> 5) {
        const int e = task / 6, s = task - 6 * e;
        const int4 si = P.side_info[(wi.x + e) * 6 + s];
        if (!(si.x & 1)) continue;
        int d, a, b;
        side_dirs(s, d, a, b);
        const int na = sel3(a, n1p, n2p, n3p), nb = sel3(b, n1p, n2p, n3p);
        int ma, mb;
        side_mortar_dims(si, ma, mb);
        const int nm = ma * mb;
        const int ub = e * per_e + (d == 0 ? 0 : d == 1 ? 2 * nf0 : 2 * (nf0 + nf1)) + (s & 1) * na * nb;
        const double* T1 = P.tables + OFF_T + ((na - 1) * 8 + (ma - 1)) * 64;
        const double* T2 = P.tables + OFF_T + ((nb - 1) * 8 + (mb - 1)) * 64;
        double* dst = P.gtrm + (long long)si.w * NTR;
        warp_proj_mma<NTR>(na, nb, T1, ma, T2, mb,
                           [&](int c, int ia, int ib) { return fvs[c * nfi + ub + ia + na * ib]; }, dst, nm,
                           [&](int A, int B) { return A + ma * B; });
      }
    }
  } else {
    item_side_traces<NG>(P, wi.x, wi.y, coupled, np, strides, T.bnd, P.gtr, P.gtrm, Gvol);
  }
  PHASE_T(7);
  PHASE_END(0, 8);
}

// BR1 lift for LGL plans whose evaluated sides all use own-order traces (no
// nonconforming face, or an isolated evaluation): the side traces of G are
// face-node values.  Three passes over the work item:
//   1. (g* form) packed over the item's face nodes, one thread per (side,
//      face node): g* and the side's signed n sigma go to shared memory, so
//      the per-node surface terms below are a few shared loads (in a warp of
//      consecutive volume nodes only a few lanes lie on any one side: the
//      gathers, orientation index math and geometry loads would otherwise
//      run at an eighth of the lanes, once per side the warp touches);
//   2. one thread per node: volume part + surface terms, times M^-1 -> grad;
//   3. packed over the face nodes again: each side's viscous trace (Navier-
//      Stokes: its own F_v.n sigma) from the gradient just written (read
//      back through L2) and the staged lifted variables.
template <int LAW, int NX>
__global__ void __launch_bounds__(VOL_THREADS, VOL_BLOCKS) k_vol_lift_own(DevPlan P, const double* __restrict__ Q,
                                                                   int coupled) {
  using L = Law<LAW>;
  constexpr int NV = L::NV, NGV = L::NGV, NG = 3 * NGV;
  __shared__ ElemTables T;
  __shared__ unsigned char side_on[MAX_ITEM_ELEMS * 6];
  extern __shared__ double sm[];
  const int2 wi = P.work[blockIdx.x];
  const int* od = P.work_ord + 3 * blockIdx.x;   // item orders: no hop through wi
  const int N1 = NX >= 0 ? NX : od[0], N2 = NX >= 0 ? NX : od[1], N3 = NX >= 0 ? NX : od[2];
  const int n1p = N1 + 1, n2p = N2 + 1, n3p = N3 + 1;
  const int n = n1p * n2p * n3p, tot = wi.y * n;
  const ItemDiv<NX> dv(P.work_mul + 8 * blockIdx.x, n, n1p, n2p, n3p);
  const int nf0 = n2p * n3p, nf1 = n1p * n3p, nf2 = n1p * n2p;
  const int per_e = 2 * (nf0 + nf1 + nf2), nfi = wi.y * per_e;
  const bool gst = coupled && P.gstar;
  double qa[NPT][NV];
  __shared__ unsigned long long qbar;
  // [sf: (NGV + 3) x nfi, g* form only] [gs: NGV x tot] [js: 9 x tot | TMA Q]
  double* sf = sm;
  double* gs = sm + (gst ? (((NGV + 3) * nfi + 1) & ~1) : 0);   // [NGV][tot], 16-byte aligned
  double* js = gs + NGV * tot;                                    // [9][tot]  (curved items only)
  const bool tma = P.tma_q != 0;
  double* qs = gs + ((NGV * tot + 1) & ~1);   // 16-byte aligned bulk-copy destination
  int shift = 0;
  if (tma) {
    // the item's slots are contiguous in Q: one bulk copy of [nv][n] x E
    // (16-byte aligned span; data starts `shift` doubles in) into shared
    // memory after the g region, while the tables and g* are staged
    const long long n0 = P.node_off[wi.x];
    const double* src = Q + n0 * NV;
    shift = static_cast<int>((reinterpret_cast<unsigned long long>(src) & 15ull) >> 3);
    if (threadIdx.x == 0) {
      mbar_init(&qbar, 1);
      mbar_fence_init();
      const unsigned long long a = reinterpret_cast<unsigned long long>(src);
      const unsigned long long lo = a & ~15ull, hi = (a + 8ull * NV * tot + 15ull) & ~15ull;
      mbar_expect_tx(&qbar, static_cast<uint32_t>(hi - lo));
      bulk_g2s(qs, reinterpret_cast<const void*>(lo), static_cast<uint32_t>(hi - lo), &qbar);
    }
  } else {
    load_item_state<NV>(P, Q, wi, n, tot, qa, dv);
    if (P.pf_item) prefetch_item_metrics(P, wi, n, 32);
  }
  if (!gst) prefetch_item_surface<NG>(P, P.lsurf, wi, N1, N2);
  if (gst) {
    // pass 1: g* and n sigma of the conforming interior sides
    for (int u = threadIdx.x; u < nfi; u += blockDim.x) {
      int s, kf, nf;
      const int e = dv.by_per_e(u);
      face_task(u, e, per_e, nf0, nf1, nf2, s, kf, nf);
      const int4 sn = P.side_nb[(wi.x + e) * 6 + s];
      if (kf == 0) side_on[e * 6 + s] = sn.x >= 0;
      if (sn.x < 0) continue;
      int tl = kf;
      if ((sn.z >> 9) & 1) {
        // right side: its face node in the left frame
        const int M1 = sn.z & 7, M2 = (sn.z >> 3) & 7, orient = (sn.z >> 6) & 7;
        int ap, bp;
        if (orient & 4) {
          bp = kf % (M2 + 1);
          ap = kf / (M2 + 1);
        } else {
          ap = kf % (M1 + 1);
          bp = kf / (M1 + 1);
        }
        tl = ((orient & 1) ? M1 - ap : ap) + (M1 + 1) * ((orient & 2) ? M2 - bp : bp);
      }
      const double* gv = P.gsf + (long long)sn.x * NGV + tl;
      const double* geo = P.face_geo + sn.y + (((sn.z >> 10) & 1) ? 0 : tl);
      const double sg = ((sn.z >> 9) & 1) ? -geo[0] : geo[0];
#pragma unroll
      for (int kk = 0; kk < NGV; ++kk) sf[kk * nfi + u] = gv[(long long)kk * nf];
#pragma unroll
      for (int d2 = 0; d2 < 3; ++d2) sf[(NGV + d2) * nfi + u] = geo[(1 + d2) * nf] * sg;
    }
  }
  load_tables(P, N1, N2, N3, T);
  if (tma) {
    __syncthreads();   // mbarrier initialised before anyone waits on it
    mbar_wait(&qbar, 0);
#pragma unroll
    for (int r = 0; r < NPT; ++r) {
      const int t = threadIdx.x + r * blockDim.x;
      if (t < tot) {
        const int e = dv.by_n(t), node = t - e * n;
#pragma unroll
        for (int v = 0; v < NV; ++v) qa[r][v] = qs[shift + (e * NV + v) * n + node];
      }
    }
  }
  const bool aff = P.work_aff[blockIdx.x] != 0;
  // staging needs no table: one barrier covers both
  stage_grad_vars<LAW>(P, wi, n, tot, aff, qa, gs, js, dv);
  __syncthreads();
  const SurfStage SS{sf, side_on, nfi, per_e};
  // pass 2
#pragma unroll 1
  for (int t = threadIdx.x; t < tot; t += blockDim.x) {
    const int e = dv.by_n(t), node = t - e * n, slot = wi.x + e;
    int i, j, k;
    dv.ijk(node, i, j, k);
    double x[NG];
    if (gst)
      lift_node<LAW, NX, 1>(P, T, gs, js, aff, tot, n, n1p, n2p, n3p, e, node, slot, i, j, k, x, SS);
    else
      lift_node<LAW, NX>(P, T, gs, js, aff, tot, n, n1p, n2p, n3p, e, node, slot, i, j, k, x);
    if (P.grad) {
      const long long gb = P.node_off[slot] * NG;
#pragma unroll
      for (int c = 0; c < NG; ++c) P.grad[gb + (long long)c * n + node] = x[c];
    }
    if constexpr (!L::FVTR) {
      // scalar laws: the side traces are the gradient's face-node values
      const int ijk[3] = {i, j, k};
      const int np[3] = {n1p, n2p, n3p};
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        int d, a, b;
        side_dirs(s, d, a, b);
        if (ijk[d] != ((s & 1) ? np[d] - 1 : 0)) continue;
        const int nf = np[a] * np[b];
        const int kf = ijk[a] + np[a] * ijk[b];
        double* dst = P.gtr + P.side_off[slot * 6 + s] * NG + kf;
#pragma unroll
        for (int c = 0; c < NG; ++c) dst[(long long)c * nf] = x[c];
      }
    }
  }
  if constexpr (L::FVTR) {
    // pass 3: this side's own F_v.n sigma at each face node (LGL: the traces
    // are the node's own lifted variables and gradient)
    __syncthreads();   // the block's gradient stores are visible to the block
    const long long so0 = P.side_off[wi.x * 6];
    for (int u = threadIdx.x; u < nfi; u += blockDim.x) {
      int s, kf, nf;
      const int e = dv.by_per_e(u);
      face_task(u, e, per_e, nf0, nf1, nf2, s, kf, nf);
      const int slot = wi.x + e;
      int d, a, b;
      side_dirs(s, d, a, b);
      const int na = sel3(a, n1p, n2p, n3p), nd = sel3(d, n1p, n2p, n3p);
      const int ib = d == 0 ? dv.by_n2p(kf) : dv.by_n1p(kf), ia = kf - ib * na;
      const int off = ia * sel3(a, 1, n1p, n1p * n2p) + ib * sel3(b, 1, n1p, n1p * n2p) +
                      ((s & 1) ? (nd - 1) * sel3(d, 1, n1p, n1p * n2p) : 0);
      const long long so = so0 + u - kf;
      const int fl = P.side_flags[slot * 6 + s];
      double sigma, nrm[3], gv[NGV], G3[3][NGV], fv[L::NTR];
      const double* gp = P.grad + P.node_off[slot] * NG + off;
#pragma unroll
      for (int c = 0; c < NG; ++c) G3[c / NGV][c % NGV] = __ldcg(gp + (long long)c * n);
      side_geometry(P, so, nf, kf, (fl >> 4) & 1, sigma, nrm);
#pragma unroll
      for (int kk = 0; kk < NGV; ++kk) gv[kk] = gs[kk * tot + e * n + off];
      L::side_visc(P.prm, gv, G3, nrm, sigma, coupled ? (fl & 15) - 1 : -1, fv);
      double* dst = P.gtr + so * L::NTR + kf;
#pragma unroll
      for (int c = 0; c < L::NTR; ++c) dst[(long long)c * nf] = fv[c];
    }
  }
}

// In-loop variant of k_vol_lift_own for low orders (P.lift_packed == 0):
// every node gathers its sides' g* and geometry itself and writes its own
// side traces.  With more face nodes than volume nodes per element (N <= 3)
// the two packed passes of k_vol_lift_own cost more than the divergence they
// remove (config 5, N = 3 curved: V-cycle 26.2 ms in-loop, 28.1 ms packed;
// config 4, N = 7: lift 0.59 ms in-loop, 0.55 ms packed).  No staging of G in shared memory and no second barrier,
// so each thread keeps one node's values at a time (80 registers, 3 blocks
// per SM: measured faster than 4 blocks with spills at 64).
template <int LAW, int NX>
__global__ void __launch_bounds__(VOL_THREADS, VOL_BLOCKS) k_vol_lift_own_inl(DevPlan P, const double* __restrict__ Q,
                                                                   int coupled) {
  using L = Law<LAW>;
  constexpr int NV = L::NV, NGV = L::NGV, NG = 3 * NGV;
  __shared__ ElemTables T;
  extern __shared__ double sm[];
  const int2 wi = P.work[blockIdx.x];
  const int* od = P.work_ord + 3 * blockIdx.x;   // item orders: no hop through wi
  const int N1 = NX >= 0 ? NX : od[0], N2 = NX >= 0 ? NX : od[1], N3 = NX >= 0 ? NX : od[2];
  const int n1p = N1 + 1, n2p = N2 + 1, n3p = N3 + 1;
  const int n = n1p * n2p * n3p, tot = wi.y * n;
  const ItemDiv<NX> dv(P.work_mul + 8 * blockIdx.x, n, n1p, n2p, n3p);
  double qa[NPT][NV];
  __shared__ unsigned long long qbar;
  double* gs = sm;               // [NGV][tot]
  double* js = sm + NGV * tot;   // [9][tot]  (curved items only)
  const bool tma = P.tma_q != 0;
  if (tma) {
    // the item's slots are contiguous in Q: one bulk copy of [nv][n] x E
    // (16-byte aligned span; data starts `shift` doubles in) into shared
    // memory after the g region, while the tables are staged
    double* qs = sm + ((NGV * tot + 1) & ~1);   // 16-byte aligned destination
    const long long n0 = P.node_off[wi.x];
    const double* src = Q + n0 * NV;
    const int shift = static_cast<int>((reinterpret_cast<unsigned long long>(src) & 15ull) >> 3);
    if (threadIdx.x == 0) {
      mbar_init(&qbar, 1);
      mbar_fence_init();
      const unsigned long long a = reinterpret_cast<unsigned long long>(src);
      const unsigned long long lo = a & ~15ull, hi = (a + 8ull * NV * tot + 15ull) & ~15ull;
      mbar_expect_tx(&qbar, static_cast<uint32_t>(hi - lo));
      bulk_g2s(qs, reinterpret_cast<const void*>(lo), static_cast<uint32_t>(hi - lo), &qbar);
    }
    if (coupled && P.gstar)
      prefetch_item_gstar<NGV>(P, wi, N1, N2, N3);
    else
      prefetch_item_surface<NG>(P, P.lsurf, wi, N1, N2);
    load_tables(P, N1, N2, N3, T);
    __syncthreads();   // mbarrier initialised before anyone waits on it
    mbar_wait(&qbar, 0);
#pragma unroll
    for (int r = 0; r < NPT; ++r) {
      const int t = threadIdx.x + r * blockDim.x;
      if (t < tot) {
        const int e = dv.by_n(t), node = t - e * n;
#pragma unroll
        for (int v = 0; v < NV; ++v) qa[r][v] = qs[shift + (e * NV + v) * n + node];
      }
    }
  } else {
    load_item_state<NV>(P, Q, wi, n, tot, qa, dv);
    if (coupled && P.gstar)
      prefetch_item_gstar<NGV>(P, wi, N1, N2, N3);
    else
      prefetch_item_surface<NG>(P, P.lsurf, wi, N1, N2);
    if (P.pf_item) prefetch_item_metrics(P, wi, n, 32);
    load_tables(P, N1, N2, N3, T);
  }
  const bool aff = P.work_aff[blockIdx.x] != 0;
  // staging needs no table: one barrier covers both
  stage_grad_vars<LAW>(P, wi, n, tot, aff, qa, gs, js, dv);
  __syncthreads();
#pragma unroll 1
  for (int t = threadIdx.x; t < tot; t += blockDim.x) {
    const int e = dv.by_n(t), node = t - e * n, slot = wi.x + e;
    int i, j, k;
    dv.ijk(node, i, j, k);
    double x[NG];
    if (coupled && P.gstar)
      lift_node<LAW, NX, 2>(P, T, gs, js, aff, tot, n, n1p, n2p, n3p, e, node, slot, i, j, k, x);
    else
      lift_node<LAW, NX>(P, T, gs, js, aff, tot, n, n1p, n2p, n3p, e, node, slot, i, j, k, x);
    if (P.grad) {
      const long long gb = P.node_off[slot] * NG;
#pragma unroll
      for (int c = 0; c < NG; ++c) P.grad[gb + (long long)c * n + node] = x[c];
    }
    const int ijk[3] = {i, j, k};
    const int np[3] = {n1p, n2p, n3p};
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      int d, a, b;
      side_dirs(s, d, a, b);
      if (ijk[d] != ((s & 1) ? np[d] - 1 : 0)) continue;
      const int nf = np[a] * np[b];
      const int kf = ijk[a] + np[a] * ijk[b];
      const long long so = P.side_off[slot * 6 + s];
      if constexpr (L::FVTR) {
        // this side's own F_v.n sigma at the node (LGL: the traces are the
        // node's own lifted variables and gradient)
        const int fl = P.side_flags[slot * 6 + s];
        double sigma, nrm[3], gv[NGV], G3[3][NGV], fv[L::NTR];
        side_geometry(P, so, nf, kf, (fl >> 4) & 1, sigma, nrm);
#pragma unroll
        for (int kk = 0; kk < NGV; ++kk) gv[kk] = gs[kk * tot + t];
#pragma unroll
        for (int c = 0; c < NG; ++c) G3[c / NGV][c % NGV] = x[c];
        L::side_visc(P.prm, gv, G3, nrm, sigma, coupled ? (fl & 15) - 1 : -1, fv);
        double* dst = P.gtr + so * L::NTR + kf;
#pragma unroll
        for (int c = 0; c < L::NTR; ++c) dst[(long long)c * nf] = fv[c];
      } else {
        double* dst = P.gtr + so * NG + kf;
#pragma unroll
        for (int c = 0; c < NG; ++c) dst[(long long)c * nf] = x[c];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Flux divergence + surface scatter + epilogue (operators.py:283-290, 337-364;
// timestep.py:100-112 for MODE_RK).
struct FluxArgs {
  const double* S;     // source (nullable)
  const double* X;     // additive term for MODE_A (nullable)
  double* out;         // output field (MODE_F/A/R) or tau by element id (MODE_TAU)
  double* W;           // RK register
  double* Qout;        // RK: updated state (== Q)
  const double* dt;
  int local;
  int stage;
  double rk_a, rk_b;
  double* norm;        // max |r|
  int* nonfinite;
  int traces;          // RK: also write the new state's own-order Q traces (LGL, conforming)
  int coupled;         // coupled (1) or isolated (0) evaluation (the lift's surface terms)
};

template <int LAW, int MODE, int NX>
__global__ void __launch_bounds__(VOL_THREADS, VOL_BLOCKS) k_vol_flux(DevPlan P, const double* Q, FluxArgs A) {
  using L = Law<LAW>;
  constexpr int NV = L::NV, NGV = L::NGV, NG = 3 * NGV;
  __shared__ ElemTables T;
  extern __shared__ double sm[];
  const int2 wi = P.work[blockIdx.x];
  const int* od = P.work_ord + 3 * blockIdx.x;   // item orders: no hop through wi
  const int N1 = NX >= 0 ? NX : od[0], N2 = NX >= 0 ? NX : od[1], N3 = NX >= 0 ? NX : od[2];
  prefetch_item_surface<NV>(P, P.fsurf, wi, N1, N2);
  // epilogue inputs, read after the contraction
  if (MODE != MODE_F) prefetch_item_nodes<NV>(P, MODE == MODE_A ? A.X : A.S, wi, 32);
  if (MODE == MODE_RK && A.stage != 0) prefetch_item_nodes<NV>(P, A.W, wi, 64);
  if (P.pf_item) {
    // the item's state and gradient spans, read node by node below (the
    // second node of each thread only after the first one's flux)
    prefetch_item_nodes<NV>(P, Q, wi, 96);
    if (L::viscous(P.prm)) prefetch_item_nodes<NG>(P, P.grad, wi, 128);
    prefetch_item_metrics(P, wi, (N1 + 1) * (N2 + 1) * (N3 + 1), 160);
  }
  const int n1p = N1 + 1, n2p = N2 + 1, n3p = N3 + 1;
  const int n = n1p * n2p * n3p, tot = wi.y * n;
  const ItemDiv<NX> dv(P.work_mul + 8 * blockIdx.x, n, n1p, n2p, n3p);
  double* ft = sm;   // [3][NV][tot]
  const bool visc = L::viscous(P.prm);
  PHASE_DECL;
  PHASE_T(0);
  // the contravariant fluxes need no table: they are formed first, the
  // tables are staged after them, and one barrier covers both
#pragma unroll 1
  for (int r = 0; r < NPT; ++r) {
    const int t = threadIdx.x + r * blockDim.x;
    if (t < tot) {
      const int e = dv.by_n(t), node = t - e * n, slot = wi.x + e;
      const long long base = P.node_off[slot] * NV;
      double q[NV], f[3][NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) q[v] = Q[base + (long long)v * n + node];
      L::adv_flux(P.prm, q, f);
      if (visc) {
        double G[3][NGV];
        const double* gp = P.grad + P.node_off[slot] * NG + node;
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int k = 0; k < NGV; ++k) G[d][k] = gp[(long long)(d * NGV + k) * n];
        L::sub_visc(P.prm, q, G, f);
      }
      int ms;
      const double* m = metric_ptr(P, slot, node, n, ms);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double j0 = m[(1 + 3 * i) * ms], j1 = m[(2 + 3 * i) * ms], j2 = m[(3 + 3 * i) * ms];
#pragma unroll
        for (int v = 0; v < NV; ++v)
          ft[(i * NV + v) * tot + t] = j0 * f[0][v] + j1 * f[1][v] + j2 * f[2][v];
      }
    }
  }
  load_tables(P, N1, N2, N3, T);
  PHASE_T(1);
  __syncthreads();
  PHASE_T(2);
  double rmax = 0.0;
#pragma unroll 1
  for (int r = 0; r < NPT; ++r) {
    const int t = threadIdx.x + r * blockDim.x;
    if (t < tot) {
      const int e = dv.by_n(t), node = t - e * n, slot = wi.x + e;
      int i, j, k;
    dv.ijk(node, i, j, k);
      const int eb = e * n;
      double F[NV], F0[NV], F1[NV], F2[NV];   // per-direction chains (ILP)
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        F[v] = 0.0;
        F0[v] = F1[v] = F2[v] = 0.0;
      }
      {
#pragma unroll
        for (int m = 0; m < (NX >= 0 ? NX + 1 : 8); ++m) {
          if (NX < 0 && m >= n1p) break;
          const int idx = eb + m + n1p * (j + n2p * k);
          const double dw = T.dh[0][m * 8 + i];
#pragma unroll
          for (int v = 0; v < NV; ++v) F0[v] += dw * ft[(0 * NV + v) * tot + idx];
        }
        const double wo = T.w[1][j] * T.w[2][k];
#pragma unroll
        for (int v = 0; v < NV; ++v) F0[v] *= wo;
      }
      {
#pragma unroll
        for (int m = 0; m < (NX >= 0 ? NX + 1 : 8); ++m) {
          if (NX < 0 && m >= n2p) break;
          const int idx = eb + i + n1p * (m + n2p * k);
          const double dw = T.dh[1][m * 8 + j];
#pragma unroll
          for (int v = 0; v < NV; ++v) F1[v] += dw * ft[(1 * NV + v) * tot + idx];
        }
        const double wo = T.w[0][i] * T.w[2][k];
#pragma unroll
        for (int v = 0; v < NV; ++v) F1[v] *= wo;
      }
      {
#pragma unroll
        for (int m = 0; m < (NX >= 0 ? NX + 1 : 8); ++m) {
          if (NX < 0 && m >= n3p) break;
          const int idx = eb + i + n1p * (j + n2p * m);
          const double dw = T.dh[2][m * 8 + k];
#pragma unroll
          for (int v = 0; v < NV; ++v) F2[v] += dw * ft[(2 * NV + v) * tot + idx];
        }
        const double wo = T.w[0][i] * T.w[1][j];
#pragma unroll
        for (int v = 0; v < NV; ++v) F2[v] *= wo;
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) F[v] -= (F0[v] + F1[v]) + F2[v];
      const int ijk[3] = {i, j, k};
      const int np[3] = {n1p, n2p, n3p};
      // (runtime-order plans only: measured slower than the branches at every
      // compile-time order of config 4, where whole warps are interior)
      const bool fast = NX < 0 && P.family == 1 && n1p > 1 && n2p > 1 && n3p > 1;
      if (fast)
        lgl_surface_gather<NV>(P, T, P.fsurf, slot, i, j, k, n1p, n2p, n3p,
                               [&](int c, double x) { F[c] += x; });
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        if (fast) break;
        int d, a, b;
        side_dirs(s, d, a, b);
        const double l = T.bnd[d][(s & 1) * 8 + ijk[d]];
        if (l == 0.0) continue;
        const int nf = np[a] * np[b];
        const int kf = ijk[a] + np[a] * ijk[b];
        const double lw = l * T.w[a][ijk[a]] * T.w[b][ijk[b]];
        const double* src = P.fsurf + P.side_off[slot * 6 + s] * NV + kf;
#pragma unroll
        for (int v = 0; v < NV; ++v) F[v] += lw * src[(long long)v * nf];
      }
      const long long base = P.node_off[slot] * NV + node;
      int ms;
      const double* mp = metric_ptr(P, slot, node, n, ms);
      const double mass = T.w[0][i] * T.w[1][j] * T.w[2][k] * mp[0];
      const double invm = 1.0 / mass;
      if (MODE == MODE_F) {
#pragma unroll
        for (int v = 0; v < NV; ++v) A.out[base + (long long)v * n] = F[v];
      } else if (MODE == MODE_A) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double a = F[v] * invm;
          if (A.X) a += A.X[base + (long long)v * n];
          A.out[base + (long long)v * n] = a;
        }
      } else if (MODE == MODE_R) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double s = A.S ? A.S[base + (long long)v * n] : 0.0;
          const double rv = s - F[v] * invm;
          if (A.out) A.out[base + (long long)v * n] = rv;
          rmax = nanmax(rmax, fabs(rv));
        }
      } else if (MODE == MODE_RK) {
        const double dtv0 = A.local ? A.dt[slot] : A.dt[0];
        // no time scale (dt = +inf): leave Q untouched; the caller raises
        // TimeScaleError as the reference does before stepping (timestep.py:133)
        const double dtv = isinf(dtv0) && dtv0 > 0.0 ? 0.0 : dtv0;
        bool bad = false;
        double qn[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const long long ix = base + (long long)v * n;
          const double s = A.S ? A.S[ix] : 0.0;
          const double rv = s - F[v] * invm;
          rmax = nanmax(rmax, fabs(rv));
          const double wv = (A.stage == 0) ? rv : A.rk_a * A.W[ix] + rv;
          A.W[ix] = wv;
          qn[v] = A.Qout[ix] + A.rk_b * dtv * wv;
          A.Qout[ix] = qn[v];
          bad |= !isfinite(qn[v]);
        }
        if (bad && A.nonfinite) *A.nonfinite = 1;
        if (A.traces) {
          // LGL face nodes: the next stage's own-order Q traces (k_trace_q skipped)
          const int ijk[3] = {i, j, k};
          const int np[3] = {n1p, n2p, n3p};
#pragma unroll
          for (int sd = 0; sd < 6; ++sd) {
            int d, a, b;
            side_dirs(sd, d, a, b);
            if (ijk[d] != ((sd & 1) ? np[d] - 1 : 0)) continue;
            const int nf = np[a] * np[b];
            double* dst = P.qtr + P.side_off[slot * 6 + sd] * NV + ijk[a] + np[a] * ijk[b];
#pragma unroll
            for (int v = 0; v < NV; ++v) dst[(long long)v * nf] = qn[v];
          }
        }
      } else if (MODE == MODE_TAU) {
        double tv = 0.0;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double s = A.S ? A.S[base + (long long)v * n] : 0.0;
          tv = nanmax(tv, fabs(mass * s - F[v]));
        }
        atomicMax(&T.emax[e], static_cast<unsigned long long>(__double_as_longlong(tv)));
      }
    }
  }
  PHASE_T(3);
  if (MODE == MODE_R || (MODE == MODE_RK)) {
    if (A.norm && (MODE == MODE_R || A.stage == 0)) block_max_to(rmax, A.norm, T.red);
  }
  PHASE_T(4);
  PHASE_END(8, 5);
  if (MODE == MODE_TAU) {
    __syncthreads();
    for (int e = threadIdx.x; e < wi.y; e += blockDim.x)
      atomic_max_nonneg(A.out + P.elem_id[wi.x + e], __longlong_as_double((long long)T.emax[e]));
  }
}

// ---------------------------------------------------------------------------
// per-element pseudo-time step (timestep.py:40-66)
template <int LAW>
__global__ void __launch_bounds__(ELEM_THREADS) k_element_dt(DevPlan P, const double* __restrict__ Q,
                                                             double cfl_a, double cfl_v,
                                                             double* dt_slot, double* dt_min) {
  using L = Law<LAW>;
  constexpr int NV = L::NV;
  __shared__ unsigned long long smax[MAX_ITEM_ELEMS];
  const int2 wi = P.work[blockIdx.x];
  const int* od = P.work_ord + 3 * blockIdx.x;   // item orders: no hop through wi
  const int No[3] = {od[0], od[1], od[2]};
  const int n = (No[0] + 1) * (No[1] + 1) * (No[2] + 1), tot = wi.y * n;
  const ItemDiv<-1> dv(P.work_mul + 8 * blockIdx.x, n, No[0] + 1, No[1] + 1, No[2] + 1);
  for (int u = threadIdx.x; u < MAX_ITEM_ELEMS; u += blockDim.x) smax[u] = 0ull;
  __syncthreads();
  for (int t = threadIdx.x; t < tot; t += blockDim.x) {
    const int e = dv.by_n(t), node = t - e * n, slot = wi.x + e;
    const long long base = P.node_off[slot] * NV;
    double q[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) q[v] = Q[base + (long long)v * n + node];
    const double s = L::wave_speed(P.prm, q);
    atomicMax(&smax[e], static_cast<unsigned long long>(__double_as_longlong(nanmax(s, 0.0))));
  }
  __syncthreads();
  const double mu = P.prm[7];
  for (int e = threadIdx.x; e < wi.y; e += blockDim.x) {
    const int slot = wi.x + e;
    const double sm = __longlong_as_double((long long)smax[e]);
    double dt = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      // collapsed directions (order 0 on every element) carry no time scale;
      // any other direction uses max(N_d, 1) (timestep.py:55)
      if ((P.collapsed >> d) & 1) continue;
      const double nn = (double)(No[d] > 1 ? No[d] : 1);
      const double h = P.sizes[slot * 3 + d];
      if (sm > 0.0) dt = fmin(dt, cfl_a * h / (sm * nn * nn));
      if (mu > 0.0) dt = fmin(dt, cfl_v * h * h / (mu * nn * nn * nn * nn));
    }
    if (sm != sm) dt = sm;   // NaN state propagates
    if (dt_slot) dt_slot[slot] = dt;
    if (dt_min) atomic_min_nonneg(dt_min, dt);
  }
}

// ---------------------------------------------------------------------------
// max |X| over everything and per element; non-finite flag (fields.py:144-162)
template <int NV>
__global__ void __launch_bounds__(ELEM_THREADS) k_norm(DevPlan P, const double* __restrict__ X,
                                                       double* gmax, double* emax_out, int* flag) {
  __shared__ unsigned long long emax[MAX_ITEM_ELEMS];
  __shared__ double red[32];
  const int2 wi = P.work[blockIdx.x];
  const int* od = P.work_ord + 3 * blockIdx.x;   // item orders: no hop through wi
  const int n = (od[0] + 1) * (od[1] + 1) * (od[2] + 1), tot = wi.y * n;
  const ItemDiv<-1> dv(P.work_mul + 8 * blockIdx.x, n, od[0] + 1, od[1] + 1, od[2] + 1);
  for (int u = threadIdx.x; u < MAX_ITEM_ELEMS; u += blockDim.x) emax[u] = 0ull;
  __syncthreads();
  double m = 0.0;
  bool bad = false;
  for (int t = threadIdx.x; t < tot; t += blockDim.x) {
    const int e = dv.by_n(t), node = t - e * n, slot = wi.x + e;
    const long long base = P.node_off[slot] * NV + node;
    double em = 0.0;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const double x = X[base + (long long)v * n];
      em = nanmax(em, fabs(x));
      bad |= !isfinite(x);
    }
    m = nanmax(m, em);
    if (emax_out) atomicMax(&emax[e], static_cast<unsigned long long>(__double_as_longlong(em)));
  }
  if (bad && flag) *flag = 1;
  if (gmax) block_max_to(m, gmax, red);
  if (emax_out) {
    __syncthreads();
    for (int e = threadIdx.x; e < wi.y; e += blockDim.x)
      emax_out[P.elem_id[wi.x + e]] = __longlong_as_double((long long)emax[e]);
  }
}

// ---------------------------------------------------------------------------
// truncation_from_avalue (operators.py:355-360): tau[elem] = max over nodes and
// unknowns of |M (S - A)|, M = w_i w_j w_k J as in the MODE_TAU epilogue.
template <int NV>
__global__ void __launch_bounds__(ELEM_THREADS) k_tau_avalue(DevPlan P, const double* __restrict__ A,
                                                             const double* __restrict__ S, double* tau) {
  __shared__ unsigned long long emax[MAX_ITEM_ELEMS];
  __shared__ double w[3][8];
  const int2 wi = P.work[blockIdx.x];
  const int* od = P.work_ord + 3 * blockIdx.x;
  const int n1p = od[0] + 1, n2p = od[1] + 1, n = n1p * n2p * (od[2] + 1), tot = wi.y * n;
  const ItemDiv<-1> dv(P.work_mul + 8 * blockIdx.x, n, n1p, n2p, od[2] + 1);
  for (int u = threadIdx.x; u < MAX_ITEM_ELEMS; u += blockDim.x) emax[u] = 0ull;
  for (int u = threadIdx.x; u < 24; u += blockDim.x)
    w[u / 8][u % 8] = P.tables[OFF_W + sel3(u / 8, od[0], od[1], od[2]) * 8 + (u % 8)];
  __syncthreads();
  for (int t = threadIdx.x; t < tot; t += blockDim.x) {
    const int e = dv.by_n(t), node = t - e * n, slot = wi.x + e;
    int i, j, k;
    dv.ijk(node, i, j, k);
    int ms;
    const double* mp = metric_ptr(P, slot, node, n, ms);
    const double mass = w[0][i] * w[1][j] * w[2][k] * mp[0];
    const long long base = P.node_off[slot] * NV + node;
    double tv = 0.0;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const long long ix = base + (long long)v * n;
      const double s = S ? S[ix] : 0.0;
      tv = nanmax(tv, fabs(mass * (s - A[ix])));
    }
    atomicMax(&emax[e], static_cast<unsigned long long>(__double_as_longlong(tv)));
  }
  __syncthreads();
  for (int e = threadIdx.x; e < wi.y; e += blockDim.x)
    tau[P.elem_id[wi.x + e]] = __longlong_as_double((long long)emax[e]);
}

}  // namespace tdg
