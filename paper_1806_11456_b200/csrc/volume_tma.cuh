// volume_tma.cuh — persistent, TMA-pipelined flux-divergence kernel.
//
// One 512-thread block per SM walks the work items (runs of same-shape
// elements, <= 512 nodes, contiguous slots).  For each item the element
// state Q and the lifted gradient G are single contiguous spans in HBM; one
// thread issues two cp.async.bulk copies into a shared-memory buffer that
// completes on an mbarrier, while the block computes the previous item from
// the other buffer (double buffering).  The surface contributions, S and the
// RK register are loaded into registers before the block barrier so their
// latency overlaps the pointwise flux work.  Arithmetic is identical to
// k_vol_flux (volume.cuh): f~ = Ja (f_a - f_v), F = -WD(f~) + scatter, then
// the MODE epilogue.
#pragma once
#include "common.cuh"
#include "laws.cuh"
#include "volume.cuh"

namespace tdg {

constexpr int TMA_THREADS = 512;

template <int NV, int NG>
constexpr int tma_flux_smem_doubles() {
  return 2 * ((NV * MAXN + 2) + (NG * MAXN + 2)) + 3 * NV * MAXN;
}

template <int LAW, int MODE, int NX>
__global__ void __launch_bounds__(TMA_THREADS, 1) k_vol_flux_tma(DevPlan P, const double* Q, FluxArgs A) {
  using L = Law<LAW>;
  constexpr int NV = L::NV, NGV = L::NGV, NG = 3 * NGV;
  constexpr int QB = NV * MAXN + 2, GB = NG * MAXN + 2;
  extern __shared__ __align__(16) double sm[];
  double* bufs = sm;                       // 2 x (QB + GB)
  double* ft = sm + 2 * (QB + GB);         // [3][NV][MAXN]
  __shared__ ElemTables T;
  __shared__ __align__(8) unsigned long long bar[2];
  __shared__ int s_off[2][2];
  const int tid = threadIdx.x;
  const bool visc = L::viscous(P.prm);

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();

  auto issue = [&](int item, int b) {   // single thread
    const int2 wi = P.work[item];
    const int* od = P.orders + 3 * wi.x;
    const long long n = (long long)(od[0] + 1) * (od[1] + 1) * (od[2] + 1);
    const long long base = P.node_off[wi.x];
    double* dst = bufs + b * (QB + GB);
    uint32_t tot = 0;
    s_off[b][0] = bulk_span(dst, Q + base * NV, n * wi.y * NV, &bar[b], tot);
    s_off[b][1] = visc ? bulk_span(dst + QB, P.grad + base * NG, n * wi.y * NG, &bar[b], tot) : 0;
    mbar_expect_tx(&bar[b], tot);
  };

  int item = blockIdx.x;
  if (item < P.nwork && tid == 0) issue(item, 0);
  int cur = -1;
  double rmax = 0.0;

  for (int it = 0; item < P.nwork; item += gridDim.x, ++it) {
    const int b = it & 1;
    const int next = item + gridDim.x;
    if (next < P.nwork && tid == 0) issue(next, b ^ 1);   // that buffer was released at the end of it-1
    const int2 wi = P.work[item];
    const int* od = P.orders + 3 * wi.x;
    const int N1 = NX >= 0 ? NX : od[0], N2 = NX >= 0 ? NX : od[1], N3 = NX >= 0 ? NX : od[2];
    const int key = N1 | (N2 << 4) | (N3 << 8);
    if (key != cur) {                      // block-uniform: reload tables on a shape change
      load_tables(P, N1, N2, N3, T);
      cur = key;
    } else if (MODE == MODE_TAU) {
      for (int u = tid; u < 64; u += blockDim.x) T.emax[u] = 0ull;
    }
    __syncthreads();
    const int n1p = N1 + 1, n2p = N2 + 1, n3p = N3 + 1;
    const int n = n1p * n2p * n3p, tot = wi.y * n;
    const int t = tid;
    const bool active = t < tot;
    const int e = active ? t / n : 0, node = t - e * n, slot = wi.x + e;
    const int i = node % n1p, j = (node / n1p) % n2p, k = node / (n1p * n2p);

    // ---- loads that do not depend on the staged state: surface, S, W ----
    double Fs[NV], Sv[NV], Wv[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) Fs[v] = Sv[v] = Wv[v] = 0.0;
    const long long gbase = P.node_off[slot] * NV + node;
    if (active) {
      const int ijk[3] = {i, j, k};
      const int np[3] = {n1p, n2p, n3p};
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        int d, a, bb;
        side_dirs(s, d, a, bb);
        const double l = T.bnd[d][(s & 1) * 8 + ijk[d]];
        if (l == 0.0) continue;
        const int nf = np[a] * np[bb];
        const int kf = ijk[a] + np[a] * ijk[bb];
        const double lw = l * T.w[a][ijk[a]] * T.w[bb][ijk[bb]];
        const double* src = P.fsurf + P.side_off[slot * 6 + s] * NV + kf;
#pragma unroll
        for (int v = 0; v < NV; ++v) Fs[v] += lw * src[(long long)v * nf];
      }
      if ((MODE == MODE_R || MODE == MODE_RK || MODE == MODE_TAU) && A.S) {
#pragma unroll
        for (int v = 0; v < NV; ++v) Sv[v] = A.S[gbase + (long long)v * n];
      }
      if (MODE == MODE_A && A.X) {
#pragma unroll
        for (int v = 0; v < NV; ++v) Sv[v] = A.X[gbase + (long long)v * n];
      }
      if (MODE == MODE_RK && A.stage != 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) Wv[v] = A.W[gbase + (long long)v * n];
      }
    }

    // ---- staged element state ----
    mbar_wait(&bar[b], (it >> 1) & 1);
    const double* qs = bufs + b * (QB + GB) + s_off[b][0] + (long long)e * n * NV + node;
    const double* gsm = bufs + b * (QB + GB) + QB + s_off[b][1] + (long long)e * n * NG + node;
    double q[NV];
    if (active) {
#pragma unroll
      for (int v = 0; v < NV; ++v) q[v] = qs[v * n];
      double f[3][NV];
      L::adv_flux(P.prm, q, f);
      if (visc) {
        double G[3][NGV];
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int kk = 0; kk < NGV; ++kk) G[d][kk] = gsm[(d * NGV + kk) * n];
        L::sub_visc(P.prm, q, G, f);
      }
      int ms;
      const double* m = metric_ptr(P, slot, node, n, ms);
#pragma unroll
      for (int ii = 0; ii < 3; ++ii) {
        const double j0 = m[(1 + 3 * ii) * ms], j1 = m[(2 + 3 * ii) * ms], j2 = m[(3 + 3 * ii) * ms];
#pragma unroll
        for (int v = 0; v < NV; ++v)
          ft[(ii * NV + v) * MAXN + t] = j0 * f[0][v] + j1 * f[1][v] + j2 * f[2][v];
      }
    }
    __syncthreads();

    if (active) {
      const int eb = e * n;
      double F[NV], F0[NV], F1[NV], F2[NV];   // per-direction chains (ILP)
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        F[v] = Fs[v];
        F0[v] = F1[v] = F2[v] = 0.0;
      }
      {
        const double wo = T.w[1][j] * T.w[2][k];
#pragma unroll
        for (int mm = 0; mm < (NX >= 0 ? NX + 1 : 8); ++mm) {
          if (NX < 0 && mm >= n1p) break;
          const int idx = eb + mm + n1p * (j + n2p * k);
          const double dw = T.dh[0][mm * 8 + i] * wo;
#pragma unroll
          for (int v = 0; v < NV; ++v) F0[v] += dw * ft[(0 * NV + v) * MAXN + idx];
        }
      }
      {
        const double wo = T.w[0][i] * T.w[2][k];
#pragma unroll
        for (int mm = 0; mm < (NX >= 0 ? NX + 1 : 8); ++mm) {
          if (NX < 0 && mm >= n2p) break;
          const int idx = eb + i + n1p * (mm + n2p * k);
          const double dw = T.dh[1][mm * 8 + j] * wo;
#pragma unroll
          for (int v = 0; v < NV; ++v) F1[v] += dw * ft[(1 * NV + v) * MAXN + idx];
        }
      }
      {
        const double wo = T.w[0][i] * T.w[1][j];
#pragma unroll
        for (int mm = 0; mm < (NX >= 0 ? NX + 1 : 8); ++mm) {
          if (NX < 0 && mm >= n3p) break;
          const int idx = eb + i + n1p * (j + n2p * mm);
          const double dw = T.dh[2][mm * 8 + k] * wo;
#pragma unroll
          for (int v = 0; v < NV; ++v) F2[v] += dw * ft[(2 * NV + v) * MAXN + idx];
        }
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) F[v] -= (F0[v] + F1[v]) + F2[v];
      int ms;
      const double* mp = metric_ptr(P, slot, node, n, ms);
      const double mass = T.w[0][i] * T.w[1][j] * T.w[2][k] * mp[0];
      const double invm = 1.0 / mass;
      if (MODE == MODE_F) {
#pragma unroll
        for (int v = 0; v < NV; ++v) A.out[gbase + (long long)v * n] = F[v];
      } else if (MODE == MODE_A) {
#pragma unroll
        for (int v = 0; v < NV; ++v) A.out[gbase + (long long)v * n] = F[v] * invm + Sv[v];
      } else if (MODE == MODE_R) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double rv = Sv[v] - F[v] * invm;
          if (A.out) A.out[gbase + (long long)v * n] = rv;
          rmax = nanmax(rmax, fabs(rv));
        }
      } else if (MODE == MODE_RK) {
        const double dtv = A.local ? A.dt[slot] : A.dt[0];
        bool bad = false;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const long long ix = gbase + (long long)v * n;
          const double rv = Sv[v] - F[v] * invm;
          rmax = nanmax(rmax, fabs(rv));
          const double wv = (A.stage == 0) ? rv : A.rk_a * Wv[v] + rv;
          A.W[ix] = wv;
          const double qn = q[v] + A.rk_b * dtv * wv;
          A.Qout[ix] = qn;
          bad |= !isfinite(qn);
        }
        if (bad && A.nonfinite) *A.nonfinite = 1;
      } else if (MODE == MODE_TAU) {
        double tv = 0.0;
#pragma unroll
        for (int v = 0; v < NV; ++v) tv = nanmax(tv, fabs(mass * Sv[v] - F[v]));
        atomicMax(&T.emax[e], static_cast<unsigned long long>(__double_as_longlong(tv)));
      }
    }
    if (MODE == MODE_TAU) {
      __syncthreads();
      for (int ee = tid; ee < wi.y; ee += blockDim.x)
        atomic_max_nonneg(A.out + P.elem_id[wi.x + ee], __longlong_as_double((long long)T.emax[ee]));
    }
    __syncthreads();   // buffer b, ft and T free for the next item
  }
  if (MODE == MODE_R || MODE == MODE_RK) {
    if (A.norm && (MODE == MODE_R || A.stage == 0)) block_max_to(rmax, A.norm, T.red);
  }
}

}  // namespace tdg
