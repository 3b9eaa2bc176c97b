// geometry.cuh — device construction of the invariant-curl volume metrics
// (the host path is paper_1806_11456_b200/geometry.py
// volume_metrics, the reference's mesh.py:132-164 in 3D).
//
// One block per element.  The control-node map is interpolated to the
// solution nodes, moved to the element-local origin (the curl form is
// translation invariant), differentiated by collocation, and the metric terms
// are formed in the conservative curl form
//     Ja^i_n = -1/2 (D_j (X_l dX_m/dxi_k - X_m dX_l/dxi_k) - D_k (... j ...)),
// (i, j, k) cyclic, (n, m, l) cyclic; J = a_1 . (a_2 x a_3) from the
// collocated derivatives a_d = dX/dxi_d, and the directional sizes
// h_d = sum w |a_d| / 4.  Outputs use the host's (ξ-slowest) array layouts so
// the plan builder consumes them unchanged.
//
// Bit-identical to the oracle (oracle/geometry.py) and the product's host
// path: every sum runs in the same fixed order, multiplies and adds are
// separately rounded (__dmul_rn / __dadd_rn: no FMA contraction), the local
// origin is node 0 and the size sums run sequentially in node order — the
// metric round-off otherwise moves an M = 0.1 residual by ~1e-12 relative
// (DESIGN.md §3), the parity bar itself.
#pragma once
#include "common.cuh"

namespace tdg {

constexpr int GEO_THREADS = 256;

// tables: [3][8][4] interpolation ctrl -> nodes (row i, col a: stride 4),
//         [3][64]   collocation derivative at the nodes (row i, col m: stride 8),
//         [3][8]    quadrature weights
struct GeoTables {
  double L[3][8][4];
  double D[3][64];
  double w[3][8];
};

__global__ void __launch_bounds__(GEO_THREADS) k_volume_metrics(const double* __restrict__ ctrl, int a1, int a2,
                                                                int a3, int n1p, int n2p, int n3p,
                                                                const GeoTables* __restrict__ tab, double* jac,
                                                                double* ja, double* coords, double* sizes) {
  extern __shared__ double sm[];
  __shared__ GeoTables T;
  const int e = blockIdx.x;
  const int n = n1p * n2p * n3p;
  for (int u = threadIdx.x; u < (int)(sizeof(GeoTables) / sizeof(double)); u += blockDim.x)
    reinterpret_cast<double*>(&T)[u] = reinterpret_cast<const double*>(tab)[u];
  __syncthreads();
  double* X = sm;            // [3][n]
  double* g = sm + 3 * n;    // [3 c][3 k][n]: dX_c / dxi_k
  double* V = sm + 12 * n;   // [3][n]
  const double* cp = ctrl + (long long)e * a1 * a2 * a3 * 3;
  const int st[3] = {n2p * n3p, n3p, 1};   // node (i, j, k), k fastest
  // 1. map the control nodes to the solution nodes: x = sum_abc ((L1 L2) L3) p
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const int i = t / st[0], j = (t / n3p) % n2p, k = t % n3p;
    double x[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < a1; ++a)
      for (int b = 0; b < a2; ++b) {
        const double lab = __dmul_rn(T.L[0][i][a], T.L[1][j][b]);
        for (int c = 0; c < a3; ++c) {
          const double l = __dmul_rn(lab, T.L[2][k][c]);
          const double* p = cp + ((a * a2 + b) * a3 + c) * 3;
          x[0] = __dadd_rn(x[0], __dmul_rn(l, p[0]));
          x[1] = __dadd_rn(x[1], __dmul_rn(l, p[1]));
          x[2] = __dadd_rn(x[2], __dmul_rn(l, p[2]));
        }
      }
    for (int c = 0; c < 3; ++c) {
      X[c * n + t] = x[c];
      coords[((long long)e * n + t) * 3 + c] = x[c];
    }
  }
  __syncthreads();
  // element-local origin: node 0 (the curl form is translation invariant)
  double org[3];
  for (int c = 0; c < 3; ++c) org[c] = X[c * n];
  __syncthreads();
  for (int t = threadIdx.x; t < n; t += blockDim.x)
    for (int c = 0; c < 3; ++c) X[c * n + t] = __dsub_rn(X[c * n + t], org[c]);
  __syncthreads();
  // 2. collocated derivatives g[c][k] = D_k X_c
  const int np[3] = {n1p, n2p, n3p};
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const int ijk[3] = {t / st[0], (t / n3p) % n2p, t % n3p};
    for (int kd = 0; kd < 3; ++kd) {
      const int base = t - ijk[kd] * st[kd];
      for (int c = 0; c < 3; ++c) {
        double s = 0.0;
        for (int m = 0; m < np[kd]; ++m)
          s = __dadd_rn(s, __dmul_rn(T.D[kd][ijk[kd] * 8 + m], X[c * n + base + m * st[kd]]));
        g[(c * 3 + kd) * n + t] = s;
      }
    }
  }
  __syncthreads();
  // 3. J and |a_d| w (staged in V for the ordered size sums) from
  //    a_d = (g[0][d], g[1][d], g[2][d])
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const int i = t / st[0], j = (t / n3p) % n2p, k = t % n3p;
    double a[3][3];
    for (int d = 0; d < 3; ++d)
      for (int c = 0; c < 3; ++c) a[d][c] = g[(c * 3 + d) * n + t];
    const double cx = __dsub_rn(__dmul_rn(a[1][1], a[2][2]), __dmul_rn(a[1][2], a[2][1]));
    const double cy = __dsub_rn(__dmul_rn(a[1][2], a[2][0]), __dmul_rn(a[1][0], a[2][2]));
    const double cz = __dsub_rn(__dmul_rn(a[1][0], a[2][1]), __dmul_rn(a[1][1], a[2][0]));
    jac[(long long)e * n + t] =
        __dadd_rn(__dadd_rn(__dmul_rn(a[0][0], cx), __dmul_rn(a[0][1], cy)), __dmul_rn(a[0][2], cz));
    const double www = __dmul_rn(__dmul_rn(T.w[0][i], T.w[1][j]), T.w[2][k]);
    for (int d = 0; d < 3; ++d) {
      const double nrm = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(a[d][0], a[d][0]), __dmul_rn(a[d][1], a[d][1])),
                                        __dmul_rn(a[d][2], a[d][2])));
      V[d * n + t] = __dmul_rn(www, nrm);
    }
  }
  __syncthreads();
  if (threadIdx.x < 3) {   // sequential in node order, as the oracle's loop
    double s = 0.0;
    for (int t = 0; t < n; ++t) s = __dadd_rn(s, V[threadIdx.x * n + t]);
    sizes[e * 3 + threadIdx.x] = s / 4.0;
  }
  // 4. curl-form metric terms, one physical component n at a time
  for (int nn = 0; nn < 3; ++nn) {
    const int mm = (nn + 1) % 3, ll = (nn + 2) % 3;
    __syncthreads();
    for (int t = threadIdx.x; t < n; t += blockDim.x)
      for (int kd = 0; kd < 3; ++kd)
        V[kd * n + t] = __dsub_rn(__dmul_rn(X[ll * n + t], g[(mm * 3 + kd) * n + t]),
                                  __dmul_rn(X[mm * n + t], g[(ll * 3 + kd) * n + t]));
    __syncthreads();
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const int ijk[3] = {t / st[0], (t / n3p) % n2p, t % n3p};
      for (int i = 0; i < 3; ++i) {
        const int j = (i + 1) % 3, k = (i + 2) % 3;
        // D_j V_k
        double s1 = 0.0, s2 = 0.0;
        {
          const int base = t - ijk[j] * st[j];
          for (int m = 0; m < np[j]; ++m)
            s1 = __dadd_rn(s1, __dmul_rn(T.D[j][ijk[j] * 8 + m], V[k * n + base + m * st[j]]));
        }
        {
          const int base = t - ijk[k] * st[k];
          for (int m = 0; m < np[k]; ++m)
            s2 = __dadd_rn(s2, __dmul_rn(T.D[k][ijk[k] * 8 + m], V[j * n + base + m * st[k]]));
        }
        ja[(((long long)e * 3 + i) * 3 + nn) * n + t] = __dmul_rn(-0.5, __dsub_rn(s1, s2));
      }
    }
  }
}

}  // namespace tdg
