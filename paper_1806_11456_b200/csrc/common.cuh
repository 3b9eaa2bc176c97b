// common.cuh — device-side plan, table layout and reduction helpers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tdg {

// spectral table layout — must match paper_1806_11456_b200/spectral.py
constexpr int PAD = 8;
constexpr int OFF_DHAT = 0;
constexpr int OFF_W = OFF_DHAT + PAD * PAD * PAD;
constexpr int OFF_BND = OFF_W + PAD * PAD;
constexpr int OFF_T = OFF_BND + PAD * 2 * PAD;
constexpr int TABLES_LEN = OFF_T + PAD * PAD * PAD * PAD;

constexpr int ELEM_THREADS = 256;     // element kernels: 8 warps
constexpr int MAXN = 512;             // nodes per element work item (<= (7+1)^3)
#ifndef TDG_VOL_THREADS
#define TDG_VOL_THREADS 256
#endif
#ifndef TDG_VOL_BLOCKS
#define TDG_VOL_BLOCKS 3
#endif
constexpr int VOL_THREADS = TDG_VOL_THREADS;   // lift / flux kernels: threads per block ...
constexpr int VOL_BLOCKS = TDG_VOL_BLOCKS;     // ... and resident blocks per SM (register cap)
constexpr int NPT = MAXN / VOL_THREADS;        // nodes per thread of a full work item
constexpr int MAX_ITEM_ELEMS = 64;    // elements per work item (per-element smem reductions)
// k_vol_lift_own (g* form): face nodes of a work item whose g* and n sigma fit
// beside the item's staged state with three blocks per SM ((4 + 3) x 8 B each)
constexpr int LIFT_FACE_NODES = 768;
constexpr size_t LIFT_OWN_SMEM_3 = 72000;       // dynamic shared memory bound for 3 blocks / SM
constexpr int FACE_THREADS = 64;      // one interior face (<= 8x8 mortar nodes) per block
constexpr int FACE_THREADS_MAX = 128; // packed uniform faces: face_pack * face_nm <= 128
constexpr int SIDE_THREADS = 256;     // four element sides per block
constexpr int SIDES_PER_BLOCK = SIDE_THREADS / 64;

enum Mode { MODE_F = 0, MODE_A = 1, MODE_R = 2, MODE_RK = 3, MODE_TAU = 4 };

struct DevPlan {
  int law;
  int family;
  double prm[8];
  const double* tables;
  int nslots;
  const int* orders;
  const int* elem_id;
  const long long* node_off;
  const long long* metric_off;
  const int* affine;
  const double* metrics;
  const double* sizes;
  const long long* side_off;
  const double* side_geo;
  int nfaces;
  const int* face_info;
  const long long* face_geo_off;
  const double* face_geo;
  int nbfaces;
  const int* bface_info;
  const long long* ghost_off;
  const double* ghost;
  // element work items: (first slot, count), uniform orders inside an item
  int nwork;
  const int2* work;
  const int* work_aff;   // per work item: 1 if every element of the item is affine
  const int* work_ord;   // per work item: its (N1, N2, N3), read without waiting for work[]
  // per work item: multipliers m(d) = ceil(2^20 / d) for d = n, n1p, n2p,
  // n1p n2p and the face nodes per element, [8] per item (mdiv below)
  const int* work_mul;
  int nsm;        // SMs: kernels prefetch the work about one wave ahead (L2)
  int pf_trace, pf_face, pf_down;   // look-ahead distances, blocks per SM
  int pf_item;    // element kernels: L2 bulk prefetch of the item's own spans
  int tma_q;      // lift (own-order plans, every item affine): the item's Q span
                  // arrives in shared memory by one TMA bulk copy
  int collapsed;  // bit d: direction d has order 0 on every element (2D extrusion)
  // side work items for side kernels: (slot, side | kind<<8), ghost offset
  int nside_iso;
  const int4* side_iso;      // isolated: every side of every element
  int nside_bnd;
  const int4* side_bnd;      // coupled: boundary faces
  // per element side (slot*6+side): x = nonconforming-interior | is_right<<1 | orient<<2,
  // y = M1 | M2<<8 (mortar orders, left frame), z = face index (-1: boundary),
  // w = mortar-trace offset (nodes) of a nonconforming side
  const int4* side_info;
  // per interior face, two int4: [2f] = (left trace offset, right trace offset,
  // M1 | M2<<3 | orient<<6 | conforming<<9, face-geometry offset) (trace
  // offsets: own side arrays when conforming, mortar traces otherwise);
  // [2f+1] = (0, left side offset, right side offset,
  // L1 | L2<<3 | R1<<6 | R2<<9 aligned own orders)
  const int4* fdesc;
  int ncface, nmface;
  // k_face packing: when every conforming face has the same node count
  // face_nm, a block of face_threads evaluates face_pack = 128 / face_nm faces
  int face_pack, face_nm, face_threads;
  const int* cface;              // conforming interior faces (k_face)
  const int* mface;              // nonconforming interior faces (k_mortar)
  // scratch (device)
  double* qtrm;   // mortar-order Q traces of nonconforming sides (own frame)
  double* gtrm;   // mortar-order viscous traces of nonconforming sides ([ntr] per node)
  double* qtr;    // [side_nodes][nv] own-order Q traces
  double* lsurf;  // [side_nodes][3*ngv]   lift surface contributions
  // [side_nodes][ntr] own-order viscous traces: the gradient (scalar laws,
  // ntr = 3 ngv) or the side's own normal viscous flux F_v.n sigma with its
  // boundary treatment applied (Navier-Stokes, ntr = 4; Law::FVTR)
  double* gtr;
  // per element side (slot*6+side): bits 0-3 = boundary kind + 1 (0: interior
  // side), bit 4 = uniform own-order side geometry (node 0's values serve)
  const int* side_flags;
  double* fsurf;  // [side_nodes][nv]      flux surface contributions
  double* grad;   // [nodes][3*ngv] lifted gradient
  // conforming-face lift in g* form (LGL plans without nonconforming faces):
  // k_face<lift> writes g* = ½(g_L + g_R) once per face node ([ngv][nm] at
  // the left side's trace offset) instead of g*·n σ for both sides (2 x 3 ngv),
  // and k_vol_lift_own forms g*·n σ from it and the face geometry
  int gstar;
  int lift_packed;   // own-order lift: packed face-node passes (k_vol_lift_own) or in-loop (k_vol_lift_own_inl)
  double* gsf;    // [side_nodes][ngv] (left-side offsets used)
  // per element side (slot*6+side) of a conforming interior face: x = the
  // left side's trace offset (nodes; -1 otherwise), y = face-geometry
  // offset, z = M1 | M2<<3 | orient<<6 | is_right<<9 (left frame)
  const int4* side_nb;
};

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  // IEEE bit patterns of non-negative doubles order like the values (NaN above +inf)
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

__device__ __forceinline__ void atomic_min_nonneg(double* addr, double v) {
  atomicMin(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// NaN-propagating max of NON-NEGATIVE values (every caller passes |x| or a
// running maximum that starts at +0): the IEEE bit patterns of non-negative
// doubles order like the values and every NaN pattern lies above +inf, so an
// unsigned integer max does it in four integer instructions (fmax drops NaN;
// a compare-and-select on doubles costs two FP64-pipe compares per call, 7 %
// of the flux kernel's instructions at five calls per node).
__device__ __forceinline__ double nanmax(double a, double b) {
  const unsigned long long x = static_cast<unsigned long long>(__double_as_longlong(a));
  const unsigned long long y = static_cast<unsigned long long>(__double_as_longlong(b));
  return __longlong_as_double(static_cast<long long>(x > y ? x : y));
}

__device__ __forceinline__ double warp_nanmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nanmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// block-wide NaN-propagating max of non-negative values -> one atomic per block
__device__ __forceinline__ void block_max_to(double v, double* out, double* red /*[32]*/) {
  v = warp_nanmax(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    double x = lane < nw ? red[lane] : 0.0;
    x = warp_nanmax(x);
    if (lane == 0 && out) atomic_max_nonneg(out, x);
  }
  __syncthreads();
}

// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col); per lane
// a = A[lane/4][lane%4], b = B[lane%4][lane/4], d = D[lane/4][2(lane%4) + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  // not volatile: a pure function of its operands, so independent components'
  // MMAs may be interleaved by the scheduler
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// One warp projects C component arrays of (na x nb) values to (ma x mb):
//   out[c][A, B] = sum_b T2[B][b] sum_a T1[A][a] in[c][a, b]      (T rows stride 8)
// on the FP64 tensor cores, one zero-padded 8x8 tile per component and pass:
// pass 1 (M = A, K = a, N = b) takes its B operand straight from ld(c, a, b).
// Its result tmp[A][b] leaves lane (g, q) holding tmp[g][2q] and tmp[g][2q+1],
// which are exactly the B operands B[k][n = g] of pass 2 (M = B, K = b, N = A)
// if its two k-steps run over the even and the odd b: step 0 pairs k = q with
// b = 2q, step 1 with b = 2q + 1, and T2 is read in the same order.  Nothing
// moves between lanes.  No shared memory, no __syncwarp; the whole warp must
// be converged.  Output (A, B) of component c is stored once, as
// out[c * cstride + idx(A, B)] (negated if NEG): the two offsets and their
// predicates of a lane are formed once, outside the component loop.
template <int C, bool NEG = false, class Load, class Index>
__device__ __forceinline__ void warp_proj_mma(int na, int nb, const double* __restrict__ T1, int ma,
                                              const double* __restrict__ T2, int mb, Load ld,
                                              double* __restrict__ out, long long cstride, Index idx) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const double t10 = (g < ma && q < na) ? T1[g * 8 + q] : 0.0;
  const double t11 = (g < ma && q + 4 < na) ? T1[g * 8 + q + 4] : 0.0;
  const double t20 = (g < mb && 2 * q < nb) ? T2[g * 8 + 2 * q] : 0.0;
  const double t21 = (g < mb && 2 * q + 1 < nb) ? T2[g * 8 + 2 * q + 1] : 0.0;
  const bool ka = na > 4, kb = nb > 1;
  const bool colv = g < nb;
  const bool p0 = g < mb && 2 * q < ma, p1 = g < mb && 2 * q + 1 < ma;
  double* const out0 = out + (p0 ? idx(2 * q, g) : 0);
  double* const out1 = out + (p1 ? idx(2 * q + 1, g) : 0);
#pragma unroll
  for (int c = 0; c < C; ++c) {
    double d0 = 0.0, d1 = 0.0;
    const double b0 = (colv && q < na) ? ld(c, q, g) : 0.0;
    const double b1 = (colv && ka && q + 4 < na) ? ld(c, q + 4, g) : 0.0;
    dmma_8x8x4(d0, d1, t10, b0);
    if (ka) dmma_8x8x4(d0, d1, t11, b1);
    double o0 = 0.0, o1 = 0.0;
    dmma_8x8x4(o0, o1, t20, d0);
    if (kb) dmma_8x8x4(o0, o1, t21, d1);
    if (p0) out0[c * cstride] = NEG ? -o0 : o0;
    if (p1) out1[c * cstride] = NEG ? -o1 : o1;
  }
}

// Bulk prefetch of a global span into L2 (one instruction, issued by one
// thread): loads that follow the span's first use then hit L2.
__device__ __forceinline__ void l2_prefetch_span(const void* p, size_t bytes) {
  if (bytes == 0) return;
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(static_cast<unsigned>(e - a))
               : "memory");
}

// x / d for 0 <= x <= 2048 and 1 <= d <= 512 as a multiply and a shift with
// m = ceil(2^20 / d) (exact: x (m d - 2^20) < 2^20).  A division by a runtime
// divisor costs ~20 instructions, three of them on the conversion pipe; the
// runtime-order kernels decompose node and face indices several times per node.
constexpr int MDIV_SHIFT = 20;
__host__ __device__ __forceinline__ int mdiv_mul(int d) { return ((1 << MDIV_SHIFT) + d - 1) / d; }
__device__ __forceinline__ int mdiv(int x, int m) {
  return static_cast<int>((static_cast<unsigned>(x) * static_cast<unsigned>(m)) >> MDIV_SHIFT);
}
// per-item divisors of the element kernels: compile-time orders divide by
// constants, runtime orders use the plan's multipliers
template <int NX>
struct ItemDiv {
  int n, n1p, n2p, n12, per_e;
  int mn, m1, m2, m12, mpe;
  __device__ __forceinline__ ItemDiv(const int* mul, int n_, int n1p_, int n2p_, int n3p_)
      : n(n_), n1p(n1p_), n2p(n2p_), n12(n1p_ * n2p_),
        per_e(2 * (n2p_ * n3p_ + n1p_ * n3p_ + n1p_ * n2p_)) {
    if (NX < 0) {
      mn = mul[0];
      m1 = mul[1];
      m2 = mul[2];
      m12 = mul[3];
      mpe = mul[4];
    } else {
      mn = m1 = m2 = m12 = mpe = 0;
    }
  }
  __device__ __forceinline__ int by_n(int x) const { return NX < 0 ? mdiv(x, mn) : x / n; }
  __device__ __forceinline__ int by_n1p(int x) const { return NX < 0 ? mdiv(x, m1) : x / n1p; }
  __device__ __forceinline__ int by_n2p(int x) const { return NX < 0 ? mdiv(x, m2) : x / n2p; }
  __device__ __forceinline__ int by_n12(int x) const { return NX < 0 ? mdiv(x, m12) : x / n12; }
  __device__ __forceinline__ int by_per_e(int x) const { return NX < 0 ? mdiv(x, mpe) : x / per_e; }
  // node -> (i, j, k)
  __device__ __forceinline__ void ijk(int node, int& i, int& j, int& k) const {
    k = by_n12(node);
    const int r = node - k * n12;
    j = by_n1p(r);
    i = r - j * n1p;
  }
};

// a[i] for i in 0..2 as selects (a runtime index into a local array would
// put the array in local memory)
__device__ __forceinline__ int sel3(int i, int a0, int a1, int a2) {
  return i == 0 ? a0 : (i == 1 ? a1 : a2);
}

// face coordinates of a side: normal direction and the two tangential ones
__device__ __forceinline__ void side_dirs(int side, int& d, int& a, int& b) {
  d = side >> 1;
  a = (d == 0) ? 1 : 0;
  b = (d == 2) ? 1 : 2;
}

}  // namespace tdg

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk) completing on an mbarrier
namespace tdg {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Copy doubles [src, src+count) into shared memory at a 16-byte aligned
// ``dst`` with one bulk copy; returns the index offset (0 or 1) at which the
// data starts in ``dst`` (the source span is widened to 16-byte boundaries,
// so buffers need >= 8 bytes of slack past their end).
__device__ __forceinline__ int bulk_span(double* dst, const double* src, long long count,
                                         unsigned long long* bar, uint32_t& bytes_total) {
  const unsigned long long a = reinterpret_cast<unsigned long long>(src);
  const unsigned long long lo = a & ~15ull;
  const unsigned long long hi = (a + 8ull * count + 15ull) & ~15ull;
  const uint32_t bytes = static_cast<uint32_t>(hi - lo);
  bulk_g2s(dst, reinterpret_cast<const void*>(lo), bytes, bar);
  bytes_total += bytes;
  return static_cast<int>((a - lo) >> 3);
}

}  // namespace tdg
