// sta_arnoldi.cu -- NEXT row f1: the Arnoldi reduced-order
// model of every net ("an Arnoldi-based reduced-order
// model"; readings A1-A7 in DESIGN.md), one warp per net,
// fp64, per corner and per update (it depends on the RC values).
//
// The driver node is driven by the ideal source; the unknowns are the other
// nodes, C v' + G v = b u.  A = G^-1 C is self-adjoint in the C-inner
// product and G^-1 b = 1, so Lanczos from v_1 = 1 / ||1||_C builds T =
// tridiag(beta, alpha, beta) (order q <= 4, breakdown truncates); each A
// application is one tree solve on the net's DFS-preorder nodes (subtree of
// node i = [i, end_i)): subtree sums S_i of C x as differences of a prefix
// sum, then root-path sums of R S by pointer jumping inside 32-node chunks
// (parents precede children, so a chunk's outside parents are final).  Full
// reorthogonalisation (classical Gram-Schmidt, twice).  T = Q diag(lam) Q^T
// by cyclic Jacobi; per sink the residues res_k = sqrt(Ctot) (V Q)_ik Q_0k.
// Outputs: lam per driver (x < 0: unstable, the forward uses Elmore), the
// residues per sink.  Vectors live in a per-corner fp64 scratch (q + 4
// values per RC node).
#include <cuda_runtime.h>
#include <math_constants.h>

#include "sta_internal.h"

namespace sta {

namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kArnThreads = 256;
constexpr uint32_t kArnBlockMin = 1024;        // nets above: one block of kArnBlock threads each
constexpr int kArnBlock = 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ double warp_incl_scan(double v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// cyclic Jacobi on the symmetric n x n (n <= 4) matrix a: eigenvalues w,
// eigenvectors in the columns of v (every lane computes the same)
__device__ void jacobi4(int n, double a[4][4], double w[4], double v[4][4]) {
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) v[i][j] = i == j;
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, nrm = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        nrm += a[i][j] * a[i][j];
        if (i != j) off += a[i][j] * a[i][j];
      }
    if (off <= 1e-30 * nrm || off == 0.0) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[p][q];
        if (apq == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
        const double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(tt * tt + 1.0), sn = tt * c;
        for (int k = 0; k < n; ++k) {
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - sn * akq;
          a[k][q] = sn * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - sn * aqk;
          a[q][k] = sn * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = c * vkp - sn * vkq;
          v[k][q] = sn * vkp + c * vkq;
        }
      }
  }
  for (int i = 0; i < n; ++i) w[i] = a[i][i];
}

struct ArnScr {                 // per-corner scratch, per internal RC node
  double* C;                    // node cap (0 at the driven root)
  double* V;                    // V[k * n + i], k = 0 .. q
  double* W;                    // the new Lanczos vector
  double* P;                    // exclusive prefix sums of C x within the net
  size_t n;
};

// W = A x over the net's nodes [x0, x0 + m) (global internal indices)
__device__ void tree_apply(const Topo& t, const float* __restrict__ R, const ArnScr& s, const double* x,
                           uint32_t x0, uint32_t m, int lane) {
  // pass A: exclusive prefix of C x
  double carry = 0.0;
  for (uint32_t c0 = 0; c0 < m; c0 += 32) {
    const uint32_t i = x0 + c0 + lane;
    const double v = c0 + lane < m ? s.C[i] * x[i] : 0.0;
    const double inc = warp_incl_scan(v, lane);
    if (c0 + lane < m) s.P[i] = carry + inc - v;
    carry += __shfl_sync(kFull, inc, 31);
  }
  const double total = carry;
  __syncwarp();
  // pass B: W_i = sum over the root path of R_a S_a, S_a = P[end_a] - P[a]
  for (uint32_t c0 = 0; c0 < m; c0 += 32) {
    const uint32_t i = x0 + c0 + lane;
    const bool act = c0 + lane < m;
    double acc = 0.0;
    uint32_t ptr = kNone;
    if (act) {
      const uint4 nd = __ldg(t.arn_node + i);
      if (nd.y != kNone) {                     // not the root
        const double S = (nd.z == x0 + m ? total : s.P[nd.z]) - s.P[i];
        acc = (double)R[nd.x] * S;
        ptr = nd.y;
      }
    }
    const uint32_t cs = x0 + c0;
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const bool in = ptr != kNone && ptr >= cs;
      const int src = in ? (int)(ptr - cs) : lane;
      const double pa = __shfl_sync(kFull, acc, src);
      const uint32_t pp = __shfl_sync(kFull, ptr, src);
      if (in) {
        acc += pa;
        ptr = pp;
      }
    }
    if (act) s.W[i] = acc + (ptr != kNone ? s.W[ptr] : 0.0);
    __syncwarp();
  }
}

__global__ void __launch_bounds__(kArnThreads) arn_reduce_kernel(Topo t, const __grid_constant__ Batch B) {
  const uint32_t w = (blockIdx.x * kArnThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= t.n_arn_nets) return;
  const CornerDev& c = B.c[blockIdx.y];
  const uint4 net = __ldg(t.arn_nets + w);
  const uint32_t x0 = net.x, m = net.y, drv = net.z;
  const int q = (int)t.arn_q;
  if (m <= 32 || m > kArnBlockMin) return;    // arn_small_kernel / arn_block_kernel
  const float* R = c.rc_vals[0];
  const float* Cw = c.rc_vals[1];
  const size_t n = t.n_rc_nodes;
  ArnScr s{c.arn_scr, c.arn_scr + n, c.arn_scr + (size_t)(q + 2) * n, c.arn_scr + (size_t)(q + 3) * n, n};
  // node caps (wire + pin + PO) and Ctot over the non-root nodes
  double ctot = 0.0;
  for (uint32_t c0 = 0; c0 < m; c0 += 32) {
    const uint32_t i = x0 + c0 + lane;
    if (c0 + lane < m) {
      const uint4 nd = __ldg(t.arn_node + i);
      const double C = nd.y == kNone ? 0.0 : (double)Cw[nd.x] + (double)__ldg(t.arn_scap + i);
      s.C[i] = C;
      ctot += C;
    }
  }
  ctot = warp_sum(ctot);
  if (!(ctot > 0.0) || m <= 1) {               // no dynamics: the output follows the input
    if (lane == 0) c.arn_lam[drv] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t c0 = 0; c0 < m; c0 += 32) {
      const uint32_t i = x0 + c0 + lane;
      if (c0 + lane < m) {
        const uint32_t tag = __ldg(t.arn_node + i).w;
        if (tag != kNone) c.arn_res[tag] = make_float4(1.f, 0.f, 0.f, 0.f);
      }
    }
    return;
  }
  const double inv = 1.0 / sqrt(ctot);
  for (uint32_t c0 = 0; c0 < m; c0 += 32) {
    const uint32_t i = x0 + c0 + lane;
    if (c0 + lane < m) s.V[i] = s.C[i] > 0.0 || __ldg(t.arn_node + i).y != kNone ? inv : 0.0;
  }
  __syncwarp();
  double alpha[4] = {0, 0, 0, 0}, beta[4] = {0, 0, 0, 0};
  int qq = 0;
  for (int j = 0; j < q; ++j) {
    const double* vj = s.V + (size_t)j * n;
    tree_apply(t, R, s, vj, x0, m, lane);
    // W -= beta_{j-1} v_{j-1}; dots with v_0 .. v_j (alpha_j = the last)
    double d[4] = {0, 0, 0, 0};
    for (uint32_t c0 = 0; c0 < m; c0 += 32) {
      const uint32_t i = x0 + c0 + lane;
      if (c0 + lane < m) {
        double wi = s.W[i];
        if (j > 0) wi -= beta[j - 1] * s.V[(size_t)(j - 1) * n + i];
        s.W[i] = wi;
        const double cw = s.C[i] * wi;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k <= j) d[k] += cw * s.V[(size_t)k * n + i];
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) d[k] = warp_sum(d[k]);
    alpha[j] = d[j];
    __syncwarp();
    // two classical Gram-Schmidt sweeps against v_0 .. v_j, then ||W||_C
    double e[4] = {0, 0, 0, 0};
    for (uint32_t c0 = 0; c0 < m; c0 += 32) {
      const uint32_t i = x0 + c0 + lane;
      if (c0 + lane < m) {
        double wi = s.W[i];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k <= j) wi -= d[k] * s.V[(size_t)k * n + i];
        s.W[i] = wi;
        const double cw = s.C[i] * wi;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k <= j) e[k] += cw * s.V[(size_t)k * n + i];
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) e[k] = warp_sum(e[k]);
    __syncwarp();
    double nn = 0.0;
    for (uint32_t c0 = 0; c0 < m; c0 += 32) {
      const uint32_t i = x0 + c0 + lane;
      if (c0 + lane < m) {
        double wi = s.W[i];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k <= j) wi -= e[k] * s.V[(size_t)k * n + i];
        s.W[i] = wi;
        nn += s.C[i] * wi * wi;
      }
    }
    beta[j] = sqrt(warp_sum(nn));
    qq = j + 1;
    if (j + 1 == q || !(beta[j] > 1e-10 * fabs(alpha[j]))) break;
    __syncwarp();
    for (uint32_t c0 = 0; c0 < m; c0 += 32) {
      const uint32_t i = x0 + c0 + lane;
      if (c0 + lane < m) s.V[(size_t)(j + 1) * n + i] = s.W[i] / beta[j];
    }
    __syncwarp();
  }
  // T = Q diag(lam) Q^T
  double T[4][4], Q[4][4], ev[4];
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b)
      T[a][b] = (a >= qq || b >= qq) ? 0.0 : a == b ? alpha[a] : (a + 1 == b ? beta[a] : (b + 1 == a ? beta[b] : 0.0));
  jacobi4(qq, T, ev, Q);
  double lmax = 0.0;
  for (int k = 0; k < qq; ++k) lmax = fmax(lmax, ev[k]);
  bool stable = true;
  float lam[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k = 0; k < qq; ++k) {
    if (ev[k] < -1e-9 * lmax) stable = false;
    lam[k] = ev[k] < 0.0 ? 0.f : (float)ev[k];
  }
  if (lane == 0) c.arn_lam[drv] = stable ? make_float4(lam[0], lam[1], lam[2], lam[3]) : make_float4(-1.f, 0.f, 0.f, 0.f);
  if (!stable) return;
  // residues of the sinks
  const double sq = sqrt(ctot);
  for (uint32_t c0 = 0; c0 < m; c0 += 32) {
    const uint32_t i = x0 + c0 + lane;
    if (c0 + lane >= m) continue;
    const uint32_t tag = __ldg(t.arn_node + i).w;
    if (tag == kNone) continue;
    float r[4] = {0.f, 0.f, 0.f, 0.f};
    for (int k = 0; k < qq; ++k) {
      double a = 0.0;
      for (int j = 0; j < qq; ++j) a += s.V[(size_t)j * n + i] * Q[j][k];
      r[k] = (float)(a * sq * Q[0][k]);
    }
    c.arn_res[tag] = make_float4(r[0], r[1], r[2], r[3]);
  }
}


// Nets of <= 32 RC nodes (nearly all): one lane per node in preorder, the
// Lanczos vectors in registers, the tree solve by a warp scan (subtree sums)
// and pointer jumping over parent lanes (root-path sums): no scratch.
__global__ void __launch_bounds__(kArnThreads) arn_small_kernel(Topo t, const __grid_constant__ Batch B) {
  const uint32_t w = (blockIdx.x * kArnThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= t.n_arn_nets) return;
  const CornerDev& c = B.c[blockIdx.y];
  const uint4 net = __ldg(t.arn_nets + w);
  const uint32_t x0 = net.x, m = net.y, drv = net.z;
  const int q = (int)t.arn_q;
  if (m == 0) {                                // lumped net: no wire delay (the Elmore path)
    if (lane == 0) c.arn_lam[drv] = make_float4(-1.f, 0.f, 0.f, 0.f);
    return;
  }
  if (m > 32) return;                          // arn_reduce_kernel
  const bool act = (uint32_t)lane < m;
  uint4 nd = make_uint4(0, kNone, 0, kNone);
  double C = 0.0, R = 0.0;
  if (act) {
    nd = __ldg(t.arn_node + x0 + lane);
    if (nd.y != kNone) {
      C = (double)c.rc_vals[1][nd.x] + (double)__ldg(t.arn_scap + x0 + lane);
      R = (double)c.rc_vals[0][nd.x];
    }
  }
  const int par = (act && nd.y != kNone) ? (int)(nd.y - x0) : -1;
  const int endl = act ? (int)(nd.z - x0) : 0;
  const double ctot = warp_sum(C);
  if (!(ctot > 0.0) || m <= 1) {               // no dynamics: the output follows the input
    if (lane == 0) c.arn_lam[drv] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (act && nd.w != kNone) c.arn_res[nd.w] = make_float4(1.f, 0.f, 0.f, 0.f);
    return;
  }
  // A x on the lanes (x = this lane's component)
  auto apply = [&](double x) {
    const double tv = C * x;
    const double inc = warp_incl_scan(tv, lane);
    const double exc = inc - tv;
    const double total = __shfl_sync(kFull, inc, 31);
    const double pend = __shfl_sync(kFull, exc, endl < 32 ? endl : lane);
    const double S = (endl == (int)m ? total : pend) - exc;
    double acc = par >= 0 ? R * S : 0.0;
    int ptr = par;
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const int src = ptr >= 0 ? ptr : lane;
      const double pa = __shfl_sync(kFull, acc, src);
      const int pp = __shfl_sync(kFull, ptr, src);
      if (ptr >= 0) {
        acc += pa;
        ptr = pp;
      }
    }
    return acc;
  };
  double V[5] = {0, 0, 0, 0, 0};
  V[0] = par >= 0 ? 1.0 / sqrt(ctot) : 0.0;
  double alpha[4] = {0, 0, 0, 0}, beta[4] = {0, 0, 0, 0};
  int qq = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (j >= q) break;
    double wv = apply(V[j]);
    if (j > 0) wv -= beta[j - 1] * V[j - 1];
    double d[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) d[k] = k <= j ? warp_sum(C * wv * V[k]) : 0.0;
    alpha[j] = d[j];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k <= j) wv -= d[k] * V[k];
#pragma unroll
    for (int k = 0; k < 4; ++k) d[k] = k <= j ? warp_sum(C * wv * V[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k <= j) wv -= d[k] * V[k];
    beta[j] = sqrt(warp_sum(C * wv * wv));
    qq = j + 1;
    if (j + 1 == q || !(beta[j] > 1e-10 * fabs(alpha[j]))) break;
    V[j + 1] = wv / beta[j];
  }
  double T[4][4], Q[4][4], ev[4];
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b)
      T[a][b] = (a >= qq || b >= qq) ? 0.0 : a == b ? alpha[a] : (a + 1 == b ? beta[a] : (b + 1 == a ? beta[b] : 0.0));
  jacobi4(qq, T, ev, Q);
  double lmax = 0.0;
  for (int k = 0; k < qq; ++k) lmax = fmax(lmax, ev[k]);
  bool stable = true;
  float lam[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k = 0; k < qq; ++k) {
    if (ev[k] < -1e-9 * lmax) stable = false;
    lam[k] = ev[k] < 0.0 ? 0.f : (float)ev[k];
  }
  if (lane == 0) c.arn_lam[drv] = stable ? make_float4(lam[0], lam[1], lam[2], lam[3]) : make_float4(-1.f, 0.f, 0.f, 0.f);
  if (!stable || !act || nd.w == kNone) return;
  const double sq = sqrt(ctot);
  float r[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k = 0; k < qq; ++k) {
    double a = 0.0;
    for (int j = 0; j < qq; ++j) a += V[j] * Q[j][k];
    r[k] = (float)(a * sq * Q[0][k]);
  }
  c.arn_res[nd.w] = make_float4(r[0], r[1], r[2], r[3]);
}


// ---- nets of more than kArnBlockMin RC nodes: one block of kArnBlock
// threads per net, the same passes in 1024-node chunks (block scans and sums
// through shared memory, the in-chunk pointer jumping in shared memory).
struct BlkSh {
  double red[kArnBlock / 32][4];
  double acc[kArnBlock];
  uint32_t ptr[kArnBlock];
  double carry;
};

// sums of up to 4 values over the block (every thread gets them)
__device__ __forceinline__ void block_sum4(double (&v)[4], int nv, BlkSh& sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = 0; k < nv; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0)
    for (int k = 0; k < nv; ++k) sh.red[wid][k] = v[k];
  __syncthreads();
  for (int k = 0; k < nv; ++k) {
    double x = lane < kArnBlock / 32 ? sh.red[lane][k] : 0.0;
    v[k] = warp_sum(x);
  }
}

// inclusive scan over the block; *total = the block's sum
__device__ __forceinline__ double block_incl_scan(double v, BlkSh& sh, double* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double inc = warp_incl_scan(v, lane);
  __syncthreads();
  if (lane == 31) sh.red[wid][0] = inc;
  __syncthreads();
  if (wid == 0) {
    const double x = lane < kArnBlock / 32 ? sh.red[lane][0] : 0.0;
    sh.red[lane][1] = warp_incl_scan(x, lane);
  }
  __syncthreads();
  *total = sh.red[kArnBlock / 32 - 1][1];
  return inc + (wid ? sh.red[wid - 1][1] : 0.0);
}

__device__ void tree_apply_blk(const Topo& t, const float* __restrict__ R, const ArnScr& s, const double* x,
                               uint32_t x0, uint32_t m, BlkSh& sh) {
  const int tid = threadIdx.x;
  double carry = 0.0;
  for (uint32_t c0 = 0; c0 < m; c0 += kArnBlock) {
    const uint32_t i = x0 + c0 + tid;
    const double v = c0 + tid < m ? s.C[i] * x[i] : 0.0;
    double tot;
    const double inc = block_incl_scan(v, sh, &tot);
    if (c0 + tid < m) s.P[i] = carry + inc - v;
    carry += tot;
  }
  const double total = carry;
  __syncthreads();
  for (uint32_t c0 = 0; c0 < m; c0 += kArnBlock) {
    const uint32_t i = x0 + c0 + tid;
    const bool act = c0 + tid < m;
    double acc = 0.0;
    uint32_t ptr = kNone;
    if (act) {
      const uint4 nd = __ldg(t.arn_node + i);
      if (nd.y != kNone) {
        const double S = (nd.z == x0 + m ? total : s.P[nd.z]) - s.P[i];
        acc = (double)R[nd.x] * S;
        ptr = nd.y;
      }
    }
    const uint32_t cs = x0 + c0;
    sh.acc[tid] = acc;
    sh.ptr[tid] = ptr;
    __syncthreads();
    for (int r = 0; r < 10; ++r) {
      const bool in = ptr != kNone && ptr >= cs;
      double pa = 0.0;
      uint32_t pp = ptr;
      if (in) {
        pa = sh.acc[ptr - cs];
        pp = sh.ptr[ptr - cs];
      }
      __syncthreads();
      if (in) {
        acc += pa;
        ptr = pp;
        sh.acc[tid] = acc;
        sh.ptr[tid] = ptr;
      }
      const int more = __syncthreads_or(ptr != kNone && ptr >= cs);
      if (!more) break;
    }
    if (act) s.W[i] = acc + (ptr != kNone ? s.W[ptr] : 0.0);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kArnBlock, 1) arn_block_kernel(Topo t, const __grid_constant__ Batch B,
                                                                 const uint32_t* __restrict__ big, uint32_t n_big) {
  __shared__ BlkSh sh;
  const int tid = threadIdx.x;
  const CornerDev& c = B.c[blockIdx.y];
  const uint4 net = __ldg(t.arn_nets + big[blockIdx.x]);
  const uint32_t x0 = net.x, m = net.y, drv = net.z;
  const int q = (int)t.arn_q;
  const float* R = c.rc_vals[0];
  const float* Cw = c.rc_vals[1];
  const size_t n = t.n_rc_nodes;
  ArnScr s{c.arn_scr, c.arn_scr + n, c.arn_scr + (size_t)(q + 2) * n, c.arn_scr + (size_t)(q + 3) * n, n};
  double v4[4] = {0, 0, 0, 0};
  for (uint32_t c0 = 0; c0 < m; c0 += kArnBlock) {
    const uint32_t i = x0 + c0 + tid;
    if (c0 + tid < m) {
      const uint4 nd = __ldg(t.arn_node + i);
      const double C = nd.y == kNone ? 0.0 : (double)Cw[nd.x] + (double)__ldg(t.arn_scap + i);
      s.C[i] = C;
      v4[0] += C;
    }
  }
  block_sum4(v4, 1, sh);
  const double ctot = v4[0];
  if (!(ctot > 0.0)) {
    if (tid == 0) c.arn_lam[drv] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t c0 = 0; c0 < m; c0 += kArnBlock) {
      const uint32_t i = x0 + c0 + tid;
      if (c0 + tid < m) {
        const uint32_t tag = __ldg(t.arn_node + i).w;
        if (tag != kNone) c.arn_res[tag] = make_float4(1.f, 0.f, 0.f, 0.f);
      }
    }
    return;
  }
  const double inv = 1.0 / sqrt(ctot);
  for (uint32_t c0 = 0; c0 < m; c0 += kArnBlock) {
    const uint32_t i = x0 + c0 + tid;
    if (c0 + tid < m) s.V[i] = __ldg(t.arn_node + i).y != kNone ? inv : 0.0;
  }
  __syncthreads();
  double alpha[4] = {0, 0, 0, 0}, beta[4] = {0, 0, 0, 0};
  int qq = 0;
  for (int j = 0; j < q; ++j) {
    tree_apply_blk(t, R, s, s.V + (size_t)j * n, x0, m, sh);
    double d[4] = {0, 0, 0, 0};
    for (uint32_t c0 = 0; c0 < m; c0 += kArnBlock) {
      const uint32_t i = x0 + c0 + tid;
      if (c0 + tid < m) {
        double wi = s.W[i];
        if (j > 0) wi -= beta[j - 1] * s.V[(size_t)(j - 1) * n + i];
        s.W[i] = wi;
        const double cw = s.C[i] * wi;
        for (int k = 0; k <= j; ++k) d[k] += cw * s.V[(size_t)k * n + i];
      }
    }
    block_sum4(d, j + 1, sh);
    alpha[j] = d[j];
    double e[4] = {0, 0, 0, 0};
    for (uint32_t c0 = 0; c0 < m; c0 += kArnBlock) {
      const uint32_t i = x0 + c0 + tid;
      if (c0 + tid < m) {
        double wi = s.W[i];
        for (int k = 0; k <= j; ++k) wi -= d[k] * s.V[(size_t)k * n + i];
        s.W[i] = wi;
        const double cw = s.C[i] * wi;
        for (int k = 0; k <= j; ++k) e[k] += cw * s.V[(size_t)k * n + i];
      }
    }
    block_sum4(e, j + 1, sh);
    double nn[4] = {0, 0, 0, 0};
    for (uint32_t c0 = 0; c0 < m; c0 += kArnBlock) {
      const uint32_t i = x0 + c0 + tid;
      if (c0 + tid < m) {
        double wi = s.W[i];
        for (int k = 0; k <= j; ++k) wi -= e[k] * s.V[(size_t)k * n + i];
        s.W[i] = wi;
        nn[0] += s.C[i] * wi * wi;
      }
    }
    block_sum4(nn, 1, sh);
    beta[j] = sqrt(nn[0]);
    qq = j + 1;
    if (j + 1 == q || !(beta[j] > 1e-10 * fabs(alpha[j]))) break;
    for (uint32_t c0 = 0; c0 < m; c0 += kArnBlock) {
      const uint32_t i = x0 + c0 + tid;
      if (c0 + tid < m) s.V[(size_t)(j + 1) * n + i] = s.W[i] / beta[j];
    }
    __syncthreads();
  }
  double T[4][4], Q[4][4], ev[4];
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b)
      T[a][b] = (a >= qq || b >= qq) ? 0.0 : a == b ? alpha[a] : (a + 1 == b ? beta[a] : (b + 1 == a ? beta[b] : 0.0));
  jacobi4(qq, T, ev, Q);
  double lmax = 0.0;
  for (int k = 0; k < qq; ++k) lmax = fmax(lmax, ev[k]);
  bool stable = true;
  float lam[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k = 0; k < qq; ++k) {
    if (ev[k] < -1e-9 * lmax) stable = false;
    lam[k] = ev[k] < 0.0 ? 0.f : (float)ev[k];
  }
  if (tid == 0) c.arn_lam[drv] = stable ? make_float4(lam[0], lam[1], lam[2], lam[3]) : make_float4(-1.f, 0.f, 0.f, 0.f);
  if (!stable) return;
  const double sq = sqrt(ctot);
  for (uint32_t c0 = 0; c0 < m; c0 += kArnBlock) {
    const uint32_t i = x0 + c0 + tid;
    if (c0 + tid >= m) continue;
    const uint32_t tag = __ldg(t.arn_node + i).w;
    if (tag == kNone) continue;
    float r[4] = {0.f, 0.f, 0.f, 0.f};
    for (int k = 0; k < qq; ++k) {
      double a = 0.0;
      for (int j = 0; j < qq; ++j) a += s.V[(size_t)j * n + i] * Q[j][k];
      r[k] = (float)(a * sq * Q[0][k]);
    }
    c.arn_res[tag] = make_float4(r[0], r[1], r[2], r[3]);
  }
}

}  // namespace

cudaError_t launch_arn_reduce(const Topo& t, const Batch& b, cudaStream_t s) {
  if (!t.n_arn_nets) return cudaSuccess;
  const dim3 g((uint32_t)((32ull * t.n_arn_nets + kArnThreads - 1) / kArnThreads), b.K);
  arn_small_kernel<<<g, kArnThreads, 0, s>>>(t, b);
  arn_reduce_kernel<<<g, kArnThreads, 0, s>>>(t, b);
  if (t.n_arn_big) arn_block_kernel<<<dim3(t.n_arn_big, b.K), kArnBlock, 0, s>>>(t, b, t.arn_big, t.n_arn_big);
  return cudaGetLastError();
}

}  // namespace sta
