// Hermitian eigendecomposition (syevd) on the GPU -- reference
// pkg/src/bcmg/solvers.py:597-910 (_householder, _tridiagonalize,
// _tridiag_eig, syevd).
//
// Same algorithm as the reference, re-planned for one B200:
//   1. the shards (block-cyclic or contiguous column layout, any number of
//      logical devices on this GPU) are gathered into ONE dense n x n working
//      copy in the compute type (double / double2): the per-column symmetric
//      matrix-vector product then streams the trailing lower triangle at HBM
//      rate instead of walking tiles device by device;
//   2. blocked Householder tridiagonalisation exactly as solvers.py:666-780:
//      per column a lazy panel-column update from the tile's U / W panels, the
//      reflector (v, tau, beta) with real beta (solvers.py:600-623), y = A v
//      over the stale trailing lower triangle (tiled, deterministic two-pass
//      reduction), the U / W correction and W = tau y - sigma v; per tile one
//      rank-2T update of the trailing lower triangle on the DMMA GEMM;
//   3. back-transformation (solvers.py:884-897) of the IDENTITY, blocked 256
//      reflectors at a time in compact WY form (Q_blk = I - V T V^H, T from
//      the forward recurrence): V = Q with three GEMMs per block.  Since
//      Q (Z_ql) = (Q Z_ql), this does not wait for the QL: the GPU forms Q
//      while the host iterates;
//   4. implicit-shift QL on the real tridiagonal (solvers.py:783-843) on the
//      host, O(n^2) without vectors; its plane rotations are recorded, streamed
//      to the GPU and replayed on V's columns (one thread per row; a complex
//      column is a real column of 2n (re, im) rows, the rotations being real);
//   5. phase normalisation (largest-magnitude component real and positive,
//      first index on ties, solvers.py:898-909) fused with the scatter back
//      into the caller's shards and the narrowing to the storage type.
// Every reduction has a fixed order: two runs give identical bits
// (reference test_solvers.py:260-271).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <string>
#include <vector>

#include "ops.h"
#include "solver.h"

namespace bcmg {
namespace {

constexpr int ET = 64;      // symv tile
constexpr int WY = 256;     // reflectors per compact-WY block of the back-transformation
constexpr int RT = 256;     // threads of the row-parallel kernels

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscl(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double d = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
__device__ __forceinline__ double2 zero2() { return make_double2(0.0, 0.0); }

// Column g of the distributed matrix -> (shard, local column).
struct ShardMap {
  void* p[16];
  int64_t off[17];  // contiguous layout: first global column of each device
  int64_t T;
  int D, cyclic;
};
__device__ __forceinline__ void map_col(const ShardMap& m, int64_t g, int& d, int64_t& lc) {
  if (m.cyclic) {
    const int64_t t = g / m.T;
    d = (int)(t % m.D);
    lc = (t / m.D) * m.T + g % m.T;
  } else {
    d = 0;
    while (d + 1 < m.D && g >= m.off[d + 1]) ++d;
    lc = g - m.off[d];
  }
}

// deterministic block sum of a double2 (fixed shuffle tree + fixed warp order)
__device__ __forceinline__ double2 block_sum(double2 v, double2* red) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double2 s = zero2();
  if (threadIdx.x == 0)
    for (int i = 0; i < nw; ++i) s = cadd(s, red[i]);
  return s;  // valid in thread 0
}

// ---------------------------------------------------------------- gather / scatter
template <class S, class X>
__global__ void eig_gather(ShardMap m, X* A, int64_t n) {
  const int64_t g = blockIdx.y + (int64_t)blockIdx.z * gridDim.y;
  if (g >= n) return;
  int d;
  int64_t lc;
  map_col(m, g, d, lc);
  const S* src = reinterpret_cast<const S*>(m.p[d]) + lc * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    A[i + g * n] = from_c<X>(to_c(src[i]));
}

// Z column j -> shard column j, scaled so that its first largest-magnitude
// component is real and positive (solvers.py:898-909).
template <class X, class S>
__global__ void eig_phase_scatter(const X* Z, const int64_t* order, int64_t n, ShardMap m) {
  __shared__ double bv[32];
  __shared__ int64_t bi[32];
  __shared__ double2 ph;
  const int64_t j = blockIdx.x;
  const X* z = Z + order[j] * n;  // eigenvectors in ascending eigenvalue order
  double best = -1.0;
  int64_t idx = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 v = to_c(z[i]);
    const double a = hypot(v.x, v.y);
    if (a > best) best = a, idx = i;  // strided ascending: first max of this thread
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_down_sync(0xffffffffu, best, o);
    const int64_t oi = __shfl_down_sync(0xffffffffu, idx, o);
    if (ob > best || (ob == best && oi < idx)) best = ob, idx = oi;
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) bv[w] = best, bi[w] = idx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (bv[k] > best || (bv[k] == best && bi[k] < idx)) best = bv[k], idx = bi[k];
    const double2 lead = to_c(z[idx]);
    const double s = hypot(lead.x, lead.y);
    ph = s == 0.0 ? make_double2(1.0, 0.0) : make_double2(lead.x / s, lead.y / s);
  }
  __syncthreads();
  const double2 p = ph;
  int d;
  int64_t lc;
  map_col(m, j, d, lc);
  S* dst = reinterpret_cast<S*>(m.p[d]) + lc * n;
  __shared__ int64_t anchor;
  if (threadIdx.x == 0) anchor = idx;
  __syncthreads();
  const int64_t ia = anchor;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double2 o = cmulc(to_c(z[i]), p);
    if (i == ia) o = make_double2(hypot(o.x, o.y), 0.0);  // the anchor exactly real and positive
    dst[i] = from_c<S>(o);
  }
}

// ---------------------------------------------------------------- tridiagonalisation
// y = sym(A[c0:, c0:]) v, lower-triangle storage (solvers.py:729-745): one CTA
// per 64x64 tile (bi >= bj) of the trailing lower triangle; the tile's row
// products go to P1[bj][rows], its conjugate-transposed column products
// (strictly below the diagonal) to P2[bi][cols]; eig_symv_reduce sums them in
// a fixed order.
template <class X>
__global__ void __launch_bounds__(256) eig_symv(const X* A, int64_t n, int64_t c0, const X* v, X* P1, X* P2,
                                               int64_t ntri, const X* U, const X* W, int jj, X* t) {
  // the first 2*jj blocks (dispatched first, so they overlap the tiles instead
  // of trailing them): t[k] = (W^H v)[k], t[jj + k] = (U^H v)[k]
  if ((int64_t)blockIdx.x < 2 * jj) {
    __shared__ double2 dred[32];
    const int b = (int)blockIdx.x;
    const X* M = b < jj ? W + (int64_t)b * n : U + (int64_t)(b - jj) * n;
    double2 acc = zero2();
#pragma unroll 4
    for (int64_t i = c0 + threadIdx.x; i < n; i += blockDim.x) acc = cadd(acc, cmul(cconj(to_c(M[i])), to_c(v[i])));
    acc = block_sum(acc, dred);
    if (threadIdx.x == 0) t[b] = from_c<X>(acc);
    return;
  }
  extern __shared__ __align__(16) unsigned char sm_raw[];
  X* sm = reinterpret_cast<X*>(sm_raw);  // 64 x 65, column-major tile
  __shared__ double2 vr[ET], vc[ET], half[2][2][ET];
  const int64_t b = blockIdx.x - 2 * jj;
  int64_t bi = (int64_t)((sqrt(8.0 * (double)b + 1.0) - 1.0) * 0.5);
  while (bi * (bi + 1) / 2 > b) --bi;
  while ((bi + 1) * (bi + 2) / 2 <= b) ++bi;
  const int64_t bj = b - bi * (bi + 1) / 2;
  const int64_t r0 = c0 + bi * ET, q0 = c0 + bj * ET;
  const int tid = threadIdx.x;
  X ld[ET * ET / 256];
#pragma unroll
  for (int q = 0; q < ET * ET / 256; ++q) {  // all loads in flight, then stage
    const int e = tid + q * 256, il = e % ET, jl = e / ET;
    const int64_t i = r0 + il, j = q0 + jl;
    ld[q] = (i < n && j < n) ? A[i + j * n] : from_c<X>(zero2());
  }
#pragma unroll
  for (int q = 0; q < ET * ET / 256; ++q) {
    const int e = tid + q * 256;
    sm[(e / ET) * (ET + 1) + e % ET] = ld[q];
  }
  if (tid < ET) vc[tid] = q0 + tid < n ? to_c(v[q0 + tid]) : zero2();
  else if (tid < 2 * ET) vr[tid - ET] = r0 + tid - ET < n ? to_c(v[r0 + tid - ET]) : zero2();
  __syncthreads();
  const bool diag = bi == bj;
  const int part = tid >> 7, h = (tid >> 6) & 1, x = tid & 63;
  double2 acc = zero2();
  if constexpr (!Traits<X>::cplx) {  // real: plain FMAs, branch-free off the diagonal
    double a = 0.0;
    if (part == 0) {  // row x, columns 32h .. 32h+31
      const double* row = reinterpret_cast<const double*>(sm) + x;
      if (!diag) {
#pragma unroll
        for (int q = 0; q < 32; ++q) a = fma(row[(32 * h + q) * (ET + 1)], vc[32 * h + q].x, a);
      } else {
        for (int jl = 32 * h; jl < 32 * h + 32 && jl <= x; ++jl) a = fma(row[jl * (ET + 1)], vc[jl].x, a);
      }
    } else {  // column x, rows 32h .. 32h+31 (strictly below the diagonal on diagonal tiles)
      const double* col = reinterpret_cast<const double*>(sm) + x * (ET + 1);
      if (!diag) {
#pragma unroll
        for (int q = 0; q < 32; ++q) a = fma(col[32 * h + q], vr[32 * h + q].x, a);
      } else {
        for (int il = max(32 * h, x + 1); il < 32 * h + 32; ++il) a = fma(col[il], vr[il].x, a);
      }
    }
    acc.x = a;
  } else {
    if (part == 0) {  // row x, columns 32h .. 32h+31
      for (int jl = 32 * h; jl < 32 * h + 32; ++jl)
        if (!diag || jl <= x) acc = cadd(acc, cmul(to_c(sm[jl * (ET + 1) + x]), vc[jl]));
    } else {  // column x, rows 32h .. 32h+31 (strictly below the diagonal on diagonal tiles)
      for (int il = 32 * h; il < 32 * h + 32; ++il)
        if (!diag || il > x) acc = cadd(acc, cmul(cconj(to_c(sm[x * (ET + 1) + il])), vr[il]));
    }
  }
  half[part][h][x] = acc;
  __syncthreads();
  if (tid < ET) {
    if (r0 + tid < n) P1[bj * n + r0 + tid] = from_c<X>(cadd(half[0][0][tid], half[0][1][tid]));
  } else if (tid < 2 * ET) {
    const int jl = tid - ET;
    if (q0 + jl < n) P2[bi * n + q0 + jl] = from_c<X>(cadd(half[1][0][jl], half[1][1][jl]));
  }
}

// ---- fused per-column kernels (3 launches per column).  Grid-wide steps use
// the last-block pattern: every block publishes its partial, the block that
// takes the last ticket reduces them in a fixed order (same bits every run)
// and does the serial tail; it also re-arms the ticket counter.
__device__ __forceinline__ bool last_block(unsigned* counter) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

template <class X>
__device__ __forceinline__ double2 ldcg_c(const X* p) {
  if constexpr (sizeof(X) == 16) {
    const double2 v = __ldcg(reinterpret_cast<const double2*>(p));
    return v;
  } else {
    return make_double2(__ldcg(reinterpret_cast<const double*>(p)), 0.0);
  }
}

// K1: lazy panel-column update A[c:, c] -= U conj(W[c]) + W conj(U[c])
// (solvers.py:705-709), then -- in the last block -- d[c] and the reflector of
// A[c+1:, c] (solvers.py:600-623, 712-716).
template <class X>
__global__ void __launch_bounds__(1024) eig_col_prep(X* A, int64_t n, int64_t c, const X* U, const X* W, int jj,
                                                     X* vbuf, X* tau, double* dd, double* ee, double* npart,
                                                     unsigned* counter) {
  __shared__ double2 sred[32];
  __shared__ double wsq[32];
  __shared__ double2 den;
  __shared__ int trivial;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;  // one warp per row, lanes over k
  const int64_t i = c + blockIdx.x * 32 + w;
  double2 s = zero2();
  if (i < n)
    for (int k = lane; k < jj; k += 32)
      s = cadd(s, cadd(cmulc(to_c(U[i + k * n]), to_c(W[c + k * n])), cmulc(to_c(W[i + k * n]), to_c(U[c + k * n]))));
  for (int o = 16; o > 0; o >>= 1) {
    s.x += __shfl_down_sync(0xffffffffu, s.x, o);
    s.y += __shfl_down_sync(0xffffffffu, s.y, o);
  }
  if (lane == 0) {
    double sq = 0.0;
    if (i < n) {
      X val = A[i + c * n];
      if (jj) {
        val = from_c<X>(csub(to_c(val), s));
        A[i + c * n] = val;
      }
      if (i >= c + 2) {
        const double2 q = to_c(val);
        sq = q.x * q.x + q.y * q.y;
      }
    }
    wsq[w] = sq;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sq = 0.0;
    for (int q = 0; q < 32; ++q) sq += wsq[q];
    npart[blockIdx.x] = sq;
  }
  if (!last_block(counter)) return;
  if (threadIdx.x == 0) {
    *counter = 0u;
    dd[c] = ldcg_c(A + c + c * n).x;
  }
  const int64_t L = n - c - 1;
  if (L <= 0) return;
  double acc = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) acc += __ldcg(npart + b);
  const double tot = block_sum(make_double2(acc, 0.0), sred).x;
  X* x = A + (c + 1) + c * n;
  if (threadIdx.x == 0) {
    const double tail = sqrt(tot);
    const double2 alpha = ldcg_c(x);
    double2 t;
    double beta;
    if (tail == 0.0 && alpha.y == 0.0) {
      t = zero2();
      beta = alpha.x;
      trivial = 1;
    } else {
      const double h = hypot(hypot(alpha.x, alpha.y), tail);
      beta = -copysign(h, alpha.x != 0.0 ? alpha.x : 1.0);  // `alpha.real or 1.0`
      den = make_double2(alpha.x - beta, alpha.y);
      t = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
      trivial = 0;
    }
    ee[c] = beta;
    tau[c] = from_c<X>(t);
  }
  __syncthreads();
  const int triv = trivial;
  const double2 dn = den;
#pragma unroll 4
  for (int64_t r = threadIdx.x; r < L; r += blockDim.x) {
    double2 v;
    if (r == 0) v = make_double2(1.0, 0.0);
    else if (triv) v = zero2();
    else v = cdiv(ldcg_c(x + r), dn);
    const X vx = from_c<X>(v);
    vbuf[c + 1 + r] = vx;
    x[r] = vx;
  }
}

// K3: y = sum of the symv partials minus U t[:jj] + W t[jj:] (solvers.py:746-750),
// then -- in the last block -- sigma = |tau|^2/2 v^H y and the panel columns
// U[:, jj] = v, W[:, jj] = tau y - sigma v (solvers.py:751-754).
template <class X>
__global__ void __launch_bounds__(1024) eig_col_finish(const X* P1, const X* P2, int64_t n, int64_t c0, int64_t nb,
                                                       X* U, X* W, int jj, const X* t, X* y, const X* v,
                                                       const X* tau, int64_t c, double2* part, unsigned* counter) {
  __shared__ double2 sred[32];
  __shared__ double2 sig;
  __shared__ double2 wc[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;  // one warp per row
  const int64_t i = c0 + blockIdx.x * 32 + w;
  double2 s = zero2(), corr = zero2();
  if (i < n) {
    const int64_t I = (i - c0) / ET;
    for (int64_t q = lane; q <= I; q += 32) s = cadd(s, to_c(P1[q * n + i]));
    for (int64_t q = I + lane; q < nb; q += 32) s = cadd(s, to_c(P2[q * n + i]));
    for (int k = lane; k < jj; k += 32)
      corr = cadd(corr, cadd(cmul(to_c(U[i + (int64_t)k * n]), to_c(t[k])),
                             cmul(to_c(W[i + (int64_t)k * n]), to_c(t[jj + k]))));
  }
  double2 yi = csub(s, corr);
  for (int o = 16; o > 0; o >>= 1) {
    yi.x += __shfl_down_sync(0xffffffffu, yi.x, o);
    yi.y += __shfl_down_sync(0xffffffffu, yi.y, o);
  }
  if (lane == 0) {
    double2 contrib = zero2();
    if (i < n) {
      const X yx = from_c<X>(yi);
      y[i] = yx;
      contrib = cmul(cconj(to_c(v[i])), to_c(yx));
    }
    wc[w] = contrib;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 tot = zero2();
    for (int q = 0; q < 32; ++q) tot = cadd(tot, wc[q]);
    part[blockIdx.x] = tot;
  }
  if (!last_block(counter)) return;
  if (threadIdx.x == 0) *counter = 0u;
  const double2 tu = to_c(tau[c]);
  if (tu.x == 0.0 && tu.y == 0.0) return;  // reflection skipped (solvers.py:718)
  double2 acc = zero2();
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) acc = cadd(acc, ldcg_c(part + b));
  acc = block_sum(acc, sred);
  if (threadIdx.x == 0) sig = cscl(acc, 0.5 * (tu.x * tu.x + tu.y * tu.y));
  __syncthreads();
  const double2 sg = sig;
#pragma unroll 4
  for (int64_t r = c0 + threadIdx.x; r < n; r += blockDim.x) {
    const double2 vi = to_c(v[r]);
    U[r + (int64_t)jj * n] = v[r];
    W[r + (int64_t)jj * n] = from_c<X>(csub(cmul(tu, ldcg_c(y + r)), cmul(sg, vi)));
  }
}

// ---------------------------------------------------------------- tridiagonal eigenvectors
// Replay the QL plane rotations on the rows of Z (solvers.py:831-835).  Sweep
// k applies rotations top_k, top_k - 1, ..., bot_k to column pairs (i, i+1),
// sweeps in order.  K consecutive sweeps run as one wavefront: at step p (p
// descending) sweep s applies its rotation at i = p + 2s.  Every rotation of
// an earlier sweep that touches columns i or i+1 sits at a position >= i - 1,
// i.e. at a step >= p + 1, so the order of operations on every column is the
// sequential one (same bits).  One thread per row keeps the 2K active columns
// in registers: one load and one store per column per K sweeps instead of per
// sweep.
template <int K>
__global__ void __launch_bounds__(32) eig_rotate_wave(double* Z, int64_t rows, int64_t ld, int64_t n, const double2* cs,
                                                      const int64_t* sw_off, const int64_t* sw_top, int64_t s0,
                                                      int64_t nsw) {
  constexpr int W = 2 * K;  // window columns == steps per parameter chunk == warp width
  static_assert(W == 32, "one parameter per lane and step");
  __shared__ double2 prm[K][W];
  const int lane = threadIdx.x;
  const int64_t r = blockIdx.x * (int64_t)W + lane;
  const bool live = r < rows;
  const int kk = (int)min((int64_t)K, nsw - s0);
  int64_t top[K], bot[K], off[K];
  int64_t pmax = INT64_MIN, pmin = INT64_MAX;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    if (s < kk) {
      off[s] = sw_off[s0 + s];
      top[s] = sw_top[s0 + s];
      bot[s] = top[s] - (sw_off[s0 + s + 1] - off[s]) + 1;
      pmax = max(pmax, top[s] - 2 * s);
      pmin = min(pmin, bot[s] - 2 * s);
    } else {
      off[s] = 0, top[s] = -1, bot[s] = 0;  // empty
    }
  }
  double* z = Z + (live ? r : 0);
  // column c lives in slot (c - pmax) mod W: every index below is static
  double win[W];
#pragma unroll
  for (int j = 0; j < W; ++j) {
    const int64_t c = pmax + j;
    win[j] = (live && c >= 0 && c < n) ? z[c * ld] : 0.0;
  }
  for (int64_t p0 = pmax; p0 >= pmin; p0 -= W) {
    __syncwarp();
#pragma unroll
    for (int s = 0; s < K; ++s) {  // lane u stages sweep s's rotation for step p0 - u (identity when idle)
      const int64_t i = p0 - lane + 2 * s;
      double2 g = make_double2(1.0, 0.0);
      if (i >= bot[s] && i <= top[s]) g = cs[off[s] + (top[s] - i)];
      prm[s][lane] = g;
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < W; ++u) {
      const int64_t p = p0 - u;
      if (p < pmin) break;
#pragma unroll
      for (int s = 0; s < K; ++s) {  // sweep s: columns p + 2s, p + 2s + 1
        const double2 g = prm[s][u];
        const int sa = ((2 * s - u) % W + W) % W, sb = ((2 * s + 1 - u) % W + W) % W;
        const double x = win[sa], y = win[sb];
        win[sb] = g.y * x + g.x * y;
        win[sa] = g.x * x - g.y * y;
      }
      const int sl = W - 1 - u;  // column p + W - 1 leaves, column p - 1 enters
      const int64_t co = p + W - 1, ci = p - 1;
      if (live && co >= 0 && co < n) z[co * ld] = win[sl];
      win[sl] = (live && ci >= 0 && ci < n) ? z[ci * ld] : 0.0;
    }
  }
  // the window now holds columns pmin - 1 .. pmin + W - 2
  const int64_t first = pmin - 1, shift = ((first - pmax) % W + W) % W;
#pragma unroll
  for (int sl = 0; sl < W; ++sl) {
    const int64_t c = first + (((int64_t)sl - shift) % W + W) % W;
    if (live && c >= 0 && c < n) z[c * ld] = win[sl];
  }
}

template <class X>
__global__ void eig_identity(X* Z, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) Z[i + i * n] = from_c<X>(make_double2(1.0, 0.0));
}

// Forward compact-WY factor of kb reflectors: T upper, T[j][j] = tau_j,
// T[:j, j] = -tau_j T[:j, :j] G[:j, j], G = V^H V (LAPACK larft, forward / columnwise).
template <class X>
__global__ void __launch_bounds__(WY) eig_larft(const X* G, const X* tau, int kb, X* Tm) {
  const int i = threadIdx.x;  // row of T, in global memory (kb x kb, ld kb)
  if (i < kb)
    for (int j = 0; j < kb; ++j) Tm[i + j * kb] = from_c<X>(zero2());
  __syncthreads();
  for (int j = 0; j < kb; ++j) {
    const double2 tj = to_c(tau[j]);
    if (i < j) {
      double2 acc = zero2();
      for (int l = i; l < j; ++l) acc = cadd(acc, cmul(to_c(Tm[i + l * kb]), to_c(G[l + j * kb])));
      Tm[i + j * kb] = from_c<X>(cscl(cmul(tj, acc), -1.0));
    } else if (i == j) {
      Tm[j + j * kb] = from_c<X>(tj);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- host QL
// Implicit-shift QL on the tridiagonal (d, e) exactly as solvers.py:783-843,
// without the vectors: the rotations of each bulge-chasing sweep are recorded.
// hypot through one correctly rounded sqrt when neither square can overflow or
// lose precision to underflow (within 1 ulp of hypot, ~4x cheaper); the
// library hypot otherwise
inline double fast_hypot(double a, double b) {
  const double m = std::fmax(std::fabs(a), std::fabs(b));
  if (m < 1e150 && m > 1e-140) return std::sqrt(a * a + b * b);
  return std::hypot(a, b);
}

struct QLRecord {
  double2* cs = nullptr;  // rotations of the pending sweeps, written straight into a pinned slot
  int64_t ncs = 0;
  std::vector<int64_t> off{0}, top;
};
template <class F>
void tridiag_ql(std::vector<double>& d, const std::vector<double>& e_in, QLRecord& rec, F&& after_sweep,
                int max_iter = 30) {
  const int64_t n = (int64_t)d.size();
  std::vector<double> e(n, 0.0);
  for (int64_t i = 0; i + 1 < n; ++i) e[i] = e_in[i];
  const double eps = 2.220446049250313e-16;
  for (int64_t l = 0; l < n; ++l) {
    int iters = 0;
    while (true) {
      int64_t m = n - 1;
      for (int64_t mm = l; mm < n - 1; ++mm) {
        const double dd = std::fabs(d[mm]) + std::fabs(d[mm + 1]);
        if (std::fabs(e[mm]) <= eps * dd) {
          m = mm;
          break;
        }
      }
      if (m == l) break;
      if (++iters > max_iter)
        throw Error(NO_CONVERGENCE, "tridiagonal eigensolver exceeded " + std::to_string(max_iter) +
                                        " iterations at index " + std::to_string(l));
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = std::hypot(g, 1.0);
      g = d[m] - d[l] + e[l] / (g + std::copysign(r, g));
      double s = 1.0, c = 1.0, p = 0.0;
      bool broke = false;
      rec.top.push_back(m - 1);
      for (int64_t i = m - 1; i >= l; --i) {
        const double f = s * e[i], b = c * e[i];
        r = fast_hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          d[i + 1] -= p;
          e[m] = 0.0;
          broke = true;
          break;
        }
        s = f / r;
        c = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * s + 2.0 * c * b;
        p = s * r;
        d[i + 1] = g + p;
        g = c * r - b;
        rec.cs[rec.ncs++] = make_double2(c, s);
      }
      if (rec.ncs == rec.off.back()) rec.top.pop_back();  // no rotation applied
      else {
        rec.off.push_back(rec.ncs);
        after_sweep();
      }
      if (!broke) {
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    }
  }
}

inline unsigned blocks_for(int64_t rows, int threads) { return (unsigned)std::max<int64_t>(1, (rows + threads - 1) / threads); }
inline dim3 col_grid(int64_t n, int64_t rows) {
  const int64_t y = std::min<int64_t>(n, 65535), z = (n + y - 1) / y;
  return dim3((unsigned)std::min<int64_t>(std::max<int64_t>(1, (rows + 255) / 256), 8), (unsigned)y, (unsigned)z);
}

template <class S>
void syevd_t(Session& ss, int64_t n, int64_t T, int ndev, void* const* shards, bool cyclic, void* w_out) {
  constexpr bool CP = Traits<S>::cplx;
  using X = typename std::conditional<CP, double2, double>::type;
  const int dtw = CP ? C128 : R64;
  cudaStream_t st = ss.user;
  const size_t es = sizeof(X);
  const int64_t nb = (n + ET - 1) / ET;
  const int64_t nparts_max = (n + 31) / 32;  // eig_col_prep / eig_col_finish blocks (one warp per row)

  // ---- workspace: everything reserved before any data moves (OUT_OF_MEMORY first)
  DevBuf* wb = ss.eig;
  wb[0].ensure((size_t)n * n * es);               // working copy A / stored reflectors V
  wb[2].ensure((size_t)n * n * es);               // V = Q, then Q times the QL rotations
  wb[3].ensure((size_t)2 * n * T * es);           // U | W panels
  wb[4].ensure((size_t)2 * nb * n * es);          // symv partials P1 | P2
  const size_t small = (size_t)(2 * n + 2 * T + n) * es + (size_t)(nparts_max + 1) * sizeof(double2) +
                       (size_t)2 * n * sizeof(double) + (size_t)2 * WY * WY * es + (size_t)2 * WY * n * es +
                       (size_t)n * sizeof(int64_t) + (size_t)nparts_max * sizeof(double) + 512;
  wb[5].ensure(small);
  X* A = static_cast<X*>(wb[0].p);
  X* Zx = static_cast<X*>(wb[2].p);
  X* U = static_cast<X*>(wb[3].p);
  X* W = U + n * T;
  X* P1 = static_cast<X*>(wb[4].p);
  X* P2 = P1 + nb * n;
  char* q = static_cast<char*>(wb[5].p);
  auto carve = [&](size_t bytes) {
    char* r = q;
    q += (bytes + 15) / 16 * 16;
    return r;
  };
  X* vbuf = reinterpret_cast<X*>(carve(n * es));
  X* ybuf = reinterpret_cast<X*>(carve(n * es));
  X* tbuf = reinterpret_cast<X*>(carve(2 * T * es));
  X* tau = reinterpret_cast<X*>(carve(n * es));
  double2* part = reinterpret_cast<double2*>(carve((nparts_max + 1) * sizeof(double2)));
  double* dd = reinterpret_cast<double*>(carve(n * sizeof(double)));
  double* ee = reinterpret_cast<double*>(carve(n * sizeof(double)));
  X* G = reinterpret_cast<X*>(carve(WY * WY * es));
  X* Tm = reinterpret_cast<X*>(carve(WY * WY * es));
  X* X1 = reinterpret_cast<X*>(carve(WY * n * es));
  X* X2 = reinterpret_cast<X*>(carve(WY * n * es));
  int64_t* order_d = reinterpret_cast<int64_t*>(carve(n * sizeof(int64_t)));
  double* npart = reinterpret_cast<double*>(carve(nparts_max * sizeof(double)));
  unsigned* tickets = reinterpret_cast<unsigned*>(carve(2 * sizeof(unsigned)));

  ShardMap map{};
  map.D = ndev;
  map.T = T;
  map.cyclic = cyclic ? 1 : 0;
  const std::vector<int64_t> counts = column_counts(n, T, ndev);
  map.off[0] = 0;
  for (int d = 0; d < ndev; ++d) {
    map.p[d] = shards[d];
    map.off[d + 1] = map.off[d] + counts[d];
  }

  // BCMG_EIG_PROFILE=1: per-phase device times on stderr
  static const bool prof = getenv("BCMG_EIG_PROFILE") != nullptr;
  cudaEvent_t pe[6];
  auto pmark = [&](int k) {
    if (!prof) return;
    if (k == 0)
      for (auto& e : pe) BCMG_CUDA(cudaEventCreate(&e));
    BCMG_CUDA(cudaEventRecord(pe[k], st));
  };
  pmark(0);
  // ---- 1. dense working copy
  eig_gather<S, X><<<col_grid(n, n), 256, 0, st>>>(map, A, n);
  BCMG_CHECK_LAUNCH();
  BCMG_CUDA(cudaMemsetAsync(tau, 0, n * es, st));
  BCMG_CUDA(cudaMemsetAsync(ee, 0, n * sizeof(double), st));
  BCMG_CUDA(cudaMemsetAsync(tickets, 0, 2 * sizeof(unsigned), st));

  // ---- 2. blocked Householder tridiagonalisation (solvers.py:666-780)
  const size_t symv_smem = (size_t)ET * (ET + 1) * sizeof(X);
  BCMG_CUDA(cudaFuncSetAttribute(eig_symv<X>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)symv_smem));
  for (int64_t start = 0; start < n; start += T) {
    const int64_t stop = std::min(start + T, n), tc = stop - start;
    BCMG_CUDA(cudaMemsetAsync(U, 0, (size_t)2 * n * T * es, st));
    for (int64_t jj = 0; jj < tc; ++jj) {
      const int64_t c = start + jj, c0 = c + 1;
      const unsigned g1 = blocks_for(n - c, 32);
      eig_col_prep<X><<<g1, 1024, 0, st>>>(A, n, c, U, W, (int)jj, vbuf, tau, dd, ee, npart, tickets);
      BCMG_CHECK_LAUNCH();
      if (c == n - 1) continue;
      const int64_t L = n - c0, nbt = (L + ET - 1) / ET, ntri = nbt * (nbt + 1) / 2;
      eig_symv<X><<<(unsigned)(ntri + 2 * jj), 256, symv_smem, st>>>(A, n, c0, vbuf, P1, P2, ntri, U, W, (int)jj,
                                                                     tbuf);
      BCMG_CHECK_LAUNCH();
      const unsigned np = blocks_for(L, 32);
      eig_col_finish<X><<<np, 1024, 0, st>>>(P1, P2, n, c0, nbt, U, W, (int)jj, tbuf, ybuf, vbuf, tau, c, part,
                                            tickets + 1);
      BCMG_CHECK_LAUNCH();
    }
    if (stop >= n) continue;
    // trailing lower triangle: A[stop:, stop:] -= U W^H + W U^H (solvers.py:771-780)
    const int64_t M = n - stop;
    Epilogue ep{};
    ep.C = A + stop + stop * n;
    ep.ldc = n;
    ep.alpha = -1.0;
    ep.beta = 1.0;
    ep.lower_only = 1;
    ep.lower_off = 0;
    gemm(dtw, M, M, tc, opA(U + stop, n, OP_N), opB(W + stop, n, OP_C), ep, nullptr, st);
    gemm(dtw, M, M, tc, opA(W + stop, n, OP_N), opB(U + stop, n, OP_C), ep, nullptr, st);
  }

  pmark(1);
  // ---- 3. tridiagonal QL on the host, rotations replayed on the GPU
  std::vector<double> d(n), e(n);
  BCMG_CUDA(cudaMemcpyAsync(d.data(), dd, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  BCMG_CUDA(cudaMemcpyAsync(e.data(), ee, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  BCMG_CUDA(cudaStreamSynchronize(st));
  e.resize(std::max<int64_t>(n - 1, 0));
  // ---- 4 (before 3). back-transformation of the identity: V = Q = H_0 ... H_{n-2}
  // (solvers.py:884-897 applies the same reflectors to Z; Q (Z_ql) = (Q Z_ql)).  It
  // does not depend on the QL, so the GPU runs it while the host iterates, and
  // the QL rotations are then replayed on V's columns directly.
  BCMG_CUDA(cudaMemsetAsync(Zx, 0, (size_t)n * n * es, st));
  eig_identity<X><<<blocks_for(n, RT), RT, 0, st>>>(Zx, n);
  BCMG_CHECK_LAUNCH();
  if (n >= 2) {
    for (int64_t c0 = ((n - 2) / WY) * WY; c0 >= 0; c0 -= WY) {
      const int64_t c1 = std::min<int64_t>(c0 + WY, n - 1), kb = c1 - c0, r0 = c0 + 1, K = n - r0;
      const X* V = A + r0 + c0 * n;  // unit lower trapezoid: V(i, k) valid for i >= k
      Operand vN = opA(V, n, OP_N), vC = opA(V, n, OP_C), vB = opB(V, n, OP_N);
      vN.mask = vC.mask = vB.mask = 1;
      vN.mask_off = vC.mask_off = vB.mask_off = 0;
      Epilogue eg{};
      eg.C = G;
      eg.ldc = kb;
      eg.alpha = 1.0;
      eg.beta = 0.0;
      gemm(dtw, kb, kb, K, vC, vB, eg, nullptr, st);  // G = V^H V
      eig_larft<X><<<1, WY, 0, st>>>(G, tau + c0, (int)kb, Tm);
      BCMG_CHECK_LAUNCH();
      Epilogue e1{};
      e1.C = X1;
      e1.ldc = kb;
      e1.alpha = 1.0;
      e1.beta = 0.0;
      gemm(dtw, kb, n, K, vC, opB(Zx + r0, n, OP_N), e1, nullptr, st);  // X1 = V^H Z[r0:, :]
      Epilogue e2{};
      e2.C = X2;
      e2.ldc = kb;
      e2.alpha = 1.0;
      e2.beta = 0.0;
      gemm(dtw, kb, n, kb, opA(Tm, kb, OP_N), opB(X1, kb, OP_N), e2, nullptr, st);  // X2 = T X1
      Epilogue e3{};
      e3.C = Zx + r0;
      e3.ldc = n;
      e3.alpha = -1.0;
      e3.beta = 1.0;
      gemm(dtw, K, n, kb, vN, opB(X2, kb, OP_N), e3, nullptr, st);  // Z[r0:, :] -= V X2
    }
  }

  pmark(2);
  // rotation parameters stream through NSLOT pinned -> device slots of CH sweeps
  constexpr int KW = 16, CH = 4 * KW, NSLOT = 8;  // enough slots that the host never waits behind the back-transformation
  const size_t cap_rot = (size_t)CH * (size_t)std::max<int64_t>(n, 1);
  const size_t slot_bytes = (cap_rot * sizeof(double2) + (2 * CH + 1) * sizeof(int64_t) + 255) / 256 * 256;
  wb[6].ensure(NSLOT * slot_bytes);
  struct Ring {
    void* host = nullptr;
    cudaEvent_t done[NSLOT] = {};
    cudaStream_t st;
    ~Ring() {
      cudaStreamSynchronize(st);  // the pinned slots are reused by the next call
      for (auto e : done)
        if (e) cudaEventDestroy(e);
    }
  } ring;
  ring.st = st;
  if (ss.eig_host_bytes < NSLOT * slot_bytes) {  // session-owned, grow-only
    if (ss.eig_host) BCMG_CUDA(cudaFreeHost(ss.eig_host));
    ss.eig_host = nullptr;
    ss.eig_host_bytes = 0;
    BCMG_CUDA(cudaHostAlloc(&ss.eig_host, NSLOT * slot_bytes, cudaHostAllocDefault));
    ss.eig_host_bytes = NSLOT * slot_bytes;
  }
  ring.host = ss.eig_host;
  for (auto& e : ring.done) BCMG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  int64_t nrot = 0, nsw = 0;
  // the rotations are real: a complex column is a real column of 2n (re, im) rows
  const int64_t zrows = CP ? 2 * n : n;
  int cur = 0;  // slot the host is writing
  QLRecord rec;
  rec.cs = reinterpret_cast<double2*>(ring.host);
  auto flush = [&] {
    const int64_t ns = (int64_t)rec.top.size(), nr = rec.ncs;
    if (!ns) return;
    char* hb = static_cast<char*>(ring.host) + cur * slot_bytes;
    char* db = static_cast<char*>(wb[6].p) + cur * slot_bytes;
    int64_t* hmeta = reinterpret_cast<int64_t*>(hb + cap_rot * sizeof(double2));
    std::copy(rec.off.begin(), rec.off.end(), hmeta);
    std::copy(rec.top.begin(), rec.top.end(), hmeta + ns + 1);
    BCMG_CUDA(cudaMemcpyAsync(db, hb, nr * sizeof(double2), cudaMemcpyHostToDevice, st));
    int64_t* dmeta = reinterpret_cast<int64_t*>(db + cap_rot * sizeof(double2));
    BCMG_CUDA(cudaMemcpyAsync(dmeta, hmeta, (2 * ns + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    for (int64_t s0 = 0; s0 < ns; s0 += KW) {
      eig_rotate_wave<KW><<<blocks_for(zrows, 32), 32, 0, st>>>(reinterpret_cast<double*>(Zx), zrows, zrows, n,
                                                                reinterpret_cast<const double2*>(db), dmeta,
                                                                dmeta + ns + 1, s0, ns);
      BCMG_CHECK_LAUNCH();
    }
    BCMG_CUDA(cudaEventRecord(ring.done[cur], st));
    nrot += nr;
    nsw += ns;
    cur = (cur + 1) % NSLOT;
    BCMG_CUDA(cudaEventSynchronize(ring.done[cur]));  // that slot's previous batch has been copied and run
    rec.cs = reinterpret_cast<double2*>(static_cast<char*>(ring.host) + cur * slot_bytes);
    rec.ncs = 0;
    rec.off.assign(1, 0);
    rec.top.clear();
  };
  const auto ql0 = std::chrono::steady_clock::now();
  tridiag_ql(d, e, rec, [&] {
    if ((int64_t)rec.top.size() >= CH) flush();
  });
  flush();
  const double host_ql_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ql0).count();
  std::vector<int64_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return d[a] < d[b]; });
  BCMG_CUDA(cudaMemcpyAsync(order_d, order.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  pmark(3);

  pmark(4);
  // ---- 5. phase normalisation + scatter into the caller's shards; eigenvalues
  eig_phase_scatter<X, S><<<(unsigned)n, 256, 0, st>>>(Zx, order_d, n, map);
  BCMG_CHECK_LAUNCH();
  pmark(5);
  if (prof) {
    BCMG_CUDA(cudaEventSynchronize(pe[5]));
    float ms[5];
    for (int k = 0; k < 5; ++k) BCMG_CUDA(cudaEventElapsedTime(&ms[k], pe[k], pe[k + 1]));
    fprintf(stderr,
            "[syevd n=%lld T=%lld] tridiag %.1f ms, back-transform of I %.1f ms (overlaps the host QL), QL + rotation "
            "replay done %.1f ms after it (host loop %.1f ms, %lld rotations, %lld sweeps), phase+scatter %.1f ms\n",
            (long long)n, (long long)T, ms[0], ms[1], ms[2], host_ql_ms, (long long)nrot, (long long)nsw, ms[4]);
    for (auto& e : pe) cudaEventDestroy(e);
  }
  std::sort(d.begin(), d.end());  // == d[order] (stable order of equal keys is immaterial for values)
  if (sizeof(S) == 4 || (CP && sizeof(S) == 8)) {  // float / complex64: float eigenvalues
    std::vector<float> wf(n);
    for (int64_t i = 0; i < n; ++i) wf[i] = (float)d[i];
    BCMG_CUDA(cudaMemcpyAsync(w_out, wf.data(), n * sizeof(float), cudaMemcpyHostToDevice, st));
    BCMG_CUDA(cudaStreamSynchronize(st));
  } else {
    BCMG_CUDA(cudaMemcpyAsync(w_out, d.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
    BCMG_CUDA(cudaStreamSynchronize(st));
  }
}

}  // namespace

// world > 1: the eigensolver's chain is serial (a reflector per column, the
// host QL loop), so the shards are gathered on rank 0 (one point-to-point
// transfer per logical device, device after device -- the all-shards layout of
// a single-process session), solved there by the single-process path, and the
// eigenvector shards / eigenvalues sent back.  The outcome (NO_CONVERGENCE,
// OUT_OF_MEMORY, ...) is agreed on by every rank before any data returns.
void Session::syevd(int dt, int64_t n, int64_t T, int ndev, void* const* shards, bool cyclic, void* w) {
  if (ndev > 16) throw Error(CONFIG, "syevd supports at most 16 logical devices");
  if (world == 1) {
    dispatch_dtype(dt, [&](auto s) { syevd_t<decltype(s)>(*this, n, T, ndev, shards, cyclic, w); });
    return;
  }
  if (ndev % world) throw Error(CONFIG, "logical device count must be a multiple of the process count");
  const size_t esz = dtype_size(dt), wsz = (dt == R32 || dt == C64) ? 4 : 8;
  const int nloc = ndev / world, dev0 = rank * nloc;
  const auto counts = column_counts(n, T, ndev);
  std::vector<int64_t> off(ndev + 1, 0);
  for (int d = 0; d < ndev; ++d) off[d + 1] = off[d] + counts[d];
  cudaStream_t st = user;
  int status = 0;  // 0 ok, else the error code of the root's solve
  std::string msg;
  if (rank == 0) {
    try {
      eig[1].ensure((size_t)n * n * esz);  // the gathered matrix, device after device (eig[1] is free)
    } catch (const Error& e) {
      status = e.code;
      msg = e.what();
    }
  }
  tmp.ensure(4096);
  status = -net->allreduce_min(-status, tmp.p, comm);  // max over ranks
  if (status) throw Error(status, rank == 0 ? msg : "syevd: the gathering rank failed");
  char* g = static_cast<char*>(eig[1].p);
  auto seg = [&](int d) { return (size_t)counts[d] * n * esz; };
  net->group_start();
  if (rank == 0) {
    for (int d = 0; d < nloc; ++d)
      if (seg(d)) BCMG_CUDA(cudaMemcpyAsync(g + off[d] * n * esz, shards[d], seg(d), cudaMemcpyDeviceToDevice, st));
    for (int d = nloc; d < ndev; ++d)
      if (seg(d)) net->recv(g + off[d] * n * esz, seg(d), d / nloc, st);
  } else {
    for (int i = 0; i < nloc; ++i)
      if (seg(dev0 + i)) net->send(shards[i], seg(dev0 + i), 0, st);
  }
  net->group_end();
  if (rank == 0) {
    std::vector<void*> all(ndev);
    for (int d = 0; d < ndev; ++d) all[d] = g + off[d] * n * esz;
    try {
      dispatch_dtype(dt, [&](auto s) { syevd_t<decltype(s)>(*this, n, T, ndev, all.data(), cyclic, w); });
    } catch (const Error& e) {
      status = e.code;
      msg = e.what();
    }
  }
  status = -net->allreduce_min(-status, tmp.p, comm);
  if (status) throw Error(status, rank == 0 ? msg : "syevd failed on the solving rank");
  net->group_start();
  if (rank == 0) {
    for (int d = 0; d < nloc; ++d)
      if (seg(d)) BCMG_CUDA(cudaMemcpyAsync(shards[d], g + off[d] * n * esz, seg(d), cudaMemcpyDeviceToDevice, st));
    for (int d = nloc; d < ndev; ++d)
      if (seg(d)) net->send(g + off[d] * n * esz, seg(d), d / nloc, st);
  } else {
    for (int i = 0; i < nloc; ++i)
      if (seg(dev0 + i)) net->recv(shards[i], seg(dev0 + i), 0, st);
  }
  net->group_end();
  net->bcast(w, (size_t)n * wsz, 0, st);
}

}  // namespace bcmg
