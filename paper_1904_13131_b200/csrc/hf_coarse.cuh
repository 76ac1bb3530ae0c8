// Coarse-level Chebyshev solve as ONE persistent cooperative kernel
// (coarse_solve, multigrid.py:255-306; LevelOperator.coarse_settings 248-252).
//
// The coarsest GMG level (e.g. 4^3 Q2: 2,187 DoFs) is latency bound: the
// reference's 99 operator applications + Chebyshev updates + every-4th
// residual test cost ~7.5 us each as separate graph launches.  Here the level
// operator is the assembled CSR of the same tangent (constrained rows and
// columns cleared, unit diagonal: exactly the matrix-free apply's zero-in /
// identity-out semantics), split over the CTAs' shared memory, and the whole
// iteration runs inside one kernel with a grid barrier per application:
//   * rows are split over the CTAs; one warp per row forms (A x)_i;
//   * the Chebyshev update of row i needs only (A x)_i and row-local vectors,
//     so it is fused into the SpMV; each CTA keeps its rows of the matrix and
//     its rows' x and d in shared memory, and per application gathers only the
//     entries of the (double-buffered) iterate its rows touch;
//   * every `degree`-th application the squared residual norm is reduced in a
//     fixed order (per-warp partials -> per-CTA partials -> every CTA sums the
//     CTA partials in index order), so every CTA takes the same stop decision
//     and the result is deterministic.
// Cooperative launch guarantees co-residency of the CTAs for the barrier.
// A level whose whole matrix fits one CTA's shared memory (2D coarsest levels,
// e.g. 4^2 Q2: 162 DoFs) runs as ONE CTA of COARSE_THREADS_1 threads: the
// iterate stays in shared memory and every grid barrier becomes a
// __syncthreads (the ~1.2 us grid barrier and the L2 round trip of the
// gather were ~3.2 us of every application at config 1).
#pragma once
#include <cooperative_groups.h>

#include "hf_common.cuh"

namespace hf {

// Per-CTA block of the level matrix, packed on the host by hf_coarse_create
// (16-byte aligned sections): the CTA's rows [r0, r0 + rows), the sorted
// distinct columns they touch (nu of them), the CSR of those rows with
// columns renumbered into that list, and the values.  The whole block is
// copied to shared memory once; per application the CTA gathers only the nu
// iterate entries it needs.
struct CoarseBlock {
  int r0, rows, nu, nnz;
  // followed by: double val[nnz]; int ucol[nu]; int rowptr[rows + 1]; unsigned short lcol[nnz]
};

__host__ __device__ __forceinline__ size_t coarse_align16(size_t b) { return (b + 15) & ~(size_t)15; }

struct CoarseArgs {
  int n;                      // rows of the level
  const unsigned char* blob;  // packed CoarseBlocks
  const long long* boff;      // byte offset of CTA c's block
  const double* b;
  const double* inv_d;
  double* x;                  // result (and buffer 0 of the iterate)
  double* xb;                 // buffer 1 of the iterate
  double* d;                  // Chebyshev direction (written back at the end)
  double* partials;           // per-CTA partial sums (gridDim.x)
  double* scal;               // scal[0] = ||b||^2, scal[1] = target, scal[2] = last ||b - A x||^2
  int* flag;                  // 1: converged (or b == 0) before the cap
  double theta, delta, sigma, rel_target;
  int max_applications, degree;
};

constexpr int COARSE_THREADS = 256;
constexpr int COARSE_THREADS_1 = 1024;  // the single-CTA form: 4 lanes per row (k_coarse_cheb<1024, 4>)

// sum over the grid of one value per thread, in a fixed order; every thread
// of every CTA returns the same total (one CTA: no partials, no grid barrier)
HF_DEV double coarse_grid_sum(double v, double* red, const CoarseArgs& a, cooperative_groups::grid_group& grid) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (gridDim.x == 1) {
    if (warp == 0) {
      double t = lane < nw ? red[lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) red[32] = t;
    }
    __syncthreads();
    const double t = red[32];
    __syncthreads();  // red is reused by the next reduction
    return t;
  }
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[w];
    a.partials[blockIdx.x] = s;
  }
  grid.sync();
  // warp 0: lane l sums partials l, l + 32, ... (independent loads, fixed
  // order), then a fixed shuffle tree; broadcast through shared memory
  if (warp == 0) {
    double t = 0.0;
    for (int c = lane; c < (int)gridDim.x; c += 32) t += __ldcg(a.partials + c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  const double t = red[0];
  __syncthreads();  // red is reused by the next reduction
  return t;
}

// dynamic shared memory: the CTA's CoarseBlock (minus header), then the
// gathered iterate entries (nu), then per own row A x, d, x, b and inv_d
template <int NT, int G>
__global__ void __launch_bounds__(NT) k_coarse_cheb(const CoarseArgs a) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  extern __shared__ __align__(16) unsigned char csm[];
  __shared__ double red[33];
  const bool single = gridDim.x == 1;  // the iterate lives in shared memory (xl)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned char* gb = a.blob + a.boff[blockIdx.x];
  const CoarseBlock hb = *reinterpret_cast<const CoarseBlock*>(gb);
  const int r0 = hb.r0, r1 = hb.r0 + hb.rows, nu = hb.nu, nnz = hb.nnz;
  HF_ASSERT(r0 >= 0 && r1 <= a.n && nu >= 0 && nnz >= 0);
  // copy the block body to shared memory (16-byte vectors)
  const size_t body = coarse_align16(8ull * nnz) + coarse_align16(4ull * nu) + coarse_align16(4ull * (hb.rows + 1)) +
                      coarse_align16(2ull * nnz);
  {
    const uint4* src = reinterpret_cast<const uint4*>(gb + 16);
    uint4* dst = reinterpret_cast<uint4*>(csm);
    for (size_t i = threadIdx.x; i < body / 16; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  const double* val = reinterpret_cast<const double*>(csm);
  const int* ucol = reinterpret_cast<const int*>(csm + coarse_align16(8ull * nnz));
  const int* rowptr = reinterpret_cast<const int*>(reinterpret_cast<const unsigned char*>(ucol) + coarse_align16(4ull * nu));
  const unsigned short* lcol =
      reinterpret_cast<const unsigned short*>(reinterpret_cast<const unsigned char*>(rowptr) + coarse_align16(4ull * (hb.rows + 1)));
  double* xs = reinterpret_cast<double*>(csm + body);
  double* axl = xs + nu;
  double* dl = axl + hb.rows;
  double* xl = dl + hb.rows;
  double* bl = xl + hb.rows;   // this CTA's rows of b and inv_d, read once
  double* idl = bl + hb.rows;
  for (int l = threadIdx.x; l < hb.rows; l += blockDim.x) {
    bl[l] = __ldg(a.b + r0 + l);
    idl[l] = __ldg(a.inv_d + r0 + l);
  }
  __syncthreads();
  // ||b||^2, target, flag = (||b|| == 0)   (hf_scalar_op op 1)
  double bb = 0.0;
  for (int l = threadIdx.x; l < hb.rows; l += blockDim.x) bb = fma(bl[l], bl[l], bb);
  const double bn2 = coarse_grid_sum(bb, red, a, grid);
  const double target = a.rel_target * sqrt(bn2);
  bool done = bn2 == 0.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.scal[0] = bn2;
    a.scal[1] = target;
    a.flag[0] = done ? 1 : 0;
  }
  // first step from x = 0: d = inv_d b / theta, x = d
  for (int l = threadIdx.x; l < hb.rows; l += blockDim.x) {
    const double dd = idl[l] * bl[l] / a.theta;
    dl[l] = dd;
    xl[l] = dd;
    if (!single) a.x[r0 + l] = dd;
  }
  if (single)
    __syncthreads();
  else
    grid.sync();
  double rho_old = 1.0 / a.sigma;
  const double* xin = a.x;
  double* xout = a.xb;
  for (int step = 2; step <= a.max_applications && !done; ++step) {
    const bool check = step % a.degree == 0;
    const double rho = 1.0 / (2.0 * a.sigma - rho_old);
    const double cd = rho * rho_old, cz = 2.0 * rho / a.delta;
    // gather the iterate entries this CTA's rows touch (one L2 round trip)
    for (int j = threadIdx.x; j < nu; j += blockDim.x) {
      HF_ASSERT(ucol[j] >= 0 && ucol[j] < a.n);
      xs[j] = single ? xl[ucol[j]] : __ldcg(xin + ucol[j]);
    }
    __syncthreads();
    // (A x)_i of this CTA's rows from shared memory, G lanes per row (G = 32:
    // one warp per row; the single-CTA form uses small groups so that each
    // warp's row rounds are few and short).  The row rounds are warp-uniform,
    // so every lane reaches the shuffles.
    double rr = 0.0;
    for (int base = warp * (32 / G); base < hb.rows; base += nw * (32 / G)) {
      const int l = base + lane / G;
      const bool on = l < hb.rows;
      double s = 0.0;
      if (on) {
        const int k0 = rowptr[l], k1 = rowptr[l + 1];
        HF_ASSERT(k0 >= 0 && k1 <= nnz && k0 <= k1);
        for (int k = k0 + lane % G; k < k1; k += G) {
          HF_ASSERT(lcol[k] < nu);
          s = fma(val[k], xs[lcol[k]], s);
        }
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (on && lane % G == 0) {
        axl[l] = s;
        const double r = bl[l] - s;
        if (check) rr = fma(r, r, rr);
      }
    }
    if (check) {
      const double rn2 = coarse_grid_sum(rr, red, a, grid);  // includes a grid barrier
      if (blockIdx.x == 0 && threadIdx.x == 0) a.scal[2] = rn2;
      if (sqrt(rn2) <= target) {
        done = true;
        if (blockIdx.x == 0 && threadIdx.x == 0) a.flag[0] = 1;
        break;
      }
    } else {
      __syncthreads();
    }
    // Chebyshev update of this CTA's rows (hf_cheb_step)
    for (int l = threadIdx.x; l < hb.rows; l += blockDim.x) {
      const double z = idl[l] * (bl[l] - axl[l]);
      const double dd = cd * dl[l] + cz * z;
      dl[l] = dd;
      const double xn = xl[l] + dd;
      xl[l] = xn;
      if (!single) xout[r0 + l] = xn;
    }
    rho_old = rho;
    xin = xout;
    xout = xout == a.x ? a.xb : a.x;
    if (single)
      __syncthreads();
    else
      grid.sync();
  }
  // the iterate (and the direction) of this CTA's rows
  for (int l = threadIdx.x; l < hb.rows; l += blockDim.x) {
    a.x[r0 + l] = xl[l];
    a.d[r0 + l] = dl[l];
  }
}

// blob value of update slot u = sum of its element-matrix entries (ascending)
__global__ void k_coarse_values(int nupd, const int* __restrict__ cptr, const int* __restrict__ cidx,
                                const double* __restrict__ elem, unsigned char* blob, const long long* __restrict__ uoff) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= nupd) return;
  double v = 0.0;
  for (int k = cptr[u]; k < cptr[u + 1]; ++k) {
    HF_ASSERT(cidx[k] >= 0);
    v += elem[cidx[k]];
  }
  HF_ASSERT(uoff[u] >= 16 && (uoff[u] & 7) == 0);
  *reinterpret_cast<double*>(blob + uoff[u]) = v;
}

}  // namespace hf
