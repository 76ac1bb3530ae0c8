// Vector, reduction and grid-transfer kernels (fp64, HBM-bound, grid-stride).
#pragma once
#include "hf_common.cuh"

namespace hf {

constexpr int RED_THREADS = 256;
constexpr int RED_MAX_BLOCKS = 592;  // 4 x 148 SMs

HF_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic grid reduction: per-block partial sums, the last block to
// finish adds them in block order.  `out` receives the total.
HF_DEV void grid_reduce(double v, double* partials, unsigned* counter, double* out) {
  __shared__ double sh[RED_THREADS / 32];
  __shared__ bool last;
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    v = warp_sum(v);
    if (lane == 0) {
      partials[blockIdx.x] = v;
      __threadfence();
      unsigned t = atomicAdd(counter, 1u);
      last = (t == gridDim.x - 1);
    }
  }
  __syncthreads();
  if (last) {
    double s = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) s += __ldcg(partials + i);
    s = warp_sum(s);
    if (lane == 0) sh[w] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
      *out = t;
      *counter = 0u;
    }
  }
}

// reverse halo add of a multi-GPU slab interface: y[i] += recv[i] on the
// unconstrained DoFs (constrained ones hold the identity value on both ranks)
__global__ void k_halo_add(long long n, double* __restrict__ y, const double* __restrict__ recv,
                           const unsigned char* __restrict__ mask) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (!mask[i]) y[i] += recv[i];
}

// interface DoFs of a box partition (distributed.py Box): buf[i] = y[idx[i]]
// packs the partial sums sent to one neighbour; y[idx[i]] += buf[i] adds a
// neighbour's partials on the unconstrained DoFs.  Within one neighbour's list
// every idx is distinct, so the add needs no atomics.
__global__ void k_pack_idx(long long n, const int* __restrict__ idx, const double* __restrict__ y,
                           double* __restrict__ buf) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    buf[i] = y[idx[i]];
}
__global__ void k_unpack_add_idx(long long n, const int* __restrict__ idx, double* __restrict__ y,
                                 const double* __restrict__ buf, const unsigned char* __restrict__ mask) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int j = idx[i];
    if (!mask[j]) y[j] += buf[i];
  }
}

// dot product over the DoFs a rank owns (own[i] != 0), deterministic order
__global__ void k_dot_owned(long long n, const double* __restrict__ a, const double* __restrict__ b,
                            const unsigned char* __restrict__ own, double* partials, unsigned* counter, double* out) {
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (own[i]) s = fma(a[i], b[i], s);
  grid_reduce(s, partials, counter, out);
}

// fp64 throughput probe (the denominator of the fp64 roofline; MEASURED_PEAKS
// has no fp64 entry): 8 independent DFMA chains per thread
__global__ void k_probe_dfma(long long iters, double* sink) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + 1e-3 * (threadIdx.x + k);
  const double m = 0.999999, c = 1e-7;
  for (long long i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) sink[0] = s;  // keep the chains alive
}

inline unsigned red_blocks(long long n) {
  long long b = (n + RED_THREADS * 4 - 1) / (RED_THREADS * 4);
  if (b < 1) b = 1;
  if (b > RED_MAX_BLOCKS) b = RED_MAX_BLOCKS;
  return (unsigned)b;
}

template <typename T = double>
__global__ void k_dot(long long n, const T* __restrict__ a, const T* __restrict__ b, double* partials,
                      unsigned* counter, double* out, const int* skip) {
  if (skip && *skip) return;
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s = fma((double)a[i], (double)b[i], s);
  grid_reduce(s, partials, counter, out);
}

// y[i] = mask[i] ? (x ? x[i] : mval) : 0
template <typename T = double>
__global__ void k_fill_masked(long long n, T* __restrict__ y, const T* __restrict__ x,
                              const uint8_t* __restrict__ mask, double mval, const int* skip) {
  asm volatile("griddepcontrol.launch_dependents;");  // a PDL secondary (the apply) may start now
  if (skip && *skip) return;
  // four elements per thread and iteration, every load issued before any use
  // (x is read whether or not the mask selects it: no load behind a branch)
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint8_t m[4];
    T v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      m[k] = mask[i + k * stride];
      v[k] = x ? x[i + k * stride] : (T)mval;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) y[i + k * stride] = m[k] ? v[k] : (T)0;
  }
  for (; i < n; i += stride) {
    const T v = x ? x[i] : (T)mval;
    y[i] = mask[i] ? v : (T)0;
  }
}

// Chebyshev step (multigrid.py:176-205, 280-296):
//   z = inv_d * (b - ax)        (ax == nullptr -> A x = 0)
//   first:  d = z / theta       else d = cd * d + cz * z
//   x = (x_zero ? 0 : x) + d
//   fill_mask != null: also y_next = mask ? x_new : 0, the initialisation of
//   the NEXT tangent apply (which is launched as this kernel's programmatic
//   dependent and skips its own fill); y_next may alias ax (read first)
//   after_apply: this launch is the programmatic dependent of the cell kernel
//   that wrote ax (hf_cheb_step_after_apply).  Its blocks become resident
//   while that kernel drains, prefetch into L2 the first operands the cell
//   kernel does not write (inv_d, b, d, x) and wait for its completion before
//   they load anything.  The cell kernel releases its dependents after its
//   own wait, so every kernel before it has completed by then.
template <typename T = double>
__global__ void k_cheb(long long n, T* __restrict__ x, T* __restrict__ d, const T* __restrict__ b, const T* ax,
                       const T* __restrict__ inv_d, int first, double theta, double cd, double cz, int x_zero,
                       const int* skip, const uint8_t* __restrict__ fill_mask, T* y_next, int after_apply) {
  asm volatile("griddepcontrol.launch_dependents;");
  const long long st = (long long)gridDim.x * blockDim.x;
  if (after_apply) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x + u * st;
      if (i < n) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(inv_d + i));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(b + i));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(x + i));
        if (!first) asm volatile("prefetch.global.L2 [%0];" ::"l"(d + i));
      }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (skip && *skip) return;
  // four elements per thread and iteration with every load issued before any
  // use (one element per iteration left the 64^3 step latency bound at 0.77 of
  // HBM); per element the arithmetic is unchanged, and ax is read before
  // y_next (which may alias it) is written
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += 4 * st) {
    double vb[4], va[4], vi[4], vd[4], vx[4];
    uint8_t vm[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * st;
      const bool in = i < n;
      vi[u] = in ? (double)inv_d[i] : 0.0;
      vb[u] = in ? (double)b[i] : 0.0;
      va[u] = (in && ax) ? (double)ax[i] : 0.0;
      vd[u] = (in && !first) ? (double)d[i] : 0.0;
      vx[u] = (in && !x_zero) ? (double)x[i] : 0.0;
      vm[u] = (in && fill_mask) ? fill_mask[i] : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * st;
      if (i >= n) break;
      double z = vi[u] * (vb[u] - va[u]);
      double di = first ? z / theta : cd * vd[u] + cz * z;
      d[i] = (T)di;
      const T xn = (T)(x_zero ? di : vx[u] + di);
      x[i] = xn;
      if (fill_mask) y_next[i] = vm[u] ? xn : (T)0;
    }
  }
}

// Chebyshev step in three-term form: the direction is not stored, it is the
// difference of the last two iterates, d_{k-1} = x_k - x_{k-1}:
//   z = inv_d * (b - ax)                     (ax == nullptr -> A x_k = 0)
//   d = first ? z / theta : cd * (x_k - x_{k-1}) + cz * z
//   x_{k+1} = x_k + d, written over x_{k-1} (xo); the caller swaps the buffers
//   xk_zero: x_k = 0 (not read); xprev_zero: x_{k-1} = 0 (not read)
// One vector write less than k_cheb (57 instead of 65 B per DoF); the iterates
// agree with the stored-direction form to rounding (x_k - x_{k-1} recovers
// d_{k-1} to an ulp of x).  fill_mask / y_next / after_apply as in k_cheb.
template <typename T = double>
__global__ void k_cheb3(long long n, const T* __restrict__ xk, T* __restrict__ xo, const T* __restrict__ b,
                        const T* ax, const T* __restrict__ inv_d, int first, double theta, double cd, double cz,
                        int xk_zero, int xprev_zero, const uint8_t* __restrict__ fill_mask, T* y_next,
                        int after_apply) {
  asm volatile("griddepcontrol.launch_dependents;");
  const long long st = (long long)gridDim.x * blockDim.x;
  if (after_apply) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x + u * st;
      if (i < n) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(inv_d + i));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(b + i));
        if (!xk_zero) asm volatile("prefetch.global.L2 [%0];" ::"l"(xk + i));
        if (!first && !xprev_zero) asm volatile("prefetch.global.L2 [%0];" ::"l"(xo + i));
      }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  const bool rd_prev = !first && !xprev_zero;
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += 4 * st) {
    double vb[4], va[4], vi[4], vp[4], vx[4];
    uint8_t vm[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * st;
      const bool in = i < n;
      vi[u] = in ? (double)inv_d[i] : 0.0;
      vb[u] = in ? (double)b[i] : 0.0;
      va[u] = (in && ax) ? (double)ax[i] : 0.0;
      vp[u] = (in && rd_prev) ? (double)xo[i] : 0.0;
      vx[u] = (in && !xk_zero) ? (double)xk[i] : 0.0;
      vm[u] = (in && fill_mask) ? fill_mask[i] : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * st;
      if (i >= n) break;
      const double z = vi[u] * (vb[u] - va[u]);
      const double di = first ? z / theta : cd * (vx[u] - vp[u]) + cz * z;
      const T xn = (T)(vx[u] + di);
      xo[i] = xn;
      if (fill_mask) y_next[i] = vm[u] ? xn : (T)0;
    }
  }
}

// r = b - ax, r[mask] = 0
template <typename T = double>
__global__ void k_resid_masked(long long n, T* __restrict__ r, const T* __restrict__ b, const T* __restrict__ ax,
                               const uint8_t* __restrict__ mask) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    r[i] = mask[i] ? (T)0 : (T)((double)b[i] - (double)ax[i]);
}

// ||b - ax||^2 -> scal[out]; if sqrt(.) <= scal[tgt] set *flag (coarse_solve check)
template <typename T = double>
__global__ void k_resnorm_check(long long n, const T* __restrict__ b, const T* __restrict__ ax, double* partials,
                                unsigned* counter, double* scal, int out, int tgt, int* flag) {
  if (*flag) return;
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double r = (double)b[i] - (double)ax[i];
    s = fma(r, r, s);
  }
  grid_reduce(s, partials, counter, scal + out);
  // the last block wrote scal[out]; the flag is set by a follow-up scalar kernel
}

// scalar bookkeeping kernels (single thread)
// op 0: flag = sqrt(scal[a]) <= scal[b]
// op 1: scal[b] = rel * sqrt(scal[a]); flag = (scal[a] == 0)
__global__ void k_scalar(int op, double* scal, int a, int b, double rel, int* flag) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (op == 0) {
    if (!*flag && sqrt(scal[a]) <= scal[b]) *flag = 1;
  } else if (op == 1) {
    scal[b] = rel * sqrt(scal[a]);
    *flag = (scal[a] == 0.0) ? 1 : 0;
  }
}

// CG updates (solver.py:57-75) with device-resident scalars
//   alpha = scal[irz] / scal[ipap];  x += alpha p;  r -= alpha ap;  scal[irr] = r.r
__global__ void k_cg_xr(long long n, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                        const double* __restrict__ ap, double* scal, int irz, int ipap, int irr, double* partials,
                        unsigned* counter) {
  const double alpha = scal[irz] / scal[ipap];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    double ri = r[i] - alpha * ap[i];
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  grid_reduce(s, partials, counter, scal + irr);
}

//   beta = scal[irzn] / scal[irz];  p = z + beta p
//   fill_mask != null: also y_next = mask ? p_new : 0, the initialisation of
//   the tangent apply A p that follows (launched as this kernel's programmatic
//   dependent, hf_tangent_apply_after_fill), as k_cheb does for the smoother
__global__ void k_cg_p(long long n, double* __restrict__ p, const double* __restrict__ z, const double* scal, int irzn,
                       int irz, const uint8_t* __restrict__ fill_mask, double* __restrict__ y_next) {
  asm volatile("griddepcontrol.launch_dependents;");
  const double beta = scal[irzn] / scal[irz];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double pn = z[i] + beta * p[i];
    p[i] = pn;
    if (fill_mask) y_next[i] = fill_mask[i] ? pn : 0.0;
  }
}

// z = inv_d * r; scal[out] = r.z  (Jacobi-preconditioned Lanczos, multigrid.py:126-153)
__global__ void k_jacobi_dot(long long n, double* __restrict__ z, const double* __restrict__ r,
                             const double* __restrict__ inv_d, double* partials, unsigned* counter, double* out) {
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double zi = inv_d[i] * r[i];
    z[i] = zi;
    s = fma(r[i], zi, s);
  }
  grid_reduce(s, partials, counter, out);
}

// y = a x + b y  (general axpby)
// ---- Jacobi-PCG / Lanczos range estimate with device-side scalars
// (estimate_eigenvalue_range, multigrid.py:112-166).  scal: [0] rz, [1] pAp,
// [2] rz_new, [3] beta; st: [0] stop flag, [1] recorded steps; ab[2k] alpha_k,
// ab[2k+1] beta_k.  No host round trip per iteration.
__global__ void k_lanczos_r(long long n, double* __restrict__ r, const double* __restrict__ ap, const double* scal,
                            const int* st) {
  if (st[0] || scal[1] <= 0.0) return;
  const double a = -(scal[0] / scal[1]);  // r -= alpha ap
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    r[i] = fma(a, ap[i], r[i]);
}

// k_lanczos_r and k_jacobi_dot in one pass (same arithmetic per element, same
// reduction tree as k_jacobi_dot): r -= alpha ap unless the run has stopped,
// z = inv_d r, scal[2] = r.z
__global__ void k_lanczos_rz(long long n, double* __restrict__ r, double* __restrict__ z,
                             const double* __restrict__ ap, const double* __restrict__ inv_d, double* scal,
                             const int* st, double* partials, unsigned* counter) {
  const bool upd = !(st[0] || scal[1] <= 0.0);
  const double a = upd ? -(scal[0] / scal[1]) : 0.0;
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double ri = upd ? fma(a, ap[i], r[i]) : r[i];
    if (upd) r[i] = ri;
    const double zi = inv_d[i] * ri;
    z[i] = zi;
    s = fma(ri, zi, s);
  }
  grid_reduce(s, partials, counter, scal + 2);
}

// one thread: the reference's tests and recording after r.z (rz_new) is known
__global__ void k_lanczos_scalar(double* scal, int* st, double* ab) {
  if (st[0]) return;
  const double rz = scal[0], pap = scal[1], rzn = scal[2];
  const int k = st[1];
  if (pap <= 0.0) {  // multigrid.py: break before recording
    st[0] = 1;
    return;
  }
  const double alpha = rz / pap;
  ab[2 * k] = alpha;
  st[1] = k + 1;
  if (rzn <= 1e-28 * rz || !isfinite(rzn)) {
    st[0] = 1;
    return;
  }
  const double beta = rzn / rz;
  ab[2 * k + 1] = beta;
  scal[0] = rzn;
  scal[3] = beta;
}

// p = z + beta p
__global__ void k_lanczos_p(long long n, double* __restrict__ p, const double* __restrict__ z, const double* scal,
                            const int* st) {
  if (st[0]) return;
  const double b = scal[3];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = fma(b, p[i], z[i]);
}

// k_lanczos_p that also writes y_next = mask ? p_new : 0, the initialisation of
// the application A p of the next iteration (its programmatic dependent)
__global__ void k_lanczos_p_fill(long long n, double* __restrict__ p, const double* __restrict__ z, const double* scal,
                                 const int* st, const uint8_t* __restrict__ mask, double* __restrict__ y_next) {
  asm volatile("griddepcontrol.launch_dependents;");
  if (st[0]) return;
  const double b = scal[3];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double pn = fma(b, p[i], z[i]);
    p[i] = pn;
    y_next[i] = mask[i] ? pn : 0.0;
  }
}

// st[0] = !(rz > 0 and finite), st[1] = 0 (the check before the first iteration)
__global__ void k_lanczos_init(const double* scal, int* st) {
  const double rz = scal[0];
  st[0] = (rz <= 0.0 || !isfinite(rz)) ? 1 : 0;
  st[1] = 0;
}

__global__ void k_axpby(long long n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = a * x[i] + (b == 0.0 ? 0.0 : b * y[i]);
}

// out[node*C + c] -= traction[c] * sw[node]; out[mask] = 0   (operators.py:221-223)
__global__ void k_resid_finalize(long long n_nodes, int C, double* __restrict__ out, const double* __restrict__ sw,
                                 double t0, double t1, double t2, int has_traction, const uint8_t* __restrict__ mask) {
  const double tr[3] = {t0, t1, t2};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n_nodes * C;
       i += (long long)gridDim.x * blockDim.x) {
    double v = out[i];
    if (has_traction) v -= tr[i % C] * sw[i / C];
    out[i] = mask[i] ? 0.0 : v;
  }
}

// One axis of a tensor-product 1D operator on a (n2, n1, n0, C) lattice array
// (multigrid.py:39-55).  Row o of the banded 1D matrix is (cols, w)[rowptr[o]..].
// mode 0: out = v;  mode 1: out = mask ? 0 : v;  mode 2: out += mask ? 0 : v
template <typename TI = double, typename TO = double>
__global__ void k_axis(const TI* __restrict__ in, TO* __restrict__ out, int n0, int n1, int n2, int C, int axis,
                       int nout, const int* __restrict__ rowptr, const int* __restrict__ cols,
                       const double* __restrict__ w, const uint8_t* __restrict__ mask, int mode) {
  // 32-bit index arithmetic: both lattices hold < 2^31 DoFs (hf_space_create),
  // and 32-bit divisions by the run-time extents are a fraction of the cost of
  // 64-bit ones (four per element)
  const unsigned m0 = axis == 0 ? nout : n0, m1 = axis == 1 ? nout : n1, m2 = axis == 2 ? nout : n2;
  const unsigned total = m0 * m1 * m2 * (unsigned)C;
  const unsigned in_stride = axis == 0 ? C : (axis == 1 ? (unsigned)n0 * C : (unsigned)n0 * n1 * C);
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    unsigned r = t;
    const unsigned c = r % (unsigned)C;
    r /= (unsigned)C;
    const unsigned i0 = r % m0;
    r /= m0;
    const unsigned i1 = r % m1;
    const unsigned i2 = r / m1;
    const unsigned o = axis == 0 ? i0 : (axis == 1 ? i1 : i2);
    const unsigned base = (((axis == 2 ? 0u : i2) * (unsigned)n1 + (axis == 1 ? 0u : i1)) * (unsigned)n0 +
                           (axis == 0 ? 0u : i0)) * (unsigned)C + c;
    double s = 0.0;
    for (int k = rowptr[o]; k < rowptr[o + 1]; ++k)
      s = fma(w[k], (double)in[base + (unsigned)cols[k] * in_stride], s);
    if (mode == 0) out[t] = (TO)s;
    else if (mode == 1) out[t] = mask[t] ? (TO)0 : (TO)s;
    else if (!mask[t]) out[t] = (TO)((double)out[t] + s);
  }
}

// nodal injection onto the coarse lattice (multigrid.py:76-92)
__global__ void k_inject(const double* __restrict__ uf, double* __restrict__ uc, int nc0, int nc1, int nc2, int nf0,
                         int nf1, int C, const uint8_t* __restrict__ cmask, int keep) {
  long long total = (long long)nc0 * nc1 * nc2 * C;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    long long r = t;
    int c = (int)(r % C);
    r /= C;
    int i0 = (int)(r % nc0);
    r /= nc0;
    int i1 = (int)(r % nc1);
    int i2 = (int)(r / nc1);
    long long f = (((long long)(2 * i2) * nf1 + 2 * i1) * nf0 + 2 * i0) * C + c;
    double v = uf[f];
    uc[t] = (!keep && cmask[t]) ? 0.0 : v;
  }
}

}  // namespace hf
