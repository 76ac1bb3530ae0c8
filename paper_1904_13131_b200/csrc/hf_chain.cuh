// Chained-contraction apply kernel of the matrix-free Neo-Hookean tangent
// (sm_100a, fp64): the same warp tiles, TMA cache ring, gather and atomic
// scatter as k_apply_line (hf_line.cuh), with fewer line-buffer round trips.
//
// k_apply_line evaluates gradients by collocation (interpolate to the Gauss
// points along every axis, then differentiate there) and hands the y and z
// derivatives to the x-line owner through shared memory, which costs 10 axis
// phases and ~23 line-buffer accesses per thread and value.  Here the unit
// gradient is evaluated the way the reference writes it (fespace.py:230-239:
// the derivative table on axis g, the value table on the others), with the
// per-axis tables applied in a chain that carries several fields:
//
//   Z  z-lines : gather x (constrained DoFs zeroed);  a = V_z u,  b = D_z u       -> buf0, buf1
//   Y  y-lines : c = V_y a,  d = D_y a,  e = V_y b                               -> buf0, buf2, buf1
//   X  x-lines : G_x = D_x c,  G_y = V_x d,  G_z = V_x e                         (registers)
//   P  x-lines : q-point physics of the caching variant (operators.py:341-392), in place
//   X' x-lines : f1 = D_x^T q_x,  f2 = V_x^T q_y,  f3 = V_x^T q_z                 -> buf0, buf1, buf2
//   Y' y-lines : g1 = V_y^T f1 + D_y^T f2,  g2 = V_y^T f3                        -> buf0, buf1
//   Z' z-lines : y_loc = V_z^T g1 + D_z^T g2, atomic scatter-add (fespace.py:307-324)
//
// Four transposes (2, 3, 3 and 2 fields) instead of the collocation path's
// ten phases; the point phase reads no gradients from shared memory and
// writes none back.  The price is 16 instead of 12 line contractions per
// component (the reference's own count).  Each Y / Y' thread writes exactly
// the sites it read, so the fields are updated in place without a barrier.
// 2D drops the Y phases (gather along y, X reads a, b).
//
// Reference correspondence: gather fespace.py:291-293 + operators.py:333-334;
// evaluate fespace.py:224-239; q-point physics operators.py:341-392; integrate
// fespace.py:258-288; scatter fespace.py:296-324.
#pragma once
#include "hf_line.cuh"

namespace hf {

template <int DIM, int N, int VAR, typename ST = double>
struct ChainPlan {
  using K = LineCfg<DIM, N>;
  static constexpr int NB = DIM;  // line buffers (3 fields in flight at the Y / X' transposes in 3D)
  static constexpr int NF = (VAR == SCALAR) ? 2 + DIM * DIM : CacheFields<DIM, VAR>::NF;
  static constexpr long long CH = TileLayout<DIM, N>::template chunk_e<sizeof(ST)>(NF);
  static constexpr size_t BUDGET = 226 * 1024;
  static constexpr size_t perw(int rw) {
    return sizeof(ST) * (size_t)rw * CH + sizeof(double) * (size_t)NB * LineMap<DIM, N>::BUF + 16 * rw;
  }
  static constexpr int RW = N < 3 ? N : 3;
  static constexpr int W0 = (int)(BUDGET / perw(RW));
  static constexpr int WMAX = VAR == SCALAR ? 8 : 12;
  static constexpr int W = W0 > WMAX ? WMAX : (W0 < 1 ? 1 : W0);
  static constexpr int NT = 32 * W;
  static constexpr size_t SMEM = (size_t)W * perw(RW);
};

// out[c] = M applied along the line (forward: out[o] = sum_l M[l][o] in[l])
template <int DIM, int N, bool TR>
HF_DEV void cl(const double (&M)[N][N], const double (&in)[DIM][N], double (&out)[DIM][N]) {
#pragma unroll
  for (int c = 0; c < DIM; ++c) c1d<N, TR>(M, in[c], out[c]);
}
// out[c] = A^T a + B^T b along the line (transposed contractions summed)
template <int DIM, int N>
HF_DEV void cl2t(const double (&A)[N][N], const double (&a)[DIM][N], const double (&B)[N][N],
                 const double (&b)[DIM][N], double (&out)[DIM][N]) {
#pragma unroll
  for (int c = 0; c < DIM; ++c)
#pragma unroll
    for (int l = 0; l < N; ++l) {
      double s = 0.0;
#pragma unroll
      for (int o = 0; o < N; ++o) s = fma(A[l][o], a[c][o], s);
#pragma unroll
      for (int o = 0; o < N; ++o) s = fma(B[l][o], b[c][o], s);
      out[c][l] = s;
    }
}

// Unit-cell gradients of the (masked) last-axis nodal line values u0 into the
// x-line owner's registers: G[a][c][iq] = d/dxi_a of component c at Gauss
// point iq of this thread's x-line.  Uses buffers b0..b(DIM-1) as scratch.
template <int DIM, int N>
HF_DEV void chain_eval(const TabLine<N>& T, const double (&u0)[DIM][N], bool live, const LineOff<DIM, N>& lo,
                       double* (&buf)[DIM], double (&G)[DIM][DIM][N]) {
  if (live) {
    double a[DIM][N], b[DIM][N];
    cl<DIM, N, false>(T.V, u0, a);
    cl<DIM, N, false>(T.D, u0, b);
    st_line<DIM, N, DIM - 1>(buf[0], lo, a);
    st_line<DIM, N, DIM - 1>(buf[1], lo, b);
  }
  __syncwarp();
  if constexpr (DIM == 3) {
    if (live) {
      double a[DIM][N], b[DIM][N], t[DIM][N];
      ld_line<DIM, N, 1>(buf[0], lo, a);
      ld_line<DIM, N, 1>(buf[1], lo, b);
      cl<DIM, N, false>(T.V, a, t);
      st_line<DIM, N, 1>(buf[0], lo, t);  // c, in place of a
      cl<DIM, N, false>(T.D, a, t);
      st_line<DIM, N, 1>(buf[2], lo, t);  // d
      cl<DIM, N, false>(T.V, b, t);
      st_line<DIM, N, 1>(buf[1], lo, t);  // e, in place of b
    }
    __syncwarp();
    if (live) {
      double c[DIM][N];
      ld_line<DIM, N, 0>(buf[0], lo, c);
      cl<DIM, N, false>(T.D, c, G[0]);
      ld_line<DIM, N, 0>(buf[2], lo, c);
      cl<DIM, N, false>(T.V, c, G[1]);
      ld_line<DIM, N, 0>(buf[1], lo, c);
      cl<DIM, N, false>(T.V, c, G[2]);
    }
  } else {
    if (live) {
      double c[DIM][N];
      ld_line<DIM, N, 0>(buf[0], lo, c);
      cl<DIM, N, false>(T.D, c, G[0]);
      ld_line<DIM, N, 0>(buf[1], lo, c);
      cl<DIM, N, false>(T.V, c, G[1]);
    }
  }
}

// Transposed chain: from the queued point values Q[a][c][iq] of this thread's
// x-line to the nodal values v of its last-axis line (before the scatter).
// The X' phase writes only this thread's own x-line sites, which it alone
// read in the X phase, so no barrier is needed before it.
template <int DIM, int N>
HF_DEV void chain_integrate(const TabLine<N>& T, const double (&Q)[DIM][DIM][N], bool live,
                            const LineOff<DIM, N>& lo, double* (&buf)[DIM], double (&v)[DIM][N]) {
  if (live) {
    double f[DIM][N];
    cl<DIM, N, true>(T.D, Q[0], f);
    st_line<DIM, N, 0>(buf[0], lo, f);
    cl<DIM, N, true>(T.V, Q[1], f);
    st_line<DIM, N, 0>(buf[1], lo, f);
    if constexpr (DIM == 3) {
      cl<DIM, N, true>(T.V, Q[2], f);
      st_line<DIM, N, 0>(buf[2], lo, f);
    }
  }
  __syncwarp();
  if constexpr (DIM == 3) {
    if (live) {
      double f1[DIM][N], f2[DIM][N], g[DIM][N];
      ld_line<DIM, N, 1>(buf[0], lo, f1);
      ld_line<DIM, N, 1>(buf[1], lo, f2);
      cl2t<DIM, N>(T.V, f1, T.D, f2, g);
      st_line<DIM, N, 1>(buf[0], lo, g);  // g1
      ld_line<DIM, N, 1>(buf[2], lo, f1);
      cl<DIM, N, true>(T.V, f1, g);
      st_line<DIM, N, 1>(buf[1], lo, g);  // g2
    }
    __syncwarp();
  }
  if (live) {
    double g1[DIM][N], g2[DIM][N];
    ld_line<DIM, N, DIM - 1>(buf[0], lo, g1);
    ld_line<DIM, N, DIM - 1>(buf[1], lo, g2);
    cl2t<DIM, N>(T.V, g1, T.D, g2, v);
  }
}

template <int DIM, int N, int VAR, typename ST = double>
__global__ void __launch_bounds__(ChainPlan<DIM, N, VAR, ST>::NT, 1)
    k_apply_chain(const LineArgs a, const TabLine<N> T) {
  using K = LineCfg<DIM, N>;
  using PL = ChainPlan<DIM, N, VAR, ST>;
  using Y = LineMap<DIM, N>;
  constexpr int NF = PL::NF;
  constexpr int NB = PL::NB;
  constexpr int W = PL::W;
  constexpr int RW = PL::RW;
  constexpr long long CH = PL::CH;
  constexpr int NV = DIM * (DIM + 1) / 2;
  constexpr int NM = NV * (NV + 1) / 2;
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(128) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ST* ring = reinterpret_cast<ST*>(smem) + (size_t)warp * RW * CH;
  double* lbuf = reinterpret_cast<double*>(reinterpret_cast<ST*>(smem) + (size_t)W * RW * CH);
  const ST* cache = reinterpret_cast<const ST*>(a.cache);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(lbuf + (size_t)W * NB * Y::BUF) + warp * RW;
  const long long ntiles = a.tile1;
  const long long tstride = (long long)N * CH;
  auto dtile = [&](long long tl) { return (a.reverse && tl < a.tile1) ? a.tile1 - 1 - (tl - a.tile0) : tl; };
  // tile of this warp's k-th work item
  // (round robin over blocks and warps; a global or per-SM dynamic schedule
  // measured slower: DESIGN.md §4.1)
  auto tile_k = [&](long long k) -> long long {
    return dtile(a.tile0 + blockIdx.x + (warp + k * W) * (long long)gridDim.x);
  };
  auto issue = [&](long long j) {
    const long long tile = tile_k(j / N);
    if (tile >= ntiles) return;
    const int s = (int)(j % RW);
    HF_ASSERT(tile * tstride + (j % N + 1) * CH <= a.cache_len);
    mbar_expect_tx(full + s, (unsigned)(CH * sizeof(ST)));
    tma_load_1d(ring + (size_t)s * CH, cache + tile * tstride + (j % N) * CH, (unsigned)(CH * sizeof(ST)), full + s);
  };
  bool synced = a.fill != 1;
  if (a.fill == 2) asm volatile("griddepcontrol.wait;" ::: "memory");
  int slot, m, t;
  bool act;
  line_slot<DIM, N>(lane, slot, m, t, act);
  Gather<DIM, N, VAR> nxt;
  gather_tile<DIM, N, VAR, ST>(a, tile_k(0), ntiles, m, t, act, nxt);  // before the TMA burst (hf_line.cuh)
  if (lane == 0) {
    for (int s = 0; s < RW; ++s) mbar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int j = 0; j < RW; ++j) issue(j);
  }
  __syncwarp();
  LineOff<DIM, N> lo;
  line_offsets<DIM, N>(lane, T, m, t, lo);
  double* const wb = lbuf + (size_t)warp * NB * Y::BUF;
  double* buf[DIM];
#pragma unroll
  for (int b = 0; b < DIM; ++b) buf[b] = wb + b * Y::BUF;

  long long jc = 0;
  for (long long k = 0;; ++k) {
    if (tile_k(k) >= ntiles) break;
    const Gather<DIM, N, VAR> g = nxt;
    gather_tile<DIM, N, VAR, ST>(a, tile_k(k + 1), ntiles, m, t, act, nxt);  // in flight during this tile
    const long long e = g.e;
    const bool live = g.live;
    double u[DIM][N];
#pragma unroll
    for (int c = 0; c < DIM; ++c)
#pragma unroll
      for (int l = 0; l < N; ++l) u[c][l] = ((g.mb >> (c * N + l)) & 1u) ? 0.0 : g.u[c][l];

    double G[DIM][DIM][N];   // [axis][component][point]: gradients, then the queued values in place
    double Gu[DIM][DIM][N];  // scalar: gradients of ubar
    if constexpr (VAR == SCALAR) {
      chain_eval<DIM, N>(T, g.ub, live, lo, buf, Gu);
      __syncwarp();  // the second evaluation reuses the buffers
    }
    chain_eval<DIM, N>(T, u, live, lo, buf, G);

    // ---------------- P: q-point physics along this thread's x-line ----------------
    double mu = 0.0, lam = 0.0;
    if (VAR == SCALAR && live) {
      mu = __ldg(a.mu + e);
      lam = __ldg(a.lam + e);
    }
    auto point = [&](const int iq, const ST* st) {
      if (!live) return;
      double f[NF];
#pragma unroll
      for (int q = 0; q < NF; ++q) f[q] = (double)st[q * K::LANES];
      double gu[DIM][DIM];
#pragma unroll
      for (int cc = 0; cc < DIM; ++cc)
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) gu[cc][ax] = G[ax][cc][iq];
      double Gq[DIM][DIM];
      if (VAR == TENSOR4) {
        double sinv[DIM][DIM], tau[DIM][DIM];
#pragma unroll
        for (int i = 0; i < DIM; ++i)
#pragma unroll
          for (int j = 0; j < DIM; ++j) {
            tau[i][j] = f[hf_slot<DIM>(i, j)];
            sinv[i][j] = f[NV + NM + i * DIM + j];
          }
        qp_action<DIM, true>(gu, sinv, tau, 0.0, 0.0, f + NV, 1.0, Gq);  // JxW folded into tau, M
      } else if (VAR == TENSOR2) {
        double sinv[DIM][DIM], tau[DIM][DIM];
#pragma unroll
        for (int i = 0; i < DIM; ++i)
#pragma unroll
          for (int j = 0; j < DIM; ++j) {
            tau[i][j] = f[2 + hf_slot<DIM>(i, j)];
            sinv[i][j] = f[2 + NV + i * DIM + j];
          }
        qp_action<DIM, false>(gu, sinv, tau, f[0], f[1], nullptr, 1.0, Gq);  // JxW folded into c1', c2', tau
      } else {
        // rebuild F, b, tau = mu b - c1 I and s_inv from ubar (operators.py:349-363)
        double ji[DIM][DIM];
#pragma unroll
        for (int r = 0; r < DIM; ++r)
#pragma unroll
          for (int q = 0; q < DIM; ++q) ji[r][q] = f[1 + r * DIM + q];
        double F[DIM * DIM];
#pragma unroll
        for (int i = 0; i < DIM; ++i)
#pragma unroll
          for (int Aa = 0; Aa < DIM; ++Aa) {
            double sm = (i == Aa) ? 1.0 : 0.0;
#pragma unroll
            for (int q = 0; q < DIM; ++q) sm = fma(Gu[q][i][iq], ji[q][Aa], sm);
            F[i * DIM + Aa] = sm;
          }
        const double c1 = f[0];
        double tau[DIM][DIM], sinv[DIM][DIM], Fi[DIM * DIM];
#pragma unroll
        for (int i = 0; i < DIM; ++i)
#pragma unroll
          for (int j = 0; j < DIM; ++j) {
            double bb = 0.0;
#pragma unroll
            for (int Aa = 0; Aa < DIM; ++Aa) bb = fma(F[i * DIM + Aa], F[j * DIM + Aa], bb);
            tau[i][j] = mu * bb - (i == j ? c1 : 0.0);
          }
        hf_inv<DIM>(F, hf_det<DIM>(F), Fi);
#pragma unroll
        for (int q = 0; q < DIM; ++q)
#pragma unroll
          for (int j = 0; j < DIM; ++j) {
            double sm = 0.0;
#pragma unroll
            for (int Aa = 0; Aa < DIM; ++Aa) sm = fma(ji[q][Aa], Fi[Aa * DIM + j], sm);
            sinv[q][j] = sm;
          }
        qp_action<DIM, false>(gu, sinv, tau, 2.0 * c1, 2.0 * lam, nullptr, f[NF - 1], Gq);
      }
#pragma unroll
      for (int cc = 0; cc < DIM; ++cc)
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) G[ax][cc][iq] = Gq[cc][ax];
    };
    if constexpr (RW >= N) {
#pragma unroll
      for (int iq = 0; iq < N; ++iq) mbar_wait(full + (int)((jc + iq) % RW), (unsigned)(((jc + iq) / RW) & 1));
#pragma unroll
      for (int iq = 0; iq < N; ++iq) point(iq, ring + (size_t)((jc + iq) % RW) * CH + slot);
      __syncwarp();
      if (lane < N) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(jc + lane + RW);
      }
      jc += N;
    } else {
#pragma unroll
      for (int iq = 0; iq < N; ++iq, ++jc) {
        const int s = (int)(jc % RW);
        mbar_wait(full + s, (unsigned)((jc / RW) & 1));
        point(iq, ring + (size_t)s * CH + slot);
        __syncwarp();
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(jc + RW);
        }
      }
    }

    double v[DIM][N];
    chain_integrate<DIM, N>(T, G, live, lo, buf, v);
    if (!synced) {  // the fill kernel (PDL primary) has completed and its writes are visible
      asm volatile("griddepcontrol.wait;" ::: "memory");
      synced = true;
    }
    if (live) {
      unsigned nb, s_last;
      last_axis_line<DIM, N>(a.lat, g.node0, t, nb, s_last);
#pragma unroll
      for (int l = 0; l < N; ++l) {
        const unsigned d0 = (nb + l * s_last) * DIM;
        HF_ASSERT((long long)d0 + DIM <= a.lat.n_nodes * DIM);
#pragma unroll
        for (int cc = 0; cc < DIM; ++cc)
          atomicAdd(reinterpret_cast<ST*>(a.y) + d0 + cc, ((g.mb >> (cc * N + l)) & 1u) ? (ST)0 : (ST)v[cc][l]);
      }
    }
    __syncwarp();  // line buffers are reused by the next tile
  }
}

}  // namespace hf
