// Plane-parallel apply kernel for 3D Q2 (N = 3), tensor2 cache (sm_100a, fp64).
// DESIGN.md §4.1 "plane owners" has the measurements.
//
// The line kernel (hf_line.cuh) hands every 1D line between axis phases
// through shared memory: ~200 8-byte accesses per thread and tile, ~140
// wavefronts per cell, and the tensor2 variant runs at 84 % of the L1/shared
// pipe with half of its HBM bandwidth unused.  Here one thread owns a whole
// z-PLANE of a cell (3 x 3 points x 3 components = 27 values in registers):
//
//  * the x and y contractions (interpolation, collocation derivatives and
//    their transposes) never leave the thread's registers;
//  * only the z contractions cross threads, among the 3 plane owners of a
//    cell, as two exchanges through a per-warp shared-memory slice:
//      E  each owner publishes its plane of (x, y)-interpolated nodal-in-z
//         values and reads the two others: values Q = V_z w and the z
//         derivative G_z = D_z w at its Gauss plane (the reference's own form of
//         the z derivative, fespace.py:230-239: derivative table on the
//         differentiated axis, value tables on the others);
//      I  each owner publishes its contributions V_z[k][k'] S + D_z[k][k'] Z to
//         the two other nodal planes k and sums what it receives;
//    27 + 54 and 54 + 54 accesses per thread and cell third: ~38 wavefronts per
//    cell instead of ~140;
//  * a warp tile is 10 cells (30 lanes).  The cache is stored
//    [tile][p][field][lane] with p the point within the plane (x fastest) and
//    lane = cell * 3 + Gauss plane, so the chunk of one (tile, p) is contiguous
//    and arrives through the warp's private TMA ring as in the line kernel;
//  * x and y derivatives at a point are formed from the plane's values Q when
//    the point is processed (3 FMAs each per component: the same count as the
//    full contraction), and the queued test-function gradients are folded
//    into the plane accumulator S the same way, so neither is stored.
//
// Reference correspondence: gather fespace.py:291-293 + operators.py:333-334;
// evaluate fespace.py:224-239; q-point physics operators.py:364-392; integrate
// fespace.py:258-288; scatter fespace.py:296-324.
#pragma once
#include "hf_line.cuh"

namespace hf {

struct PlaneCfg {
  static constexpr int N = 3;
  static constexpr int CPW = 10;        // cells per warp tile
  static constexpr int LANES = 30;      // active lanes
  static constexpr int NPP = 9;         // points per plane
};

// 1D tables of the plane kernel: V and Dc indexed with compile-time constants
// (constant-bank operands); the z tables are read per lane (its plane index).
struct TabPlane {
  double V[3][3];   // V[l][o]  = N_l(xi_o)
  double D[3][3];   // D[l][o]  = N_l'(xi_o)
  double Dc[3][3];  // collocation derivative at Gauss point o of Gauss-basis l
};

template <int VAR, typename ST = double>
struct PlanePlan {
  static constexpr int NF = CacheFields<3, VAR>::NF;
  // ST elements per (tile, p) chunk, 16-byte padded
  static constexpr long long CH = (((long long)NF * PlaneCfg::LANES * sizeof(ST) + 15) & ~15ll) / sizeof(ST);
  static constexpr int RW = 3;                    // ring stages per warp (one row of the plane)
  static constexpr int XB = 27 * 32;              // doubles of the exchange slice per warp
  static constexpr int GS = 27 * 32;              // ST elements of the gather staging slice per warp
  static constexpr size_t perw() {
    return sizeof(ST) * ((size_t)RW * CH + GS) + sizeof(double) * XB + 16 * RW;
  }
  static constexpr size_t BUDGET = 226 * 1024;
  static constexpr int W0 = (int)(BUDGET / perw());
  static constexpr int W = W0 > 8 ? 8 : W0;       // 255 registers per thread: 8 warps per SM
  static constexpr int NT = 32 * W;
  static constexpr size_t SMEM = (size_t)W * perw();
};

// 4- or 8-byte asynchronous global -> shared copy (LDGSTS: no register staging)
template <int BYTES>
HF_DEV void cp_async(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(BYTES) : "memory");
}
HF_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

#ifndef HF_PLANE_GROUP
#define HF_PLANE_GROUP 1  // points processed per ring wait (1, or 3 = a whole row)
#endif

template <int VAR, typename ST = double>
__global__ void __launch_bounds__(PlanePlan<VAR, ST>::NT, 1)
    k_apply_plane(const LineArgs a, const TabPlane T, const uint32_t* __restrict__ pmask) {
  using PL = PlanePlan<VAR, ST>;
  constexpr int NF = PL::NF;
  constexpr int W = PL::W;
  constexpr int RW = PL::RW;
  constexpr long long CH = PL::CH;
  constexpr int NV = 6;
  constexpr int CPW = PlaneCfg::CPW;
  constexpr int LANES = PlaneCfg::LANES;
  constexpr int GRP = HF_PLANE_GROUP;
  static_assert(VAR == TENSOR2, "plane kernel: tensor2 only");
  static_assert(RW == 3 && (GRP == 1 || GRP == 3), "one ring turn per row of the plane");
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(128) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // shared memory: W rings | W gather slices (ST) | W exchange slices (double) | mbarriers
  ST* ring = reinterpret_cast<ST*>(smem) + (size_t)warp * RW * CH;
  ST* gs = reinterpret_cast<ST*>(smem) + (size_t)W * RW * CH + (size_t)warp * PL::GS;
  double* xb0 = reinterpret_cast<double*>(reinterpret_cast<ST*>(smem) + (size_t)W * (RW * CH + PL::GS));
  double* xb = xb0 + (size_t)warp * PL::XB;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(xb0 + (size_t)W * PL::XB) + warp * RW;
  const ST* cache = reinterpret_cast<const ST*>(a.cache);
  const ST* xs = reinterpret_cast<const ST*>(a.x);
  const long long ntiles = a.tile1;
  constexpr long long tstride = 9 * CH;
  auto dtile = [&](long long tl) { return (a.reverse && tl < a.tile1) ? a.tile1 - 1 - (tl - a.tile0) : tl; };
  auto tile_k = [&](int k) -> long long {
    return dtile(a.tile0 + blockIdx.x + (warp + k * W) * (long long)gridDim.x);
  };
  // chunk p of a tile's cache block into stage p % RW (cb == nullptr: no such tile)
  auto issue = [&](const ST* cb, int p) {
    if (!cb) return;
    const int s = p % RW;
    mbar_expect_tx(full + s, (unsigned)(CH * sizeof(ST)));
    tma_load_1d(ring + (size_t)s * CH, cb + p * CH, (unsigned)(CH * sizeof(ST)), full + s);
  };
  auto cblock = [&](long long tile) -> const ST* {
    HF_ASSERT(tile >= ntiles || (tile + 1) * tstride <= a.cache_len);
    return tile < ntiles ? cache + tile * tstride : nullptr;
  };
  bool synced = a.fill != 1;
  if (a.fill == 2) asm volatile("griddepcontrol.wait;" ::: "memory");

  const bool act = lane < LANES;
  const int m = act ? lane / 3 : 0;        // cell within the tile
  const int kp = act ? lane - 3 * m : 0;   // this thread's plane (nodal plane k and Gauss plane k')
  // lanes of the cell's other planes, in the order (kp + 1) % 3, (kp + 2) % 3
  const int l1 = 3 * m + (kp + 1) % 3, l2 = 3 * m + (kp + 2) % 3;
  // z tables of this plane, re-read from the constant bank where they are
  // used (12 registers less across the point loop): zV[r] = V[(kp + r) % 3][kp]
  // for the source plane (kp + r) % 3 -> Gauss plane kp; the transposed pass
  // uses the same entries
  auto ztab = [&](double (&zV)[3], double (&zD)[3]) {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      zV[r] = T.V[(kp + r) % 3][kp];
      zD[r] = T.D[(kp + r) % 3][kp];
    }
  };
  const unsigned sy = (unsigned)a.lat.nodes[0];
  const unsigned sz = sy * (unsigned)a.lat.nodes[1];
  // gather of a tile, one tile ahead of use: the nodal plane kp of the lane's
  // cell copied asynchronously into the warp's staging slice ([c * 9 + q][lane]),
  // and the plane's constraint bits
  auto gather = [&](long long tile, unsigned& mbits) {
    const long long e = tile * CPW + m;
    mbits = 0;
    if (!(act && tile < ntiles && e < a.lat.n_el)) return;
    const unsigned nb = cell_node0<3>(a.lat, (unsigned)e, a.degree) + (unsigned)kp * sz;
    mbits = __ldg(pmask + (unsigned)e * 3u + (unsigned)kp);
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int aa = 0; aa < 3; ++aa) {
        const unsigned d0 = (nb + aa + b * sy) * 3u;
        HF_ASSERT((long long)d0 + 3 <= a.lat.n_nodes * 3);
#pragma unroll
        for (int c = 0; c < 3; ++c) cp_async<sizeof(ST)>(gs + (c * 9 + aa + 3 * b) * 32 + lane, xs + d0 + c);
      }
  };

  long long t_cur = tile_k(0);
  unsigned mb_nxt;
  gather(t_cur, mb_nxt);
  const ST* cb_cur = cblock(t_cur);
  if (lane == 0) {
    for (int s = 0; s < RW; ++s) mbar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int j = 0; j < RW; ++j) issue(cb_cur, j);
  }
  __syncwarp();

  for (int k = 0;; ++k) {
    if (t_cur >= ntiles) break;
    const long long t_nxt = tile_k(k + 1);
    const ST* cb_nxt = cblock(t_nxt);
    const long long e = t_cur * CPW + m;
    const bool live = act && e < a.lat.n_el;
    const unsigned mb = mb_nxt;
    // ---------------- the gathered nodal plane, constrained DoFs zeroed ----------------
    double u[3][9];  // [component][a + 3 b]
    cp_async_wait_all();
    if (live) {
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int q = 0; q < 9; ++q) u[c][q] = ((mb >> (c * 9 + q)) & 1u) ? 0.0 : (double)gs[(c * 9 + q) * 32 + lane];
      // in-plane interpolation: x, then y
#pragma unroll
      for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          double o[3];
          c1d<3, false>(T.V, &u[c][3 * b], o);
#pragma unroll
          for (int i = 0; i < 3; ++i) u[c][3 * b + i] = o[i];
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double in[3] = {u[c][i], u[c][i + 3], u[c][i + 6]};
          double o[3];
          c1d<3, false>(T.V, in, o);
#pragma unroll
          for (int j = 0; j < 3; ++j) u[c][i + 3 * j] = o[j];
        }
      }
      // ---------------- E: publish the plane, read the cell's two others ----------------
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int q = 0; q < 9; ++q) xb[(c * 9 + q) * 32 + lane] = u[c][q];
    }
    __syncwarp();
    gather(t_nxt, mb_nxt);  // the staged values are in registers (they fed the interpolation)
    double Q[3][9], Z[3][9];  // values at the Gauss plane; z derivative, later the queued z part
    if (live) {
      double cV[3], cD[3];
      ztab(cV, cD);
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int q = 0; q < 9; ++q) {
          const double w1 = xb[(c * 9 + q) * 32 + l1], w2 = xb[(c * 9 + q) * 32 + l2];
          Q[c][q] = fma(cV[2], w2, fma(cV[1], w1, cV[0] * u[c][q]));
          Z[c][q] = fma(cD[2], w2, fma(cD[1], w1, cD[0] * u[c][q]));
        }
    }
    __syncwarp();  // the slice is written again in I
    // ---------------- P: the 9 points of the plane ----------------
    double S[3][9];  // accumulates Dc_x^T X + Dc_y^T Y
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int q = 0; q < 9; ++q) S[c][q] = 0.0;
    auto point = [&](const int p) {
      const int i = p % 3, j = p / 3;
      const ST* st = ring + (size_t)(p % RW) * CH + lane;
      double f[NF];
#pragma unroll
      for (int q = 0; q < NF; ++q) f[q] = (double)st[q * LANES];
      double gu[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double gx = 0.0, gy = 0.0;
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          gx = fma(T.Dc[l][i], Q[c][l + 3 * j], gx);
          gy = fma(T.Dc[l][j], Q[c][i + 3 * l], gy);
        }
        gu[c][0] = gx;
        gu[c][1] = gy;
        gu[c][2] = Z[c][p];
      }
      double sinv[3][3], tau[3][3], G[3][3];
#pragma unroll
      for (int ii = 0; ii < 3; ++ii)
#pragma unroll
        for (int jj = 0; jj < 3; ++jj) {
          tau[ii][jj] = f[2 + hf_slot<3>(ii, jj)];
          sinv[ii][jj] = f[2 + NV + ii * 3 + jj];
        }
      qp_action<3, false>(gu, sinv, tau, f[0], f[1], nullptr, 1.0, G);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          S[c][l + 3 * j] = fma(T.Dc[l][i], G[c][0], S[c][l + 3 * j]);
          S[c][i + 3 * l] = fma(T.Dc[l][j], G[c][1], S[c][i + 3 * l]);
        }
        Z[c][p] = G[c][2];
      }
    };
    constexpr int RPT = 9 / RW;  // ring turns per tile
#pragma unroll
    for (int p0 = 0; p0 < 9; p0 += GRP) {
#pragma unroll
      for (int g = 0; g < GRP; ++g)
        mbar_wait(full + (p0 + g) % RW, (unsigned)((k * RPT + (p0 + g) / RW) & 1));
      if (live) {
#pragma unroll
        for (int g = 0; g < GRP; ++g) point(p0 + g);
      }
      __syncwarp();
      if (lane < GRP) {  // stages consumed by every lane: refill them with the chunks RW ahead
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const int pn = p0 + lane + RW;
        if (pn < 9) issue(cb_cur, pn); else issue(cb_nxt, pn - 9);
      }
    }
    // ---------------- I: contributions to the cell's two other nodal planes ----------------
    // two rounds through the slice: round r carries what plane (kp - r) % 3 adds to plane kp
    double cV[3], cD[3];
    ztab(cV, cD);
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int q = 0; q < 9; ++q) u[c][q] = fma(cD[0], Z[c][q], cV[0] * S[c][q]);
#pragma unroll
    for (int r = 1; r <= 2; ++r) {
      if (live) {
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int q = 0; q < 9; ++q) xb[(c * 9 + q) * 32 + lane] = fma(cD[r], Z[c][q], cV[r] * S[c][q]);  // to plane (kp + r) % 3
      }
      __syncwarp();
      if (live) {
        const int src = r == 1 ? l2 : l1;  // the owner whose "+r" plane is kp
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int q = 0; q < 9; ++q) u[c][q] += xb[(c * 9 + q) * 32 + src];
      }
      __syncwarp();
    }
    if (live) {
      // transposed in-plane interpolation: y, then x
#pragma unroll
      for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double in[3] = {u[c][i], u[c][i + 3], u[c][i + 6]};
          double o[3];
          c1d<3, true>(T.V, in, o);
#pragma unroll
          for (int b = 0; b < 3; ++b) u[c][i + 3 * b] = o[b];
        }
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          double o[3];
          c1d<3, true>(T.V, &u[c][3 * b], o);
#pragma unroll
          for (int aa = 0; aa < 3; ++aa) u[c][3 * b + aa] = o[aa];
        }
      }
    }
    if (!synced) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      synced = true;
    }
    if (live) {
      const unsigned nb = cell_node0<3>(a.lat, (unsigned)e, a.degree) + (unsigned)kp * sz;
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int aa = 0; aa < 3; ++aa) {
          const unsigned d0 = (nb + aa + b * sy) * 3u;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            atomicAdd(reinterpret_cast<ST*>(a.y) + d0 + c,
                      ((mb >> (c * 9 + aa + 3 * b)) & 1u) ? (ST)0 : (ST)u[c][aa + 3 * b]);
        }
    }
    t_cur = t_nxt;
    cb_cur = cb_nxt;
  }
}

}  // namespace hf
