// Line-parallel, TMA-fed apply kernel of the matrix-free Neo-Hookean tangent
// (sm_100a, fp64).  DESIGN.md §4.1 has the measurements behind each choice.
//
//  * One thread owns one 1D LINE of a cell (N points along one axis). Every 1D
//    contraction of the sum factorisation runs in registers with a warp-uniform
//    table index. The tables are kernel parameters (constant-bank operands of
//    DFMA), so no shared-memory table traffic.
//  * A consumer warp holds CPW = 32 / N^(DIM-1) whole cells (a "warp tile").
//    The only synchronisation between axis phases is __syncwarp. Lines are
//    handed from one axis to the next through a per-warp shared-memory slice
//    whose layout (cells interleaved, padded strides) is chosen per (DIM, N) to
//    minimise bank conflicts of the 64-bit accesses.
//  * The quadrature cache is stored per tile as [tile][iq][field][lane], so the
//    data of one (tile, iq) is a contiguous chunk. Every warp streams its own
//    chunks through a private ring of RW shared-memory stages with 1D TMA bulk
//    copies (cp.async.bulk ... mbarrier::complete_tx): it issues chunk j+RW as
//    soon as chunk j is consumed, and waits on a stage's mbarrier only right
//    before the point phase. Private rings keep every wait at most one phase
//    ahead of its barrier (a ring shared by several consumers lets a fast warp
//    alias the parity of a slow one's stage).
//    The HBM stream therefore never occupies registers: the bytes in flight are
//    bounded by the rings, not by occupancy. The first kernel generation was
//    latency bound at 16 warps/SM with the cache loaded into registers.
//
// Phases of one warp tile (3D; 2D drops axis 2):
//   E1  z-lines : gather x (constrained DoFs zeroed), interpolate along z      -> A
//   E2  y-lines : interpolate along y                                         A -> B
//   E3  x-lines : interpolate along x (values Q at Gauss points), collocation
//                 derivative along x kept in registers (Gx)                    B -> A(Q)
//   E4  y-/z-lines : collocation derivatives along y and z                   A -> B(G1), C(G2)
//   P   x-lines : q-point physics of the caching variant (operators.py:341-392)
//                 from the TMA stage; queued G[c][a]*JxW written to A/B/C
//   I1  a-lines : transposed collocation derivative along axis a (in place)
//   I2  x-lines : sum of the three, transposed interpolation along x           A
//   I3  y-lines : transposed interpolation along y                             A
//   I4  z-lines : transposed interpolation along z + atomic scatter-add,
//                 constrained rows dropped (fespace.py:307-324)
//
// Reference correspondence: gather fespace.py:291-293 + operators.py:333-334;
// evaluate fespace.py:224-239; q-point physics operators.py:341-392; integrate
// fespace.py:258-288; scatter fespace.py:296-324.
#pragma once
#include "hf_cell.cuh"
#include "hf_dispatch.h"
#include "hf_lanemap.h"

namespace hf {

// Per-warp timeline of the apply kernel (instrumented build only:
// HF_TIMELINE=1 python -m paper_1904_13131_b200.build -> libhf_tl.so;
// hf_timeline_fetch; tools/timeline.py).  Slot 0: kernel entry; per tile k:
// 1 + 4k tile start, 2 + 4k gradients done, 3 + 4k point phase done, 4 + 4k
// tile end; the last slot: exit.  %globaltimer, ns.
#ifdef HF_TIMELINE
static __device__ unsigned long long hf_tl_buf[HF_TL_WARPS * HF_TL_SLOTS];  // one per translation unit
HF_DEV unsigned long long hf_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define HF_TL(slot)                                                                                   \
  do {                                                                                                \
    const int _s = (slot);                                                                            \
    const unsigned _w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);                          \
    if ((threadIdx.x & 31) == 0 && _w < HF_TL_WARPS && _s < HF_TL_SLOTS) hf_tl_buf[_w * HF_TL_SLOTS + _s] = hf_gtime(); \
  } while (0)
#else
#define HF_TL(slot) \
  do {              \
  } while (0)
#endif

// 1D tables as a kernel parameter: indexed with compile-time constants only,
// so they are constant-bank operands.
template <int N>
struct TabLine {
  double V[N][N];   // V[l][o]  = N_l(xi_o)
  double Dc[N][N];  // Dc[l][o] = collocation derivative at Gauss point o of Gauss-basis l
  // per-lane packed site offsets of a generated conflict-free layout
  // (LaneMapT::TABLE); read from the constant bank with a per-lane index
  unsigned long long loff[32][2];
};

struct LineArgs {
  HfLattice lat;
  int degree;
  const double* x;
  double* y;
  const double* cache;  // tiled [tile][iq][field][lane]
  const double* ubar;   // scalar strategy
  const double* mu;     // scalar strategy
  const double* lam;
  const uint8_t* mask;
  const uint32_t* lmask;  // constraint bits per (cell, last-axis line)
  const int* skip;
  // 0: plain launch (y already initialised by an earlier kernel)
  // 1: PDL secondary of the y = mask ? x : 0 fill (operators.py:333-338): wait before the first scatter
  // 2: PDL secondary of a kernel that wrote x and y (hf_cheb_step_fill): wait before the first gather
  int fill;
  long long tile0, tile1;  // tile range of this launch (interior/boundary split of a slab)
  int reverse;             // walk the tile range backwards (alternating sweeps reuse L2, hf_tangent_set_alternate)
  long long cache_len;     // cache elements (bounds checks of the debug build)
};

// Per-warp line-buffer layout: element (cell m, component c, point i,j,k) at
// ((c*NP + i + j*SJ + k*SK) * CPWP + m).  (CPWP, PJ, PK) from a bank-conflict
// search over the 64-bit access patterns of every axis phase.
template <int DIM, int N>
struct LineLay {
  static constexpr int CPWP = DIM == 3 ? (N == 2 ? 12 : (N == 5 ? 1 : 3))
                                       : (N == 2 ? 18 : N == 3 ? 11 : N == 4 ? 12 : N == 5 ? 9 : N == 6 ? 5
                                          : N == 7 ? 6 : N == 8 ? 6 : 9);
  static constexpr int PJ = DIM == 3 ? (N == 4 ? 1 : 0) : (N == 2 || N == 9 ? 2 : (N == 3 || N == 4 || N == 8) ? 1 : 0);
  static constexpr int PK = (DIM == 3 && N == 2) ? 2 : 0;
  static constexpr int SJ = N + PJ;
  static constexpr int SK = DIM == 3 ? N * SJ + PK : 0;
  static constexpr int NP = DIM == 3 ? N * SK : N * SJ;  // points incl. padding
  static constexpr int BUF = DIM * NP * CPWP;           // doubles per buffer per warp
};

template <int DIM, int N, int AX>
HF_DEV constexpr int lstride() {
  using Y = LineLay<DIM, N>;
  return AX == 0 ? 1 : (AX == 1 ? Y::SJ : Y::SK);
}
// padded offset of point 0 of line t along axis AX
template <int DIM, int N, int AX>
HF_DEV int lbase(int t) {
  using Y = LineLay<DIM, N>;
  if (DIM == 2) return AX == 0 ? t * Y::SJ : t;
  if (AX == 0) return (t % N) * Y::SJ + (t / N) * Y::SK;
  if (AX == 1) return (t % N) + (t / N) * Y::SK;
  return (t % N) + (t / N) * Y::SJ;
}

// out[o] = sum_l M[l][o] in[l]   (forward)      out[l] = sum_o M[l][o] in[o]   (transposed)
template <int N, bool TR>
HF_DEV void c1d(const double (&M)[N][N], const double* in, double* out) {
#pragma unroll
  for (int o = 0; o < N; ++o) {
    double s = 0.0;
#pragma unroll
    for (int l = 0; l < N; ++l) s = fma(TR ? M[o][l] : M[l][o], in[l], s);
    out[o] = s;
  }
}

// Where a thread's line sites live in its warp's line buffers: off[AX][l] is
// the offset (component 0) of the site at position l along axis AX of the
// line the thread owns in an AX phase.  3D Q2 uses the generated
// bank-conflict-free map (hf_lanemap.h: lane -> (cell, line) slot, sites
// coloured over the 16 banks of each half-warp); other (DIM, N) the padded
// interleaved layout of LineLay.
template <int DIM, int N>
struct LineMap {
  static constexpr bool CUSTOM = LaneMapT<DIM, N>::ENABLED;
  static constexpr int CS = CUSTOM ? LaneMapT<DIM, N>::COMP : LineLay<DIM, N>::NP * LineLay<DIM, N>::CPWP;  // component stride
  static constexpr int BUF = DIM * CS;                                                      // doubles per buffer
};

template <int DIM, int N>
struct LineOff {
  int off[DIM][N];
};

// lane -> (slot = cell * L + line, cell m, line t, active): immediates only,
// no memory access (the kernel issues its first gather right after)
template <int DIM, int N>
HF_DEV void line_slot(int lane, int& slot, int& m, int& t, bool& act) {
  using K = LineCfg<DIM, N>;
  if constexpr (LineMap<DIM, N>::CUSTOM) {
    using Z = LaneMapT<DIM, N>;
    const unsigned long long w = lane < 12 ? Z::B0 : (lane < 24 ? Z::B1 : Z::B2);
    const int sl = (int)((w >> (5 * (lane % 12))) & 31ull);
    act = sl != 31;
    slot = act ? sl : 0;
  } else {
    act = lane < K::LANES;
    slot = act ? lane : 0;
  }
  m = slot / K::L;
  t = slot - m * K::L;
}

// the lane's line-buffer site offsets (the generated layout reads a per-lane
// table from the kernel parameters: a constant-cache miss at kernel start)
template <int DIM, int N>
HF_DEV void line_offsets(int lane, const TabLine<N>& T, int m, int t, LineOff<DIM, N>& o) {
  using Y = LineLay<DIM, N>;
  if constexpr (LineMap<DIM, N>::CUSTOM) {
    using Z = LaneMapT<DIM, N>;
    constexpr int per = 64 / Z::OFF_BITS;
    unsigned long long ow[Z::OFF_WORDS];
#pragma unroll
    for (int i = 0; i < Z::OFF_WORDS; ++i) ow[i] = T.loff[lane][i];
#pragma unroll
    for (int k = 0; k < DIM * N; ++k)
      o.off[k / N][k % N] = (int)((ow[k / per] >> (Z::OFF_BITS * (k % per))) & ((1ull << Z::OFF_BITS) - 1));
  } else {
#pragma unroll
    for (int l = 0; l < N; ++l) {
      o.off[0][l] = (lbase<DIM, N, 0>(t) + l * lstride<DIM, N, 0>()) * Y::CPWP + m;
      o.off[1][l] = (lbase<DIM, N, 1>(t) + l * lstride<DIM, N, 1>()) * Y::CPWP + m;
      if (DIM == 3) o.off[DIM - 1][l] = (lbase<DIM, N, DIM - 1>(t) + l * lstride<DIM, N, DIM - 1>()) * Y::CPWP + m;
    }
  }
}

template <int DIM, int N, int AX>
HF_DEV void ld_line(const double* buf, const LineOff<DIM, N>& o, double (&v)[DIM][N]) {
  constexpr int CS = LineMap<DIM, N>::CS;
#pragma unroll
  for (int c = 0; c < DIM; ++c)
#pragma unroll
    for (int l = 0; l < N; ++l) v[c][l] = buf[c * CS + o.off[AX][l]];
}
template <int DIM, int N, int AX>
HF_DEV void st_line(double* buf, const LineOff<DIM, N>& o, const double (&v)[DIM][N]) {
  constexpr int CS = LineMap<DIM, N>::CS;
#pragma unroll
  for (int c = 0; c < DIM; ++c)
#pragma unroll
    for (int l = 0; l < N; ++l) buf[c * CS + o.off[AX][l]] = v[c][l];
}
template <int DIM, int N, bool TR>
HF_DEV void c_line(const double (&M)[N][N], double (&v)[DIM][N]) {
#pragma unroll
  for (int c = 0; c < DIM; ++c) {
    double o[N];
    c1d<N, TR>(M, v[c], o);
#pragma unroll
    for (int l = 0; l < N; ++l) v[c][l] = o[l];
  }
}

// First lattice node of cell e, and the first node and stride (in nodes) of
// line t along the last axis.  32-bit index arithmetic: hf_space_create
// guarantees n_dofs < 2^31; the cell coordinates come from multiply-shift
// divisions by the invariant cell counts (HfLattice::dm/ds).
template <int DIM>
HF_DEV unsigned cell_node0(const HfLattice& lat, unsigned e, int degree) {
  const unsigned r = hf_fastdiv(e, lat.dm[0], lat.ds[0]);
  const unsigned ex = e - r * (unsigned)lat.cells[0];
  unsigned ey = r, ez = 0;
  if (DIM == 3) {
    ez = hf_fastdiv(r, lat.dm[1], lat.ds[1]);
    ey = r - ez * (unsigned)lat.cells[1];
  }
  return (ex + (unsigned)lat.nodes[0] * (ey + (unsigned)lat.nodes[1] * ez)) * (unsigned)degree;
}

template <int DIM, int N>
HF_DEV void last_axis_line(const HfLattice& lat, unsigned node0, int t, unsigned& nb, unsigned& s_last) {
  const unsigned i = (unsigned)(t % N);
  const unsigned j = DIM == 3 ? (unsigned)(t / N) : 0u;
  const unsigned sy = (unsigned)lat.nodes[0];
  s_last = DIM == 3 ? sy * (unsigned)lat.nodes[1] : sy;
  nb = node0 + i + (DIM == 3 ? j * sy : 0u);
}

// The scatter's reductions are evict-last in L2: the kernel after an apply
// (Chebyshev or CG update, dot) reads y, and the evict-first cache stream
// leaves room for it.  Config-4 CG iteration with tensor2 8.04 -> 7.95 ms,
// k_cheb 1.36 -> 1.27 ms per iteration (profiles/r02/ab_l2_evict_first.txt);
// the same hint on the x gathers moved time from k_cheb into the apply.
HF_DEV unsigned long long l2_keep_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
HF_DEV void red_keep(double* p, double v, unsigned long long pol) {
#ifndef HF_NO_L2HINT
  asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
#else
  atomicAdd(p, v);
#endif
}
HF_DEV void red_keep(float* p, float v, unsigned long long pol) {
#ifndef HF_NO_L2HINT
  asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
#else
  atomicAdd(p, v);
#endif
}

// The last-axis line of one tile gathered ahead of use (software pipelining
// one tile deep): nodal values of x (and ubar for the scalar strategy) and the
// line's constraint bits (bit c*N + l).
template <int DIM, int N, int VAR>
struct Gather {  // values held in fp64 whatever the storage type
  double u[DIM][N];
  double ub[DIM][N];  // scalar strategy only
  unsigned mb;
  unsigned e, node0;
  bool live;
};

template <int DIM, int N, int VAR, typename ST = double>
HF_DEV void gather_tile(const LineArgs& a, long long tile, long long ntiles, int m, int t, bool act,
                        Gather<DIM, N, VAR>& g) {
  using K = LineCfg<DIM, N>;
  const ST* xs = reinterpret_cast<const ST*>(a.x);  // fp64, or fp32 vectors of a mixed-precision level
  const long long e = tile * K::CPW + m;
  g.live = act && tile < ntiles && e < a.lat.n_el;
  g.e = (unsigned)e;
  g.mb = 0;
  g.node0 = g.live ? cell_node0<DIM>(a.lat, g.e, a.degree) : 0u;
  if (!g.live) return;
  unsigned nb, s_last;
  last_axis_line<DIM, N>(a.lat, g.node0, t, nb, s_last);
#pragma unroll
  for (int l = 0; l < N; ++l) {
    const unsigned d0 = (nb + l * s_last) * DIM;
    HF_ASSERT((long long)d0 + DIM <= a.lat.n_nodes * DIM);
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      g.u[c][l] = (double)__ldg(xs + d0 + c);
      if (VAR == SCALAR) g.ub[c][l] = __ldg(a.ubar + d0 + c);
    }
  }
  g.mb = __ldg(a.lmask + (g.e * (unsigned)K::L + (unsigned)t));
}

// Unit-cell gradients of the nodal line values u0 (last axis, already masked)
// of the warp's cells: Gx in registers (x-line owners), the axis-1 derivative
// in buffer g1, the axis-2 derivative (3D) in g2.  a and b are scratch; g1 may
// be a (the y-derivative then overwrites the values in place, line by line,
// after the z-lines have read them) and g2 may be b.
template <int DIM, int N, bool KEEPQ = false>
HF_DEV void eval_line(const TabLine<N>& T, const double (&u0)[DIM][N], bool live, const LineOff<DIM, N>& t,
                      double* a, double* b, double* g1, double* g2, double (&Gx)[DIM][N]) {
  double u[DIM][N];
  if (live) {
#pragma unroll
    for (int c = 0; c < DIM; ++c)
#pragma unroll
      for (int l = 0; l < N; ++l) u[c][l] = u0[c][l];
    c_line<DIM, N, false>(T.V, u);
    st_line<DIM, N, DIM - 1>(DIM == 3 ? a : b, t, u);
  }
  __syncwarp();
  if (DIM == 3) {
    if (live) {
      ld_line<DIM, N, 1>(a, t, u);
      c_line<DIM, N, false>(T.V, u);
      st_line<DIM, N, 1>(b, t, u);
    }
    __syncwarp();
  }
  if (live) {
    ld_line<DIM, N, 0>(b, t, u);
    c_line<DIM, N, false>(T.V, u);
    st_line<DIM, N, 0>(a, t, u);  // Q at Gauss points
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      if constexpr (KEEPQ) {  // the point phase differentiates along x itself
#pragma unroll
        for (int l = 0; l < N; ++l) Gx[c][l] = u[c][l];
      } else {
        c1d<N, false>(T.Dc, u[c], Gx[c]);
      }
    }
  }
  __syncwarp();
  if (DIM == 3) {
    if (live) {
      ld_line<DIM, N, DIM - 1>(a, t, u);
      c_line<DIM, N, false>(T.Dc, u);
      st_line<DIM, N, DIM - 1>(g2, t, u);
    }
    if (g1 == a) __syncwarp();  // the y-lines overwrite sites the z-lines read
  }
  if (live) {
    ld_line<DIM, N, 1>(a, t, u);
    c_line<DIM, N, false>(T.Dc, u);
    st_line<DIM, N, 1>(g1, t, u);
  }
  __syncwarp();
}

// eval_line for two fields at once (the scalar strategy's x and ubar): every
// axis phase handles both, so the evaluation takes half the phases and each
// phase has twice the independent work.  Field 1 uses scratch a, b and writes
// g1, g2 (g1 may be a); field 2 uses c, d and writes its y-derivative in place
// in c and its z-derivative in d.
template <int DIM, int N, bool KEEPQ = false>
HF_DEV void eval_line2(const TabLine<N>& T, const double (&u0)[DIM][N], const double (&w0)[DIM][N], bool live,
                       const LineOff<DIM, N>& t, double* a, double* b, double* g1, double* g2, double* c, double* d,
                       double (&Gx)[DIM][N], double (&Gw)[DIM][N]) {
  double u[DIM][N], w[DIM][N];
  if (live) {
#pragma unroll
    for (int k = 0; k < DIM; ++k)
#pragma unroll
      for (int l = 0; l < N; ++l) {
        u[k][l] = u0[k][l];
        w[k][l] = w0[k][l];
      }
    c_line<DIM, N, false>(T.V, u);
    c_line<DIM, N, false>(T.V, w);
    st_line<DIM, N, DIM - 1>(DIM == 3 ? a : b, t, u);
    st_line<DIM, N, DIM - 1>(DIM == 3 ? c : d, t, w);
  }
  __syncwarp();
  if (DIM == 3) {
    if (live) {
      ld_line<DIM, N, 1>(a, t, u);
      ld_line<DIM, N, 1>(c, t, w);
      c_line<DIM, N, false>(T.V, u);
      c_line<DIM, N, false>(T.V, w);
      st_line<DIM, N, 1>(b, t, u);
      st_line<DIM, N, 1>(d, t, w);
    }
    __syncwarp();
  }
  if (live) {
    ld_line<DIM, N, 0>(b, t, u);
    ld_line<DIM, N, 0>(d, t, w);
    c_line<DIM, N, false>(T.V, u);
    c_line<DIM, N, false>(T.V, w);
    st_line<DIM, N, 0>(a, t, u);
    st_line<DIM, N, 0>(c, t, w);
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      if constexpr (KEEPQ) {
#pragma unroll
        for (int l = 0; l < N; ++l) {
          Gx[k][l] = u[k][l];
          Gw[k][l] = w[k][l];
        }
      } else {
        c1d<N, false>(T.Dc, u[k], Gx[k]);
        c1d<N, false>(T.Dc, w[k], Gw[k]);
      }
    }
  }
  __syncwarp();
  if (DIM == 3) {
    if (live) {
      ld_line<DIM, N, DIM - 1>(a, t, u);
      ld_line<DIM, N, DIM - 1>(c, t, w);
      c_line<DIM, N, false>(T.Dc, u);
      c_line<DIM, N, false>(T.Dc, w);
      st_line<DIM, N, DIM - 1>(g2, t, u);
      st_line<DIM, N, DIM - 1>(d, t, w);
    }
    __syncwarp();  // the y-lines overwrite sites the z-lines read (c always, a when g1 == a)
  }
  if (live) {
    ld_line<DIM, N, 1>(a, t, u);
    ld_line<DIM, N, 1>(c, t, w);
    c_line<DIM, N, false>(T.Dc, u);
    c_line<DIM, N, false>(T.Dc, w);
    st_line<DIM, N, 1>(g1, t, u);
    st_line<DIM, N, 1>(c, t, w);
  }
  __syncwarp();
}

// ---- mbarrier / TMA bulk-copy primitives (PTX) ----
HF_DEV unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
HF_DEV void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
HF_DEV bool mbar_try(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// wait for the phase of parity `parity`; a wait that cannot complete traps
// after ~10 s instead of hanging the device
HF_DEV void mbar_wait(unsigned long long* b, unsigned parity) {
  if (mbar_try(b, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(b, parity))
    if (clock64() - t0 > 20000000000ll) __trap();
}
HF_DEV void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
HF_DEV void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
HF_DEV void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
#ifndef HF_NO_L2HINT
  // The q-point cache is read once per application: its lines are evict-first
  // in L2, so the stream does not displace the vectors (x gathered ~3.4 times,
  // y under reduction, the operands of the neighbouring vector kernels).
  // Measured (profiles/r02/ab_l2_evict_first.txt): tensor4 49.4 vs 50.8 us at
  // config 2, 37.3 vs 39.4 us at config 3, a config-4 CG iteration -5 %.
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
#endif
}

// x-derivative at Gauss point iq (a loop variable) of the Gauss-point values q
// of a line: sum_l Dc[l][iq] q[l], the table column read warp-uniformly from
// the kernel parameters
template <int N>
HF_DEV double dc_at(const TabLine<N>& T, const double (&q)[N], int iq) {
  double s = 0.0;
#pragma unroll
  for (int l = 0; l < N; ++l) s = fma(T.Dc[l][iq], q[l], s);
  return s;
}

// shared-memory plan of one block of W warps, each with NB line buffers and a
// private ring of RW cache stages
template <int DIM, int N, int VAR, typename ST = double>
struct LinePlan {
  using K = LineCfg<DIM, N>;
  // line buffers: A (values at the Gauss points, finally the integration
  // result) and B (scratch, then G2 and the queued z part).  The queued x part
  // stays in the x-line owner's registers (XREG, and G1 overwrites the values
  // in A in place) or replaces the values in A (and G1 takes a third buffer).  XREG measured faster for tensor2 and scalar at Q2
  // (tensor2 b2b 47.7 -> 44.4 us: the smaller slice admits a 12th warp) and
  // slower for tensor4 (55.6 -> 56.4 us at 7 warps, 59 us at the 8 warps the
  // freed buffer admits); at Q4 the 15 extra registers spill.  The scalar
  // strategy adds two buffers for the gradients of ubar.
  static constexpr bool XREG = N <= 3 && VAR != TENSOR4;
  static constexpr int NB = (XREG ? 2 : 3) + (VAR == SCALAR ? 2 : 0);
  static constexpr int NF = (VAR == SCALAR) ? 2 + DIM * DIM : CacheFields<DIM, VAR>::NF;
  // ST elements per (tile, iq) chunk (fp64, or the fp32 storage of a mixed-precision level)
  static constexpr long long CH = TileLayout<DIM, N>::template chunk_e<sizeof(ST)>(NF);
  static constexpr size_t BUDGET = 226 * 1024;
  static constexpr size_t perw(int rw) {
    return sizeof(ST) * (size_t)rw * CH + sizeof(double) * (size_t)NB * LineMap<DIM, N>::BUF + 16 * rw;
  }
  // RW = min(N, 3) stages: at Q2 the chunks of the next tile are issued while
  // the current tile's point phase consumes its own, one tile period ahead of
  // use (RW = 2 < N stalled the point phase on the TMA barrier); at Q4 a full
  // tile of stages would cost 3 of 7 resident warps, so the ring stays 3 deep.
  static constexpr int RW = N < 3 ? N : 3;
  static constexpr int W0 = (int)(BUDGET / perw(RW));
  // warps per block: shared memory bound, capped so the registers of the
  // heaviest variant still fit (scalar ~210 regs -> 8 warps, others ~170 -> 12)
  static constexpr int WMAX = VAR == SCALAR ? 8 : 12;
  static constexpr int W = W0 > WMAX ? WMAX : (W0 < 1 ? 1 : W0);
  static constexpr int NT = 32 * W;
  static constexpr size_t SMEM = (size_t)W * perw(RW);
};

template <int DIM, int N, int VAR, typename ST = double>
__global__ void __launch_bounds__(LinePlan<DIM, N, VAR, ST>::NT, 1)
    k_apply_line(const LineArgs a, const TabLine<N> T) {
  using K = LineCfg<DIM, N>;
  using PL = LinePlan<DIM, N, VAR, ST>;
  using Y = LineMap<DIM, N>;
  constexpr int NF = PL::NF;
  constexpr int NB = PL::NB;
  constexpr int W = PL::W;
  constexpr int RW = PL::RW;
  // rolled point loop (see below): tensor4 only -- at Q4 it made tensor4 10 %
  // faster (3,528 -> 2,352 instructions, 45.8 -> 41.4 us at config 3) and
  // tensor2 / scalar 4-5 % slower (their point phases are cheap, the per-point
  // x-derivative is not)
  constexpr bool ROLL = RW < N && VAR == TENSOR4;
  constexpr long long CH = PL::CH;
  constexpr int NV = DIM * (DIM + 1) / 2;
  constexpr int NM = NV * (NV + 1) / 2;
  if (a.skip && *a.skip) return;
  HF_TL(0);
#ifdef HF_TIMELINE
  {  // the SM this block runs on (slot SLOTS - 5), for per-SM speed statistics
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const unsigned w_ = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if ((threadIdx.x & 31) == 0 && w_ < HF_TL_WARPS) hf_tl_buf[w_ * HF_TL_SLOTS + HF_TL_SLOTS - 5] = smid + 1;
  }
#endif
  extern __shared__ __align__(128) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ST* ring = reinterpret_cast<ST*>(smem) + (size_t)warp * RW * CH;  // this warp's stages (16-byte aligned)
  double* lbuf = reinterpret_cast<double*>(reinterpret_cast<ST*>(smem) + (size_t)W * RW * CH);  // W x NB x BUF
  const ST* cache = reinterpret_cast<const ST*>(a.cache);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(lbuf + (size_t)W * NB * Y::BUF) + warp * RW;
  const long long ntiles = a.tile1;  // tiles [a.tile0, a.tile1) of the (CPW-cell) tiling
  const long long tstride = (long long)N * CH;
  // the tile whose data a work slot processes: the range walked forwards, or
  // backwards when a.reverse (slots past the range stay past it)
  auto dtile = [&](long long tl) { return (a.reverse && tl < a.tile1) ? a.tile1 - 1 - (tl - a.tile0) : tl; };
  // tile of this warp's k-th work item
  // (round robin over blocks and warps; a global or per-SM dynamic schedule
  // measured slower: DESIGN.md §4.1)
  auto tile_k = [&](int k) -> long long {
    return dtile(a.tile0 + blockIdx.x + (warp + (long long)k * W) * (long long)gridDim.x);
  };
  // a tile's cache block (nullptr past the range): formed once per tile, so
  // that issuing a chunk is a multiply-free handful of instructions (the
  // per-chunk 64-bit tile arithmetic was 12 % of the Q4 kernel's instructions)
  auto cblock = [&](long long tile) -> const ST* {
    HF_ASSERT(tile >= ntiles || (tile + 1) * tstride <= a.cache_len);
    return tile < ntiles ? cache + tile * tstride : nullptr;
  };
  // chunk c (iq) of the cache block cb into ring stage s
  auto issue = [&](const ST* cb, int c, int s) {
    if (!cb) return;
    mbar_expect_tx(full + s, (unsigned)(CH * sizeof(ST)));
    tma_load_1d(ring + (size_t)s * CH, cb + (size_t)c * CH, (unsigned)(CH * sizeof(ST)), full + s);
  };
  // y = mask ? x : 0 is written by the preceding k_fill_masked launch.  With
  // programmatic dependent launch (a.fill != 0) this kernel starts while that
  // fill is still running: TMA loads, gathers and the evaluation overlap it,
  // and griddepcontrol.wait orders only the first scatter-add after it.
  bool synced = a.fill != 1;
#ifdef HF_EARLY_XWAIT
  const bool late_x = false;
  if (a.fill == 2) asm volatile("griddepcontrol.wait;" ::: "memory");  // x comes from the primary
#else
  // a.fill == 2: x comes from the primary, but the cache does not.  On small
  // levels (at most two rounds of tiles) the first TMA chunks and the lane
  // offsets are issued while the primary still runs and the wait stands only
  // in front of the first gather: a smoothing at 8^3 47.0 -> 43.2 us, at 16^3
  // 84.2 -> 82.2 us; at 32^3 the early burst competes with the primary's own
  // traffic (+0.6 %), so larger launches wait first
  // (profiles/r02/experiments/ab_pdl_cheb.txt).
  const bool late_x = a.fill == 2 && (a.tile1 - a.tile0) <= 2ll * W * (long long)gridDim.x;
  if (a.fill == 2 && !late_x) asm volatile("griddepcontrol.wait;" ::: "memory");
#endif

  // Start-up order: the first tile's gather, then its TMA chunks, then the
  // constant-bank offsets.  Every warp of the grid starts at once and the TMA
  // burst (23 KB per warp at config 2) would otherwise queue the 9 gather
  // loads behind it; the first tile waited ~3 us for them (tools/timeline.py).
  int slot, m, t;
  bool act;
  line_slot<DIM, N>(lane, slot, m, t, act);
  Gather<DIM, N, VAR> nxt;
  long long t_cur = tile_k(0);  // this work item's tile and the next one's
  if (!late_x) gather_tile<DIM, N, VAR, ST>(a, t_cur, ntiles, m, t, act, nxt);
  HF_TL(HF_TL_SLOTS - 4);
  const ST* cb_cur = cblock(t_cur);
  if (lane == 0) {
    for (int s = 0; s < RW; ++s) mbar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int j = 0; j < RW; ++j) issue(cb_cur, j, j);  // RW <= N: chunks of the first tile
  }
  __syncwarp();
  HF_TL(HF_TL_SLOTS - 3);
  LineOff<DIM, N> lo;
  line_offsets<DIM, N>(lane, T, m, t, lo);
#ifdef HF_TIMELINE
  if (lo.off[0][0] == 12345) lbuf[0] = 0;  // the timestamp below waits for the offsets
#endif
  HF_TL(HF_TL_SLOTS - 2);
  if (late_x) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    gather_tile<DIM, N, VAR, ST>(a, t_cur, ntiles, m, t, act, nxt);
  }
  double* wb = lbuf + (size_t)warp * NB * Y::BUF;
  double* bufs[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) bufs[b] = wb + b * Y::BUF;
  double* A = bufs[0];  // values at the Gauss points -> G1 (in place) -> queued y part -> result
  double* B = bufs[1];  // scratch -> G2 -> queued z part

  unsigned jc = 0;  // this warp's chunk counter
  int k = 0;
  for (;; ++k) {
    if (t_cur >= ntiles) break;
    HF_TL(1 + 4 * (int)k);
    const long long t_nxt = tile_k(k + 1);
    // A kernel launched as this one's programmatic dependent (the Chebyshev
    // update of a small level, hf_cheb_step_after_apply) may become resident
    // once every warp has reached its last tile; it waits for this grid's
    // completion before it reads y.  Released only after this kernel's own
    // wait, so that everything before this kernel has completed by then.
    const bool last = t_nxt >= ntiles;
    if (last && synced) asm volatile("griddepcontrol.launch_dependents;");
    const ST* cb_nxt = cblock(t_nxt);
    const Gather<DIM, N, VAR> g = nxt;
    gather_tile<DIM, N, VAR, ST>(a, t_nxt, ntiles, m, t, act, nxt);  // in flight during this tile
    const long long e = g.e;
    const bool live = g.live;
    double u[DIM][N];
#pragma unroll
    for (int c = 0; c < DIM; ++c)
#pragma unroll
      for (int l = 0; l < N; ++l) u[c][l] = ((g.mb >> (c * N + l)) & 1u) ? 0.0 : g.u[c][l];

    double Gx[DIM][N];
    double Gxu[DIM][N];  // scalar: x part of the gradient of ubar
    // XREG: G1 overwrites the values in A in place; else G1 goes to the third
    // buffer and the queued x part later replaces the values in A
    double* G1 = PL::XREG ? A : bufs[2];
    double* G2 = B;
    double* X = A;
    double vx[DIM][N];  // queued x part of this thread's x-line (XREG)
    // scalar: gradients of x and ubar in one pass (ubar's land in bufs[NB-2]
    // (y) and bufs[NB-1] (z)); above Q4 the doubled line registers spill, so
    // the two fields are evaluated one after the other there
    // the point loop runs rolled when the ring does not hold a whole tile; the
    // x-line owner then keeps its values at the Gauss points and differentiates
    // them point by point (dc_at) instead of holding all N x-derivatives
    static_assert(!ROLL || !LineMap<DIM, N>::CUSTOM, "rolled point loop needs the padded layout");
    constexpr bool FUSED = VAR == SCALAR && N <= 5;
    if (VAR == SCALAR && !FUSED) eval_line<DIM, N, ROLL>(T, g.ub, live, lo, A, B, bufs[NB - 2], bufs[NB - 1], Gxu);
    if (FUSED)
      eval_line2<DIM, N, ROLL>(T, u, g.ub, live, lo, A, B, G1, G2, bufs[NB - 2], bufs[NB - 1], Gx, Gxu);
    else
      eval_line<DIM, N, ROLL>(T, u, live, lo, A, B, G1, G2, Gx);
    HF_TL(2 + 4 * (int)k);

    // ---------------- P: q-point physics along this thread's x-line ----------------
    double mu = 0.0, lam = 0.0;
    if (VAR == SCALAR && live) {
      mu = __ldg(a.mu + e);
      lam = __ldg(a.lam + e);
    }
    // one Gauss point of this thread's x-line from its cache chunk
    auto point = [&](const int iq, const ST* st) {
      if (live) {
      // this thread's x-line site iq (ROLL: iq is a loop variable; the padded
      // layout puts the sites of an x-line CPWP doubles apart)
      const int pt = ROLL ? lo.off[0][0] + iq * LineLay<DIM, N>::CPWP : lo.off[0][iq];
      double f[NF];
#pragma unroll
      for (int q = 0; q < NF; ++q) f[q] = (double)st[q * K::LANES];
      double gu[DIM][DIM];
#pragma unroll
      for (int cc = 0; cc < DIM; ++cc) {
        gu[cc][0] = ROLL ? dc_at(T, Gx[cc], iq) : Gx[cc][iq];
        gu[cc][1] = G1[cc * Y::CS + pt];
        if (DIM == 3) gu[cc][DIM - 1] = G2[cc * Y::CS + pt];
      }
      double G[DIM][DIM];
      if (VAR == TENSOR4) {
        double sinv[DIM][DIM], tau[DIM][DIM];
#pragma unroll
        for (int i = 0; i < DIM; ++i)
#pragma unroll
          for (int j = 0; j < DIM; ++j) {
            tau[i][j] = f[hf_slot<DIM>(i, j)];
            sinv[i][j] = f[NV + NM + i * DIM + j];
          }
        qp_action<DIM, true>(gu, sinv, tau, 0.0, 0.0, f + NV, 1.0, G);  // JxW folded into tau, M
      } else if (VAR == TENSOR2) {
        double sinv[DIM][DIM], tau[DIM][DIM];
#pragma unroll
        for (int i = 0; i < DIM; ++i)
#pragma unroll
          for (int j = 0; j < DIM; ++j) {
            tau[i][j] = f[2 + hf_slot<DIM>(i, j)];
            sinv[i][j] = f[2 + NV + i * DIM + j];
          }
        qp_action<DIM, false>(gu, sinv, tau, f[0], f[1], nullptr, 1.0, G);  // JxW folded into c1', c2', tau
      } else {
        // rebuild F, b, tau = mu b - c1 I and s_inv from ubar (operators.py:349-363)
        double ji[DIM][DIM];
#pragma unroll
        for (int r = 0; r < DIM; ++r)
#pragma unroll
          for (int q = 0; q < DIM; ++q) ji[r][q] = f[1 + r * DIM + q];
        double gub[DIM][DIM];
#pragma unroll
        for (int cc = 0; cc < DIM; ++cc) {
          gub[cc][0] = ROLL ? dc_at(T, Gxu[cc], iq) : Gxu[cc][iq];
          gub[cc][1] = bufs[NB - 2][cc * Y::CS + pt];
          if (DIM == 3) gub[cc][DIM - 1] = bufs[NB - 1][cc * Y::CS + pt];
        }
        double F[DIM * DIM];
#pragma unroll
        for (int i = 0; i < DIM; ++i)
#pragma unroll
          for (int Aa = 0; Aa < DIM; ++Aa) {
            double sm = (i == Aa) ? 1.0 : 0.0;
#pragma unroll
            for (int q = 0; q < DIM; ++q) sm = fma(gub[i][q], ji[q][Aa], sm);
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
        qp_action<DIM, false>(gu, sinv, tau, 2.0 * c1, 2.0 * lam, nullptr, f[NF - 1], G);
      }
#pragma unroll
      for (int cc = 0; cc < DIM; ++cc) {
        if (PL::XREG)
          vx[cc][iq] = G[cc][0];
        else
          X[cc * Y::CS + pt] = G[cc][0];
        G1[cc * Y::CS + pt] = G[cc][1];
        if (DIM == 3) G2[cc * Y::CS + pt] = G[cc][DIM - 1];
      }
    }
    };
    if constexpr (RW >= N) {
      static_assert(RW <= N, "a ring at least a tile deep is exactly a tile deep");
      // the whole tile's chunks are resident: wait once, then the N points
      // are free of barriers and the compiler interleaves their chains
      // tensor4's first tile waits per point: at kernel start every warp's
      // chunks are in one 24 MB burst that HBM delivers in ~3.7 us, chunk 0 of
      // every warp first, so the point phase can start on chunk 0 while
      // chunks 1 and 2 arrive (config 2 back to back 50.3 -> 49.6 us).  Later
      // tiles find their chunks resident; per-point waits there would only
      // keep the compiler from interleaving the points' chains.  tensor2 and
      // scalar chunks are small and gain nothing (+0.5 % with the extra code).
      if (VAR == TENSOR4 && k == 0) {
#pragma unroll
        for (int iq = 0; iq < N; ++iq) {
          mbar_wait(full + iq, 0u);
          point(iq, ring + (size_t)iq * CH + slot);
        }
      } else {
#pragma unroll
        for (int iq = 0; iq < N; ++iq) mbar_wait(full + iq, (unsigned)k & 1u);  // RW == N: chunk iq sits in stage iq
#pragma unroll
        for (int iq = 0; iq < N; ++iq) point(iq, ring + (size_t)iq * CH + slot);
      }
      __syncwarp();
      if (lane < N) {  // stages consumed by every lane: lanes 0..N-1 refill them with the next tile's chunks
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(cb_nxt, lane, lane);  // RW == N: the next tile's chunks
      }
      jc += N;
    } else {
      // Q4 (N = 5 > RW): tensor4's point phase as a rolled loop; five unrolled
      // copies of its point code made the kernel 3,500 instructions long and
      // 12 % of the warp stalls were instruction fetches
#pragma unroll(ROLL ? 1 : N)
      for (int iq = 0; iq < N; ++iq, ++jc) {
        const int s = (int)(jc % RW);
        mbar_wait(full + s, (jc / RW) & 1u);
        point(iq, ring + (size_t)s * CH + slot);
        __syncwarp();
        if (lane == 0) {  // stage consumed by every lane: refill it with chunk jc + RW
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          if (iq + RW < N)
            issue(cb_cur, iq + RW, s);
          else
            issue(cb_nxt, iq + RW - N, s);
        }
      }
    }
    __syncwarp();
    HF_TL(3 + 4 * (int)k);
    // ---------------- I1: transposed collocation derivative per axis (x in registers, y/z in place) ----------------
    if (live) {
      double v[DIM][N];
      if (PL::XREG) {
        c_line<DIM, N, true>(T.Dc, vx);
      } else {
        ld_line<DIM, N, 0>(X, lo, v);
        c_line<DIM, N, true>(T.Dc, v);
        st_line<DIM, N, 0>(X, lo, v);
      }
      ld_line<DIM, N, 1>(G1, lo, v);
      c_line<DIM, N, true>(T.Dc, v);
      st_line<DIM, N, 1>(G1, lo, v);
      if (DIM == 3) {
        ld_line<DIM, N, DIM - 1>(G2, lo, v);
        c_line<DIM, N, true>(T.Dc, v);
        st_line<DIM, N, DIM - 1>(G2, lo, v);
      }
    }
    __syncwarp();
    // ---------------- I2: sum, transposed interpolation along x ----------------
    if (live) {
      double v[DIM][N], w[DIM][N];
      if (PL::XREG) {
#pragma unroll
        for (int cc = 0; cc < DIM; ++cc)
#pragma unroll
          for (int l = 0; l < N; ++l) v[cc][l] = vx[cc][l];
      } else {
        ld_line<DIM, N, 0>(X, lo, v);
      }
      ld_line<DIM, N, 0>(G1, lo, w);
#pragma unroll
      for (int cc = 0; cc < DIM; ++cc)
#pragma unroll
        for (int l = 0; l < N; ++l) v[cc][l] += w[cc][l];
      if (DIM == 3) {
        ld_line<DIM, N, 0>(G2, lo, w);
#pragma unroll
        for (int cc = 0; cc < DIM; ++cc)
#pragma unroll
          for (int l = 0; l < N; ++l) v[cc][l] += w[cc][l];
      }
      c_line<DIM, N, true>(T.V, v);
      st_line<DIM, N, 0>(A, lo, v);
    }
    __syncwarp();
    if (DIM == 3) {
      if (live) {
        double v[DIM][N];
        ld_line<DIM, N, 1>(A, lo, v);
        c_line<DIM, N, true>(T.V, v);
        st_line<DIM, N, 1>(A, lo, v);
      }
      __syncwarp();
    }
    // ---------------- I4: last axis, scatter-add ----------------
    if (!synced) {  // the fill kernel (PDL primary) has completed and its writes are visible
      asm volatile("griddepcontrol.wait;" ::: "memory");
      if (last) asm volatile("griddepcontrol.launch_dependents;");
      synced = true;
    }
    if (live) {
      double v[DIM][N];
      ld_line<DIM, N, DIM - 1>(A, lo, v);
      c_line<DIM, N, true>(T.V, v);
      unsigned nb, s_last;
      last_axis_line<DIM, N>(a.lat, g.node0, t, nb, s_last);
      const unsigned long long polk = l2_keep_policy();
#pragma unroll
      for (int l = 0; l < N; ++l) {
        const unsigned d0 = (nb + l * s_last) * DIM;
        HF_ASSERT((long long)d0 + DIM <= a.lat.n_nodes * DIM);
        // constrained rows take +0 (their identity value x is unchanged):
        // no branch per DoF around the reductions
#pragma unroll
        for (int cc = 0; cc < DIM; ++cc)
          red_keep(reinterpret_cast<ST*>(a.y) + d0 + cc, ((g.mb >> (cc * N + l)) & 1u) ? (ST)0 : (ST)v[cc][l], polk);
      }
    }
    __syncwarp();  // line buffers are reused by the next tile
    t_cur = t_nxt;
    cb_cur = cb_nxt;
    HF_TL(4 + 4 * (int)k);
  }
  HF_TL(HF_TL_SLOTS - 1);
}

}  // namespace hf
