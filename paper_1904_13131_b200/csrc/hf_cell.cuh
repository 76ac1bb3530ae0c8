// Cell kernels of the matrix-free Neo-Hookean tangent (sm_100a, fp64).
//
// One "team" of NQ = N^DIM threads processes one cell; thread (i,j,k) owns the
// lattice node (i,j,k) of the cell AND the Gauss point (i,j,k) (the kernels are
// instantiated for n_qpoints = degree+1, so nloc == nq).  CPB cells share a
// block of NT threads; every sum-factorisation stage is one 1D contraction in
// shared memory followed by a block barrier.
//
// Reference correspondence (/root/reference/pkg/src/hyperfree):
//   gather            fespace.py:291-293 (+ operators.py:333-334 zeroing)
//   evaluate grads    fespace.py:224-239   -> interpolate to Gauss points with V
//                                             along every axis, then collocation
//                                             derivatives (Dco) per direction
//   q-point physics   operators.py:341-392 (three caching strategies)
//   integrate         fespace.py:258-288   -> transposed collocation + V^T chain
//   scatter-add       fespace.py:296-324   -> fp64 atomics, constrained rows dropped
//   cache build       operators.py:179-202, 292-311; material.py:121-124, 195-230
//   diagonal          operators.py:395-410 -> direct sum-factorised diagonal
//   residual          operators.py:205-224
#pragma once
#include "hf_common.cuh"

namespace hf {

enum Variant { SCALAR = 0, TENSOR2 = 1, TENSOR4 = 2 };

template <int DIM, int N>
struct Cfg {
  static constexpr int NQ = (DIM == 2) ? N * N : N * N * N;
  static constexpr int C = DIM;
  static constexpr int CPB = (256 / NQ) > 0 ? (256 / NQ) : 1;
  static constexpr int NT = ((CPB * NQ + 31) / 32) * 32;
  static constexpr int SBUF = C * NQ;        // doubles per cell per ping-pong buffer
  static constexpr int NV = DIM * (DIM + 1) / 2;
  static constexpr int NM = NV * (NV + 1) / 2;
  // shared memory: 4 tables (+3 diagonal tables) + A, B, G buffers
  static constexpr int TAB = 7 * N * N;
  static constexpr size_t SMEM = sizeof(double) * (TAB + (size_t)CPB * SBUF * (2 + DIM));
};

// number of cached doubles per q-point (SoA fields)
template <int DIM, int VAR>
struct CacheFields {
  static constexpr int NV = DIM * (DIM + 1) / 2;
  static constexpr int NM = NV * (NV + 1) / 2;
  // tensor4: JxW tau(NV), JxW M(NM), sinv(D*D) ; tensor2: JxW 2c1, JxW 2lambda, JxW tau(NV), sinv ;
  // scalar: c1 J^-1(D*D) JxW (the geometry it re-reads, stored beside c1 in the tile layout).
  // tensor4/tensor2 fold the quadrature weight JxW into the fields the q-point
  // action is linear in (deal.II's practice), so it is neither stored nor
  // multiplied per point: 36 / 17 doubles per q-point instead of the
  // reference's 37 / 18 (operators.py:259-289 keep JxW in the geometry).
  static constexpr int NF = VAR == TENSOR4 ? NV + NM + DIM * DIM
                                           : (VAR == TENSOR2 ? 2 + NV + DIM * DIM : 2 + DIM * DIM);
};

struct CellArgs {
  HfTables tab;
  HfLattice lat;
  int degree;
  const double* x;          // input vector (apply) / state (build, residual)
  double* y;                // output (atomic accumulation)
  const double* cache;      // SoA [field][n_qp]
  double* cache_out;        // build output
  const double* jinv;       // SoA [DIM*DIM][n_qp], entry (a, A) = dxi_a/dX_A
  const double* jxw;        // [n_qp]
  const double* mu;         // [n_el]
  const double* lam;        // [n_el]
  const double* ubar;       // scalar strategy: snapshot of the linearisation point
  const uint8_t* mask;      // [n_dofs] constrained DoFs
  const uint32_t* lmask;    // [n_el * lines] constraint bits per last-axis line (k_line_masks)
  const int* skip;          // optional device flag; non-zero -> kernel is a no-op
  int fill;                 // apply: 0 plain, 1/2 PDL secondary (hf_line.cuh LineArgs::fill)
  int fp32;                 // apply/build: cache and x/y stored as float (mixed-precision levels)
  long long cache_len;      // cache elements (bounds checks of the debug build)
  long long tile0, tile1;   // apply: tile range; tile1 < 0 means all tiles
  int reserve_sms = 0;      // apply: leave this many SMs' worth of blocks free (a concurrent NCCL kernel)
  int reverse = 0;          // apply: walk the tile range backwards
  unsigned long long* detmin;  // ordered-double min of det F (build / residual / range)
  unsigned long long* detmax;
};

struct Team {
  int slot, lq, idx[3];
  long long e;
  bool act;
  long long node;  // global lattice node of (cell, lq)
};

template <int DIM, int N>
HF_DEV Team make_team(const HfLattice& lat, int degree) {
  using K = Cfg<DIM, N>;
  Team t;
  t.slot = threadIdx.x / K::NQ;
  t.lq = threadIdx.x - t.slot * K::NQ;
  t.idx[0] = t.lq % N;
  t.idx[1] = (t.lq / N) % N;
  t.idx[2] = (DIM == 3) ? t.lq / (N * N) : 0;
  t.e = (long long)blockIdx.x * K::CPB + t.slot;
  t.act = (t.slot < K::CPB) && (t.e < lat.n_el);
  if (t.slot >= K::CPB) t.slot = 0;  // keep pointers in range for idle lanes
  long long node = 0;
  if (t.act) {
    long long r = t.e;
    int ex = (int)(r % lat.cells[0]);
    r /= lat.cells[0];
    int ey = (int)(r % lat.cells[1]);
    int ez = (DIM == 3) ? (int)(r / lat.cells[1]) : 0;
    node = (long long)(ex * degree + t.idx[0]) +
           (long long)lat.nodes[0] * ((long long)(ey * degree + t.idx[1]) +
                                       (long long)lat.nodes[1] * (long long)(ez * degree + t.idx[2]));
  }
  t.node = node;
  return t;
}

// smem table offsets
template <int N> struct Tab {
  static constexpr int V = 0, VT = N * N, DC = 2 * N * N, DCT = 3 * N * N;
  static constexpr int VV = 4 * N * N, DD = 5 * N * N, VD = 6 * N * N;  // diagonal tables, [l=q][o=node]
};

template <int DIM, int N>
HF_DEV void load_tables(double* sm, const HfTables& tb, bool diag_tables) {
  for (int t = threadIdx.x; t < N * N; t += blockDim.x) {
    int l = t / N, o = t - l * N;
    sm[Tab<N>::V + t] = tb.V[l * N + o];
    sm[Tab<N>::VT + t] = tb.V[o * N + l];
    sm[Tab<N>::DC + t] = tb.Dc[l * N + o];
    sm[Tab<N>::DCT + t] = tb.DcT[l * N + o];
    if (diag_tables) {  // M[l=q][o=node] products of the ORIGINAL tables (no collocation)
      double v = tb.V[o * N + l], d = tb.D[o * N + l];
      sm[Tab<N>::VV + t] = v * v;
      sm[Tab<N>::DD + t] = d * d;
      sm[Tab<N>::VD + t] = v * d;
    }
  }
}

template <int AX, int N>
HF_DEV constexpr int ax_stride() { return AX == 0 ? 1 : (AX == 1 ? N : N * N); }

// out[c][pt] = sum_l M[l*N + o] * in[c][pt with axis AX -> l]
template <int DIM, int N, int NC, int AX>
HF_DEV void contract(const double* __restrict__ in, double* __restrict__ out, const double* __restrict__ M,
                     const Team& t) {
  constexpr int NQ = Cfg<DIM, N>::NQ;
  constexpr int STR = ax_stride<AX, N>();
  const int o = t.idx[AX];
  const int base = t.lq - o * STR;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double acc = 0.0;
#pragma unroll
    for (int l = 0; l < N; ++l) acc = fma(M[l * N + o], in[c * NQ + base + l * STR], acc);
    out[c * NQ + t.lq] = acc;
  }
}

template <int DIM, int N, int NC, int AX>
HF_DEV void contract_reg(const double* __restrict__ in, double* out, const double* __restrict__ M, const Team& t) {
  constexpr int NQ = Cfg<DIM, N>::NQ;
  constexpr int STR = ax_stride<AX, N>();
  const int o = t.idx[AX];
  const int base = t.lq - o * STR;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double acc = 0.0;
#pragma unroll
    for (int l = 0; l < N; ++l) acc = fma(M[l * N + o], in[c * NQ + base + l * STR], acc);
    out[c] = acc;
  }
}

// Unit-cell gradients g[c][a] at this thread's Gauss point from the nodal
// values already stored in A (per-cell slice).  Uses B as scratch.  Ends with
// a barrier so A/B may be reused.
template <int DIM, int N>
HF_DEV void eval_gradients(double* A, double* B, const double* sm, const Team& t, double (&g)[DIM][DIM]) {
  constexpr int NC = DIM;
  constexpr int NQ = Cfg<DIM, N>::NQ;
  const double* U;
  if (t.act) contract<DIM, N, NC, 0>(A, B, sm + Tab<N>::V, t);
  __syncthreads();
  if (t.act) contract<DIM, N, NC, 1>(B, A, sm + Tab<N>::V, t);
  __syncthreads();
  if (DIM == 3) {
    if (t.act) contract<DIM, N, NC, 2>(A, B, sm + Tab<N>::V, t);
    __syncthreads();
    U = B;
  } else {
    U = A;
  }
  if (t.act) {
    double tmp[NC];
    contract_reg<DIM, N, NC, 0>(U, tmp, sm + Tab<N>::DC, t);
#pragma unroll
    for (int c = 0; c < NC; ++c) g[c][0] = tmp[c];
    contract_reg<DIM, N, NC, 1>(U, tmp, sm + Tab<N>::DC, t);
#pragma unroll
    for (int c = 0; c < NC; ++c) g[c][1] = tmp[c];
    if (DIM == 3) {
      contract_reg<DIM, N, NC, (DIM == 3 ? 2 : 1)>(U, tmp, sm + Tab<N>::DC, t);
#pragma unroll
      for (int c = 0; c < NC; ++c) g[c][DIM - 1] = tmp[c];
    }
  }
  (void)NQ;
  __syncthreads();
}

// Local vector y_loc[c] at this thread's node from queued q-point data
// G[c][a] (already multiplied by JxW).  Uses A, B, Gs buffers.
template <int DIM, int N>
HF_DEV void integrate_gradients(double* A, double* B, double* Gs, const double* sm, const Team& t,
                                const double (&G)[DIM][DIM], double (&yl)[DIM]) {
  constexpr int NC = DIM;
  constexpr int NQ = Cfg<DIM, N>::NQ;
  if (t.act) {
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int a = 0; a < DIM; ++a) Gs[(c * DIM + a) * NQ + t.lq] = G[c][a];
  }
  __syncthreads();
  if (t.act) {
    const double* M = sm + Tab<N>::DCT;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const int STR = a == 0 ? 1 : (a == 1 ? N : N * N);
        const int o = t.idx[a];
        const int base = t.lq - o * STR;
        const double* src = Gs + (c * DIM + a) * NQ;
#pragma unroll
        for (int l = 0; l < N; ++l) acc = fma(M[l * N + o], src[base + l * STR], acc);
      }
      A[c * NQ + t.lq] = acc;
    }
  }
  __syncthreads();
  if (DIM == 3) {
    if (t.act) contract<DIM, N, NC, 0>(A, B, sm + Tab<N>::VT, t);
    __syncthreads();
    if (t.act) contract<DIM, N, NC, 1>(B, A, sm + Tab<N>::VT, t);
    __syncthreads();
    if (t.act) contract_reg<DIM, N, NC, (DIM == 3 ? 2 : 1)>(A, yl, sm + Tab<N>::VT, t);
  } else {
    if (t.act) contract<DIM, N, NC, 0>(A, B, sm + Tab<N>::VT, t);
    __syncthreads();
    if (t.act) contract_reg<DIM, N, NC, 1>(B, yl, sm + Tab<N>::VT, t);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// q-point constitutive kernels
// ---------------------------------------------------------------------------

// F, J, F^-1, b, tau, sinv from unit gradients of u, the geometry J^-1 and (mu, lam).
template <int DIM>
struct Kin {
  double J, c1;
  double tau[DIM][DIM];
  double sinv[DIM][DIM];
};

template <int DIM>
HF_DEV void kinematics(const double (&gu)[DIM][DIM], const double (&ji)[DIM][DIM], double mu, double lam, Kin<DIM>& k,
                       bool with_sinv = true) {
  double F[DIM * DIM];
#pragma unroll
  for (int i = 0; i < DIM; ++i)
#pragma unroll
    for (int A = 0; A < DIM; ++A) {
      double s = (i == A) ? 1.0 : 0.0;
#pragma unroll
      for (int a = 0; a < DIM; ++a) s = fma(gu[i][a], ji[a][A], s);
      F[i * DIM + A] = s;
    }
  k.J = hf_det<DIM>(F);
  k.c1 = mu - 2.0 * lam * log(k.J);
#pragma unroll
  for (int i = 0; i < DIM; ++i)
#pragma unroll
    for (int j = 0; j < DIM; ++j) {
      double b = 0.0;
#pragma unroll
      for (int A = 0; A < DIM; ++A) b = fma(F[i * DIM + A], F[j * DIM + A], b);
      k.tau[i][j] = mu * b - (i == j ? k.c1 : 0.0);
    }
  if (with_sinv) {
    double Fi[DIM * DIM];
    hf_inv<DIM>(F, k.J, Fi);
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int j = 0; j < DIM; ++j) {
        double s = 0.0;
#pragma unroll
        for (int A = 0; A < DIM; ++A) s = fma(ji[a][A], Fi[A * DIM + j], s);
        k.sinv[a][j] = s;
      }
  }
}

// queued G[i][a] = jxw * sum_j P[i][j] sinv[a][j] with
// P = C:grad_s(g) + g.tau,  g = gu . sinv.
// material action: closed form (c1p g_s + c2p tr(g_s) I) or Voigt matrix M.
template <int DIM, bool VOIGT>
HF_DEV void qp_action(const double (&gu)[DIM][DIM], const double (&sinv)[DIM][DIM], const double (&tau)[DIM][DIM],
                      double c1p, double c2p, const double* Mp, double jxw, double (&G)[DIM][DIM]) {
  constexpr int NV = DIM * (DIM + 1) / 2;
  double g[DIM][DIM];
#pragma unroll
  for (int i = 0; i < DIM; ++i)
#pragma unroll
    for (int j = 0; j < DIM; ++j) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < DIM; ++a) s = fma(gu[i][a], sinv[a][j], s);
      g[i][j] = s;
    }
  double P[DIM][DIM];
  if (VOIGT) {
    double gam[NV], sig[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      int a = k < DIM ? k : (DIM == 2 ? 0 : (k == 3 ? 1 : 0));
      int b = k < DIM ? k : (DIM == 2 ? 1 : (k == 5 ? 1 : 2));
      gam[k] = (k < DIM) ? g[a][a] : (g[a][b] + g[b][a]);  // engineering shear = 2 sym
    }
#pragma unroll
    for (int r = 0; r < NV; ++r) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        int idx = r <= c ? hf_triu<NV>(r, c) : hf_triu<NV>(c, r);
        s = fma(Mp[idx], gam[c], s);
      }
      sig[r] = s;
    }
#pragma unroll
    for (int i = 0; i < DIM; ++i)
#pragma unroll
      for (int j = 0; j < DIM; ++j) P[i][j] = sig[hf_slot<DIM>(i, j)];
  } else {
    double tr = 0.0;
#pragma unroll
    for (int i = 0; i < DIM; ++i) tr += g[i][i];
#pragma unroll
    for (int i = 0; i < DIM; ++i)
#pragma unroll
      for (int j = 0; j < DIM; ++j) P[i][j] = c1p * 0.5 * (g[i][j] + g[j][i]) + (i == j ? c2p * tr : 0.0);
  }
#pragma unroll
  for (int i = 0; i < DIM; ++i)
#pragma unroll
    for (int j = 0; j < DIM; ++j) {
      double s = P[i][j];
#pragma unroll
      for (int k = 0; k < DIM; ++k) s = fma(g[i][k], tau[k][j], s);
      P[i][j] = s;
    }
#pragma unroll
  for (int i = 0; i < DIM; ++i)
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < DIM; ++j) s = fma(P[i][j], sinv[a][j], s);
      G[i][a] = s * jxw;
    }
}

// warp-aggregated ordered min/max (all 32 lanes must call; invalid lanes pass valid=false)
HF_DEV void warp_minmax_atomic(unsigned long long* amin, unsigned long long* amax, double v, bool valid) {
  unsigned long long mn = valid ? hf_ord(v) : ~0ull;
  unsigned long long mx = valid ? hf_ord(v) : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, o);
    unsigned long long b = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    if (amin && mn != ~0ull) atomicMin(amin, mn);
    if (amax && mx != 0ull) atomicMax(amax, mx);
  }
}

template <int DIM>
HF_DEV void load_jinv(const CellArgs& a, long long qi, double (&ji)[DIM][DIM]) {
  const long long nqp = a.lat.n_qp;
#pragma unroll
  for (int r = 0; r < DIM; ++r)
#pragma unroll
    for (int c = 0; c < DIM; ++c) ji[r][c] = __ldg(a.jinv + (r * DIM + c) * nqp + qi);
}

template <int DIM, int N>
HF_DEV void gather_nodal(const double* __restrict__ v, const uint8_t* __restrict__ mask, const Team& t, double* A) {
  constexpr int NQ = Cfg<DIM, N>::NQ;
  if (t.act) {
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      long long d = t.node * DIM + c;
      double xv = __ldg(v + d);
      if (mask && mask[d]) xv = 0.0;
      A[c * NQ + t.lq] = xv;
    }
  }
}

// ---------------------------------------------------------------------------
// cache build (operators.py:292-311); also records min det F
// ---------------------------------------------------------------------------
template <int DIM, int N, int VAR, typename ST = double>
__global__ void __launch_bounds__(Cfg<DIM, N>::NT) k_build(const CellArgs a) {
  using K = Cfg<DIM, N>;
  constexpr int NQ = K::NQ;
  constexpr int NV = K::NV;
  extern __shared__ double sm[];
  load_tables<DIM, N>(sm, a.tab, false);
  Team t = make_team<DIM, N>(a.lat, a.degree);
  double* A = sm + K::TAB + t.slot * K::SBUF;
  double* B = A + K::CPB * K::SBUF;
  const long long qi = t.e * NQ + t.lq;
  gather_nodal<DIM, N>(a.x, nullptr, t, A);
  __syncthreads();
  double gu[DIM][DIM];
  eval_gradients<DIM, N>(A, B, sm, t, gu);
  double ji[DIM][DIM];
  Kin<DIM> k;
  double lam = 0.0;
  if (t.act) {
    load_jinv<DIM>(a, qi, ji);
    const double mu = __ldg(a.mu + t.e);
    lam = __ldg(a.lam + t.e);
    kinematics<DIM>(gu, ji, mu, lam, k, VAR != SCALAR);
  }
  warp_minmax_atomic(a.detmin, nullptr, t.act ? k.J : 0.0, t.act);
  if (!t.act) return;
  constexpr int NF = CacheFields<DIM, VAR>::NF;
  using TL = TileLayout<DIM, N>;
  ST* o = reinterpret_cast<ST*>(a.cache_out);  // fp64, or fp32 storage of a mixed-precision level
  auto put = [&](int f, double v) {
    const long long i = TL::template index_e<sizeof(ST)>(t.e, t.lq, f, NF);
    HF_ASSERT(i >= 0 && i < a.cache_len);
    o[i] = (ST)v;
  };
  int f = 0;
  if (VAR == SCALAR) {
    put(f++, k.c1);
#pragma unroll
    for (int r = 0; r < DIM; ++r)
#pragma unroll
      for (int c = 0; c < DIM; ++c) put(f++, ji[r][c]);
    put(f++, __ldg(a.jxw + qi));
    return;
  }
  const double w = __ldg(a.jxw + qi);  // folded into the fields below (CacheFields)
  if (VAR == TENSOR2) {
    put(f++, w * (2.0 * k.c1));
    put(f++, w * (2.0 * lam));
  }
#pragma unroll
  for (int s = 0; s < NV; ++s) {
    int i = s < DIM ? s : (DIM == 2 ? 0 : (s == 3 ? 1 : 0));
    int j = s < DIM ? s : (DIM == 2 ? 1 : (s == 5 ? 1 : 2));
    put(f++, w * k.tau[i][j]);
  }
  if (VAR == TENSOR4) {
    // Voigt matrix of J c (material.py:195-208), packed upper (218-222)
#pragma unroll
    for (int r = 0; r < NV; ++r)
#pragma unroll
      for (int c = r; c < NV; ++c) {
        double v = 0.0;
        if (r < DIM && c < DIM) v = 2.0 * lam + (r == c ? 2.0 * k.c1 : 0.0);
        else if (r == c) v = k.c1;
        put(f++, w * v);
      }
  }
#pragma unroll
  for (int r = 0; r < DIM; ++r)
#pragma unroll
    for (int c = 0; c < DIM; ++c) put(f++, k.sinv[r][c]);
}

// ---------------------------------------------------------------------------
// direct diagonal: diag(n,c) = sum_q sum_ab dN_a dN_b K^c_ab,
//   K^c = JxW * sinv (H^c + tau) sinv^T,  H^c[j][k] = M[slot(c,j)][slot(c,k)]
// (closed form strategies: H^c = c1'/2 I + (c1'/2 + c2') e_c e_c^T).
// Sum-factorised with the squared/product 1D tables; equals the reference's
// unit-vector local applies (operators.py:395-410).
// ---------------------------------------------------------------------------
template <int DIM, int N, int VAR>
__global__ void __launch_bounds__(Cfg<DIM, N>::NT) k_diag(const CellArgs a) {
  using K = Cfg<DIM, N>;
  constexpr int NQ = K::NQ;
  constexpr int NF = CacheFields<DIM, VAR>::NF;
  constexpr int NV = K::NV;
  extern __shared__ double sm[];
  load_tables<DIM, N>(sm, a.tab, true);
  Team t = make_team<DIM, N>(a.lat, a.degree);
  double* A = sm + K::TAB + t.slot * K::SBUF;
  double* B = A + K::CPB * K::SBUF;
  const long long qi = t.e * NQ + t.lq;

  double sinv[DIM][DIM], tau[DIM][DIM], jxw = 0.0;
  double Hc[DIM][DIM][DIM];  // [c][j][k]
  if (VAR == SCALAR) {
    gather_nodal<DIM, N>(a.ubar, nullptr, t, A);
    __syncthreads();
    double gub[DIM][DIM];
    eval_gradients<DIM, N>(A, B, sm, t, gub);
    if (t.act) {
      double ji[DIM][DIM];
      load_jinv<DIM>(a, qi, ji);
      const double mu = __ldg(a.mu + t.e), lam = __ldg(a.lam + t.e);
      Kin<DIM> k;
      kinematics<DIM>(gub, ji, mu, lam, k, true);
      const double c1 = a.cache[TileLayout<DIM, N>::index(t.e, t.lq, 0, NF)];  // cached c1 (same value as k.c1)
#pragma unroll
      for (int i = 0; i < DIM; ++i)
#pragma unroll
        for (int j = 0; j < DIM; ++j) {
          sinv[i][j] = k.sinv[i][j];
          tau[i][j] = k.tau[i][j] + (i == j ? k.c1 - c1 : 0.0);
        }
      jxw = __ldg(a.jxw + qi);
      const double c1p = 2.0 * c1, c2p = 2.0 * lam;
#pragma unroll
      for (int c = 0; c < DIM; ++c)
#pragma unroll
        for (int j = 0; j < DIM; ++j)
#pragma unroll
          for (int k2 = 0; k2 < DIM; ++k2)
            Hc[c][j][k2] = (j == k2 ? 0.5 * c1p : 0.0) + (j == c && k2 == c ? 0.5 * c1p + c2p : 0.0);
    }
  } else if (t.act) {
    double cf[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) cf[f] = a.cache[TileLayout<DIM, N>::index(t.e, t.lq, f, NF)];
    const int off = (VAR == TENSOR2) ? 2 : 0;
#pragma unroll
    for (int i = 0; i < DIM; ++i)
#pragma unroll
      for (int j = 0; j < DIM; ++j) {
        tau[i][j] = cf[off + hf_slot<DIM>(i, j)];
        sinv[i][j] = cf[off + NV + (VAR == TENSOR4 ? K::NM : 0) + i * DIM + j];
      }
    jxw = 1.0;  // folded into the cached fields (CacheFields)
#pragma unroll
    for (int c = 0; c < DIM; ++c)
#pragma unroll
      for (int j = 0; j < DIM; ++j)
#pragma unroll
        for (int k2 = 0; k2 < DIM; ++k2) {
          if (VAR == TENSOR4) {
            int r = hf_slot<DIM>(c, j), s = hf_slot<DIM>(c, k2);
            Hc[c][j][k2] = cf[NV + (r <= s ? hf_triu<NV>(r, s) : hf_triu<NV>(s, r))];
          } else {
            Hc[c][j][k2] = (j == k2 ? 0.5 * cf[0] : 0.0) + (j == c && k2 == c ? 0.5 * cf[0] + cf[1] : 0.0);
          }
        }
  }
  // K^c_ab (symmetric); off-diagonal pairs carry a factor 2
  double Kc[DIM][DIM * (DIM + 1) / 2];
  if (t.act) {
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      double W[DIM][DIM];  // (H + tau) sinv^T
#pragma unroll
      for (int j = 0; j < DIM; ++j)
#pragma unroll
        for (int b = 0; b < DIM; ++b) {
          double s = 0.0;
#pragma unroll
          for (int k2 = 0; k2 < DIM; ++k2) s = fma(Hc[c][j][k2] + tau[j][k2], sinv[b][k2], s);
          W[j][b] = s;
        }
      int p = 0;
#pragma unroll
      for (int aa = 0; aa < DIM; ++aa)
#pragma unroll
        for (int b = aa; b < DIM; ++b) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < DIM; ++j) s = fma(sinv[aa][j], W[j][b], s);
          Kc[c][p++] = s * jxw * (aa == b ? 1.0 : 2.0);
        }
    }
  }
  double acc[DIM];
#pragma unroll
  for (int c = 0; c < DIM; ++c) acc[c] = 0.0;
  int p = 0;
#pragma unroll
  for (int aa = 0; aa < DIM; ++aa)
#pragma unroll
    for (int b = aa; b < DIM; ++b, ++p) {
      if (t.act) {
#pragma unroll
        for (int c = 0; c < DIM; ++c) A[c * NQ + t.lq] = Kc[c][p];
      }
      __syncthreads();
      // contract q -> node along each axis with the product table of (aa, b)
      const double* T0 = sm + ((aa == 0 && b == 0) ? Tab<N>::DD : ((aa == 0 || b == 0) ? Tab<N>::VD : Tab<N>::VV));
      const double* T1 = sm + ((aa == 1 && b == 1) ? Tab<N>::DD : ((aa == 1 || b == 1) ? Tab<N>::VD : Tab<N>::VV));
      const double* T2 = sm + ((aa == 2 && b == 2) ? Tab<N>::DD : ((aa == 2 || b == 2) ? Tab<N>::VD : Tab<N>::VV));
      double r[DIM];
      if (t.act) contract<DIM, N, DIM, 0>(A, B, T0, t);
      __syncthreads();
      if (DIM == 3) {
        if (t.act) contract<DIM, N, DIM, 1>(B, A, T1, t);
        __syncthreads();
        if (t.act) contract_reg<DIM, N, DIM, (DIM == 3 ? 2 : 1)>(A, r, T2, t);
      } else {
        if (t.act) contract_reg<DIM, N, DIM, 1>(B, r, T1, t);
      }
      __syncthreads();
      if (t.act) {
#pragma unroll
        for (int c = 0; c < DIM; ++c) acc[c] += r[c];
      }
    }
  if (t.act) {
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      long long d = t.node * DIM + c;
      if (!a.mask[d]) atomicAdd(a.y + d, acc[c]);
    }
  }
}

// ---------------------------------------------------------------------------
// residual internal force (operators.py:205-220): all rows accumulated; the
// traction and constraint finalisation is a vector kernel.
// ---------------------------------------------------------------------------
template <int DIM, int N>
__global__ void __launch_bounds__(Cfg<DIM, N>::NT) k_residual(const CellArgs a) {
  using K = Cfg<DIM, N>;
  constexpr int NQ = K::NQ;
  extern __shared__ double sm[];
  load_tables<DIM, N>(sm, a.tab, false);
  Team t = make_team<DIM, N>(a.lat, a.degree);
  double* A = sm + K::TAB + t.slot * K::SBUF;
  double* B = A + K::CPB * K::SBUF;
  double* Gs = sm + K::TAB + 2 * K::CPB * K::SBUF + t.slot * DIM * K::SBUF;
  const long long qi = t.e * NQ + t.lq;
  gather_nodal<DIM, N>(a.x, nullptr, t, A);
  __syncthreads();
  double gu[DIM][DIM];
  eval_gradients<DIM, N>(A, B, sm, t, gu);
  double G[DIM][DIM];
  double detv = 0.0;
  if (t.act) {
    double ji[DIM][DIM];
    load_jinv<DIM>(a, qi, ji);
    const double mu = __ldg(a.mu + t.e), lam = __ldg(a.lam + t.e);
    Kin<DIM> k;
    kinematics<DIM>(gu, ji, mu, lam, k, true);
    detv = k.J;
    const double jxw = __ldg(a.jxw + qi);
#pragma unroll
    for (int i = 0; i < DIM; ++i)
#pragma unroll
      for (int aa = 0; aa < DIM; ++aa) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < DIM; ++j) s = fma(k.tau[i][j], k.sinv[aa][j], s);
        G[i][aa] = s * jxw;
      }
  }
  warp_minmax_atomic(a.detmin, nullptr, detv, t.act);
  double yl[DIM];
  integrate_gradients<DIM, N>(A, B, Gs, sm, t, G, yl);
  if (t.act) {
#pragma unroll
    for (int c = 0; c < DIM; ++c) atomicAdd(a.y + t.node * DIM + c, yl[c]);
  }
}

// ---------------------------------------------------------------------------
// det F range (operators.py:192-196) and the first q-point attaining a value
// (argmin search for NonPositiveJacobian, operators.py:184-188).
//   mode 0: min/max into detmin/detmax;  mode 1: smallest flat (e*nq+q) index
//   whose det equals *target -> atomicMin into (unsigned long long*)y
// ---------------------------------------------------------------------------
template <int DIM, int N>
__global__ void __launch_bounds__(Cfg<DIM, N>::NT) k_jrange(const CellArgs a, int mode, double target,
                                                            unsigned long long* first) {
  using K = Cfg<DIM, N>;
  constexpr int NQ = K::NQ;
  extern __shared__ double sm[];
  load_tables<DIM, N>(sm, a.tab, false);
  Team t = make_team<DIM, N>(a.lat, a.degree);
  double* A = sm + K::TAB + t.slot * K::SBUF;
  double* B = A + K::CPB * K::SBUF;
  const long long qi = t.e * NQ + t.lq;
  gather_nodal<DIM, N>(a.x, nullptr, t, A);
  __syncthreads();
  double gu[DIM][DIM];
  eval_gradients<DIM, N>(A, B, sm, t, gu);
  double J = 0.0;
  if (t.act) {
    double ji[DIM][DIM];
    load_jinv<DIM>(a, qi, ji);
    double F[DIM * DIM];
#pragma unroll
    for (int i = 0; i < DIM; ++i)
#pragma unroll
      for (int Aa = 0; Aa < DIM; ++Aa) {
        double s = (i == Aa) ? 1.0 : 0.0;
#pragma unroll
        for (int q = 0; q < DIM; ++q) s = fma(gu[i][q], ji[q][Aa], s);
        F[i * DIM + Aa] = s;
      }
    J = hf_det<DIM>(F);
  }
  if (mode == 0) {
    warp_minmax_atomic(a.detmin, a.detmax, J, t.act);
  } else if (t.act && J == target) {
    atomicMin(first, (unsigned long long)qi);
  }
}

// ---------------------------------------------------------------------------
// total strain energy sum_q psi(F) JxW (operators.py:227-236, material.py:98-106):
// psi = mu/2 (tr C - d - 2 ln J) + lam (ln J)^2, block partials atomically
// added into *a.y; min det F into a.detmin (NonPositiveJacobian)
// ---------------------------------------------------------------------------
template <int DIM, int N>
__global__ void __launch_bounds__(Cfg<DIM, N>::NT) k_energy(const CellArgs a) {
  using K = Cfg<DIM, N>;
  constexpr int NQ = K::NQ;
  extern __shared__ double sm[];
  load_tables<DIM, N>(sm, a.tab, false);
  Team t = make_team<DIM, N>(a.lat, a.degree);
  double* A = sm + K::TAB + t.slot * K::SBUF;
  double* B = A + K::CPB * K::SBUF;
  const long long qi = t.e * NQ + t.lq;
  gather_nodal<DIM, N>(a.x, nullptr, t, A);
  __syncthreads();
  double gu[DIM][DIM];
  eval_gradients<DIM, N>(A, B, sm, t, gu);
  double J = 1.0, psi = 0.0;
  if (t.act) {
    double ji[DIM][DIM];
    load_jinv<DIM>(a, qi, ji);
    double F[DIM * DIM];
#pragma unroll
    for (int i = 0; i < DIM; ++i)
#pragma unroll
      for (int Aa = 0; Aa < DIM; ++Aa) {
        double s = (i == Aa) ? 1.0 : 0.0;
#pragma unroll
        for (int q = 0; q < DIM; ++q) s = fma(gu[i][q], ji[q][Aa], s);
        F[i * DIM + Aa] = s;
      }
    J = hf_det<DIM>(F);
    double trc = 0.0;
#pragma unroll
    for (int k = 0; k < DIM * DIM; ++k) trc = fma(F[k], F[k], trc);  // tr C = |F|^2
    const double lnj = log(J);
    const double mu = __ldg(a.mu + t.e), lam = __ldg(a.lam + t.e);
    psi = (0.5 * mu * (trc - DIM - 2.0 * lnj) + lam * lnj * lnj) * __ldg(a.jxw + qi);
  }
  warp_minmax_atomic(a.detmin, nullptr, J, t.act);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) psi += __shfl_xor_sync(0xffffffffu, psi, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(a.y, psi);
}

// ---------------------------------------------------------------------------
// geometry cache (mesh.py:290-307): one thread per (cell, q-point)
// ---------------------------------------------------------------------------
template <int DIM>
__global__ void k_geometry(const HfTables tab, const HfLattice lat, int nq1, const double* __restrict__ verts,
                           double* __restrict__ jinv, double* __restrict__ jxw, unsigned long long* detmin) {
  long long qi = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = qi < lat.n_qp;
  if (!valid) qi = lat.n_qp - 1;  // idle lanes recompute the last point (keeps the warp reduction full)
  int nq = nq1 * nq1 * (DIM == 3 ? nq1 : 1);
  long long e = qi / nq;
  int lq = (int)(qi - e * nq);
  int qx = lq % nq1, qy = (lq / nq1) % nq1, qz = DIM == 3 ? lq / (nq1 * nq1) : 0;
  long long r = e;
  int ex = (int)(r % lat.cells[0]);
  r /= lat.cells[0];
  int ey = (int)(r % lat.cells[1]);
  int ez = DIM == 3 ? (int)(r / lat.cells[1]) : 0;
  double xi[3] = {tab.qp[qx], tab.qp[qy], tab.qp[qz]};
  double Jm[DIM * DIM];
#pragma unroll
  for (int i = 0; i < DIM * DIM; ++i) Jm[i] = 0.0;
  const long long vx = lat.cells[0] + 1, vy = lat.cells[1] + 1;
#pragma unroll
  for (int c = 0; c < (1 << DIM); ++c) {
    int b0 = c & 1, b1 = (c >> 1) & 1, b2 = (c >> 2) & 1;
    long long vid = (ex + b0) + vx * ((ey + b1) + vy * (long long)(ez + b2));
    int bits[3] = {b0, b1, b2};
    double dn[DIM];
#pragma unroll
    for (int aa = 0; aa < DIM; ++aa) {
      double s = 1.0;
#pragma unroll
      for (int k = 0; k < DIM; ++k) {
        double fac = bits[k] ? xi[k] : 1.0 - xi[k];
        double dfac = bits[k] ? 1.0 : -1.0;
        s *= (aa == k) ? dfac : fac;
      }
      dn[aa] = s;
    }
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      double X = verts[vid * DIM + i];
#pragma unroll
      for (int aa = 0; aa < DIM; ++aa) Jm[i * DIM + aa] = fma(X, dn[aa], Jm[i * DIM + aa]);
    }
  }
  double det = hf_det<DIM>(Jm);
  warp_minmax_atomic(detmin, nullptr, det, true);
  if (!valid) return;
  double Ji[DIM * DIM];
  hf_inv<DIM>(Jm, det, Ji);
#pragma unroll
  for (int i = 0; i < DIM * DIM; ++i) jinv[i * lat.n_qp + qi] = Ji[i];
  double w = tab.qw[qx] * tab.qw[qy] * (DIM == 3 ? tab.qw[qz] : 1.0);
  jxw[qi] = det * w;
}

// Per (cell, last-axis line) constraint bits for the line kernels
// (hf_line.cuh): bit c*N + l is set when DoF c of node l of line t is
// constrained.  One coalesced 32-bit load per lane replaces N*DIM byte loads
// and the data-dependent branch on them.
static __global__ void k_line_masks(const HfLattice lat, int dim, int degree, const uint8_t* __restrict__ mask,
                                    uint32_t* __restrict__ bits) {
  const int n1 = degree + 1;
  const int L = dim == 3 ? n1 * n1 : n1;
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= lat.n_el * L) return;
  const long long e = id / L;
  const int t = (int)(id - e * L);
  long long r = e;
  const int ex = (int)(r % lat.cells[0]);
  r /= lat.cells[0];
  const int ey = (int)(r % lat.cells[1]);
  const int ez = dim == 3 ? (int)(r / lat.cells[1]) : 0;
  const int i = t % n1, j = dim == 3 ? t / n1 : 0;
  uint32_t b = 0;
  for (int l = 0; l < n1; ++l) {
    const long long node = dim == 3 ? (long long)(ex * degree + i) +
                                          (long long)lat.nodes[0] * ((long long)(ey * degree + j) +
                                                                     (long long)lat.nodes[1] * (long long)(ez * degree + l))
                                    : (long long)(ex * degree + i) + (long long)lat.nodes[0] * (long long)(ey * degree + l);
    for (int c = 0; c < dim; ++c)
      if (mask[node * dim + c]) b |= 1u << (c * n1 + l);
  }
  bits[id] = b;
}

}  // namespace hf
