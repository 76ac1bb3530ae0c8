// Shared device helpers for the hyperfree-B200 kernels (sm_100a, fp64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define HF_DEV __device__ __forceinline__

// Device-side bounds checks of the debug build (HF_DEBUG=1 python -m
// paper_1904_13131_b200.build -> libhf_debug.so): compute-sanitizer is not
// available on the GPU pool, so index arithmetic is checked by the kernels.
#ifdef HF_DEBUG
#include <cstdio>
#define HF_ASSERT(c)                                                                  \
  do {                                                                                \
    if (!(c)) {                                                                       \
      printf("HF_ASSERT %s:%d: %s\n", __FILE__, __LINE__, #c);                        \
      __trap();                                                                       \
    }                                                                                 \
  } while (0)
#else
#define HF_ASSERT(c) \
  do {               \
  } while (0)
#endif

// Largest 1D table the cell kernels are instantiated for (2D p<=8).
#define HF_MAXN 9

// 1D data of one level, passed by value as a kernel parameter (lives in the
// constant bank) and copied to shared memory at kernel start.
//   V[l*N+o]   = N_l(xi_o)           value of node-basis l at Gauss point o
//   D[l*N+o]   = N_l'(xi_o)
//   Dc[l*N+o]  = Dco(o,l)            collocation derivative at point o of the
//                                    Gauss-point Lagrange basis l  (Dco = D^T V^-T)
//   DcT[l*N+o] = Dco(l,o)
//   qp[o], qw[o]                     Gauss points / weights on [0,1]
struct HfTables {
  double V[HF_MAXN * HF_MAXN];
  double D[HF_MAXN * HF_MAXN];
  double Dc[HF_MAXN * HF_MAXN];
  double DcT[HF_MAXN * HF_MAXN];
  double qp[HF_MAXN];
  double qw[HF_MAXN];
};

// Per-level geometry/lattice description shared by every cell kernel.
struct HfLattice {
  int cells[3];   // cells per axis (x, y, z)
  int nodes[3];   // lattice nodes per axis (cells*p+1)
  long long n_el;
  long long n_nodes;
  long long n_qp;  // n_el * nq
  // n / cells[a] for 0 <= n < 2^31 as (umulhi(n, dm[a]) + n) >> ds[a]
  // (division by an invariant through a multiply; hf_fastdiv_init)
  unsigned dm[2], ds[2];
};

inline void hf_fastdiv_init(unsigned d, unsigned& m, unsigned& s) {
  unsigned l = 0;
  while ((1ull << l) < d) ++l;  // l = ceil(log2 d)
  m = (unsigned)((((1ull << 32) * ((1ull << l) - d)) / d) + 1);
  s = l;
}
HF_DEV unsigned hf_fastdiv(unsigned n, unsigned m, unsigned s) { return (__umulhi(n, m) + n) >> s; }

// ---- ordered-double atomics (min/max of doubles through uint64 atomics) ----
HF_DEV unsigned long long hf_ord(double v) {
  unsigned long long b = __double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
static inline __host__ __device__ double hf_unord(unsigned long long o) {
  unsigned long long b = (o & 0x8000000000000000ull) ? (o & 0x7fffffffffffffffull) : ~o;
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  union { unsigned long long u; double d; } cv;
  cv.u = b;
  return cv.d;
#endif
}
HF_DEV void hf_atomic_min_d(unsigned long long* a, double v) { atomicMin(a, hf_ord(v)); }
HF_DEV void hf_atomic_max_d(unsigned long long* a, double v) { atomicMax(a, hf_ord(v)); }

// 3x3 / 2x2 helpers on row-major arrays
template <int D>
HF_DEV double hf_det(const double* a);
template <>
HF_DEV double hf_det<2>(const double* a) { return a[0] * a[3] - a[1] * a[2]; }
template <>
HF_DEV double hf_det<3>(const double* a) {
  return a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
         a[2] * (a[3] * a[7] - a[4] * a[6]);
}
// inverse via adjugate / det
template <int D>
HF_DEV void hf_inv(const double* a, double det, double* o);
template <>
HF_DEV void hf_inv<2>(const double* a, double det, double* o) {
  double r = 1.0 / det;
  o[0] = a[3] * r; o[1] = -a[1] * r; o[2] = -a[2] * r; o[3] = a[0] * r;
}
template <>
HF_DEV void hf_inv<3>(const double* a, double det, double* o) {
  double r = 1.0 / det;
  o[0] = (a[4] * a[8] - a[5] * a[7]) * r;
  o[1] = (a[2] * a[7] - a[1] * a[8]) * r;
  o[2] = (a[1] * a[5] - a[2] * a[4]) * r;
  o[3] = (a[5] * a[6] - a[3] * a[8]) * r;
  o[4] = (a[0] * a[8] - a[2] * a[6]) * r;
  o[5] = (a[2] * a[3] - a[0] * a[5]) * r;
  o[6] = (a[3] * a[7] - a[4] * a[6]) * r;
  o[7] = (a[1] * a[6] - a[0] * a[7]) * r;
  o[8] = (a[0] * a[4] - a[1] * a[3]) * r;
}

// Symmetric packing order of the reference (material.py:161-164)
//   2D: (00, 11, 01)       3D: (00, 11, 22, 12, 02, 01)
template <int D> struct HfSym;
template <> struct HfSym<2> {
  static constexpr int NV = 3;
  HF_DEV static int a(int k) { return k == 2 ? 0 : k; }
  HF_DEV static int b(int k) { return k == 2 ? 1 : k; }
};
template <> struct HfSym<3> {
  static constexpr int NV = 6;
  HF_DEV static int a(int k) { return k < 3 ? k : (k == 3 ? 1 : 0); }
  HF_DEV static int b(int k) { return k < 3 ? k : (k == 5 ? 1 : 2); }
};
// index of the symmetric slot holding (i, j)
//   3D: (1,2)->3, (0,2)->4, (0,1)->5
template <int D>
HF_DEV constexpr int hf_slot(int i, int j) {
  return (i == j) ? i : (D == 2 ? 2 : (i + j == 3 ? 3 : (i + j == 2 ? 4 : 5)));
}

// packed upper-triangle (row-major) index of Voigt entry (r, c), r <= c
template <int NV>
HF_DEV constexpr int hf_triu(int r, int c) {
  return r * NV - (r * (r - 1)) / 2 + (c - r);
}

// ---- warp-tile geometry of the line kernels and the tiled q-point cache ----
// (hf_line.cuh).  A warp tile holds CPW whole cells; its cache block is
// [field][iq][lane] with lane = cell_in_tile * L + line (x-lines).
template <int DIM, int N>
struct LineCfg {
  static constexpr int NQ = (DIM == 2) ? N * N : N * N * N;
  static constexpr int L = NQ / N;        // lines per cell
  static constexpr int CPW = 32 / L;      // cells per warp tile
  static constexpr int LANES = CPW * L;   // active lanes of a warp
  static constexpr int TS = CPW * NQ;     // q-points per tile
};

// Tiled q-point cache: [tile][iq][field][lane], one contiguous "chunk" of
// nf*LANES doubles (rounded to 16 bytes) per (tile, iq) -- the unit a TMA bulk
// copy moves into shared memory (hf_line.cuh).
template <int DIM, int N>
struct TileLayout {
  using K = LineCfg<DIM, N>;
  // elements per chunk for ESZ-byte elements, rounded to 16 bytes
  template <int ESZ = 8>
  HF_DEV static constexpr long long chunk_e(int nf) {
    return ((long long)nf * K::LANES + (16 / ESZ - 1)) & ~(long long)(16 / ESZ - 1);
  }
  HF_DEV static constexpr long long chunk(int nf) { return chunk_e<8>(nf); }
  HF_DEV static constexpr long long stride(int nf) { return N * chunk(nf); }
  // flat index of field f of (cell e, local q-point lq, x fastest)
  HF_DEV static long long index(long long e, int lq, int f, int nf) {
    const long long tile = e / K::CPW;
    const int m = (int)(e - tile * K::CPW);
    const int iq = lq % N, line = lq / N;
    return tile * stride(nf) + iq * chunk(nf) + (long long)f * K::LANES + m * K::L + line;
  }
  // same for ESZ-byte elements (the fp32 storage of mixed-precision levels)
  template <int ESZ>
  HF_DEV static long long index_e(long long e, int lq, int f, int nf) {
    const long long tile = e / K::CPW;
    const int m = (int)(e - tile * K::CPW);
    const int iq = lq % N, line = lq / N;
    return tile * (N * chunk_e<ESZ>(nf)) + iq * chunk_e<ESZ>(nf) + (long long)f * K::LANES + m * K::L + line;
  }
};
inline long long tile_cache_doubles(int dim, int n1, int nf, long long n_el, int esz = 8) {
  int nq = dim == 2 ? n1 * n1 : n1 * n1 * n1;
  int lanes = (32 / (nq / n1)) * (nq / n1);
  int cpw = 32 / (nq / n1);
  long long tiles = (n_el + cpw - 1) / cpw;
  const long long r = 16 / esz - 1;
  long long ch = ((long long)nf * lanes + r) & ~r;
  return tiles * n1 * ch;  // elements of esz bytes
}
