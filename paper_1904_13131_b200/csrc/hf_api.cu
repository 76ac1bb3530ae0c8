// C-ABI of the hyperfree-B200 library (libhf.so).  See include/hf.h for the
// contract and the reference interface each entry point replaces.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/hf.h"
#include "hf_dispatch.h"
#include "hf_vec.cuh"
#include "hf_coarse.cuh"

using namespace hf;

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define HF_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess) return fail(HF_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// Device block pool.  Every device allocation of this library goes through
// dmalloc/dfree.  A Newton iteration rebuilds the tangent and the whole GMG
// hierarchy (solver.py:174, multigrid.py:358-369) with the same sizes as the
// previous one; returning blocks to cudaFree and asking cudaMalloc again costs
// tens of ms per iteration at 64^3 (page unmapping/mapping of GB-sized caches).
// Freed blocks are kept per device and handed out again for requests of the
// same size (within +12.5 %).  dfree synchronises the device before pooling a
// block, the same ordering guarantee cudaFree gives, so no queued kernel still
// reads a block when it is reused.  Pooled bytes are capped (HF_POOL_MAX_MB,
// default 32768); hf_pool_release() returns every pooled block to the driver,
// and an allocation that fails releases the pool and retries once.
struct DevPool {
  std::mutex m;
  std::multimap<std::pair<int, size_t>, void*> free_blocks;
  std::unordered_map<void*, std::pair<int, size_t>> owned;
  size_t pooled = 0, live = 0, cap = 0;
  DevPool() {
    const char* e = std::getenv("HF_POOL_MAX_MB");
    cap = (size_t)(e ? std::atoll(e) : 32768) << 20;
  }
  void release_locked() {
    for (auto& kv : free_blocks) {
      cudaFree(kv.second);
      owned.erase(kv.second);
    }
    free_blocks.clear();
    pooled = 0;
  }
};

DevPool& dev_pool() {
  static DevPool* p = new DevPool();  // never destroyed: outlives static teardown order
  return *p;
}

cudaError_t dmalloc(void** ptr, size_t bytes) {
  DevPool& P = dev_pool();
  int dev = 0;
  cudaGetDevice(&dev);
  if (bytes == 0) bytes = 1;
  std::lock_guard<std::mutex> g(P.m);
  auto it = P.free_blocks.lower_bound({dev, bytes});
  if (it != P.free_blocks.end() && it->first.first == dev && it->first.second <= bytes + bytes / 8) {
    *ptr = it->second;
    P.pooled -= it->first.second;
    P.live += it->first.second;
    P.free_blocks.erase(it);
    return cudaSuccess;
  }
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e == cudaErrorMemoryAllocation && !P.free_blocks.empty()) {
    cudaGetLastError();
    P.release_locked();
    e = cudaMalloc(ptr, bytes);
  }
  if (e == cudaSuccess) {
    P.owned[*ptr] = {dev, bytes};
    P.live += bytes;
  }
  return e;
}

cudaError_t dfree(void* ptr) {
  if (!ptr) return cudaSuccess;
  DevPool& P = dev_pool();
  std::lock_guard<std::mutex> g(P.m);
  auto it = P.owned.find(ptr);
  if (it == P.owned.end()) return cudaFree(ptr);
  const auto key = it->second;
  P.live -= key.second;
  if (P.pooled + key.second > P.cap) {
    P.owned.erase(it);
    return cudaFree(ptr);
  }
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != key.first) cudaSetDevice(key.first);
  cudaError_t e = cudaDeviceSynchronize();
  if (cur != key.first) cudaSetDevice(cur);
  P.free_blocks.emplace(key, ptr);
  P.pooled += key.second;
  return e;
}

inline unsigned vec_blocks(long long n) {
  long long b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)b;
}

// the fill: four elements per thread per iteration, one resident wave (148 SMs x 8 blocks of 256)
inline unsigned fill_blocks(long long n) {
  static const int per_sm = [] {  // HF_FILL_BLOCKS: A/B knob (blocks of 256 threads per SM)
    const char* e = std::getenv("HF_FILL_BLOCKS");
    const int v = e ? std::atoi(e) : 8;
    return v > 0 ? v : 8;
  }();
  long long b = (n + 1023) / 1024;
  if (b < 1) b = 1;
  if (b > 148ll * per_sm) b = 148ll * per_sm;
  return (unsigned)b;
}

// Gauss-Jordan inverse of a small dense matrix (row-major), returns false if singular
bool invert(std::vector<double> a, int n, std::vector<double>& inv) {
  inv.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(a[r * n + c]) > std::fabs(a[piv * n + c])) piv = r;
    if (a[piv * n + c] == 0.0) return false;
    for (int k = 0; k < n; ++k) {
      std::swap(a[c * n + k], a[piv * n + k]);
      std::swap(inv[c * n + k], inv[piv * n + k]);
    }
    double d = a[c * n + c];
    for (int k = 0; k < n; ++k) {
      a[c * n + k] /= d;
      inv[c * n + k] /= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      double f = a[r * n + c];
      if (f == 0.0) continue;
      for (int k = 0; k < n; ++k) {
        a[r * n + k] -= f * a[c * n + k];
        inv[r * n + k] -= f * inv[c * n + k];
      }
    }
  }
  return true;
}
}  // namespace

struct hf_space {
  int dim, degree, n1;
  HfTables tab;
  HfLattice lat;
  long long n_dofs;
  double* d_jinv = nullptr;
  double* d_jxw = nullptr;
  double* d_mu = nullptr;
  double* d_lam = nullptr;
  uint8_t* d_mask = nullptr;
  uint32_t* d_lmask = nullptr;  // per (cell, last-axis line): constraint bits (k_line_masks)
  unsigned long long* d_u64 = nullptr;  // [0] detmin [1] detmax [2] first-index
};

// Host-to-host apply (hf_tangent_apply_host): device staging vectors, copy
// streams, and the pipelines already captured as CUDA graphs, keyed by the
// host buffers and the slab count.
struct HostPipe {
  static constexpr int NG = 4;
  double* xd = nullptr;
  double* yd = nullptr;
  cudaStream_t cap = nullptr, s_in = nullptr, s_out = nullptr;
  std::vector<cudaEvent_t> ev;
  struct Entry {
    const void* x;
    void* y;
    int chunks;
    cudaGraphExec_t exec;  // null: enqueue directly (variant 2 overlap / 3 serial)
    unsigned long long used;
    int variant;
    unsigned uses;  // calls of this entry
    int recal;      // the one recalibration after RECAL_AT calls is done
  } g[NG] = {};
  // A first calibration can fall into a window in which the host link runs
  // ~1.7x slow (tens of ms at a time, early in a process on some boxes), and
  // then picks a variant that is not the fastest in steady state.  With
  // HF_E2E_RECAL=1 each entry is calibrated once more after this many calls
  // (opt-in: the recalibration synchronises and stalls the caller's loop).
  static constexpr unsigned RECAL_AT = 256;
  cudaEvent_t done = nullptr;  // recorded after every enqueued step (any caller stream)
  int ng = 0;
  unsigned long long clock = 0;
  int last_order = -1;           // variant of the last calibration: 0 graph overlap, 1 graph serial,
                                 // 2 direct overlap, 3 direct serial
  float last_us[4] = {0, 0, 0, 0};  // their calibration times
};

struct hf_tangent {
  hf_space* sp;
  int strategy;
  int nf;
  long long cache_len = 0;  // elements
  int fp32 = 0;  // cache and x/y stored as float (mixed-precision multigrid levels)
  double* d_cache = nullptr;
  double* d_ubar = nullptr;
  HostPipe* host = nullptr;
  int alternate = 0;  // whole-range applies alternate their sweep direction (hf_tangent_set_alternate)
  int flip = 0;
};

struct hf_transfer {
  const hf_space* coarse;
  const hf_space* fine;
  // per axis CSR of prolongation (rows: fine) and restriction (rows: coarse)
  int* d_pp[3] = {nullptr, nullptr, nullptr};
  int* d_pc[3] = {nullptr, nullptr, nullptr};
  double* d_pw[3] = {nullptr, nullptr, nullptr};
  int* d_rp[3] = {nullptr, nullptr, nullptr};
  int* d_rc[3] = {nullptr, nullptr, nullptr};
  double* d_rw[3] = {nullptr, nullptr, nullptr};
  double* d_tmp[2] = {nullptr, nullptr};
  long long tmp_len = 0;
};

struct hf_coarse {
  int n = 0;
  long long nnz = 0;
  int grid = 1;
  size_t smem = 0;
  unsigned char* blob = nullptr;
  size_t blob_bytes = 0;
  long long* boff = nullptr;
  double* xb = nullptr;
  double* partials = nullptr;
  // value refresh from element matrices (hf_coarse_create_space / hf_coarse_update)
  const hf_space* sp = nullptr;
  int nupd = 0;                 // CSR slots with element contributions
  int* cptr = nullptr;          // [nupd + 1] contributions of slot u
  int* cidx = nullptr;          // element-matrix entry indices, ascending per slot
  long long* uoff = nullptr;    // blob byte offset of slot u's value
  double* elem = nullptr;       // element matrices scratch
};

struct hf_ws {
  double* d_partials = nullptr;
  unsigned* d_counter = nullptr;
};

static cudaError_t update_cell_flags(hf_space* sp, cudaStream_t s) {
  if (sp->lat.n_el <= 0) return cudaSuccess;
  const long long n = sp->lat.n_el * (sp->dim == 3 ? sp->n1 * sp->n1 : sp->n1);
  k_line_masks<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sp->lat, sp->dim, sp->degree, sp->d_mask, sp->d_lmask);
  return cudaGetLastError();
}

// mode: 0 plain, 1 zero constrained outputs, 2 add into out with constrained dropped.
// Input/output element types may differ (the boundary of fp32 multigrid
// levels); intermediate passes and all arithmetic are fp64.
template <typename TI, typename TO>
static int transfer_run(hf_transfer* t, bool prolong, const TI* in, TO* out, int mode, cudaStream_t s) {
  const hf_space* src = prolong ? t->coarse : t->fine;
  const hf_space* dst = prolong ? t->fine : t->coarse;
  int dim = src->dim, C = dim;
  int n[3] = {src->lat.nodes[0], src->lat.nodes[1], dim == 3 ? src->lat.nodes[2] : 1};
  const double* cur = nullptr;
  for (int a = 0; a < dim; ++a) {
    bool last = (a == dim - 1);
    int nout = dst->lat.nodes[a];
    long long total;
    if (a == 0) total = (long long)C * nout * n[1] * n[2];
    else if (a == 1) total = (long long)C * n[0] * nout * n[2];
    else total = (long long)C * n[0] * n[1] * nout;
    const int* rp = prolong ? t->d_pp[a] : t->d_rp[a];
    const int* cl = prolong ? t->d_pc[a] : t->d_rc[a];
    const double* w = prolong ? t->d_pw[a] : t->d_rw[a];
    double* tmp = t->d_tmp[a & 1];
    const unsigned blocks = vec_blocks(total);
    if (a == 0 && last) {
      k_axis<TI, TO><<<blocks, 256, 0, s>>>(in, out, n[0], n[1], n[2], C, a, nout, rp, cl, w, dst->d_mask, mode);
    } else if (a == 0) {
      k_axis<TI, double><<<blocks, 256, 0, s>>>(in, tmp, n[0], n[1], n[2], C, a, nout, rp, cl, w, dst->d_mask, 0);
    } else if (last) {
      k_axis<double, TO><<<blocks, 256, 0, s>>>(cur, out, n[0], n[1], n[2], C, a, nout, rp, cl, w, dst->d_mask, mode);
    } else {
      k_axis<double, double><<<blocks, 256, 0, s>>>(cur, tmp, n[0], n[1], n[2], C, a, nout, rp, cl, w, dst->d_mask, 0);
    }
    HF_CUDA(cudaGetLastError());
    n[a] = nout;
    cur = tmp;
  }
  return HF_OK;
}

static int transfer_dispatch(hf_transfer* t, bool prolong, const void* in, int in_bits, void* out, int out_bits,
                             int mode, cudaStream_t s) {
  if ((in_bits != 32 && in_bits != 64) || (out_bits != 32 && out_bits != 64)) return fail(HF_ERR_ARG, "bits: 32|64");
  if (in_bits == 64 && out_bits == 64)
    return transfer_run(t, prolong, (const double*)in, (double*)out, mode, s);
  if (in_bits == 64) return transfer_run(t, prolong, (const double*)in, (float*)out, mode, s);
  if (out_bits == 64) return transfer_run(t, prolong, (const float*)in, (double*)out, mode, s);
  return transfer_run(t, prolong, (const float*)in, (float*)out, mode, s);
}

// hf_cheb_step / hf_cheb_step_fill / hf_cheb_step_f32 launched as the
// programmatic dependent of the cell kernel that wrote ax (the apply of the
// same smoothing step, immediately before on the stream)
template <typename T>
static cudaError_t launch_cheb_after_apply(long long n, T* x, T* d, const T* b, const T* ax, const T* inv_d, int first,
                                           double theta, double cd, double cz, const unsigned char* fill_mask,
                                           T* y_next, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(vec_blocks(n));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int* skip = nullptr;
  return cudaLaunchKernelEx(&cfg, k_cheb<T>, n, x, d, b, ax, inv_d, first, theta, cd, cz, 0, skip, fill_mask, y_next,
                            1);
}

extern "C" {

HF_API const char* hf_last_error(void) { return g_err.c_str(); }
HF_API int hf_abi_version(void) { return HF_ABI_VERSION; }

HF_API int hf_pool_release(void) {
  DevPool& P = dev_pool();
  std::lock_guard<std::mutex> g(P.m);
  P.release_locked();
  return HF_OK;
}

HF_API int hf_pool_info(long long* pooled_bytes, long long* live_bytes) {
  DevPool& P = dev_pool();
  std::lock_guard<std::mutex> g(P.m);
  if (pooled_bytes) *pooled_bytes = (long long)P.pooled;
  if (live_bytes) *live_bytes = (long long)P.live;
  return HF_OK;
}

HF_API int hf_max_degree(int dim) { return dim == 2 ? 8 : (dim == 3 ? 4 : 0); }

// ---------------------------------------------------------------------------
HF_API int hf_space_create(int dim, int degree, int nq1, const int* cells, const double* values_1d,
                           const double* derivs_1d, const double* qpoints_1d, const double* qweights_1d,
                           const double* vertices, const double* mu_el, const double* lam_el,
                           const unsigned char* mask, void* stream, hf_space** out) {
  if (!out || !cells || !values_1d || !derivs_1d || !qpoints_1d || !qweights_1d || !vertices || !mu_el || !lam_el ||
      !mask)
    return fail(HF_ERR_ARG, "hf_space_create: null argument");
  if (dim != 2 && dim != 3) return fail(HF_ERR_ARG, "dim must be 2 or 3");
  if (degree < 1 || degree > hf_max_degree(dim))
    return fail(HF_ERR_UNSUPPORTED, "degree " + std::to_string(degree) + " not instantiated for dim " + std::to_string(dim));
  if (nq1 != degree + 1)
    return fail(HF_ERR_UNSUPPORTED, "the B200 kernels are instantiated for n_qpoints = degree + 1 only");
  hf_space* sp = new hf_space();
  sp->dim = dim;
  sp->degree = degree;
  sp->n1 = degree + 1;
  const int N = sp->n1;
  std::memset(&sp->tab, 0, sizeof(HfTables));
  std::vector<double> V(N * N), Vinv;
  for (int i = 0; i < N * N; ++i) {
    sp->tab.V[i] = values_1d[i];
    sp->tab.D[i] = derivs_1d[i];
    V[i] = values_1d[i];
  }
  for (int i = 0; i < N; ++i) {
    sp->tab.qp[i] = qpoints_1d[i];
    sp->tab.qw[i] = qweights_1d[i];
  }
  if (!invert(V, N, Vinv)) {
    delete sp;
    return fail(HF_ERR_ARG, "singular 1D value table");
  }
  // Dco(o, l) = sum_i D[i][o] Vinv[l][i]
  for (int o = 0; o < N; ++o)
    for (int l = 0; l < N; ++l) {
      double s = 0.0;
      for (int i = 0; i < N; ++i) s += derivs_1d[i * N + o] * Vinv[l * N + i];
      sp->tab.Dc[l * N + o] = s;   // Dc[l][o]  = Dco(o, l)
      sp->tab.DcT[o * N + l] = s;  // DcT[o][l] = Dco(o, l)
    }
  sp->lat.cells[2] = 1;
  sp->lat.nodes[2] = 1;
  long long nel = 1, nn = 1;
  for (int a = 0; a < dim; ++a) {
    if (cells[a] < 1) {
      delete sp;
      return fail(HF_ERR_ARG, "cells per axis must be >= 1");
    }
    sp->lat.cells[a] = cells[a];
    sp->lat.nodes[a] = cells[a] * degree + 1;
    nel *= cells[a];
    nn *= sp->lat.nodes[a];
  }
  long long nq = 1;
  for (int a = 0; a < dim; ++a) nq *= N;
  sp->lat.n_el = nel;
  sp->lat.n_nodes = nn;
  sp->lat.n_qp = nel * nq;
  sp->n_dofs = nn * dim;
  if (sp->n_dofs >= (1ll << 31)) {  // the cell kernels index DoFs in 32 bits
    delete sp;
    return fail(HF_ERR_UNSUPPORTED, "n_dofs must be < 2^31 on one device (partition the mesh over more GPUs)");
  }
  for (int a = 0; a < 2; ++a) hf_fastdiv_init((unsigned)sp->lat.cells[a], sp->lat.dm[a], sp->lat.ds[a]);
  cudaStream_t s = S(stream);
  long long nverts = 1;
  for (int a = 0; a < dim; ++a) nverts *= (cells[a] + 1);
  double* d_verts = nullptr;
#define ALLOC(ptr, bytes) HF_CUDA(dmalloc((void**)&(ptr), (bytes)))
  ALLOC(sp->d_jinv, sizeof(double) * dim * dim * sp->lat.n_qp);
  ALLOC(sp->d_jxw, sizeof(double) * sp->lat.n_qp);
  ALLOC(sp->d_mu, sizeof(double) * nel);
  ALLOC(sp->d_lam, sizeof(double) * nel);
  ALLOC(sp->d_mask, sp->n_dofs);
  ALLOC(sp->d_lmask, sizeof(uint32_t) * (nel > 0 ? nel : 1) * (dim == 3 ? N * N : N));
  ALLOC(sp->d_u64, sizeof(unsigned long long) * 4);
  ALLOC(d_verts, sizeof(double) * nverts * dim);
  HF_CUDA(cudaMemcpyAsync(d_verts, vertices, sizeof(double) * nverts * dim, cudaMemcpyHostToDevice, s));
  HF_CUDA(cudaMemcpyAsync(sp->d_mu, mu_el, sizeof(double) * nel, cudaMemcpyHostToDevice, s));
  HF_CUDA(cudaMemcpyAsync(sp->d_lam, lam_el, sizeof(double) * nel, cudaMemcpyHostToDevice, s));
  HF_CUDA(cudaMemcpyAsync(sp->d_mask, mask, sp->n_dofs, cudaMemcpyHostToDevice, s));
  HF_CUDA(update_cell_flags(sp, s));
  unsigned long long init = ~0ull;
  HF_CUDA(cudaMemcpyAsync(sp->d_u64, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  HF_CUDA(launch_geometry(dim, sp->tab, sp->lat, N, d_verts, sp->d_jinv, sp->d_jxw, sp->d_u64, s));
  unsigned long long o = 0;
  HF_CUDA(cudaMemcpyAsync(&o, sp->d_u64, sizeof(o), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  dfree(d_verts);
  if (nel > 0 && !(hf_unord(o) > 0.0)) {
    hf_space_destroy(sp);
    char buf[128];
    std::snprintf(buf, sizeof(buf), "non-positive mapping Jacobian (det=%.3e)", hf_unord(o));
    return fail(HF_ERR_GEOMETRY, buf);
  }
  *out = sp;
  return HF_OK;
}

HF_API int hf_space_set_mask(hf_space* sp, const unsigned char* mask, void* stream) {
  if (!sp || !mask) return fail(HF_ERR_ARG, "null argument");
  HF_CUDA(cudaMemcpyAsync(sp->d_mask, mask, sp->n_dofs, cudaMemcpyHostToDevice, S(stream)));
  HF_CUDA(update_cell_flags(sp, S(stream)));
  HF_CUDA(cudaStreamSynchronize(S(stream)));
  return HF_OK;
}

HF_API int hf_space_info(const hf_space* sp, long long* n_dofs, long long* n_el, long long* n_qp) {
  if (!sp) return fail(HF_ERR_ARG, "null space");
  if (n_dofs) *n_dofs = sp->n_dofs;
  if (n_el) *n_el = sp->lat.n_el;
  if (n_qp) *n_qp = sp->lat.n_qp;
  return HF_OK;
}

HF_API int hf_space_pointers(const hf_space* sp, const double** jinv, const double** jxw,
                             const unsigned char** mask) {
  if (!sp) return fail(HF_ERR_ARG, "null space");
  if (jinv) *jinv = sp->d_jinv;
  if (jxw) *jxw = sp->d_jxw;
  if (mask) *mask = sp->d_mask;
  return HF_OK;
}

HF_API int hf_space_geometry_copy(const hf_space* sp, double* jinv_dev, double* jxw_dev, void* stream) {
  if (!sp || !jinv_dev || !jxw_dev) return fail(HF_ERR_ARG, "null argument");
  cudaStream_t s = S(stream);
  HF_CUDA(cudaMemcpyAsync(jinv_dev, sp->d_jinv, sizeof(double) * sp->dim * sp->dim * sp->lat.n_qp,
                          cudaMemcpyDeviceToDevice, s));
  HF_CUDA(cudaMemcpyAsync(jxw_dev, sp->d_jxw, sizeof(double) * sp->lat.n_qp, cudaMemcpyDeviceToDevice, s));
  return HF_OK;
}

HF_API int hf_space_destroy(hf_space* sp) {
  if (!sp) return HF_OK;
  dfree(sp->d_jinv);
  dfree(sp->d_jxw);
  dfree(sp->d_mu);
  dfree(sp->d_lam);
  dfree(sp->d_mask);
  dfree(sp->d_lmask);
  dfree(sp->d_u64);
  delete sp;
  return HF_OK;
}

// ---------------------------------------------------------------------------
static CellArgs base_args(const hf_space* sp) {
  CellArgs a;
  std::memset(&a, 0, sizeof(a));
  a.tile1 = -1;
  a.tab = sp->tab;
  a.lat = sp->lat;
  a.degree = sp->degree;
  a.jinv = sp->d_jinv;
  a.jxw = sp->d_jxw;
  a.mu = sp->d_mu;
  a.lam = sp->d_lam;
  a.mask = sp->d_mask;
  a.lmask = sp->d_lmask;
  return a;
}

static cudaError_t cell(const hf_space* sp, int op, int var, const CellArgs& a, cudaStream_t s, int mode = 0,
                        double target = 0.0, unsigned long long* first = nullptr) {
  if (sp->dim == 2) return launch_cell_2d(op, sp->n1, var, a, mode, target, first, s);
  return launch_cell_3d(op, sp->n1, var, a, mode, target, first, s);
}

static int nfields(int dim, int strategy) {
  int nv = dim * (dim + 1) / 2, nm = nv * (nv + 1) / 2;
  if (strategy == HF_TENSOR4) return nv + nm + dim * dim;  // JxW folded into tau, M (CacheFields)
  if (strategy == HF_TENSOR2) return 2 + nv + dim * dim;
  return 2 + dim * dim;  // c1 + J^-1 + JxW (tile layout, hf_line.cuh)
}

// locate the first q-point (flat e*nq+q) attaining min det F of state u
static int locate_min_det(hf_space* sp, const double* u, cudaStream_t s, hf_error_info* err) {
  CellArgs a = base_args(sp);
  a.x = u;
  a.detmin = sp->d_u64;
  a.detmax = sp->d_u64 + 1;
  unsigned long long init[3] = {~0ull, 0ull, ~0ull};
  HF_CUDA(cudaMemcpyAsync(sp->d_u64, init, sizeof(init), cudaMemcpyHostToDevice, s));
  HF_CUDA(cell(sp, OP_JRANGE, 0, a, s, 0));
  unsigned long long mm[2];
  HF_CUDA(cudaMemcpyAsync(mm, sp->d_u64, sizeof(mm), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  double jmin = hf_unord(mm[0]);
  HF_CUDA(cell(sp, OP_JRANGE, 0, a, s, 1, jmin, sp->d_u64 + 2));
  unsigned long long idx;
  HF_CUDA(cudaMemcpyAsync(&idx, sp->d_u64 + 2, sizeof(idx), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  long long nq = sp->lat.n_qp / (sp->lat.n_el > 0 ? sp->lat.n_el : 1);
  if (err) {
    err->code = HF_ERR_JACOBIAN;
    err->det = jmin;
    err->element = (long long)(idx / (unsigned long long)nq);
    err->qpoint = (int)(idx % (unsigned long long)nq);
  }
  char buf[160];
  std::snprintf(buf, sizeof(buf), "det F = %.3e <= 0 in element %lld (quadrature point %d)", jmin,
                (long long)(idx / (unsigned long long)nq), (int)(idx % (unsigned long long)nq));
  return fail(HF_ERR_JACOBIAN, buf);
}

HF_API int hf_jacobian_range(hf_space* sp, const double* u_dev, void* stream, double* jmin, double* jmax,
                             long long* argmin_element, int* argmin_qpoint) {
  if (!sp || !u_dev) return fail(HF_ERR_ARG, "null argument");
  cudaStream_t s = S(stream);
  hf_error_info e;
  int rc = locate_min_det(sp, u_dev, s, &e);
  if (rc != HF_ERR_JACOBIAN) return rc;
  unsigned long long mm[2];
  HF_CUDA(cudaMemcpyAsync(mm, sp->d_u64, sizeof(mm), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  if (jmin) *jmin = hf_unord(mm[0]);
  if (jmax) *jmax = hf_unord(mm[1]);
  if (argmin_element) *argmin_element = e.element;
  if (argmin_qpoint) *argmin_qpoint = e.qpoint;
  g_err.clear();
  return HF_OK;
}

HF_API int hf_tangent_create_ex(hf_space* sp, int strategy, int storage_bits, const double* ubar_dev, void* stream,
                                hf_tangent** out, hf_error_info* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!sp || !ubar_dev || !out) return fail(HF_ERR_ARG, "null argument");
  if (strategy < HF_SCALAR || strategy > HF_TENSOR4) return fail(HF_ERR_ARG, "unknown strategy");
  if (storage_bits != 32 && storage_bits != 64) return fail(HF_ERR_ARG, "storage_bits must be 32 or 64");
  cudaStream_t s = S(stream);
  hf_tangent* op = new hf_tangent();
  op->sp = sp;
  op->strategy = strategy;
  op->nf = nfields(sp->dim, strategy);
  op->fp32 = storage_bits == 32;
  const int esz = op->fp32 ? 4 : 8;
  const long long ncache = tile_cache_doubles(sp->dim, sp->n1, op->nf, sp->lat.n_el, esz);
  op->cache_len = ncache;
  HF_CUDA(dmalloc((void**)&op->d_cache, (size_t)esz * (ncache > 0 ? ncache : 1)));
  if (strategy == HF_SCALAR) {
    HF_CUDA(dmalloc((void**)&op->d_ubar, sizeof(double) * sp->n_dofs));
    HF_CUDA(cudaMemcpyAsync(op->d_ubar, ubar_dev, sizeof(double) * sp->n_dofs, cudaMemcpyDeviceToDevice, s));
  }
  unsigned long long init = ~0ull;
  HF_CUDA(cudaMemcpyAsync(sp->d_u64, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  CellArgs a = base_args(sp);
  a.x = ubar_dev;
  a.cache_out = op->d_cache;
  a.detmin = sp->d_u64;
  a.fp32 = op->fp32;
  a.cache_len = op->cache_len;
  HF_CUDA(cell(sp, OP_BUILD, strategy, a, s));
  unsigned long long o;
  HF_CUDA(cudaMemcpyAsync(&o, sp->d_u64, sizeof(o), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  if (sp->lat.n_el > 0 && !(hf_unord(o) > 0.0)) {
    hf_tangent_destroy(op);
    return locate_min_det(sp, ubar_dev, s, err);
  }
  *out = op;
  return HF_OK;
}

HF_API int hf_tangent_create(hf_space* sp, int strategy, const double* ubar_dev, void* stream, hf_tangent** out,
                             hf_error_info* err) {
  return hf_tangent_create_ex(sp, strategy, 64, ubar_dev, stream, out, err);
}

// Host-pointer form for FFI callers that hold numpy arrays (the reference-side
// ctypes binding): u_bar is staged through a pooled device
// buffer; synchronous on the default stream.
HF_API int hf_tangent_create_host(hf_space* sp, int strategy, const double* ubar_host, hf_tangent** out,
                                  hf_error_info* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!sp || !ubar_host || !out) return fail(HF_ERR_ARG, "null argument");
  double* d = nullptr;
  HF_CUDA(dmalloc((void**)&d, sizeof(double) * (sp->n_dofs > 0 ? sp->n_dofs : 1)));
  int rc = HF_OK;
  if (cudaMemcpy(d, ubar_host, sizeof(double) * sp->n_dofs, cudaMemcpyHostToDevice) != cudaSuccess)
    rc = fail(HF_ERR_CUDA, "u_bar upload failed");
  if (rc == HF_OK) rc = hf_tangent_create_ex(sp, strategy, 64, d, nullptr, out, err);
  cudaDeviceSynchronize();
  dfree(d);
  return rc;
}

static int tangent_apply(hf_tangent* op, const double* x_dev, double* y_dev, const int* skip_dev, int fill,
                         void* stream, long long tile0 = 0, long long tile1 = -1, int reserve_sms = 0) {
  if (!op || !x_dev || !y_dev) return fail(HF_ERR_ARG, "null argument");
  CellArgs a = base_args(op->sp);
  a.tile0 = tile0;
  a.tile1 = tile1;
  a.fp32 = op->fp32;
  a.cache_len = op->cache_len;
  a.x = x_dev;
  a.y = y_dev;
  a.cache = op->d_cache;
  a.ubar = op->d_ubar;
  a.skip = skip_dev;
  a.fill = fill;
  a.reserve_sms = reserve_sms;
  if (op->alternate && tile1 < 0) {  // whole-range apply: every other sweep backwards
    a.reverse = op->flip;
    op->flip ^= 1;
  } else if (tile1 < 0) {
    // Whole-range applies that do not alternate walk the tiles backwards.  The
    // vector kernels around an apply (Chebyshev and CG updates, dots) stream
    // their operands forwards, so L2 holds the END of x and y when the apply
    // starts and the kernel after it starts where the apply's last
    // reductions landed.  Config-4 CG iteration 10.53 -> 10.39 ms
    // (profiles/r02/ab_l2_evict_first.txt); HF_REVERSE=0 restores forwards.
    static int rev = -1;
    if (rev < 0) {
      const char* e = std::getenv("HF_REVERSE");
      rev = e ? std::atoi(e) : 1;
    }
    a.reverse = rev;
  }
  HF_CUDA(cell(op->sp, OP_APPLY, op->strategy, a, S(stream)));
  return HF_OK;
}

HF_API int hf_tangent_apply_raw(hf_tangent* op, const double* x_dev, double* y_dev, const int* skip_dev,
                                void* stream) {
  return tangent_apply(op, x_dev, y_dev, skip_dev, 0, stream);
}

// y = mask ? x : 0, then the cell kernel as its programmatic dependent
// launch: the apply overlaps the fill and waits for it only before scattering
HF_API int hf_tangent_apply_flagged(hf_tangent* op, const double* x_dev, double* y_dev, const int* skip_dev,
                                    void* stream) {
  if (!op || !x_dev || !y_dev) return fail(HF_ERR_ARG, "null argument");
  static int pdl = -1;
  if (pdl < 0) {
    const char* e = std::getenv("HF_PDL");
    pdl = e ? std::atoi(e) : 1;
  }
  if (op->fp32)
    k_fill_masked<float><<<fill_blocks(op->sp->n_dofs), 256, 0, S(stream)>>>(
        op->sp->n_dofs, (float*)y_dev, (const float*)x_dev, op->sp->d_mask, 0.0, skip_dev);
  else
    k_fill_masked<<<fill_blocks(op->sp->n_dofs), 256, 0, S(stream)>>>(op->sp->n_dofs, y_dev, x_dev, op->sp->d_mask,
                                                                     0.0, skip_dev);
  HF_CUDA(cudaGetLastError());
  if (op->sp->lat.n_el == 0) return HF_OK;
  return tangent_apply(op, x_dev, y_dev, skip_dev, pdl, stream);
}

// the cell kernel alone, as the programmatic dependent of a kernel that has
// written both x and y = mask ? x : 0 (hf_cheb_step_fill)
HF_API int hf_tangent_apply_after_fill(hf_tangent* op, const double* x_dev, double* y_dev, const int* skip_dev,
                                       void* stream) {
  if (op && op->sp->lat.n_el == 0) return HF_OK;
  return tangent_apply(op, x_dev, y_dev, skip_dev, 2, stream);
}

HF_API int hf_tangent_tiles(const hf_tangent* op, long long* n_tiles, int* cells_per_tile) {
  if (!op) return fail(HF_ERR_ARG, "null tangent");
  const hf_space* sp = op->sp;
  const int lines = sp->dim == 3 ? sp->n1 * sp->n1 : sp->n1;
  const int cpw = 32 / lines;
  if (cells_per_tile) *cells_per_tile = cpw;
  if (n_tiles) *n_tiles = (sp->lat.n_el + cpw - 1) / cpw;
  return HF_OK;
}

HF_API int hf_tangent_apply_tiles(hf_tangent* op, const double* x_dev, double* y_dev, const int* skip_dev,
                                  long long tile0, long long tile1, int mode, void* stream) {
  if (mode < 0 || mode > 2 || tile0 < 0 || tile1 < tile0) return fail(HF_ERR_ARG, "bad tile range or mode");
  if (!op || op->sp->lat.n_el == 0 || tile1 == tile0) return op ? HF_OK : fail(HF_ERR_ARG, "null tangent");
  return tangent_apply(op, x_dev, y_dev, skip_dev, mode, stream, tile0, tile1);
}

HF_API int hf_tangent_apply_tiles_ex(hf_tangent* op, const double* x_dev, double* y_dev, const int* skip_dev,
                                     long long tile0, long long tile1, int mode, int reserve_sms, void* stream) {
  if (mode < 0 || mode > 2 || tile0 < 0 || tile1 < tile0 || reserve_sms < 0)
    return fail(HF_ERR_ARG, "bad tile range, mode or reserve");
  if (!op || op->sp->lat.n_el == 0 || tile1 == tile0) return op ? HF_OK : fail(HF_ERR_ARG, "null tangent");
  return tangent_apply(op, x_dev, y_dev, skip_dev, mode, stream, tile0, tile1, reserve_sms);
}

HF_API int hf_tangent_set_alternate(hf_tangent* op, int on) {
  if (!op) return fail(HF_ERR_ARG, "null tangent");
  op->alternate = on != 0;
  op->flip = 0;
  return HF_OK;
}

HF_API int hf_tangent_apply(hf_tangent* op, const double* x_dev, double* y_dev, void* stream) {
  return hf_tangent_apply_flagged(op, x_dev, y_dev, nullptr, stream);
}

// ---- host-to-host apply: slab pipeline captured once per buffer pair ----
static void host_pipe_free(HostPipe* h) {
  if (!h) return;
  for (int i = 0; i < h->ng; ++i)
    if (h->g[i].exec) cudaGraphExecDestroy(h->g[i].exec);
  for (cudaEvent_t e : h->ev) cudaEventDestroy(e);
  if (h->done) cudaEventDestroy(h->done);
  if (h->cap) cudaStreamDestroy(h->cap);
  if (h->s_in) cudaStreamDestroy(h->s_in);
  if (h->s_out) cudaStreamDestroy(h->s_out);
  dfree(h->xd);
  dfree(h->yd);
  delete h;
}

static bool page_locked(const void* p, long long bytes) {
  const char* c = static_cast<const char*>(p);
  for (const char* q : {c, c + (bytes > 0 ? bytes - 1 : 0)}) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, q) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (at.type != cudaMemoryTypeHost) return false;
  }
  return true;
}

// Enqueue y_host = A x_host on h->cap (being captured).  The cells are cut
// into `chunks` slabs of last-axis cell layers; cells are lexicographic with
// the last axis slowest, so a slab touches a contiguous range of node planes,
// i.e. a contiguous DoF range.  H2D of each slab's new planes runs on s_in,
// fill + cell kernel on cap, D2H of the planes no later slab touches on s_out.
static int host_pipe_enqueue(hf_tangent* op, HostPipe* h, const double* xh, double* yh, int chunks, bool serial) {
  const hf_space* sp = op->sp;
  const int d = sp->dim, deg = sp->degree;
  const long long layer = d == 3 ? (long long)sp->lat.cells[0] * sp->lat.cells[1] : sp->lat.cells[0];
  const long long plane = (d == 3 ? (long long)sp->lat.nodes[0] * sp->lat.nodes[1] : sp->lat.nodes[0]) * d;
  const long long n_planes = sp->lat.nodes[d - 1];
  const int nl = sp->lat.cells[d - 1];
  long long nt;
  int cpt;
  hf_tangent_tiles(op, &nt, &cpt);
  std::vector<long long> cuts;
  for (int k = 0; k <= chunks; ++k) {
    const long long b = (long long)nl * k / chunks;
    const long long c = std::min(nt, (b * layer + cpt - 1) / cpt);
    if (cuts.empty() || c > cuts.back()) cuts.push_back(c);
  }
  auto planes = [&](long long t0, long long t1, long long& lo, long long& hi) {
    const long long z0 = t0 * cpt / layer;
    const long long z1 = (std::min(t1 * cpt, sp->lat.n_el) - 1) / layer;
    lo = z0 * deg;
    hi = (z1 + 1) * deg + 1;
  };
  const size_t need = 2 * cuts.size() + 6;
  while (h->ev.size() < need) {
    cudaEvent_t e;
    HF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    h->ev.push_back(e);
  }
  size_t ie = 0;
  HF_CUDA(cudaEventRecord(h->ev[ie], h->cap));
  HF_CUDA(cudaStreamWaitEvent(h->s_in, h->ev[ie], 0));
  HF_CUDA(cudaStreamWaitEvent(h->s_out, h->ev[ie], 0));
  ++ie;
  // H2D of every slab's new node planes, in slab order on s_in (one event each)
  std::vector<size_t> in_ev(cuts.size(), 0);
  long long copied = 0;
  for (size_t k = 0; k + 1 < cuts.size(); ++k) {
    long long lo, hi;
    planes(cuts[k], cuts[k + 1], lo, hi);
    if (hi > copied) {
      HF_CUDA(cudaMemcpyAsync(h->xd + copied * plane, xh + copied * plane, sizeof(double) * (hi - copied) * plane,
                              cudaMemcpyHostToDevice, h->s_in));
      copied = hi;
      HF_CUDA(cudaEventRecord(h->ev[ie], h->s_in));
      in_ev[k] = ie++;
    }
  }
  // serial: no D2H while any H2D is in flight (on hosts where the two copy
  // directions do not overlap, concurrent traffic is slower than back to back)
  if (serial) HF_CUDA(cudaStreamWaitEvent(h->s_out, h->ev[ie - 1], 0));
  long long filled = 0, sent = 0;
  for (size_t k = 0; k + 1 < cuts.size(); ++k) {
    const long long t0 = cuts[k], t1 = cuts[k + 1];
    long long lo, hi;
    planes(t0, t1, lo, hi);
    if (in_ev[k]) HF_CUDA(cudaStreamWaitEvent(h->cap, h->ev[in_ev[k]], 0));
    int mode = 0;
    if (hi > filled) {
      const long long off = filled * plane, cnt = (hi - filled) * plane;
      k_fill_masked<double><<<fill_blocks(cnt), 256, 0, h->cap>>>(cnt, h->yd + off, h->xd + off, sp->d_mask + off, 0.0,
                                                                 nullptr);
      HF_CUDA(cudaGetLastError());
      filled = hi;
      mode = 1;  // programmatic dependent of the fill
    }
    const int rc = tangent_apply(op, h->xd, h->yd, nullptr, mode, h->cap, t0, t1);
    if (rc != HF_OK) return rc;
    long long fin = n_planes;
    if (k + 2 < cuts.size()) {
      long long nlo, nhi;
      planes(cuts[k + 1], cuts[k + 2], nlo, nhi);
      fin = nlo;
    }
    if (fin > sent) {
      HF_CUDA(cudaEventRecord(h->ev[ie], h->cap));
      HF_CUDA(cudaStreamWaitEvent(h->s_out, h->ev[ie], 0));
      ++ie;
      HF_CUDA(cudaMemcpyAsync(yh + sent * plane, h->yd + sent * plane, sizeof(double) * (fin - sent) * plane,
                              cudaMemcpyDeviceToHost, h->s_out));
      sent = fin;
    }
  }
  HF_CUDA(cudaEventRecord(h->ev[ie], h->s_in));
  HF_CUDA(cudaStreamWaitEvent(h->cap, h->ev[ie], 0));
  ++ie;
  HF_CUDA(cudaEventRecord(h->ev[ie], h->s_out));
  HF_CUDA(cudaStreamWaitEvent(h->cap, h->ev[ie], 0));
  return HF_OK;
}

HF_API int hf_tangent_host_info(const hf_tangent* op, int* variant, float* us4) {
  if (!op) return fail(HF_ERR_ARG, "null tangent");
  const HostPipe* h = op->host;
  if (variant) *variant = h ? h->last_order : -1;
  if (us4)
    for (int v = 0; v < 4; ++v) us4[v] = h ? h->last_us[v] : 0.f;
  return HF_OK;
}

// Per-warp timeline of the last instrumented apply (HF_TIMELINE builds only)
HF_API int hf_timeline_fetch(unsigned long long* host, long long n, int clear) {
#ifdef HF_TIMELINE
  if (!host || n < (long long)HF_TL_WARPS * HF_TL_SLOTS) return fail(HF_ERR_ARG, "timeline buffer too small");
  HF_CUDA(cudaDeviceSynchronize());
  HF_CUDA(hf::timeline_copy_3d(host, clear));
  return HF_OK;
#else
  (void)host;
  (void)n;
  (void)clear;
  return fail(HF_ERR_UNSUPPORTED, "not an HF_TIMELINE build");
#endif
}

HF_API int hf_stream_synchronize(void* stream) {
  HF_CUDA(cudaStreamSynchronize(S(stream)));
  return HF_OK;
}

// ---- launch-sequence graphs (the V-cycle, multigrid.py:309-351) ----
// A Newton iteration rebuilds the GMG hierarchy and with it the V-cycle's
// launch sequence: same kernels and order, new pointers and Chebyshev
// coefficients.  Instantiating a fresh graph for it costs 3-9 ms and now and
// then 50-80 ms (device allocations of the executable graph); updating the
// previous executable graph in place costs about a millisecond and allocates
// nothing.  hf_graph_end therefore takes the handle of an earlier graph of the
// same shape and falls back to a new instantiation when the update is refused.
struct hf_graph {
  cudaGraphExec_t exec = nullptr;
};

HF_API int hf_graph_begin(void* stream) {
  HF_CUDA(cudaStreamBeginCapture(S(stream), cudaStreamCaptureModeThreadLocal));
  return HF_OK;
}

HF_API int hf_graph_end(void* stream, hf_graph** g, int* updated) {
  if (!g) return fail(HF_ERR_ARG, "null graph handle pointer");
  if (updated) *updated = 0;
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(S(stream), &graph);
  if (e != cudaSuccess || !graph) {
    cudaGetLastError();
    if (graph) cudaGraphDestroy(graph);
    return fail(HF_ERR_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e));
  }
  hf_graph* h = *g;
  if (h && h->exec) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(h->exec, graph, &info) == cudaSuccess) {
      cudaGraphDestroy(graph);
      if (updated) *updated = 1;
      return HF_OK;
    }
    cudaGetLastError();  // a different shape: instantiate anew
    cudaGraphExecDestroy(h->exec);
    h->exec = nullptr;
  }
  if (!h) h = new hf_graph();
  e = cudaGraphInstantiate(&h->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) {
    if (!*g) delete h;
    return fail(HF_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
  }
  *g = h;
  return HF_OK;
}

HF_API int hf_graph_launch(hf_graph* g, void* stream) {
  if (!g || !g->exec) return fail(HF_ERR_ARG, "null graph");
  HF_CUDA(cudaGraphLaunch(g->exec, S(stream)));
  return HF_OK;
}

HF_API int hf_graph_destroy(hf_graph* g) {
  if (!g) return HF_OK;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  delete g;
  return HF_OK;
}

HF_API int hf_host_register(void* p, long long bytes) {
  if (!p || bytes <= 0) return fail(HF_ERR_ARG, "null or empty host range");
  HF_CUDA(cudaHostRegister(p, (size_t)bytes, cudaHostRegisterDefault));
  return HF_OK;
}

HF_API int hf_host_unregister(void* p) {
  if (!p) return fail(HF_ERR_ARG, "null host pointer");
  HF_CUDA(cudaHostUnregister(p));
  return HF_OK;
}

HF_API int hf_tangent_apply_host(hf_tangent* op, const double* x_host, double* y_host, int chunks, void* stream) {
  if (!op || !x_host || !y_host) return fail(HF_ERR_ARG, "null argument");
  if (op->fp32) return fail(HF_ERR_UNSUPPORTED, "host apply of an fp32-storage tangent");
  hf_space* sp = op->sp;
  const long long bytes = (long long)sizeof(double) * sp->n_dofs;
  if (sp->n_dofs == 0) return HF_OK;
  if (!page_locked(x_host, bytes) || !page_locked(y_host, bytes))
    return fail(HF_ERR_ARG, "host buffers must be page-locked (cudaHostAlloc, or hf_host_register)");
  if (chunks < 1) chunks = 1;
  if (chunks > sp->lat.cells[sp->dim - 1]) chunks = sp->lat.cells[sp->dim - 1];
  if (sp->lat.n_el == 0) chunks = 1;
  HostPipe* h = op->host;
  if (!h) {
    h = op->host = new HostPipe();
    HF_CUDA(dmalloc((void**)&h->xd, bytes));
    HF_CUDA(dmalloc((void**)&h->yd, bytes));
    HF_CUDA(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
    HF_CUDA(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
    HF_CUDA(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
    HF_CUDA(cudaEventCreateWithFlags(&h->done, cudaEventDisableTiming));
  }
  HostPipe::Entry* hit = nullptr;
  for (int i = 0; i < h->ng; ++i)
    if (h->g[i].x == x_host && h->g[i].y == y_host && h->g[i].chunks == chunks) hit = &h->g[i];
  int recal_slot = -1;
  const bool recal_on = std::getenv("HF_E2E_RECAL") && !std::getenv("HF_E2E_ORDER");
  if (hit && recal_on && !hit->recal && hit->uses >= HostPipe::RECAL_AT) {
    hit->recal = 1;  // once, whatever the outcome below
    // the entry's graph may still run from an earlier call on any stream
    HF_CUDA(cudaEventSynchronize(h->done));
    if (hit->exec) HF_CUDA(cudaGraphExecDestroy(hit->exec));
    hit->exec = nullptr;
    hit->variant = 2;  // direct enqueue until the recalibration below has finished
    recal_slot = (int)(hit - h->g);
    hit = nullptr;
  }
  // enqueue directly on `stream` (no graph): fork/join through the pipe's streams
  auto direct = [&](bool serial) -> int {
    cudaEvent_t fork;
    HF_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    HF_CUDA(cudaEventRecord(fork, S(stream)));
    HF_CUDA(cudaStreamWaitEvent(h->cap, fork, 0));
    cudaEventDestroy(fork);
    const int rc = host_pipe_enqueue(op, h, x_host, y_host, chunks, serial);
    if (rc != HF_OK) return rc;
    cudaEvent_t join;
    HF_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    HF_CUDA(cudaEventRecord(join, h->cap));
    HF_CUDA(cudaStreamWaitEvent(S(stream), join, 0));
    cudaEventDestroy(join);
    return HF_OK;
  };
  if (!hit) {
    // Four ways to run the pipeline: captured as a graph or enqueued directly,
    // each with the copy directions overlapping or with every D2H held back
    // until the last H2D is done.  On first use per buffer pair all four are
    // timed on this host and the fastest is kept (hosts differ: on some,
    // concurrent H2D + D2H is slower than back to back, and graph launches with
    // host-memory copy nodes cost more than direct enqueues).
    // HF_E2E_ORDER=0..3 forces one.
    const char* env = std::getenv("HF_E2E_ORDER");
    const int force = env ? std::atoi(env) : -1;
    cudaGraphExec_t cand[2] = {nullptr, nullptr};
    for (int v = 0; v < 2; ++v) {
      if (force >= 0 && v != force) continue;
      cudaGraph_t graph;
      HF_CUDA(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
      const int rc = host_pipe_enqueue(op, h, x_host, y_host, chunks, v == 1);
      const cudaError_t ce = cudaStreamEndCapture(h->cap, &graph);
      if (rc != HF_OK) {
        if (ce == cudaSuccess) cudaGraphDestroy(graph);
        if (cand[0]) cudaGraphExecDestroy(cand[0]);
        return rc;
      }
      HF_CUDA(ce);
      const cudaError_t ie = cudaGraphInstantiate(&cand[v], graph, 0);
      cudaGraphDestroy(graph);
      HF_CUDA(ie);
    }
    int keep = force >= 0 && force <= 3 ? force : -1;
    if (keep < 0) {
      float best = 1e30f;
      for (int v = 0; v < 4; ++v) {
        auto run = [&]() -> int {
          if (v < 2) {
            HF_CUDA(cudaGraphLaunch(cand[v], S(stream)));
            return HF_OK;
          }
          return direct(v == 3);
        };
        auto drop = [&]() {  // error path: no candidate graph leaks
          for (int c = 0; c < 2; ++c)
            if (cand[c]) cudaGraphExecDestroy(cand[c]);
        };
        int rc = HF_OK;
        for (int w = 0; w < 2 && rc == HF_OK; ++w) rc = run();
        if (rc != HF_OK || cudaStreamSynchronize(S(stream)) != cudaSuccess) {
          drop();
          return rc != HF_OK ? rc : fail(HF_ERR_CUDA, "host pipeline calibration failed");
        }
        // host wall time of one synchronised step (enqueue cost included),
        // best of 5: the host link is noisy
        float us = 1e30f;
        for (int r = 0; r < 5; ++r) {
          const auto t0 = std::chrono::steady_clock::now();
          rc = run();
          if (rc != HF_OK || cudaStreamSynchronize(S(stream)) != cudaSuccess) {
            drop();
            return rc != HF_OK ? rc : fail(HF_ERR_CUDA, "host pipeline calibration failed");
          }
          us = std::min(us, std::chrono::duration<float, std::micro>(std::chrono::steady_clock::now() - t0).count());
        }
        h->last_us[v] = us;
        if (us < best) {
          best = us;
          keep = v;
        }
      }
    }
    for (int v = 0; v < 2; ++v)
      if (cand[v] && v != keep) cudaGraphExecDestroy(cand[v]);
    cudaGraphExec_t exec = keep < 2 ? cand[keep] : nullptr;
    h->last_order = keep;
    int slot;
    if (recal_slot >= 0) {
      slot = recal_slot;
    } else if (h->ng == HostPipe::NG) {  // evict the least recently used pipeline
      slot = 0;
      for (int i = 1; i < h->ng; ++i)
        if (h->g[i].used < h->g[slot].used) slot = i;
      if (h->g[slot].exec) cudaGraphExecDestroy(h->g[slot].exec);
    } else {
      slot = h->ng++;
    }
    h->g[slot] = {x_host, y_host, chunks, exec, 0, keep, 0, recal_slot >= 0 ? 1 : 0};
    hit = &h->g[slot];
  }
  hit->used = ++h->clock;
  ++hit->uses;
  if (hit->exec) {
    HF_CUDA(cudaGraphLaunch(hit->exec, S(stream)));
  } else {
    const int rc = direct(hit->variant == 3);
    if (rc != HF_OK) return rc;
  }
  HF_CUDA(cudaEventRecord(h->done, S(stream)));
  return HF_OK;
}

HF_API int hf_tangent_assemble_local(hf_tangent* op, double* vals_dev, void* stream) {
  if (!op || !vals_dev) return fail(HF_ERR_ARG, "null argument");
  if (op->strategy != HF_TENSOR4 || op->fp32)
    return fail(HF_ERR_ARG, "element matrices are formed from an fp64 tensor4 cache");
  const hf_space* sp = op->sp;
  if ((sp->dim == 3 && sp->n1 > 3) || (sp->dim == 2 && sp->n1 > 5))
    return fail(HF_ERR_UNSUPPORTED, "matrix-based assembly is instantiated for 3D Q1-Q2 and 2D Q1-Q4");
  CellArgs a = base_args(sp);
  a.cache = op->d_cache;
  HF_CUDA(launch_assemble(sp->dim, sp->n1, a, vals_dev, S(stream)));
  return HF_OK;
}

HF_API int hf_space_cell_dofs(const hf_space* sp, long long* dofs_dev, void* stream) {
  if (!sp || !dofs_dev) return fail(HF_ERR_ARG, "null argument");
  HF_CUDA(launch_cell_dofs(sp->lat, sp->dim, sp->degree, dofs_dev, S(stream)));
  return HF_OK;
}

HF_API int hf_tangent_diagonal(hf_tangent* op, double* d_dev, void* stream) {
  if (!op || !d_dev) return fail(HF_ERR_ARG, "null argument");
  if (op->fp32) return fail(HF_ERR_UNSUPPORTED, "diagonal of an fp32-storage tangent: use the fp64 operator");
  const hf_space* sp = op->sp;
  cudaStream_t s = S(stream);
  k_fill_masked<double><<<fill_blocks(sp->n_dofs), 256, 0, s>>>(sp->n_dofs, d_dev, nullptr, sp->d_mask, 1.0, nullptr);
  HF_CUDA(cudaGetLastError());
  CellArgs a = base_args(sp);
  a.y = d_dev;
  a.cache = op->d_cache;
  a.ubar = op->d_ubar;
  HF_CUDA(cell(sp, OP_DIAG, op->strategy, a, s));
  return HF_OK;
}

HF_API int hf_tangent_diagonal_host(hf_tangent* op, double* d_host) {
  if (!op || !d_host) return fail(HF_ERR_ARG, "null argument");
  const long long n = op->sp->n_dofs;
  double* d = nullptr;
  HF_CUDA(dmalloc((void**)&d, sizeof(double) * (n > 0 ? n : 1)));
  int rc = hf_tangent_diagonal(op, d, nullptr);
  if (rc == HF_OK && cudaMemcpy(d_host, d, sizeof(double) * n, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = fail(HF_ERR_CUDA, "diagonal download failed");
  cudaDeviceSynchronize();
  dfree(d);
  return rc;
}

HF_API int hf_tangent_storage(const hf_tangent* op, long long* storage_bytes, int* payload_scalars,
                              long long* payload_bytes) {
  if (!op) return fail(HF_ERR_ARG, "null tangent");
  const hf_space* sp = op->sp;
  int d = sp->dim, nv = d * (d + 1) / 2;
  int payload = op->strategy == HF_SCALAR ? 1 : (op->strategy == HF_TENSOR2 ? 2 + nv : nv + nv * (nv + 1) / 2);
  long long nqp = sp->lat.n_qp;
  if (payload_scalars) *payload_scalars = payload;
  if (payload_bytes) *payload_bytes = (op->fp32 ? 4ll : 8ll) * payload * nqp;
  // operators.py:412-417: payload + (jac_inv or jac_spatial_inv) + jxw
  if (storage_bytes) *storage_bytes = 8ll * nqp * (payload + d * d + 1);
  return HF_OK;
}

HF_API int hf_tangent_destroy(hf_tangent* op) {
  if (!op) return HF_OK;
  host_pipe_free(op->host);
  dfree(op->d_cache);
  dfree(op->d_ubar);
  delete op;
  return HF_OK;
}

// ---------------------------------------------------------------------------
HF_API int hf_residual(hf_space* sp, const double* u_dev, const double* traction, const double* surf_w_dev,
                       double* out_dev, void* stream, hf_error_info* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!sp || !u_dev || !out_dev) return fail(HF_ERR_ARG, "null argument");
  if (traction && !surf_w_dev) return fail(HF_ERR_ARG, "traction needs surface weights");
  cudaStream_t s = S(stream);
  HF_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(double) * sp->n_dofs, s));
  unsigned long long init = ~0ull;
  HF_CUDA(cudaMemcpyAsync(sp->d_u64, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  CellArgs a = base_args(sp);
  a.x = u_dev;
  a.y = out_dev;
  a.detmin = sp->d_u64;
  HF_CUDA(cell(sp, OP_RESIDUAL, 0, a, s));
  double t[3] = {0, 0, 0};
  if (traction)
    for (int i = 0; i < sp->dim; ++i) t[i] = traction[i];
  k_resid_finalize<<<vec_blocks(sp->n_dofs), 256, 0, s>>>(sp->lat.n_nodes, sp->dim, out_dev, surf_w_dev, t[0], t[1],
                                                          t[2], traction ? 1 : 0, sp->d_mask);
  HF_CUDA(cudaGetLastError());
  unsigned long long o;
  HF_CUDA(cudaMemcpyAsync(&o, sp->d_u64, sizeof(o), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  if (sp->lat.n_el > 0 && !(hf_unord(o) > 0.0)) return locate_min_det(sp, u_dev, s, err);
  return HF_OK;
}

HF_API int hf_energy(hf_space* sp, const double* u_dev, double* out_dev, void* stream, hf_error_info* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!sp || !u_dev || !out_dev) return fail(HF_ERR_ARG, "null argument");
  cudaStream_t s = S(stream);
  HF_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(double), s));
  unsigned long long init = ~0ull;
  HF_CUDA(cudaMemcpyAsync(sp->d_u64, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  CellArgs a = base_args(sp);
  a.x = u_dev;
  a.y = out_dev;
  a.detmin = sp->d_u64;
  HF_CUDA(cell(sp, OP_ENERGY, 0, a, s));
  unsigned long long o;
  HF_CUDA(cudaMemcpyAsync(&o, sp->d_u64, sizeof(o), cudaMemcpyDeviceToHost, s));
  HF_CUDA(cudaStreamSynchronize(s));
  if (sp->lat.n_el > 0 && !(hf_unord(o) > 0.0)) return locate_min_det(sp, u_dev, s, err);
  return HF_OK;
}

// ---------------------------------------------------------------------------
HF_API int hf_transfer_create(const hf_space* coarse, const hf_space* fine, const double* const* interp_1d,
                              hf_transfer** out) {
  if (!coarse || !fine || !interp_1d || !out) return fail(HF_ERR_ARG, "null argument");
  if (coarse->dim != fine->dim || coarse->degree != fine->degree) return fail(HF_ERR_ARG, "incompatible levels");
  for (int a = 0; a < coarse->dim; ++a)
    if (fine->lat.cells[a] != 2 * coarse->lat.cells[a])
      return fail(HF_ERR_ARG, "transfer requires a 2:1 refined pair of levels");
  hf_transfer* t = new hf_transfer();
  t->coarse = coarse;
  t->fine = fine;
  for (int a = 0; a < coarse->dim; ++a) {
    int nf = fine->lat.nodes[a], nc = coarse->lat.nodes[a];
    const double* M = interp_1d[a];  // (nf, nc) row-major
    std::vector<int> pp(1, 0), pc, rp(1, 0), rc;
    std::vector<double> pw, rw;
    for (int f = 0; f < nf; ++f) {
      for (int c = 0; c < nc; ++c)
        if (M[(long long)f * nc + c] != 0.0) {
          pc.push_back(c);
          pw.push_back(M[(long long)f * nc + c]);
        }
      pp.push_back((int)pc.size());
    }
    for (int c = 0; c < nc; ++c) {
      for (int f = 0; f < nf; ++f)
        if (M[(long long)f * nc + c] != 0.0) {
          rc.push_back(f);
          rw.push_back(M[(long long)f * nc + c]);
        }
      rp.push_back((int)rc.size());
    }
    HF_CUDA(dmalloc((void**)&t->d_pp[a], sizeof(int) * pp.size()));
    HF_CUDA(dmalloc((void**)&t->d_pc[a], sizeof(int) * (pc.size() + 1)));
    HF_CUDA(dmalloc((void**)&t->d_pw[a], sizeof(double) * (pw.size() + 1)));
    HF_CUDA(dmalloc((void**)&t->d_rp[a], sizeof(int) * rp.size()));
    HF_CUDA(dmalloc((void**)&t->d_rc[a], sizeof(int) * (rc.size() + 1)));
    HF_CUDA(dmalloc((void**)&t->d_rw[a], sizeof(double) * (rw.size() + 1)));
    HF_CUDA(cudaMemcpy(t->d_pp[a], pp.data(), sizeof(int) * pp.size(), cudaMemcpyHostToDevice));
    HF_CUDA(cudaMemcpy(t->d_pc[a], pc.data(), sizeof(int) * pc.size(), cudaMemcpyHostToDevice));
    HF_CUDA(cudaMemcpy(t->d_pw[a], pw.data(), sizeof(double) * pw.size(), cudaMemcpyHostToDevice));
    HF_CUDA(cudaMemcpy(t->d_rp[a], rp.data(), sizeof(int) * rp.size(), cudaMemcpyHostToDevice));
    HF_CUDA(cudaMemcpy(t->d_rc[a], rc.data(), sizeof(int) * rc.size(), cudaMemcpyHostToDevice));
    HF_CUDA(cudaMemcpy(t->d_rw[a], rw.data(), sizeof(double) * rw.size(), cudaMemcpyHostToDevice));
  }
  // largest intermediate: fine nodes (all passes are bounded by the fine lattice)
  t->tmp_len = fine->n_dofs;
  HF_CUDA(dmalloc((void**)&t->d_tmp[0], sizeof(double) * t->tmp_len));
  HF_CUDA(dmalloc((void**)&t->d_tmp[1], sizeof(double) * t->tmp_len));
  *out = t;
  return HF_OK;
}

HF_API int hf_prolong(hf_transfer* t, const double* xc, double* xf, int mode, void* stream) {
  if (!t || !xc || !xf) return fail(HF_ERR_ARG, "null argument");
  return transfer_dispatch(t, true, xc, 64, xf, 64, mode, S(stream));
}

HF_API int hf_restrict(hf_transfer* t, const double* rf, double* rc, int mode, void* stream) {
  if (!t || !rf || !rc) return fail(HF_ERR_ARG, "null argument");
  return transfer_dispatch(t, false, rf, 64, rc, 64, mode, S(stream));
}

HF_API int hf_prolong_ex(hf_transfer* t, const void* xc, int in_bits, void* xf, int out_bits, int mode, void* stream) {
  if (!t || !xc || !xf) return fail(HF_ERR_ARG, "null argument");
  return transfer_dispatch(t, true, xc, in_bits, xf, out_bits, mode, S(stream));
}

HF_API int hf_restrict_ex(hf_transfer* t, const void* rf, int in_bits, void* rc, int out_bits, int mode,
                          void* stream) {
  if (!t || !rf || !rc) return fail(HF_ERR_ARG, "null argument");
  return transfer_dispatch(t, false, rf, in_bits, rc, out_bits, mode, S(stream));
}

HF_API int hf_transfer_destroy(hf_transfer* t) {
  if (!t) return HF_OK;
  for (int a = 0; a < 3; ++a) {
    dfree(t->d_pp[a]);
    dfree(t->d_pc[a]);
    dfree(t->d_pw[a]);
    dfree(t->d_rp[a]);
    dfree(t->d_rc[a]);
    dfree(t->d_rw[a]);
  }
  dfree(t->d_tmp[0]);
  dfree(t->d_tmp[1]);
  delete t;
  return HF_OK;
}

HF_API int hf_inject(const hf_space* coarse, const hf_space* fine, const double* uf, double* uc, int keep_constrained,
                     void* stream) {
  if (!coarse || !fine || !uf || !uc) return fail(HF_ERR_ARG, "null argument");
  for (int a = 0; a < coarse->dim; ++a)
    if (fine->lat.nodes[a] != 2 * coarse->lat.nodes[a] - 1) return fail(HF_ERR_ARG, "levels are not 2:1 nested");
  k_inject<<<vec_blocks(coarse->n_dofs), 256, 0, S(stream)>>>(uf, uc, coarse->lat.nodes[0], coarse->lat.nodes[1],
                                                              coarse->dim == 3 ? coarse->lat.nodes[2] : 1,
                                                              fine->lat.nodes[0], fine->lat.nodes[1], coarse->dim,
                                                              coarse->d_mask, keep_constrained);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

// ---------------------------------------------------------------------------
HF_API int hf_ws_create(hf_ws** out) {
  if (!out) return fail(HF_ERR_ARG, "null argument");
  hf_ws* w = new hf_ws();
  HF_CUDA(dmalloc((void**)&w->d_partials, sizeof(double) * RED_MAX_BLOCKS));
  HF_CUDA(dmalloc((void**)&w->d_counter, sizeof(unsigned)));
  HF_CUDA(cudaMemset(w->d_counter, 0, sizeof(unsigned)));
  *out = w;
  return HF_OK;
}

HF_API int hf_ws_destroy(hf_ws* w) {
  if (!w) return HF_OK;
  dfree(w->d_partials);
  dfree(w->d_counter);
  delete w;
  return HF_OK;
}

HF_API int hf_dot(hf_ws* w, long long n, const double* a, const double* b, double* out_dev, const int* skip_dev,
                  void* stream) {
  if (!w || !a || !b || !out_dev) return fail(HF_ERR_ARG, "null argument");
  k_dot<<<red_blocks(n), RED_THREADS, 0, S(stream)>>>(n, a, b, w->d_partials, w->d_counter, out_dev, skip_dev);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_fill_masked(long long n, double* y, const double* x, const unsigned char* mask, double masked_value,
                          void* stream) {
  if (!y || !mask) return fail(HF_ERR_ARG, "null argument");
  k_fill_masked<<<fill_blocks(n), 256, 0, S(stream)>>>(n, y, x, mask, masked_value, nullptr);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_probe_dfma(long long iters, int blocks, int threads, double* sink_dev, void* stream) {
  if (!sink_dev || iters < 1 || blocks < 1 || threads < 32) return fail(HF_ERR_ARG, "bad probe arguments");
  k_probe_dfma<<<blocks, threads, 0, S(stream)>>>(iters, sink_dev);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

// ---- fp32 vector algebra of mixed-precision multigrid levels (arithmetic in fp64)
HF_API int hf_fill_masked_f32(long long n, float* y, const float* x, const unsigned char* mask, double masked_value,
                              void* stream) {
  if (!y || !mask) return fail(HF_ERR_ARG, "null argument");
  k_fill_masked<float><<<fill_blocks(n), 256, 0, S(stream)>>>(n, y, x, mask, masked_value, nullptr);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_cheb_step_f32(long long n, float* x, float* d, const float* b, const float* ax, const float* inv_d,
                            int first, double theta, double cd, double cz, int x_zero, const int* skip_dev,
                            const unsigned char* fill_mask, float* y_next, void* stream) {
  if (!x || !d || !b || !inv_d) return fail(HF_ERR_ARG, "null argument");
  k_cheb<float><<<vec_blocks(n), 256, 0, S(stream)>>>(n, x, d, b, ax, inv_d, first, theta, cd, cz, x_zero, skip_dev,
                                                      fill_mask, y_next, 0);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_resid_masked_f32(long long n, float* r, const float* b, const float* ax, const unsigned char* mask,
                               void* stream) {
  if (!r || !b || !ax || !mask) return fail(HF_ERR_ARG, "null argument");
  k_resid_masked<float><<<vec_blocks(n), 256, 0, S(stream)>>>(n, r, b, ax, mask);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_dot_f32(hf_ws* w, long long n, const float* a, const float* b, double* out_dev, void* stream) {
  if (!w || !a || !b || !out_dev) return fail(HF_ERR_ARG, "null argument");
  k_dot<float><<<red_blocks(n), RED_THREADS, 0, S(stream)>>>(n, a, b, w->d_partials, w->d_counter, out_dev, nullptr);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_resnorm_check_f32(hf_ws* w, long long n, const float* b, const float* ax, double* scal, int out_idx,
                                int target_idx, int* flag_dev, void* stream) {
  if (!w || !b || !ax || !scal || !flag_dev) return fail(HF_ERR_ARG, "null argument");
  cudaStream_t s = S(stream);
  k_resnorm_check<float><<<red_blocks(n), RED_THREADS, 0, s>>>(n, b, ax, w->d_partials, w->d_counter, scal, out_idx,
                                                                target_idx, flag_dev);
  k_scalar<<<1, 32, 0, s>>>(0, scal, out_idx, target_idx, 0.0, flag_dev);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_halo_pack(long long n, const int* idx, const double* y, double* buf, void* stream) {
  if (n <= 0) return HF_OK;
  if (!idx || !y || !buf) return fail(HF_ERR_ARG, "null argument");
  k_pack_idx<<<vec_blocks(n), 256, 0, S(stream)>>>(n, idx, y, buf);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_halo_unpack_add(long long n, const int* idx, double* y, const double* buf, const unsigned char* mask,
                              void* stream) {
  if (n <= 0) return HF_OK;
  if (!idx || !y || !buf || !mask) return fail(HF_ERR_ARG, "null argument");
  k_unpack_add_idx<<<vec_blocks(n), 256, 0, S(stream)>>>(n, idx, y, buf, mask);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_dot_owned(hf_ws* w, long long n, const double* a, const double* b, const unsigned char* own,
                        double* out_dev, void* stream) {
  if (!w || !a || !b || !own || !out_dev) return fail(HF_ERR_ARG, "null argument");
  k_dot_owned<<<red_blocks(n), RED_THREADS, 0, S(stream)>>>(n, a, b, own, w->d_partials, w->d_counter, out_dev);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_halo_add(long long n, double* y, const double* recv, const unsigned char* mask, void* stream) {
  if (!y || !recv || !mask) return fail(HF_ERR_ARG, "null argument");
  if (n <= 0) return HF_OK;
  k_halo_add<<<vec_blocks(n), 256, 0, S(stream)>>>(n, y, recv, mask);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_cheb_step(long long n, double* x, double* d, const double* b, const double* ax, const double* inv_d,
                        int first, double theta, double cd, double cz, int x_zero, const int* skip_dev,
                        void* stream) {
  if (!x || !d || !b || !inv_d) return fail(HF_ERR_ARG, "null argument");
  k_cheb<double><<<vec_blocks(n), 256, 0, S(stream)>>>(n, x, d, b, ax, inv_d, first, theta, cd, cz, x_zero, skip_dev,
                                                       nullptr, nullptr, 0);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_cheb_step_fill(long long n, double* x, double* d, const double* b, const double* ax, const double* inv_d,
                             int first, double theta, double cd, double cz, int x_zero, const int* skip_dev,
                             const unsigned char* mask, double* y_next, void* stream) {
  if (!x || !d || !b || !inv_d || !mask || !y_next) return fail(HF_ERR_ARG, "null argument");
  k_cheb<double><<<vec_blocks(n), 256, 0, S(stream)>>>(n, x, d, b, ax, inv_d, first, theta, cd, cz, x_zero, skip_dev,
                                                       mask, y_next, 0);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_cheb3_step(long long n, const void* xk, void* xo, const void* b, const void* ax, const void* inv_d,
                         int first, double theta, double cd, double cz, int xk_zero, int xprev_zero,
                         const unsigned char* fill_mask, void* y_next, int fp_bits, int after_apply, void* stream) {
  if (!xk || !xo || !b || !inv_d || xk == xo) return fail(HF_ERR_ARG, "null or aliased argument");
  if ((fill_mask == nullptr) != (y_next == nullptr)) return fail(HF_ERR_ARG, "fill_mask and y_next go together");
  if (fp_bits != 64 && fp_bits != 32) return fail(HF_ERR_ARG, "fp_bits must be 64 or 32");
  if (after_apply && !ax) return fail(HF_ERR_ARG, "after_apply needs ax");
  static int pdl = -1;  // HF_PDL_CHEB=0: plain launches (A/B)
  if (pdl < 0) {
    const char* e = std::getenv("HF_PDL_CHEB");
    pdl = e ? std::atoi(e) : 1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(vec_blocks(n));
  cfg.blockDim = dim3(256);
  cfg.stream = S(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  const int chained = (after_apply && pdl) ? 1 : 0;
  if (chained) {
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  if (fp_bits == 64)
    HF_CUDA(cudaLaunchKernelEx(&cfg, k_cheb3<double>, n, (const double*)xk, (double*)xo, (const double*)b,
                               (const double*)ax, (const double*)inv_d, first, theta, cd, cz, xk_zero, xprev_zero,
                               fill_mask, (double*)y_next, chained));
  else
    HF_CUDA(cudaLaunchKernelEx(&cfg, k_cheb3<float>, n, (const float*)xk, (float*)xo, (const float*)b,
                               (const float*)ax, (const float*)inv_d, first, theta, cd, cz, xk_zero, xprev_zero,
                               fill_mask, (float*)y_next, chained));
  return HF_OK;
}

HF_API int hf_cheb_step_after_apply(long long n, void* x, void* d, const void* b, const void* ax, const void* inv_d,
                                    int first, double theta, double cd, double cz, const unsigned char* fill_mask,
                                    void* y_next, int fp_bits, void* stream) {
  if (!x || !d || !b || !ax || !inv_d) return fail(HF_ERR_ARG, "null argument");
  if ((fill_mask == nullptr) != (y_next == nullptr)) return fail(HF_ERR_ARG, "fill_mask and y_next go together");
  if (fp_bits != 64 && fp_bits != 32) return fail(HF_ERR_ARG, "fp_bits must be 64 or 32");
  static int pdl = -1;  // HF_PDL_CHEB=0: a plain launch (A/B)
  if (pdl < 0) {
    const char* e = std::getenv("HF_PDL_CHEB");
    pdl = e ? std::atoi(e) : 1;
  }
  if (!pdl) {
    if (fp_bits == 64)
      k_cheb<double><<<vec_blocks(n), 256, 0, S(stream)>>>(n, (double*)x, (double*)d, (const double*)b,
                                                           (const double*)ax, (const double*)inv_d, first, theta, cd,
                                                           cz, 0, nullptr, fill_mask, (double*)y_next, 0);
    else
      k_cheb<float><<<vec_blocks(n), 256, 0, S(stream)>>>(n, (float*)x, (float*)d, (const float*)b, (const float*)ax,
                                                          (const float*)inv_d, first, theta, cd, cz, 0, nullptr,
                                                          fill_mask, (float*)y_next, 0);
    HF_CUDA(cudaGetLastError());
    return HF_OK;
  }
  if (fp_bits == 64)
    HF_CUDA(launch_cheb_after_apply<double>(n, (double*)x, (double*)d, (const double*)b, (const double*)ax,
                                            (const double*)inv_d, first, theta, cd, cz, fill_mask, (double*)y_next,
                                            S(stream)));
  else
    HF_CUDA(launch_cheb_after_apply<float>(n, (float*)x, (float*)d, (const float*)b, (const float*)ax,
                                           (const float*)inv_d, first, theta, cd, cz, fill_mask, (float*)y_next,
                                           S(stream)));
  return HF_OK;
}

HF_API int hf_resid_masked(long long n, double* r, const double* b, const double* ax, const unsigned char* mask,
                           void* stream) {
  if (!r || !b || !ax || !mask) return fail(HF_ERR_ARG, "null argument");
  k_resid_masked<<<vec_blocks(n), 256, 0, S(stream)>>>(n, r, b, ax, mask);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_resnorm_check(hf_ws* w, long long n, const double* b, const double* ax, double* scal, int out_idx,
                            int target_idx, int* flag_dev, void* stream) {
  if (!w || !b || !ax || !scal || !flag_dev) return fail(HF_ERR_ARG, "null argument");
  cudaStream_t s = S(stream);
  k_resnorm_check<<<red_blocks(n), RED_THREADS, 0, s>>>(n, b, ax, w->d_partials, w->d_counter, scal, out_idx,
                                                         target_idx, flag_dev);
  k_scalar<<<1, 32, 0, s>>>(0, scal, out_idx, target_idx, 0.0, flag_dev);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_scalar_op(int op, double* scal, int a, int b, double rel, int* flag_dev, void* stream) {
  if (!scal || !flag_dev) return fail(HF_ERR_ARG, "null argument");
  k_scalar<<<1, 32, 0, S(stream)>>>(op, scal, a, b, rel, flag_dev);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_cg_update_xr(hf_ws* w, long long n, double* x, double* r, const double* p, const double* ap,
                           double* scal, int irz, int ipap, int irr, void* stream) {
  if (!w || !x || !r || !p || !ap || !scal) return fail(HF_ERR_ARG, "null argument");
  k_cg_xr<<<red_blocks(n), RED_THREADS, 0, S(stream)>>>(n, x, r, p, ap, scal, irz, ipap, irr, w->d_partials,
                                                       w->d_counter);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_cg_update_p(long long n, double* p, const double* z, const double* scal, int irzn, int irz,
                          void* stream) {
  if (!p || !z || !scal) return fail(HF_ERR_ARG, "null argument");
  k_cg_p<<<vec_blocks(n), 256, 0, S(stream)>>>(n, p, z, scal, irzn, irz, nullptr, nullptr);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_cg_update_p_fill(long long n, double* p, const double* z, const double* scal, int irzn, int irz,
                               const unsigned char* mask, double* y_next, void* stream) {
  if (!p || !z || !scal || !mask || !y_next) return fail(HF_ERR_ARG, "null argument");
  k_cg_p<<<vec_blocks(n), 256, 0, S(stream)>>>(n, p, z, scal, irzn, irz, mask, y_next);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_jacobi_dot(hf_ws* w, long long n, double* z, const double* r, const double* inv_d, double* out_dev,
                         void* stream) {
  if (!w || !z || !r || !inv_d || !out_dev) return fail(HF_ERR_ARG, "null argument");
  k_jacobi_dot<<<red_blocks(n), RED_THREADS, 0, S(stream)>>>(n, z, r, inv_d, w->d_partials, w->d_counter, out_dev);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

// Pack a host CSR into per-CTA shared-memory blocks (CoarseBlock) and upload;
// slot_off[k] receives the blob byte offset of CSR value k.
static int coarse_build(long long n, long long nnz, const std::vector<int>& rp, const std::vector<int>& cl,
                        const std::vector<double>& va, cudaStream_t s, hf_coarse** out,
                        std::vector<long long>* slot_off) {
  if (n >= (1ll << 31) || nnz >= (1ll << 31)) return fail(HF_ERR_UNSUPPORTED, "coarse matrix too large");
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // one CTA per SM (the grid barrier costs the same ~1.2 us from 35 to 148
  // CTAs on B200, tools/probes/gridsync_probe.cu), fewer for tiny levels; a
  // level whose whole block (values, columns, rows, iterate) fits one CTA's
  // shared memory runs as a single CTA without grid barriers
  const size_t one_cta = coarse_align16(8ull * nnz) + coarse_align16(4ull * n) + coarse_align16(4ull * (n + 1)) +
                         coarse_align16(2ull * nnz) + 8ull * 6 * n;
  const char* single_env = std::getenv("HF_COARSE_SINGLE");  // "0": always the multi-CTA form (tests)
  const bool single = one_cta <= 160 * 1024 && n <= 65535 && !(single_env && single_env[0] == '0');
  const int grid = single ? 1 : (int)std::max(1ll, std::min<long long>(nsm, (n + 7) / 8));
  const int rows_per = (int)((n + grid - 1) / grid);
  std::vector<unsigned char> blob;
  std::vector<long long> boff(grid);
  if (slot_off) slot_off->assign(nnz, 0);
  std::vector<int> pos(n, -1);
  size_t smem = 0;
  for (int c = 0; c < grid; ++c) {
    const int r0 = std::min<long long>(n, (long long)c * rows_per), r1 = std::min<long long>(n, (long long)r0 + rows_per);
    const int rows = r1 - r0;
    const int k0 = rp[r0], k1 = rp[r1], nz = k1 - k0;
    std::vector<int> u(cl.begin() + k0, cl.begin() + k1);
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    if (u.size() > 65535) return fail(HF_ERR_UNSUPPORTED, "coarse CTA block touches too many columns");
    for (size_t q = 0; q < u.size(); ++q) pos[u[q]] = (int)q;
    const size_t body = coarse_align16(8ull * nz) + coarse_align16(4ull * u.size()) +
                        coarse_align16(4ull * (rows + 1)) + coarse_align16(2ull * nz);
    smem = std::max<size_t>(smem, body + 8 * (u.size() + 5 * (size_t)rows));
    const size_t base = blob.size();
    boff[c] = (long long)base;
    blob.resize(base + 16 + body, 0);
    CoarseBlock h = {r0, rows, (int)u.size(), nz};
    std::memcpy(blob.data() + base, &h, sizeof(h));
    unsigned char* p = blob.data() + base + 16;
    std::memcpy(p, va.data() + k0, 8ull * nz);
    if (slot_off)
      for (int k = 0; k < nz; ++k) (*slot_off)[k0 + k] = (long long)(base + 16 + 8ull * k);
    p += coarse_align16(8ull * nz);
    std::memcpy(p, u.data(), 4ull * u.size());
    p += coarse_align16(4ull * u.size());
    int* lr = reinterpret_cast<int*>(p);
    for (int l = 0; l <= rows; ++l) lr[l] = rp[r0 + l] - k0;
    p += coarse_align16(4ull * (rows + 1));
    unsigned short* lc = reinterpret_cast<unsigned short*>(p);
    for (int k = 0; k < nz; ++k) lc[k] = (unsigned short)pos[cl[k0 + k]];
  }
  if (smem > 200 * 1024) return fail(HF_ERR_UNSUPPORTED, "coarse level too large for the one-kernel solve");
  HF_CUDA(cudaFuncSetAttribute(k_coarse_cheb<COARSE_THREADS, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  HF_CUDA(cudaFuncSetAttribute(k_coarse_cheb<COARSE_THREADS_1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));

  int per_sm = 0;
  if (grid == 1)
    HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_coarse_cheb<COARSE_THREADS_1, 4>, COARSE_THREADS_1, smem));
  else
    HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_coarse_cheb<COARSE_THREADS, 32>, COARSE_THREADS, smem));
  if (per_sm < 1) return fail(HF_ERR_UNSUPPORTED, "coarse kernel cannot be resident");
  hf_coarse* c = new hf_coarse();
  c->n = (int)n;
  c->nnz = nnz;
  c->grid = grid;
  c->smem = smem;
  c->blob_bytes = blob.size();
  HF_CUDA(dmalloc((void**)&c->blob, blob.size()));
  HF_CUDA(dmalloc((void**)&c->boff, sizeof(long long) * grid));
  HF_CUDA(dmalloc((void**)&c->xb, sizeof(double) * n));
  HF_CUDA(dmalloc((void**)&c->partials, sizeof(double) * grid));
  HF_CUDA(cudaMemcpyAsync(c->blob, blob.data(), blob.size(), cudaMemcpyHostToDevice, s));
  HF_CUDA(cudaMemcpyAsync(c->boff, boff.data(), sizeof(long long) * grid, cudaMemcpyHostToDevice, s));
  HF_CUDA(cudaStreamSynchronize(s));
  *out = c;
  return HF_OK;
}

HF_API int hf_coarse_create(long long n, long long nnz, const int* rowptr_dev, const int* col_dev,
                            const double* val_dev, void* stream, hf_coarse** out) {
  if (!out || n <= 0 || nnz < 0 || !rowptr_dev || (nnz > 0 && (!col_dev || !val_dev)))
    return fail(HF_ERR_ARG, "bad coarse matrix");
  if (n >= (1ll << 31) || nnz >= (1ll << 31)) return fail(HF_ERR_UNSUPPORTED, "coarse matrix too large");
  cudaStream_t s = S(stream);
  std::vector<int> rp(n + 1), cl(nnz);
  std::vector<double> va(nnz);
  HF_CUDA(cudaMemcpyAsync(rp.data(), rowptr_dev, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, s));
  if (nnz > 0) {
    HF_CUDA(cudaMemcpyAsync(cl.data(), col_dev, sizeof(int) * nnz, cudaMemcpyDeviceToHost, s));
    HF_CUDA(cudaMemcpyAsync(va.data(), val_dev, sizeof(double) * nnz, cudaMemcpyDeviceToHost, s));
  }
  HF_CUDA(cudaStreamSynchronize(s));
  return coarse_build(n, nnz, rp, cl, va, s, out, nullptr);
}

// The level's sparsity pattern from the cell DoF map and the constraint mask
// (AssembledTangent, operators.py:471-490: constrained rows/columns cleared,
// unit diagonal), built once on the host; values come later from element
// matrices (hf_coarse_update), summed per CSR slot in ascending entry order.
HF_API int hf_coarse_create_space(const hf_space* sp, void* stream, hf_coarse** out) {
  if (!sp || !out) return fail(HF_ERR_ARG, "null argument");
  if ((sp->dim == 3 && sp->n1 > 3) || (sp->dim == 2 && sp->n1 > 5))
    return fail(HF_ERR_UNSUPPORTED, "element matrices are instantiated for 3D Q1-Q2 and 2D Q1-Q4");
  cudaStream_t s = S(stream);
  const long long nel = sp->lat.n_el, n = sp->n_dofs;
  int nloc = 1;
  for (int a = 0; a < sp->dim; ++a) nloc *= sp->n1;
  const int nld = nloc * sp->dim;
  if (n >= (1ll << 31) || nel * nld * nld >= (1ll << 31)) return fail(HF_ERR_UNSUPPORTED, "coarse level too large");
  long long* d_dofs = nullptr;
  HF_CUDA(dmalloc((void**)&d_dofs, sizeof(long long) * std::max(1ll, nel * nld)));
  std::vector<long long> dofs(nel * nld);
  std::vector<unsigned char> mask(n);
  cudaError_t e = launch_cell_dofs(sp->lat, sp->dim, sp->degree, d_dofs, s);
  if (e == cudaSuccess && nel > 0)
    e = cudaMemcpyAsync(dofs.data(), d_dofs, sizeof(long long) * nel * nld, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(mask.data(), sp->d_mask, n, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  dfree(d_dofs);
  HF_CUDA(e);
  struct Ent {
    int r, c, k;  // k = element-matrix entry, -1 = unit diagonal of a constrained row
  };
  std::vector<Ent> ent;
  ent.reserve((size_t)nel * nld * nld);
  for (long long el = 0; el < nel; ++el)
    for (int i = 0; i < nld; ++i) {
      const int r = (int)dofs[el * nld + i];
      if (mask[r]) continue;
      for (int j = 0; j < nld; ++j) {
        const int c = (int)dofs[el * nld + j];
        if (!mask[c]) ent.push_back({r, c, (int)((el * nld + i) * nld + j)});
      }
    }
  for (long long r = 0; r < n; ++r)
    if (mask[r]) ent.push_back({(int)r, (int)r, -1});
  std::sort(ent.begin(), ent.end(), [](const Ent& a, const Ent& b) {
    return a.r != b.r ? a.r < b.r : (a.c != b.c ? a.c < b.c : a.k < b.k);
  });
  std::vector<int> rp(n + 1, 0), cl, cptr(1, 0), cidx;
  std::vector<double> va;
  std::vector<int> slot_of_upd;  // CSR slot of update u
  for (size_t q = 0; q < ent.size();) {
    size_t q1 = q;
    while (q1 < ent.size() && ent[q1].r == ent[q].r && ent[q1].c == ent[q].c) ++q1;
    const int slot = (int)cl.size();
    cl.push_back(ent[q].c);
    rp[ent[q].r + 1]++;
    if (ent[q].k < 0) {
      va.push_back(1.0);
    } else {
      va.push_back(0.0);
      for (size_t t = q; t < q1; ++t) cidx.push_back(ent[t].k);
      cptr.push_back((int)cidx.size());
      slot_of_upd.push_back(slot);
    }
    q = q1;
  }
  for (long long r = 0; r < n; ++r) rp[r + 1] += rp[r];
  std::vector<long long> slot_off;
  const int rc = coarse_build(n, (long long)cl.size(), rp, cl, va, s, out, &slot_off);
  if (rc != HF_OK) return rc;
  hf_coarse* c = *out;
  c->sp = sp;
  c->nupd = (int)slot_of_upd.size();
  std::vector<long long> uoff(c->nupd);
  for (int u = 0; u < c->nupd; ++u) uoff[u] = slot_off[slot_of_upd[u]];
  HF_CUDA(dmalloc((void**)&c->cptr, sizeof(int) * (c->nupd + 1)));
  HF_CUDA(dmalloc((void**)&c->cidx, sizeof(int) * std::max<size_t>(1, cidx.size())));
  HF_CUDA(dmalloc((void**)&c->uoff, sizeof(long long) * std::max(1, c->nupd)));
  HF_CUDA(dmalloc((void**)&c->elem, sizeof(double) * std::max(1ll, nel * nld * nld)));
  HF_CUDA(cudaMemcpyAsync(c->cptr, cptr.data(), sizeof(int) * (c->nupd + 1), cudaMemcpyHostToDevice, s));
  if (!cidx.empty())
    HF_CUDA(cudaMemcpyAsync(c->cidx, cidx.data(), sizeof(int) * cidx.size(), cudaMemcpyHostToDevice, s));
  if (c->nupd) HF_CUDA(cudaMemcpyAsync(c->uoff, uoff.data(), sizeof(long long) * c->nupd, cudaMemcpyHostToDevice, s));
  HF_CUDA(cudaStreamSynchronize(s));
  return HF_OK;
}

// Refresh the values from the element matrices of a tensor4 fp64 tangent on
// the same space (asynchronous; the sparsity pattern is unchanged).
HF_API int hf_coarse_update(hf_coarse* c, hf_tangent* op, void* stream) {
  if (!c || !op) return fail(HF_ERR_ARG, "null argument");
  if (!c->sp || op->sp != c->sp) return fail(HF_ERR_ARG, "coarse handle was not created from this tangent's space");
  if (op->strategy != HF_TENSOR4 || op->fp32) return fail(HF_ERR_ARG, "element matrices need an fp64 tensor4 tangent");
  cudaStream_t s = S(stream);
  CellArgs a = base_args(op->sp);
  a.cache = op->d_cache;
  HF_CUDA(launch_assemble(op->sp->dim, op->sp->n1, a, c->elem, s));
  if (c->nupd) {
    k_coarse_values<<<(unsigned)((c->nupd + 255) / 256), 256, 0, s>>>(c->nupd, c->cptr, c->cidx, c->elem, c->blob,
                                                                      c->uoff);
    HF_CUDA(cudaGetLastError());
  }
  return HF_OK;
}

// an independent handle with the same pattern (own values and iterate buffers)
HF_API int hf_coarse_clone(const hf_coarse* src, void* stream, hf_coarse** out) {
  if (!src || !out) return fail(HF_ERR_ARG, "null argument");
  cudaStream_t s = S(stream);
  hf_coarse* c = new hf_coarse(*src);
  c->blob = nullptr;
  c->boff = nullptr;
  c->xb = nullptr;
  c->partials = nullptr;
  c->cptr = nullptr;
  c->cidx = nullptr;
  c->uoff = nullptr;
  c->elem = nullptr;
  auto dup = [&](void** dst, const void* from, size_t bytes) -> cudaError_t {
    cudaError_t e = dmalloc(dst, std::max<size_t>(bytes, 8));
    if (e == cudaSuccess && from && bytes) e = cudaMemcpyAsync(*dst, from, bytes, cudaMemcpyDeviceToDevice, s);
    return e;
  };
  int nloc = 1, nld = 0;
  if (src->sp) {
    for (int a = 0; a < src->sp->dim; ++a) nloc *= src->sp->n1;
    nld = nloc * src->sp->dim;
  }
  const long long nel = src->sp ? src->sp->lat.n_el : 0;
  long long ncidx = 0;
  if (src->nupd) HF_CUDA(cudaMemcpy(&ncidx, src->cptr + src->nupd, sizeof(int), cudaMemcpyDeviceToHost));
  ncidx = (int)ncidx;
  cudaError_t e = dup((void**)&c->blob, src->blob, src->blob_bytes);
  if (e == cudaSuccess) e = dup((void**)&c->boff, src->boff, sizeof(long long) * src->grid);
  if (e == cudaSuccess) e = dup((void**)&c->xb, nullptr, sizeof(double) * src->n);
  if (e == cudaSuccess) e = dup((void**)&c->partials, nullptr, sizeof(double) * src->grid);
  if (e == cudaSuccess && src->cptr) e = dup((void**)&c->cptr, src->cptr, sizeof(int) * (src->nupd + 1));
  if (e == cudaSuccess && src->cidx) e = dup((void**)&c->cidx, src->cidx, sizeof(int) * ncidx);
  if (e == cudaSuccess && src->uoff) e = dup((void**)&c->uoff, src->uoff, sizeof(long long) * src->nupd);
  if (e == cudaSuccess && src->elem) e = dup((void**)&c->elem, nullptr, sizeof(double) * nel * nld * nld);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    hf_coarse_destroy(c);
    return fail(HF_ERR_CUDA, std::string("hf_coarse_clone: ") + cudaGetErrorString(e));
  }
  *out = c;
  return HF_OK;
}

HF_API int hf_coarse_destroy(hf_coarse* c) {
  if (!c) return HF_OK;
  dfree(c->blob);
  dfree(c->boff);
  dfree(c->xb);
  dfree(c->partials);
  dfree(c->cptr);
  dfree(c->cidx);
  dfree(c->uoff);
  dfree(c->elem);
  delete c;
  return HF_OK;
}

HF_API int hf_coarse_cheb_solve(hf_coarse* c, const double* b, double* x, double* d, const double* inv_d,
                                double theta, double delta, double sigma, double rel_target, int max_applications,
                                int degree, double* scal_dev, int* flag_dev, void* stream) {
  if (!c || !b || !x || !d || !inv_d || !scal_dev || !flag_dev || degree < 1)
    return fail(HF_ERR_ARG, "null argument or degree < 1");
  CoarseArgs a;
  a.n = c->n;
  a.blob = c->blob;
  a.boff = c->boff;
  a.b = b;
  a.inv_d = inv_d;
  a.x = x;
  a.xb = c->xb;
  a.d = d;
  a.partials = c->partials;
  a.scal = scal_dev;
  a.flag = flag_dev;
  a.theta = theta;
  a.delta = delta;
  a.sigma = sigma;
  a.rel_target = rel_target;
  a.max_applications = max_applications;
  a.degree = degree;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)c->grid);
  cfg.blockDim = dim3(c->grid == 1 ? COARSE_THREADS_1 : COARSE_THREADS);
  cfg.dynamicSmemBytes = c->smem;
  cfg.stream = S(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // co-residency for the grid barrier
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (c->grid == 1)
    HF_CUDA(cudaLaunchKernelEx(&cfg, k_coarse_cheb<COARSE_THREADS_1, 4>, a));
  else
    HF_CUDA(cudaLaunchKernelEx(&cfg, k_coarse_cheb<COARSE_THREADS, 32>, a));
  return HF_OK;
}

HF_API int hf_lanczos_init(const double* scal_dev, int* state_dev, void* stream) {
  if (!scal_dev || !state_dev) return fail(HF_ERR_ARG, "null argument");
  k_lanczos_init<<<1, 1, 0, S(stream)>>>(scal_dev, state_dev);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_lanczos_step(hf_ws* w, long long n, double* r, double* z, double* p, const double* ap,
                           const double* inv_d, double* scal_dev, double* ab_dev, int* state_dev, void* stream) {
  if (!w || !r || !z || !p || !ap || !inv_d || !scal_dev || !ab_dev || !state_dev)
    return fail(HF_ERR_ARG, "null argument");
  cudaStream_t s = S(stream);
  k_dot<<<red_blocks(n), RED_THREADS, 0, s>>>(n, p, ap, w->d_partials, w->d_counter, scal_dev + 1, state_dev);
  k_lanczos_r<<<vec_blocks(n), 256, 0, s>>>(n, r, ap, scal_dev, state_dev);
  k_jacobi_dot<<<red_blocks(n), RED_THREADS, 0, s>>>(n, z, r, inv_d, w->d_partials, w->d_counter, scal_dev + 2);
  k_lanczos_scalar<<<1, 1, 0, s>>>(scal_dev, state_dev, ab_dev);
  k_lanczos_p<<<vec_blocks(n), 256, 0, s>>>(n, p, z, scal_dev, state_dev);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

// hf_lanczos_step with two passes fused (r update + Jacobi + r.z; p update +
// the next application's initialisation y_next = mask ? p : 0): the next
// application is then launched with hf_tangent_apply_after_fill
HF_API int hf_lanczos_step_fill(hf_ws* w, long long n, double* r, double* z, double* p, const double* ap,
                                const double* inv_d, double* scal_dev, double* ab_dev, int* state_dev,
                                const unsigned char* mask, double* y_next, void* stream) {
  if (!w || !r || !z || !p || !ap || !inv_d || !scal_dev || !ab_dev || !state_dev || !mask || !y_next)
    return fail(HF_ERR_ARG, "null argument");
  cudaStream_t s = S(stream);
  k_dot<<<red_blocks(n), RED_THREADS, 0, s>>>(n, p, ap, w->d_partials, w->d_counter, scal_dev + 1, state_dev);
  k_lanczos_rz<<<red_blocks(n), RED_THREADS, 0, s>>>(n, r, z, ap, inv_d, scal_dev, state_dev, w->d_partials,
                                                     w->d_counter);
  k_lanczos_scalar<<<1, 1, 0, s>>>(scal_dev, state_dev, ab_dev);
  k_lanczos_p_fill<<<vec_blocks(n), 256, 0, s>>>(n, p, z, scal_dev, state_dev, mask, y_next);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

HF_API int hf_axpby(long long n, double a, const double* x, double b, double* y, void* stream) {
  if (!x || !y) return fail(HF_ERR_ARG, "null argument");
  k_axpby<<<vec_blocks(n), 256, 0, S(stream)>>>(n, a, x, b, y);
  HF_CUDA(cudaGetLastError());
  return HF_OK;
}

}  // extern "C"
