// Instantiation/dispatch of the cell kernels for one dimension.
#pragma once
#include "hf_dispatch.h"
#include "hf_line.cuh"


namespace hf {

inline int nsm_cached() {
  static int n = -1;
  if (n < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// Launch of the line-parallel apply (hf_line.cuh): persistent warps, grid
// sized to the resident capacity (148 SMs x blocks per SM) or the tile count.
template <int DIM, int N, int VAR, typename ST>
cudaError_t launch_apply_line_t(const CellArgs& c, cudaStream_t s) {
  using K = LineCfg<DIM, N>;
  using PL = LinePlan<DIM, N, VAR, ST>;
  constexpr auto kern = k_apply_line<DIM, N, VAR, ST>;
  static int resident = -1;
  if (resident < 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PL::SMEM);
    if (e != cudaSuccess) return e;
    int per_sm = 0, dev = 0, nsm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PL::NT, PL::SMEM);
    if (e != cudaSuccess) return e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    resident = (per_sm > 0 ? per_sm : 1) * (nsm > 0 ? nsm : 148);
  }
  LineArgs a;
  a.lat = c.lat;
  a.degree = c.degree;
  a.x = c.x;
  a.y = c.y;
  a.cache = c.cache;
  a.ubar = c.ubar;
  a.mu = c.mu;
  a.lam = c.lam;
  a.mask = c.mask;
  a.lmask = c.lmask;
  a.skip = c.skip;
  a.fill = c.fill;
  a.cache_len = c.cache_len;
  a.reverse = c.reverse;


  const long long all_tiles = (c.lat.n_el + K::CPW - 1) / K::CPW;
  a.tile0 = c.tile1 < 0 ? 0 : c.tile0;
  a.tile1 = c.tile1 < 0 ? all_tiles : (c.tile1 < all_tiles ? c.tile1 : all_tiles);
  TabLine<N> T = {};
  for (int l = 0; l < N; ++l)
    for (int o = 0; o < N; ++o) {
      T.V[l][o] = c.tab.V[l * N + o];
      T.Dc[l][o] = c.tab.Dc[l * N + o];
    }
  if constexpr (LaneMapT<DIM, N>::ENABLED) {
    using Z = LaneMapT<DIM, N>;
    static_assert(Z::OFF_WORDS <= 2, "TabLine::loff holds two words per lane");
    for (int lane = 0; lane < 32; ++lane)
      for (int i = 0; i < Z::OFF_WORDS; ++i) T.loff[lane][i] = Z::TABLE[lane][i];
  }
  // One block per tile up to the resident capacity: a small level (fewer
  // tiles than SMs) runs one warp per SM instead of W warps sharing a few SMs,
  // which shortens its latency chain; larger levels fill every SM.
  const long long tiles = a.tile1 - a.tile0;
  long long nb = tiles;
  long long cap = resident;
  if (c.reserve_sms > 0 && cap > 2ll * c.reserve_sms) cap -= (cap / (nsm_cached() > 0 ? nsm_cached() : 148)) * c.reserve_sms;
  if (nb > cap) nb = cap;
  if (nb <= 0) return cudaSuccess;
  if (!c.fill) {
    kern<<<(unsigned)nb, PL::NT, PL::SMEM, s>>>(a, T);
    return cudaGetLastError();
  }
  // programmatic dependent launch after the fill kernel (hf_api.cu)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nb);
  cfg.blockDim = dim3(PL::NT);
  cfg.dynamicSmemBytes = PL::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, T);
}

template <int DIM, int N, int VAR>
cudaError_t launch_apply_line(const CellArgs& c, cudaStream_t s) {
  return c.fp32 ? launch_apply_line_t<DIM, N, VAR, float>(c, s) : launch_apply_line_t<DIM, N, VAR, double>(c, s);
}

template <int DIM, int N>
cudaError_t launch_one(int op, int var, const CellArgs& a, int mode, double target, unsigned long long* first,
                       cudaStream_t s) {
  using K = Cfg<DIM, N>;
  long long nb = (a.lat.n_el + K::CPB - 1) / K::CPB;
  if (nb <= 0) return cudaSuccess;
  dim3 grid((unsigned)nb), block(K::NT);
  size_t sm = K::SMEM;
  switch (op) {
    case OP_APPLY:
      if (var == SCALAR) return launch_apply_line<DIM, N, SCALAR>(a, s);
      if (var == TENSOR2) return launch_apply_line<DIM, N, TENSOR2>(a, s);
      return launch_apply_line<DIM, N, TENSOR4>(a, s);
    case OP_BUILD:
      if (a.fp32) {
        if (var == SCALAR) k_build<DIM, N, SCALAR, float><<<grid, block, sm, s>>>(a);
        else if (var == TENSOR2) k_build<DIM, N, TENSOR2, float><<<grid, block, sm, s>>>(a);
        else k_build<DIM, N, TENSOR4, float><<<grid, block, sm, s>>>(a);
      } else {
        if (var == SCALAR) k_build<DIM, N, SCALAR><<<grid, block, sm, s>>>(a);
        else if (var == TENSOR2) k_build<DIM, N, TENSOR2><<<grid, block, sm, s>>>(a);
        else k_build<DIM, N, TENSOR4><<<grid, block, sm, s>>>(a);
      }
      break;
    case OP_DIAG:
      if (var == SCALAR) k_diag<DIM, N, SCALAR><<<grid, block, sm, s>>>(a);
      else if (var == TENSOR2) k_diag<DIM, N, TENSOR2><<<grid, block, sm, s>>>(a);
      else k_diag<DIM, N, TENSOR4><<<grid, block, sm, s>>>(a);
      break;
    case OP_RESIDUAL:
      k_residual<DIM, N><<<grid, block, sm, s>>>(a);
      break;
    case OP_ENERGY:
      k_energy<DIM, N><<<grid, block, sm, s>>>(a);
      break;
    case OP_JRANGE:
      k_jrange<DIM, N><<<grid, block, sm, s>>>(a, mode, target, first);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace hf
