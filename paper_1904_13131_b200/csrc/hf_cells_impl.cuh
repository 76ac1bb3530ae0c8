// Instantiation/dispatch of the cell kernels for one dimension.
#pragma once
#include "hf_dispatch.h"

namespace hf {

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
      if (var == SCALAR) k_apply<DIM, N, SCALAR><<<grid, block, sm, s>>>(a);
      else if (var == TENSOR2) k_apply<DIM, N, TENSOR2><<<grid, block, sm, s>>>(a);
      else k_apply<DIM, N, TENSOR4><<<grid, block, sm, s>>>(a);
      break;
    case OP_BUILD:
      if (var == SCALAR) k_build<DIM, N, SCALAR><<<grid, block, sm, s>>>(a);
      else if (var == TENSOR2) k_build<DIM, N, TENSOR2><<<grid, block, sm, s>>>(a);
      else k_build<DIM, N, TENSOR4><<<grid, block, sm, s>>>(a);
      break;
    case OP_DIAG:
      if (var == SCALAR) k_diag<DIM, N, SCALAR><<<grid, block, sm, s>>>(a);
      else if (var == TENSOR2) k_diag<DIM, N, TENSOR2><<<grid, block, sm, s>>>(a);
      else k_diag<DIM, N, TENSOR4><<<grid, block, sm, s>>>(a);
      break;
    case OP_RESIDUAL:
      k_residual<DIM, N><<<grid, block, sm, s>>>(a);
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
