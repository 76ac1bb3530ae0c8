// 3D cell-kernel instantiations: degree 1..4 (n1 = 2..5), n_qpoints = degree+1.
#include "hf_cells_impl.cuh"

namespace hf {

cudaError_t launch_cell_3d(int op, int n1, int var, const CellArgs& a, int mode, double target,
                           unsigned long long* first, cudaStream_t s) {
  switch (n1) {
    case 2: return launch_one<3, 2>(op, var, a, mode, target, first, s);
    case 3: return launch_one<3, 3>(op, var, a, mode, target, first, s);
    case 4: return launch_one<3, 4>(op, var, a, mode, target, first, s);
    case 5: return launch_one<3, 5>(op, var, a, mode, target, first, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_geometry(int dim, const HfTables& tab, const HfLattice& lat, int nq1, const double* verts,
                            double* jinv, double* jxw, unsigned long long* detmin, cudaStream_t s) {
  if (lat.n_qp == 0) return cudaSuccess;
  unsigned nb = (unsigned)((lat.n_qp + 255) / 256);
  if (dim == 2) k_geometry<2><<<nb, 256, 0, s>>>(tab, lat, nq1, verts, jinv, jxw, detmin);
  else k_geometry<3><<<nb, 256, 0, s>>>(tab, lat, nq1, verts, jinv, jxw, detmin);
  return cudaGetLastError();
}

cudaError_t timeline_copy_3d(unsigned long long* host, int clear) {
#ifdef HF_TIMELINE
  cudaError_t e = cudaMemcpyFromSymbol(host, hf_tl_buf, sizeof(unsigned long long) * HF_TL_WARPS * HF_TL_SLOTS);
  if (e != cudaSuccess || !clear) return e;
  static unsigned long long zero[HF_TL_WARPS * HF_TL_SLOTS];
  return cudaMemcpyToSymbol(hf_tl_buf, zero, sizeof(zero));
#else
  (void)host;
  (void)clear;
  return cudaErrorNotSupported;
#endif
}

int cells_per_block(int dim, int n1) {
  int nq = dim == 2 ? n1 * n1 : n1 * n1 * n1;
  return (256 / nq) > 0 ? 256 / nq : 1;
}

}  // namespace hf
