// 2D cell-kernel instantiations: degree 1..8 (n1 = 2..9), n_qpoints = degree+1.
#include "hf_cells_impl.cuh"

namespace hf {

cudaError_t launch_cell_2d(int op, int n1, int var, const CellArgs& a, int mode, double target,
                           unsigned long long* first, cudaStream_t s) {
  switch (n1) {
    case 2: return launch_one<2, 2>(op, var, a, mode, target, first, s);
    case 3: return launch_one<2, 3>(op, var, a, mode, target, first, s);
    case 4: return launch_one<2, 4>(op, var, a, mode, target, first, s);
    case 5: return launch_one<2, 5>(op, var, a, mode, target, first, s);
    case 6: return launch_one<2, 6>(op, var, a, mode, target, first, s);
    case 7: return launch_one<2, 7>(op, var, a, mode, target, first, s);
    case 8: return launch_one<2, 8>(op, var, a, mode, target, first, s);
    case 9: return launch_one<2, 9>(op, var, a, mode, target, first, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hf
