// Internal launch interface between the C-ABI (hf_api.cu) and the templated
// cell kernels instantiated per dimension (hf_cells2d.cu / hf_cells3d.cu).
#pragma once
#include "hf_cell.cuh"

namespace hf {

enum CellOp { OP_APPLY = 0, OP_BUILD = 1, OP_DIAG = 2, OP_RESIDUAL = 3, OP_JRANGE = 4, OP_ENERGY = 5 };

// Returns cudaErrorInvalidValue when (dim, n1) is not instantiated.
cudaError_t launch_cell_2d(int op, int n1, int var, const CellArgs& a, int mode, double target,
                           unsigned long long* first, cudaStream_t s);
cudaError_t launch_cell_3d(int op, int n1, int var, const CellArgs& a, int mode, double target,
                           unsigned long long* first, cudaStream_t s);
cudaError_t launch_geometry(int dim, const HfTables& tab, const HfLattice& lat, int nq1, const double* verts,
                            double* jinv, double* jxw, unsigned long long* detmin, cudaStream_t s);

// element matrices of the matrix-based baseline (hf_assemble.cu)
cudaError_t launch_assemble(int dim, int n1, const CellArgs& a, double* vals, cudaStream_t s);
cudaError_t launch_cell_dofs(const HfLattice& lat, int dim, int degree, long long* dofs, cudaStream_t s);

// the 3D apply kernels' per-warp timeline (HF_TIMELINE builds, hf_line.cuh):
// HF_TL_WARPS warps x HF_TL_SLOTS timestamps
#define HF_TL_WARPS (148 * 16)
#define HF_TL_SLOTS 72
cudaError_t timeline_copy_3d(unsigned long long* host, int clear);

// blocks per grid and cells per block of the cell kernels
int cells_per_block(int dim, int n1);

}  // namespace hf
