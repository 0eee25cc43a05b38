// egs_kern.cu — the solve kernels (egs_solve.cuh) for one edge-record
// format.  Built twice (Makefile): -DEGS_EDGE_BYTES=8 -DEGS_FMT_NS=e8 and
// -DEGS_EDGE_BYTES=4 -DEGS_FMT_NS=e4; the host driver (egs_solver.cu) picks
// the format per arena and launches through these entry points.
#include "egs_solve.cuh"

namespace egs {
namespace EGS_FMT_NS {

const void* solve_kernel(int vbits) {
  return vbits == 32 ? reinterpret_cast<const void*>(&k_solve<uint32_t>)
                     : reinterpret_cast<const void*>(&k_solve<uint64_t>);
}

}  // namespace EGS_FMT_NS
}  // namespace egs
