// Stand-in for the one reference routine that needs Eigen (absent from this
// image): dense_solve (/root/reference/proj/src/reference.cpp:48-64).  It is
// off the fast-matvec path; the stub throws so imq_dense_solve reports an error.
// Compiled only into oracle/_ref/ (test infrastructure, never shipped).
#include <stdexcept>
#include <vector>
#include "imq/reference.hpp"
namespace imq {
DenseSolveResult dense_solve(const DenseMatrix&, const std::vector<double>&) {
  throw std::runtime_error("dense_solve: Eigen is not available in this build of the reference");
}
}  // namespace imq
