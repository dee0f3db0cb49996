// Instantiation of the small-n path for n = 3 (see ks_small_impl.cuh).
#include "ks_small_impl.cuh"

namespace ks {
namespace smalld {
template cudaError_t factor_n<3>(const SmallFactorArgs &, cudaStream_t);
template cudaError_t backward_n<3>(const SmallBackwardArgs &, cudaStream_t);
template cudaError_t whiten_n<3>(const SmallWhitenArgs &, cudaStream_t, int *);
template cudaError_t factor_tail_n<3>(const SmallTailArgs &, cudaStream_t);
template int tail_cols_n<3>();
template cudaError_t backward_tail_n<3>(const SmallBwdTailArgs &, cudaStream_t);
}  // namespace smalld
}  // namespace ks
