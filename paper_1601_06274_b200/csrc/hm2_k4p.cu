// One explicit instantiation set of the packed chain-pair kernels
// (hm2_impl.cuh): LPL = 4 labels per lane, padded K.  Split per
// translation unit so the kernels compile in parallel.
#include "hm2_impl.cuh"

namespace dmm {
namespace p2 {
template void launch_win<4, true>(const PassArgs&, int, int, cudaStream_t);
}  // namespace p2
}  // namespace dmm
