// One explicit instantiation set of the int32 chain-DP kernels (hm_impl.cuh):
// LPL = 1 labels per lane, dense K.  Split per translation unit so the
// kernels compile in parallel.
#include "hm_impl.cuh"

namespace dmm {
template void hm_launch_win<1, false>(const PassArgs&, int, int, cudaStream_t);
}  // namespace dmm
