// hm2.cu -- dispatcher of the packed chain-pair half-step kernels
// (hm2_impl.cuh): picks the instantiation for LPL = KP/32 and padded / dense
// K.  The kernels themselves are instantiated in hm2_k{1,2,4,8}{d,p}.cu.
#include "dmm_internal.cuh"

namespace dmm {
namespace p2 {

template <int LPL, bool PAD>
void launch_win(const PassArgs& a, int vertical, int nframes, cudaStream_t s);

namespace {
constexpr int kCMax = kLeafMax;    // longest leaf block (nodes), as hm2_impl.cuh

int leaf_level(int n) {
    int l = 0;
    while (((n + (1 << l) - 1) >> l) > kCMax) ++l;
    return l;
}

template <int LPL>
void launch_lpl(const PassArgs& a, int vertical, int nframes, cudaStream_t s) {
    if (a.L.K != 32 * LPL) launch_win<LPL, true>(a, vertical, nframes, s);
    else launch_win<LPL, false>(a, vertical, nframes, s);
}
}  // namespace
}  // namespace p2

int hm2_launches_per_pass(const PassArgs& a, int vertical) {
    const int n = vertical ? a.L.H : a.L.W;
    return p2::leaf_level(n) + 1;
}

void launch_hm2_pass(const PassArgs& a, int vertical, int nframes, cudaStream_t s) {
    switch (a.L.KP / 32) {
        case 1: p2::launch_lpl<1>(a, vertical, nframes, s); break;
        case 2: p2::launch_lpl<2>(a, vertical, nframes, s); break;
        case 4: p2::launch_lpl<4>(a, vertical, nframes, s); break;
        default: p2::launch_lpl<8>(a, vertical, nframes, s); break;
    }
}

}  // namespace dmm
