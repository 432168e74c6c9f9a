// hm.cu -- dispatcher of the int32 chain-DP half-step kernels (hm_impl.cuh):
// picks the instantiation for LPL = KP/32 and padded / dense K.  The kernels
// themselves are instantiated in hm_k{1,2,4,8}{d,p}.cu.
#include "dmm_internal.cuh"

namespace dmm {

template <int LPL, bool PAD>
void hm_launch_win(const PassArgs& a, int vertical, int nframes, cudaStream_t s);

namespace {
constexpr int kCMax = 12;    // longest leaf block (nodes), as hm_impl.cuh

int leaf_level(int n) {
    int l = 0;
    while (((n + (1 << l) - 1) >> l) > kCMax) ++l;
    return l;
}

template <int LPL>
void launch_lpl(const PassArgs& a, int vertical, int nframes, cudaStream_t s) {
    if (a.L.K != 32 * LPL) hm_launch_win<LPL, true>(a, vertical, nframes, s);
    else hm_launch_win<LPL, false>(a, vertical, nframes, s);
}
}  // namespace

int hm_launches_per_pass(const PassArgs& a, int vertical, int /*wave*/) {
    const int n = vertical ? a.L.H : a.L.W;
    return leaf_level(n) + 1;      // root + levels 1..l*-1 + leaf blocks
}

void launch_hm_pass(const PassArgs& a, int vertical, int nframes, int /*wave*/, cudaStream_t s) {
    switch (a.L.KP / 32) {
        case 1: launch_lpl<1>(a, vertical, nframes, s); break;
        case 2: launch_lpl<2>(a, vertical, nframes, s); break;
        case 4: launch_lpl<4>(a, vertical, nframes, s); break;
        default: launch_lpl<8>(a, vertical, nframes, s); break;
    }
}

}  // namespace dmm
