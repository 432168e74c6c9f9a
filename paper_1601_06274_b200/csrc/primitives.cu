// primitives.cu -- the chain-DP primitives of the hot path exposed on their
// own (include/dmm.h: dmm_msg, dmm_handshake), running exactly the device code
// the Dual MM kernels use (hm_device.cuh): one warp per K-vector.
#include "../../include/dmm.h"
#include "hm_device.cuh"

namespace dmm {

template <int LPL>
__device__ __forceinline__ void ld_dense(const int32_t* p, int K, int lane, int (&v)[LPL]) {
#pragma unroll
    for (int e = 0; e < LPL; ++e) {
        const int k = lane * LPL + e;
        v[e] = k < K ? p[k] : 0;
    }
}
template <int LPL>
__device__ __forceinline__ void st_dense(int32_t* p, int K, int lane, const int (&v)[LPL]) {
#pragma unroll
    for (int e = 0; e < LPL; ++e) {
        const int k = lane * LPL + e;
        if (k < K) p[k] = v[e];
    }
}

template <int LPL, bool PAD, int WIN>
__global__ void msg_batch_kernel(const int32_t* a, int32_t* out, int count, int K, int ws, int wsT) {
    const int v = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (v >= count) return;
    int x[LPL];
    ld_dense<LPL>(a + (size_t)v * K, K, lane, x);
    msg<LPL, PAD, WIN>(x, ws, wsT, lane, K);
    st_dense<LPL>(out + (size_t)v * K, K, lane, x);
}

template <int LPL, bool PAD, int WIN>
__global__ void handshake_batch_kernel(const int32_t* Fi, const int32_t* Fj, const int32_t* pL,
                                       const int32_t* pR, int32_t* oij, int32_t* oji, int count, int K, int ws,
                                       int wsT) {
    const int v = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (v >= count) return;
    const size_t o = (size_t)v * K;
    int fi[LPL], fj[LPL], pl[LPL], pr[LPL];
    ld_dense<LPL>(Fi + o, K, lane, fi);
    ld_dense<LPL>(Fj + o, K, lane, fj);
    ld_dense<LPL>(pL + o, K, lane, pl);
    ld_dense<LPL>(pR + o, K, lane, pr);
    handshake_regs<LPL, PAD, WIN>(fi, fj, pl, pr, ws, wsT, lane, K);
    st_dense<LPL>(oij + o, K, lane, pl);
    st_dense<LPL>(oji + o, K, lane, pr);
}

template <int LPL, bool PAD, int WIN>
static void launch_prim(bool hs, const int32_t* a0, const int32_t* a1, const int32_t* a2, const int32_t* a3,
                        int32_t* o0, int32_t* o1, int count, int K, int ws, int wsT, cudaStream_t s) {
    const int grid = (count + 3) / 4;
    if (hs)
        handshake_batch_kernel<LPL, PAD, WIN><<<grid, 128, 0, s>>>(a0, a1, a2, a3, o0, o1, count, K, ws, wsT);
    else
        msg_batch_kernel<LPL, PAD, WIN><<<grid, 128, 0, s>>>(a0, o0, count, K, ws, wsT);
}

template <int LPL>
static void dispatch(bool hs, const int32_t* a0, const int32_t* a1, const int32_t* a2, const int32_t* a3,
                     int32_t* o0, int32_t* o1, int count, int K, int ws, int T, cudaStream_t s) {
    const bool pad = K != 32 * LPL, win = T <= LPL + 1, t4 = LPL >= 4 && T == 4;
    const int wsT = ws * T;
    if (pad && t4) launch_prim<LPL, true, 4>(hs, a0, a1, a2, a3, o0, o1, count, K, ws, wsT, s);
    else if (pad && win) launch_prim<LPL, true, -1>(hs, a0, a1, a2, a3, o0, o1, count, K, ws, wsT, s);
    else if (pad) launch_prim<LPL, true, 0>(hs, a0, a1, a2, a3, o0, o1, count, K, ws, wsT, s);
    else if (t4) launch_prim<LPL, false, 4>(hs, a0, a1, a2, a3, o0, o1, count, K, ws, wsT, s);
    else if (win) launch_prim<LPL, false, -1>(hs, a0, a1, a2, a3, o0, o1, count, K, ws, wsT, s);
    else launch_prim<LPL, false, 0>(hs, a0, a1, a2, a3, o0, o1, count, K, ws, wsT, s);
}

static dmm_status run(bool hs, const int32_t* a0, const int32_t* a1, const int32_t* a2, const int32_t* a3,
                      int32_t* o0, int32_t* o1, int count, int K, int32_t ws, int32_t T, void* stream) {
    if (count < 0 || K < 1 || K > 256 || ws < 0 || ws > (1 << 16) || T < 1) return DMM_E_ARG;
    if (count == 0) return DMM_OK;
    if (T > K) T = K;     // min(|a-b|, T) with |a-b| <= K-1: T >= K is untruncated
    cudaStream_t s = (cudaStream_t)stream;
    const int lpl = K <= 32 ? 1 : K <= 64 ? 2 : K <= 128 ? 4 : 8;
    switch (lpl) {
        case 1: dispatch<1>(hs, a0, a1, a2, a3, o0, o1, count, K, ws, T, s); break;
        case 2: dispatch<2>(hs, a0, a1, a2, a3, o0, o1, count, K, ws, T, s); break;
        case 4: dispatch<4>(hs, a0, a1, a2, a3, o0, o1, count, K, ws, T, s); break;
        default: dispatch<8>(hs, a0, a1, a2, a3, o0, o1, count, K, ws, T, s); break;
    }
    return cudaGetLastError() == cudaSuccess ? DMM_OK : DMM_E_CUDA;
}

}  // namespace dmm

extern "C" {

dmm_status dmm_msg(const int32_t* a, int32_t* out, int count, int K, int32_t ws, int32_t T, void* stream) {
    if (!a || !out) return count == 0 ? DMM_OK : DMM_E_ARG;
    return dmm::run(false, a, nullptr, nullptr, nullptr, out, nullptr, count, K, ws, T, stream);
}

dmm_status dmm_handshake(const int32_t* Fi, const int32_t* Fj, const int32_t* phiL, const int32_t* phiR,
                         int32_t* phi_ij, int32_t* phi_ji, int count, int K, int32_t ws, int32_t T,
                         void* stream) {
    if (!Fi || !Fj || !phiL || !phiR || !phi_ij || !phi_ji) return count == 0 ? DMM_OK : DMM_E_ARG;
    return dmm::run(true, Fi, Fj, phiL, phiR, phi_ij, phi_ji, count, K, ws, T, stream);
}

}  // extern "C"
