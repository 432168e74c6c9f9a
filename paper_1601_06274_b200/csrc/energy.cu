// energy.cu -- primal energy of the labelling (Eq.3, with f_i = D_i
// and f_ij = w*min(|x_i - x_j|, T)), exact int64, scaled by 2^F; plus
// the de-padding copies used by the parity taps.
#include "dmm_internal.cuh"

namespace dmm {

__global__ void __launch_bounds__(256)
energy_kernel(Layout L, int frame0, int w_h, int w_v, int T, int fbits, const uint8_t* __restrict__ ext,
              int32_t* bad) {
    FramePtrs P = frame_ptrs(L, frame0 + blockIdx.y);
    const int W = L.W, H = L.H, KP = L.KP, K = L.K;
    const uint8_t* __restrict__ lab = ext ? ext : P.labels;
    long long e = 0;
    bool oob = false;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < W * H; q += gridDim.x * blockDim.x) {
        const int y = q / W, x = q - y * W;
        const int l = lab[q];
        oob |= l >= K;
        e += P.D[(size_t)q * KP + min(l, K - 1)];
        if (x + 1 < W) e += (long long)w_h * min(abs(l - (int)lab[q + 1]), T);
        if (y + 1 < H) e += (long long)w_v * min(abs(l - (int)lab[q + W]), T);
    }
    if (oob && bad) *bad = 1;
    for (int d = 16; d > 0; d >>= 1) e += __shfl_down_sync(kFull, e, d);
    __shared__ long long part[8];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long s = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[w];
        atomicAdd(reinterpret_cast<unsigned long long*>(P.energy), (unsigned long long)(s << fbits));
    }
}

void launch_energy(const Layout& L, int frame0, int nframes, int w_h, int w_v, int T, int fbits,
                   const uint8_t* labels, int32_t* bad, cudaStream_t s) {
    int blocks = (L.W * L.H + 255) / 256;
    if (blocks > 4 * 148) blocks = 4 * 148;
    energy_kernel<<<dim3(blocks, nframes), 256, 0, s>>>(L, frame0, w_h, w_v, T, fbits, labels, bad);
}

template <typename T>
__global__ void unpad_kernel(const T* __restrict__ src, T* __restrict__ dst, long long cells, int K,
                             int KP) {
    const long long n = cells * K;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long c = i / K;
        dst[i] = src[c * KP + (i - c * K)];
    }
}

void launch_unpad_u8(const uint8_t* src, uint8_t* dst, long long cells, int K, int KP, cudaStream_t s) {
    unpad_kernel<uint8_t><<<4 * 148, 256, 0, s>>>(src, dst, cells, K, KP);
}
__global__ void pad_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, long long cells, int K,
                           int KP) {
    const long long n = cells * KP;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long c = i / KP;
        const int k = (int)(i - c * KP);
        dst[i] = k < K ? src[c * K + k] : 0;
    }
}

void launch_pad_u8(const uint8_t* src, uint8_t* dst, long long cells, int K, int KP, cudaStream_t s) {
    pad_kernel<<<4 * 148, 256, 0, s>>>(src, dst, cells, K, KP);
}

__global__ void decode_rec_kernel(const uint8_t* __restrict__ rec, const uint8_t* __restrict__ D, int fbits,
                                  int32_t* __restrict__ dst, long long cells, int K, int KP) {
    const int R = rec_bytes(KP);
    const long long n = cells * K;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long c = i / K;
        const int k = (int)(i - c * K);
        const uint8_t* r = rec + c * R;
        int v = *reinterpret_cast<const int32_t*>(r + 2 * KP) + reinterpret_cast<const uint16_t*>(r)[k];
        if (D) v -= (int)D[c * KP + k] << fbits;
        dst[i] = v;
    }
}

__global__ void decode_dense_kernel(const int32_t* __restrict__ src, const uint8_t* __restrict__ D, int fbits,
                                    int32_t* __restrict__ dst, long long cells, int K, int KP) {
    const long long n = cells * K;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long c = i / K;
        const int k = (int)(i - c * K);
        int v = src[c * KP + k];
        if (D) v -= (int)D[c * KP + k] << fbits;
        dst[i] = v;
    }
}

void launch_decode_dense(const int32_t* src, const uint8_t* D, int fbits, int32_t* dst, long long cells, int K, int KP,
                         cudaStream_t s) {
    decode_dense_kernel<<<4 * 148, 256, 0, s>>>(src, D, fbits, dst, cells, K, KP);
}

void launch_decode_rec(const uint8_t* rec, const uint8_t* D, int fbits, int32_t* dst, long long cells, int K,
                       int KP, cudaStream_t s) {
    decode_rec_kernel<<<4 * 148, 256, 0, s>>>(rec, D, fbits, dst, cells, K, KP);
}

}  // namespace dmm
