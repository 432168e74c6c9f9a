// flow.cu -- the discrete stage of optical flow (NEXT-1):
// optimistic decoupled data costs of the 2-D label window (Eq. "flow
// decoupled costs"; Sec. 3.2),
//   f1(a) = min_b D(a,b),  f2(b) = min_a D(a,b),
//   D(a,b) = popcount(c1(x,y) ^ c2(x + u1(a), y + u2(b))), oob outside the image,
// with u1(a) = u1_min + a, u2(b) = u2_min + b (a, b < K), computed by one fused
// kernel that never materialises the K*K volume: each thread evaluates the
// K*K Hamming distances of two vertically adjacent pixels from a
// shared-memory tile of the second image's census codes (pixel (x, y+1)'s
// window row b is pixel (x, y)'s row b+1, so one shared load serves both) and
// keeps f1 as packed bytes (__vminu4) and f2 as a running minimum.  The two
// layers land in two frames of one context, which then solves them as two
// independent K-label Dual MM problems in the same launches ("decouple into
// two independent stereo-like problems").
#include "dmm_internal.cuh"

namespace dmm {

constexpr int kFTX = 32, kFTY = 8;      // threads: 32 x 8, each 2 pixels stacked -> 32 x 16 pixel tile

template <int K, bool FAST>
__device__ __forceinline__ void flow_pixels(const uint32_t* sr, int SW, int ty, int px, int x, int y0, int W, int H,
                                            int KP, int u1_min, int u2_min, int oob, const uint32_t* __restrict__ c1,
                                            uint8_t* __restrict__ D1, uint8_t* __restrict__ D2) {
    const uint32_t cA = c1[(size_t)y0 * W + x];
    const bool hasB = y0 + 1 < H;
    const uint32_t cB = hasB ? c1[(size_t)(y0 + 1) * W + x] : 0u;
    uint32_t f1A[K / 4], f1B[K / 4], f2A[K / 4], f2B[K / 4];
#pragma unroll
    for (int j = 0; j < K / 4; ++j) { f1A[j] = f1B[j] = 0xffffffffu; f2A[j] = f2B[j] = 0u; }
    uint32_t keepx[K / 4];     // general path: bytes whose displaced column is inside the image
    if constexpr (!FAST) {
#pragma unroll
        for (int j = 0; j < K / 4; ++j) {
            uint32_t k = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) k |= ((unsigned)(x + u1_min + 4 * j + e) < (unsigned)W ? 0xffu : 0u) << (8 * e);
            keepx[j] = k;
        }
    }
    const uint32_t oobP = (uint32_t)oob * 0x01010101u;
    // window row r of the shared tile serves pixel A at b = r and pixel B at b = r - 1
#pragma unroll 1
    for (int r = 0; r <= K; ++r) {
        const uint32_t* row = sr + (2 * ty + r) * SW + px;
        bool vy = true;
        if constexpr (!FAST) vy = (unsigned)(y0 + u2_min + r) < (unsigned)H;   // same frame row for A (b=r), B (b=r-1)
        uint32_t mA = 0xffu, mB = 0xffu;
#pragma unroll
        for (int j = 0; j < K / 4; ++j) {
            uint32_t dA = 0, dB = 0;
#pragma unroll
            for (int e = 3; e >= 0; --e) {
                const uint32_t code = row[4 * j + e];
                dA = dA * 256u + __popc(cA ^ code);
                dB = dB * 256u + __popc(cB ^ code);
            }
            if constexpr (!FAST) {
                const uint32_t keep = vy ? keepx[j] : 0u;
                dA = (dA & keep) | (oobP & ~keep);
                dB = (dB & keep) | (oobP & ~keep);
            }
            if (r < K) {
                f1A[j] = __vminu4(f1A[j], dA);
                mA = min(mA, min(min(dA & 0xffu, (dA >> 8) & 0xffu), min((dA >> 16) & 0xffu, dA >> 24)));
            }
            if (r > 0) {
                f1B[j] = __vminu4(f1B[j], dB);
                mB = min(mB, min(min(dB & 0xffu, (dB >> 8) & 0xffu), min((dB >> 16) & 0xffu, dB >> 24)));
            }
        }
        if (r < K) f2A[r >> 2] |= mA << (8 * (r & 3));
        if (r > 0) f2B[(r - 1) >> 2] |= mB << (8 * ((r - 1) & 3));
    }
    auto put = [&](uint8_t* D, int y, const uint32_t (&v)[K / 4]) {
        uint4* o = reinterpret_cast<uint4*>(D + ((size_t)y * W + x) * KP);
#pragma unroll
        for (int j = 0; j < K / 16; ++j) o[j] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        for (int j = K / 16; j < KP / 16; ++j) o[j] = make_uint4(0u, 0u, 0u, 0u);
    };
    put(D1, y0, f1A);
    put(D2, y0, f2A);
    if (hasB) {
        put(D1, y0 + 1, f1B);
        put(D2, y0 + 1, f2B);
    }
}

template <int K>
__global__ void __launch_bounds__(kFTX* kFTY)
flow_cost_kernel(const uint32_t* __restrict__ c1, const uint32_t* __restrict__ c2, int W, int H, int KP, int u1_min,
                 int u2_min, int oob, uint8_t* __restrict__ D1, uint8_t* __restrict__ D2) {
    extern __shared__ uint32_t sr[];     // [2*kFTY + K][kFTX + K - 1]
    constexpr int SW = kFTX + K - 1, SH = 2 * kFTY + K;
    const int tx0 = blockIdx.x * kFTX, ty0 = blockIdx.y * 2 * kFTY;
    const int bx = tx0 + u1_min, by = ty0 + u2_min;       // frame coordinates of sr[0][0]
    for (int q = threadIdx.y * kFTX + threadIdx.x; q < SW * SH; q += kFTX * kFTY) {
        const int r = q / SW, cc = q - r * SW;
        const int ys = by + r, xs = bx + cc;
        sr[q] = (ys >= 0 && ys < H && xs >= 0 && xs < W) ? c2[(size_t)ys * W + xs] : 0u;
    }
    __syncthreads();
    const int px = threadIdx.x, x = tx0 + px;
    const int y0 = ty0 + 2 * threadIdx.y;
    if (x >= W || y0 >= H) return;
    // CTA-uniform: the whole window region of the tile inside the image -> no checks
    const bool fast = bx >= 0 && bx + SW <= W && by >= 0 && by + SH <= H;
    if (fast)
        flow_pixels<K, true>(sr, SW, threadIdx.y, px, x, y0, W, H, KP, u1_min, u2_min, oob, c1, D1, D2);
    else
        flow_pixels<K, false>(sr, SW, threadIdx.y, px, x, y0, W, H, KP, u1_min, u2_min, oob, c1, D1, D2);
}

template <int K>
static void launch_k(const uint32_t* c1, const uint32_t* c2, int W, int H, int KP, int u1_min, int u2_min, int oob,
                     uint8_t* D1, uint8_t* D2, cudaStream_t s) {
    const int smem = (2 * kFTY + K) * (kFTX + K - 1) * 4;
    static int set = 0;
    if (!set) {
        cudaFuncSetAttribute(flow_cost_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        set = 1;
    }
    dim3 grid((W + kFTX - 1) / kFTX, (H + 2 * kFTY - 1) / (2 * kFTY));
    flow_cost_kernel<K><<<grid, dim3(kFTX, kFTY), smem, s>>>(c1, c2, W, H, KP, u1_min, u2_min, oob, D1, D2);
}

bool flow_k_ok(int K) { return K == 16 || K == 32 || K == 48 || K == 64; }

void launch_flow_costs(const uint32_t* c1, const uint32_t* c2, int W, int H, int K, int KP, int u1_min, int u2_min,
                       int oob, uint8_t* D1, uint8_t* D2, cudaStream_t s) {
    switch (K) {
        case 16: launch_k<16>(c1, c2, W, H, KP, u1_min, u2_min, oob, D1, D2, s); break;
        case 32: launch_k<32>(c1, c2, W, H, KP, u1_min, u2_min, oob, D1, D2, s); break;
        case 48: launch_k<48>(c1, c2, W, H, KP, u1_min, u2_min, oob, D1, D2, s); break;
        default: launch_k<64>(c1, c2, W, H, KP, u1_min, u2_min, oob, D1, D2, s); break;
    }
}

}  // namespace dmm
