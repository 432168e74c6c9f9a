// census.cu -- census transform and Hamming cost volume (Sec. 3.1;
// P:161 "f_i(x_i) = D_i(u(x_i))"), sm_100a.
//
// census_kernel: one thread per pixel, 2-D 32x8 tiles staged through shared
// memory with a replicated (clamped) border of `radius` pixels (reading R17).
// cost_kernel: one CTA per image row; the row's left and right codes are
// staged in shared memory and every thread emits 16 consecutive labels of one
// pixel as a single 16-byte store, so a warp writes 512 contiguous bytes of the
// label-contiguous volume D[y][x][KP] (coalesced, vectorised).
#include "dmm_internal.cuh"

namespace dmm {

constexpr int kTX = 32, kTY = 8, kMaxR = 2;

__global__ void __launch_bounds__(kTX* kTY)
census_kernel(Layout L, int frame0, int radius, long long pitch, const uint8_t* __restrict__ left,
              const uint8_t* __restrict__ right) {
    __shared__ uint8_t tile[2][kTY + 2 * kMaxR][kTX + 2 * kMaxR];
    const int f = frame0 + blockIdx.z;
    FramePtrs P = frame_ptrs(L, f);
    const int W = L.W, H = L.H;
    // images: external (pitch) for the first frame of a call, or the staging copies
    const uint8_t* srcs[2] = {left ? left + (size_t)blockIdx.z * pitch * H : P.img_l,
                              right ? right + (size_t)blockIdx.z * pitch * H : P.img_r};
    const long long pitches[2] = {left ? pitch : (long long)W, right ? pitch : (long long)W};
    const int x0 = blockIdx.x * kTX - radius, y0 = blockIdx.y * kTY - radius;
    const int tw = kTX + 2 * radius, th = kTY + 2 * radius;
    for (int s = 0; s < 2; ++s)
        for (int q = threadIdx.y * kTX + threadIdx.x; q < tw * th; q += kTX * kTY) {
            int yy = min(max(y0 + q / tw, 0), H - 1);
            int xx = min(max(x0 + q % tw, 0), W - 1);
            tile[s][q / tw][q % tw] = srcs[s][(size_t)yy * pitches[s] + xx];
        }
    __syncthreads();
    const int x = blockIdx.x * kTX + threadIdx.x, y = blockIdx.y * kTY + threadIdx.y;
    if (x >= W || y >= H) return;
    for (int s = 0; s < 2; ++s) {
        const int c = tile[s][threadIdx.y + radius][threadIdx.x + radius];
        uint32_t code = 0;
        int bit = 0;
        for (int dy = -radius; dy <= radius; ++dy)
            for (int dx = -radius; dx <= radius; ++dx) {
                if (dx == 0 && dy == 0) continue;
                code |= (uint32_t)(tile[s][threadIdx.y + radius + dy][threadIdx.x + radius + dx] < c)
                        << bit;
                ++bit;
            }
        (s == 0 ? P.codes_l : P.codes_r)[(size_t)y * W + x] = code;
    }
}

void launch_census(const Layout& L, int frame0, int nframes, int radius, int64_t pitch,
                   const uint8_t* left, const uint8_t* right, cudaStream_t s) {
    dim3 grid((L.W + kTX - 1) / kTX, (L.H + kTY - 1) / kTY, nframes);
    census_kernel<<<grid, dim3(kTX, kTY), 0, s>>>(L, frame0, radius, pitch, left, right);
}

// D[y][x][k] = popc(cL[y][x] ^ cR[y][x - d_min - k]) or oob; pads (k >= K) = 0.
__global__ void __launch_bounds__(256) cost_kernel(Layout L, int frame0, int d_min, int oob) {
    extern __shared__ uint32_t srow[];   // [2][W]
    const int f = frame0 + blockIdx.z, y = blockIdx.x;
    FramePtrs P = frame_ptrs(L, f);
    const int W = L.W, K = L.K, KP = L.KP;
    uint32_t* sl = srow;
    uint32_t* sr = srow + W;
    for (int x = threadIdx.x; x < W; x += blockDim.x) {
        sl[x] = P.codes_l[(size_t)y * W + x];
        sr[x] = P.codes_r[(size_t)y * W + x];
    }
    __syncthreads();
    const int chunks = KP / 16;
    uint4* out = reinterpret_cast<uint4*>(P.D + (size_t)y * W * KP);
    // blockIdx.y splits the row's output into gridDim.y contiguous parts
    const int nq = W * chunks, per = (nq + gridDim.y - 1) / gridDim.y;
    const int q0 = blockIdx.y * per, q1 = min(nq, q0 + per);
    for (int q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
        const int x = q / chunks, k0 = (q % chunks) * 16;
        const uint32_t cl = sl[x];
        uint32_t w[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            uint32_t v = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int k = k0 + g * 4 + b;
                const int xr = x - d_min - k;
                uint32_t c = (xr >= 0 && xr < W) ? (uint32_t)__popc(cl ^ sr[xr]) : (uint32_t)oob;
                if (k >= K) c = 0;
                v |= c << (8 * b);
            }
            w[g] = v;
        }
        out[q] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

void launch_cost(const Layout& L, int frame0, int nframes, int d_min, int oob, cudaStream_t s) {
    const size_t smem = 2 * (size_t)L.W * sizeof(uint32_t);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(cost_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cost_kernel<<<dim3(L.H, 4, nframes), 256, smem, s>>>(L, frame0, d_min, oob);
}

}  // namespace dmm
