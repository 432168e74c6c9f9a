// census.cu -- census transform and Hamming cost volume (Sec. 3.1;
// P:161 "f_i(x_i) = D_i(u(x_i))"), sm_100a.
//
// census_kernel: one thread per pixel, 2-D 32x8 tiles staged through shared
// memory with a replicated (clamped) border of `radius` pixels (reading R17).
// cost_kernel: one CTA per 64-pixel tile of a row (any rectangle of the
// frame: the whole frame, or a rank's row / column band); see below.
#include "hm_device.cuh"

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

// D[y][x][k] = popc(cL[y][x] ^ cR[y][x - d_min - k]) or oob; pads (k >= K) = 0,
// over the rectangle [x0, x0 + w) x [y0, y0 + h) of a frame whose codes are
// full-frame rows of W codes; D rows of the rectangle have pitch w*KP.  One CTA
// per (kCostTX-pixel tile, row, frame), one thread per pixel computing all KP
// labels (two threads per pixel, half each, at KP = 256) (per label: one shared load, XOR, POPC, byte packing; the per-CTA
// setup is amortised over KP labels per thread): the right codes the tile can
// reach (kCostTX + KP - 1) are staged in shared memory (consecutive lanes read
// consecutive codes), the labels go to a padded shared tile (row stride KP + 16
// bytes: conflict-free 16-byte stores) that leaves with 16-byte coalesced
// stores -- or, for KP = 256, one TMA bulk store (cp.async.bulk shared ->
// global) per pixel row.  A thread whose samples are all inside the image
// (and K = KP) takes the test-free path; the others (the left ~KP pixels of a
// row, padded K) select oob / 0 per label.  KP is a template parameter.
constexpr int kCostTX = 128;

template <int KP>
constexpr int kCostTPP = KP >= 256 ? 2 : 1;    // threads per pixel (each a contiguous half of the labels)

template <int KP>
__global__ void __launch_bounds__(kCostTX * kCostTPP<KP>)
cost_kernel(const uint32_t* __restrict__ codes_l, const uint32_t* __restrict__ codes_r, size_t code_fstride,
            int W, int K, int d_min, int oob, int x0, int y0, int w, uint8_t* __restrict__ D, size_t d_fstride) {
    constexpr int chunks = KP / 16, stride = KP + 16, NT = kCostTX * kCostTPP<KP>;
    constexpr int cpt = chunks / kCostTPP<KP>;             // 16-label chunks per thread
    __shared__ uint32_t sr[kCostTX + KP];
    __shared__ __align__(16) uint8_t tile[kCostTX * stride];
    const int tx0 = x0 + blockIdx.x * kCostTX;            // first pixel of the tile (frame x)
    const int y = y0 + blockIdx.y;
    const size_t fo = (size_t)blockIdx.z * code_fstride + (size_t)y * W;
    const int npx = min(kCostTX, x0 + w - tx0);
    const int base = tx0 - d_min - (KP - 1);               // frame x of sr[0]
    for (int j = threadIdx.x; j < kCostTX + KP - 1; j += NT) {
        const int xr = base + j;
        sr[j] = (xr >= 0 && xr < W) ? codes_r[fo + xr] : 0u;
    }
    const int px = threadIdx.x % kCostTX, part = threadIdx.x / kCostTX;
    const int x = tx0 + px;
    const uint32_t cl = px < npx ? codes_l[fo + x] : 0u;
    __syncthreads();
    // label k samples x - d_min - k: inside the image for x - d_min - W < k <= x - d_min
    const bool clean = x - d_min >= KP - 1 && x - d_min < W && K == KP;
    const int s0 = px + KP - 1;                            // sr index of label 0 (label k at s0 - k)
#pragma unroll
    for (int cc = 0; cc < cpt; ++cc) {
        const int k0 = 16 * (part * cpt + cc);
        uint32_t wv[4];
        if (clean) {
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                const int sg = s0 - k0 - 4 * g;
                uint32_t v = __popc(cl ^ sr[sg - 3]);
                v = v * 256u + __popc(cl ^ sr[sg - 2]);
                v = v * 256u + __popc(cl ^ sr[sg - 1]);
                wv[g] = v * 256u + __popc(cl ^ sr[sg]);
            }
        } else {
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                uint32_t v = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int k = k0 + g * 4 + b;
                    const int xr = x - d_min - k;
                    DMM_CHECK((unsigned)xr >= (unsigned)W || (xr - base >= 0 && xr - base < kCostTX + KP - 1));
                    const uint32_t cst =
                        (unsigned)xr < (unsigned)W ? (uint32_t)__popc(cl ^ sr[xr - base]) : (uint32_t)oob;
                    v |= (k < K ? cst : 0u) << (8 * b);
                }
                wv[g] = v;
            }
        }
        *reinterpret_cast<uint4*>(tile + px * stride + k0) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
    uint8_t* out = D + (size_t)blockIdx.z * d_fstride + ((size_t)blockIdx.y * w + (tx0 - x0)) * KP;
    if constexpr (KP >= 256) {
        fence_proxy_async();                               // the tile's generic stores -> the async proxy
        __syncthreads();
        if (part == 0 && px < npx) {
            tma_store_s(out + px * KP, (unsigned)__cvta_generic_to_shared(tile + px * stride), KP);
            bulk_commit();
            bulk_wait_read();                              // the tile stays valid until read
        }
    } else {
        __syncthreads();
        uint4* o4 = reinterpret_cast<uint4*>(out);
#pragma unroll 4
        for (int q = threadIdx.x; q < npx * chunks; q += NT) {
            const int p = q / chunks, c = q % chunks;      // compile-time power of two: shifts
            o4[q] = *reinterpret_cast<const uint4*>(tile + p * stride + 16 * c);
        }
    }
}

void launch_cost_rect(const uint32_t* codes_l, const uint32_t* codes_r, size_t code_fstride, int W, int K, int KP,
                      int d_min, int oob, int x0, int y0, int w, int h, uint8_t* D, size_t d_fstride, int nframes,
                      cudaStream_t s) {
    if (w <= 0 || h <= 0) return;
    dim3 grid((w + kCostTX - 1) / kCostTX, h, nframes);
#define DMM_COST_CASE(KPV)                                                                                   \
    case KPV:                                                                                                \
        cost_kernel<KPV><<<grid, kCostTX * kCostTPP<KPV>, 0, s>>>(codes_l, codes_r, code_fstride, W, K, d_min, \
                                                                   oob, x0, y0, w, D, d_fstride);            \
        break;
    switch (KP) {
        DMM_COST_CASE(32)
        DMM_COST_CASE(64)
        DMM_COST_CASE(128)
        default: DMM_COST_CASE(256)
    }
#undef DMM_COST_CASE
}

void launch_cost(const Layout& L, int frame0, int nframes, int d_min, int oob, cudaStream_t s) {
    FramePtrs P = frame_ptrs(L, frame0);
    launch_cost_rect(P.codes_l, P.codes_r, L.frame_bytes / 4, L.W, L.K, L.KP, d_min, oob, 0, 0, L.W, L.H, P.D,
                     L.frame_bytes, nframes, s);
}

}  // namespace dmm
