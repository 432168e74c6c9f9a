// refine.cu -- continuous refinement of the discrete labelling (NEXT-2, SURVEY
// 8(f)): the non-convex primal-dual method of Sec. 2.4 with the
// two-slope data approximation of Sec. 3.1 for stereo, or the
// quadratic model of Eq. 19 and the prox of Eq. 20 for flow (Sec. 3.2,
// P:449-467), in float64.
//
//   u+ = prox_{tau D~}(u - tau A^T (p - q))            (Eq. cont_iterates, P:306-311,
//   q+ = prox_{tau R_-^*}(q + tau A u)                   grad A of P:350-355, d = 1)
//   p+ = prox_{sigma R_+^*}(p + sigma A(2 u+ - u))
//   prox of (w r_{a,b})^*: Eq. pprox; r = r_{eps,delta} - r_{0,C+delta-eps delta}
//   (Eq. r-decompose); data prox P:431-440; warping P:441.
// Readings R24-R28 as the oracle (oracle/refine.py).
//
// Per pixel state (double [H][W] each): u, p_h, p_v, q_h, q_v (two buffers
// each: every launch reads one and writes the other, so no thread reads a
// value another thread of the same launch updates), u0 (expansion point), s1,
// s2 (slopes); edge arrays are indexed by the edge's first pixel.  The
// iterations run kHalo at a time in refine_tile_kernel / flow_tile_kernel
// (temporal blocking on chip); the state (112 B/pixel, 52 MB at C2) stays
// L2-resident across launches.  A warp's launches are captured once into a
// CUDA graph per (frame, parameters) and replayed.
#include <cmath>
#include <cstring>

#include "ctx.cuh"

namespace dmm {

namespace {

constexpr int kRX = 32, kRY = 8;
// u (buffers 0, 1), u0 (expansion point), s1, s2 (flow: L, Q_kk), then per
// buffer b: ph, pv, qh, qv at 5 + 4b; 13: flow's Q_12 (first component's area)
constexpr int kRefArrays = 14;
using real = double;             // float64, the oracle's precision

struct RefArgs {
    real* rf;            // kRefArrays x [H][W]
    const uint8_t* D;    // [H][W][KP]
    const uint8_t* labels;
    int W, H, K, KP;
    real wh, wv, eps, delta, C, h, tau, sigma;
};

__device__ __forceinline__ real* arr(const RefArgs& a, int k) { return a.rf + (size_t)k * a.W * a.H; }

// D at a real label (reading R26): linear interpolation, label clamped to [0, K-1]
__device__ __forceinline__ real d_interp(const uint8_t* Dp, int K, real u) {
    const real uc = fmin(fmax(u, 0.0), (real)(K - 1));
    const int k0 = min((int)floor(uc), K - 1);
    const int k1 = min(k0 + 1, K - 1);
    const real f = uc - (real)k0;
    return (1.0 - f) * (real)Dp[k0] + f * (real)Dp[k1];
}


__device__ __forceinline__ real r_dc(real t, real eps, real delta, real C) {
    const real at = fabs(t);
    const real bp = C + delta - eps * delta;
    const real rp = at <= delta ? eps * at : at - delta * (1.0 - eps);
    const real rm = at <= bp ? 0.0 : at - bp;
    return rp - rm;
}

__global__ void refine_init_kernel(RefArgs a) {
    const int x = blockIdx.x * kRX + threadIdx.x, y = blockIdx.y * kRY + threadIdx.y;
    if (x >= a.W || y >= a.H) return;
    const size_t i = (size_t)y * a.W + x;
    arr(a, 0)[i] = (real)a.labels[i];
    for (int k = 5; k < kRefArrays; ++k) arr(a, k)[i] = 0.0;
}

// a new expansion point: u0 = u, two-slope approximation (R24)
__global__ void refine_warp_kernel(RefArgs a) {
    const int x = blockIdx.x * kRX + threadIdx.x, y = blockIdx.y * kRY + threadIdx.y;
    if (x >= a.W || y >= a.H) return;
    const size_t i = (size_t)y * a.W + x;
    const real u0 = arr(a, 0)[i];
    const uint8_t* Dp = a.D + i * a.KP;
    const real dc = d_interp(Dp, a.K, u0);
    real s1 = (dc - d_interp(Dp, a.K, u0 - a.h)) / a.h;
    real s2 = (d_interp(Dp, a.K, u0 + a.h) - dc) / a.h;
    if (s2 < s1) { const real m = 0.5 * (s1 + s2); s1 = m; s2 = m; }
    arr(a, 2)[i] = u0;
    arr(a, 3)[i] = s1;
    arr(a, 4)[i] = s2;
}

// One PDHG iteration (Eq. cont_iterates), per pixel i (edges indexed by their
// first pixel, reading buffer cur, writing 1 - cur):
//   u+_i = clip(prox_{tau D~}(u_i - tau (A^T (p - q))_i), u0_i - h, u0_i + h)
//          (two slopes P:431-440, R25; or the quadratic of flow, Eq. 19/20, R34)
//   q+_e = prox_{tau R_-^*}(q_e + tau (A u)_e)
//   p+_e = prox_{sigma R_+^*}(p_e + sigma (A (2 u+ - u))_e)
// in the oracle's operation order (oracle/refine.py refine / flow_refine).
//
// Temporal blocking: one launch runs nt <= kHalo iterations on a kTX x TY
// tile held on chip, writing back only the inner (kTX - 2 kHalo) x
// (TY - 2 kHalo) pixels.  Every iteration's dependence cone has Chebyshev
// radius 1 (u+ at j reads the duals of j's left / upper edges; p+, q+ of i's
// edges read u, u+ at i's right / lower neighbour), so after nt iterations
// the values at distance >= nt from the tile border are exactly those of nt
// single-iteration sweeps: the same operations in the same order on the same
// operands (bit-exact, -fmad=false).  Each thread
// owns TPX pixels of one column: its u, u0, s1 / s2 (or L / Q) and its
// edges' p, q live in registers; shared memory holds what neighbours read:
// u (two buffers: before / after the primal step) and p - q per direction
// (the operand A^T(p - q) consumes; the subtraction is the one the iteration
// kernel does).  Outside the image a pixel is inert; a term whose neighbour is
// off the tile is dropped (the apron's garbage, never reaching the inner tile).
// Stereo tile 64 x 40, 5 pixels per thread: 276 CTAs of 512 threads at C2,
// under two waves of 148 SMs (measured against 64 x 32 / 4 and 64 x 48 / 6)
constexpr int kTX = 64, kHalo = 4, kTY = 40, kTPX = 5;
constexpr int kTileThreads = kTX * kTY / kTPX, kOX = kTX - 2 * kHalo, kOY = kTY - 2 * kHalo;
constexpr size_t kTileSmem = 5 * sizeof(real) * kTX * kTY;

// max / min / clip as numpy evaluates them on non-NaN operands (a compare and
// a select; the libm fmax / fmin add NaN handling the finite iterates never need)
__device__ __forceinline__ real dmax(real a, real b) { return a > b ? a : b; }
__device__ __forceinline__ real dmin(real a, real b) { return a < b ? a : b; }
__device__ __forceinline__ real dclip(real v, real lo, real hi) { return dmin(dmax(v, lo), hi); }

// prox of step * (w r_{a,b})^* (Eq. pprox) with its loop-invariant
// products hoisted: aw = a * w, bs = b * step
__device__ __forceinline__ real prox_conj_h(real t, real w, real aw, real bs) {
    const real at = fabs(t);
    const real tp = at <= aw ? t : copysign(dmax(aw, at - bs), t);
    return dclip(tp, -w, w);
}

__global__ void __launch_bounds__(kTileThreads) refine_tile_kernel(RefArgs a, int cur, int nt) {
    extern __shared__ real tsm[];            // u [2][kTY][kTX], bi, p_h - q_h, p_v - q_v
    real* sbi = tsm + 2 * kTX * kTY;
    real* sdh = tsm + 3 * kTX * kTY;
    real* sdv = tsm + 4 * kTX * kTY;
    const int W = a.W, H = a.H;
    const real tau = a.tau, sigma = a.sigma, h = a.h, wh = a.wh, wv = a.wv;
    const real bp = a.C + a.delta - a.eps * a.delta;
    // the products prox_conj forms from its constant arguments, formed once
    const real q_awh = 0.0 * wh, q_awv = 0.0 * wv, q_bs = bp * tau;
    const real p_awh = a.eps * wh, p_awv = a.eps * wv, p_bs = a.delta * sigma;
    const int lx = threadIdx.x % kTX, ly0 = (threadIdx.x / kTX) * kTPX;
    const int gx = blockIdx.x * kOX - kHalo + lx, gy0 = blockIdx.y * kOY - kHalo + ly0;
    const int b0 = 5 + 4 * cur, b1 = 5 + 4 * (1 - cur);
    const bool inx = gx >= 0 && gx < W;
    const bool hasr = gx + 1 < W && lx + 1 < kTX, hasl = gx > 0 && lx > 0, inr = gx + 1 < W;
    // per pixel: u, the data prox's constants c1 = tau s1, c2 = tau s2 (its
    // own subexpressions), u0, the duals of the pixel's two edges
    real u[kTPX], u0[kTPX], c1[kTPX], c2[kTPX], ph[kTPX], pv[kTPX], qh[kTPX], qv[kTPX], un[kTPX];
#pragma unroll
    for (int r = 0; r < kTPX; ++r) {
        const int gy = gy0 + r, l = (ly0 + r) * kTX + lx;
        u[r] = u0[r] = c1[r] = c2[r] = ph[r] = pv[r] = qh[r] = qv[r] = 0.0;
        if (inx && gy >= 0 && gy < H) {
            const size_t i = (size_t)gy * W + gx;
            u[r] = arr(a, cur)[i];
            u0[r] = arr(a, 2)[i];
            c1[r] = tau * arr(a, 3)[i];
            c2[r] = tau * arr(a, 4)[i];
            ph[r] = arr(a, b0)[i];
            pv[r] = arr(a, b0 + 1)[i];
            qh[r] = arr(a, b0 + 2)[i];
            qv[r] = arr(a, b0 + 3)[i];
        }
        tsm[l] = u[r];
        sdh[l] = ph[r] - qh[r];
        sdv[l] = pv[r] - qv[r];
    }
    __syncthreads();
    // all kTPX pixels are computed unconditionally (independent chains the
    // scheduler interleaves); a pixel off the image computes on zeros and is
    // never read by an image pixel (the neighbour tests are the image's)
    for (int t = 0; t < nt; ++t) {
        const real* uo = tsm + (t & 1) * (kTX * kTY);
        real* us = tsm + ((t + 1) & 1) * (kTX * kTY);
        real bi[kTPX];
#pragma unroll
        for (int r = 0; r < kTPX; ++r) {          // primal step
            const int gy = gy0 + r, ly = ly0 + r, l = ly * kTX + lx;
            real div = 0.0;
            if (inr) div += ph[r] - qh[r];
            if (hasl) div -= sdh[l - 1];
            if (gy + 1 < H) div += pv[r] - qv[r];
            if (gy > 0 && ly > 0) div -= sdv[l - kTX];
            const real uh = u[r] - tau * div;
            const real v = uh > u0[r] + c2[r] ? uh - c2[r] : (uh < u0[r] + c1[r] ? uh - c1[r] : u0[r]);
            un[r] = dclip(v, u0[r] - h, u0[r] + h);
            bi[r] = 2.0 * un[r] - u[r];
            us[l] = un[r];
            sbi[l] = bi[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kTPX; ++r) {          // dual steps of the pixel's own edges
            const int gy = gy0 + r, ly = ly0 + r, l = ly * kTX + lx;
            // a neighbour's 2 u+ - u is its own bi (the same operations on the
            // same operands).  Computed branch-free and selected: an absent
            // edge keeps its dual (its operands, read past the row / tile end,
            // stay inside the shared allocation and are discarded)
            const bool hasd = gy + 1 < H && ly + 1 < kTY;
            const real ur = uo[l + 1], ud = uo[l + kTX];
            const real nqh = prox_conj_h(qh[r] + tau * (u[r] - ur), wh, q_awh, q_bs);
            const real nph = prox_conj_h(ph[r] + sigma * (bi[r] - sbi[l + 1]), wh, p_awh, p_bs);
            const real nqv = prox_conj_h(qv[r] + tau * (u[r] - ud), wv, q_awv, q_bs);
            const real npv = prox_conj_h(pv[r] + sigma * (bi[r] - sbi[l + kTX]), wv, p_awv, p_bs);
            qh[r] = hasr ? nqh : qh[r];
            ph[r] = hasr ? nph : ph[r];
            qv[r] = hasd ? nqv : qv[r];
            pv[r] = hasd ? npv : pv[r];
            u[r] = un[r];
        }
        // the next primal step reads the neighbours' p - q (and rewrites `uo`
        // and bi) only after the barrier below
#pragma unroll
        for (int r = 0; r < kTPX; ++r) {
            const int l = (ly0 + r) * kTX + lx;
            sdh[l] = ph[r] - qh[r];
            sdv[l] = pv[r] - qv[r];
        }
        __syncthreads();
    }
    if (!inx || lx < kHalo || lx >= kTX - kHalo) return;
#pragma unroll
    for (int r = 0; r < kTPX; ++r) {
        const int gy = gy0 + r, ly = ly0 + r;
        if (gy < 0 || gy >= H || ly < kHalo || ly >= kTY - kHalo) continue;
        const size_t i = (size_t)gy * W + gx;
        arr(a, 1 - cur)[i] = u[r];
        if (inr) {
            arr(a, b1)[i] = ph[r];
            arr(a, b1 + 2)[i] = qh[r];
        }
        if (gy + 1 < H) {
            arr(a, b1 + 1)[i] = pv[r];
            arr(a, b1 + 3)[i] = qv[r];
        }
    }
}

__global__ void refine_swap_kernel(RefArgs a) {     // odd iteration count: the state back to buffer 0
    const int x = blockIdx.x * kRX + threadIdx.x, y = blockIdx.y * kRY + threadIdx.y;
    if (x >= a.W || y >= a.H) return;
    const size_t i = (size_t)y * a.W + x;
    arr(a, 0)[i] = arr(a, 1)[i];
    for (int k = 0; k < 4; ++k) arr(a, 5 + k)[i] = arr(a, 9 + k)[i];
}

// output (disparity units) and the energy E(u) = D(u) + R(Au), double accumulation
__global__ void refine_out_kernel(RefArgs a, real d_min, float* out, double* energy) {
    const int x = blockIdx.x * kRX + threadIdx.x, y = blockIdx.y * kRY + threadIdx.y;
    double e = 0.0;
    if (x < a.W && y < a.H) {
        const int W = a.W;
        const size_t i = (size_t)y * W + x;
        const real* u = arr(a, 0);
        const real ui = u[i];
        if (out) out[i] = (float)(d_min + ui);
        e = d_interp(a.D + i * a.KP, a.K, ui);
        if (x + 1 < W) e += a.wh * r_dc(ui - u[i + 1], a.eps, a.delta, a.C);
        if (y + 1 < a.H) e += a.wv * r_dc(ui - u[i + W], a.eps, a.delta, a.C);
    }
    for (int d = 16; d > 0; d >>= 1) e += __shfl_down_sync(0xffffffffu, e, d);
    __shared__ double part[kRX * kRY / 32];
    const int t = threadIdx.y * kRX + threadIdx.x;
    if ((t & 31) == 0) part[t >> 5] = e;
    __syncthreads();
    if (t == 0 && energy) {
        double s = 0.0;
        for (int k = 0; k < kRX * kRY / 32; ++k) s += part[k];
        atomicAdd(energy, s);
    }
}

// ------------------------------------------------------------- optical flow
// D at a real displacement (reading R35): bilinear over the census Hamming
// costs of the four surrounding integer displacements (oob outside the image),
// in the oracle's operation order.
struct FlowArgs {
    const uint32_t* c1;
    const uint32_t* c2;
    int W, H;
    real oob;
};

__device__ __forceinline__ real flow_cost_int(const FlowArgs& f, int x, int y, long long a, long long b) {
    const long long xs = x + a, ys = y + b;
    if (xs < 0 || xs >= f.W || ys < 0 || ys >= f.H) return f.oob;
    return (real)__popc(f.c1[(size_t)y * f.W + x] ^ f.c2[(size_t)ys * f.W + xs]);
}

__device__ __forceinline__ real flow_cost_bilinear(const FlowArgs& f, int x, int y, real u1, real u2) {
    const real a0 = floor(u1), b0 = floor(u2);
    const real fx = u1 - a0, fy = u2 - b0;
    const long long ia = (long long)a0, ib = (long long)b0;
    const real d00 = flow_cost_int(f, x, y, ia, ib), d10 = flow_cost_int(f, x, y, ia + 1, ib);
    const real d01 = flow_cost_int(f, x, y, ia, ib + 1), d11 = flow_cost_int(f, x, y, ia + 1, ib + 1);
    return ((1.0 - fx) * (1.0 - fy) * d00 + fx * (1.0 - fy) * d10) + ((1.0 - fx) * fy * d01 + fx * fy * d11);
}

// the layers' labels -> displacements; duals of both components 0
__global__ void flow_init_kernel(RefArgs a1, RefArgs a2, real u1_min, real u2_min) {
    const int x = blockIdx.x * kRX + threadIdx.x, y = blockIdx.y * kRY + threadIdx.y;
    if (x >= a1.W || y >= a1.H) return;
    const size_t i = (size_t)y * a1.W + x;
    arr(a1, 0)[i] = u1_min + (real)a1.labels[i];
    arr(a2, 0)[i] = u2_min + (real)a2.labels[i];
    for (int k = 5; k < kRefArrays; ++k) { arr(a1, k)[i] = 0.0; arr(a2, k)[i] = 0.0; }
}

// the quadratic model of Eq. 19 at the current (u1, u2) (readings R34-R36):
// central differences (nine bilinear census costs), the PSD part of the 2x2
// Hessian [[Qa, Qb], [Qb, Qc]] (negative eigenvalue clipped), in the oracle's
// operation order (oracle/refine.py flow_quadratic, psd_part).  Slots: u0 ->
// 2, L -> 3 of each component, Qa -> a1's 4, Qc -> a2's 4, Qb -> a1's 13.
__global__ void flow_warp_kernel(RefArgs a1, RefArgs a2, FlowArgs f) {
    const int x = blockIdx.x * kRX + threadIdx.x, y = blockIdx.y * kRY + threadIdx.y;
    if (x >= a1.W || y >= a1.H) return;
    const size_t i = (size_t)y * a1.W + x;
    const real u1 = arr(a1, 0)[i], u2 = arr(a2, 0)[i], h = a1.h;
    const real d0 = flow_cost_bilinear(f, x, y, u1, u2);
    const real dp1 = flow_cost_bilinear(f, x, y, u1 + h, u2), dm1 = flow_cost_bilinear(f, x, y, u1 - h, u2);
    const real dp2 = flow_cost_bilinear(f, x, y, u1, u2 + h), dm2 = flow_cost_bilinear(f, x, y, u1, u2 - h);
    const real dpp = flow_cost_bilinear(f, x, y, u1 + h, u2 + h), dpm = flow_cost_bilinear(f, x, y, u1 + h, u2 - h);
    const real dmp = flow_cost_bilinear(f, x, y, u1 - h, u2 + h), dmm = flow_cost_bilinear(f, x, y, u1 - h, u2 - h);
    const real qa = (dp1 - 2.0 * d0 + dm1) / (h * h);
    const real qc = (dp2 - 2.0 * d0 + dm2) / (h * h);
    const real qb = ((dpp - dpm) - (dmp - dmm)) / (4.0 * h * h);
    // PSD part: eigenvalues m +- rad; l1 > 0 > l2 keeps l1 (Q - l2 I) / (l1 - l2)
    const real m = 0.5 * (qa + qc), dl = 0.5 * (qa - qc);
    const real rad = sqrt(dl * dl + qb * qb);
    const real l1 = m + rad, l2 = m - rad;
    const bool mixed = l1 > 0.0 && l2 < 0.0;
    const real sc = mixed ? l1 / (2.0 * rad) : 0.0;
    arr(a1, 2)[i] = u1;
    arr(a1, 3)[i] = (dp1 - dm1) / (2.0 * h);
    arr(a1, 4)[i] = l2 >= 0.0 ? qa : (mixed ? sc * (qa - l2) : 0.0);
    arr(a1, 13)[i] = l2 >= 0.0 ? qb : (mixed ? sc * qb : 0.0);
    arr(a2, 2)[i] = u2;
    arr(a2, 3)[i] = (dp2 - dm2) / (2.0 * h);
    arr(a2, 4)[i] = l2 >= 0.0 ? qc : (mixed ? sc * (qc - l2) : 0.0);
}

// Flow tile kernel: the stereo tile kernel's temporal blocking with both
// components in lockstep, because the primal step is the joint 2-D prox of
// Eq. 20 (reading R34): r = uh + tau (Q u0 - L), (I + tau Q) v = r by Cramer's
// rule, each component clamped to [u0 - h, u0 + h]; each component's duals
// (its own regulariser) as in stereo.  Per-pixel constants of the prox (u0,
// tau (Q u0 - L), the entries and determinant of I + tau Q) live in shared
// memory, the duals in registers, u (before / after the primal step) and
// p - q per component and direction in shared memory.  Tile 64 x 24, three
// pixels per thread.
#ifndef DMM_FTY
#define DMM_FTY 24
#endif
#ifndef DMM_FTPX
#define DMM_FTPX 3
#endif
constexpr int kFTY = DMM_FTY, kFTPX = DMM_FTPX, kFOY = kFTY - 2 * kHalo;
constexpr int kFThreads = kTX * kFTY / kFTPX, kFN = kTX * kFTY;
constexpr size_t kFSmem = 16 * sizeof(real) * kFN;
static_assert(kFSmem <= 227 * 1024, "flow tile: shared memory per CTA");   // (measured: 24 x 3 beats 16 x 2, 24 x 2)

__global__ void __launch_bounds__(kFThreads) flow_tile_kernel(RefArgs a1, RefArgs a2, int cur, int nt) {
    extern __shared__ real fsm[];
    // [0, 4): u1 (2 buffers), u2 (2 buffers); [4, 8): dh1, dv1, dh2, dv2;
    // [8, 16): u01, u02, k1, k2, m11, m22, m12, det
    auto S = [&](int k) { return fsm + (size_t)k * kFN; };
    const int W = a1.W, H = a1.H;
    const real tau = a1.tau, sigma = a1.sigma, h = a1.h, wh = a1.wh, wv = a1.wv;
    const real bp = a1.C + a1.delta - a1.eps * a1.delta;
    const real q_awh = 0.0 * wh, q_awv = 0.0 * wv, q_bs = bp * tau;
    const real p_awh = a1.eps * wh, p_awv = a1.eps * wv, p_bs = a1.delta * sigma;
    const int lx = threadIdx.x % kTX, ly0 = (threadIdx.x / kTX) * kFTPX;
    const int gx = blockIdx.x * kOX - kHalo + lx, gy0 = blockIdx.y * kFOY - kHalo + ly0;
    const int b0 = 5 + 4 * cur, b1 = 5 + 4 * (1 - cur);
    const bool inx = gx >= 0 && gx < W;
    const bool hasr = gx + 1 < W && lx + 1 < kTX, hasl = gx > 0 && lx > 0, inr = gx + 1 < W;
    real u[2][kFTPX], ph[2][kFTPX], pv[2][kFTPX], qh[2][kFTPX], qv[2][kFTPX], un[2][kFTPX];
#pragma unroll
    for (int r = 0; r < kFTPX; ++r) {
        const int gy = gy0 + r, l = (ly0 + r) * kTX + lx;
        real u01 = 0.0, u02 = 0.0, k1 = 0.0, k2 = 0.0, m11 = 1.0, m22 = 1.0, m12 = 0.0, det = 1.0;
#pragma unroll
        for (int c = 0; c < 2; ++c) u[c][r] = ph[c][r] = pv[c][r] = qh[c][r] = qv[c][r] = 0.0;
        if (inx && gy >= 0 && gy < H) {
            const size_t i = (size_t)gy * W + gx;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const RefArgs& a = c ? a2 : a1;
                u[c][r] = arr(a, cur)[i];
                ph[c][r] = arr(a, b0)[i];
                pv[c][r] = arr(a, b0 + 1)[i];
                qh[c][r] = arr(a, b0 + 2)[i];
                qv[c][r] = arr(a, b0 + 3)[i];
            }
            u01 = arr(a1, 2)[i];
            u02 = arr(a2, 2)[i];
            const real L1 = arr(a1, 3)[i], L2 = arr(a2, 3)[i];
            const real qa = arr(a1, 4)[i], qc = arr(a2, 4)[i], qb = arr(a1, 13)[i];
            // the prox's subexpressions, as oracle/refine.py prox_quadratic forms them
            k1 = tau * ((qa * u01 + qb * u02) - L1);
            k2 = tau * ((qb * u01 + qc * u02) - L2);
            m11 = 1.0 + tau * qa;
            m22 = 1.0 + tau * qc;
            m12 = tau * qb;
            det = m11 * m22 - m12 * m12;
        }
        S(8)[l] = u01; S(9)[l] = u02; S(10)[l] = k1; S(11)[l] = k2;
        S(12)[l] = m11; S(13)[l] = m22; S(14)[l] = m12; S(15)[l] = det;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            S(2 * c)[l] = u[c][r];
            S(4 + 2 * c)[l] = ph[c][r] - qh[c][r];
            S(5 + 2 * c)[l] = pv[c][r] - qv[c][r];
        }
    }
    __syncthreads();
    for (int t = 0; t < nt; ++t) {
        const int ob = t & 1, nb = (t + 1) & 1;      // u buffers: old, new
#pragma unroll
        for (int r = 0; r < kFTPX; ++r) {          // joint primal step
            const int gy = gy0 + r, ly = ly0 + r, l = ly * kTX + lx;
            real uh[2];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const real* sdh = S(4 + 2 * c);
                const real* sdv = S(5 + 2 * c);
                real div = 0.0;
                if (inr) div += ph[c][r] - qh[c][r];
                if (hasl) div -= sdh[l - 1];
                if (gy + 1 < H) div += pv[c][r] - qv[c][r];
                if (gy > 0 && ly > 0) div -= sdv[l - kTX];
                uh[c] = u[c][r] - tau * div;
            }
            const real u01 = S(8)[l], u02 = S(9)[l];
            const real m11 = S(12)[l], m22 = S(13)[l], m12 = S(14)[l], det = S(15)[l];
            const real r1 = uh[0] + S(10)[l], r2 = uh[1] + S(11)[l];
            const real v1 = (m22 * r1 - m12 * r2) / det;
            const real v2 = (m11 * r2 - m12 * r1) / det;
            un[0][r] = dclip(v1, u01 - h, u01 + h);
            un[1][r] = dclip(v2, u02 - h, u02 + h);
            S(2 * 0 + nb)[l] = un[0][r];
            S(2 * 1 + nb)[l] = un[1][r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kFTPX; ++r) {          // each component's dual steps
            const int gy = gy0 + r, ly = ly0 + r, l = ly * kTX + lx;
            const bool hasd = gy + 1 < H && ly + 1 < kFTY;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const real* uo = S(2 * c + ob);
                const real* us = S(2 * c + nb);
                const real bi = 2.0 * un[c][r] - u[c][r];
                const real ur = uo[l + 1], ud = uo[l + kTX];
                const real nqh = prox_conj_h(qh[c][r] + tau * (u[c][r] - ur), wh, q_awh, q_bs);
                const real nph = prox_conj_h(ph[c][r] + sigma * (bi - (2.0 * us[l + 1] - ur)), wh, p_awh, p_bs);
                const real nqv = prox_conj_h(qv[c][r] + tau * (u[c][r] - ud), wv, q_awv, q_bs);
                const real npv = prox_conj_h(pv[c][r] + sigma * (bi - (2.0 * us[l + kTX] - ud)), wv, p_awv, p_bs);
                qh[c][r] = hasr ? nqh : qh[c][r];
                ph[c][r] = hasr ? nph : ph[c][r];
                qv[c][r] = hasd ? nqv : qv[c][r];
                pv[c][r] = hasd ? npv : pv[c][r];
                u[c][r] = un[c][r];
            }
        }
#pragma unroll
        for (int r = 0; r < kFTPX; ++r) {
            const int l = (ly0 + r) * kTX + lx;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                S(4 + 2 * c)[l] = ph[c][r] - qh[c][r];
                S(5 + 2 * c)[l] = pv[c][r] - qv[c][r];
            }
        }
        __syncthreads();
    }
    if (!inx || lx < kHalo || lx >= kTX - kHalo) return;
#pragma unroll
    for (int r = 0; r < kFTPX; ++r) {
        const int gy = gy0 + r, ly = ly0 + r;
        if (gy < 0 || gy >= H || ly < kHalo || ly >= kFTY - kHalo) continue;
        const size_t i = (size_t)gy * W + gx;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const RefArgs& a = c ? a2 : a1;
            arr(a, 1 - cur)[i] = u[c][r];
            if (inr) {
                arr(a, b1)[i] = ph[c][r];
                arr(a, b1 + 2)[i] = qh[c][r];
            }
            if (gy + 1 < H) {
                arr(a, b1 + 1)[i] = pv[c][r];
                arr(a, b1 + 3)[i] = qv[c][r];
            }
        }
    }
}

__global__ void flow_out_kernel(RefArgs a1, RefArgs a2, FlowArgs f, float* out1, float* out2, double* energy) {
    const int x = blockIdx.x * kRX + threadIdx.x, y = blockIdx.y * kRY + threadIdx.y;
    double e = 0.0;
    if (x < a1.W && y < a1.H) {
        const int W = a1.W;
        const size_t i = (size_t)y * W + x;
        const real* u1 = arr(a1, 0);
        const real* u2 = arr(a2, 0);
        if (out1) out1[i] = (float)u1[i];
        if (out2) out2[i] = (float)u2[i];
        e = flow_cost_bilinear(f, x, y, u1[i], u2[i]);
        const real* us[2] = {u1, u2};
        for (int k = 0; k < 2; ++k) {
            if (x + 1 < W) e += a1.wh * r_dc(us[k][i] - us[k][i + 1], a1.eps, a1.delta, a1.C);
            if (y + 1 < a1.H) e += a1.wv * r_dc(us[k][i] - us[k][i + W], a1.eps, a1.delta, a1.C);
        }
    }
    for (int d = 16; d > 0; d >>= 1) e += __shfl_down_sync(0xffffffffu, e, d);
    __shared__ double part[kRX * kRY / 32];
    const int t = threadIdx.y * kRX + threadIdx.x;
    if ((t & 31) == 0) part[t >> 5] = e;
    __syncthreads();
    if (t == 0 && energy) {
        double s = 0.0;
        for (int k = 0; k < kRX * kRY / 32; ++k) s += part[k];
        atomicAdd(energy, s);
    }
}

// `iters` iterations as ceil(iters / kHalo) tile launches (stereo: a0; flow:
// a0, a1 = the two components), then the state back to buffer 0; returns the
// number of launches
int launch_iters(const RefArgs& a0, const RefArgs* a1, int iters, cudaStream_t s) {
    static bool attr = [] {
        cudaFuncSetAttribute(refine_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmem);
        cudaFuncSetAttribute(flow_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFSmem);
        return true;
    }();
    (void)attr;
    int cur = 0, n = 0;
    for (int it = 0; it < iters; it += kHalo, ++n, cur ^= 1) {
        const int nt = min(kHalo, iters - it);
        if (a1)
            flow_tile_kernel<<<dim3((a0.W + kOX - 1) / kOX, (a0.H + kFOY - 1) / kFOY), kFThreads, kFSmem, s>>>(
                a0, *a1, cur, nt);
        else
            refine_tile_kernel<<<dim3((a0.W + kOX - 1) / kOX, (a0.H + kOY - 1) / kOY), kTileThreads, kTileSmem, s>>>(
                a0, cur, nt);
    }
    if (cur) {
        const dim3 g2((a0.W + kRX - 1) / kRX, (a0.H + kRY - 1) / kRY), blk(kRX, kRY);
        refine_swap_kernel<<<g2, blk, 0, s>>>(a0);
        ++n;
        if (a1) { refine_swap_kernel<<<g2, blk, 0, s>>>(*a1); ++n; }
    }
    return n;
}

RefArgs ref_args(dmm_ctx* ctx, int frame, const dmm_refine_params* prm) {
    FramePtrs P = frame_ptrs(ctx->L, frame);
    RefArgs a;
    a.rf = reinterpret_cast<real*>(P.rf);
    a.D = P.D;
    a.labels = P.labels;
    a.W = ctx->L.W; a.H = ctx->L.H; a.K = ctx->K; a.KP = ctx->KP;
    a.wh = (real)ctx->cfg.w_h; a.wv = (real)ctx->cfg.w_v;
    a.eps = prm->eps; a.delta = prm->delta; a.C = prm->C; a.h = prm->h; a.tau = prm->tau; a.sigma = prm->sigma;
    return a;
}

}  // namespace

size_t refine_bytes(int W, int H) { return (size_t)kRefArrays * sizeof(real) * W * H; }

dmm_status refine_run(dmm_ctx* ctx, int frame, const dmm_refine_params* prm, float* out, double* energy_dev,
                      cudaStream_t s) {
    FramePtrs P = frame_ptrs(ctx->L, frame);
    RefArgs a = ref_args(ctx, frame, prm);
    const dim3 grid((a.W + kRX - 1) / kRX, (a.H + kRY - 1) / kRY), blk(kRX, kRY);
    refine_init_kernel<<<grid, blk, 0, s>>>(a);
    ++ctx->launches;
    // one warp = the expansion kernel + `iters` iteration kernels (+ a swap for
    // an odd count, so the state ends in buffer 0).  Captured once per (frame,
    // parameters) into a graph on the context's capture stream, replayed on `s`.
    RefineGraph& g = ctx->rg;
    const bool same = g.exec && g.frame == frame && memcmp(&g.prm, prm, sizeof(*prm)) == 0 && g.rf == P.rf;
    if (!same) {
        if (g.exec) { cudaGraphExecDestroy(g.exec); g.exec = nullptr; }
        if (!g.cap && cudaStreamCreateWithFlags(&g.cap, cudaStreamNonBlocking) != cudaSuccess)
            return cuda_status(ctx, cudaGetLastError(), "refine capture stream");
        cudaGraph_t graph = nullptr;
        int launches_per_warp = 0;
        cudaError_t e = cudaStreamBeginCapture(g.cap, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) return cuda_status(ctx, e, "refine capture");
        refine_warp_kernel<<<grid, blk, 0, g.cap>>>(a);
        launches_per_warp = 1 + launch_iters(a, nullptr, prm->iters, g.cap);
        g.launches_per_warp = launches_per_warp;
        e = cudaStreamEndCapture(g.cap, &graph);
        if (e != cudaSuccess) return cuda_status(ctx, e, "refine capture end");
        e = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return cuda_status(ctx, e, "refine graph instantiate");
        g.frame = frame;
        g.prm = *prm;
        g.rf = P.rf;
    }
    for (int w = 0; w < prm->warps; ++w) {
        cudaError_t e = cudaGraphLaunch(g.exec, s);
        if (e != cudaSuccess) return cuda_status(ctx, e, "refine graph launch");
        ctx->launches += g.launches_per_warp;
    }
    refine_out_kernel<<<grid, blk, 0, s>>>(a, (real)ctx->cfg.d_min, out, energy_dev);
    ++ctx->launches;
    return cuda_status(ctx, cudaGetLastError(), "refine");
}


// Flow refinement (Sec. 3.2): layer frames `frame` (u1) and `frame + 1` (u2)
// of a flow context; census codes of frame `frame`.
dmm_status refine_flow_run(dmm_ctx* ctx, int frame, double u1_min, double u2_min, const dmm_refine_params* prm,
                           float* out1, float* out2, double* energy_dev, cudaStream_t s) {
    RefArgs a1 = ref_args(ctx, frame, prm), a2 = ref_args(ctx, frame + 1, prm);
    FramePtrs P = frame_ptrs(ctx->L, frame);
    FlowArgs f{P.codes_l, P.codes_r, ctx->L.W, ctx->L.H, (real)ctx->oob};
    const dim3 grid((a1.W + kRX - 1) / kRX, (a1.H + kRY - 1) / kRY), blk(kRX, kRY);
    flow_init_kernel<<<grid, blk, 0, s>>>(a1, a2, u1_min, u2_min);
    ++ctx->launches;
    RefineGraph& g = ctx->rgf;
    const bool same = g.exec && g.frame == frame && memcmp(&g.prm, prm, sizeof(*prm)) == 0 && g.rf == P.rf;
    if (!same) {
        if (g.exec) { cudaGraphExecDestroy(g.exec); g.exec = nullptr; }
        if (!g.cap && cudaStreamCreateWithFlags(&g.cap, cudaStreamNonBlocking) != cudaSuccess)
            return cuda_status(ctx, cudaGetLastError(), "refine capture stream");
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamBeginCapture(g.cap, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) return cuda_status(ctx, e, "flow refine capture");
        flow_warp_kernel<<<grid, blk, 0, g.cap>>>(a1, a2, f);
        g.launches_per_warp = 1 + launch_iters(a1, &a2, prm->iters, g.cap);
        e = cudaStreamEndCapture(g.cap, &graph);
        if (e != cudaSuccess) return cuda_status(ctx, e, "flow refine capture end");
        e = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return cuda_status(ctx, e, "flow refine graph instantiate");
        g.frame = frame;
        g.prm = *prm;
        g.rf = P.rf;
    }
    for (int w = 0; w < prm->warps; ++w) {
        cudaError_t e = cudaGraphLaunch(g.exec, s);
        if (e != cudaSuccess) return cuda_status(ctx, e, "flow refine graph launch");
        ctx->launches += g.launches_per_warp;
    }
    flow_out_kernel<<<grid, blk, 0, s>>>(a1, a2, f, out1, out2, energy_dev);
    ++ctx->launches;
    return cuda_status(ctx, cudaGetLastError(), "flow refine");
}

void refine_release(dmm_ctx* ctx) {
    for (RefineGraph* g : {&ctx->rg, &ctx->rgf}) {
        if (g->exec) cudaGraphExecDestroy(g->exec);
        if (g->cap) cudaStreamDestroy(g->cap);
        g->exec = nullptr;
        g->cap = nullptr;
    }
}

}  // namespace dmm
