// hmg.cu -- Dual MM half-steps for the GENERAL pairwise model (NEXT-3, SURVEY
// 8(f)): the three-piece penalty of Fig.2 (r = r_{eps,delta} -
// r_{0,C+delta-eps*delta}, Eq. r-decompose) sampled at integer label
// differences, times quantised edge-aware weights (Eq. regularizer-form
// omega_ij "reducing the penalty around sharp edges"):
//   R(d) = min(e1*min(d,delta) + e2*max(d-delta,0), c)    (units 2^-F)
//   V_ij(d) = floor(w * om_ij * R(|d|) / 16),   om_ij in [1,16]
// (readings R29-R31).  Such V is in general NOT a metric (eps < 1 breaks the
// triangle inequality), so the Handshake keeps Alg.5's literal three Msg
// (the bounce identity of the truncated-linear kernels does not apply), and
// every Msg is evaluated from its own edge's weight.
//
// Layout: the duals are dense int32 [H][W][KP] (the classic compact u16
// records' span bound does not hold for arbitrary penalties): gfv = f_ (H
// output, V input), ggh = D*2^F + g_ (V output, H input).  The hierarchy runs
// level-synchronously, one warp per (chain, subchain) task; the boundary
// messages of the subchains of a level live in two int32 [H][W][KP] arrays
// Lb / Rb at the subchain's first / last node (distinct across a level), so
// a split writes Rb[i] = phi_ji' (left child) and Lb[j] = phi_ij (right
// child) and leaves the parent's boundaries in place.  A final kernel emits
// lambda_p = Lb[p] + F_p + Rb[p] (reading R8) per node: the output record
// Lb + Rb + D*2^F, the node minimum into the dual bound, and (last V) the
// lowest-index argmin as the label.
//
// Msg over one edge: x is staged in the warp's shared-memory row and every
// label b takes min(min(x) + V(dc), min_{|d| < dc} x(b+d) + V(|d|)), where dc
// is the first distance with R(d) = c (V is constant beyond) -- exact.
#include "ctx.cuh"

namespace dmm {

int genR_host(const dmm_config& c, int d);
void pen_of(const dmm_config& c, int& e1, int& e2, int& delta, int& cc);

namespace {

#ifndef DMM_GW
#define DMM_GW 4
#endif
constexpr int kGW = DMM_GW;      // warps per CTA
constexpr int kBigG = 1 << 29;   // padded labels

struct GenArgs {
    const uint8_t* D;            // [H][W][KP]
    const int32_t* src;          // F of the pass ([H][W][KP]), unused when first
    int32_t* dst;                // output records
    int32_t* Lb;
    int32_t* Rb;
    const uint8_t* om;           // edge weights of this orientation [H][W] (nullptr: 16)
    uint8_t* labels;
    long long* bound;
    int W, H, K, KP, vert, first, last, fbits;
    int w, e1, e2, delta, c, dc;
    int passes, gshift;          // iterative minorant (NEXT-4)
};

__device__ __forceinline__ int genR(const GenArgs& a, int d) {
    const int lin = a.e1 * min(d, a.delta) + a.e2 * max(d - a.delta, 0);
    return min(lin, a.c);
}

// `rows` Msg staging rows of 3 KP ints at base (KP = 32 LPL): the pads
// [0, KP) and [2 KP, 3 KP) of each hold kBigG so the windowed Msg reads its
// sources x(b +- d), d < dc <= K, without bounds tests; returns the centre
// of the first row (the next row's centre is 3 KP further)
template <int LPL>
__device__ __forceinline__ int* padded_rows(int* base, int rows, int lane) {
    constexpr int KP = 32 * LPL;
    for (int r = 0; r < rows; ++r)
        for (int k = lane; k < KP; k += 32) {
            base[r * 3 * KP + k] = kBigG;
            base[r * 3 * KP + 2 * KP + k] = kBigG;
        }
    __syncwarp();
    return base + KP;
}

// The CTA's table of V values: vt[om * (dc + 1) + d] = floor(w om R(d) / 16)
// for om in [0, 16], d in [0, dc] (d = dc: the cap value), filled once per
// kernel -- the Msg reads V(d) with one broadcast shared load instead of
// evaluating R(d) and a 64-bit product per distance.
__device__ __forceinline__ int* fill_vtab(int* vt, const GenArgs& a) {
    const int vs = a.dc + 1;
    for (int idx = threadIdx.x; idx < 17 * vs; idx += blockDim.x) {
        const int om = idx / vs, d = idx - om * vs;
        vt[idx] = (int)((((long long)a.w * om) * genR(a, d)) >> 4);
    }
    __syncthreads();
    return vt;
}
inline size_t vtab_bytes(int dc) { return (size_t)17 * (dc + 1) * sizeof(int); }

template <int LPL>
struct GenPass {
    const GenArgs& a;
    int chain, n, lane;
    int* sx;                     // this warp's shared row: [KP] at sx, kBigG pads [-KP, 0) and [KP, 2 KP)
    const int* vt;               // the CTA's V table (fill_vtab)
    __device__ GenPass(const GenArgs& a_, int chain_, int lane_, int* sx_, const int* vt_)
        : a(a_), chain(chain_), lane(lane_), sx(sx_), vt(vt_) {
        n = a.vert ? a.H : a.W;
    }
    __device__ __forceinline__ size_t q(int p) const {
        return a.vert ? (size_t)p * a.W + chain : (size_t)chain * a.W + p;
    }
    __device__ __forceinline__ int om(int e) const {   // weight of edge (e, e+1) of this chain
        return a.om ? (int)a.om[q(e)] : 16;
    }
    __device__ __forceinline__ void ldF(int p, int (&F)[LPL]) const {
        const size_t base = q(p) * a.KP + lane * LPL;
#pragma unroll
        for (int e = 0; e < LPL; ++e) {
            const int k = lane * LPL + e;
            F[e] = a.first ? ((int)a.D[base + e] << a.fbits) : a.src[base + e];
            if (k >= a.K) F[e] = kBigG;
        }
    }
    __device__ __forceinline__ void ld(const int32_t* arr, int p, int (&v)[LPL]) const {
        const size_t base = q(p) * a.KP + lane * LPL;
#pragma unroll
        for (int e = 0; e < LPL; ++e) v[e] = arr[base + e];
    }
    __device__ __forceinline__ void st(int32_t* arr, int p, const int (&v)[LPL]) const {
        const size_t base = q(p) * a.KP + lane * LPL;
#pragma unroll
        for (int e = 0; e < LPL; ++e) arr[base + e] = v[e];
    }
    // Software-pipelined loads (the passes are latency-bound: one dependent Msg
    // per node): a node's costs are fetched R steps before use as raw words --
    // D bytes (first pass) or int32 records -- and expanded only at use, so
    // the load's latency overlaps the R Msg in between.
    static constexpr int kRawW = LPL;              // words per lane (D bytes use the first ceil(LPL / 4))
    template <bool FIRST>
    __device__ __forceinline__ void ldraw(int p, uint32_t (&r)[kRawW]) const {
        const size_t base = q(p) * a.KP + lane * LPL;
        if constexpr (FIRST) {
            if constexpr (LPL == 8) {
                const uint2 v = *reinterpret_cast<const uint2*>(a.D + base);
                r[0] = v.x; r[1] = v.y;
            } else if constexpr (LPL == 4) {
                r[0] = *reinterpret_cast<const uint32_t*>(a.D + base);
            } else if constexpr (LPL == 2) {
                r[0] = *reinterpret_cast<const uint16_t*>(a.D + base);
            } else {
                r[0] = a.D[base];
            }
        } else {
#pragma unroll
            for (int e = 0; e < LPL; ++e) r[e] = (uint32_t)a.src[base + e];
        }
    }
    template <bool FIRST>
    __device__ __forceinline__ void expand(const uint32_t (&r)[kRawW], int (&F)[LPL]) const {
#pragma unroll
        for (int e = 0; e < LPL; ++e) {
            F[e] = FIRST ? (int)((r[e >> 2] >> (8 * (e & 3))) & 0xffu) << a.fbits : (int)r[e];
            if (lane * LPL + e >= a.K) F[e] = kBigG;
        }
    }
    // two independent Msg (their instructions interleave): x over an edge of
    // weight omx staged in sx, y over omy staged in sy -- each exactly msg()
    __device__ __forceinline__ void msg2(int (&x)[LPL], int omx, int (&y)[LPL], int omy, int* sy) const {
        int lx = kBigG, ly = kBigG;
#pragma unroll
        for (int e = 0; e < LPL; ++e) {
            if (lane * LPL + e >= a.K) { x[e] = kBigG; y[e] = kBigG; }
            lx = min(lx, x[e]);
            ly = min(ly, y[e]);
        }
        const int mx = __reduce_min_sync(0xffffffffu, lx), my = __reduce_min_sync(0xffffffffu, ly);
        __syncwarp();
#pragma unroll
        for (int e = 0; e < LPL; ++e) { sx[lane * LPL + e] = x[e]; sy[lane * LPL + e] = y[e]; }
        __syncwarp();
        const int* tx = vt + omx * (a.dc + 1);
        const int* ty = vt + omy * (a.dc + 1);
        const int capx = mx + tx[a.dc], capy = my + ty[a.dc];
        int bx[LPL], by[LPL];
#pragma unroll
        for (int e = 0; e < LPL; ++e) { bx[e] = min(capx, x[e]); by[e] = min(capy, y[e]); }
        for (int d = 1; d < a.dc; ++d) {
            const int vx = tx[d], vy = ty[d];
#pragma unroll
            for (int e = 0; e < LPL; ++e) {
                const int b = lane * LPL + e;
                // out-of-range sources read kBigG (pads, labels >= K): never the minimum
                bx[e] = min(bx[e], sx[b - d] + vx);
                by[e] = min(by[e], sy[b - d] + vy);
                bx[e] = min(bx[e], sx[b + d] + vx);
                by[e] = min(by[e], sy[b + d] + vy);
            }
        }
#pragma unroll
        for (int e = 0; e < LPL; ++e) {
            const bool in = lane * LPL + e < a.K;
            x[e] = in ? bx[e] : capx;
            y[e] = in ? by[e] : capy;
        }
        __syncwarp();
    }
    // x := Msg over an edge of weight om: out(b) = min_a x(a) + V(|a-b|), exact
    __device__ __forceinline__ void msg(int (&x)[LPL], int omw) const {
        int lm = kBigG;
#pragma unroll
        for (int e = 0; e < LPL; ++e) {
            if (lane * LPL + e >= a.K) x[e] = kBigG;
            lm = min(lm, x[e]);
        }
        const int m = __reduce_min_sync(0xffffffffu, lm);
        __syncwarp();
#pragma unroll
        for (int e = 0; e < LPL; ++e) sx[lane * LPL + e] = x[e];
        __syncwarp();
        const int* tv = vt + omw * (a.dc + 1);
        const int cap = m + tv[a.dc];
        int best[LPL];
#pragma unroll
        for (int e = 0; e < LPL; ++e) best[e] = min(cap, x[e]);
        // distance d < dc (beyond, V = its cap value): V(d) computed once per
        // distance (warp-uniform), the lane's LPL labels read their two
        // neighbours at distance d from the staged row
        for (int d = 1; d < a.dc; ++d) {
            const int v = tv[d];
#pragma unroll
            for (int e = 0; e < LPL; ++e) {
                const int b = lane * LPL + e;
                best[e] = min(best[e], sx[b - d] + v);
                best[e] = min(best[e], sx[b + d] + v);
            }
        }
#pragma unroll
        for (int e = 0; e < LPL; ++e) x[e] = lane * LPL + e < a.K ? best[e] : cap;
        __syncwarp();
    }
};

// One level of the hierarchy: one warp per (chain, subchain) task.  The
// task's two passes (into i from the left, into j from the right) are
// independent chains of Msg: they run interleaved (msg2), their node costs
// and edge weights fetched kPre steps ahead (register rings, static slots).
#ifndef DMM_GPRE
#define DMM_GPRE 4
#endif
template <int LPL>
constexpr int kPre = LPL >= 8 ? DMM_GPRE / 2 : DMM_GPRE;

template <int LPL, bool FIRST>
__global__ void __launch_bounds__(kGW * 32) hmg_level_kernel(GenArgs a, int lev, int ntasks) {
    constexpr int R = kPre<LPL>;
    extern __shared__ int gsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int* sx = padded_rows<LPL>(gsm + warp * 6 * 32 * LPL, 2, lane);
    int* sy = sx + 3 * 32 * LPL;
    const int* vt = fill_vtab(gsm + kGW * 6 * 32 * LPL, a);
    for (int t = blockIdx.x * kGW + warp; t < ntasks; t += gridDim.x * kGW) {
        const int chain = t >> lev, s = t & ((1 << lev) - 1);
        GenPass<LPL> g(a, chain, lane, sx, vt);
        int lo = 0, hi = g.n - 1;
        for (int b = lev - 1; b >= 0; --b) {
            const int mid = lo + (hi - lo + 1) / 2 - 1;
            if ((s >> b) & 1) lo = mid + 1; else hi = mid;
        }
        if (hi <= lo) continue;                       // single node: nothing to split
        DMM_CHECK(lo >= 0 && hi < g.n);
        const int len = hi - lo + 1, i = lo + len / 2 - 1, j = i + 1;
        int pl[LPL], pr[LPL], F[LPL];
        if (lev == 0) {
#pragma unroll
            for (int e = 0; e < LPL; ++e) { pl[e] = 0; pr[e] = 0; }
        } else {
            g.ld(a.Lb, lo, pl);
            g.ld(a.Rb, hi, pr);
        }
        // left pass: step u adds F(lo + u) and crosses edge lo + u; right pass:
        // step u adds F(hi - u) and crosses edge hi - u - 1
        const int nl = i - lo, nr = hi - j, ns = max(nl, nr);
        uint32_t rl[R][LPL], rr[R][LPL];
        int ol[R], orr[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            // a pass shorter than the other runs idle steps on unloaded slots: their
            // weight must still index the V table (their results are discarded)
            ol[k] = orr[k] = 16;
            if (k < nl) { g.template ldraw<FIRST>(lo + k, rl[k]); ol[k] = g.om(lo + k); }
            if (k < nr) { g.template ldraw<FIRST>(hi - k, rr[k]); orr[k] = g.om(hi - k - 1); }
        }
        for (int u0 = 0; u0 < ns; u0 += R) {
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const int u = u0 + k;
                if (u >= ns) break;
                int Fl[LPL], Fr[LPL];
                g.template expand<FIRST>(rl[k], Fl);
                g.template expand<FIRST>(rr[k], Fr);
                const int oml = ol[k], omr = orr[k];
                if (u + R < nl) { g.template ldraw<FIRST>(lo + u + R, rl[k]); ol[k] = g.om(lo + u + R); }
                if (u + R < nr) { g.template ldraw<FIRST>(hi - u - R, rr[k]); orr[k] = g.om(hi - u - R - 1); }
                int xl[LPL], xr[LPL];
#pragma unroll
                for (int e = 0; e < LPL; ++e) { xl[e] = pl[e] + Fl[e]; xr[e] = pr[e] + Fr[e]; }
                g.msg2(xl, oml, xr, omr, sy);
                const bool dl = u < nl, dr = u < nr;
#pragma unroll
                for (int e = 0; e < LPL; ++e) {
                    pl[e] = dl ? xl[e] : pl[e];
                    pr[e] = dr ? xr[e] : pr[e];
                }
            }
        }
        // Handshake (Alg.5, literal three Msg; readings R9, R10)
        const int omij = g.om(i);
        int pji[LPL], t_[LPL], Fi[LPL];
        g.ldF(j, F);
#pragma unroll
        for (int e = 0; e < LPL; ++e) pji[e] = F[e] + pr[e];
        g.msg(pji, omij);                                            // phi_ji := Msg(f_j + phi_{j+1,j})
        g.ldF(i, Fi);
#pragma unroll
        for (int e = 0; e < LPL; ++e) t_[e] = (pl[e] + Fi[e] - pji[e]) >> 1;   // floor(m_i/2 - phi_ji)
        g.msg(t_, omij);                                             // phi_ij
        int b_[LPL];
#pragma unroll
        for (int e = 0; e < LPL; ++e) b_[e] = -t_[e];
        g.msg(b_, omij);                                             // phi_ji' := Msg(-phi_ij)
        g.st(a.Rb, i, b_);
        g.st(a.Lb, j, t_);
    }
}

// The top levels (few, long tasks: latency-bound) with one CTA of KP threads
// per task, one label per thread -- the same task as hmg_level_kernel (its two
// passes interleaved, then Alg.5's three Msg), each Msg CTA-wide: the
// thread stages its value in one of two padded rows per pass (alternating, so
// one barrier per step orders rows and warp minima), the CTA minimum gives the
// cap, the window is two shared loads per distance.  Node data fetched
// kPreIt steps ahead.
constexpr int kPreLv = 4;

template <int KP, bool FIRST>
__global__ void __launch_bounds__(KP) hmg_level_cta_kernel(GenArgs a, int lev, int ntasks) {
    constexpr int NW = KP / 32, R = kPreLv;
    extern __shared__ int gsm[];
    int* rows = gsm;                                  // [2 parities][2 passes] x [pad KP | row KP | pad KP]
    int* wmin = gsm + 12 * KP;                        // [2 parities][2 passes][NW]
    const int k = threadIdx.x, lane = k & 31, warp = k >> 5;
    for (int r = 0; r < 4; ++r) { rows[r * 3 * KP + k] = kBigG; rows[r * 3 * KP + 2 * KP + k] = kBigG; }
    const int* vt = fill_vtab(gsm + 12 * KP + 4 * NW, a);
    const bool in = k < a.K;
    int par = 0;
    // Msg of the values x (pass 0) and y (pass 1) over edges of weights ox, oy
    auto msg2 = [&](int& x, int ox, int& y, int oy) {
        if (!in) { x = kBigG; y = kBigG; }
        int* rx = rows + (2 * par) * 3 * KP + KP;
        int* ry = rows + (2 * par + 1) * 3 * KP + KP;
        rx[k] = x;
        ry[k] = y;
        const int mx = __reduce_min_sync(0xffffffffu, x), my = __reduce_min_sync(0xffffffffu, y);
        if (lane == 0) { wmin[(2 * par) * NW + warp] = mx; wmin[(2 * par + 1) * NW + warp] = my; }
        __syncthreads();
        int m0 = wmin[(2 * par) * NW], m1 = wmin[(2 * par + 1) * NW];
#pragma unroll
        for (int w = 1; w < NW; ++w) { m0 = min(m0, wmin[(2 * par) * NW + w]); m1 = min(m1, wmin[(2 * par + 1) * NW + w]); }
        const int* tx = vt + ox * (a.dc + 1);
        const int* ty = vt + oy * (a.dc + 1);
        const int capx = m0 + tx[a.dc], capy = m1 + ty[a.dc];
        int bx = min(capx, x), by = min(capy, y);
#pragma unroll 4
        for (int d = 1; d < a.dc; ++d) {
            const int vx = tx[d], vy = ty[d];
            bx = min(bx, rx[k - d] + vx);
            by = min(by, ry[k - d] + vy);
            bx = min(bx, rx[k + d] + vx);
            by = min(by, ry[k + d] + vy);
        }
        par ^= 1;
        x = in ? bx : capx;
        y = in ? by : capy;
    };
    auto msg1 = [&](int& x, int ox) { int y = 0; msg2(x, ox, y, 16); };
    const int n = a.vert ? a.H : a.W;
    const int fbits = a.fbits;
    const long long pst = a.vert ? a.W : 1;
    for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
        const int chain = t >> lev, s = t & ((1 << lev) - 1);
        int lo = 0, hi = n - 1;
        for (int b = lev - 1; b >= 0; --b) {
            const int mid = lo + (hi - lo + 1) / 2 - 1;
            if ((s >> b) & 1) lo = mid + 1; else hi = mid;
        }
        if (hi <= lo) continue;                       // single node: nothing to split
        const long long c0 = a.vert ? chain : (long long)chain * a.W;
        const long long cb = c0 * KP + k, est = pst * KP;
        const uint8_t* Dp = a.D + cb;
        const int32_t* Sp = a.src + cb;
        const uint8_t* Op = a.om ? a.om + c0 : nullptr;
        auto ldF = [&](int p) -> int { return FIRST ? (int)Dp[p * est] : Sp[p * est]; };
        auto F_of = [&](int raw) -> int { return !in ? kBigG : (FIRST ? raw << fbits : raw); };
        auto om_of = [&](int e) -> int { return Op ? (int)Op[e * pst] : 16; };
        const int len = hi - lo + 1, i = lo + len / 2 - 1, j = i + 1;
        int pl = lev == 0 ? 0 : a.Lb[cb + lo * est];
        int pr = lev == 0 ? 0 : a.Rb[cb + hi * est];
        const int nl = i - lo, nr = hi - j, ns = max(nl, nr);
        int rl[R], rr[R], ol[R], orr[R];
#pragma unroll
        for (int q = 0; q < R; ++q) {
            ol[q] = orr[q] = 16;                      // idle steps of the shorter pass: a valid weight
            rl[q] = rr[q] = 0;
            if (q < nl) { rl[q] = ldF(lo + q); ol[q] = om_of(lo + q); }
            if (q < nr) { rr[q] = ldF(hi - q); orr[q] = om_of(hi - q - 1); }
        }
        // the prefetch cursors: node lo + u + R (left), hi - u - R (right), stepped per step
        const uint8_t* dL = FIRST ? Dp + (lo + R) * est : nullptr;
        const uint8_t* dR = FIRST ? Dp + (hi - R) * est : nullptr;
        const int32_t* sL = FIRST ? nullptr : Sp + (lo + R) * est;
        const int32_t* sR = FIRST ? nullptr : Sp + (hi - R) * est;
        const uint8_t* oL = Op ? Op + (lo + R) * pst : nullptr;
        const uint8_t* oR = Op ? Op + (hi - R - 1) * pst : nullptr;
        for (int u0 = 0; u0 < ns; u0 += R) {
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int u = u0 + q;
                if (u >= ns) break;
                int xl = pl + F_of(rl[q]), xr = pr + F_of(rr[q]);
                const int oml = ol[q], omr = orr[q];
                if (u + R < nl) { rl[q] = FIRST ? (int)*dL : *sL; ol[q] = oL ? (int)*oL : 16; }
                if (u + R < nr) { rr[q] = FIRST ? (int)*dR : *sR; orr[q] = oR ? (int)*oR : 16; }
                if (FIRST) { dL += est; dR -= est; } else { sL += est; sR -= est; }
                if (Op) { oL += pst; oR -= pst; }
                msg2(xl, oml, xr, omr);
                if (u < nl) pl = xl;
                if (u < nr) pr = xr;
            }
        }
        // Handshake (Alg.5, literal three Msg; readings R9, R10)
        const int omij = om_of(i);
        int pji = F_of(ldF(j)) + pr;
        msg1(pji, omij);                              // phi_ji := Msg(f_j + phi_{j+1,j})
        int t_ = (pl + F_of(ldF(i)) - pji) >> 1;      // floor(m_i/2 - phi_ji)
        msg1(t_, omij);                               // phi_ij
        int b_ = -t_;
        msg1(b_, omij);                               // phi_ji' := Msg(-phi_ij)
        a.Rb[cb + i * est] = b_;
        a.Lb[cb + j * est] = t_;
    }
}

// Chain ends: Lb[first] = Rb[last] = 0 (the boundary messages of level 0).
__global__ void hmg_ends_kernel(GenArgs a, int chains, int n) {
    const int KP = a.KP;
    for (long long z = blockIdx.x * (long long)blockDim.x + threadIdx.x; z < (long long)chains * KP;
         z += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(z / KP), k = (int)(z - (long long)c * KP);
        const size_t q0 = a.vert ? (size_t)c : (size_t)c * a.W;
        const size_t q1 = a.vert ? (size_t)(n - 1) * a.W + c : (size_t)c * a.W + n - 1;
        a.Lb[q0 * KP + k] = 0;
        a.Rb[q1 * KP + k] = 0;
    }
}

// Output of the iterative minorant (Alg.4): lambda (in Rb) per node; record
// lambda - F + D*2^F (the other orientation's input), bound += min lambda,
// last V: lowest argmin label.  One warp per node (grid-stride).  (The
// hierarchical path emits from its leaf kernel.)
template <int LPL>
__global__ void __launch_bounds__(kGW * 32) hmg_emit_kernel(GenArgs a) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    long long bsum = 0;
    for (long long qn = gw; qn < (long long)a.W * a.H; qn += nw) {
        const size_t base = (size_t)qn * a.KP + lane * LPL;
        int lmin = kBigG, arg = 0x7fffffff;
        int lam[LPL];
#pragma unroll
        for (int e = 0; e < LPL; ++e) {
            const int k = lane * LPL + e;
            const int Ds = (int)a.D[base + e] << a.fbits;
            const int F = a.first ? Ds : a.src[base + e];
            const int lr = a.Rb[base + e] - F;
            lam[e] = lr + F;
            a.dst[base + e] = k < a.K ? lr + Ds : 0;
            if (k < a.K) lmin = min(lmin, lam[e]);
        }
        const int m = __reduce_min_sync(0xffffffffu, lmin);
        bsum += m;
        if (a.last && a.vert) {
#pragma unroll
            for (int e = LPL - 1; e >= 0; --e)
                if (lane * LPL + e < a.K && lam[e] == m) arg = lane * LPL + e;
            arg = __reduce_min_sync(0xffffffffu, arg);
            if (lane == 0) a.labels[qn] = (uint8_t)arg;
        }
    }
    if (lane == 0 && bsum != 0) atomicAdd(reinterpret_cast<unsigned long long*>(a.bound), (unsigned long long)bsum);
}

__global__ void hmg_weights_kernel(const uint8_t* __restrict__ img, long long pitch, int W, int H, const uint8_t* lut,
                                   uint8_t* om_h, uint8_t* om_v) {
    for (int qn = blockIdx.x * blockDim.x + threadIdx.x; qn < W * H; qn += gridDim.x * blockDim.x) {
        const int y = qn / W, x = qn - y * W;
        const int i = img[(size_t)y * pitch + x];
        om_h[qn] = x + 1 < W ? lut[abs(i - (int)img[(size_t)y * pitch + x + 1])] : 16;
        om_v[qn] = y + 1 < H ? lut[abs(i - (int)img[(size_t)(y + 1) * pitch + x])] : 16;
    }
}

__global__ void __launch_bounds__(256)
hmg_energy_kernel(const uint8_t* __restrict__ D, const uint8_t* __restrict__ lab, int W, int H, int K, int KP,
                  int fbits, int w_h, int w_v, int e1, int e2, int delta, int c, const uint8_t* om_h,
                  const uint8_t* om_v, long long* energy, int32_t* bad) {
    long long e = 0;
    bool oob = false;
    auto V = [&](int w, int om, int d) -> long long {
        d = abs(d);
        const int lin = e1 * min(d, delta) + e2 * max(d - delta, 0);
        return ((long long)w * om * min(lin, c)) >> 4;
    };
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < W * H; q += gridDim.x * blockDim.x) {
        const int y = q / W, x = q - y * W;
        const int l = lab[q];
        oob |= l >= K;
        e += (long long)D[(size_t)q * KP + min(l, K - 1)] << fbits;
        if (x + 1 < W) e += V(w_h, om_h ? om_h[q] : 16, l - (int)lab[q + 1]);
        if (y + 1 < H) e += V(w_v, om_v ? om_v[q] : 16, l - (int)lab[q + W]);
    }
    if (oob && bad) *bad = 1;
    for (int d = 16; d > 0; d >>= 1) e += __shfl_down_sync(0xffffffffu, e, d);
    __shared__ long long part[8];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long s = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[w];
        atomicAdd(reinterpret_cast<unsigned long long*>(energy), (unsigned long long)s);
    }
}

// Leaf blocks: every subchain of level `lev` (<= kGLeaf nodes) is finished
// on chip by one warp -- the remaining levels of the hierarchy depth first
// (a pending right part with its boundary messages on a shared-memory stack),
// then each single node emitted: lambda = L + F + R
// (R8), record L + R + D 2^F, the node minimum into the bound, last V: the
// lowest-index argmin label.  The same operations on the same operands as
// the level kernels + emit (bit-identical); the block's costs and edge
// weights are staged once, the boundary messages never leave the SM.
#ifndef DMM_GLEAF
#define DMM_GLEAF 12          // measured: 8 -> 15.5, 12 -> 15.0, 16 -> 16.3 ms (C2, general penalty)
#endif
constexpr int kGLeaf = DMM_GLEAF;
static_assert(kGLeaf >= 2 && kGLeaf <= 16, "leaf stack: 4 pending right parts");

template <int LPL>   // ints per warp: F rows, 2 padded Msg rows, stack (4 x 2 vectors), edge weights
constexpr int kLeafInts = kGLeaf * 32 * LPL + 6 * 32 * LPL + 8 * 32 * LPL + kGLeaf;

template <int LPL, bool FIRST>
__global__ void __launch_bounds__(kGW * 32) hmg_leaf_kernel(GenArgs a, int lev, int ntasks) {
    constexpr int KP = 32 * LPL;
    extern __shared__ int gsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int* wbase = gsm + warp * kLeafInts<LPL>;
    int* sF = wbase;                                          // [kGLeaf][KP]
    int* sx = padded_rows<LPL>(wbase + kGLeaf * KP, 2, lane);
    int* sy = sx + 3 * KP;
    int* stk = wbase + kGLeaf * KP + 6 * KP;                  // [4][2][KP]: pending (L, R)
    int* som = stk + 8 * KP;                                  // [kGLeaf] edge weights
    const int* vt = fill_vtab(gsm + kGW * kLeafInts<LPL>, a);
    long long bsum = 0;
    for (int t = blockIdx.x * kGW + warp; t < ntasks; t += gridDim.x * kGW) {
        const int chain = t >> lev, s = t & ((1 << lev) - 1);
        GenPass<LPL> g(a, chain, lane, sx, vt);
        int lo = 0, hi = g.n - 1;
        for (int b = lev - 1; b >= 0; --b) {
            const int mid = lo + (hi - lo + 1) / 2 - 1;
            if ((s >> b) & 1) lo = mid + 1; else hi = mid;
        }
        if (hi < lo) continue;                                // empty (a single node's left part)
        DMM_CHECK(lo >= 0 && hi < g.n && hi - lo + 1 <= kGLeaf);
        __syncwarp();
        for (int p = lo; p <= hi; ++p) {                      // stage the block's costs and weights
            uint32_t r[LPL];
            g.template ldraw<FIRST>(p, r);
            int F[LPL];
            g.template expand<FIRST>(r, F);
#pragma unroll
            for (int e = 0; e < LPL; ++e) sF[(p - lo) * KP + lane * LPL + e] = F[e];
        }
        if (lane < hi - lo) som[lane] = g.om(lo + lane);
        int L[LPL], R[LPL];
        if (lev == 0) {
#pragma unroll
            for (int e = 0; e < LPL; ++e) { L[e] = 0; R[e] = 0; }
        } else {
            g.ld(a.Lb, lo, L);
            g.ld(a.Rb, hi, R);
        }
        __syncwarp();
        auto Fof = [&](int p, int e) { return sF[(p - lo) * KP + lane * LPL + e]; };
        int sl[4], sh[4], depth = 0;                          // pending right parts [sl, sh]
        int cl = lo, ch = hi;
        while (true) {
            if (cl == ch) {                                   // a leaf node: emit
                const size_t base = g.q(cl) * a.KP + lane * LPL;
                int lmin = kBigG, arg = 0x7fffffff, lam[LPL];
#pragma unroll
                for (int e = 0; e < LPL; ++e) {
                    const int k = lane * LPL + e;
                    const int Ds = (int)a.D[base + e] << a.fbits;
                    const int F = FIRST ? Ds : a.src[base + e];
                    const int lr = L[e] + R[e];
                    lam[e] = lr + F;
                    a.dst[base + e] = k < a.K ? lr + Ds : 0;
                    if (k < a.K) lmin = min(lmin, lam[e]);
                }
                const int m = __reduce_min_sync(0xffffffffu, lmin);
                bsum += m;
                if (a.last && a.vert) {
#pragma unroll
                    for (int e = LPL - 1; e >= 0; --e)
                        if (lane * LPL + e < a.K && lam[e] == m) arg = lane * LPL + e;
                    arg = __reduce_min_sync(0xffffffffu, arg);
                    if (lane == 0) a.labels[g.q(cl)] = (uint8_t)arg;
                }
                if (depth == 0) break;
                --depth;                                      // the pending right part
                cl = sl[depth];
                ch = sh[depth];
#pragma unroll
                for (int e = 0; e < LPL; ++e) {
                    L[e] = stk[(2 * depth) * KP + lane * LPL + e];
                    R[e] = stk[(2 * depth + 1) * KP + lane * LPL + e];
                }
                continue;
            }
            const int len = ch - cl + 1, i = cl + len / 2 - 1, j = i + 1;
            int pl[LPL], pr[LPL];
#pragma unroll
            for (int e = 0; e < LPL; ++e) { pl[e] = L[e]; pr[e] = R[e]; }
            const int nl = i - cl, nr = ch - j, ns = max(nl, nr);
            for (int u = 0; u < ns; ++u) {                    // the two passes, interleaved
                const bool dl = u < nl, dr = u < nr;
                const int pL = dl ? cl + u : cl, pR = dr ? ch - u : ch;
                int xl[LPL], xr[LPL];
#pragma unroll
                for (int e = 0; e < LPL; ++e) { xl[e] = pl[e] + Fof(pL, e); xr[e] = pr[e] + Fof(pR, e); }
                g.msg2(xl, som[pL - lo], xr, som[max(pR - 1, lo) - lo], sy);
#pragma unroll
                for (int e = 0; e < LPL; ++e) {
                    pl[e] = dl ? xl[e] : pl[e];
                    pr[e] = dr ? xr[e] : pr[e];
                }
            }
            // Handshake (Alg.5, literal three Msg; readings R9, R10)
            const int omij = som[i - lo];
            int pji[LPL], t_[LPL], b_[LPL];
#pragma unroll
            for (int e = 0; e < LPL; ++e) pji[e] = Fof(j, e) + pr[e];
            g.msg(pji, omij);
#pragma unroll
            for (int e = 0; e < LPL; ++e) t_[e] = (pl[e] + Fof(i, e) - pji[e]) >> 1;
            g.msg(t_, omij);
#pragma unroll
            for (int e = 0; e < LPL; ++e) b_[e] = -t_[e];
            g.msg(b_, omij);
            // push [j, ch] with (phi_ij, R); continue with [cl, i] and (L, phi_ji')
            DMM_CHECK(depth < 4);
            sl[depth] = j;
            sh[depth] = ch;
#pragma unroll
            for (int e = 0; e < LPL; ++e) {
                stk[(2 * depth) * KP + lane * LPL + e] = t_[e];
                stk[(2 * depth + 1) * KP + lane * LPL + e] = R[e];
                R[e] = b_[e];
            }
            ++depth;
            ch = i;
        }
    }
    if (lane == 0 && bsum != 0) atomicAdd(reinterpret_cast<unsigned long long*>(a.bound), (unsigned long long)bsum);
}

#ifndef DMM_CTA_TASKS
#define DMM_CTA_TASKS 1024
#endif
constexpr int kCtaTasks = DMM_CTA_TASKS;          // levels with at most this many tasks: hmg_level_cta_kernel

template <int LPL>
void run_half(const GenArgs& a, int chains, int n, cudaStream_t s, long long& launches) {
    hmg_ends_kernel<<<148, 256, 0, s>>>(a, chains, n);
    // level kernels down to the first level whose subchains (<= ceil(n / 2^l)
    // nodes) fit a leaf block; the leaf kernel finishes and emits
    int lstar = 0;
    while (((n + (1 << lstar) - 1) >> lstar) > kGLeaf) ++lstar;
    const int smem = 6 * kGW * 32 * LPL * 4 + (int)vtab_bytes(a.dc);
    static bool lattr = [] {          // over 48 KB for large kGW x LPL
        const int b = 6 * kGW * 32 * LPL * 4 + (int)vtab_bytes(256);
        cudaFuncSetAttribute(hmg_level_kernel<LPL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
        cudaFuncSetAttribute(hmg_level_kernel<LPL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
        return true;
    }();
    (void)lattr;
    for (int lev = 0; lev < lstar; ++lev) {
        const long long nt = (long long)chains << lev;
        const int ntasks = (int)nt;
        if (ntasks <= kCtaTasks) {                  // few long tasks: a CTA per task
            constexpr int KP = 32 * LPL;
            const size_t cs = (12 * KP + 4 * (KP / 32)) * sizeof(int) + vtab_bytes(a.dc);
            if (a.first)
                hmg_level_cta_kernel<KP, true><<<ntasks, KP, cs, s>>>(a, lev, ntasks);
            else
                hmg_level_cta_kernel<KP, false><<<ntasks, KP, cs, s>>>(a, lev, ntasks);
            continue;
        }
        int grid = (ntasks + kGW - 1) / kGW;
        if (grid > 148 * 16) grid = 148 * 16;
        if (a.first)
            hmg_level_kernel<LPL, true><<<grid, kGW * 32, smem, s>>>(a, lev, ntasks);
        else
            hmg_level_kernel<LPL, false><<<grid, kGW * 32, smem, s>>>(a, lev, ntasks);
    }
    {
        static bool attr = [] {
            const int b = kGW * kLeafInts<LPL> * 4 + (int)vtab_bytes(256);
            cudaFuncSetAttribute(hmg_leaf_kernel<LPL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
            cudaFuncSetAttribute(hmg_leaf_kernel<LPL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
            return true;
        }();
        (void)attr;
        const int ntasks = chains << lstar;
        int grid = (ntasks + kGW - 1) / kGW;
        if (grid > 148 * 8) grid = 148 * 8;
        const int lsm = kGW * kLeafInts<LPL> * 4 + (int)vtab_bytes(a.dc);
        if (a.first)
            hmg_leaf_kernel<LPL, true><<<grid, kGW * 32, lsm, s>>>(a, lstar, ntasks);
        else
            hmg_leaf_kernel<LPL, false><<<grid, kGW * 32, lsm, s>>>(a, lstar, ntasks);
    }
    launches += 2 + lstar;
}

// Iterative minorant (Alg.4, readings R32): one CTA of KP threads
// per chain, one label per thread (the sweeps are one long dependent chain of
// Msg per chain, so the per-step latency is what counts: a label per thread
// keeps each Msg's window loop at two shared loads per distance).  `passes`
// sweeps alternating direction (the first from node 0), each preceded by the
// far-side messages of the current remainder f - lambda (stored in Lb);
// lambda (in Rb) += floor(m_i / 2^gshift) with the dynamic min-marginal m_i,
// the last pass with gamma = 1.  A Msg: the thread stages its value in one of
// two padded rows (alternating, so one CTA barrier per Msg orders both the
// row and the warp minima), the CTA minimum gives the cap, then the window.
// Node costs / Lb / Rb of the next kPreIt steps are fetched ahead.
constexpr int kPreIt = 4;

template <int KP, bool FIRST>
__global__ void __launch_bounds__(KP) hmg_iter_kernel(GenArgs a, int chains) {
    constexpr int NW = KP / 32, R = kPreIt;
    extern __shared__ int gsm[];
    int* rows = gsm;                                  // 2 x [pad KP | row KP | pad KP]
    int* wmin = gsm + 6 * KP;                         // 2 x NW warp minima
    const int k = threadIdx.x, lane = k & 31, warp = k >> 5;
    for (int r = 0; r < 2; ++r) { rows[r * 3 * KP + k] = kBigG; rows[r * 3 * KP + 2 * KP + k] = kBigG; }
    const int* vt = fill_vtab(gsm + 6 * KP + 2 * NW, a);     // (its barrier also covers the pads)
    const bool in = k < a.K;
    int par = 0;
    auto msg = [&](int x, int om) -> int {            // Msg over an edge of weight om, at label k
        if (!in) x = kBigG;
        int* row = rows + par * 3 * KP + KP;
        row[k] = x;
        const int mw = __reduce_min_sync(0xffffffffu, x);
        if (lane == 0) wmin[par * NW + warp] = mw;
        __syncthreads();
        int m = wmin[par * NW];
#pragma unroll
        for (int w = 1; w < NW; ++w) m = min(m, wmin[par * NW + w]);
        const int* tv = vt + om * (a.dc + 1);
        const int cap = m + tv[a.dc];
        int best = min(cap, x);
#pragma unroll 4
        for (int d = 1; d < a.dc; ++d) {              // out-of-range sources: kBigG pads / labels >= K
            const int v = tv[d];
            best = min(best, row[k - d] + v);
            best = min(best, row[k + d] + v);
        }
        par ^= 1;
        return in ? best : cap;
    };
    const int n = a.vert ? a.H : a.W;
    const int fbits = a.fbits;
    const long long pst = a.vert ? a.W : 1;           // node stride of a chain (pixels)
    for (int ch = blockIdx.x; ch < chains; ch += gridDim.x) {
        // this thread's label of the chain's node p in the [H][W][KP] arrays: cb + p * est
        const long long c0 = a.vert ? ch : (long long)ch * a.W;
        const long long cb = c0 * KP + k, est = pst * KP;
        const uint8_t* Dp = a.D + cb;
        const int32_t* Sp = a.src + cb;
        int32_t* Lp = a.Lb + cb;
        int32_t* Rp = a.Rb + cb;
        const uint8_t* Op = a.om ? a.om + c0 : nullptr;
        auto ldF = [&](int p) -> int {                // raw: D byte (FIRST) or the int32 record
            return FIRST ? (int)Dp[p * est] : Sp[p * est];
        };
        auto F_of = [&](int raw) -> int { return !in ? kBigG : (FIRST ? raw << fbits : raw); };
        auto om_of = [&](int e) -> int { return Op ? (int)Op[e * pst] : 16; };
        for (int p = 0; p < n; ++p) Rp[p * est] = 0;
        for (int s = 0; s < a.passes; ++s) {
            const int dir = (s & 1) ? -1 : 1;
            const int sh = s == a.passes - 1 ? 0 : a.gshift;
            const int start = dir > 0 ? n - 1 : 0;  // far end
            int psi = 0;
            Lp[start * est] = psi;
            {   // far-side messages: step u reads node src = start - dir u, writes i = src - dir
                int rf[R], rl[R], ro[R];
#pragma unroll
                for (int j = 0; j < R; ++j)
                    if (j < n - 1) {
                        const int src = start - dir * j;
                        rf[j] = ldF(src);
                        rl[j] = Rp[src * est];
                        ro[j] = om_of(dir > 0 ? src - 1 : src);
                    }
                for (int u0 = 0; u0 < n - 1; u0 += R) {
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const int u = u0 + j;
                        if (u >= n - 1) break;
                        psi += F_of(rf[j]) - rl[j];
                        const int om = ro[j];
                        if (u + R < n - 1) {
                            const int src = start - dir * (u + R);
                            rf[j] = ldF(src);
                            rl[j] = Rp[src * est];
                            ro[j] = om_of(dir > 0 ? src - 1 : src);
                        }
                        psi = msg(psi, om);
                        Lp[(start - dir * (u + 1)) * est] = psi;
                    }
                }
            }
            int phi = 0;
            {   // the sweep: step u at node i = i0 + dir u (edge min(i, i + dir) when u < n - 1)
                const int i0 = dir > 0 ? 0 : n - 1;
                int rf[R], rl[R], rp[R], ro[R];
#pragma unroll
                for (int j = 0; j < R; ++j)
                    if (j < n) {
                        const int i = i0 + dir * j;
                        rf[j] = ldF(i);
                        rl[j] = Rp[i * est];
                        rp[j] = Lp[i * est];
                        ro[j] = j < n - 1 ? om_of(dir > 0 ? i : i - 1) : 16;
                    }
                for (int u0 = 0; u0 < n; u0 += R) {
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const int u = u0 + j;
                        if (u >= n) break;
                        const int i = i0 + dir * u;
                        const int F = F_of(rf[j]);
                        int lam = rl[j];
                        const int m = phi + F - lam + rp[j];      // min-marginal of f - lambda at i
                        lam += sh ? (m >> sh) : m;
                        const int om = ro[j];
                        if (u + R < n) {
                            const int i2 = i0 + dir * (u + R);
                            rf[j] = ldF(i2);
                            rl[j] = Rp[i2 * est];
                            rp[j] = Lp[i2 * est];
                            ro[j] = u + R < n - 1 ? om_of(dir > 0 ? i2 : i2 - 1) : 16;
                        }
                        Rp[i * est] = lam;
                        if (u < n - 1) phi = msg(phi + F - lam, om);
                    }
                }
            }
        }
    }
}

template <int LPL>
void run_iter(const GenArgs& a, int chains, cudaStream_t s, long long& launches) {
    constexpr int KP = 32 * LPL;
    const size_t smem = (6 * KP + 2 * (KP / 32)) * sizeof(int) + vtab_bytes(a.dc);
    int grid = chains < 148 * 16 ? chains : 148 * 16;
    if (a.first)
        hmg_iter_kernel<KP, true><<<grid, KP, smem, s>>>(a, chains);
    else
        hmg_iter_kernel<KP, false><<<grid, KP, smem, s>>>(a, chains);
    hmg_emit_kernel<LPL><<<148 * 8, kGW * 32, 0, s>>>(a);
    launches += 2;
}

}  // namespace

size_t gen_bytes(int W, int H, int KP) { return 2 * (size_t)W * H * KP * 4 + 2 * (size_t)W * H + 256; }

bool gen_mode(const dmm_config* c) {
    return c->pen_e1 || c->pen_e2 || c->pen_delta || c->pen_c || c->edge_weights || c->minorant;
}

void gen_weights(dmm_ctx* ctx, int frame, const uint8_t* left, int64_t pitch, cudaStream_t s) {
    FramePtrs P = frame_ptrs(ctx->L, frame);
    uint8_t* lut = P.gom_v + (size_t)ctx->L.W * ctx->L.H;
    hmg_weights_kernel<<<4 * 148, 256, 0, s>>>(left, pitch, ctx->L.W, ctx->L.H, lut, P.gom_h, P.gom_v);
    ++ctx->launches;
}

void gen_half(dmm_ctx* ctx, int frame, int nframes, int t, int v, int iterations, cudaStream_t s) {
    const dmm_config& c = ctx->cfg;
    for (int f = frame; f < frame + nframes; ++f) {
        FramePtrs P = frame_ptrs(ctx->L, f);
        GenArgs a;
        a.D = P.D;
        a.src = v ? P.gfv : P.ggh;
        a.dst = v ? P.ggh : P.gfv;
        a.Lb = P.fwd;
        a.Rb = P.bwd;
        a.om = c.edge_weights ? (v ? P.gom_v : P.gom_h) : nullptr;
        a.labels = P.labels;
        a.bound = P.bounds + 2 * t + v;
        a.W = ctx->L.W; a.H = ctx->L.H; a.K = ctx->K; a.KP = ctx->KP;
        a.vert = v; a.first = (t == 0 && v == 0); a.last = (t == iterations - 1 && v == 1);
        a.fbits = c.frac_bits;
        a.w = v ? c.w_v : c.w_h;
        pen_of(c, a.e1, a.e2, a.delta, a.c);
        int dc = 0;
        while (dc < ctx->K && genR_host(c, dc) < a.c) ++dc;
        a.dc = dc;
        a.passes = c.iter_passes; a.gshift = c.iter_gshift;
        const int chains = v ? a.W : a.H, n = v ? a.H : a.W;
        if (c.minorant == 1) {
            switch (ctx->KP / 32) {
                case 1: run_iter<1>(a, chains, s, ctx->launches); break;
                case 2: run_iter<2>(a, chains, s, ctx->launches); break;
                case 4: run_iter<4>(a, chains, s, ctx->launches); break;
                default: run_iter<8>(a, chains, s, ctx->launches); break;
            }
            continue;
        }
        switch (ctx->KP / 32) {
            case 1: run_half<1>(a, chains, n, s, ctx->launches); break;
            case 2: run_half<2>(a, chains, n, s, ctx->launches); break;
            case 4: run_half<4>(a, chains, n, s, ctx->launches); break;
            default: run_half<8>(a, chains, n, s, ctx->launches); break;
        }
    }
}

void gen_energy(dmm_ctx* ctx, int frame, int nframes, const uint8_t* labels, int32_t* bad, cudaStream_t s) {
    const dmm_config& c = ctx->cfg;
    for (int f = frame; f < frame + nframes; ++f) {
        FramePtrs P = frame_ptrs(ctx->L, f);
        int blocks = (ctx->L.W * ctx->L.H + 255) / 256;
        if (blocks > 4 * 148) blocks = 4 * 148;
        int e1, e2, dl, cc;
        pen_of(c, e1, e2, dl, cc);
        hmg_energy_kernel<<<blocks, 256, 0, s>>>(P.D, labels ? labels : P.labels, ctx->L.W, ctx->L.H, ctx->K, ctx->KP,
                                                 c.frac_bits, c.w_h, c.w_v, e1, e2, dl, cc,
                                                 c.edge_weights ? P.gom_h : nullptr, c.edge_weights ? P.gom_v : nullptr,
                                                 P.energy, bad);
        ++ctx->launches;
    }
}

// The penalty of the general kernels: the config's, or (all zero: the classic
// model in general storage, e.g. for the iterative minorant) e1 = e2 = 2^F,
// delta = 0, c = T 2^F, i.e. V = w min(|d|, T) 2^F with om = 16.
void pen_of(const dmm_config& c, int& e1, int& e2, int& delta, int& cc) {
    if (c.pen_e1 || c.pen_e2 || c.pen_delta || c.pen_c) {
        e1 = c.pen_e1; e2 = c.pen_e2; delta = c.pen_delta; cc = c.pen_c;
    } else {
        e1 = e2 = 1 << c.frac_bits; delta = 0; cc = c.trunc << c.frac_bits;
    }
}

int genR_host(const dmm_config& c, int d) {
    int e1, e2, delta, cc;
    pen_of(c, e1, e2, delta, cc);
    const long long lin = (long long)e1 * (d < delta ? d : delta) + (long long)e2 * (d > delta ? d - delta : 0);
    return (int)(lin < cc ? lin : cc);
}

}  // namespace dmm
