// hm.cu -- Dual MM half-steps (Algorithm 2) for sm_100a: every row
// (H pass) or column (V pass) chain builds its hierarchical minorant
// with Handshakes (Alg.5).
//
// Mapping:
//  * one CTA per chain, NW warps; a warp owns one K-vector at a time with the
//    label dimension in registers, LPL = KP/32 consecutive labels per lane.
//  * Msg (Eq. msg-pass, Msg of Alg.5) for
//    f_ij = ws*min(|a-b|, T) is computed exactly: in-lane forward/backward
//    envelopes, a one-hop neighbour exchange (2 shuffles) when T <= LPL + 1 or a
//    Kogge-Stone min-plus scan otherwise, and the truncation cap
//    min(a) + ws*T from one redux.sync.min.
//  * "global levels" (subchains longer than kCMax): processed breadth first,
//    one warp per subchain; only the message direction whose boundary changed
//    is recomputed (Fig.11's dots are reused: the "spine" messages a later level
//    needs are kept in the fwd/bwd scratch arrays, L2-resident).  Node data
//    F = D*2^F + g_ (H) or f_ (V) streams through a per-warp cp.async ring of
//    kRing slots whose producer runs ahead across level barriers (the data
//    does not depend on the messages).
//  * "leaf blocks" (the 2^l* subchains of length <= kCMax): one warp stages the
//    block's F in shared memory and finishes its whole sub-hierarchy on chip,
//    depth first, with the forward and backward passes of each piece
//    interleaved (two independent Msg chains -> ILP).  Leaves [p,p] with
//    boundary messages L, R give lambda = L + F + R (reading R8):
//    H writes f_ = lambda - g_ = L + D*2^F + R, V writes g_ = lambda - f_ = L + R;
//    the node minima sum to the dual bound (exactness) and the last V pass
//    writes the lowest-index argmin as the label (R13, R14).
//  * chains are launched in L2-sized waves (host side) so the global levels'
//    re-reads of F hit the 126 MB L2.
// All arithmetic is exact int32 (ranges in DESIGN.md): bit-identical to the
// CPU oracle whatever the evaluation order.
#include "hm_device.cuh"

namespace dmm {

// ------------------------------------------------------------ the kernel
struct HmShared {   // per-warp shared memory carve-up (bytes)
    int ring, leafF, leafD, stack, stackIdx, total;
    __host__ __device__ HmShared(int KP, bool vert) {
        const int rec = vert ? KP * 4 : KP * 5;
        ring = 0;
        leafF = ring + kRing * rec;
        leafD = leafF + kCMax * KP * 4;
        stack = leafD + (vert ? 0 : kCMax * KP);
        stackIdx = stack + kDepth * 2 * KP * 4;
        total = stackIdx + kDepth * 8;
        total = (total + 127) & ~127;
    }
};

// [lo, hi] of subchain s (bit-path from the root, MSB first) at level lev.
__device__ __forceinline__ void task_bounds(int n, int lev, int s, int& lo, int& hi) {
    lo = 0; hi = n - 1;
    for (int b = lev - 1; b >= 0; --b) {
        const int mid = lo + (hi - lo + 1) / 2 - 1;
        if ((s >> b) & 1) lo = mid + 1; else hi = mid;
    }
}

// Producer side of the ring: enumerates, in consumption order, the nodes whose
// F this warp will read (global-level passes, Handshake nodes j then i, then
// the leaf blocks' nodes in ascending order).
struct NodeSeq {
    int n, lstar, warp, nw;
    int lev, s, p, step, left, hs, hj, hi_;
    bool done;
    __device__ __forceinline__ void start() {
        while (true) {
            if (lev > lstar) { done = true; return; }
            if (lev == 0 && lstar > 0) {
                if (s <= 1) {
                    const int i = n / 2 - 1, j = i + 1;
                    if (s == 0) { p = 0; step = 1; left = i; hs = 2; hj = j; hi_ = i; }
                    else { p = n - 1; step = -1; left = n - 1 - j; hs = 0; }
                    return;
                }
            } else if (s < (1 << lev)) {
                int lo, hi;
                task_bounds(n, lev, s, lo, hi);
                if (lev == lstar) { p = lo; step = 1; left = hi - lo + 1; hs = 0; return; }
                const int i = lo + (hi - lo + 1) / 2 - 1, j = i + 1;
                if (!(s & 1)) { p = hi; step = -1; left = hi - j; }
                else { p = lo; step = 1; left = i - lo; }
                hs = 2; hj = j; hi_ = i;
                return;
            }
            ++lev; s = warp;
        }
    }
    __device__ __forceinline__ void init(int n_, int lstar_, int warp_, int nw_) {
        n = n_; lstar = lstar_; warp = warp_; nw = nw_; lev = 0; s = warp_; done = false;
        start();
    }
    __device__ __forceinline__ bool next(int& node) {
        while (!done) {
            if (left > 0) { node = p; p += step; --left; return true; }
            if (hs == 2) { node = hj; hs = 1; return true; }
            if (hs == 1) { node = hi_; hs = 0; return true; }
            s += nw;
            start();
        }
        return false;
    }
};

template <int LPL, bool VERT, bool PAD, bool WIN>
struct Hm {
    static constexpr int KP = 32 * LPL;
    FramePtrs P;
    int W, K, c, lane, n;
    int fbits, ws, wsT;
    bool first, last;
    char* ring;
    int rec;
    NodeSeq seq;
    int t, issued;
    long long bsum;

    __device__ __forceinline__ size_t q_of(int p) const {
        return VERT ? (size_t)p * W + c : (size_t)c * W + p;
    }
    __device__ __forceinline__ size_t off(int p) const { return q_of(p) * KP + lane * LPL; }
    __device__ __forceinline__ void msg_(int (&x)[LPL]) const { msg<LPL, PAD, WIN>(x, ws, wsT, lane, K); }

    // ---- ring
    __device__ __forceinline__ void issue() {
        int node;
        if (seq.next(node)) {
            char* slot = ring + (issued % kRing) * rec;
            const size_t q = q_of(node);
            if constexpr (VERT) {
                const char* src = reinterpret_cast<const char*>(P.fdual + q * KP);
#pragma unroll
                for (int ch = lane; ch < KP / 4; ch += 32) cp_async16(slot + 16 * ch, src + 16 * ch);
            } else {
                if (!first) {
                    const char* src = reinterpret_cast<const char*>(P.gdual + q * KP);
#pragma unroll
                    for (int ch = lane; ch < KP / 4; ch += 32) cp_async16(slot + 16 * ch, src + 16 * ch);
                }
                const char* srcd = reinterpret_cast<const char*>(P.D + q * KP);
                if (lane < KP / 16) cp_async16(slot + KP * 4 + 16 * lane, srcd + 16 * lane);
            }
        }
        cp_async_commit();
        ++issued;
    }
    __device__ __forceinline__ void prologue() {
#pragma unroll 1
        for (int k = 0; k < kRing - 1; ++k) issue();
    }
    // Next F (and D for H) in consumption order.
    __device__ __forceinline__ void pop(int (&F)[LPL], int (&Dv)[LPL]) {
        issue();
        cp_async_wait<kRing - 1>();
        __syncwarp();
        const char* slot = ring + (t % kRing) * rec;
        ++t;
        if constexpr (VERT) {
            ld_i32<LPL>(reinterpret_cast<const int32_t*>(slot) + lane * LPL, F);
        } else {
            ld_u8<LPL>(reinterpret_cast<const uint8_t*>(slot + KP * 4) + lane * LPL, Dv);
            if (!first) {
                ld_i32<LPL>(reinterpret_cast<const int32_t*>(slot) + lane * LPL, F);
#pragma unroll
                for (int e = 0; e < LPL; ++e) F[e] += Dv[e] << fbits;
            } else {
#pragma unroll
                for (int e = 0; e < LPL; ++e) F[e] = Dv[e] << fbits;
            }
        }
        __syncwarp();
    }

    // ---- global-level passes (messages in the fwd/bwd scratch arrays)
    __device__ __forceinline__ void pass_fwd(int lo, int end, int (&phi)[LPL]) {
        const int len0 = end - lo + 1;
        if (len0 < 2) return;
        int kk = (31 - __clz(len0)) - 1;          // spine: nodes lo + (len0 >> k) - 1
        int target = len0 >> kk;
#pragma unroll 1
        for (int p = lo; p < end; ++p) {
            int F[LPL], Dv[LPL];
            pop(F, Dv);
#pragma unroll
            for (int e = 0; e < LPL; ++e) phi[e] += F[e];
            msg_(phi);
            if (p + 2 - lo == target) {
                st_i32<LPL>(P.fwd + off(p + 1), phi);
                --kk;
                target = kk >= 0 ? (len0 >> kk) : INT_MAX;
            }
        }
    }
    __device__ __forceinline__ void pass_bwd(int hi, int end, int (&phi)[LPL]) {
        const int lenB = hi - end + 1;
        if (lenB < 2) return;
        int kk = 31 - __clz(lenB - 1);            // spine: nodes hi - ceil(lenB/2^k) + 1
        int target = ((lenB - 1) >> kk) + 1;
#pragma unroll 1
        for (int p = hi; p > end; --p) {
            int F[LPL], Dv[LPL];
            pop(F, Dv);
#pragma unroll
            for (int e = 0; e < LPL; ++e) phi[e] += F[e];
            msg_(phi);
            if (hi - p + 2 == target) {
                st_i32<LPL>(P.bwd + off(p - 1), phi);
                --kk;
                target = kk >= 0 ? (((lenB - 1) >> kk) + 1) : INT_MAX;
            }
        }
    }
    // Handshake (Alg.5, R9/R10); Fj, Fi popped in that order.  On exit pl =
    // phi_ij (left boundary of the right piece), pr = phi_ji' (right boundary
    // of the left piece).
    __device__ __forceinline__ void handshake(const int (&Fi)[LPL], const int (&Fj)[LPL], int (&pl)[LPL],
                                              int (&pr)[LPL]) {
        handshake_regs<LPL, PAD, WIN>(Fi, Fj, pl, pr, ws, wsT, lane, K);
    }
    __device__ __forceinline__ void global_handshake(int i, int (&pl)[LPL], int (&pr)[LPL]) {
        int Fi[LPL], Fj[LPL], Dv[LPL];
        pop(Fj, Dv);
        pop(Fi, Dv);
        handshake(Fi, Fj, pl, pr);
        st_i32<LPL>(P.fwd + off(i + 1), pl);
        st_i32<LPL>(P.bwd + off(i), pr);
    }

    // ---- leaves
    __device__ __forceinline__ void emit(int node, const int (&L)[LPL], const int (&F)[LPL], const int (&Dv)[LPL],
                                         const int (&R)[LPL]) {
        int lam[LPL], o[LPL];
        int lmin = INT_MAX;
#pragma unroll
        for (int e = 0; e < LPL; ++e) {
            const int lr = L[e] + R[e];
            o[e] = VERT ? lr : lr + (Dv[e] << fbits);
            lam[e] = lr + F[e];
            if (PAD && lane * LPL + e >= K) { o[e] = 0; lam[e] = INT_MAX; }
            lmin = min(lmin, lam[e]);
        }
        st_i32<LPL>((VERT ? P.gdual : P.fdual) + off(node), o);
        const int gmin = __reduce_min_sync(kFull, lmin);
        bsum += gmin;
        if (VERT && last) {
            int kmin = INT_MAX;
#pragma unroll
            for (int e = LPL - 1; e >= 0; --e)
                if (lam[e] == gmin) kmin = lane * LPL + e;
            kmin = __reduce_min_sync(kFull, kmin);
            if (lane == 0) P.labels[q_of(node)] = (uint8_t)kmin;
        }
    }

    // Whole sub-hierarchy of the block [lo0, lo0+m-1] on chip (depth first; the
    // pieces' forward / backward passes recompute both directions).
    __device__ __forceinline__ void leaf_block(int lo0, int m, int (&L)[LPL], int (&R)[LPL], int32_t* sF,
                                               uint8_t* sD, int32_t* stk, int* stkIdx) {
#pragma unroll 1
        for (int k = 0; k < m; ++k) {
            int F[LPL], Dv[LPL];
            pop(F, Dv);
            st_i32<LPL>(sF + k * KP + lane * LPL, F);
            if constexpr (!VERT) st_u8<LPL>(sD + k * KP + lane * LPL, Dv);
        }
        __syncwarp();
        int lo = 0, hi = m - 1, sp = 0;
#pragma unroll 1
        while (true) {
            if (lo == hi) {
                int F[LPL], Dv[LPL];
                ld_i32<LPL>(sF + lo * KP + lane * LPL, F);
                if constexpr (!VERT) ld_u8<LPL>(sD + lo * KP + lane * LPL, Dv);
                emit(lo0 + lo, L, F, Dv, R);
                if (sp == 0) break;
                --sp;
                __syncwarp();
                lo = stkIdx[2 * sp]; hi = stkIdx[2 * sp + 1];
                ld_i32<LPL>(stk + (2 * sp) * KP + lane * LPL, L);
                ld_i32<LPL>(stk + (2 * sp + 1) * KP + lane * LPL, R);
                continue;
            }
            const int len = hi - lo + 1, i = lo + len / 2 - 1, j = i + 1;
            int pl[LPL], pr[LPL];
#pragma unroll
            for (int e = 0; e < LPL; ++e) { pl[e] = L[e]; pr[e] = R[e]; }
            const int nf = i - lo, nb = hi - j;
#pragma unroll 1
            for (int s = 0; s < nf || s < nb; ++s) {
                if (s < nf) {
                    int F[LPL];
                    ld_i32<LPL>(sF + (lo + s) * KP + lane * LPL, F);
#pragma unroll
                    for (int e = 0; e < LPL; ++e) pl[e] += F[e];
                    msg_(pl);
                }
                if (s < nb) {
                    int F[LPL];
                    ld_i32<LPL>(sF + (hi - s) * KP + lane * LPL, F);
#pragma unroll
                    for (int e = 0; e < LPL; ++e) pr[e] += F[e];
                    msg_(pr);
                }
            }
            int Fi[LPL], Fj[LPL];
            ld_i32<LPL>(sF + i * KP + lane * LPL, Fi);
            ld_i32<LPL>(sF + j * KP + lane * LPL, Fj);
            handshake(Fi, Fj, pl, pr);
            // push the right piece (j, hi, phi_ij, R); continue with (lo, i, L, phi_ji')
            if (lane == 0) { stkIdx[2 * sp] = j; stkIdx[2 * sp + 1] = hi; }
            st_i32<LPL>(stk + (2 * sp) * KP + lane * LPL, pl);
            st_i32<LPL>(stk + (2 * sp + 1) * KP + lane * LPL, R);
            ++sp;
            hi = i;
#pragma unroll
            for (int e = 0; e < LPL; ++e) R[e] = pr[e];
        }
    }
};

template <int LPL, bool VERT, bool PAD, bool WIN, int NW>
__global__ void __launch_bounds__(NW * 32) hm_kernel(PassArgs a, int chain0, int lstar) {
    extern __shared__ __align__(128) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int KP = 32 * LPL;
    const HmShared lay(KP, VERT);
    char* wsm = smem + warp * lay.total;

    Hm<LPL, VERT, PAD, WIN> h;
    h.P = frame_ptrs(a.L, a.frame0 + blockIdx.y);
    h.W = a.L.W; h.K = a.L.K; h.c = chain0 + blockIdx.x; h.lane = lane;
    h.n = VERT ? a.L.H : a.L.W;
    h.fbits = a.fbits; h.ws = a.ws; h.wsT = a.wsT;
    h.first = a.first != 0; h.last = a.last != 0;
    h.ring = wsm + lay.ring;
    h.rec = VERT ? KP * 4 : KP * 5;
    h.t = 0; h.issued = 0; h.bsum = 0;
    const int n = h.n;
    h.seq.init(n, lstar, warp, NW);
    h.prologue();

    int32_t* sF = reinterpret_cast<int32_t*>(wsm + lay.leafF);
    uint8_t* sD = reinterpret_cast<uint8_t*>(wsm + lay.leafD);
    int32_t* stk = reinterpret_cast<int32_t*>(wsm + lay.stack);
    int* stkIdx = reinterpret_cast<int*>(wsm + lay.stackIdx);
    int zero[LPL];
#pragma unroll
    for (int e = 0; e < LPL; ++e) zero[e] = 0;

    if (lstar > 0) {
        // ---- level 0: the whole chain, zero boundary messages
        const int i = n / 2 - 1;
        int pl[LPL], pr[LPL];
#pragma unroll
        for (int e = 0; e < LPL; ++e) { pl[e] = 0; pr[e] = 0; }
        if (warp == 0) { st_i32<LPL>(h.P.fwd + h.off(0), zero); h.pass_fwd(0, i, pl); }
        if (warp == 1) { st_i32<LPL>(h.P.bwd + h.off(n - 1), zero); h.pass_bwd(n - 1, i + 1, pr); st_i32<LPL>(h.P.bwd + h.off(i + 1), pr); }
        __syncthreads();
        if (warp == 0) {
            ld_i32<LPL>(h.P.bwd + h.off(i + 1), pr);
            h.global_handshake(i, pl, pr);
        }
        __syncthreads();
        // ---- global levels 1 .. lstar-1
#pragma unroll 1
        for (int lev = 1; lev < lstar; ++lev) {
#pragma unroll 1
            for (int s = warp; s < (1 << lev); s += NW) {
                int lo, hi;
                task_bounds(n, lev, s, lo, hi);
                const int ii = lo + (hi - lo + 1) / 2 - 1, j = ii + 1;
                if (!(s & 1)) {   // left piece: left boundary kept -> reuse fwd, recompute bwd
                    ld_i32<LPL>(h.P.bwd + h.off(hi), pr);
                    ld_i32<LPL>(h.P.fwd + h.off(ii), pl);
                    h.pass_bwd(hi, j, pr);
                } else {          // right piece: right boundary kept -> reuse bwd, recompute fwd
                    ld_i32<LPL>(h.P.fwd + h.off(lo), pl);
                    ld_i32<LPL>(h.P.bwd + h.off(j), pr);
                    h.pass_fwd(lo, ii, pl);
                }
                h.global_handshake(ii, pl, pr);
            }
            __syncthreads();
        }
    } else {
        if (warp == 0) { st_i32<LPL>(h.P.fwd + h.off(0), zero); st_i32<LPL>(h.P.bwd + h.off(n - 1), zero); }
        __syncthreads();
    }
    // ---- leaf blocks at level lstar
    const int nb = 1 << lstar;
    int L[LPL], R[LPL];
    if (warp < nb) {
        int lo, hi;
        task_bounds(n, lstar, warp, lo, hi);
        ld_i32<LPL>(h.P.fwd + h.off(lo), L);
        ld_i32<LPL>(h.P.bwd + h.off(hi), R);
    }
#pragma unroll 1
    for (int s = warp; s < nb; s += NW) {
        int lo, hi;
        task_bounds(n, lstar, s, lo, hi);
        int L2[LPL], R2[LPL];
        const int s2 = s + NW;
        if (s2 < nb) {      // prefetch the next block's boundary messages
            int lo2, hi2;
            task_bounds(n, lstar, s2, lo2, hi2);
            ld_i32<LPL>(h.P.fwd + h.off(lo2), L2);
            ld_i32<LPL>(h.P.bwd + h.off(hi2), R2);
        }
        h.leaf_block(lo, hi - lo + 1, L, R, sF, sD, stk, stkIdx);
        if (s2 < nb) {
#pragma unroll
            for (int e = 0; e < LPL; ++e) { L[e] = L2[e]; R[e] = R2[e]; }
        }
    }
    cp_async_wait<0>();
    if (lane == 0 && h.bsum != 0)
        atomicAdd(reinterpret_cast<unsigned long long*>(&h.P.bounds[a.bound_slot]),
                  (unsigned long long)h.bsum);
}

// Leaf level: smallest l with ceil(n / 2^l) <= kCMax.
static int leaf_level(int n) {
    int l = 0;
    while (((n + (1 << l) - 1) >> l) > kCMax) ++l;
    return l;
}

template <int LPL, bool PAD, bool WIN>
static void launch_cfg(const PassArgs& a, int vertical, int nframes, int wave_chains, cudaStream_t s) {
    constexpr int NW = 4;
    constexpr int KP = 32 * LPL;
    const int chains = vertical ? a.L.W : a.L.H;
    const int n = vertical ? a.L.H : a.L.W;
    const int lstar = leaf_level(n);
    const HmShared lay(KP, vertical != 0);
    const int smem = NW * lay.total;
    auto kern = vertical ? hm_kernel<LPL, true, PAD, WIN, NW> : hm_kernel<LPL, false, PAD, WIN, NW>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int wave = wave_chains > 0 ? wave_chains : chains;
    for (int c0 = 0; c0 < chains; c0 += wave) {
        const int nc = chains - c0 < wave ? chains - c0 : wave;
        kern<<<dim3(nc, nframes), NW * 32, smem, s>>>(a, c0, lstar);
    }
}

template <int LPL>
static void launch_lpl(const PassArgs& a, int vertical, int nframes, int wave, cudaStream_t s) {
    const bool pad = a.L.K != 32 * LPL;
    const bool win = a.T <= LPL + 1;
    if (pad) {
        if (win) launch_cfg<LPL, true, true>(a, vertical, nframes, wave, s);
        else launch_cfg<LPL, true, false>(a, vertical, nframes, wave, s);
    } else {
        if (win) launch_cfg<LPL, false, true>(a, vertical, nframes, wave, s);
        else launch_cfg<LPL, false, false>(a, vertical, nframes, wave, s);
    }
}

int hm_launches_per_pass(const PassArgs& a, int vertical, int wave) {
    const int chains = vertical ? a.L.W : a.L.H;
    const int w = wave > 0 ? wave : chains;
    return (chains + w - 1) / w;
}

void launch_hm_pass(const PassArgs& a, int vertical, int nframes, int wave, cudaStream_t s) {
    switch (a.L.KP / 32) {
        case 1: launch_lpl<1>(a, vertical, nframes, wave, s); break;
        case 2: launch_lpl<2>(a, vertical, nframes, wave, s); break;
        case 4: launch_lpl<4>(a, vertical, nframes, wave, s); break;
        default: launch_lpl<8>(a, vertical, nframes, wave, s); break;
    }
}

}  // namespace dmm
