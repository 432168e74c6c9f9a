// hm.cu -- Dual MM half-steps (Algorithm 2) for sm_100a: every row
// (H pass) or column (V pass) chain builds its hierarchical minorant
// with Handshakes (Alg.5).
//
// Mapping:
//  * one CTA per chain, NW warps; a warp owns one K-vector at a time with the
//    label dimension in registers, LPL = KP/32 consecutive labels per lane;
//  * Msg (Eq. msg-pass, Msg of Alg.5) for
//    f_ij = ws*min(|a-b|,T) is the exact two-sided distance transform: in-lane
//    forward/backward envelopes, a Kogge-Stone min-plus scan across lanes with
//    shuffles (weights ws*LPL*d), and the truncation cap min(a) + ws*T from a
//    redux.sync min;
//  * the Handshake recursion is processed level by level (breadth first); at
//    level l each subchain recomputes only the message direction whose
//    boundary changed (Fig.11's "dots" are reused), so one warp runs one pass
//    per subchain.  The messages a later level needs ("spine" messages at the
//    midpoints of the descendants that keep this boundary) and the final
//    leaf boundary messages live in the fwd/bwd scratch arrays;
//  * epilogue: every node is a leaf [p,p] with boundary messages L = fwd[p],
//    R = bwd[p]; its minorant is lambda = L + F + R (reading R8), so
//    H: f_ = lambda - g_ = L + D*2^F + R, V: g_ = lambda - f_ = L + R; the
//    node minima sum to the dual bound (exactness) and the last V pass writes
//    the lowest-index argmin as the label (R13, R14).
// All arithmetic is exact int32 (ranges in DESIGN.md), so the result is
// bit-identical to the CPU oracle regardless of evaluation order.
#include <climits>

#include "dmm_internal.cuh"

namespace dmm {

template <int LPL>
__device__ __forceinline__ void ld_i32(const int32_t* __restrict__ p, int (&v)[LPL]) {
    if constexpr (LPL == 1) {
        v[0] = p[0];
    } else if constexpr (LPL == 2) {
        int2 t = *reinterpret_cast<const int2*>(p);
        v[0] = t.x; v[1] = t.y;
    } else {
#pragma unroll
        for (int q = 0; q < LPL / 4; ++q) {
            int4 t = reinterpret_cast<const int4*>(p)[q];
            v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
        }
    }
}

template <int LPL>
__device__ __forceinline__ void st_i32(int32_t* p, const int (&v)[LPL]) {
    if constexpr (LPL == 1) {
        p[0] = v[0];
    } else if constexpr (LPL == 2) {
        *reinterpret_cast<int2*>(p) = make_int2(v[0], v[1]);
    } else {
#pragma unroll
        for (int q = 0; q < LPL / 4; ++q)
            reinterpret_cast<int4*>(p)[q] = make_int4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
}

template <int LPL>
__device__ __forceinline__ void ld_u8(const uint8_t* __restrict__ p, int (&v)[LPL]) {
    if constexpr (LPL == 1) {
        v[0] = p[0];
    } else if constexpr (LPL == 2) {
        unsigned t = *reinterpret_cast<const unsigned short*>(p);
        v[0] = t & 0xff; v[1] = t >> 8;
    } else {
#pragma unroll
        for (int q = 0; q < LPL / 4; ++q) {
            unsigned t = reinterpret_cast<const unsigned*>(p)[q];
#pragma unroll
            for (int b = 0; b < 4; ++b) v[4 * q + b] = (t >> (8 * b)) & 0xff;
        }
    }
}

// out(b) = min_a x(a) + ws*min(|a-b|, T), computed in place (exact).
template <int LPL>
__device__ __forceinline__ void msg(int (&x)[LPL], int ws, int wsT, int lane, int K) {
#pragma unroll
    for (int e = 0; e < LPL; ++e)
        if (lane * LPL + e >= K) x[e] = kBig;
    int lmin = x[0];
#pragma unroll
    for (int e = 1; e < LPL; ++e) lmin = min(lmin, x[e]);
    const int gmin = __reduce_min_sync(kFull, lmin);
    int fw[LPL], bw[LPL];
    fw[0] = x[0];
#pragma unroll
    for (int e = 1; e < LPL; ++e) fw[e] = __viaddmin_s32(fw[e - 1], ws, x[e]);
    bw[LPL - 1] = x[LPL - 1];
#pragma unroll
    for (int e = LPL - 2; e >= 0; --e) bw[e] = __viaddmin_s32(bw[e + 1], ws, x[e]);
    int cf = fw[LPL - 1], cb = bw[0];
    const int step = ws * LPL;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int tf = __shfl_up_sync(kFull, cf, d);
        const int tb = __shfl_down_sync(kFull, cb, d);
        if (lane >= d) cf = __viaddmin_s32(tf, step * d, cf);
        if (lane + d < 32) cb = __viaddmin_s32(tb, step * d, cb);
    }
    int inf = __shfl_up_sync(kFull, cf, 1);
    int inb = __shfl_down_sync(kFull, cb, 1);
    if (lane == 0) inf = kBig;
    if (lane == 31) inb = kBig;
    const int cap = gmin + wsT;
#pragma unroll
    for (int e = 0; e < LPL; ++e) {
        const int vf = __viaddmin_s32(inf, ws * (e + 1), fw[e]);
        const int vb = __viaddmin_s32(inb, ws * (LPL - e), bw[e]);
        x[e] = min(min(vf, vb), cap);
    }
}

template <int LPL, bool VERT>
struct Chain {
    FramePtrs P;
    int W, KP, K, c, lane;
    int fbits, ws, wsT;
    bool first;

    __device__ __forceinline__ size_t off(int p) const {
        const size_t q = VERT ? (size_t)p * W + c : (size_t)c * W + p;
        return q * KP + lane * LPL;
    }
    // F = D * 2^F + g_ (H pass) or f_ (V pass)
    __device__ __forceinline__ void loadF(int p, int (&F)[LPL]) const {
        const size_t o = off(p);
        if constexpr (VERT) {
            ld_i32<LPL>(P.fdual + o, F);
        } else {
            ld_u8<LPL>(P.D + o, F);
#pragma unroll
            for (int e = 0; e < LPL; ++e) F[e] <<= fbits;
            if (!first) {
                int g[LPL];
                ld_i32<LPL>(P.gdual + o, g);
#pragma unroll
                for (int e = 0; e < LPL; ++e) F[e] += g[e];
            }
        }
    }
    __device__ __forceinline__ void msg_(int (&x)[LPL]) const { msg<LPL>(x, ws, wsT, lane, K); }
};

// Forward messages from `lo` (phi = message into lo) up to `end` (exclusive
// source).  Stores the messages into the spine nodes lo + (len0 >> k) - 1,
// k >= 1 (midpoints of the left-lineage descendants of [lo, end], which keep
// the left boundary), and the final message into `end` (k = 0).
template <int LPL, bool VERT>
__device__ __forceinline__ void pass_fwd(const Chain<LPL, VERT>& ch, int lo, int end, int (&phi)[LPL]) {
    const int len0 = end - lo + 1;
    if (len0 < 2) return;
    int kk = (31 - __clz(len0)) - 1;              // largest k with len0 >> k >= 2
    int target = len0 >> kk;
    int F[LPL];
    ch.loadF(lo, F);
    for (int p = lo; p < end; ++p) {
        int Fn[LPL];
        if (p + 1 < end) ch.loadF(p + 1, Fn);
#pragma unroll
        for (int e = 0; e < LPL; ++e) phi[e] += F[e];
        ch.msg_(phi);
        if (p + 2 - lo == target) {
            st_i32<LPL>(ch.P.fwd + ch.off(p + 1), phi);
            --kk;
            target = kk >= 0 ? (len0 >> kk) : INT_MAX;
        }
#pragma unroll
        for (int e = 0; e < LPL; ++e) F[e] = Fn[e];
    }
}

// Backward messages from `hi` (phi = message into hi) down to `end`.  Spine:
// nodes hi - R_k + 1 with R_k = ((lenB - 1) >> k) + 1 = ceil(lenB / 2^k)
// (midpoint + 1 of the right-lineage descendants of [end, hi]).
template <int LPL, bool VERT>
__device__ __forceinline__ void pass_bwd(const Chain<LPL, VERT>& ch, int hi, int end, int (&phi)[LPL]) {
    const int lenB = hi - end + 1;
    if (lenB < 2) return;
    int kk = 31 - __clz(lenB - 1);                // largest k with R_k >= 2
    int target = ((lenB - 1) >> kk) + 1;
    int F[LPL];
    ch.loadF(hi, F);
    for (int p = hi; p > end; --p) {
        int Fn[LPL];
        if (p - 1 > end) ch.loadF(p - 1, Fn);
#pragma unroll
        for (int e = 0; e < LPL; ++e) phi[e] += F[e];
        ch.msg_(phi);
        if (hi - p + 2 == target) {
            st_i32<LPL>(ch.P.bwd + ch.off(p - 1), phi);
            --kk;
            target = kk >= 0 ? (((lenB - 1) >> kk) + 1) : INT_MAX;
        }
#pragma unroll
        for (int e = 0; e < LPL; ++e) F[e] = Fn[e];
    }
}

// Handshake over edge (i, j = i+1), Alg.5 with reading R9/R10:
// phiL = message into i from the left, phiR = message into j from the right.
template <int LPL, bool VERT>
__device__ __forceinline__ void handshake(const Chain<LPL, VERT>& ch, int i, int (&phiL)[LPL],
                                       int (&phiR)[LPL]) {
    const int j = i + 1;
    int Fi[LPL], Fj[LPL], pji[LPL], t[LPL];
    ch.loadF(i, Fi);
    ch.loadF(j, Fj);
#pragma unroll
    for (int e = 0; e < LPL; ++e) pji[e] = Fj[e] + phiR[e];
    ch.msg_(pji);                                           // phi_ji := Msg(f_j + phi_{j+1,j})
#pragma unroll
    for (int e = 0; e < LPL; ++e) {
        const int m = phiL[e] + Fi[e] + pji[e];             // m_i
        t[e] = (m - 2 * pji[e]) >> 1;                       // floor(m_i/2 - phi_ji)
    }
    ch.msg_(t);                                             // phi_ij
    st_i32<LPL>(ch.P.fwd + ch.off(j), t);                   // right piece's left boundary
#pragma unroll
    for (int e = 0; e < LPL; ++e) t[e] = -t[e];
    ch.msg_(t);                                             // bounce back: phi_ji := Msg(-phi_ij)
    st_i32<LPL>(ch.P.bwd + ch.off(i), t);                   // left piece's right boundary
}

template <int LPL, bool VERT, int NW>
__global__ void __launch_bounds__(NW * 32) hm_kernel(PassArgs a) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Chain<LPL, VERT> ch;
    ch.P = frame_ptrs(a.L, a.frame0 + blockIdx.y);
    ch.W = a.L.W; ch.KP = a.L.KP; ch.K = a.L.K; ch.c = blockIdx.x; ch.lane = lane;
    ch.fbits = a.fbits; ch.ws = a.ws; ch.wsT = a.wsT; ch.first = a.first != 0;
    const int n = VERT ? a.L.H : a.L.W;
    int zero[LPL];
#pragma unroll
    for (int e = 0; e < LPL; ++e) zero[e] = 0;

    // ---- level 0: the whole chain [0, n-1] with zero boundary messages
    if (warp == 0) st_i32<LPL>(ch.P.fwd + ch.off(0), zero);
    if (warp == (NW > 1 ? 1 : 0)) st_i32<LPL>(ch.P.bwd + ch.off(n - 1), zero);
    if (n >= 2) {
        const int i = n / 2 - 1, j = i + 1;
        int phi[LPL];
#pragma unroll
        for (int e = 0; e < LPL; ++e) phi[e] = 0;
        if (warp == 0) pass_fwd<LPL, VERT>(ch, 0, i, phi);
        if (warp == (NW > 1 ? 1 : 0)) {
#pragma unroll
            for (int e = 0; e < LPL; ++e) phi[e] = 0;
            pass_bwd<LPL, VERT>(ch, n - 1, j, phi);
        }
        __syncthreads();
        if (warp == 0) {
            int pl[LPL], pr[LPL];
            ld_i32<LPL>(ch.P.fwd + ch.off(i), pl);
            ld_i32<LPL>(ch.P.bwd + ch.off(j), pr);
            handshake<LPL, VERT>(ch, i, pl, pr);
        }
        __syncthreads();
    }
    // ---- levels 1..: one new-direction pass + one Handshake per subchain
    const int nlev = n >= 2 ? 32 - __clz(n - 1) : 0;      // ceil(log2 n)
    for (int lev = 1; lev < nlev; ++lev) {
        for (int s = warp; s < (1 << lev); s += NW) {
            int lo = 0, hi = n - 1, right = 0;
            bool exists = true;
            for (int b = lev - 1; b >= 0; --b) {
                const int len = hi - lo + 1;
                if (len < 2) { exists = false; break; }
                const int mid = lo + len / 2 - 1;
                if ((s >> b) & 1) { lo = mid + 1; right = 1; } else { hi = mid; right = 0; }
            }
            if (!exists || hi - lo + 1 < 2) continue;
            const int len = hi - lo + 1, i = lo + len / 2 - 1, j = i + 1;
            int pl[LPL], pr[LPL];
            if (!right) {     // left child: left boundary unchanged -> reuse fwd, redo bwd
                ld_i32<LPL>(ch.P.bwd + ch.off(hi), pr);
                pass_bwd<LPL, VERT>(ch, hi, j, pr);
                ld_i32<LPL>(ch.P.fwd + ch.off(i), pl);
            } else {          // right child: right boundary unchanged -> reuse bwd, redo fwd
                ld_i32<LPL>(ch.P.fwd + ch.off(lo), pl);
                pass_fwd<LPL, VERT>(ch, lo, i, pl);
                ld_i32<LPL>(ch.P.bwd + ch.off(j), pr);
            }
            handshake<LPL, VERT>(ch, i, pl, pr);
        }
        __syncthreads();
    }

    // ---- epilogue: leaves
    long long bsum = 0;
    int32_t* out = VERT ? ch.P.gdual : ch.P.fdual;
    for (int p = warp; p < n; p += NW) {
        const size_t o = ch.off(p);
        int Lm[LPL], Rm[LPL], lam[LPL], o_[LPL];
        ld_i32<LPL>(ch.P.fwd + o, Lm);
        ld_i32<LPL>(ch.P.bwd + o, Rm);
        if constexpr (VERT) {
            int F[LPL];
            ld_i32<LPL>(ch.P.fdual + o, F);
#pragma unroll
            for (int e = 0; e < LPL; ++e) { o_[e] = Lm[e] + Rm[e]; lam[e] = o_[e] + F[e]; }
        } else {
            int Dv[LPL], g[LPL];
            ld_u8<LPL>(ch.P.D + o, Dv);
            if (!ch.first) ld_i32<LPL>(ch.P.gdual + o, g);
#pragma unroll
            for (int e = 0; e < LPL; ++e) {
                o_[e] = Lm[e] + (Dv[e] << ch.fbits) + Rm[e];
                lam[e] = o_[e] + (ch.first ? 0 : g[e]);
            }
        }
        int lmin = INT_MAX;
#pragma unroll
        for (int e = 0; e < LPL; ++e) {
            if (lane * LPL + e >= ch.K) { o_[e] = 0; lam[e] = INT_MAX; }
            lmin = min(lmin, lam[e]);
        }
        st_i32<LPL>(out + o, o_);
        const int gmin = __reduce_min_sync(kFull, lmin);
        bsum += gmin;
        if (VERT && a.last) {
            int kmin = INT_MAX;
#pragma unroll
            for (int e = LPL - 1; e >= 0; --e)
                if (lam[e] == gmin) kmin = lane * LPL + e;
            kmin = __reduce_min_sync(kFull, kmin);
            if (lane == 0) {
                const size_t q = (size_t)p * ch.W + ch.c;
                ch.P.labels[q] = (uint8_t)kmin;
            }
        }
    }
    if (lane == 0)
        atomicAdd(reinterpret_cast<unsigned long long*>(&ch.P.bounds[a.bound_slot]),
                  (unsigned long long)bsum);
}

template <int LPL>
static void launch_lpl(const PassArgs& a, int vertical, int nframes, cudaStream_t s) {
    constexpr int NW = 4;
    if (vertical)
        hm_kernel<LPL, true, NW><<<dim3(a.L.W, nframes), NW * 32, 0, s>>>(a);
    else
        hm_kernel<LPL, false, NW><<<dim3(a.L.H, nframes), NW * 32, 0, s>>>(a);
}

void launch_hm_pass(const PassArgs& a, int vertical, int nframes, cudaStream_t s) {
    switch (a.L.KP / 32) {
        case 1: launch_lpl<1>(a, vertical, nframes, s); break;
        case 2: launch_lpl<2>(a, vertical, nframes, s); break;
        case 4: launch_lpl<4>(a, vertical, nframes, s); break;
        default: launch_lpl<8>(a, vertical, nframes, s); break;
    }
}

}  // namespace dmm
