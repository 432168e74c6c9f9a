// hm2_device.cuh -- packed two-chain primitives of the chain DP (hm2.cu).
//
// A warp carries two chains of the same orientation at once: every 32-bit
// register holds one label of chain A in its low 16 bits and the same label
// of chain B in its high 16 bits, and the sm_100a packed integer ops
// (VIADDMNMX.S16x2, VIMNMX3.S16x2, VIADD.16x2) advance both chains with one
// instruction.  Every K-vector is held relative to a per-chain int32 offset
// (warp-uniform), so the 16-bit parts stay small: messages are normalised to
// min = 0 after every Msg (Msg(a + c) = Msg(a) + c exactly), record values
// are the compact records' u16 spans.  dmm_create's range check
// (pair_range_ok in capi.cu) guarantees every operand and every candidate of
// the distance transform fits in signed 16 bits, so the packed path computes
// exactly the int32 values of the oracle (same integers, different
// bookkeeping).
#pragma once
#include "hm_device.cuh"

namespace dmm {
namespace p2 {

// +/- "infinity" of the packed path: > every real operand + addend, and
// -kBig16 - addend >= -32768 (range check).
constexpr int kBig16 = 16383;
constexpr unsigned kBigP = 0x3fff3fffu;
constexpr unsigned kNegBigP = 0xc001c001u;

__device__ __forceinline__ unsigned pk(int lo, int hi) { return __byte_perm((unsigned)lo, (unsigned)hi, 0x5410); }
// PTX prmt with the sign-replicate selector bit (__byte_perm masks it off)
__device__ __forceinline__ unsigned prmt_sgn(unsigned a, unsigned b, unsigned sel) {
    unsigned r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
__device__ __forceinline__ int lo16(unsigned x) { return (int)(short)(x & 0xffffu); }
__device__ __forceinline__ int hi16(unsigned x) { return ((int)x) >> 16; }

template <bool MAX>
__device__ __forceinline__ unsigned op2(unsigned a, unsigned b) { return MAX ? __vmaxs2(a, b) : __vmins2(a, b); }
template <bool MAX>
__device__ __forceinline__ unsigned addop2(unsigned a, unsigned w, unsigned c) {   // op(a + w, c) per half
    return MAX ? __viaddmax_s16x2(a, w, c) : __viaddmin_s16x2(a, w, c);
}
template <bool MAX>
__device__ __forceinline__ unsigned op3_2(unsigned a, unsigned b, unsigned c) {
    return MAX ? __vimax3_s16x2(a, b, c) : __vimin3_s16x2(a, b, c);
}

// Loop-invariant operands of the packed distance transform, built once per
// kernel (per lane): ws, wsT, and the min-plus addends of the one-hop window,
// with wsT + 1 at lanes 0 / 31 (no neighbour: the shuffle returned one of the
// lane's own values, >= min, so that candidate lands above the cap without a
// select).  Addends beyond the truncation are clamped to wsT + 1: such a
// candidate exceeds the cap g + wsT, clamped or not.
template <int LPL>
struct DtK {
    int ws, wsT, K, lane;
    int ksd;                          // Kogge-Stone path: last round distance needed (see dtrans2)
    unsigned wsP, capP;               // pk(ws), pk(wsT)
    unsigned aL[LPL], aR[LPL];        // per label e: left (e+1)*ws, right (LPL-e)*ws
    __device__ __forceinline__ void init(int ws_, int wsT_, int K_, int lane_, int T_) {
        ws = ws_; wsT = wsT_; K = K_; lane = lane_;
        // labels of the lane j lanes away are >= (j-1)*LPL + 1 labels apart;
        // candidates at distance >= T are beaten by the truncation cap, so only
        // lanes j <= (T-2)/LPL + 1 matter: the scan may stop at the first round
        // distance d with 2d >= that (the envelope then spans 2d lanes)
        const int jmax = T_ >= 2 ? (T_ - 2) / LPL + 1 : 1;
        ksd = 1;
        while (2 * ksd < jmax && ksd < 16) ksd <<= 1;
        const int cl = wsT + 1;
        const int w1 = min(ws, cl);
        wsP = pk(w1, w1);
        capP = pk(wsT, wsT);
#pragma unroll
        for (int e = 0; e < LPL; ++e) {
            const int al = lane == 0 ? cl : min(ws * (e + 1), cl);
            const int ar = lane == 31 ? cl : min(ws * (LPL - e), cl);
            aL[e] = pk(al, al);
            aR[e] = pk(ar, ar);
        }
    }
};

// Packed distance transform of two K-vectors (see dtrans in hm_device.cuh for
// the windowed / Kogge-Stone structure):
//   MAX = false: x(b) := min_a x(a) + ws*min(|a-b|, T)      (Msg)
//   MAX = true:  x(b) := max_a x(a) - ws*min(|a-b|, T)
// Returns G = pk(gA, gB), the per-chain min (MAX: max) of the input, which is
// also the min (max) of the output.
template <int LPL, bool PAD, int WIN, bool MAX = false>
__device__ __forceinline__ unsigned dtrans2(unsigned (&x)[LPL], const DtK<LPL>& k, int& gA, int& gB) {
    const unsigned big = MAX ? kNegBigP : kBigP;
    const int lane = k.lane;
    if constexpr (PAD) {
#pragma unroll
        for (int e = 0; e < LPL; ++e)
            if (lane * LPL + e >= k.K) x[e] = big;
    }
    unsigned lred = x[0];
#pragma unroll
    for (int e = 1; e < LPL; ++e) lred = op2<MAX>(lred, x[e]);
    gA = MAX ? __reduce_max_sync(kFull, lo16(lred)) : __reduce_min_sync(kFull, lo16(lred));
    gB = MAX ? __reduce_max_sync(kFull, hi16(lred)) : __reduce_min_sync(kFull, hi16(lred));
    const int clampv = k.wsT + 1;
    const unsigned G = pk(gA, gB);
    unsigned cap, wsP;
    if constexpr (MAX) {
        cap = __vsub2(G, k.capP);
        wsP = __vsub2(0u, k.wsP);
    } else {
        cap = __vadd2(G, k.capP);
        wsP = k.wsP;
    }
    unsigned fw[LPL], bw[LPL];
    fw[0] = x[0];
#pragma unroll
    for (int e = 1; e < LPL; ++e) fw[e] = addop2<MAX>(fw[e - 1], wsP, x[e]);
    bw[LPL - 1] = x[LPL - 1];
#pragma unroll
    for (int e = LPL - 2; e >= 0; --e) bw[e] = addop2<MAX>(bw[e + 1], wsP, x[e]);
    unsigned inf, inb;
    if constexpr (WIN != 0) {
        inf = __shfl_up_sync(kFull, fw[LPL - 1], 1);
        inb = __shfl_down_sync(kFull, bw[0], 1);
    } else {
        unsigned cf = fw[LPL - 1], cb = bw[0];
        const int sg = MAX ? -1 : 1;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int st = min(k.ws * LPL * d, clampv);
            const unsigned stP = pk(sg * st, sg * st);
            const unsigned tf = __shfl_up_sync(kFull, cf, d);
            const unsigned tb = __shfl_down_sync(kFull, cb, d);
            if (lane >= d) cf = addop2<MAX>(tf, stP, cf);
            if (lane + d < 32) cb = addop2<MAX>(tb, stP, cb);
            if (d >= k.ksd) break;        // farther lanes only hold candidates above the cap
        }
        inf = __shfl_up_sync(kFull, cf, 1);
        inb = __shfl_down_sync(kFull, cb, 1);
    }
#pragma unroll
    for (int e = 0; e < LPL; ++e) {
        const bool needL = WIN > 0 ? (e + 1 < WIN) : true;
        const bool needR = WIN > 0 ? (LPL - e < WIN) : true;
        const unsigned aL = MAX ? __vsub2(0u, k.aL[e]) : k.aL[e];
        const unsigned aR = MAX ? __vsub2(0u, k.aR[e]) : k.aR[e];
        const unsigned vf = needL ? addop2<MAX>(inf, aL, fw[e]) : fw[e];
        const unsigned vb = needR ? addop2<MAX>(inb, aR, bw[e]) : bw[e];
        x[e] = op3_2<MAX>(vf, vb, cap);
    }
    return G;
}

// ---- message pairs: packed normalised values + per-chain offsets
template <int LPL>
struct MP {
    unsigned m[LPL];
    int a, b;
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int e = 0; e < LPL; ++e) m[e] = 0u;
        a = 0; b = 0;
    }
};

// Msg on a pair: x (packed, offsets oa/ob) -> normalised Msg output.
template <int LPL, bool PAD, int WIN>
__device__ __forceinline__ void msg2(unsigned (&x)[LPL], int& oa, int& ob, const DtK<LPL>& k) {
    int gA, gB;
    const unsigned G = dtrans2<LPL, PAD, WIN, false>(x, k, gA, gB);
#pragma unroll
    for (int e = 0; e < LPL; ++e) x[e] = __vsub2(x[e], G);   // per half (values may be negative)
    oa += gA; ob += gB;
}

// spine storage: packed words [q][KP] (u32 view of the int32 scratch) + offsets [q][2]
template <int LPL>
__device__ __forceinline__ void st_mp(int32_t* arr, int32_t* off, size_t q, int lane, const MP<LPL>& v) {
    constexpr int KP = 32 * LPL;
    st_i32<LPL>(arr + q * KP + lane * LPL, reinterpret_cast<const int(&)[LPL]>(v.m));
    if (lane == 0) *reinterpret_cast<int2*>(off + 2 * q) = make_int2(v.a, v.b);
}
template <int LPL>
__device__ __forceinline__ void ld_mp(const int32_t* arr, const int32_t* off, size_t q, int lane, MP<LPL>& v) {
    constexpr int KP = 32 * LPL;
    ld_i32<LPL>(arr + q * KP + lane * LPL, reinterpret_cast<int(&)[LPL]>(v.m));
    const int2 o = *reinterpret_cast<const int2*>(off + 2 * q);
    v.a = o.x; v.b = o.y;
}

// record pair at shared addresses ra / rb -> packed u16 values v, bases
template <int LPL>
__device__ __forceinline__ void ld_rec_pair_s(unsigned ra, unsigned rb, int lane, unsigned (&v)[LPL], int& ba,
                                              int& bb) {
    constexpr int KP = 32 * LPL;
    ba = (int)lds32(ra + 2 * KP);
    bb = (int)lds32(rb + 2 * KP);
    const unsigned o = 2 * LPL * lane;
    if constexpr (LPL == 1) {
        v[0] = __byte_perm(lds16(ra + o), lds16(rb + o), 0x5410);
    } else if constexpr (LPL == 2) {
        const unsigned a = lds32(ra + o), b = lds32(rb + o);
        v[0] = __byte_perm(a, b, 0x5410); v[1] = __byte_perm(a, b, 0x7632);
    } else if constexpr (LPL == 4) {
        const uint2 a = lds64(ra + o), b = lds64(rb + o);
        v[0] = __byte_perm(a.x, b.x, 0x5410); v[1] = __byte_perm(a.x, b.x, 0x7632);
        v[2] = __byte_perm(a.y, b.y, 0x5410); v[3] = __byte_perm(a.y, b.y, 0x7632);
    } else {
        const uint4 a = lds128(ra + o), b = lds128(rb + o);
        v[0] = __byte_perm(a.x, b.x, 0x5410); v[1] = __byte_perm(a.x, b.x, 0x7632);
        v[2] = __byte_perm(a.y, b.y, 0x5410); v[3] = __byte_perm(a.y, b.y, 0x7632);
        v[4] = __byte_perm(a.z, b.z, 0x5410); v[5] = __byte_perm(a.z, b.z, 0x7632);
        v[6] = __byte_perm(a.w, b.w, 0x5410); v[7] = __byte_perm(a.w, b.w, 0x7632);
    }
}

// D-row pair (u8 labels) at shared addresses da / db -> packed D << fbits
template <int LPL>
__device__ __forceinline__ void ld_u8_pair_s(unsigned da, unsigned db, int lane, int fbits, unsigned (&v)[LPL]) {
    const unsigned o = LPL * lane;
    if constexpr (LPL == 1) {
        v[0] = (lds8(da + o) | (lds8(db + o) << 16)) << fbits;
    } else if constexpr (LPL == 2) {
        const unsigned a = lds16(da + o), b = lds16(db + o);     // bytes 2, 3 are zero
        v[0] = __byte_perm(a, b, 0x3420) << fbits;
        v[1] = __byte_perm(a, b, 0x3521) << fbits;
    } else if constexpr (LPL == 4) {
        // bytes [a_e, sign(a_e), b_e, sign(b_e)]: D < 128 (pair_range_ok) makes
        // the sign-replicated bytes zero; the scale runs on the FMA pipe
        const unsigned a = lds32(da + o), b = lds32(db + o);
        const unsigned sc = 1u << fbits;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const unsigned sel = (unsigned)(e | ((e | 8) << 4) | ((4 + e) << 8) | (((4 + e) | 8) << 12));
            v[e] = prmt_sgn(a, b, sel) * sc;
        }
    } else {
        const uint2 a = lds64(da + o), b = lds64(db + o);
        const unsigned sc = 1u << fbits;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const unsigned sel = (unsigned)(e | ((e | 8) << 4) | ((4 + e) << 8) | (((4 + e) | 8) << 12));
            v[e] = prmt_sgn(a.x, b.x, sel) * sc;
            v[4 + e] = prmt_sgn(a.y, b.y, sel) * sc;
        }
    }
}

// Store the pair o (packed, 0 <= o <= span bound per half, offsets oa / ob)
// as two compact records with base = the offset and v = o: a valid record
// (base <= min, span < 2^16) without a warp reduction.  B only if wb.
template <int LPL, bool PAD>
__device__ __forceinline__ void st_rec_pair(uint8_t* ra, uint8_t* rb, bool wb, int lane, const unsigned (&o)[LPL],
                                            int oa, int ob, int K) {
    constexpr int KP = 32 * LPL;
    unsigned v[LPL];
#pragma unroll
    for (int e = 0; e < LPL; ++e) v[e] = (!PAD || lane * LPL + e < K) ? o[e] : 0u;
    uint8_t* pa = ra + 2 * LPL * lane;
    uint8_t* pb = rb + 2 * LPL * lane;
    if constexpr (LPL == 1) {
        *reinterpret_cast<uint16_t*>(pa) = (uint16_t)(v[0] & 0xffffu);
        if (wb) *reinterpret_cast<uint16_t*>(pb) = (uint16_t)(v[0] >> 16);
    } else if constexpr (LPL == 2) {
        *reinterpret_cast<unsigned*>(pa) = __byte_perm(v[0], v[1], 0x5410);
        if (wb) *reinterpret_cast<unsigned*>(pb) = __byte_perm(v[0], v[1], 0x7632);
    } else if constexpr (LPL == 4) {
        *reinterpret_cast<uint2*>(pa) = make_uint2(__byte_perm(v[0], v[1], 0x5410), __byte_perm(v[2], v[3], 0x5410));
        if (wb)
            *reinterpret_cast<uint2*>(pb) =
                make_uint2(__byte_perm(v[0], v[1], 0x7632), __byte_perm(v[2], v[3], 0x7632));
    } else {
        *reinterpret_cast<uint4*>(pa) =
            make_uint4(__byte_perm(v[0], v[1], 0x5410), __byte_perm(v[2], v[3], 0x5410),
                       __byte_perm(v[4], v[5], 0x5410), __byte_perm(v[6], v[7], 0x5410));
        if (wb)
            *reinterpret_cast<uint4*>(pb) =
                make_uint4(__byte_perm(v[0], v[1], 0x7632), __byte_perm(v[2], v[3], 0x7632),
                           __byte_perm(v[4], v[5], 0x7632), __byte_perm(v[6], v[7], 0x7632));
    }
    if (lane == 0) {
        *reinterpret_cast<int32_t*>(ra + 2 * KP) = oa;
        if (wb) *reinterpret_cast<int32_t*>(rb + 2 * KP) = ob;
    }
}

// As st_rec_pair, into shared-memory records at ra / rb (both always
// written; the caller bulk-stores B only if the pair has a B chain).
template <int LPL, bool PAD>
__device__ __forceinline__ void st_rec_pair_s(unsigned ra, unsigned rb, int lane, const unsigned (&o)[LPL], int oa,
                                              int ob, int K) {
    constexpr int KP = 32 * LPL;
    unsigned v[LPL];
#pragma unroll
    for (int e = 0; e < LPL; ++e) v[e] = (!PAD || lane * LPL + e < K) ? o[e] : 0u;
    const unsigned pa = ra + 2 * LPL * lane;
    const unsigned pb = rb + 2 * LPL * lane;
    if constexpr (LPL == 1) {
        sts16(pa, v[0] & 0xffffu);
        sts16(pb, v[0] >> 16);
    } else if constexpr (LPL == 2) {
        sts32(pa, __byte_perm(v[0], v[1], 0x5410));
        sts32(pb, __byte_perm(v[0], v[1], 0x7632));
    } else if constexpr (LPL == 4) {
        sts64(pa, make_uint2(__byte_perm(v[0], v[1], 0x5410), __byte_perm(v[2], v[3], 0x5410)));
        sts64(pb, make_uint2(__byte_perm(v[0], v[1], 0x7632), __byte_perm(v[2], v[3], 0x7632)));
    } else {
        sts128(pa, make_uint4(__byte_perm(v[0], v[1], 0x5410), __byte_perm(v[2], v[3], 0x5410),
                              __byte_perm(v[4], v[5], 0x5410), __byte_perm(v[6], v[7], 0x5410)));
        sts128(pb, make_uint4(__byte_perm(v[0], v[1], 0x7632), __byte_perm(v[2], v[3], 0x7632),
                              __byte_perm(v[4], v[5], 0x7632), __byte_perm(v[6], v[7], 0x7632)));
    }
    if (lane == 0) {
        sts32(ra + 2 * KP, (unsigned)oa);
        sts32(rb + 2 * KP, (unsigned)ob);
    }
}

// floor(z / 2) per signed 16-bit half
__device__ __forceinline__ unsigned sra1_2(unsigned z) {
    const unsigned s = (unsigned)(((int)z) >> 1);
    return (s & ~0x8000u) | (z & 0x8000u);
}

// Handshake (Alg.5, readings R9/R10) on a pair.  In: pl = message
// into i from the left, pr = message into j from the right, (vi, bi*) and
// (vj, bj*) = the node costs.  Out: pl = phi_ij, pr = phi_ji'.
//
// OPT: also return the two chains' optima min_k m_i(k) (optA, optB): with
// pl / pr the exact messages from the chain ends (the root Handshake), m_i is
// the min-marginal at i, whose minimum is the chain optimum F* -- which
// equals the sum of the node minima of the hierarchical minorant (exactness,
// Lemma 1; pinned by tests/test_oracle_chain.py), i.e. the chain's
// share of the dual bound (Eq.7).
template <int LPL, bool PAD, int WIN, bool OPT = false>
__device__ __forceinline__ void handshake2(const unsigned (&vi)[LPL], int bia, int bib, const unsigned (&vj)[LPL],
                                           int bja, int bjb, MP<LPL>& pl, MP<LPL>& pr, const DtK<LPL>& k,
                                           int* opt = nullptr) {
    // phi_ji := Msg(f_j + phi_{j+1,j})
    unsigned pji[LPL];
#pragma unroll
    for (int e = 0; e < LPL; ++e) pji[e] = pr.m[e] + vj[e];
    const int ja = pr.a + bja, jb = pr.b + bjb;       // phi_ji left unnormalised
    {
        int g0, g1;
        dtrans2<LPL, PAD, WIN, false>(pji, k, g0, g1);
    }
    if constexpr (OPT) {
        unsigned l = kBigP;
#pragma unroll
        for (int e = 0; e < LPL; ++e)
            if (!PAD || k.lane * LPL + e < k.K) l = __vmins2(l, pl.m[e] + vi[e] + pji[e]);   // halves >= 0: no carry
        opt[0] = __reduce_min_sync(kFull, lo16(l)) + pl.a + bia + ja;
        opt[1] = __reduce_min_sync(kFull, hi16(l)) + pl.b + bib + jb;
    }
    // t = floor((m_i - 2 phi_ji) / 2), m_i = phi_L + f_i + phi_ji; true offset C = pl.o + bi - pji.o
    const int ca = pl.a + bia - ja, cb = pl.b + bib - jb;
    const unsigned c0 = pk(ca & 1, cb & 1);
    unsigned t[LPL];
#pragma unroll
    for (int e = 0; e < LPL; ++e) t[e] = sra1_2(__vsub2(pl.m[e] + vi[e] + c0, pji[e]));
    int ta = ca >> 1, tb = cb >> 1;
    msg2<LPL, PAD, WIN>(t, ta, tb, k);                           // phi_ij
    // phi_ji' = Msg(-phi_ij) = -phi_ij: a Msg output is V-Lipschitz
    // (phi(a) - phi(b) <= V(a,b), V = ws*min(|a-b|,T) is a metric), so
    // max_a phi(a) - V(a,b) = phi(b) and Msg(-phi) = -phi exactly (DESIGN.md
    // "Bounce identity"; pinned in tests/test_oracle_chain.py).  The
    // normalised t lies in [0, wsT]; -t is stored as wsT - t >= 0 with the
    // offset -t_off - wsT.
#pragma unroll
    for (int e = 0; e < LPL; ++e) { pr.m[e] = __vsub2(k.capP, t[e]); pl.m[e] = t[e]; }
    pr.a = -ta - k.wsT; pr.b = -tb - k.wsT;
    pl.a = ta; pl.b = tb;
}

}  // namespace p2
}  // namespace dmm
