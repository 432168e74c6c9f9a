// hm_device.cuh -- device primitives of the chain DP shared by the Dual MM
// half-step kernels (hm.cu) and the primitive entry points (primitives.cu):
// register-vector loads / stores, compact K-vector records, TMA bulk copies
// with mbarriers, and Msg (Eq. msg-pass; Msg of Alg.5).
#pragma once
#include <climits>

#include "dmm_internal.cuh"

namespace dmm {

// ------------------------------------------------------------ small helpers
template <int LPL>
__device__ __forceinline__ void ld_i32(const int32_t* p, int (&v)[LPL]) {
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
__device__ __forceinline__ void ld_u8(const uint8_t* p, int (&v)[LPL]) {
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
            for (int b = 0; b < 4; ++b) v[4 * q + b] = __byte_perm(t, 0, 0x4440 + b);
        }
    }
}

template <int LPL>
__device__ __forceinline__ void st_u8(uint8_t* p, const int (&v)[LPL]) {
    if constexpr (LPL == 1) {
        p[0] = (uint8_t)v[0];
    } else if constexpr (LPL == 2) {
        *reinterpret_cast<unsigned short*>(p) = (unsigned short)((v[0] & 0xff) | (v[1] << 8));
    } else {
#pragma unroll
        for (int q = 0; q < LPL / 4; ++q)
            reinterpret_cast<unsigned*>(p)[q] =
                __byte_perm(__byte_perm(v[4 * q], v[4 * q + 1], 0x0040), __byte_perm(v[4 * q + 2], v[4 * q + 3], 0x0040),
                            0x5410);
    }
}

// ---- explicit shared-memory loads on 32-bit shared addresses (keeps the
// generic->shared window conversion out of the inner loops)
__device__ __forceinline__ unsigned lds32(unsigned a) {
    unsigned v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint2 lds64(unsigned a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint4 lds128(unsigned a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a)
                 : "memory");
    return v;
}
__device__ __forceinline__ unsigned lds16(unsigned a) {
    unsigned v;   // ld.u16 into a 32-bit register zero-extends
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned lds8(unsigned a) {
    unsigned v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}

// record at shared address `rec`: F[e] = base + v[lane*LPL + e]
template <int LPL>
__device__ __forceinline__ void ld_rec_s(unsigned rec, int lane, int (&F)[LPL]) {
    constexpr int KP = 32 * LPL;
    const int base = (int)lds32(rec + 2 * KP);
    const unsigned p = rec + 2 * LPL * lane;
    if constexpr (LPL == 1) {
        F[0] = base + (int)lds16(p);
    } else {
        unsigned w[LPL / 2];
        if constexpr (LPL == 2) {
            w[0] = lds32(p);
        } else if constexpr (LPL == 4) {
            uint2 t = lds64(p);
            w[0] = t.x; w[1] = t.y;
        } else {
            uint4 t = lds128(p);
            w[0] = t.x; w[1] = t.y; w[2] = t.z; w[3] = t.w;
        }
#pragma unroll
        for (int q = 0; q < LPL / 2; ++q) {
            F[2 * q] = base + (int)(w[q] & 0xffffu);
            F[2 * q + 1] = base + (int)(w[q] >> 16);
        }
    }
}

// LPL bytes at shared address p (this lane's D labels)
template <int LPL>
__device__ __forceinline__ void ld_u8_s(unsigned p, int (&v)[LPL]) {
    if constexpr (LPL == 1) {
        v[0] = (int)lds8(p);
    } else if constexpr (LPL == 2) {
        const unsigned t = lds16(p);
        v[0] = t & 0xff; v[1] = t >> 8;
    } else if constexpr (LPL == 4) {
        const unsigned t = lds32(p);
#pragma unroll
        for (int b = 0; b < 4; ++b) v[b] = __byte_perm(t, 0, 0x4440 + b);
    } else {
        const uint2 t = lds64(p);
#pragma unroll
        for (int b = 0; b < 4; ++b) { v[b] = __byte_perm(t.x, 0, 0x4440 + b); v[4 + b] = __byte_perm(t.y, 0, 0x4440 + b); }
    }
}

// ---- compact records: u16 v[KP] | int32 base | pad  (value = base + v)
template <int LPL>
__device__ __forceinline__ void ld_rec(const uint8_t* rec, int lane, int (&F)[LPL]) {
    constexpr int KP = 32 * LPL;
    const int base = *reinterpret_cast<const int32_t*>(rec + 2 * KP);
    const uint8_t* p = rec + 2 * LPL * lane;
    if constexpr (LPL == 1) {
        F[0] = base + *reinterpret_cast<const uint16_t*>(p);
    } else {
        unsigned w[LPL / 2];
        if constexpr (LPL == 2) {
            w[0] = *reinterpret_cast<const unsigned*>(p);
        } else if constexpr (LPL == 4) {
            uint2 t = *reinterpret_cast<const uint2*>(p);
            w[0] = t.x; w[1] = t.y;
        } else {
            uint4 t = *reinterpret_cast<const uint4*>(p);
            w[0] = t.x; w[1] = t.y; w[2] = t.z; w[3] = t.w;
        }
#pragma unroll
        for (int q = 0; q < LPL / 2; ++q) {
            F[2 * q] = base + (int)(w[q] & 0xffffu);
            F[2 * q + 1] = base + (int)(w[q] >> 16);
        }
    }
}

// Store v (labels >= K ignored) as a record; base = min over labels < K.
template <int LPL, bool PAD>
__device__ __forceinline__ void st_rec(uint8_t* rec, int lane, const int (&v)[LPL], int K) {
    constexpr int KP = 32 * LPL;
    int lmin = INT_MAX;
#pragma unroll
    for (int e = 0; e < LPL; ++e)
        if (!PAD || lane * LPL + e < K) lmin = min(lmin, v[e]);
    const int base = __reduce_min_sync(kFull, lmin);
    unsigned u[LPL];
#pragma unroll
    for (int e = 0; e < LPL; ++e) u[e] = (!PAD || lane * LPL + e < K) ? (unsigned)(v[e] - base) : 0u;
    uint8_t* p = rec + 2 * LPL * lane;
    if constexpr (LPL == 1) {
        *reinterpret_cast<uint16_t*>(p) = (uint16_t)u[0];
    } else if constexpr (LPL == 2) {
        *reinterpret_cast<unsigned*>(p) = u[0] | (u[1] << 16);
    } else if constexpr (LPL == 4) {
        *reinterpret_cast<uint2*>(p) = make_uint2(u[0] | (u[1] << 16), u[2] | (u[3] << 16));
    } else {
        *reinterpret_cast<uint4*>(p) =
            make_uint4(u[0] | (u[1] << 16), u[2] | (u[3] << 16), u[4] | (u[5] << 16), u[6] | (u[7] << 16));
    }
    if (lane == 0) *reinterpret_cast<int32_t*>(rec + 2 * KP) = base;
}

// ---- TMA bulk copies (cp.async.bulk) completing on an mbarrier
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_s(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// 2-D tensor TMA: box at (x, y) of the tensor map at generic address tmap
__device__ __forceinline__ void tma_load_2d(unsigned dst, const void* tmap, int x, int y, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(tmap), "r"(x), "r"(y), "r"(bar)
        : "memory");
}

// ---- TMA bulk stores shared -> global (cp.async.bulk ... bulk_group)
__device__ __forceinline__ void tma_store_s(void* dst, unsigned src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// this thread's committed bulk stores have finished reading shared memory
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// ... and completed (writes performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void sts32(unsigned a, unsigned v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts16(unsigned a, unsigned v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void sts64(unsigned a, uint2 v) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void sts128(unsigned a, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// ------------------------------------------------------------------- Msg
// Generic exact distance transform on a warp-held K-vector:
//   MAX = false: x(b) := min_a x(a) + ws*min(|a-b|, T)      (Msg, min-plus)
//   MAX = true:  x(b) := max_a x(a) - ws*min(|a-b|, T)      (= -Msg(-x))
// The max-plus form computes the bounce-back Msg(-phi_ij) of Alg.5 without
// negating first: ptxas 12.9 (sm_100a) folds the negations of a neg -> min
// tree into VIMNMX3 and drops one of them (SASS VIMNMX3 R8, R15, R27, R8 with
// R27 = +out1), which gave wrong phi_ji' for LPL >= 4.
//  WIN: T <= LPL + 1, so every label within distance T-1 lies in this lane or
//  a neighbouring one; candidates from lanes further away are beaten by the
//  truncation term.  Lanes 0 / 31 have no left / right neighbour: the shuffle
//  returns their own value, which must be masked (own fw[LPL-1] + ws*(e+1)
//  would understate the distance to in-lane labels a > e when LPL >= 3).
template <bool MAX>
__device__ __forceinline__ int dt_op(int a, int b) { return MAX ? max(a, b) : min(a, b); }
template <bool MAX>
__device__ __forceinline__ int dt_addop(int a, int w, int c) {      // op(a + w, c), w signed
    return MAX ? __viaddmax_s32(a, w, c) : __viaddmin_s32(a, w, c);
}
template <bool MAX>
__device__ __forceinline__ int dt_op3(int a, int b, int c) {
    return MAX ? __vimax3_s32(a, b, c) : __vimin3_s32(a, b, c);
}

// WIN: 0 = full Kogge-Stone scan across lanes (any T); -1 = one-hop window,
// runtime T <= LPL+1; > 0 = one-hop window with compile-time T == WIN, so the
// candidates that are provably >= the truncation term (left-lane candidates of
// labels e with e+1 >= T, right-lane ones with LPL-e >= T) are never formed.
template <int LPL, bool PAD, int WIN, bool MAX = false>
__device__ __forceinline__ void dtrans(int (&x)[LPL], int ws_, int wsT_, int lane, int K) {
    const int big = MAX ? -kBig : kBig;
    const int ws = MAX ? -ws_ : ws_;
    const int wsT = MAX ? -wsT_ : wsT_;
    if constexpr (PAD) {
#pragma unroll
        for (int e = 0; e < LPL; ++e)
            if (lane * LPL + e >= K) x[e] = big;
    }
    int lred = x[0];
#pragma unroll
    for (int e = 1; e < LPL; ++e) lred = dt_op<MAX>(lred, x[e]);
    const int cap = (MAX ? __reduce_max_sync(kFull, lred) : __reduce_min_sync(kFull, lred)) + wsT;
    int fw[LPL], bw[LPL];
    fw[0] = x[0];
#pragma unroll
    for (int e = 1; e < LPL; ++e) fw[e] = dt_addop<MAX>(fw[e - 1], ws, x[e]);
    bw[LPL - 1] = x[LPL - 1];
#pragma unroll
    for (int e = LPL - 2; e >= 0; --e) bw[e] = dt_addop<MAX>(bw[e + 1], ws, x[e]);
    int inf, inb;
    if constexpr (WIN != 0) {
        inf = __shfl_up_sync(kFull, fw[LPL - 1], 1);
        inb = __shfl_down_sync(kFull, bw[0], 1);
    } else {
        int cf = fw[LPL - 1], cb = bw[0];
        const int step = ws * LPL;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int tf = __shfl_up_sync(kFull, cf, d);
            const int tb = __shfl_down_sync(kFull, cb, d);
            if (lane >= d) cf = dt_addop<MAX>(tf, step * d, cf);
            if (lane + d < 32) cb = dt_addop<MAX>(tb, step * d, cb);
        }
        inf = __shfl_up_sync(kFull, cf, 1);
        inb = __shfl_down_sync(kFull, cb, 1);
    }
    if (lane == 0) inf = big;
    if (lane == 31) inb = big;
#pragma unroll
    for (int e = 0; e < LPL; ++e) {
        const bool needL = WIN > 0 ? (e + 1 < WIN) : true;
        const bool needR = WIN > 0 ? (LPL - e < WIN) : true;
        const int vf = needL ? dt_addop<MAX>(inf, ws * (e + 1), fw[e]) : fw[e];
        const int vb = needR ? dt_addop<MAX>(inb, ws * (LPL - e), bw[e]) : bw[e];
        x[e] = dt_op3<MAX>(vf, vb, cap);
    }
}

// out(b) = min_a x(a) + ws*min(|a-b|, T), in place, exact (Msg).
template <int LPL, bool PAD, int WIN>
__device__ __forceinline__ void msg(int (&x)[LPL], int ws, int wsT, int lane, int K) {
    dtrans<LPL, PAD, WIN, false>(x, ws, wsT, lane, K);
}

// Handshake (Alg.5, readings R9/R10) on register vectors.
// In: pl = message into i from the left, pr = message into j from the right,
// Fi, Fj = node costs.  Out: pl = phi_ij (into j), pr = phi_ji' (into i).
template <int LPL, bool PAD, int WIN>
__device__ __forceinline__ void handshake_regs(const int (&Fi)[LPL], const int (&Fj)[LPL], int (&pl)[LPL],
                                               int (&pr)[LPL], int ws, int wsT, int lane, int K) {
    int pji[LPL], t_[LPL];
#pragma unroll
    for (int e = 0; e < LPL; ++e) pji[e] = Fj[e] + pr[e];
    msg<LPL, PAD, WIN>(pji, ws, wsT, lane, K);               // phi_ji := Msg(f_j + phi_{j+1,j})
#pragma unroll
    for (int e = 0; e < LPL; ++e) t_[e] = (pl[e] + Fi[e] - pji[e]) >> 1;   // floor(m_i/2 - phi_ji)
    msg<LPL, PAD, WIN>(t_, ws, wsT, lane, K);                // phi_ij
    // bounce back: Msg(-phi_ij) = -phi_ij exactly, because a Msg output is
    // V-Lipschitz for the metric V = ws*min(|a-b|,T)
#pragma unroll
    for (int e = 0; e < LPL; ++e) { pl[e] = t_[e]; pr[e] = -t_[e]; }
}

}  // namespace dmm
