// hm.cu -- Dual MM half-steps (Algorithm 2) for sm_100a: every row
// (H pass) or column (V pass) chain builds its hierarchical minorant
// with Handshakes (Alg.5).
//
// Mapping:
//  * one CTA per chain, NW warps; a warp owns one K-vector at a time with the
//    label dimension in registers, LPL = KP/32 consecutive labels per lane;
//    Msg / Handshake are the register-level primitives of hm_device.cuh.
//  * node data F (the pass's unaries: D*2^F + g_ for H, f_ for V) are compact
//    u16-span records (dmm_internal.cuh); they stream into a per-warp ring of
//    kNSlot chunks x kCH nodes filled by TMA bulk copies (cp.async.bulk, one
//    lane per node, one mbarrier per chunk).  The producer walks the warp's
//    whole consumption order (RunSeq) and runs ahead across level barriers:
//    node data never depend on the messages.
//  * "global levels" (subchains longer than kCMax): breadth first, one warp
//    per subchain; only the message direction whose boundary changed is
//    recomputed (Fig.11's dots are reused: "spine" messages a later level needs
//    are kept in the fwd/bwd scratch arrays, L2-resident); each task's two
//    message loads are issued one task ahead.
//  * "leaf blocks" (the 2^l* subchains of length <= kCMax): one warp copies
//    the block's F (decoded to int32) and D rows into shared memory and
//    finishes the sub-hierarchy on chip, depth first, the forward and backward
//    passes of each piece interleaved (two independent Msg chains -> ILP).
//    A leaf [p,p] with boundary messages L, R has lambda = L + F + R (reading
//    R8); the pass writes L + R + D*2^F, which is f_ = lambda - g_ for H and
//    D*2^F + g_ (the next H pass's unaries) for V, as a compact record.  Node
//    minima of lambda sum to the dual bound (exactness); the last V pass
//    writes the lowest-index argmin as the label (R13, R14).
// All arithmetic is exact int32 (ranges in DESIGN.md): bit-identical to the
// CPU oracle whatever the evaluation order.
#include "hm_device.cuh"

namespace dmm {

constexpr int kCMax = 12;    // longest leaf block (nodes); < 16 (4-bit piece starts)
constexpr int kDepth = 4;    // pending right pieces in a leaf block (ceil(log2 kCMax))
constexpr int kCH = 4;       // nodes per ring chunk
constexpr int kNSlot = 4;    // ring chunks per warp (prefetch depth kNSlot * kCH nodes)

__host__ __device__ constexpr int align_up(int x, int a) { return (x + a - 1) / a * a; }

struct HmShared {   // per-warp shared memory carve-up (bytes)
    int rec, slot, ring, mbar, leafF, leafD, stack, total;
    __host__ __device__ HmShared(int KP) {
        rec = rec_bytes(KP);
        slot = kCH * (rec + KP);               // kCH F records, then kCH D rows
        ring = 0;
        mbar = align_up(ring + kNSlot * slot, 8);
        leafF = align_up(mbar + kNSlot * 8, 16);
        leafD = leafF + kCMax * KP * 4;
        stack = leafD + kCMax * KP;
        total = align_up(stack + kDepth * 2 * KP * 4, 128);
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

// The warp's node consumption order as runs of consecutive nodes: per global
// task its pass (forward lo..i-1 or backward hi..j+1) then the Handshake pair
// j, i; per leaf block lo..hi (these runs also carry the D rows).
struct RunSeq {
    int n, lstar, warp, nw, lev, s, phase;
    bool done;
    __device__ __forceinline__ void init(int n_, int lstar_, int warp_, int nw_) {
        n = n_; lstar = lstar_; warp = warp_; nw = nw_; lev = 0; s = warp_; phase = 0; done = false;
    }
    // next non-empty run; false when exhausted
    __device__ __forceinline__ bool next(int& start, int& dir, int& count, bool& leaf) {
        while (!done) {
            if (lev > lstar) { done = true; break; }
            leaf = false;
            if (lev == 0 && lstar > 0) {
                if (s > 1) { ++lev; s = warp; phase = 0; continue; }
                const int i = n / 2 - 1, j = i + 1;
                if (s == 0) {
                    if (phase == 0) { phase = 1; start = 0; dir = 1; count = i; if (count > 0) return true; continue; }
                    phase = 0; s += nw; start = j; dir = -1; count = 2; return true;
                }
                phase = 0; s += nw; start = n - 1; dir = -1; count = n - 1 - j;
                if (count > 0) return true;
                continue;
            }
            if (s >= (1 << lev)) { ++lev; s = warp; phase = 0; continue; }
            int lo, hi;
            task_bounds(n, lev, s, lo, hi);
            if (lev == lstar) { s += nw; start = lo; dir = 1; count = hi - lo + 1; leaf = true; return true; }
            const int i = lo + (hi - lo + 1) / 2 - 1, j = i + 1;
            if (phase == 0) {
                phase = 1;
                if (!(s & 1)) { start = hi; dir = -1; count = hi - j; }
                else { start = lo; dir = 1; count = i - lo; }
                if (count > 0) return true;
                continue;
            }
            phase = 0; s += nw; start = j; dir = -1; count = 2; return true;
        }
        return false;
    }
};

template <int LPL, bool VERT, bool PAD, bool WIN, bool FIRST>
struct Hm {
    static constexpr int KP = 32 * LPL;
    static constexpr int REC = rec_bytes(KP);
    static constexpr int SREC = FIRST ? KP : REC;   // bytes of a source record (FIRST: the D row)
    FramePtrs P;
    const uint8_t* src;     // source records: FIRST ? D : (VERT ? fv : fh)
    uint8_t* dst;           // output records: VERT ? fh : fv
    int W, K, c, lane, n;
    int fbits, ws, wsT;
    bool last;
    long long bsum;
    // ring
    uint8_t* ring;
    uint64_t* mbar;
    unsigned clen;                  // chunk length of slot s in bits 8s..8s+7 (per-lane copy:
                                    // every lane runs the producer logic; no shared state)
    int slotB;
    RunSeq seq;
    int r_start, r_dir, r_left;     // producer: rest of the current run
    bool r_leaf;
    int cslot, cidx, ccount;        // consumer position
    unsigned cphase;                // consumer parity bit per slot
    bool cwait;

    __device__ __forceinline__ int q_of(int p) const { return VERT ? p * W + c : c * W + p; }
    __device__ __forceinline__ size_t moff(int p) const { return (size_t)q_of(p) * KP + lane * LPL; }
    __device__ __forceinline__ void msg_(int (&x)[LPL]) const { msg<LPL, PAD, WIN>(x, ws, wsT, lane, K); }

    // ---- producer: fill `slot` with the next chunk (<= kCH nodes of one run)
    __device__ __forceinline__ void fill(int slot) {
        while (r_left == 0) {
            if (!seq.next(r_start, r_dir, r_left, r_leaf)) return;
        }
        const int cnt = r_left < kCH ? r_left : kCH;
        uint8_t* sbase = ring + slot * slotB;
        clen = (clen & ~(0xffu << (8 * slot))) | ((unsigned)cnt << (8 * slot));
        if (lane == 0) mbar_expect_tx(&mbar[slot], (unsigned)(cnt * (SREC + (r_leaf && !FIRST ? KP : 0))));
        __syncwarp();
        // every lane read this slot through the generic proxy: order those reads
        // before the async-proxy (TMA) overwrite
        fence_proxy_async();
        __syncwarp();
        if (lane < cnt) {
            const int node = r_start + r_dir * lane;
            const size_t q = (size_t)q_of(node);
            tma_load(sbase + lane * REC, src + q * SREC, SREC, &mbar[slot]);
            if (!FIRST && r_leaf) tma_load(sbase + kCH * REC + lane * KP, P.D + q * KP, KP, &mbar[slot]);
        }
        r_start += r_dir * cnt;
        r_left -= cnt;
    }
    __device__ __forceinline__ void ring_init(char* wsm, const HmShared& lay) {
        ring = reinterpret_cast<uint8_t*>(wsm + lay.ring);
        mbar = reinterpret_cast<uint64_t*>(wsm + lay.mbar);
        slotB = lay.slot;
        if (lane == 0) {
            for (int k = 0; k < kNSlot; ++k) mbar_init(&mbar[k], 1);
            fence_mbar_init();
        }
        __syncwarp();
        r_left = 0;
        clen = 0;
        cslot = 0; cidx = 0; ccount = 0; cphase = 0; cwait = true;
        for (int k = 0; k < kNSlot; ++k) fill(k);
    }
    // ---- consumer: next node's F (decoded) and, for leaf runs, its D row
    template <bool WANT_D>
    __device__ __forceinline__ void pop(int (&F)[LPL], int (&Dv)[LPL]) {
        if (cwait) {
            mbar_wait(&mbar[cslot], (cphase >> cslot) & 1u);
            __syncwarp();     // the whole warp has observed the phase before any lane reads or refills
            cphase ^= 1u << cslot;
            ccount = (int)((clen >> (8 * cslot)) & 0xffu);
            cidx = 0;
            cwait = false;
        }
        const uint8_t* sb = ring + cslot * slotB;
        if constexpr (FIRST) {
            ld_u8<LPL>(sb + cidx * REC + lane * LPL, Dv);
#pragma unroll
            for (int e = 0; e < LPL; ++e) F[e] = Dv[e] << fbits;
        } else {
            ld_rec<LPL>(sb + cidx * REC, lane, F);
            if constexpr (WANT_D) ld_u8<LPL>(sb + kCH * REC + cidx * KP + lane * LPL, Dv);
        }
        if (++cidx == ccount) {
            __syncwarp();
            fill(cslot);
            cslot = cslot + 1 == kNSlot ? 0 : cslot + 1;
            cwait = true;
        }
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
            pop<false>(F, Dv);
#pragma unroll
            for (int e = 0; e < LPL; ++e) phi[e] += F[e];
            msg_(phi);
            if (p + 2 - lo == target) {
                st_i32<LPL>(P.fwd + moff(p + 1), phi);
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
            pop<false>(F, Dv);
#pragma unroll
            for (int e = 0; e < LPL; ++e) phi[e] += F[e];
            msg_(phi);
            if (hi - p + 2 == target) {
                st_i32<LPL>(P.bwd + moff(p - 1), phi);
                --kk;
                target = kk >= 0 ? (((lenB - 1) >> kk) + 1) : INT_MAX;
            }
        }
    }
    // Handshake (Alg.5); the ring delivers F_j then F_i.  Writes the
    // children's new boundaries: fwd[j] = phi_ij, bwd[i] = phi_ji'.
    __device__ __forceinline__ void global_handshake(int i, int (&pl)[LPL], int (&pr)[LPL]) {
        int Fi[LPL], Fj[LPL], Dv[LPL];
        pop<false>(Fj, Dv);
        pop<false>(Fi, Dv);
        handshake_regs<LPL, PAD, WIN>(Fi, Fj, pl, pr, ws, wsT, lane, K);
        st_i32<LPL>(P.fwd + moff(i + 1), pl);
        st_i32<LPL>(P.bwd + moff(i), pr);
    }

    // ---- leaves
    __device__ __forceinline__ void emit(int node, const int (&L)[LPL], const int (&F)[LPL], const int (&Dv)[LPL],
                                         const int (&R)[LPL]) {
        int lam[LPL], o[LPL];
        int lmin = INT_MAX;
#pragma unroll
        for (int e = 0; e < LPL; ++e) {
            const int lr = L[e] + R[e];
            o[e] = lr + (Dv[e] << fbits);
            lam[e] = lr + F[e];
            if (PAD && lane * LPL + e >= K) lam[e] = INT_MAX;
            lmin = min(lmin, lam[e]);
        }
        st_rec<LPL, PAD>(dst + (size_t)q_of(node) * REC, lane, o, K);
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
                                               uint8_t* sD, int32_t* stk) {
#pragma unroll 1
        for (int k = 0; k < m; ++k) {
            int F[LPL], Dv[LPL];
            pop<true>(F, Dv);
            st_i32<LPL>(sF + k * KP + lane * LPL, F);
            st_u8<LPL>(sD + k * KP + lane * LPL, Dv);
        }
        int lo = 0, hi = m - 1, sp = 0;
        unsigned stkJ = 0;
#pragma unroll 1
        while (true) {
            if (lo == hi) {
                int F[LPL], Dv[LPL];
                ld_i32<LPL>(sF + lo * KP + lane * LPL, F);
                ld_u8<LPL>(sD + lo * KP + lane * LPL, Dv);
                emit(lo0 + lo, L, F, Dv, R);
                if (sp == 0) break;
                --sp;
                __syncwarp();
                // pending piece k = [j_k, hi_k] with hi_0 = m-1 and
                // hi_k = j_{k-1} - 1: only the j's are kept, 4 bits each, in a
                // per-lane register (no lane reads shared state another lane
                // may be rewriting)
                lo = (int)((stkJ >> (4 * sp)) & 0xfu);
                hi = sp == 0 ? m - 1 : (int)((stkJ >> (4 * (sp - 1))) & 0xfu) - 1;
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
            handshake_regs<LPL, PAD, WIN>(Fi, Fj, pl, pr, ws, wsT, lane, K);
            // push the right piece (j, hi, phi_ij, R); continue with (lo, i, L, phi_ji')
            stkJ = (stkJ & ~(0xfu << (4 * sp))) | ((unsigned)j << (4 * sp));
            st_i32<LPL>(stk + (2 * sp) * KP + lane * LPL, pl);
            st_i32<LPL>(stk + (2 * sp + 1) * KP + lane * LPL, R);
            ++sp;
            hi = i;
#pragma unroll
            for (int e = 0; e < LPL; ++e) R[e] = pr[e];
        }
    }
};

template <int LPL, bool VERT, bool PAD, bool WIN, bool FIRST, int NW>
__global__ void __launch_bounds__(NW * 32) hm_kernel(PassArgs a, int chain0, int lstar) {
    extern __shared__ __align__(128) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int KP = 32 * LPL;
    const HmShared lay(KP);
    char* wsm = smem + warp * lay.total;

    Hm<LPL, VERT, PAD, WIN, FIRST> h;
    h.P = frame_ptrs(a.L, a.frame0 + blockIdx.y);
    h.src = FIRST ? h.P.D : (VERT ? h.P.fv : h.P.fh);
    h.dst = VERT ? h.P.fh : h.P.fv;
    h.W = a.L.W; h.K = a.L.K; h.c = chain0 + blockIdx.x; h.lane = lane;
    h.n = VERT ? a.L.H : a.L.W;
    h.fbits = a.fbits; h.ws = a.ws; h.wsT = a.wsT;
    h.last = a.last != 0;
    h.bsum = 0;
    const int n = h.n;
    h.seq.init(n, lstar, warp, NW);
    h.ring_init(wsm, lay);

    int32_t* sF = reinterpret_cast<int32_t*>(wsm + lay.leafF);
    uint8_t* sD = reinterpret_cast<uint8_t*>(wsm + lay.leafD);
    int32_t* stk = reinterpret_cast<int32_t*>(wsm + lay.stack);
    int zero[LPL];
#pragma unroll
    for (int e = 0; e < LPL; ++e) zero[e] = 0;

    if (lstar > 0) {
        // ---- level 0: the whole chain, zero boundary messages
        const int i = n / 2 - 1;
        int pl[LPL], pr[LPL];
#pragma unroll
        for (int e = 0; e < LPL; ++e) { pl[e] = 0; pr[e] = 0; }
        if (warp == 0) { st_i32<LPL>(h.P.fwd + h.moff(0), zero); h.pass_fwd(0, i, pl); }
        if (warp == 1) {
            st_i32<LPL>(h.P.bwd + h.moff(n - 1), zero);
            h.pass_bwd(n - 1, i + 1, pr);
            st_i32<LPL>(h.P.bwd + h.moff(i + 1), pr);
        }
        __syncthreads();
        if (warp == 0) {
            ld_i32<LPL>(h.P.bwd + h.moff(i + 1), pr);
            h.global_handshake(i, pl, pr);
        }
        __syncthreads();
        // ---- global levels 1 .. lstar-1; message loads issued one task ahead
#pragma unroll 1
        for (int lev = 1; lev < lstar; ++lev) {
            int nb_[LPL], ns_[LPL];    // next task's boundary and spine messages
            auto load_msgs = [&](int s, int (&bnd)[LPL], int (&spn)[LPL]) {
                int lo, hi;
                task_bounds(n, lev, s, lo, hi);
                const int ii = lo + (hi - lo + 1) / 2 - 1;
                if (!(s & 1)) { ld_i32<LPL>(h.P.bwd + h.moff(hi), bnd); ld_i32<LPL>(h.P.fwd + h.moff(ii), spn); }
                else { ld_i32<LPL>(h.P.fwd + h.moff(lo), bnd); ld_i32<LPL>(h.P.bwd + h.moff(ii + 1), spn); }
            };
            if (warp < (1 << lev)) load_msgs(warp, nb_, ns_);
#pragma unroll 1
            for (int s = warp; s < (1 << lev); s += NW) {
                int bnd[LPL], spn[LPL];
#pragma unroll
                for (int e = 0; e < LPL; ++e) { bnd[e] = nb_[e]; spn[e] = ns_[e]; }
                if (s + NW < (1 << lev)) load_msgs(s + NW, nb_, ns_);
                int lo, hi;
                task_bounds(n, lev, s, lo, hi);
                const int ii = lo + (hi - lo + 1) / 2 - 1, j = ii + 1;
                if (!(s & 1)) {   // left piece: left boundary kept -> reuse fwd, recompute bwd
                    h.pass_bwd(hi, j, bnd);
                    h.global_handshake(ii, spn, bnd);
                } else {          // right piece: right boundary kept -> reuse bwd, recompute fwd
                    h.pass_fwd(lo, ii, bnd);
                    h.global_handshake(ii, bnd, spn);
                }
            }
            __syncthreads();
        }
    } else {
        if (warp == 0) { st_i32<LPL>(h.P.fwd + h.moff(0), zero); st_i32<LPL>(h.P.bwd + h.moff(n - 1), zero); }
        __syncthreads();
    }
    // ---- leaf blocks at level lstar (boundary messages loaded one block ahead)
    const int nb = 1 << lstar;
    int L[LPL], R[LPL];
    if (warp < nb) {
        int lo, hi;
        task_bounds(n, lstar, warp, lo, hi);
        ld_i32<LPL>(h.P.fwd + h.moff(lo), L);
        ld_i32<LPL>(h.P.bwd + h.moff(hi), R);
    }
#pragma unroll 1
    for (int s = warp; s < nb; s += NW) {
        int lo, hi;
        task_bounds(n, lstar, s, lo, hi);
        int L2[LPL], R2[LPL];
        const int s2 = s + NW;
        if (s2 < nb) {
            int lo2, hi2;
            task_bounds(n, lstar, s2, lo2, hi2);
            ld_i32<LPL>(h.P.fwd + h.moff(lo2), L2);
            ld_i32<LPL>(h.P.bwd + h.moff(hi2), R2);
        }
        h.leaf_block(lo, hi - lo + 1, L, R, sF, sD, stk);
        if (s2 < nb) {
#pragma unroll
            for (int e = 0; e < LPL; ++e) { L[e] = L2[e]; R[e] = R2[e]; }
        }
    }
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

template <int LPL, bool PAD, bool WIN, bool FIRST>
static void launch_cfg(const PassArgs& a, int vertical, int nframes, int wave_chains, cudaStream_t s) {
    constexpr int NW = 4;
    constexpr int KP = 32 * LPL;
    const int chains = vertical ? a.L.W : a.L.H;
    const int n = vertical ? a.L.H : a.L.W;
    const int lstar = leaf_level(n);
    const HmShared lay(KP);
    const int smem = NW * lay.total;
    auto kern = vertical ? hm_kernel<LPL, true, PAD, WIN, false, NW> : hm_kernel<LPL, false, PAD, WIN, FIRST, NW>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int wave = wave_chains > 0 ? wave_chains : chains;
    for (int c0 = 0; c0 < chains; c0 += wave) {
        const int nc = chains - c0 < wave ? chains - c0 : wave;
        kern<<<dim3(nc, nframes), NW * 32, smem, s>>>(a, c0, lstar);
    }
}

template <int LPL, bool PAD, bool WIN>
static void launch_first(const PassArgs& a, int vertical, int nframes, int wave, cudaStream_t s) {
    if (a.first && !vertical) launch_cfg<LPL, PAD, WIN, true>(a, vertical, nframes, wave, s);
    else launch_cfg<LPL, PAD, WIN, false>(a, vertical, nframes, wave, s);
}

template <int LPL>
static void launch_lpl(const PassArgs& a, int vertical, int nframes, int wave, cudaStream_t s) {
    const bool pad = a.L.K != 32 * LPL;
    const bool win = a.T <= LPL + 1;
    if (pad) {
        if (win) launch_first<LPL, true, true>(a, vertical, nframes, wave, s);
        else launch_first<LPL, true, false>(a, vertical, nframes, wave, s);
    } else {
        if (win) launch_first<LPL, false, true>(a, vertical, nframes, wave, s);
        else launch_first<LPL, false, false>(a, vertical, nframes, wave, s);
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
