/*
 * dmm_oracle.c -- CPU oracle for census + Dual MM with hierarchical minorants.
 *
 * TEST INFRASTRUCTURE ONLY (see dmm_oracle.h).  Plain C11, exact int64
 * arithmetic, no blocking / fusion / reordering beyond what the paper's
 * algorithms state.  Each function cites the PAPER.md passage it follows.
 */
#include "dmm_oracle.h"
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

/* floor(x / 2) for any sign (reading R9: "m_i / 2" of Alg.5 P:820 is taken
 * in fixed point with floor). */
static int64_t floor_half(int64_t x) { return x >= 0 ? x / 2 : -((-x + 1) / 2); }
static int64_t floor_div(int64_t x, int64_t n) { return x >= 0 ? x / n : -((-x + n - 1) / n); }

static int64_t penalty(int64_t ws, int T, int a, int b) {
    int d = a > b ? a - b : b - a;
    return ws * (d < T ? d : T);
}

/* ------------------------------------------------------------------ census */
/* P:416 (Sec. 3.1): "Census Transform computed on a small local patch";
 * window / comparison / border per reading R17. */
int oracle_census(const uint8_t* img, int W, int H, int r, uint32_t* codes) {
    if (!img || !codes || W < 1 || H < 1 || r < 1 || r > 2) return 1;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            int c = img[(size_t)y * W + x];
            uint32_t code = 0;
            int bit = 0;
            for (int dy = -r; dy <= r; ++dy)
                for (int dx = -r; dx <= r; ++dx) {
                    if (dx == 0 && dy == 0) continue;
                    int yy = y + dy, xx = x + dx;
                    if (yy < 0) yy = 0;
                    if (yy > H - 1) yy = H - 1;
                    if (xx < 0) xx = 0;
                    if (xx > W - 1) xx = W - 1;
                    if (img[(size_t)yy * W + xx] < c) code |= (uint32_t)1 << bit;
                    ++bit;
                }
            codes[(size_t)y * W + x] = code;
        }
    return 0;
}

static int popcount32(uint32_t v) {
    int n = 0;
    while (v) { n += (int)(v & 1u); v >>= 1; }
    return n;
}

/* "The cost is given by the pixel-wise Hamming distance on the
 * transformed images"; f_i(x_i) = D_i(u(x_i)); reading R18 (left image
 * is the reference, match x - d). */
int oracle_cost_volume(const uint32_t* cl, const uint32_t* cr, int W, int H,
                       int d_min, int K, int oob, uint8_t* D) {
    if (!cl || !cr || !D || W < 1 || H < 1 || K < 1 || K > 256 || oob < 0 || oob > 255) return 1;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int k = 0; k < K; ++k) {
                int xr = x - (d_min + k);
                int v = (xr >= 0 && xr < W)
                            ? popcount32(cl[(size_t)y * W + x] ^ cr[(size_t)y * W + xr])
                            : oob;
                D[((size_t)y * W + x) * K + k] = (uint8_t)v;
            }
    return 0;
}

/* Eq. flow-decoupled-costs: the 2-D data cost D_i(x_i1, x_i2)
 * of the flow label pair is reduced to one optimistic cost per layer by a
 * minimum over the other layer's label.  Plain enumeration, K1*K2 Hamming
 * distances per pixel. */
int oracle_flow_costs(const uint32_t* c1, const uint32_t* c2, int W, int H, int u1_min, int K1,
                      int u2_min, int K2, int oob, uint8_t* f1, uint8_t* f2) {
    if (!c1 || !c2 || !f1 || !f2 || W < 1 || H < 1 || K1 < 1 || K2 < 1 || K1 > 256 || K2 > 256 || oob < 0 ||
        oob > 255)
        return 1;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            uint8_t* o1 = f1 + ((size_t)y * W + x) * K1;
            uint8_t* o2 = f2 + ((size_t)y * W + x) * K2;
            for (int a = 0; a < K1; ++a) o1[a] = 255;
            for (int b = 0; b < K2; ++b) o2[b] = 255;
            for (int a = 0; a < K1; ++a)
                for (int b = 0; b < K2; ++b) {
                    const int xs = x + u1_min + a, ys = y + u2_min + b;
                    const int d = (xs >= 0 && xs < W && ys >= 0 && ys < H)
                                      ? popcount32(c1[(size_t)y * W + x] ^ c2[(size_t)ys * W + xs])
                                      : oob;
                    if (d < o1[a]) o1[a] = (uint8_t)d;
                    if (d < o2[b]) o2[b] = (uint8_t)d;
                }
        }
    return 0;
}

/* ------------------------------------------------------------- messages */
/* Eq. msg-pass, Msg_ij of Alg.5:
 * phi(x_j) = min_{x_i} [a(x_i) + f_ij(x_i, x_j)], by enumeration. */
void oracle_msg_direct(const int64_t* a, int K, int64_t ws, int T, int64_t* out) {
    for (int b = 0; b < K; ++b) {
        int64_t best = a[0] + penalty(ws, T, 0, b);
        for (int x = 1; x < K; ++x) best = min64(best, a[x] + penalty(ws, T, x, b));
        out[b] = best;
    }
}

/* The same minimum for f_ij = ws*min(|a-b|,T), ws >= 0: the untruncated part
 * min_a a(a) + ws|a-b| is the two-pass lower envelope (forward, backward); the
 * truncated part is min_a a(a) + ws*T.  Pinned to oracle_msg_direct. */
void oracle_msg(const int64_t* a, int K, int64_t ws, int T, int64_t* out) {
    int64_t amin = a[0];
    for (int k = 0; k < K; ++k) { out[k] = a[k]; amin = min64(amin, a[k]); }
    for (int k = 1; k < K; ++k) out[k] = min64(out[k], out[k - 1] + ws);
    for (int k = K - 2; k >= 0; --k) out[k] = min64(out[k], out[k + 1] + ws);
    for (int k = 0; k < K; ++k) out[k] = min64(out[k], amin + ws * (int64_t)T);
}

/* -------------------------------------------------------- chain dynamic prog */
/* Left / right min-marginal messages and Eq. P:646-649. */
void oracle_min_marginals(const int64_t* F, int n, int K, int64_t ws, int T, int64_t* m) {
    if (n < 1 || K < 1) return;
    int64_t* left = (int64_t*)calloc((size_t)n * K, sizeof(int64_t));
    int64_t* right = (int64_t*)calloc((size_t)n * K, sizeof(int64_t));
    int64_t* tmp = (int64_t*)malloc((size_t)K * sizeof(int64_t));
    for (int i = 1; i < n; ++i) {           /* phi_{i-1,i} */
        for (int k = 0; k < K; ++k) tmp[k] = left[(size_t)(i - 1) * K + k] + F[(size_t)(i - 1) * K + k];
        oracle_msg(tmp, K, ws, T, &left[(size_t)i * K]);
    }
    for (int i = n - 2; i >= 0; --i) {      /* phi_{i+1,i} */
        for (int k = 0; k < K; ++k) tmp[k] = right[(size_t)(i + 1) * K + k] + F[(size_t)(i + 1) * K + k];
        oracle_msg(tmp, K, ws, T, &right[(size_t)i * K]);
    }
    for (size_t q = 0; q < (size_t)n * K; ++q) m[q] = left[q] + F[q] + right[q];
    free(left); free(right); free(tmp);
}

/* Plain Viterbi with back-pointers (O(n K^2)); lowest-index tie-breaks give
 * the lexicographically smallest optimal labelling. */
int64_t oracle_chain_min(const int64_t* F, int n, int K, int64_t ws, int T, int32_t* x_opt) {
    if (n < 1 || K < 1) return 0;
    /* right-to-left: c[i][k] = F_i(k) + min_j (pen(k,j) + c[i+1][j]) */
    int64_t* c = (int64_t*)malloc((size_t)n * K * sizeof(int64_t));
    int32_t* nxt = (int32_t*)malloc((size_t)n * K * sizeof(int32_t));
    for (int k = 0; k < K; ++k) c[(size_t)(n - 1) * K + k] = F[(size_t)(n - 1) * K + k];
    for (int i = n - 2; i >= 0; --i)
        for (int k = 0; k < K; ++k) {
            int64_t best = 0; int32_t arg = -1;
            for (int j = 0; j < K; ++j) {
                int64_t v = penalty(ws, T, k, j) + c[(size_t)(i + 1) * K + j];
                if (arg < 0 || v < best) { best = v; arg = j; }
            }
            c[(size_t)i * K + k] = F[(size_t)i * K + k] + best;
            nxt[(size_t)i * K + k] = arg;
        }
    int64_t opt = c[0]; int32_t x0 = 0;
    for (int k = 1; k < K; ++k) if (c[k] < opt) { opt = c[k]; x0 = k; }
    if (x_opt) {
        x_opt[0] = x0;
        for (int i = 1; i < n; ++i) x_opt[i] = nxt[(size_t)(i - 1) * K + x_opt[i - 1]];
    }
    free(c); free(nxt);
    return opt;
}

/* ------------------------------------------------- hierarchical minorant */
typedef struct {
    const int64_t* F; int K; int64_t ws; int T; int64_t* lam;
} hm_job;

static void vadd(int64_t* o, const int64_t* a, const int64_t* b, int K) {
    for (int k = 0; k < K; ++k) o[k] = a[k] + b[k];
}

/* rec(lo, hi, L, R): subchain lo..hi decorrelated from the rest of the chain,
 * with L the message into lo from the left and R the message into hi from the
 * right (both 0 at the chain ends).  P:809-810: split into two parts "of
 * approximately the same size" (reading R7: left part floor(len/2)), run the
 * Handshake over the middle edge ij (Alg.5, reading R10: the
 * input message is the one into j from the right), recurse "down to
 * two-variable pieces" and then single nodes (reading R8), where the minorant
 * is lambda_i = L + F_i + R (the min-marginal of the decorrelated piece). */
static void hm_rec(const hm_job* J, int lo, int hi, const int64_t* L, const int64_t* R) {
    const int K = J->K;
    if (lo == hi) {
        for (int k = 0; k < K; ++k) J->lam[(size_t)lo * K + k] = L[k] + J->F[(size_t)lo * K + k] + R[k];
        return;
    }
    int len = hi - lo + 1;
    int i = lo + len / 2 - 1, j = i + 1;
    int64_t* buf = (int64_t*)malloc((size_t)7 * K * sizeof(int64_t));
    int64_t *phiL = buf, *phiR = buf + K, *tmp = buf + 2 * K, *phi_ji = buf + 3 * K;
    int64_t *m = buf + 4 * K, *phi_ij = buf + 5 * K, *phi_ji2 = buf + 6 * K;
    /* left message into i: phi_{i-1,i} (P:638-641 restricted to lo..i) */
    memcpy(phiL, L, (size_t)K * sizeof(int64_t));
    for (int p = lo; p < i; ++p) {
        vadd(tmp, phiL, &J->F[(size_t)p * K], K);
        oracle_msg(tmp, K, J->ws, J->T, phiL);
    }
    /* right message into j: phi_{j+1,j} (P:642-645 restricted to j..hi) */
    memcpy(phiR, R, (size_t)K * sizeof(int64_t));
    for (int p = hi; p > j; --p) {
        vadd(tmp, phiR, &J->F[(size_t)p * K], K);
        oracle_msg(tmp, K, J->ws, J->T, phiR);
    }
    /* Alg.5 line 1: phi_ji := Msg_ji(f_j + phi_{j+1,j}) */
    vadd(tmp, &J->F[(size_t)j * K], phiR, K);
    oracle_msg(tmp, K, J->ws, J->T, phi_ji);
    /* Alg.5 line 2: m_i := phi_{i-1,i} + f_i + phi_ji */
    for (int k = 0; k < K; ++k) m[k] = phiL[k] + J->F[(size_t)i * K + k] + phi_ji[k];
    /* Alg.5 line 3: phi_ij := Msg_ij(m_i/2 - phi_ji), fixed point floor (R9) */
    for (int k = 0; k < K; ++k) tmp[k] = floor_half(m[k] - 2 * phi_ji[k]);
    oracle_msg(tmp, K, J->ws, J->T, phi_ij);
    /* Alg.5 line 4 (bounce back): phi_ji := Msg_ji(-phi_ij) */
    for (int k = 0; k < K; ++k) tmp[k] = -phi_ij[k];
    oracle_msg(tmp, K, J->ws, J->T, phi_ji2);
    /* the two decorrelated subchains (Fig.11) */
    hm_rec(J, lo, i, L, phi_ji2);
    hm_rec(J, j, hi, phi_ij, R);
    free(buf);
}

void oracle_hm(const int64_t* F, int n, int K, int64_t ws, int T, int64_t* lam) {
    if (n < 1 || K < 1) return;
    hm_job J = {F, K, ws, T, lam};
    int64_t* zero = (int64_t*)calloc((size_t)K, sizeof(int64_t));
    hm_rec(&J, 0, n - 1, zero, zero);
    free(zero);
}

/* ------------------------------------------------------------ energy */
/* Eq.3 with f_i = D_i and f_ij = w min(|x_i - x_j|, T). */
int64_t oracle_energy(const uint8_t* D, const int32_t* labels, int W, int H, int K,
                      int w_h, int w_v, int T) {
    int64_t e = 0;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            int32_t l = labels[(size_t)y * W + x];
            e += D[((size_t)y * W + x) * K + l];
            if (x + 1 < W) e += penalty(w_h, T, l, labels[(size_t)y * W + x + 1]);
            if (y + 1 < H) e += penalty(w_v, T, l, labels[(size_t)(y + 1) * W + x]);
        }
    return e;
}

/* ------------------------------------------------------------ Dual MM */
/* Algorithm 2.  f holds all unaries D (reading R3), g only the
 * vertical pairwise terms.  lambda^{2t} = g_^{2t}, lambda^{2t+1} = -f_^{2t+1}
 * (P:255).  Minimize + minorize of f + g_ (lines 1-2) is done per row by the
 * hierarchical minorant h = HM(D + g_); f_ = h - g_ so that f_ + g_ = h is the
 * modular minorant of the row chain f + g_ (side conditions, reading R6).
 * Lines 3-4 likewise per column: v = HM(f_), g_ = v - f_.  The dual bound
 * after each half step is the sum over chains of min_x (chain + modular
 * part) = sum of per-node minima of the minorant (exactness). */
int oracle_dmm(const uint8_t* D, int W, int H, int K, int w_h, int w_v, int T,
               int Fbits, int iters, int64_t* fdual, int64_t* gdual,
               int32_t* labels, int64_t* bound_hist, int64_t* energy, int nthreads) {
    if (!D || W < 1 || H < 1 || K < 1 || K > 256 || w_h < 0 || w_v < 0 || T < 1 ||
        Fbits < 0 || Fbits > 16 || iters < 1)
        return 1;
    const size_t N = (size_t)W * H * K;
    const int64_t scale = (int64_t)1 << Fbits;
    const int64_t wsh = (int64_t)w_h * scale, wsv = (int64_t)w_v * scale;
    int64_t* f = (int64_t*)calloc(N, sizeof(int64_t));
    int64_t* g = (int64_t*)calloc(N, sizeof(int64_t));     /* g_^0 = 0, reading R4 */
    int32_t* lab = (int32_t*)malloc((size_t)W * H * sizeof(int32_t));
#ifdef _OPENMP
    int nth = nthreads > 1 ? nthreads : 1;
#endif
    (void)nthreads;
    for (int t = 0; t < iters; ++t) {
        const int last = (t == iters - 1);
        int64_t bh = 0, bv = 0;
        /* H half step (Alg.2 lines 1-2): every row chain independently */
#ifdef _OPENMP
#pragma omp parallel for num_threads(nth) reduction(+ : bh) schedule(dynamic, 1)
#endif
        for (int y = 0; y < H; ++y) {
            int64_t* Fr = (int64_t*)malloc((size_t)W * K * sizeof(int64_t));
            int64_t* h = (int64_t*)malloc((size_t)W * K * sizeof(int64_t));
            for (int x = 0; x < W; ++x)
                for (int k = 0; k < K; ++k) {
                    size_t q = ((size_t)y * W + x) * K + k;
                    Fr[(size_t)x * K + k] = (int64_t)D[q] * scale + g[q];
                }
            oracle_hm(Fr, W, K, wsh, T, h);
            for (int x = 0; x < W; ++x) {
                int64_t mn = h[(size_t)x * K];
                for (int k = 0; k < K; ++k) {
                    size_t q = ((size_t)y * W + x) * K + k;
                    f[q] = h[(size_t)x * K + k] - g[q];
                    mn = min64(mn, h[(size_t)x * K + k]);
                }
                bh += mn;
            }
            free(Fr); free(h);
        }
        /* V half step (Alg.2 lines 3-4): every column chain independently */
#ifdef _OPENMP
#pragma omp parallel for num_threads(nth) reduction(+ : bv) schedule(dynamic, 1)
#endif
        for (int x = 0; x < W; ++x) {
            int64_t* Gc = (int64_t*)malloc((size_t)H * K * sizeof(int64_t));
            int64_t* v = (int64_t*)malloc((size_t)H * K * sizeof(int64_t));
            for (int y = 0; y < H; ++y)
                for (int k = 0; k < K; ++k)
                    Gc[(size_t)y * K + k] = f[((size_t)y * W + x) * K + k];
            oracle_hm(Gc, H, K, wsv, T, v);
            for (int y = 0; y < H; ++y) {
                int64_t mn = v[(size_t)y * K];
                int32_t arg = 0;
                for (int k = 0; k < K; ++k) {
                    size_t q = ((size_t)y * W + x) * K + k;
                    g[q] = v[(size_t)y * K + k] - f[q];
                    if (v[(size_t)y * K + k] < mn) { mn = v[(size_t)y * K + k]; arg = k; }
                }
                bv += mn;
                if (last) lab[(size_t)y * W + x] = arg;   /* reading R13/R14 */
            }
            free(Gc); free(v);
        }
        if (bound_hist) { bound_hist[2 * t] = bh; bound_hist[2 * t + 1] = bv; }
    }
    if (fdual) memcpy(fdual, f, N * sizeof(int64_t));
    if (gdual) memcpy(gdual, g, N * sizeof(int64_t));
    if (labels) memcpy(labels, lab, (size_t)W * H * sizeof(int32_t));
    if (energy) *energy = oracle_energy(D, lab, W, H, K, w_h, w_v, T) * scale;
    free(f); free(g); free(lab);
    return 0;
}


/* =========================================================================
 * NEXT-3: general penalty + edge weights.  A separate, literal implementation
 * (direct enumeration of every Msg, three Msg per Handshake as Alg.5 prints
 * it) so that the classic path above stays exactly as pinned.
 * ========================================================================= */
#include <math.h>

static int64_t gen_R(const oracle_pen* p, int64_t d) {
    if (d < 0) d = -d;
    const int64_t lin = (int64_t)p->e1 * (d < p->delta ? d : p->delta) +
                        (int64_t)p->e2 * (d > p->delta ? d - p->delta : 0);
    return lin < p->c ? lin : p->c;
}

/* V_ij(d) = floor(w * om * R(|d|) / 16) */
static int64_t gen_V(const oracle_pen* p, int64_t w, int om, int64_t d) {
    return (w * (int64_t)om * gen_R(p, d)) / 16;
}

void oracle_edge_weights(const uint8_t* img, int W, int H, uint8_t* om_h, uint8_t* om_v) {
    uint8_t lut[256];
    for (int g = 0; g < 256; ++g) {
        double v = floor(16.0 * exp(-5.0 * (double)g / 255.0) + 0.5);
        lut[g] = (uint8_t)(v < 1.0 ? 1 : (v > 16.0 ? 16 : v));
    }
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const int i = img[(size_t)y * W + x];
            om_h[(size_t)y * W + x] = x + 1 < W ? lut[abs(i - img[(size_t)y * W + x + 1])] : 16;
            om_v[(size_t)y * W + x] = y + 1 < H ? lut[abs(i - img[(size_t)(y + 1) * W + x])] : 16;
        }
}

/* Msg over one edge (Eq. msg-pass) by enumeration. */
static void gen_msg(const int64_t* a, int K, const oracle_pen* p, int64_t w, int om, int64_t* out) {
    for (int b = 0; b < K; ++b) {
        int64_t best = a[0] + gen_V(p, w, om, b);
        for (int x = 1; x < K; ++x) best = min64(best, a[x] + gen_V(p, w, om, x - b));
        out[b] = best;
    }
}

typedef struct {
    const int64_t* F; int K; int64_t w; const oracle_pen* p; const uint8_t* om; int64_t* lam;
} hmg_job;

static int gen_om(const hmg_job* J, int e) { return J->om ? J->om[e] : 16; }

/* hm_rec of the general model (same recursion, readings R5/R7/R8/R9/R10);
 * edge e joins nodes e and e+1. */
static void hmg_rec(const hmg_job* J, int lo, int hi, const int64_t* L, const int64_t* R) {
    const int K = J->K;
    if (lo == hi) {
        for (int k = 0; k < K; ++k) J->lam[(size_t)lo * K + k] = L[k] + J->F[(size_t)lo * K + k] + R[k];
        return;
    }
    int len = hi - lo + 1;
    int i = lo + len / 2 - 1, j = i + 1;
    int64_t* buf = (int64_t*)malloc((size_t)7 * K * sizeof(int64_t));
    int64_t *phiL = buf, *phiR = buf + K, *tmp = buf + 2 * K, *phi_ji = buf + 3 * K;
    int64_t *m = buf + 4 * K, *phi_ij = buf + 5 * K, *phi_ji2 = buf + 6 * K;
    memcpy(phiL, L, (size_t)K * sizeof(int64_t));
    for (int p = lo; p < i; ++p) {                 /* into p+1 over edge p */
        vadd(tmp, phiL, &J->F[(size_t)p * K], K);
        gen_msg(tmp, K, J->p, J->w, gen_om(J, p), phiL);
    }
    memcpy(phiR, R, (size_t)K * sizeof(int64_t));
    for (int p = hi; p > j; --p) {                 /* into p-1 over edge p-1 */
        vadd(tmp, phiR, &J->F[(size_t)p * K], K);
        gen_msg(tmp, K, J->p, J->w, gen_om(J, p - 1), phiR);
    }
    const int om = gen_om(J, i);                   /* the Handshake edge ij */
    vadd(tmp, &J->F[(size_t)j * K], phiR, K);
    gen_msg(tmp, K, J->p, J->w, om, phi_ji);                          /* Alg.5 line 1 */
    for (int k = 0; k < K; ++k) m[k] = phiL[k] + J->F[(size_t)i * K + k] + phi_ji[k];   /* line 2 */
    for (int k = 0; k < K; ++k) tmp[k] = floor_half(m[k] - 2 * phi_ji[k]);
    gen_msg(tmp, K, J->p, J->w, om, phi_ij);                          /* line 3 (R9) */
    for (int k = 0; k < K; ++k) tmp[k] = -phi_ij[k];
    gen_msg(tmp, K, J->p, J->w, om, phi_ji2);                         /* line 4: bounce back */
    hmg_rec(J, lo, i, L, phi_ji2);
    hmg_rec(J, j, hi, phi_ij, R);
    free(buf);
}

void oracle_hm_general(const int64_t* F, int n, int K, int w, oracle_pen pen, const uint8_t* om, int64_t* lam) {
    if (n < 1 || K < 1) return;
    hmg_job J = {F, K, w, &pen, om, lam};
    int64_t* zero = (int64_t*)calloc((size_t)K, sizeof(int64_t));
    hmg_rec(&J, 0, n - 1, zero, zero);
    free(zero);
}

int64_t oracle_energy_general(const uint8_t* D, const int32_t* labels, int W, int H, int K, int w_h, int w_v,
                              oracle_pen pen, const uint8_t* om_h, const uint8_t* om_v, int Fbits) {
    int64_t e = 0;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const size_t q = (size_t)y * W + x;
            const int32_t l = labels[q];
            e += (int64_t)D[q * K + l] << Fbits;
            if (x + 1 < W) e += gen_V(&pen, w_h, om_h ? om_h[q] : 16, l - labels[q + 1]);
            if (y + 1 < H) e += gen_V(&pen, w_v, om_v ? om_v[q] : 16, l - labels[q + W]);
        }
    return e;
}

/* NEXT-4 minorants of a chain under the general model (om[n-1] edge weights).
 * Iterative minorant, Algorithm 4: lambda := 0; for s = 1..max_pass:
 * for i along the chain, m_i := min-marginal of f - lambda at i computed
 * dynamically (Eq. msg-pass, min-marginal expression P:646-649),
 * lambda_i += gamma_s m_i; reverse the chain.  gamma_s = 2^-gshift for
 * s < max_pass and 1 for the last pass ("For the last pass gamma_s is set to 1
 * to ensure that the output minorant is maximal"); fixed point:
 * gamma m = floor(m / 2^gshift) (reading R32).  The first pass runs from node
 * 0 to node n-1.
 * Naive minorant: lambda = m / n, the min-marginals of f divided
 * by the chain length, floor in fixed point (reading R33). */
static void gen_messages_into(const int64_t* F, const int64_t* lam, int n, int K, const oracle_pen* p, int64_t w,
                              const uint8_t* om, int dir, int64_t* psi) {
    /* psi[i] = message into i from the far side (dir = +1: from the right;
     * dir = -1: from the left) of the chain with unaries F - lam */
    int64_t* tmp = (int64_t*)malloc((size_t)K * sizeof(int64_t));
    const int start = dir > 0 ? n - 1 : 0;
    for (int k = 0; k < K; ++k) psi[(size_t)start * K + k] = 0;
    for (int i = start - dir; i >= 0 && i < n; i -= dir) {
        const int src = i + dir, e = dir > 0 ? i : i - 1;   /* edge (i, i+1) or (i-1, i) */
        for (int k = 0; k < K; ++k)
            tmp[k] = psi[(size_t)src * K + k] + F[(size_t)src * K + k] - lam[(size_t)src * K + k];
        gen_msg(tmp, K, p, w, om ? om[e] : 16, &psi[(size_t)i * K]);
    }
    free(tmp);
}

void oracle_iter_minorant(const int64_t* F, int n, int K, int w, oracle_pen pen, const uint8_t* om, int max_pass,
                          int gshift, int64_t* lam) {
    if (n < 1 || K < 1) return;
    int64_t* psi = (int64_t*)malloc((size_t)n * K * sizeof(int64_t));
    int64_t* phi = (int64_t*)malloc((size_t)K * sizeof(int64_t));
    int64_t* tmp = (int64_t*)malloc((size_t)K * sizeof(int64_t));
    memset(lam, 0, (size_t)n * K * sizeof(int64_t));
    for (int s = 0; s < max_pass; ++s) {
        const int dir = (s % 2 == 0) ? 1 : -1;     /* sweep direction; "Reverse the chain" after each pass */
        const int sh = (s == max_pass - 1) ? 0 : gshift;
        gen_messages_into(F, lam, n, K, &pen, w, om, dir, psi);   /* far side, current remainder */
        for (int k = 0; k < K; ++k) phi[k] = 0;
        const int first = dir > 0 ? 0 : n - 1;
        for (int i = first; i >= 0 && i < n; i += dir) {
            for (int k = 0; k < K; ++k) {
                const size_t q = (size_t)i * K + k;
                const int64_t m = phi[k] + F[q] - lam[q] + psi[q];            /* min-marginal of f - lambda at i */
                lam[q] += sh ? (m >> sh) : m;                                 /* lambda_i += gamma_s m_i (R32) */
            }
            if (i + dir >= 0 && i + dir < n) {
                const int e = dir > 0 ? i : i - 1;
                for (int k = 0; k < K; ++k) tmp[k] = phi[k] + F[(size_t)i * K + k] - lam[(size_t)i * K + k];
                gen_msg(tmp, K, &pen, w, om ? om[e] : 16, phi);
            }
        }
    }
    free(psi); free(phi); free(tmp);
}

void oracle_naive_minorant(const int64_t* F, int n, int K, int w, oracle_pen pen, const uint8_t* om, int64_t* lam) {
    if (n < 1 || K < 1) return;
    int64_t* zero = (int64_t*)calloc((size_t)n * K, sizeof(int64_t));
    int64_t* L = (int64_t*)malloc((size_t)n * K * sizeof(int64_t));
    int64_t* R = (int64_t*)malloc((size_t)n * K * sizeof(int64_t));
    gen_messages_into(F, zero, n, K, &pen, w, om, -1, L);
    gen_messages_into(F, zero, n, K, &pen, w, om, 1, R);
    for (size_t q = 0; q < (size_t)n * K; ++q) lam[q] = floor_div(L[q] + F[q] + R[q], n);
    free(zero); free(L); free(R);
}

static void chain_minorant(int minorant, const int64_t* F, int n, int K, int w, oracle_pen pen, const uint8_t* om,
                           int max_pass, int gshift, int64_t* lam) {
    if (minorant == 1) oracle_iter_minorant(F, n, K, w, pen, om, max_pass, gshift, lam);
    else if (minorant == 2) oracle_naive_minorant(F, n, K, w, pen, om, lam);
    else oracle_hm_general(F, n, K, w, pen, om, lam);
}

/* Algorithm 2 as oracle_dmm, with the general chains and a choice
 * of minorant (0 hierarchical, 1 iterative, 2 naive). */
int oracle_dmm_minorant(const uint8_t* D, int W, int H, int K, int w_h, int w_v, oracle_pen pen,
                        const uint8_t* om_h, const uint8_t* om_v, int Fbits, int iters, int minorant, int max_pass,
                        int gshift, int64_t* fdual, int64_t* gdual, int32_t* labels, int64_t* bound_hist,
                        int64_t* energy, int nthreads);

int oracle_dmm_general(const uint8_t* D, int W, int H, int K, int w_h, int w_v, oracle_pen pen,
                       const uint8_t* om_h, const uint8_t* om_v, int Fbits, int iters, int64_t* fdual,
                       int64_t* gdual, int32_t* labels, int64_t* bound_hist, int64_t* energy, int nthreads) {
    return oracle_dmm_minorant(D, W, H, K, w_h, w_v, pen, om_h, om_v, Fbits, iters, 0, 0, 0, fdual, gdual, labels,
                               bound_hist, energy, nthreads);
}

int oracle_dmm_minorant(const uint8_t* D, int W, int H, int K, int w_h, int w_v, oracle_pen pen,
                        const uint8_t* om_h, const uint8_t* om_v, int Fbits, int iters, int minorant, int max_pass,
                        int gshift, int64_t* fdual, int64_t* gdual, int32_t* labels, int64_t* bound_hist,
                        int64_t* energy, int nthreads) {
    if (minorant < 0 || minorant > 2 || (minorant == 1 && (max_pass < 1 || gshift < 0 || gshift > 30))) return 1;
    if (!D || W < 1 || H < 1 || K < 1 || K > 256 || w_h < 0 || w_v < 0 || pen.e1 < 0 || pen.e2 < pen.e1 ||
        pen.delta < 0 || pen.c < 0 || Fbits < 0 || Fbits > 16 || iters < 1)
        return 1;
    const size_t N = (size_t)W * H * K;
    const int64_t scale = (int64_t)1 << Fbits;
    int64_t* f = (int64_t*)calloc(N, sizeof(int64_t));
    int64_t* g = (int64_t*)calloc(N, sizeof(int64_t));
    int32_t* lab = (int32_t*)malloc((size_t)W * H * sizeof(int32_t));
#ifdef _OPENMP
    int nth = nthreads > 1 ? nthreads : 1;
#endif
    (void)nthreads;
    for (int t = 0; t < iters; ++t) {
        const int last = (t == iters - 1);
        int64_t bh = 0, bv = 0;
#ifdef _OPENMP
#pragma omp parallel for num_threads(nth) reduction(+ : bh) schedule(dynamic, 1)
#endif
        for (int y = 0; y < H; ++y) {
            int64_t* Fr = (int64_t*)malloc((size_t)W * K * sizeof(int64_t));
            int64_t* h = (int64_t*)malloc((size_t)W * K * sizeof(int64_t));
            uint8_t* om = (uint8_t*)malloc((size_t)W);
            for (int x = 0; x < W; ++x) {
                om[x] = om_h ? om_h[(size_t)y * W + x] : 16;
                for (int k = 0; k < K; ++k) {
                    size_t q = ((size_t)y * W + x) * K + k;
                    Fr[(size_t)x * K + k] = (int64_t)D[q] * scale + g[q];
                }
            }
            chain_minorant(minorant, Fr, W, K, w_h, pen, om, max_pass, gshift, h);
            for (int x = 0; x < W; ++x) {
                int64_t mn = h[(size_t)x * K];
                for (int k = 0; k < K; ++k) {
                    size_t q = ((size_t)y * W + x) * K + k;
                    f[q] = h[(size_t)x * K + k] - g[q];
                    mn = min64(mn, h[(size_t)x * K + k]);
                }
                bh += mn;
            }
            free(Fr); free(h); free(om);
        }
#ifdef _OPENMP
#pragma omp parallel for num_threads(nth) reduction(+ : bv) schedule(dynamic, 1)
#endif
        for (int x = 0; x < W; ++x) {
            int64_t* Gc = (int64_t*)malloc((size_t)H * K * sizeof(int64_t));
            int64_t* v = (int64_t*)malloc((size_t)H * K * sizeof(int64_t));
            uint8_t* om = (uint8_t*)malloc((size_t)H);
            for (int y = 0; y < H; ++y) {
                om[y] = om_v ? om_v[(size_t)y * W + x] : 16;
                for (int k = 0; k < K; ++k) Gc[(size_t)y * K + k] = f[((size_t)y * W + x) * K + k];
            }
            chain_minorant(minorant, Gc, H, K, w_v, pen, om, max_pass, gshift, v);
            for (int y = 0; y < H; ++y) {
                int64_t mn = v[(size_t)y * K];
                int32_t arg = 0;
                for (int k = 0; k < K; ++k) {
                    size_t q = ((size_t)y * W + x) * K + k;
                    g[q] = v[(size_t)y * K + k] - f[q];
                    if (v[(size_t)y * K + k] < mn) { mn = v[(size_t)y * K + k]; arg = k; }
                }
                bv += mn;
                if (last) lab[(size_t)y * W + x] = arg;
            }
            free(Gc); free(v); free(om);
        }
        if (bound_hist) { bound_hist[2 * t] = bh; bound_hist[2 * t + 1] = bv; }
    }
    if (fdual) memcpy(fdual, f, N * sizeof(int64_t));
    if (gdual) memcpy(gdual, g, N * sizeof(int64_t));
    if (labels) memcpy(labels, lab, (size_t)W * H * sizeof(int32_t));
    if (energy) *energy = oracle_energy_general(D, lab, W, H, K, w_h, w_v, pen, om_h, om_v, Fbits);
    free(f); free(g); free(lab);
    return 0;
}
