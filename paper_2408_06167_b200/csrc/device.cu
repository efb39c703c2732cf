// device.cu -- sm_100a kernels and the device-facing C ABI of libblindmatch.
//
// Hot path (bm_match, HE-C^3) per (query, set) pair, hoisted order
// (reading R8); every transform is one 8192-point NTT held by a 512-thread CTA (ntt3.cuh):
//   K1 k_tensor  (tile of pairs, limb)   a4: d0, d1, d2 = sum_i tensor(C_u,i, C_s,i) (Karatsuba),
//                                        a contraction over the parts tiled through shared memory
//   K2 k_digits  (pair, digit l)         a5: x_l = INTT_{q_l}(d2[q_l]); ModUp: x0 -> NTT_{q1,P},
//                                        x1 -> NTT_{q0,P}  (3 transforms)
//   K3 k_relin   (pair, component c)     a5+a6: KS_c = sum_j x_j rlk_j over {q0,q1,P}; ModDown fused
//                                        with the rescale by q1 (exact, R22):
//                                        INTT_P, INTT_q1, NTT_q0 (3 transforms) -> C_c (level 0)
//   K4 k_ladder  (pair)                  a7+a8: the log2(s) rotate-and-add steps with C resident in
//                                        shared memory and per-thread scratch in TMEM, 6 transforms
//                                        per step, coefficient-domain output
//   K5 k_out_intt (pair, c)              a8 when s = 1 (no ladder): INTT_q0 of C
// Also here: K6 k_hrot (f2, the hoisted rotation sum), the f3/f4 kernels (query expansion and
// server-side enrollment: k_exp_mask, k_rot1_digits, k_rot1_ks, k_enroll_add) and the f1 kernels
// (compressed scan one level up: k_tensor<3>, k_digits3, k_relin3, k_cmp_mask, k_cmp_rot,
// k_cmp_add), encryption / conversion / key upload, and the host side of the device C ABI.
// Memory-access conventions: NTT-domain data in the pair-coalesced M4 order,
// twiddles in load order (tw_pos), Shoup keys planar (ldkey2).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "bm_common.cuh"
#include "bm_host.h"
#include "ntt3.cuh"
#include "ntt3f.cuh"
using namespace bm::v3;

using namespace bm;
typedef unsigned __int128 u128;

// ================================================================== device constants
__constant__ uint64_t c_cdt[19];

// Workspace per (query, set) pair, 12 N u64:
//   D01 [c][l][N]  d_c[q_l] (NTT)                       K1 -> K3
//   D2  [l][N]     d2[q_l] (NTT)                        K1 -> K2, K3; then the ladder's scratch
//   XC  [2][N]     C = (c0, c1), level 0 (NTT)          K3 -> ladder
//   XU  [4][N]     ModUp'd digits x0~[q1], x0~[P], x1~[q0], x1~[P] (NTT)   K2 -> K3
// The paper order adds a level-0 accumulator ACC [2][N] (K3 sums into it across parts).
struct MatchK {
    PrimeK pr[4];       // q0, q1, P, q2 (f1)
    ulonglong2 pinv[2]; // P^-1 mod q0, q1
    ulonglong2 q1inv;   // q1^-1 mod q0
    uint64_t pmod[2];   // P mod q0, q1
    const uint64_t *rlk, *gk; // PLANAR Shoup keys: poly k at [2k N, 2k N + N) = w, [2k N + N, 2k N + 2N) = w'
    const uint64_t *db, *qry;
    uint64_t *out;
    int64_t n_sets;       // sets in the DB (output row length)
    int64_t jq0, t0, ct;  // chunk = queries [jq0, jq0+cq) x sets [t0, t0+ct); pair pi = a*ct + b
    int32_t cq;
    int32_t p;
    BM_D int64_t out_row(int64_t pi) const { return (jq0 + pi / ct) * n_sets + t0 + pi % ct; }
    uint64_t *D01, *D2, *XC, *XU, *ACC;
    uint64_t *XR, *XO;  // f1: level-0 masked results (NTT), rotated results (coefficients)
};

// a level-0 ciphertext buffer inside the workspace: pair pi, component c at base + pi*stride + c*N
struct CtBuf {
    uint64_t *base;
    int64_t stride;
    BM_D uint64_t *at(int64_t pi, int c) const { return base + pi * stride + (int64_t)c * N; }
};

constexpr int WS_POLYS = 12;      // u64 polynomials of workspace per pair (hoisted order)
constexpr int WS_POLYS_PAPER = 14;

BM_D ulonglong2 ld2(const uint64_t *p) { return __ldg(reinterpret_cast<const ulonglong2 *>(p)); }
BM_D ulonglong2 ld2k(const ulonglong2 *p) { return __ldg(p); }
BM_D void st2(uint64_t *p, uint64_t x, uint64_t y) { *reinterpret_cast<ulonglong2 *>(p) = make_ulonglong2(x, y); }

BM_D uint64_t submod_d(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }

// Planar Shoup keys (rlk, ladder gk): plane w at kp[0, N), plane w' at kp[N, 2N).  One 16-byte load per
// plane gives positions pos, pos + 1 (pos even, lane-contiguous across a warp, like the twiddles' tw_pos):
// ka = (w, w') of pos, kb = (w, w') of pos + 1.
BM_D void ldkey2(const uint64_t *kp, int pos, ulonglong2 &ka, ulonglong2 &kb)
{
    const ulonglong2 w = ld2(kp + pos), wp = ld2(kp + N + pos);
    ka = make_ulonglong2(w.x, wp.x);
    kb = make_ulonglong2(w.y, wp.y);
}
// the same for a poly addressed as ulonglong2 * (a planar poly occupies the bytes of N pairs)
BM_D void ldkey2(const ulonglong2 *kp, int pos, ulonglong2 &ka, ulonglong2 &kb)
{
    ldkey2(reinterpret_cast<const uint64_t *>(kp), pos, ka, kb);
}
// one position of a planar key (pos of any parity: two 8-byte loads)
BM_D ulonglong2 ldkey1(const ulonglong2 *kp, int pos)
{
    const uint64_t *p = reinterpret_cast<const uint64_t *>(kp);
    return make_ulonglong2(__ldg(p + pos), __ldg(p + N + pos));
}

// ================================================================== K1: tensor (a4)
// d0 = sum_i x0_i y0_i, d2 = sum_i x1_i y1_i, d1 = sum_i (x0_i + x1_i)(y0_i + y1_i) - d0 - d2 per
// (query x, set y) pair, limb and NTT-domain coefficient (Karatsuba over the ciphertext
// components, exact mod q) -- for each coefficient a small "query tile x set tile" contraction
// over the parts, tiled like one: a CTA owns TQB queries x TSB sets x CS coefficients of one limb
// and stages the operands of up to PCH parts in shared memory with cp.async (each query / set
// value is fetched from L2 once per CTA and reused TSB / TQB times); every thread then
// accumulates a 2 x 2 block of pairs for one coefficient in 128-bit sums.  A product is
// < (2q)^2 < 2^118, so the sums are folded mod q every 512 parts.
constexpr int TT = 256;                 // threads per tensor CTA
constexpr int TQB = 8, TSB = 4;         // queries x sets per CTA
constexpr int CS = 32;                  // coefficients per CTA
constexpr int PCH = 8;                  // parts staged per round
#ifndef BM_TSL
#define BM_TSL 8
#endif
constexpr int TSL = BM_TSL;             // coefficient slices per CTA (rounds double-buffered)
constexpr size_t TENSOR_SMEM_BYTES = 2 * (size_t)(TQB + TSB) * PCH * 2 * CS * sizeof(uint64_t); // 2 x 48 KiB

BM_D void cp_async16(void *smem, const void *gmem)
{
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem));
}
BM_D uint64_t red128(u128 v, const PrimeK &P) { return reduce128((uint64_t)(v >> 64), (uint64_t)v, P.q, P.r64, P.one_p); }
// x mod q for any x < 2^64, canonical (q1: fold 2^40 = c1 once so that reduce_bnd's x < 2^62 holds)
template <int PI> BM_D uint64_t reduce_any(uint64_t x)
{
    if (Q40<PI>) x = (x & ((1ull << 40) - 1)) + (x >> 40) * ((1ull << 40) - PrimeC<PI>::q); // < 2^40 + 2^44
    return reduce_bnd<PI>(x);
}
// v mod q for a 128-bit v with the prime-specialised lazy Shoup product: hi (2^64 mod q) + lo
template <int PI> BM_D uint64_t red128s(u128 v, ulonglong2 r64)
{
    const uint64_t t = shoup4<PI>((uint64_t)(v >> 64), r64) + reduce_any<PI>((uint64_t)v); // < 5 q
    return reduce_bnd<PI>(t);
}

// q1 limb on the FP64 pipe, exactly: for 0 <= a, b < 2^42 (integers held in doubles),
// r = a b - floor(a b / q1) q1 up to +-q1: hi = fl(a b) and lo = a b - hi (one FMA, exact), the
// quotient from fl(hi / q1) by a round-down add of 1.5 2^52, r = (hi - qt q1) + lo (the FMA's
// exact result is an integer below 2^43, so nothing rounds).  |r| < 3 q1.  7 FP64 instructions,
// which run on their own pipe: the q1-limb CTAs of k_tensor share each SM with q0-limb CTAs whose
// 128-bit integer products load the FMA pipe.
constexpr double MAGIC52 = 6755399441055744.0; // 1.5 2^52: x + M has ulp 1 for |x| < 2^51
BM_D double f64_floor(double x) { return __dadd_rd(x, MAGIC52) - MAGIC52; }
BM_D double mulmod_q1_f64(double a, double b)
{
    constexpr double q = (double)Q1, qinv = 1.0 / (double)Q1;
    const double hi = a * b;
    const double lo = __fma_rn(a, b, -hi);
    const double qt = f64_floor(hi * qinv);
    return __fma_rn(-qt, q, hi) + lo;
}
// exact u64 (< 2^52) <-> double through the 2^52 exponent pattern (one LOP3 + one DADD)
BM_D double u2d(uint64_t x) { return __longlong_as_double((long long)(x | 0x4330000000000000ull)) - 4503599627370496.0; }
// x mod q1 for an integer-valued double |x| < 2^51, as a canonical u64
BM_D uint64_t f64_mod_q1(double x)
{
    constexpr double q = (double)Q1, qinv = 1.0 / (double)Q1;
    double r = __fma_rn(-f64_floor(x * qinv), q, x); // in (-q1, 2 q1)
    r = r < 0 ? r + q : r;
    r = r >= q ? r - q : r;
    return (uint64_t)__double_as_longlong(r + 4503599627370496.0) & ((1ull << 52) - 1);
}

// grid: ((qt * (N / CS) + slice) * nst + st) * 2 + l  (limbs alternate, so each SM holds one
// q0-limb CTA on the integer pipe and one q1-limb CTA on the FP64 pipe; set tiles next: the CTAs
// that share a query slice run together and the query data streams from HBM once)
// NL = limbs per ciphertext (2: level 1; 3: level 2, f1), L = limb index; L = 1 (q1) runs on the FP64
// pipe, L = 0 (q0) and L = 2 (q2, prime index 3) on the integer pipe
// stage the operands of one round (coefficient slice sl, parts i0 .. i0 + pc - 1) with cp.async
template <int L, int NL> BM_D void tensor_stage(const MatchK &K, uint64_t *Qs, uint64_t *Ss, int qt, int sl, int st,
                                                int i0, int pc)
{
    const int tid = threadIdx.x;
    const int c0 = sl * CS;
    const int lpc = __ffs(pc) - 1;
    // rows (tile row, part, comp) of CS u64 = 16 chunks of 16 B
    const int rows = (TQB + TSB) * pc * 2;
#pragma unroll 4
    for (int k = tid; k < rows * (CS / 2); k += TT) {
        const int row = k >> 4, ch = k & 15;
        const int comp = row & 1, part = (row >> 1) & (pc - 1), tr = (row >> 1) >> lpc;
        const uint64_t *src;
        uint64_t *dst;
        if (tr < TQB) {
            int64_t a = (int64_t)qt * TQB + tr;
            a = a < K.cq ? a : K.cq - 1;
            src = K.qry + ((size_t)(K.jq0 + a) * K.p + i0 + part) * 2 * NL * N;
            dst = Qs + ((tr * PCH + part) * 2 + comp) * CS;
        } else {
            int64_t bb = (int64_t)st * TSB + (tr - TQB);
            bb = bb < K.ct ? bb : K.ct - 1;
            src = K.db + ((size_t)(K.t0 + bb) * K.p + i0 + part) * 2 * NL * N;
            dst = Ss + (((tr - TQB) * PCH + part) * 2 + comp) * CS;
        }
        cp_async16(dst + 2 * ch, src + (size_t)(NL * comp + L) * N + c0 + 2 * ch);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// NL = limbs per ciphertext (2: level 1; 3: level 2, f1), L = limb index; L = 1 (q1) runs on the FP64
// pipe, L = 0 (q0) and L = 2 (q2, prime index 3) on the integer pipe.  The CTA walks TSL consecutive
// coefficient slices; the rounds (slice, chunk of PCH parts) are double-buffered: round r + 1's
// operands are copied by cp.async while round r is computed.
template <int L, int NL> BM_D void tensor_tile(const MatchK &K, uint64_t *stage, int qt, int sl0, int st, int part_lo,
                                               int part_hi)
{
    const int tid = threadIdx.x;
    constexpr int PI = L == 2 ? 3 : L;
    constexpr bool INTL = L != 1;
    const PrimeK &P = K.pr[PI];
    constexpr int BUF = (TQB + TSB) * PCH * 2 * CS; // u64 per buffer: Qs [TQB] then Ss [TSB]
    // this thread: coefficient c, pairs (2 su + {0,1}) x (2 sv + {0,1}) of the tile
    const int c = tid & (CS - 1), su = tid >> 6, sv = (tid >> 5) & 1;
    const int n_chunks = (part_hi - part_lo + PCH - 1) / PCH;
    const int R = TSL * n_chunks;
    auto chunk_pc = [&](int j) { const int i0 = part_lo + j * PCH; return part_hi - i0 < PCH ? part_hi - i0 : PCH; };
    tensor_stage<L, NL>(K, stage, stage + TQB * PCH * 2 * CS, qt, sl0, st, part_lo, chunk_pc(0));
    u128 a0[2][2], a1[2][2], a2[2][2];     // q0, q2: 128-bit integer sums
    double f0[2][2], f1[2][2], f2[2][2];   // q1: exact FP64 sums of signed residues
#pragma unroll 1
    for (int r = 0; r < R; r++) {
        const int sl = sl0 + r / n_chunks, j = r % n_chunks, i0 = part_lo + j * PCH, pc = chunk_pc(j);
        if (r + 1 < R) {
            const int r1 = r + 1, j1 = r1 % n_chunks;
            uint64_t *b1 = stage + (size_t)(r1 & 1) * BUF;
            tensor_stage<L, NL>(K, b1, b1 + TQB * PCH * 2 * CS, qt, sl0 + r1 / n_chunks, st, part_lo + j1 * PCH,
                                chunk_pc(j1));
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const uint64_t *Qs = stage + (size_t)(r & 1) * BUF, *Ss = Qs + TQB * PCH * 2 * CS;
        if (j == 0) {
#pragma unroll
            for (int u = 0; u < 2; u++)
#pragma unroll
                for (int v = 0; v < 2; v++) {
                    if (INTL) a0[u][v] = a1[u][v] = a2[u][v] = 0;
                    else f0[u][v] = f1[u][v] = f2[u][v] = 0.0;
                }
        }
#pragma unroll
        for (int i = 0; i < PCH; i++) {
            if (i >= pc) break;
            uint64_t x0[2], x1[2], y0[2], y1[2];
#pragma unroll
            for (int u = 0; u < 2; u++) {
                const uint64_t *rr = Qs + (((2 * su + u) * PCH + i) * 2) * CS + c;
                x0[u] = rr[0];
                x1[u] = rr[CS];
            }
#pragma unroll
            for (int v = 0; v < 2; v++) {
                const uint64_t *rr = Ss + (((2 * sv + v) * PCH + i) * 2) * CS + c;
                y0[v] = rr[0];
                y1[v] = rr[CS];
            }
            if (INTL) {
#pragma unroll
                for (int u = 0; u < 2; u++)
#pragma unroll
                    for (int v = 0; v < 2; v++) {
                        a0[u][v] += (u128)x0[u] * y0[v];
                        a2[u][v] += (u128)x1[u] * y1[v];
                        a1[u][v] += (u128)(x0[u] + x1[u]) * (y0[v] + y1[v]);
                    }
            } else {
                double dx0[2], dx1[2], dxs[2], dy0[2], dy1[2], dys[2];
#pragma unroll
                for (int u = 0; u < 2; u++) dx0[u] = u2d(x0[u]), dx1[u] = u2d(x1[u]), dxs[u] = dx0[u] + dx1[u];
#pragma unroll
                for (int v = 0; v < 2; v++) dy0[v] = u2d(y0[v]), dy1[v] = u2d(y1[v]), dys[v] = dy0[v] + dy1[v];
#pragma unroll
                for (int u = 0; u < 2; u++)
#pragma unroll
                    for (int v = 0; v < 2; v++) {
                        f0[u][v] += mulmod_q1_f64(dx0[u], dy0[v]);
                        f2[u][v] += mulmod_q1_f64(dx1[u], dy1[v]);
                        f1[u][v] += mulmod_q1_f64(dxs[u], dys[v]); // operands < 2 q1 < 2^41
                    }
            }
        }
        // folds: (2q)^2 < 2^118 in 128 bits (q0) / 3 q1 per part below 2^51 (q1): every 512 parts
        if (((i0 + pc - part_lo) & 511) == 0 && i0 + pc < part_hi) {
#pragma unroll
            for (int u = 0; u < 2; u++)
#pragma unroll
                for (int v = 0; v < 2; v++) {
                    if (INTL) {
                        a0[u][v] = red128s<PI>(a0[u][v], P.r64);
                        a1[u][v] = red128s<PI>(a1[u][v], P.r64);
                        a2[u][v] = red128s<PI>(a2[u][v], P.r64);
                    } else {
                        f0[u][v] = (double)f64_mod_q1(f0[u][v]);
                        f1[u][v] = (double)f64_mod_q1(f1[u][v]);
                        f2[u][v] = (double)f64_mod_q1(f2[u][v]);
                    }
                }
        }
        if (j == n_chunks - 1) { // the slice is complete: write its d0, d1, d2
            const uint64_t q = P.q;
#pragma unroll
            for (int u = 0; u < 2; u++)
#pragma unroll
                for (int v = 0; v < 2; v++) {
                    const int64_t a = (int64_t)qt * TQB + 2 * su + u, bb = (int64_t)st * TSB + 2 * sv + v;
                    if (a >= K.cq || bb >= K.ct) continue;
                    const int64_t pi = a * K.ct + bb;
                    const int jj = sl * CS + c;
                    uint64_t d0, d2, kk;
                    if (INTL) {
                        d0 = red128s<PI>(a0[u][v], P.r64);
                        d2 = red128s<PI>(a2[u][v], P.r64);
                        kk = red128s<PI>(a1[u][v], P.r64);
                    } else {
                        d0 = f64_mod_q1(f0[u][v]);
                        d2 = f64_mod_q1(f2[u][v]);
                        kk = f64_mod_q1(f1[u][v]);
                    }
                    K.D01[((size_t)pi * 2 * NL + 0 + L) * N + jj] = d0;
                    K.D01[((size_t)pi * 2 * NL + NL + L) * N + jj] = submod_d(submod_d(kk, d0, q), d2, q);
                    K.D2[((size_t)pi * NL + L) * N + jj] = d2;
                }
        }
        __syncthreads(); // every read of buffer r & 1 is done before round r + 2 overwrites it
    }
}

template <int NL> __global__ void __launch_bounds__(TT, 2) k_tensor(MatchK K, int part_lo, int part_hi)
{
    extern __shared__ uint64_t sm[];
    const int nst = (int)((K.ct + TSB - 1) / TSB);
    int64_t b = blockIdx.x;
    const int l = (int)(b % NL);
    b /= NL;
    const int st = (int)(b % nst);
    b /= nst;
    const int sg = (int)(b % (N / CS / TSL));
    const int qt = (int)(b / (N / CS / TSL));
    if (l == 0) tensor_tile<0, NL>(K, sm, qt, sg * TSL, st, part_lo, part_hi);
    else if (l == 1) tensor_tile<1, NL>(K, sm, qt, sg * TSL, st, part_lo, part_hi);
    else if (NL == 3) tensor_tile<2, NL>(K, sm, qt, sg * TSL, st, part_lo, part_hi);
}

// ================================================================== prime-specialised pointwise helpers
// reduce_bnd<PI>: exact x mod q for x < 2^64 (q0, P) / x < 2^62 (q1), ntt2.cuh.
// x < 8q -> [0, 4q)
template <int PI> BM_D uint64_t red8to4(uint64_t x)
{
    constexpr uint64_t q4 = 4 * PrimeC<PI>::q;
    return x >= q4 ? x - q4 : x;
}

// ================================================================== K2: digits + ModUp + NTT
// CTA (pair, l): x_l = INTT_{q_l}(d2[q_l]) in [0, q_l) (non-centred digit, reading R4), kept in
// shared memory (thread-private slots) between its two ModUp targets:
//   l = 0: x0 mod q1 -> NTT_q1 -> XU[0],  x0 -> NTT_P -> XU[1]
//   l = 1: x1 (< q1 < q0) -> NTT_q0 -> XU[2],  x1 -> NTT_P -> XU[3]
constexpr size_t K2_SMEM_BYTES = (SMEM_WORDS + (size_t)N) * sizeof(uint64_t);
__global__ void __launch_bounds__(T, 1) k_digits(MatchK K)
{
    extern __shared__ uint64_t sm[];
    uint64_t *xs = sm + SMEM_WORDS;
    const int tid = threadIdx.x;
    const int64_t pi = blockIdx.x >> 1;
    const int l = blockIdx.x & 1;
    uint64_t a[E];
    load_eval(a, K.D2 + ((size_t)pi * 2 + l) * N);
    uint64_t *xu = K.XU + ((size_t)pi * 4 + 2 * l) * N;
    if (l == 0) {
        inv<0>(a, sm, K.pr[0]);
#pragma unroll
        for (int e = 0; e < E; e++) {
            xs[tid + T * e] = a[e];
            a[e] = reduce_bnd<1>(a[e]); // x0 < q0 < 2^58: x0 mod q1
        }
        fwd_f<1>(a, sm, K.pr[1].fwdf); // the FP64 pipe (ntt3f.cuh)
    } else {
        inv_f<1>(a, sm, K.pr[1].invf, K.pr[1].ninvf, K.pr[1].ninv_w1f); // the FP64 pipe
#pragma unroll
        for (int e = 0; e < E; e++) xs[tid + T * e] = a[e];
        fwd<0, false>(a, sm, K.pr[0]); // lazy [0, 2 q0): only ever a Shoup-product operand
    }
    store_eval(xu, a);
#pragma unroll
    for (int e = 0; e < E; e++) a[e] = xs[tid + T * e];
    fwd<2, false>(a, sm, K.pr[2]);
    store_eval(xu + N, a);
}

// ================================================================== K3: key switch + ModDown + rescale
// CTA (pair, c), R22 (exact rewriting of ModDown followed by the rescale by q1):
// (the device rlk carries P^-1 in its Q limbs, so the Q-limb inner products below are P^-1 KS_c)
//   KS_c[P]  = x0~[P] rlk0[c][P] + x1~[P] rlk1[c][P]          -> Y = INTT_P  (kept in shared memory)
//   KS_c[q1] = x0~[q1] rlk0[c][q1] + d2[q1] rlk1[c][q1]        -> U = INTT_q1(d_c[q1] + P^-1 KS_c[q1])
//   y^ = centred_P(Y);  R = U - P^-1 y^ (mod q1);  z^ = centred_q1(R)
//   A  = NTT_q0(P^-1 y^ + z^)
//   KS_c[q0] = d2[q0] rlk0[c][q0] + x1~[q0] rlk1[c][q0]
//   C_c = q1^-1 (d_c[q0] + P^-1 KS_c[q0] - A)   (level 0; accumulate: dst += C_c, paper order)
// (the digit of limb j in its own limb is d2[q_j] itself: no transform needed there)
constexpr size_t K3_SMEM_BYTES = (SMEM_WORDS + (size_t)N) * sizeof(uint64_t);
__global__ void __launch_bounds__(T, 1) k_relin(MatchK K, CtBuf dst, int accumulate)
{
    extern __shared__ uint64_t sm[];
    uint64_t *ys = sm + SMEM_WORDS;
    const int tid = threadIdx.x;
    const int64_t pi = blockIdx.x >> 1;
    const int c = blockIdx.x & 1;
    // rlk layout [j][c][l] planar polys of 2N u64.  K3 reads only the w planes (8-byte keys): each limb's
    // inner product x0 k0 + x1 k1 is formed exactly in 128 bits and reduced once (red128s), half the
    // key bytes of two Shoup products (K3 is load-bound: 5.94 -> 5.63 ms)
    const uint64_t *r0 = K.rlk + (size_t)(0 * 2 + c) * 3 * 2 * N, *r1 = K.rlk + (size_t)(1 * 2 + c) * 3 * 2 * N;
    const uint64_t *xu = K.XU + (size_t)pi * 4 * N;
    const uint64_t *d2 = K.D2 + (size_t)pi * 2 * N;
    const uint64_t *dc = K.D01 + ((size_t)pi * 4 + c * 2) * N; // d_c[q0], d_c[q1]
    uint64_t a[E];
    // ---- P limb
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int j = pos_M4(tid, e);
        const ulonglong2 u = ld2(xu + 1 * N + j), v = ld2(xu + 3 * N + j);
        const ulonglong2 w0 = ld2(r0 + 2 * 2 * N + j), w1 = ld2(r1 + 2 * 2 * N + j);
        a[e] = red128s<2>((u128)u.x * w0.x + (u128)v.x * w1.x, K.pr[2].r64);
        a[e + 1] = red128s<2>((u128)u.y * w0.y + (u128)v.y * w1.y, K.pr[2].r64);
    }
    inv<2>(a, sm, K.pr[2]);
#pragma unroll
    for (int e = 0; e < E; e++) ys[tid + T * e] = a[e]; // Y, canonical [0, P), coefficient j_M1(tid, e)
    // ---- q1 limb
    const ulonglong2 pinv1 = K.pinv[1];
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int j = pos_M4(tid, e);
        const ulonglong2 u = ld2(xu + 0 * N + j), v = ld2(d2 + 1 * N + j), dd = ld2(dc + 1 * N + j);
        const ulonglong2 w0 = ld2(r0 + 1 * 2 * N + j), w1 = ld2(r1 + 1 * 2 * N + j);
        const uint64_t ka = red128s<1>((u128)u.x * w0.x + (u128)v.x * w1.x, K.pr[1].r64);
        const uint64_t kb = red128s<1>((u128)u.y * w0.y + (u128)v.y * w1.y, K.pr[1].r64);
        a[e] = reduce_bnd<1>(dd.x + ka);
        a[e + 1] = reduce_bnd<1>(dd.y + kb);
    }
    inv_f<1>(a, sm, K.pr[1].invf, K.pr[1].ninvf, K.pr[1].ninv_w1f); // U, canonical (FP64 pipe)
    // ---- rescale in coefficient form
    const ulonglong2 pinv0 = K.pinv[0];
    // y^ = y - [y > P/2] P, so P^-1 y^ = P^-1 y - [y > P/2] in every q limb (no centring reduction)
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint64_t y = ys[tid + T * e];
        const uint64_t f = y > (QP >> 1) ? 1 : 0;
        const uint64_t R = reduce_bnd<1>(a[e] + f + 4 * Q1 - shoup4<1>(y, pinv1)); // U - P^-1 y^
        const uint64_t z = R > (Q1 >> 1) ? R + (Q0 - Q1) : R;                      // centred, in q0
        a[e] = shoup4<0>(y, pinv0) + z + (f ? Q0 - 1 : 0);                         // < 6 q0
    }
    fwd<0, false>(a, sm, K.pr[0]); // A, in [0, 2 q0)
    // ---- q0 limb and output
    const ulonglong2 q1inv = K.q1inv;
    uint64_t *co = dst.at(pi, c);
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int j = pos_M4(tid, e);
        const ulonglong2 u = ld2(d2 + 0 * N + j), v = ld2(xu + 2 * N + j), dd = ld2(dc + j);
        const ulonglong2 w0 = ld2(r0 + j), w1 = ld2(r1 + j);
        const uint64_t ka = red128s<0>((u128)u.x * w0.x + (u128)v.x * w1.x, K.pr[0].r64);
        const uint64_t kb = red128s<0>((u128)u.y * w0.y + (u128)v.y * w1.y, K.pr[0].r64);
        // d + P^-1 KS - A + 2 q0 < 11 q0
        uint64_t oa = reduce_bnd<0>(shoup4<0>(dd.x + ka + 2 * Q0 - a[e], q1inv));
        uint64_t ob = reduce_bnd<0>(shoup4<0>(dd.y + kb + 2 * Q0 - a[e + 1], q1inv));
        if (accumulate) {
            const ulonglong2 cc = *reinterpret_cast<const ulonglong2 *>(co + j);
            oa = csub(oa + cc.x, Q0);
            ob = csub(ob + cc.y, Q0);
        }
        st2(co + j, oa, ob);
    }
}

// ================================================================== TMEM as thread-private scratch
// The ladder's two per-thread scratch arrays (component 1's P-limb key-switch product, waiting for
// component 0's INTT_P; the last step's t_1) live in tensor memory instead of global memory: 16 u64
// per thread each, written and read back by the same thread.  With the 32x32b shape a warp reaches the
// 32 TMEM lanes of its quarter (warp & 3); the four warps sharing a quarter use disjoint 64-column
// ranges (warp >> 2), so the CTA allocates 256 of the SM's 512 columns (one CTA per SM).
// COLS: the CTA's allocation (power of two, <= 512); each thread owns COLS / 4 columns of its lane
template <uint32_t COLS> BM_D uint32_t tmem_alloc(uint32_t *s_addr) // all threads; this thread's base
{
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(s_addr)),
                     "n"(COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    return *s_addr + ((uint32_t)(32 * (warp & 3)) << 16) + (COLS / 4) * (uint32_t)(warp >> 2);
}
template <uint32_t COLS> BM_D void tmem_free(uint32_t base) // all threads, after every TMEM access of the CTA
{
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if ((threadIdx.x >> 5) == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(COLS) : "memory");
}
BM_D void tmem_st2(uint32_t taddr, uint64_t x, uint64_t y) // 2 u64 <-> 4 columns (wait::st before reading)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"((uint32_t)x),
                 "r"((uint32_t)(x >> 32)), "r"((uint32_t)y), "r"((uint32_t)(y >> 32))
                 : "memory");
}
// 16 u64 of this thread <-> 32 TMEM columns of its lane
BM_D void tmem_st16(uint32_t taddr, const uint64_t v[E])
{
    uint32_t r[32];
#pragma unroll
    for (int i = 0; i < 16; i++) r[2 * i] = (uint32_t)v[i], r[2 * i + 1] = (uint32_t)(v[i] >> 32);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                 "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, "
                 "%32};" ::"r"(taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
                 "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
                 "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
                 "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
                 : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
BM_D void tmem_st8(uint32_t taddr, const uint64_t v[8]) // 8 u64 <-> 16 columns
{
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 8; i++) r[2 * i] = (uint32_t)v[i], r[2 * i + 1] = (uint32_t)(v[i] >> 32);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                 "%13, %14, %15, %16};" ::"r"(taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
                 "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
                 : "memory");
}
BM_D void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
BM_D void tmem_ld16(uint32_t taddr, uint64_t v[E])
{
    uint32_t r[32];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                 "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
                 "[%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                   "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                   "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr)
                 : "memory");
    // the registers are valid only after wait::ld: make them operands of it so nothing reads them earlier
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                   "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                   "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
                 :
                 : "memory");
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = (uint64_t)r[2 * i] | ((uint64_t)r[2 * i + 1] << 32);
}

// ================================================================== fused ladder (a7 + a8)
// One CTA runs the whole log2(s)-step rotate-and-add ladder of one pair with
// the level-0 ciphertext C = (c0, c1) resident in shared memory (NTT domain, indexed by NTT index
// j, padded), so C never leaves the SM between steps.  Per step r = 2^i, g = 5^r mod 2N:
//   digit   x   = INTT_q0(sigma_g(c1)) in [0, q0), lifted to P as is (reading R4); XP = NTT_P(x)
//   comp c  y^c = centred_P(INTT_P(XP gk_r[c][P]))
//           c_c <- c_c + [c = 0] sigma_g(c0) + sigma_g(c1) (P^-1 gk_r[c][q0]) - NTT_q0(P^-1 y^c)
// (P^-1 is folded into the device Galois keys' q0 limb, and P^-1 y^c = P^-1 y - [y > P/2] needs
// no centring reduction)
// The last step leaves the NTT domain directly (INTT is linear, the rounding term y^c is already
// in coefficient form): out_c = INTT_q0(c_c + [c = 0] sigma(c0) + P^-1 sigma(c1) gk[c][q0])
// - P^-1 y^c, i.e. 6 transforms per step and none for the output conversion.
constexpr size_t LADDER_SMEM_BYTES = 3 * SMEM_WORDS * sizeof(uint64_t);


__global__ void __launch_bounds__(T, 1) k_ladder(MatchK K, CtBuf cin, int L)
{
    extern __shared__ uint64_t sm[];
    uint64_t *XB = sm, *S0 = sm + SMEM_WORDS, *S1 = sm + 2 * SMEM_WORDS;
    const int tid = threadIdx.x;
    const int64_t pi = blockIdx.x;
    __shared__ uint32_t s_tmem;
    const uint32_t tks1 = tmem_alloc<256>(&s_tmem), ttsc = tks1 + 32; // TMEM scratch (see tmem_alloc)
    const ulonglong2 pinv = K.pinv[0];
    stage_by_j(S0, cin.at(pi, 0));
    stage_by_j(S1, cin.at(pi, 1));
    uint64_t a[E];
    uint32_t g = 5; // 5^(2^i) mod 2N
#pragma unroll 1
    for (int i = 0; i < L; i++, g = (g * g) & (2 * N - 1)) {
        const bool last = i == L - 1;
        // [rot][c][q0|P] planar polys of 2N u64
        const uint64_t *gq0 = K.gk + (size_t)(i * 4 + 0) * 2 * N, *gp0 = gq0 + 2 * N;
        const uint64_t *gq1 = K.gk + (size_t)(i * 4 + 2) * 2 * N, *gp1 = gq1 + 2 * N;
        __syncthreads(); // S0 / S1 of the previous step (or the initial staging) are complete
        // digit: sigma_g(c1) -> INTT_q0 -> NTT_P
#pragma unroll
        for (int e = 0; e < E; e++) a[e] = S1[pidx(auto_perm(j_M4(tid, e), g))];
        inv<0>(a, XB, K.pr[0]);
        fwd<2, false>(a, XB, K.pr[2]); // lazy [0, 2P): Shoup operand only
        // P-limb key-switch products for both components; component 1's waits in the workspace
#pragma unroll
        for (int h = 0; h < 2; h++) { // two halves of 8 (fewer live registers)
            uint64_t k1[8];
#pragma unroll
            for (int e = 8 * h; e < 8 * h + 8; e += 2) {
                const int pos = pos_M4(tid, e);
                ulonglong2 w0, w0b, w1, w1b;
                ldkey2(gp0, pos, w0, w0b);
                ldkey2(gp1, pos, w1, w1b);
                k1[e - 8 * h] = shoup4<2>(a[e], w1);
                k1[e - 8 * h + 1] = shoup4<2>(a[e + 1], w1b);
                a[e] = shoup4<2>(a[e], w0);
                a[e + 1] = shoup4<2>(a[e + 1], w0b);
            }
            tmem_st8(tks1 + 16 * h, k1);
        }
        tmem_wait_st();
#pragma unroll 1
        for (int c = 0; c < 2; c++) {
            if (c == 1) tmem_ld16(tks1, a); // component 1's P-limb product, parked in TMEM above
            inv<2>(a, XB, K.pr[2]);
            // P^-1 y^c mod q0 with y^c = y - [y > P/2] P:  P^-1 y - [y > P/2], < 5 q0
#pragma unroll
            for (int e = 0; e < E; e++) a[e] = shoup4<0>(a[e], pinv) + (a[e] > (QP >> 1) ? Q0 - 1 : 0);
            uint64_t *S = c ? S1 : S0;
            const uint64_t *gq = c ? gq1 : gq0;
            if (!last) {
                fwd<0, false>(a, XB, K.pr[0]); // NTT_q0(P^-1 y^c), lazy [0, 2 q0)
                ulonglong2 kk[2];
#pragma unroll
                for (int e = 0; e < E; e++) {
                    const int j = j_M4(tid, e), jp = auto_perm(j, g);
                    if (!(e & 1)) ldkey2(gq, pos_M4(tid, e), kk[0], kk[1]);
                    // sigma(c1) P^-1 gk[c][q0] (P^-1 folded into the device key), [0, 4 q0)
                    const uint64_t ks = shoup4<0>(S1[pidx(jp)], kk[e & 1]);
                    uint64_t v = ks + 2 * Q0 - a[e] + S[pidx(j)]; // < 7 q0
                    if (c == 0) v += S0[pidx(jp)];           // < 7 q0
                    a[e] = reduce_bnd<0>(v);
                }
                __syncthreads(); // every read of the old c_c is done
#pragma unroll
                for (int e = 0; e < E; e++) S[pidx(j_M4(tid, e))] = a[e];
            } else {
                tmem_st16(ttsc, a); // P^-1 y^c (coefficient j_M1(tid, e)), < 5 q0
                ulonglong2 kk[2];
#pragma unroll
                for (int e = 0; e < E; e++) {
                    const int j = j_M4(tid, e), jp = auto_perm(j, g);
                    if (!(e & 1)) ldkey2(gq, pos_M4(tid, e), kk[0], kk[1]);
                    const uint64_t ks = shoup4<0>(S1[pidx(jp)], kk[e & 1]);
                    uint64_t v = ks + S[pidx(j)]; // < 5 q0
                    if (c == 0) v += S0[pidx(jp)];
                    a[e] = reduce_bnd<0>(v);
                }
                inv<0>(a, XB, K.pr[0]);
                uint64_t *o = K.out + ((size_t)K.out_row(pi) * 2 + c) * N;
                uint64_t t[E];
                tmem_ld16(ttsc, t);
#pragma unroll
                for (int e = 0; e < E; e++) o[j_M1(tid, e)] = submod_d(a[e], reduce_bnd<0>(t[e]), Q0);
            }
        }
    }
    tmem_free<256>(s_tmem);
}

// ================================================================== f2: hoisted rotation sum
// SURVEY.md sec. 8f, order BM_ORDER_HOISTED_ROT -- NOT the paper's ladder (oracle: hoisted_rot_sum).
// One CTA per pair computes out = sum_{r<s} Rot(C, r) with ONE key switch (Halevi-Shoup hoisting):
//   x = INTT_q0(c1) in [0, q0) (non-centred digit, R4), X~P = NTT_P(x); for r = 1..s-1 the
//   automorphism acts on each NTT-domain digit limb as an index permutation, and
//   A[c][q0] = sum_r sigma_r(c1) (P^-1 hgk_r[c][q0]),  A[c][P] = sum_r sigma_r(X~P) hgk_r[c][P]
//   are accumulated exactly in 128 bits (8-byte keys, no Shoup companions; folded every 64 terms);
//   then one ModDown per component straight to the coefficient-domain output:
//   out_c = INTT_q0(base_c + A[c][q0]) - P^-1 y^c,  y^c = centred_P(INTT_P(A[c][P])),
//   base_0 = sum_{r<s} sigma_r(c0), base_1 = c1.   6 transforms per pair (the ladder: 6 log2 s).
constexpr size_t HROT_SMEM_BYTES = 3 * SMEM_WORDS * sizeof(uint64_t);

__global__ void __launch_bounds__(T, 1) k_hrot(MatchK K, CtBuf cin, const uint64_t *hgk, int s)
{
    extern __shared__ uint64_t sm[];
    // XB: transform exchanges; SX: (c1, X~P) pairs by NTT index (one 16-byte gather per rotation)
    uint64_t *XB = sm;
    ulonglong2 *SX = reinterpret_cast<ulonglong2 *>(sm + SMEM_WORDS);
    uint64_t *SP = sm + SMEM_WORDS; // reused for c0 after the rotation products
    const int tid = threadIdx.x;
    const int64_t pi = blockIdx.x;
    // A [c][q0 | P] (thread-private: 16 u64 per thread and polynomial) lives in TMEM, columns 32 v + 2 e,
    // and P^-1 y^c reuses A[c][P]'s columns once consumed; base_0 waits in the D2 scratch (dead after K3)
    __shared__ uint32_t s_tmem;
    const uint32_t tA = tmem_alloc<512>(&s_tmem);
    uint64_t *b0s = K.D2 + (size_t)pi * 2 * N;
    const ulonglong2 pinv = K.pinv[0];
    // Phases share one call site per transform (an instruction-cache concern: every unrolled
    // transform is ~40 KB of SASS): ph 0 = the digit, ph 1, 2 = the ModDown of component ph - 1.
    uint64_t a[E];
#pragma unroll 1
    for (int ph = 0; ph < 3; ph++) {
        const int c = ph - 1;
        if (ph == 0) { // (c1, .) staged by NTT index; a = c1
            load_eval(a, cin.at(pi, 1));
#pragma unroll
            for (int e = 0; e < E; e++) SX[pidx(j_M4(tid, e))].x = a[e];
        } else {       // y^c = INTT_P(A[c][P]); a = base_c + A[c][q0]
            tmem_ld16(tA + 32 * (2 * c + 1), a); // A[c][P]
            inv<2>(a, XB, K.pr[2]); // y^c (canonical [0, P))
#pragma unroll
            for (int e = 0; e < E; e++) a[e] = shoup4<0>(a[e], pinv) + (a[e] > (QP >> 1) ? Q0 - 1 : 0);
            tmem_st16(tA + 32 * (2 * c + 1), a); // P^-1 y^c (coefficient j_M1(tid, e)) over A[c][P]
            const uint64_t *base = c ? cin.at(pi, 1) : b0s;
#pragma unroll
            for (int e = 0; e < E; e += 2) {
                const int pos = pos_M4(tid, e);
                const ulonglong2 bv = *reinterpret_cast<const ulonglong2 *>(base + pos);
                a[e] = bv.x;
                a[e + 1] = bv.y;
            }
            {
                uint64_t av[E];
                tmem_ld16(tA + 32 * (2 * c), av); // A[c][q0]
#pragma unroll
                for (int e = 0; e < E; e++) a[e] = csub(a[e] + av[e], Q0);
            }
        }
        inv<0>(a, XB, K.pr[0]);
        if (ph > 0) { // out_c = INTT_q0(base_c + A[c][q0]) - P^-1 y^c
            uint64_t *o = K.out + ((size_t)K.out_row(pi) * 2 + c) * N;
            uint64_t t[E];
            tmem_ld16(tA + 32 * (2 * c + 1), t);
#pragma unroll
            for (int e = 0; e < E; e++) o[j_M1(tid, e)] = submod_d(a[e], reduce_bnd<0>(t[e]), Q0);
            continue;
        }
        // ---- digit: X~P = NTT_P(x), staged next to c1
        fwd<2, false>(a, XB, K.pr[2]); // lazy [0, 2P): Shoup / 128-bit product operand
#pragma unroll
        for (int e = 0; e < E; e++) SX[pidx(j_M4(tid, e))].y = a[e];
        __syncthreads();
        // ---- the s-1 rotations' key-switch products, two coefficients (one 16-byte key position) at a
        //      time, the next rotation's keys loaded while this one's are used
#pragma unroll 1
        for (int g2 = 0; g2 < E / 2; g2++) {
            const int e0 = 2 * g2, pos = pos_M4(tid, e0);
            const int j0 = j_M4(tid, e0), j1 = j_M4(tid, e0 + 1);
            u128 A[2][4]; // [coefficient][c * 2 + limb (q0, P)]
#pragma unroll
            for (int u = 0; u < 2; u++)
#pragma unroll
                for (int v = 0; v < 4; v++) A[u][v] = 0;
            ulonglong2 kc[4], kn[4];
#pragma unroll
            for (int v = 0; v < 4; v++) kc[v] = ld2(hgk + (size_t)v * N + pos);
            uint32_t gr = 1;
#pragma unroll 1
            for (int r = 1; r < s; r++) {
                gr = (gr * 5u) & (2 * N - 1); // 5^r mod 2N
                if (r + 1 < s) {
#pragma unroll
                    for (int v = 0; v < 4; v++) kn[v] = ld2(hgk + ((size_t)r * 4 + v) * N + pos);
                }
                const ulonglong2 x0 = SX[pidx(auto_perm(j0, gr))], x1 = SX[pidx(auto_perm(j1, gr))];
#pragma unroll
                for (int c = 0; c < 2; c++) {
                    A[0][2 * c] += (u128)x0.x * kc[2 * c].x;
                    A[1][2 * c] += (u128)x1.x * kc[2 * c].y;
                    A[0][2 * c + 1] += (u128)x0.y * kc[2 * c + 1].x;
                    A[1][2 * c + 1] += (u128)x1.y * kc[2 * c + 1].y;
                }
                if ((r & 63) == 0) { // 64 products of < 2^60 x 2^60 stay below 2^128
#pragma unroll
                    for (int u = 0; u < 2; u++)
#pragma unroll
                        for (int v = 0; v < 4; v++)
                            A[u][v] = (v & 1) ? red128s<2>(A[u][v], K.pr[2].r64) : red128s<0>(A[u][v], K.pr[0].r64);
                }
#pragma unroll
                for (int v = 0; v < 4; v++) kc[v] = kn[v];
            }
#pragma unroll
            for (int v = 0; v < 4; v++) {
                if (v & 1) tmem_st2(tA + 32 * v + 4 * g2, red128s<2>(A[0][v], K.pr[2].r64), red128s<2>(A[1][v], K.pr[2].r64));
                else tmem_st2(tA + 32 * v + 4 * g2, red128s<0>(A[0][v], K.pr[0].r64), red128s<0>(A[1][v], K.pr[0].r64));
            }
        }
        tmem_wait_st(); // the A stores above complete before phases 1, 2 read them back
        // ---- base_0 = sum_{r<s} sigma_r(c0) by log2(s) doublings t <- t + sigma_{2^i}(t) (exact sums mod
        //      q0: the same residues as the term-by-term sum), c0 staged by NTT index over X~P
        __syncthreads();
        stage_by_j(SP, cin.at(pi, 0));
#pragma unroll 1
        for (uint32_t g = 5, w = 1; w < (uint32_t)s; w <<= 1, g = (g * g) & (2 * N - 1)) {
            __syncthreads();
#pragma unroll
            for (int e = 0; e < E; e++) {
                const int j = j_M4(tid, e);
                a[e] = csub(SP[pidx(j)] + SP[pidx(auto_perm(j, g))], Q0);
            }
            __syncthreads();
#pragma unroll
            for (int e = 0; e < E; e++) SP[pidx(j_M4(tid, e))] = a[e];
        }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; e++) b0s[pos_M4(tid, e)] = SP[pidx(j_M4(tid, e))];
    tmem_free<512>(s_tmem);
}
}

// K7: output INTT when there is no ladder (s = 1)
__global__ void __launch_bounds__(T, 1) k_out_intt(MatchK K, CtBuf cin)
{
    extern __shared__ uint64_t sm[];
    const int64_t pi = blockIdx.x >> 1;
    const int c = blockIdx.x & 1;
    uint64_t a[E];
    load_eval(a, cin.at(pi, c));
    inv<0>(a, sm, K.pr[0]);
    store_coef(K.out + ((size_t)K.out_row(pi) * 2 + c) * N, a);
}

// ================================================================== f3: server-side query expansion
// Algorithm 1 "Input Ciphertext Expansion" on the chain
// extended by q2 (readings R24-R26).  Per query ciphertext (level 2 = {q0, q1, q2}, NTT
// domain) and part i < p -- a "ct" below is one (query, part) output:
//   X1 k_exp_mask   (ct, c)  C_i = Res_q2(C (.) X_i): the mask product in all three limbs, y = INTT_q2
//                            of the q2 limb, then per Q limb out = c X_i q2^-1 - NTT(q2^-1 y^) with
//                            q2^-1 y^ = q2^-1 y - [y > q2/2] (q2^-1 is folded into the device masks'
//                            Q limbs, like P^-1 into the key-switching keys): 3 transforms
//   for t < log2 p, r = s 2^t, g = 5^r:  C_i <- C_i + Rot(C_i, r) at level 1 (2-digit key switch):
//   X2 k_rot1_digits (ct, l) sigma_g(c1)[q_l] (an NTT-index gather), x_l = INTT_{q_l} of it, ModUp:
//                            x0 -> NTT_{q1}, NTT_P; x1 -> NTT_{q0}, NTT_P: 3 transforms
//   X3 k_rot1_ks    (ct, c)  KS_c over {q0, q1, P} with gk1 (P^-1 in its Q limbs), y = INTT_P(KS_c[P]),
//                            c_c <- c_c + [c = 0] sigma_g(c0) + P^-1 KS_c - NTT(P^-1 y^) per Q limb: 3
// XU per ct: [0] sigma(c1)[q0] (digit 0 in its own limb), [1] x0~[q1], [2] x0~[P], [3] x1~[q0],
//            [4] sigma(c1)[q1] (digit 1 in its own limb), [5] x1~[P]   (all NTT domain)
struct ExpK {
    PrimeK pr[4];            // q0, q1, P, q2
    ulonglong2 pinv[2];      // P^-1 mod q0, q1
    ulonglong2 q2inv[2];     // q2^-1 mod q0, q1
    const ulonglong2 *mask;  // [p][3 limbs q0,q1,q2][N]; the Q limbs carry q2^-1
    const ulonglong2 *gk;    // this step's level-1 Galois key [2 digits][2 comps][3 limbs q0,q1,P][N]
    const uint64_t *in;      // [n_q][2][3][N] level 2 (the chunk's first query)
    uint64_t *out;           // [n_q][p][2][2][N] level 1 (the chunk's first query)
    uint64_t *XU;            // [cts][6][N]
    int p;
    uint32_t g;              // Galois element of this step
    // f4 enrollment mode (enroll = 1): pure rotation C <- Rot(C) (no add), applied only to the parts
    // whose amount m = (i - k) mod B has bit `bit` set (template u = u0 + ct / p, k = u mod B)
    int enroll, Bk, bit;
    int64_t u0;
    BM_D bool skip(int64_t ct) const
    {
        if (!enroll) return false;
        const int64_t u = u0 + ct / p;
        const int i = (int)(ct % p), k = (int)(u % Bk);
        const int m = ((i - k) % Bk + Bk) % Bk;
        return !((m >> bit) & 1);
    }
};
constexpr int XU_POLYS = 6;
constexpr size_t X1_SMEM_BYTES = (SMEM_WORDS + (size_t)N) * sizeof(uint64_t);
constexpr size_t X2_SMEM_BYTES = 2 * SMEM_WORDS * sizeof(uint64_t);
constexpr size_t X3_SMEM_BYTES = (2 * SMEM_WORDS + (size_t)N) * sizeof(uint64_t);

__global__ void __launch_bounds__(T, 1) k_exp_mask(ExpK K)
{
    extern __shared__ uint64_t sm[];
    uint64_t *ys = sm + SMEM_WORDS;
    const int tid = threadIdx.x;
    const int64_t ct = blockIdx.x >> 1;
    const int c = blockIdx.x & 1;
    const int64_t jq = ct / K.p;
    const int i = (int)(ct % K.p);
    const uint64_t *cin = K.in + ((size_t)jq * 2 + c) * 3 * N; // [l][N]
    const ulonglong2 *mk = K.mask + (size_t)i * 3 * N;
    uint64_t *co = K.out + ((size_t)ct * 2 + c) * 2 * N;     // [l][N]
    uint64_t a[E];
    // q2 limb: y = INTT_q2(c[q2] X_i[q2]) (canonical)
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int pos = pos_M4(tid, e);
        const ulonglong2 v = ld2(cin + 2 * N + pos);
        ulonglong2 ma, mb;
        ldkey2(mk + 2 * N, pos, ma, mb);
        a[e] = reduce_bnd<3>(shoup4<3>(v.x, ma));
        a[e + 1] = reduce_bnd<3>(shoup4<3>(v.y, mb));
    }
    inv_f<3>(a, sm, K.pr[3].invf, K.pr[3].ninvf, K.pr[3].ninv_w1f); // canonical (FP64 pipe)
#pragma unroll
    for (int e = 0; e < E; e++) ys[tid + T * e] = a[e];
    // q1 limb (FP64-pipe transform): q2^-1 y^ mod q1 = q2^-1 y - [y > q2/2]
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint64_t y = a[e];
        a[e] = reduce_bnd<1>(shoup4<1>(y, K.q2inv[1]) + (y > (Q2 >> 1) ? Q1 - 1 : 0));
    }
    fwd_f<1>(a, sm, K.pr[1].fwdf);
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int pos = pos_M4(tid, e);
        const ulonglong2 v = ld2(cin + 1 * N + pos);
        ulonglong2 ma, mb;
        ldkey2(mk + 1 * N, pos, ma, mb);
        const uint64_t xa = shoup4<1>(v.x, ma), xb = shoup4<1>(v.y, mb);
        st2(co + 1 * N + pos, reduce_bnd<1>(xa + Q1 - a[e]), reduce_bnd<1>(xb + Q1 - a[e + 1]));
    }
    // q0 limb
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint64_t y = ys[tid + T * e];
        a[e] = shoup4<0>(y, K.q2inv[0]) + (y > (Q2 >> 1) ? Q0 - 1 : 0); // < 5 q0
    }
    fwd<0>(a, sm, K.pr[0]); // canonical
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int pos = pos_M4(tid, e);
        const ulonglong2 v = ld2(cin + pos);
        ulonglong2 ma, mb;
        ldkey2(mk, pos, ma, mb);
        const uint64_t xa = shoup4<0>(v.x, ma), xb = shoup4<0>(v.y, mb);
        st2(co + pos, reduce_bnd<0>(xa + Q0 - a[e]), reduce_bnd<0>(xb + Q0 - a[e + 1]));
    }
}

// X2: digits of sigma_g(c1) and their ModUp (the rotation's half of k_digits)
__global__ void __launch_bounds__(T, 1) k_rot1_digits(ExpK K)
{
    extern __shared__ uint64_t sm[];
    uint64_t *S = sm + SMEM_WORDS, *xs = S; // xs reuses S once the gather is done (the INTT's barriers)
    const int tid = threadIdx.x;
    const int64_t ct = blockIdx.x >> 1;
    const int l = blockIdx.x & 1;
    if (K.skip(ct)) return;
    const uint64_t *c1 = K.out + ((size_t)ct * 2 + 1) * 2 * N + (size_t)l * N;
    uint64_t *xu = K.XU + (size_t)ct * XU_POLYS * N;
    stage_by_j(S, c1);
    __syncthreads();
    uint64_t a[E];
#pragma unroll
    for (int e = 0; e < E; e++) a[e] = S[pidx(auto_perm(j_M4(tid, e), K.g))];
    store_eval(xu + (size_t)(l == 0 ? 0 : 4) * N, a); // the digit in its own limb: sigma(c1)[q_l]
    if (l == 0) {
        inv<0>(a, sm, K.pr[0]);
#pragma unroll
        for (int e = 0; e < E; e++) {
            xs[tid + T * e] = a[e];
            a[e] = reduce_bnd<1>(a[e]); // x0 < q0 < 2^58: x0 mod q1
        }
        fwd_f<1>(a, sm, K.pr[1].fwdf);
        store_eval(xu + 1 * N, a);
    } else {
        inv_f<1>(a, sm, K.pr[1].invf, K.pr[1].ninvf, K.pr[1].ninv_w1f);
#pragma unroll
        for (int e = 0; e < E; e++) xs[tid + T * e] = a[e];
        fwd<0, false>(a, sm, K.pr[0]); // x1 < q1 < q0; lazy [0, 2 q0): a Shoup operand only
        store_eval(xu + 3 * N, a);
    }
#pragma unroll
    for (int e = 0; e < E; e++) a[e] = xs[tid + T * e];
    fwd<2, false>(a, sm, K.pr[2]);
    store_eval(xu + (size_t)(l == 0 ? 2 : 5) * N, a);
}

// X3: key switch + ModDown + add, one CTA per (ct, component), c_c updated in place
__global__ void __launch_bounds__(T, 1) k_rot1_ks(ExpK K)
{
    extern __shared__ uint64_t sm[];
    uint64_t *S = sm + SMEM_WORDS, *ys = sm + 2 * SMEM_WORDS;
    const int tid = threadIdx.x;
    const int64_t ct = blockIdx.x >> 1;
    const int c = blockIdx.x & 1;
    if (K.skip(ct)) return;
    const uint64_t *xu = K.XU + (size_t)ct * XU_POLYS * N;
    uint64_t *cc = K.out + ((size_t)ct * 2 + c) * 2 * N; // [l][N]
    const uint64_t *c0 = K.out + (size_t)ct * 4 * N;
    const ulonglong2 *k0 = K.gk + (size_t)(0 * 2 + c) * 3 * N, *k1 = K.gk + (size_t)(1 * 2 + c) * 3 * N;
    uint64_t a[E];
    // P limb: y = INTT_P(x0~[P] gk[0][c][P] + x1~[P] gk[1][c][P])
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int pos = pos_M4(tid, e);
        const ulonglong2 u = ld2(xu + 2 * N + pos), v = ld2(xu + 5 * N + pos);
        // 8-byte keys (w planes), exact 128-bit inner products, one reduction (as K3)
        const ulonglong2 w0 = ld2(reinterpret_cast<const uint64_t *>(k0 + 2 * N) + pos);
        const ulonglong2 w1 = ld2(reinterpret_cast<const uint64_t *>(k1 + 2 * N) + pos);
        a[e] = red128s<2>((u128)u.x * w0.x + (u128)v.x * w1.x, K.pr[2].r64);
        a[e + 1] = red128s<2>((u128)u.y * w0.y + (u128)v.y * w1.y, K.pr[2].r64);
    }
    inv<2>(a, sm, K.pr[2]);
#pragma unroll
    for (int e = 0; e < E; e++) ys[tid + T * e] = a[e];
#pragma unroll 1
    for (int l = 1; l >= 0; l--) { // q1 (FP64-pipe transform), then q0
        // P^-1 y^ mod q_l = P^-1 y - [y > P/2]
        if (l == 1) {
#pragma unroll
            for (int e = 0; e < E; e++) {
                const uint64_t y = ys[tid + T * e];
                a[e] = reduce_bnd<1>(shoup4<1>(y, K.pinv[1]) + (y > (QP >> 1) ? Q1 - 1 : 0));
            }
            fwd_f<1>(a, sm, K.pr[1].fwdf);
        } else {
#pragma unroll
            for (int e = 0; e < E; e++) {
                const uint64_t y = ys[tid + T * e];
                a[e] = shoup4<0>(y, K.pinv[0]) + (y > (QP >> 1) ? Q0 - 1 : 0); // < 5 q0
            }
            fwd<0>(a, sm, K.pr[0]);
        }
        if (c == 0) { // sigma_g(c0)[q_l] by an NTT-index gather (c0 is this CTA's to overwrite)
            __syncthreads(); // previous limb's gathers from S are done
            stage_by_j(S, c0 + (size_t)l * N);
            __syncthreads();
        }
        const uint64_t q = l ? Q1 : Q0;
        const ulonglong2 *kl0 = k0 + (size_t)l * N, *kl1 = k1 + (size_t)l * N;
        const uint64_t *x0 = xu + (size_t)(l == 0 ? 0 : 1) * N, *x1 = xu + (size_t)(l == 0 ? 3 : 4) * N;
#pragma unroll
        for (int e = 0; e < E; e += 2) {
            const int pos = pos_M4(tid, e);
            const ulonglong2 u = ld2(x0 + pos), v = ld2(x1 + pos);
            // C + Rot(C) (expansion) or Rot(C) alone (enrollment)
            const ulonglong2 cv = K.enroll ? make_ulonglong2(0, 0)
                                           : *reinterpret_cast<const ulonglong2 *>(cc + (size_t)l * N + pos);
            uint64_t ka, kb;
            const ulonglong2 w0 = ld2(reinterpret_cast<const uint64_t *>(kl0) + pos);
            const ulonglong2 w1 = ld2(reinterpret_cast<const uint64_t *>(kl1) + pos);
            const u128 sa = (u128)u.x * w0.x + (u128)v.x * w1.x, sb = (u128)u.y * w0.y + (u128)v.y * w1.y;
            if (l) {
                ka = red128s<1>(sa, K.pr[1].r64);
                kb = red128s<1>(sb, K.pr[1].r64);
            } else {
                ka = red128s<0>(sa, K.pr[0].r64);
                kb = red128s<0>(sb, K.pr[0].r64);
            }
            uint64_t va = cv.x + ka + q - a[e], vb = cv.y + kb + q - a[e + 1]; // < 11 q
            if (c == 0) {
                va += S[pidx(auto_perm(j_M4(tid, e), K.g))];
                vb += S[pidx(auto_perm(j_M4(tid, e + 1), K.g))];
            }
            a[e] = l ? reduce_bnd<1>(va) : reduce_bnd<0>(va);
            a[e + 1] = l ? reduce_bnd<1>(vb) : reduce_bnd<0>(vb);
        }
        if (c == 0) __syncthreads(); // every gather of the old c0[q_l] is done before it is overwritten
#pragma unroll
        for (int e = 0; e < E; e += 2) st2(cc + (size_t)l * N + pos_M4(tid, e), a[e], a[e + 1]);
    }
}

// f4: set[t][i] += the rotated parts of its templates (elementwise in the NTT domain, canonical)
// grid: (local set, part, comp x limb, N / 256 slices); W [n][p][2][2][N] holds templates u0 .. u0+n-1
__global__ void __launch_bounds__(256) k_enroll_add(const uint64_t *W, int64_t u0, int64_t n, int p, int Bk,
                                                    int64_t t0, uint64_t *db)
{
    const int slice = blockIdx.x % (N / 256);
    int64_t b = blockIdx.x / (N / 256);
    const int cl = (int)(b % 4);
    b /= 4;
    const int i = (int)(b % p);
    const int64_t t = t0 + b / p;
    const uint64_t q = (cl & 1) ? Q1 : Q0;
    const int k = slice * 256 + threadIdx.x;
    const int64_t lo = t * Bk > u0 ? t * Bk : u0, hi = (t + 1) * Bk < u0 + n ? (t + 1) * Bk : u0 + n;
    uint64_t *dst = db + (((size_t)t * p + i) * 4 + cl) * N + k;
    uint64_t acc = *dst;
    for (int64_t u = lo; u < hi; u++) acc = csub(acc + W[(((size_t)(u - u0) * p + i) * 4 + cl) * N + k], q);
    *dst = acc;
}

// ================================================================== f1: output compression
// SURVEY.md sec. 8f row f1 (reading R28): HE-C^3 one
// level up on the extended chain, then the compression.  Per chunk of (query, set) pairs:
//   k_tensor<3>                        tensor + part sum over the three level-2 limbs
//   C1 k_digits3   (pair, digit j)     x_j = INTT_{q_j}(d2[q_j]), ModUp to the other two Q primes and P
//   C2 k_relin3    (pair, c)           KS_c over {q0,q1,q2,P} (rlk2, P^-1 in its Q limbs), ModDown fused
//                                      with Res by q2 (the R22 rewriting with q2 in q1's role): level 1
//   ladder at level 1: log2 s x (k_rot1_digits, k_rot1_ks) with the ladder's level-1 Galois keys
//   C3 k_cmp_mask  (pair, c)           Res_q1(Mul(P)(C, M)): level 0 (q1^-1 folded into M's q0 limb)
//   C4 k_cmp_rot   (pair)              right rotation by u = t mod s (left by S - u) at level 0 and the
//                                      output INTT (u = 0: the INTT only); coefficient domain
//   C5 k_cmp_add                        packed[g] += the s rotated results of group g
constexpr int D2X_POLYS = 9; // XU at level 2: per digit j its 3 ModUp targets (other two Q limbs, P)
constexpr size_t C1_SMEM_BYTES = (SMEM_WORDS + (size_t)N) * sizeof(uint64_t);
constexpr size_t C2_SMEM_BYTES = (SMEM_WORDS + 2 * (size_t)N) * sizeof(uint64_t);
constexpr size_t C4_SMEM_BYTES = 3 * SMEM_WORDS * sizeof(uint64_t);

BM_D uint32_t pow5_mod2n(uint32_t r) // 5^r mod 2N
{
    uint32_t x = 1, b = 5;
    for (; r; r >>= 1, b = (b * b) & (2 * N - 1))
        if (r & 1) x = (x * b) & (2 * N - 1);
    return x;
}

struct CmpK {
    MatchK m;                 // pr[4], pinv[2], q1inv, D01/D2/XU/XC/XR/XO, chunk geometry
    ulonglong2 pinv2;         // P^-1 mod q2
    ulonglong2 q2inv[2];      // q2^-1 mod q0, q1
    const ulonglong2 *rlk2;   // [3 j][2 c][4 limbs q0,q1,q2,P][N]
    const ulonglong2 *gkc;    // [s-1][2 c][2 limbs q0,P][N]
    const ulonglong2 *mask;   // [2 limbs q0,q1][N], q1^-1 in the q0 limb
    uint64_t *scr;            // [pairs][2][N] scratch of k_cmp_rot
    int s;
};

__global__ void __launch_bounds__(T, 1) k_digits3(CmpK C)
{
    extern __shared__ uint64_t sm[];
    uint64_t *xs = sm + SMEM_WORDS;
    const MatchK &K = C.m;
    const int tid = threadIdx.x;
    const int64_t pi = blockIdx.x / 3;
    const int j = (int)(blockIdx.x % 3);
    uint64_t a[E];
    load_eval(a, K.D2 + ((size_t)pi * 3 + j) * N);
    uint64_t *xu = K.XU + ((size_t)pi * D2X_POLYS + 3 * j) * N; // targets: other Q limbs ascending, then P
    if (j == 0) inv<0>(a, sm, K.pr[0]);
    else if (j == 1) inv_f<1>(a, sm, K.pr[1].invf, K.pr[1].ninvf, K.pr[1].ninv_w1f);
    else inv_f<3>(a, sm, K.pr[3].invf, K.pr[3].ninvf, K.pr[3].ninv_w1f);
#pragma unroll
    for (int e = 0; e < E; e++) xs[tid + T * e] = a[e]; // x_j in [0, q_j), non-centred (reading R4)
#pragma unroll 1
    for (int k = 0; k < 3; k++) {
        // target k: the other two Q limbs ascending, then P (prime indices: 0 q0, 1 q1, 2 P, 3 q2)
        const int tp = k == 2 ? 2 : j == 0 ? (k == 0 ? 1 : 3) : j == 1 ? (k == 0 ? 0 : 3) : (k == 0 ? 0 : 1);
#pragma unroll
        for (int e = 0; e < E; e++) {
            const uint64_t x = xs[tid + T * e];
            if (tp == 1) a[e] = j == 0 ? reduce_bnd<1>(x) : x;                 // q1: x0 < 2^58; x2 < q2 < q1
            else if (tp == 3) a[e] = j == 0 ? reduce_bnd<3>(x) : csub(x, Q2);  // q2: x0 < 2^58; x1 < q1 < 2 q2
            else a[e] = x;                                                     // q0 (x1, x2 < q0), P (x < P)
        }
        if (tp == 2) fwd<2, false>(a, sm, K.pr[2]);       // lazy [0, 2P): a Shoup operand only
        else if (tp == 1) fwd_f<1>(a, sm, K.pr[1].fwdf);   // canonical (FP64 pipe)
        else if (tp == 3) fwd_f<3>(a, sm, K.pr[3].fwdf);  // canonical (FP64 pipe)
        else fwd<0, false>(a, sm, K.pr[0]);               // lazy [0, 2 q0)
        store_eval(xu + (size_t)k * N, a);
    }
}

// the digit j's residue in limb tp (prime index) as stored by k_digits3 / k_tensor<3>
BM_D const uint64_t *digit_poly(const MatchK &K, int64_t pi, int j, int tp)
{
    const int lj = j == 2 ? 3 : j; // prime index of digit j's own limb
    if (tp == lj) return K.D2 + ((size_t)pi * 3 + j) * N;
    const int k = tp == 2 ? 2 : j == 0 ? (tp == 1 ? 0 : 1) : j == 1 ? (tp == 0 ? 0 : 1) : (tp == 0 ? 0 : 1);
    return K.XU + ((size_t)pi * D2X_POLYS + 3 * j + k) * N;
}

// C2: key switch with rlk2 + ModDown + Res by q2, per (pair, c) (reading R28; the R22 rewriting):
//   y = INTT_P(KS_c[P]);  U = INTT_q2(d_c[q2] + P^-1 KS_c[q2]);  R = U - P^-1 y^ (mod q2);  z^ = c_q2(R)
//   out_c[q_l] = q2^-1 (d_c[q_l] + P^-1 KS_c[q_l] - NTT_l(P^-1 y^ + z^)),  l = 0, 1
__global__ void __launch_bounds__(T, 1) k_relin3(CmpK C)
{
    extern __shared__ uint64_t sm[];
    uint64_t *ys = sm + SMEM_WORDS, *zs = ys + N;
    const MatchK &K = C.m;
    const int tid = threadIdx.x;
    const int64_t pi = blockIdx.x >> 1;
    const int c = blockIdx.x & 1;
    const uint64_t *dc = K.D01 + ((size_t)pi * 6 + c * 3) * N; // d_c[q0], d_c[q1], d_c[q2]
    // rlk2 [j][c][l][N], l: 0 q0, 1 q1, 2 q2, 3 P
    auto key = [&](int j, int l) { return C.rlk2 + (((size_t)j * 2 + c) * 4 + l) * N; };
    // 8-byte keys: the w plane of a planar poly (positions pos, pos + 1); exact 128-bit inner products
    auto kw = [&](int j, int l, int pos) { return ld2(reinterpret_cast<const uint64_t *>(key(j, l)) + pos); };
    uint64_t a[E];
    // ---- P limb
    {
        const uint64_t *x0 = digit_poly(K, pi, 0, 2), *x1 = digit_poly(K, pi, 1, 2), *x2 = digit_poly(K, pi, 2, 2);
#pragma unroll
        for (int e = 0; e < E; e += 2) {
            const int pos = pos_M4(tid, e);
            const ulonglong2 u = ld2(x0 + pos), v = ld2(x1 + pos), w = ld2(x2 + pos);
            const ulonglong2 k0 = kw(0, 3, pos), k1 = kw(1, 3, pos), k2 = kw(2, 3, pos);
            a[e] = red128s<2>((u128)u.x * k0.x + (u128)v.x * k1.x + (u128)w.x * k2.x, K.pr[2].r64);
            a[e + 1] = red128s<2>((u128)u.y * k0.y + (u128)v.y * k1.y + (u128)w.y * k2.y, K.pr[2].r64);
        }
    }
    inv<2>(a, sm, K.pr[2]);
#pragma unroll
    for (int e = 0; e < E; e++) ys[tid + T * e] = a[e]; // y, canonical
    // ---- q2 limb
    {
        const uint64_t *x0 = digit_poly(K, pi, 0, 3), *x1 = digit_poly(K, pi, 1, 3), *x2 = digit_poly(K, pi, 2, 3);
#pragma unroll
        for (int e = 0; e < E; e += 2) {
            const int pos = pos_M4(tid, e);
            const ulonglong2 u = ld2(x0 + pos), v = ld2(x1 + pos), w = ld2(x2 + pos), dd = ld2(dc + 2 * N + pos);
            const ulonglong2 k0 = kw(0, 2, pos), k1 = kw(1, 2, pos), k2 = kw(2, 2, pos);
            a[e] = reduce_bnd<3>(dd.x + red128s<3>((u128)u.x * k0.x + (u128)v.x * k1.x + (u128)w.x * k2.x, K.pr[3].r64));
            a[e + 1] =
                reduce_bnd<3>(dd.y + red128s<3>((u128)u.y * k0.y + (u128)v.y * k1.y + (u128)w.y * k2.y, K.pr[3].r64));
        }
    }
    inv_f<3>(a, sm, K.pr[3].invf, K.pr[3].ninvf, K.pr[3].ninv_w1f); // U, canonical (FP64 pipe)
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint64_t y = ys[tid + T * e];
        const uint64_t f = y > (QP >> 1) ? 1 : 0;
        zs[tid + T * e] = reduce_bnd<3>(a[e] + f + 4 * Q2 - shoup4<3>(y, C.pinv2)); // R = U - P^-1 y^ (mod q2)
    }
    // ---- q1 (FP64-pipe transform), then q0
#pragma unroll 1
    for (int l = 1; l >= 0; l--) {
        const uint64_t q = l ? Q1 : Q0;
#pragma unroll
        for (int e = 0; e < E; e++) {
            const uint64_t y = ys[tid + T * e], R = zs[tid + T * e];
            const uint64_t f = y > (QP >> 1) ? 1 : 0;
            const uint64_t z = R > (Q2 >> 1) ? R + (q - Q2) : R; // z^ mod q_l
            if (l) a[e] = reduce_bnd<1>(shoup4<1>(y, K.pinv[1]) + (f ? Q1 - 1 : 0) + z);
            else a[e] = shoup4<0>(y, K.pinv[0]) + (f ? Q0 - 1 : 0) + z; // < 6 q0
        }
        if (l) fwd_f<1>(a, sm, K.pr[1].fwdf); // canonical
        else fwd<0, false>(a, sm, K.pr[0]);  // [0, 2 q0)
        const uint64_t *x0 = digit_poly(K, pi, 0, l), *x1 = digit_poly(K, pi, 1, l), *x2 = digit_poly(K, pi, 2, l);
        uint64_t *co = K.XC + ((size_t)pi * 2 + c) * 2 * N + (size_t)l * N;
#pragma unroll
        for (int e = 0; e < E; e += 2) {
            const int pos = pos_M4(tid, e);
            const ulonglong2 u = ld2(x0 + pos), v = ld2(x1 + pos), w = ld2(x2 + pos), dd = ld2(dc + (size_t)l * N + pos);
            uint64_t va, vb;
            const ulonglong2 k0 = kw(0, l, pos), k1 = kw(1, l, pos), k2 = kw(2, l, pos);
            const u128 sa = (u128)u.x * k0.x + (u128)v.x * k1.x + (u128)w.x * k2.x;
            const u128 sb = (u128)u.y * k0.y + (u128)v.y * k1.y + (u128)w.y * k2.y;
            if (l) {
                va = dd.x + red128s<1>(sa, K.pr[1].r64) + Q1 - a[e];
                vb = dd.y + red128s<1>(sb, K.pr[1].r64) + Q1 - a[e + 1];
                st2(co + pos, reduce_bnd<1>(shoup4<1>(va, C.q2inv[1])), reduce_bnd<1>(shoup4<1>(vb, C.q2inv[1])));
            } else {
                va = dd.x + red128s<0>(sa, K.pr[0].r64) + 2 * Q0 - a[e];
                vb = dd.y + red128s<0>(sb, K.pr[0].r64) + 2 * Q0 - a[e + 1];
                st2(co + pos, reduce_bnd<0>(shoup4<0>(va, C.q2inv[0])), reduce_bnd<0>(shoup4<0>(vb, C.q2inv[0])));
            }
        }
    }
}

// C3: Res_q1(Mul(P)(C, M)) per (pair, c): y = INTT_q1(c[q1] M[q1]); out = c[q0] M'[q0] - NTT_q0(q1^-1 y^)
__global__ void __launch_bounds__(T, 1) k_cmp_mask(CmpK C)
{
    extern __shared__ uint64_t sm[];
    const MatchK &K = C.m;
    const int tid = threadIdx.x;
    const int64_t pi = blockIdx.x >> 1;
    const int c = blockIdx.x & 1;
    const uint64_t *ci = K.XC + ((size_t)pi * 2 + c) * 2 * N;
    uint64_t a[E];
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int pos = pos_M4(tid, e);
        const ulonglong2 v = ld2(ci + N + pos);
        ulonglong2 ma, mb;
        ldkey2(C.mask + N, pos, ma, mb);
        a[e] = reduce_bnd<1>(shoup4<1>(v.x, ma));
        a[e + 1] = reduce_bnd<1>(shoup4<1>(v.y, mb));
    }
    inv_f<1>(a, sm, K.pr[1].invf, K.pr[1].ninvf, K.pr[1].ninv_w1f); // y, canonical
#pragma unroll
    for (int e = 0; e < E; e++) a[e] = shoup4<0>(a[e], K.q1inv) + (a[e] > (Q1 >> 1) ? Q0 - 1 : 0); // < 5 q0
    fwd<0>(a, sm, K.pr[0]); // canonical
    uint64_t *co = K.XR + ((size_t)pi * 2 + c) * N;
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int pos = pos_M4(tid, e);
        const ulonglong2 v = ld2(ci + pos);
        ulonglong2 ma, mb;
        ldkey2(C.mask, pos, ma, mb);
        st2(co + pos, reduce_bnd<0>(shoup4<0>(v.x, ma) + Q0 - a[e]), reduce_bnd<0>(shoup4<0>(v.y, mb) + Q0 - a[e + 1]));
    }
}

// C4: right rotation by u = t mod s of the level-0 ciphertext XR (left rotation by S - u with key gkc[u-1]),
// straight to the coefficient domain:  out_0 = INTT_q0(sigma(c0) + sigma(c1) P^-1 gk[0][q0]) - P^-1 y^0,
// out_1 = INTT_q0(sigma(c1) P^-1 gk[1][q0]) - P^-1 y^1;  u = 0: out_c = INTT_q0(c_c).
__global__ void __launch_bounds__(T, 1) k_cmp_rot(CmpK C)
{
    extern __shared__ uint64_t sm[];
    uint64_t *XB = sm, *S0 = sm + SMEM_WORDS, *S1 = sm + 2 * SMEM_WORDS;
    const MatchK &K = C.m;
    const int tid = threadIdx.x;
    const int64_t pi = blockIdx.x;
    const int u = (int)((K.t0 + pi % K.ct) % C.s);
    const uint64_t *ci = K.XR + (size_t)pi * 2 * N;
    uint64_t *co = K.XO + (size_t)pi * 2 * N;
    uint64_t a[E];
    if (u == 0) {
#pragma unroll 1
        for (int c = 0; c < 2; c++) {
            load_eval(a, ci + (size_t)c * N);
            inv<0>(a, XB, K.pr[0]);
            store_coef(co + (size_t)c * N, a);
        }
        return;
    }
    const uint32_t g = (uint32_t)pow5_mod2n(SLOTS - u);
    const ulonglong2 *gk = C.gkc + (size_t)(u - 1) * 4 * N; // [c][q0 | P][N]
    uint64_t *ks1 = C.scr + (size_t)pi * 2 * N, *tsc = ks1 + N;
    stage_by_j(S0, ci);
    stage_by_j(S1, ci + N);
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; e++) a[e] = S1[pidx(auto_perm(j_M4(tid, e), g))];
    inv<0>(a, XB, K.pr[0]);
    fwd<2, false>(a, XB, K.pr[2]); // lazy [0, 2P): Shoup operand only
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int pos = pos_M4(tid, e);
        ulonglong2 w0, w0b, w1, w1b;
        ldkey2(gk + N, pos, w0, w0b);
        ldkey2(gk + 3 * N, pos, w1, w1b);
        st2(ks1 + pos, shoup4<2>(a[e], w1), shoup4<2>(a[e + 1], w1b));
        a[e] = shoup4<2>(a[e], w0);
        a[e + 1] = shoup4<2>(a[e + 1], w0b);
    }
#pragma unroll 1
    for (int c = 0; c < 2; c++) {
        if (c == 1) { // written by this thread above: coherent loads
#pragma unroll
            for (int e = 0; e < E; e += 2) {
                const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(ks1 + pos_M4(tid, e));
                a[e] = v.x;
                a[e + 1] = v.y;
            }
        }
        inv<2>(a, XB, K.pr[2]);
#pragma unroll
        for (int e = 0; e < E; e++) tsc[j_M1(tid, e)] = shoup4<0>(a[e], K.pinv[0]) + (a[e] > (QP >> 1) ? Q0 - 1 : 0);
        const ulonglong2 *gq = gk + (size_t)(2 * c) * N;
#pragma unroll
        for (int e = 0; e < E; e++) {
            const int j = j_M4(tid, e), jp = auto_perm(j, g);
            uint64_t v = shoup4<0>(S1[pidx(jp)], ldkey1(gq, pos_M4(tid, e))); // [0, 4 q0)
            if (c == 0) v += S0[pidx(jp)];
            a[e] = reduce_bnd<0>(v);
        }
        inv<0>(a, XB, K.pr[0]);
        uint64_t *o = co + (size_t)c * N;
#pragma unroll
        for (int e = 0; e < E; e++) {
            const int j = j_M1(tid, e);
            o[j] = submod_d(a[e], reduce_bnd<0>(tsc[j]), Q0);
        }
    }
}

// C5: d_out[query][group] += sum of its rotated results in this chunk (coefficient domain, canonical)
__global__ void __launch_bounds__(256) k_cmp_add(CmpK C, uint64_t *out, int64_t n_groups, int64_t g0, int64_t ng)
{
    const MatchK &K = C.m;
    const int slice = blockIdx.x % (N / 256);
    int64_t b = blockIdx.x / (N / 256);
    const int c = (int)(b & 1);
    b >>= 1;
    const int64_t g = g0 + b % ng, a = b / ng;
    const int k = slice * 256 + threadIdx.x;
    const int64_t tlo = g * C.s > K.t0 ? g * C.s : K.t0;
    const int64_t thi = (g + 1) * C.s < K.t0 + K.ct ? (g + 1) * C.s : K.t0 + K.ct;
    uint64_t *dst = out + (((size_t)(K.jq0 + a) * n_groups + g) * 2 + c) * N + k;
    uint64_t acc = *dst;
    for (int64_t t = tlo; t < thi; t++) acc = csub(acc + K.XO[(((size_t)a * K.ct + (t - K.t0)) * 2 + c) * N + k], Q0);
    *dst = acc;
}

// ================================================================== encryption / conversion / keys
struct EncK {
    PrimeK pr[4];
    const ulonglong2 *pk; // [2][n_limbs][N]
    const int64_t *pt;    // [n][N]
    uint64_t *out;        // [n][2][n_limbs][N]
    uint64_t first_obj, seed;
    int n_limbs;          // 2 (level 1: q0, q1) or 3 (f3 level 2: q0, q1, q2)
    int lp[3];            // prime index of each limb
};

// sample a small polynomial of stream st into sm (residues mod q), adding pt if given
BM_D void sample_to_smem(uint64_t *sm, const Stream &st, int gauss, uint64_t q, uint64_t one_p, const int64_t *pt)
{
    for (int r = 0; r < N / 8 / T; r++) {
        const int b = threadIdx.x + T * r;
        uint64_t d[8];
        chacha_draws(st, (uint32_t)b, d);
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int k = 8 * b + i;
            const int v = gauss ? gauss_of(d[i], c_cdt) : ternary_of(d[i]);
            uint64_t x = v >= 0 ? (uint64_t)v : q - (uint64_t)(-v);
            if (pt) {
                const int64_t m = pt[k];
                uint64_t mr = m >= 0 ? reduce64((uint64_t)m, q, one_p) : submod_d(0, reduce64((uint64_t)(-m), q, one_p), q);
                x = csub(x + mr, q);
            }
            sm[pidx(k)] = x;
        }
    }
}

__global__ void __launch_bounds__(T, 1) k_encrypt(EncK Ek)
{
    extern __shared__ uint64_t sm[];
    const int tid = threadIdx.x;
    const int nl = Ek.n_limbs;
    const int64_t ct = blockIdx.x / nl;
    const int l = (int)(blockIdx.x % nl), pi = Ek.lp[l];
    const uint64_t o = Ek.first_obj + (uint64_t)ct;
    const PrimeK P = Ek.pr[pi];
    const uint64_t q = P.q;
    uint64_t *c0 = Ek.out + ((size_t)ct * 2 * nl + 0 + l) * N;
    uint64_t *c1 = Ek.out + ((size_t)ct * 2 * nl + nl + l) * N;
    const ulonglong2 *pb = Ek.pk + (size_t)(0 + l) * N, *pa = Ek.pk + (size_t)(nl + l) * N;
    uint64_t a[E];
    // phase 0: NTT(u) -> kept in c0 until phase 2;  phase 1: c1 = u a + e1;  phase 2: c0 = u b + e0 + pt
    for (int ph = 0; ph < 3; ph++) {
        __syncthreads();
        const uint32_t purpose = ph == 0 ? P_ENC_U : ph == 1 ? P_ENC_E1 : P_ENC_E0;
        sample_to_smem(sm, make_stream(Ek.seed, purpose, o, 0), ph != 0, q, P.one_p,
                       ph == 2 ? Ek.pt + (size_t)ct * N : nullptr);
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; e++) a[e] = sm[pidx(j_M1(tid, e))];
        fwd_rt(a, sm, P, pi);
        if (ph == 0) {
            store_eval(c0, a);
            continue;
        }
        uint64_t *dst = ph == 1 ? c1 : c0;
        const ulonglong2 *key = ph == 1 ? pa : pb;
#pragma unroll
        for (int e = 0; e < E; e++) {
            const int j = pos_M4(tid, e);
            dst[j] = csub(csub(shoup(c0[j], ldkey1(key, j), q) + a[e], 2 * q), q);
        }
    }
}

struct ConvK {
    PrimeK pr[4];
    const uint64_t *in;
    uint64_t *out;
    int n_limbs;
    int lp[4];          // prime index of each limb
    uint64_t scale[4];  // k_key_ntt: constant folded into each limb (canonical, < q)
    int planar;         // k_key_ntt: write (w, w') as two planes per polynomial (ldkey2) instead of pairs
};

// one block per polynomial; dir 0: coefficient -> NTT, 1: NTT -> coefficient
__global__ void __launch_bounds__(T, 1) k_convert(ConvK C, int dir)
{
    extern __shared__ uint64_t sm[];
    const int64_t poly = blockIdx.x;
    const int li = (int)(poly % C.n_limbs);
    const int pidx_ = C.lp[li];
    const PrimeK P = C.pr[pidx_];
    const uint64_t *in = C.in + (size_t)poly * N;
    uint64_t *out = C.out + (size_t)poly * N;
    uint64_t a[E];
    if (dir == 0) {
        load_coef(a, in);
        fwd_rt(a, sm, P, pidx_);
        __syncthreads(); // in may alias out
        store_eval(out, a);
    } else {
        load_eval(a, in);
        inv_rt(a, sm, P, pidx_);
        __syncthreads();
        store_coef(out, a);
    }
}

// keys: canonical coefficients -> NTT domain Shoup pairs (storage order pos_L3)
__global__ void __launch_bounds__(T, 1) k_key_ntt(ConvK C, ulonglong2 *dst)
{
    extern __shared__ uint64_t sm[];
    const int tid = threadIdx.x;
    const int64_t poly = blockIdx.x;
    const int li = (int)(poly % C.n_limbs);
    const int pidx_ = C.lp[li];
    const PrimeK P = C.pr[pidx_];
    uint64_t a[E];
    load_coef(a, C.in + (size_t)poly * N);
    fwd_rt(a, sm, P, pidx_);
    const uint64_t sc = C.scale[li];
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint64_t w = (uint64_t)((u128)a[e] * sc % P.q); // setup only: plain 128-bit remainder
        const uint64_t wp = (uint64_t)(((u128)w << 64) / P.q);
        if (C.planar) {
            uint64_t *d = reinterpret_cast<uint64_t *>(dst) + (size_t)poly * 2 * N;
            d[pos_M4(tid, e)] = w;
            d[N + pos_M4(tid, e)] = wp;
        } else {
            dst[(size_t)poly * N + pos_M4(tid, e)] = make_ulonglong2(w, wp);
        }
    }
}

// ================================================================== host side: device context
namespace {

struct DevCtx {
    int dev = -1;
    ulonglong2 *tw = nullptr;  // [4][2][N]: q0, q1, P, q2 (f3)
    ulonglong2 *twf = nullptr; // [q1, q2][fwd, inv][N], FP64 form
    PrimeK pr[4] = {};
    ulonglong2 pinv[2], q1inv;
    ulonglong2 q2inv[2];       // f3: q2^-1 mod q0, q1
    ulonglong2 pinv2;          // f1: P^-1 mod q2
    uint64_t pmod[2];
};

std::mutex g_mu;
std::vector<DevCtx *> g_ctx;

ulonglong2 shoup_pair(uint64_t w, uint64_t q) { return make_ulonglong2(w, shoup_companion(w, q)); }
uint64_t powmod_d(uint64_t a, uint64_t e, uint64_t q)
{
    uint64_t r = 1;
    a %= q;
    for (; e; e >>= 1, a = mulmod_h(a, a, q))
        if (e & 1) r = mulmod_h(r, a, q);
    return r;
}

const size_t SMEM_BYTES = SMEM_WORDS * sizeof(uint64_t);

template <typename F> void set_smem(F f) { cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES); }

int ctx_get(DevCtx **out)
{
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) {
        cudaGetLastError();
        return BM_ERR_CUDA;
    }
    std::lock_guard<std::mutex> lk(g_mu);
    if ((int)g_ctx.size() <= dev) g_ctx.resize(dev + 1, nullptr);
    if (g_ctx[dev]) {
        *out = g_ctx[dev];
        return BM_OK;
    }
    DevCtx *C = new DevCtx;
    C->dev = dev;
    std::vector<ulonglong2> h(8 * (size_t)N);
    for (int i = 0; i < 4; i++) {
        const HostPrime &H = host_prime(i);
        for (int k = 0; k < N; k++) {
            h[(size_t)(2 * i) * N + tw_pos(k)] = shoup_pair(H.fwd[k], H.q);     // load-order storage
            h[(size_t)(2 * i + 1) * N + tw_pos(k)] = shoup_pair(H.inv[k], H.q);
        }
    }
    if (cudaMalloc(&C->tw, h.size() * sizeof(ulonglong2)) != cudaSuccess) {
        delete C;
        cudaGetLastError();
        return BM_ERR_OOM;
    }
    cudaMemcpy(C->tw, h.data(), h.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice);
    // q1 and q2 twiddles for the FP64-pipe transforms (ntt3f.cuh): (w, fl(w / q)) as double bit patterns
    auto fpair = [](uint64_t w, uint64_t q) {
        const double dw = (double)w, dq = dw / (double)q;
        uint64_t a, b;
        memcpy(&a, &dw, 8);
        memcpy(&b, &dq, 8);
        return make_ulonglong2(a, b);
    };
    {
        const int fp[2] = {1, 3};
        std::vector<ulonglong2> hf(4 * (size_t)N);
        for (int f = 0; f < 2; f++) {
            const HostPrime &H = host_prime(fp[f]);
            for (int k = 0; k < N; k++)
                hf[(size_t)(2 * f) * N + tw_pos(k)] = fpair(H.fwd[k], H.q),
                                       hf[(size_t)(2 * f + 1) * N + tw_pos(k)] = fpair(H.inv[k], H.q);
        }
        if (cudaMalloc(&C->twf, hf.size() * sizeof(ulonglong2)) != cudaSuccess) {
            cudaFree(C->tw);
            delete C;
            cudaGetLastError();
            return BM_ERR_OOM;
        }
        cudaMemcpy(C->twf, hf.data(), hf.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice);
        for (int f = 0; f < 2; f++) {
            const HostPrime &H = host_prime(fp[f]);
            PrimeK &P = C->pr[fp[f]];
            P.fwdf = C->twf + (size_t)(2 * f) * N;
            P.invf = C->twf + (size_t)(2 * f + 1) * N;
            P.ninvf = fpair(H.ninv, H.q);
            P.ninv_w1f = fpair(mulmod_h(H.ninv, H.inv[1], H.q), H.q);
        }
    }
    for (int i = 0; i < 4; i++) {
        const HostPrime &H = host_prime(i);
        PrimeK &P = C->pr[i];
        P.q = H.q;
        P.q2 = 2 * H.q;
        P.fwd = C->tw + (size_t)(2 * i) * N;
        P.inv = C->tw + (size_t)(2 * i + 1) * N;
        P.ninv = shoup_pair(H.ninv, H.q);
        P.ninv_w1 = shoup_pair(mulmod_h(H.ninv, H.inv[1], H.q), H.q);
        uint64_t r64 = (uint64_t)(((u128)1 << 64) % H.q);
        P.r64 = shoup_pair(r64, H.q);
        P.one_p = (uint64_t)((((u128)1) << 64) / H.q);
    }
    for (int l = 0; l < 2; l++) {
        uint64_t q = C->pr[l].q;
        C->pmod[l] = QP % q;
        C->pinv[l] = shoup_pair(powmod_d(QP % q, q - 2, q), q);
    }
    C->q1inv = shoup_pair(powmod_d(Q1 % Q0, Q0 - 2, Q0), Q0);
    for (int l = 0; l < 2; l++) C->q2inv[l] = shoup_pair(powmod_d(Q2 % C->pr[l].q, C->pr[l].q - 2, C->pr[l].q), C->pr[l].q);
    C->pinv2 = shoup_pair(powmod_d(QP % Q2, Q2 - 2, Q2), Q2);
    cudaMemcpyToSymbol(c_cdt, host_cdt(), sizeof(uint64_t) * 19);
    cudaFuncSetAttribute(k_tensor<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TENSOR_SMEM_BYTES);
    cudaFuncSetAttribute(k_tensor<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TENSOR_SMEM_BYTES);
    cudaFuncSetAttribute(k_digits, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K2_SMEM_BYTES);
    cudaFuncSetAttribute(k_relin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K3_SMEM_BYTES);
    set_smem(k_out_intt);
    cudaFuncSetAttribute(k_ladder, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LADDER_SMEM_BYTES);
    cudaFuncSetAttribute(k_hrot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HROT_SMEM_BYTES);
    set_smem(k_encrypt);
    cudaFuncSetAttribute(k_exp_mask, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)X1_SMEM_BYTES);
    cudaFuncSetAttribute(k_rot1_digits, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)X2_SMEM_BYTES);
    cudaFuncSetAttribute(k_rot1_ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)X3_SMEM_BYTES);
    cudaFuncSetAttribute(k_digits3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C1_SMEM_BYTES);
    cudaFuncSetAttribute(k_relin3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C2_SMEM_BYTES);
    set_smem(k_cmp_mask);
    cudaFuncSetAttribute(k_cmp_rot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C4_SMEM_BYTES);
    set_smem(k_convert);
    set_smem(k_key_ntt);
    if (cudaDeviceSynchronize() != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        cudaFree(C->tw);
        delete C;
        return BM_ERR_CUDA;
    }
    g_ctx[dev] = C;
    *out = C;
    return BM_OK;
}

int launch_check()
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "blindmatch: CUDA error %s\n", cudaGetErrorString(e));
        return BM_ERR_CUDA;
    }
    return BM_OK;
}

// ------------------------------------------------------------------ profiling
struct Prof {
    bool on = false;
    double ms[7] = {0};
    int64_t launches[7] = {0};
    int64_t units[7] = {0};
};
Prof g_prof;
std::mutex g_prof_mu;

struct Rec {
    int cls;
    int64_t units;
    cudaEvent_t a, b;
};

} // namespace

struct bm_pk_dev {
    int dev;
    uint8_t digest[32];
    ulonglong2 *pk;
};
struct bm_xk_dev {
    int dev;
    uint8_t digest[32];
    int32_t d, p, s, n_rot;
    ulonglong2 *pk2;   // [2][3 limbs q0,q1,q2][N] level-2 public key
    ulonglong2 *gk1;   // [n_rot][2][2][3 limbs q0,q1,P][N], P^-1 in the Q limbs
    ulonglong2 *mask;  // [p][3 limbs q0,q1,q2][N] expansion masks X_i, q2^-1 in the Q limbs
    ulonglong2 *emask; // [p][3][N] enrollment masks E_i (f4; nullptr if not uploaded)
};
struct bm_ck_dev {
    int dev;
    uint8_t digest[32];
    int32_t d, p, s, log_s;
    ulonglong2 *rlk2; // [3][2][4 limbs q0,q1,q2,P][N], P^-1 in the Q limbs
    ulonglong2 *gkl;  // [log_s][2][2][3 limbs q0,q1,P][N], P^-1 in the Q limbs
    ulonglong2 *gkc;  // [s-1][2][2 limbs q0,P][N], P^-1 in the q0 limb
    ulonglong2 *mask; // [2 limbs q0,q1][N], q1^-1 in the q0 limb
};
struct bm_evk_dev {
    int dev;
    uint8_t digest[32];
    int32_t n_rot;
    ulonglong2 *rlk; // [2][2][3] planar polys (ldkey2): 2N u64 each
    ulonglong2 *gk;  // [n_rot][2][2] planar polys
    int32_t n_hrot;  // f2 hoisted rotation keys (0: none)
    uint64_t *hgk;   // [n_hrot][2][2][N], NTT domain, plain residues (no Shoup companion), P^-1 in q0
};

// keys -> device NTT-domain Shoup pairs; limb li is multiplied by scale[li] (nullptr: 1); planar
// (default): per polynomial the w plane then the w' plane (read with ldkey2 / ldkey1)
static int upload_key_polys(DevCtx *C, const uint64_t *h, int64_t n_polys, int n_limbs, const int *lp, ulonglong2 **out,
                            const uint64_t *scale = nullptr, bool planar = true)
{
    uint64_t *tmp = nullptr;
    ulonglong2 *dst = nullptr;
    if (cudaMalloc(&tmp, (size_t)n_polys * N * 8) != cudaSuccess ||
        cudaMalloc(&dst, (size_t)n_polys * N * sizeof(ulonglong2)) != cudaSuccess) {
        cudaFree(tmp);
        cudaGetLastError();
        return BM_ERR_OOM;
    }
    cudaMemcpy(tmp, h, (size_t)n_polys * N * 8, cudaMemcpyHostToDevice);
    ConvK K;
    for (int i = 0; i < 4; i++) K.pr[i] = C->pr[i];
    K.in = tmp;
    K.out = nullptr;
    K.n_limbs = n_limbs;
    for (int i = 0; i < 4; i++) K.lp[i] = i < n_limbs ? lp[i] : 0;
    for (int i = 0; i < 4; i++) K.scale[i] = scale && i < n_limbs ? scale[i] : 1;
    K.planar = planar ? 1 : 0;
    k_key_ntt<<<(unsigned)n_polys, T, SMEM_BYTES>>>(K, dst);
    int rc = launch_check();
    if (!rc && cudaDeviceSynchronize() != cudaSuccess) rc = BM_ERR_CUDA;
    cudaFree(tmp);
    if (rc) {
        cudaFree(dst);
        return rc;
    }
    *out = dst;
    return BM_OK;
}

extern "C" {

int bm_pk_to_device(const bm_params *prm, const bm_pk *pk, bm_pk_dev **out)
{
    if (!prm || !pk || !out) return BM_ERR_INVALID_ARG;
    if (memcmp(pk->digest, prm->digest, 32)) return BM_ERR_KEY_MISMATCH;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    bm_pk_dev *d = new bm_pk_dev;
    d->dev = C->dev;
    memcpy(d->digest, prm->digest, 32);
    const int lp[2] = {0, 1};
    rc = upload_key_polys(C, pk->v.data(), 4, 2, lp, &d->pk);
    if (rc) {
        delete d;
        return rc;
    }
    *out = d;
    return BM_OK;
}

int bm_evk_to_device(const bm_params *prm, const bm_evk *evk, bm_evk_dev **out)
{
    if (!prm || !evk || !out) return BM_ERR_INVALID_ARG;
    if (memcmp(evk->digest, prm->digest, 32)) return BM_ERR_KEY_MISMATCH;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    bm_evk_dev *d = new bm_evk_dev;
    d->dev = C->dev;
    memcpy(d->digest, prm->digest, 32);
    d->n_rot = evk->n_rot;
    d->gk = nullptr;
    d->n_hrot = 0;
    d->hgk = nullptr;
    const int lr[3] = {0, 1, 2}, lg[2] = {0, 2};
    // device convention: P^-1 is folded into the Q limbs of the key-switching keys (the ModDown
    // multiplies every Q-limb inner product by P^-1 anyway; exact mod q, saves one product)
    const uint64_t sr[3] = {C->pinv[0].x, C->pinv[1].x, 1}, sg[2] = {C->pinv[0].x, 1};
    rc = upload_key_polys(C, evk->rlk.data(), 12, 3, lr, &d->rlk, sr, true);
    if (!rc && evk->n_rot > 0)
        rc = upload_key_polys(C, evk->gk.data(), 4 * (int64_t)evk->n_rot, 2, lg, &d->gk, sg, true);
    if (!rc && evk->n_hrot > 0) { // f2 keys: keep only the residues (the hoisted sum accumulates in 128 bits)
        ulonglong2 *pairs = nullptr;
        const int64_t np = 4 * (int64_t)evk->n_hrot;
        rc = upload_key_polys(C, evk->hgk.data(), np, 2, lg, &pairs, sg, false); // interleaved: w at +0
        if (!rc && cudaMalloc(&d->hgk, (size_t)np * N * 8) != cudaSuccess) rc = BM_ERR_OOM;
        if (!rc && cudaMemcpy2D(d->hgk, 8, pairs, 16, 8, (size_t)np * N, cudaMemcpyDeviceToDevice) != cudaSuccess)
            rc = BM_ERR_CUDA;
        cudaFree(pairs);
        if (!rc) d->n_hrot = evk->n_hrot;
    }
    if (rc) {
        cudaFree(d->rlk);
        cudaFree(d->gk);
        cudaFree(d->hgk);
        cudaGetLastError();
        delete d;
        return rc;
    }
    *out = d;
    return BM_OK;
}

void bm_pk_dev_free(bm_pk_dev *d)
{
    if (!d) return;
    cudaFree(d->pk);
    delete d;
}
void bm_evk_dev_free(bm_evk_dev *d)
{
    if (!d) return;
    cudaFree(d->rlk);
    cudaFree(d->gk);
    cudaFree(d->hgk);
    delete d;
}

int bm_encrypt(const bm_params *prm, const bm_pk_dev *pk, const int64_t *d_pt, int64_t n_cts, uint64_t first_obj,
               uint64_t seed, uint64_t *d_out, void *stream)
{
    if (!prm || !pk || n_cts < 0 || (n_cts > 0 && (!d_pt || !d_out))) return BM_ERR_INVALID_ARG;
    if (memcmp(pk->digest, prm->digest, 32)) return BM_ERR_KEY_MISMATCH;
    if (n_cts == 0) return BM_OK;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    EncK Ek;
    for (int i = 0; i < 4; i++) Ek.pr[i] = C->pr[i];
    Ek.pk = pk->pk;
    Ek.pt = d_pt;
    Ek.out = d_out;
    Ek.first_obj = first_obj;
    Ek.seed = seed;
    Ek.n_limbs = 2;
    Ek.lp[0] = 0;
    Ek.lp[1] = 1;
    Ek.lp[2] = 3;
    k_encrypt<<<(unsigned)(2 * n_cts), T, SMEM_BYTES, (cudaStream_t)stream>>>(Ek);
    return launch_check();
}

static int encrypt_host_pt(const bm_params *prm, const bm_pk_dev *pk, const std::vector<int64_t> &pt, int64_t n_cts,
                           uint64_t first_obj, uint64_t seed, uint64_t *d_out, void *stream)
{
    int64_t *d_pt = nullptr;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMallocAsync(&d_pt, pt.size() * 8, s) != cudaSuccess) {
        cudaGetLastError();
        return BM_ERR_OOM;
    }
    cudaMemcpyAsync(d_pt, pt.data(), pt.size() * 8, cudaMemcpyHostToDevice, s);
    int rc = bm_encrypt(prm, pk, d_pt, n_cts, first_obj, seed, d_out, stream);
    cudaFreeAsync(d_pt, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) rc = BM_ERR_CUDA;
    return rc;
}

int bm_encrypt_db(const bm_params *prm, const bm_pk_dev *pk, const double *tmpl, int64_t n, int64_t first_set,
                  int64_t n_sets, uint64_t seed, uint64_t *d_out, void *stream)
{
    if (!prm || !pk || n_sets < 0) return BM_ERR_INVALID_ARG;
    if (n_sets == 0) return BM_OK;
    std::vector<int64_t> pt((size_t)n_sets * prm->p * N);
    int rc = bm_encode_db(prm, tmpl, n, first_set, n_sets, pt.data());
    if (rc) return rc;
    return encrypt_host_pt(prm, pk, pt, n_sets * prm->p, (uint64_t)first_set * prm->p, seed, d_out, stream);
}

int bm_encrypt_query(const bm_params *prm, const bm_pk_dev *pk, const double *q, int64_t nq, int64_t first_query,
                     uint64_t seed, uint64_t *d_out, void *stream)
{
    if (!prm || !pk || nq < 0 || first_query < 0) return BM_ERR_INVALID_ARG;
    if (nq == 0) return BM_OK;
    std::vector<int64_t> pt((size_t)nq * prm->p * N);
    int rc = bm_encode_query(prm, q, nq, pt.data());
    if (rc) return rc;
    return encrypt_host_pt(prm, pk, pt, nq * prm->p, (uint64_t)first_query * prm->p, seed, d_out, stream);
}

static int convert(const bm_params *prm, const uint64_t *in, int64_t n_cts, int32_t n_limbs, uint64_t *out,
                   void *stream, int dir)
{
    if (!prm || n_cts < 0 || n_limbs < 1 || n_limbs > 3 || (n_cts && (!in || !out))) return BM_ERR_INVALID_ARG;
    if (n_cts == 0) return BM_OK;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    ConvK K;
    for (int i = 0; i < 4; i++) K.pr[i] = C->pr[i];
    K.in = in;
    K.out = out;
    K.n_limbs = n_limbs;
    K.lp[0] = 0;
    K.lp[1] = 1;
    K.lp[2] = 3; // level-2 limb q2 (f3)
    k_convert<<<(unsigned)(n_cts * 2 * n_limbs), T, SMEM_BYTES, (cudaStream_t)stream>>>(K, dir);
    return launch_check();
}

int bm_ct_to_coeff(const bm_params *prm, const uint64_t *d_in, int64_t n_cts, int32_t n_limbs, uint64_t *d_out,
                   void *stream)
{
    return convert(prm, d_in, n_cts, n_limbs, d_out, stream, 1);
}
int bm_ct_from_coeff(const bm_params *prm, const uint64_t *d_in, int64_t n_cts, int32_t n_limbs, uint64_t *d_out,
                     void *stream)
{
    return convert(prm, d_in, n_cts, n_limbs, d_out, stream, 0);
}

// ------------------------------------------------------------------ f3: query expansion
static int upload_masks(DevCtx *C, const bm_params *prm, const int64_t *h_masks, ulonglong2 **out)
{
    // integer plaintexts -> residues per limb (q0, q1, q2), q2^-1 folded into the Q limbs
    std::vector<uint64_t> m(3 * (size_t)prm->p * N);
    const uint64_t qs[3] = {Q0, Q1, Q2};
    for (int i = 0; i < prm->p; i++)
        for (int l = 0; l < 3; l++)
            for (int k = 0; k < N; k++) {
                const int64_t x = h_masks[(size_t)i * N + k];
                const uint64_t q = qs[l];
                m[((size_t)i * 3 + l) * N + k] = x >= 0 ? (uint64_t)x % q : q - 1 - (uint64_t)(-(x + 1)) % q;
            }
    const uint64_t sm[3] = {C->q2inv[0].x, C->q2inv[1].x, 1};
    const int l2[3] = {0, 1, 3};
    return upload_key_polys(C, m.data(), 3 * (int64_t)prm->p, 3, l2, out, sm);
}

int bm_xk_to_device(const bm_params *prm, const bm_pk *pk, const bm_xk *xk, const int64_t *h_masks,
                    const int64_t *h_emasks, bm_xk_dev **out)
{
    if (!prm || !pk || !xk || !h_masks || !out) return BM_ERR_INVALID_ARG;
    if (memcmp(pk->digest, prm->digest, 32) || memcmp(xk->digest, prm->digest, 32) || xk->d != prm->d ||
        xk->p != prm->p)
        return BM_ERR_KEY_MISMATCH;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    bm_xk_dev *d = new bm_xk_dev;
    d->dev = C->dev;
    memcpy(d->digest, prm->digest, 32);
    d->d = prm->d;
    d->p = prm->p;
    d->s = prm->s;
    d->n_rot = xk->n_rot;
    d->pk2 = d->gk1 = d->mask = d->emask = nullptr;
    // level-2 pk: pk's limbs q0, q1 and xk's q2 limb
    std::vector<uint64_t> h(6 * (size_t)N);
    for (int c = 0; c < 2; c++) {
        memcpy(&h[(size_t)(c * 3 + 0) * N], &pk->v[(size_t)(c * 2 + 0) * N], 8 * (size_t)N);
        memcpy(&h[(size_t)(c * 3 + 1) * N], &pk->v[(size_t)(c * 2 + 1) * N], 8 * (size_t)N);
        memcpy(&h[(size_t)(c * 3 + 2) * N], &xk->pk_q2[(size_t)c * N], 8 * (size_t)N);
    }
    const int l2[3] = {0, 1, 3}, lk[3] = {0, 1, 2};
    rc = upload_key_polys(C, h.data(), 6, 3, l2, &d->pk2);
    // Galois keys: P^-1 folded into the Q limbs (the ModDown multiplies by it anyway)
    const uint64_t sk[3] = {C->pinv[0].x, C->pinv[1].x, 1};
    if (!rc && xk->n_rot > 0) rc = upload_key_polys(C, xk->gk1.data(), 12 * (int64_t)xk->n_rot, 3, lk, &d->gk1, sk);
    if (!rc) rc = upload_masks(C, prm, h_masks, &d->mask);
    if (!rc && h_emasks) rc = upload_masks(C, prm, h_emasks, &d->emask);
    if (rc) {
        cudaFree(d->pk2);
        cudaFree(d->gk1);
        cudaFree(d->mask);
        cudaFree(d->emask);
        cudaGetLastError();
        delete d;
        return rc;
    }
    *out = d;
    return BM_OK;
}

void bm_xk_dev_free(bm_xk_dev *d)
{
    if (!d) return;
    cudaFree(d->pk2);
    cudaFree(d->gk1);
    cudaFree(d->mask);
    cudaFree(d->emask);
    delete d;
}

int bm_encrypt_l2(const bm_params *prm, const bm_xk_dev *xk, const int64_t *d_pt, int64_t n_cts, uint64_t first_obj,
                  uint64_t seed, uint64_t *d_out, void *stream)
{
    if (!prm || !xk || n_cts < 0 || (n_cts > 0 && (!d_pt || !d_out))) return BM_ERR_INVALID_ARG;
    if (memcmp(xk->digest, prm->digest, 32)) return BM_ERR_KEY_MISMATCH;
    if (n_cts == 0) return BM_OK;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    EncK Ek;
    for (int i = 0; i < 4; i++) Ek.pr[i] = C->pr[i];
    Ek.pk = xk->pk2;
    Ek.pt = d_pt;
    Ek.out = d_out;
    Ek.first_obj = first_obj;
    Ek.seed = seed;
    Ek.n_limbs = 3;
    Ek.lp[0] = 0;
    Ek.lp[1] = 1;
    Ek.lp[2] = 3;
    k_encrypt<<<(unsigned)(3 * n_cts), T, SMEM_BYTES, (cudaStream_t)stream>>>(Ek);
    return launch_check();
}

static int64_t expand_chunk_cts(const bm_params *prm, int32_t nq)
{
    int64_t ch = 2048; // (query, part) outputs per launch: 6 N u64 of workspace each (768 MiB)
    if (const char *e = getenv("BM_EXPAND_CHUNK")) {
        long v = atol(e);
        if (v > 0) ch = v;
    }
    ch = ch / prm->p * prm->p; // whole queries
    if (ch < prm->p) ch = prm->p;
    const int64_t total = (int64_t)nq * prm->p;
    return total < ch ? total : ch;
}

size_t bm_expand_ws_bytes(const bm_params *prm, int32_t nq)
{
    if (!prm || nq <= 0) return 0;
    return (size_t)expand_chunk_cts(prm, nq) * XU_POLYS * N * sizeof(uint64_t);
}

int bm_expand(const bm_params *prm, const bm_xk_dev *xk, const uint64_t *d_in, int32_t nq, uint64_t *d_out, void *d_ws,
              size_t ws_bytes, void *stream)
{
    if (!prm || !xk || nq < 0) return BM_ERR_INVALID_ARG;
    if (memcmp(xk->digest, prm->digest, 32) || xk->p != prm->p || xk->d != prm->d) return BM_ERR_KEY_MISMATCH;
    int log_p = 0;
    while ((1 << log_p) < prm->p) log_p++;
    if (xk->n_rot < log_p) return BM_ERR_MISSING_ROTATION_KEY;
    if (nq == 0) return BM_OK;
    if (!d_in || !d_out || !d_ws) return BM_ERR_INVALID_ARG;
    if (ws_bytes < bm_expand_ws_bytes(prm, nq)) return BM_ERR_WORKSPACE;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    ExpK K;
    for (int i = 0; i < 4; i++) K.pr[i] = C->pr[i];
    K.pinv[0] = C->pinv[0];
    K.pinv[1] = C->pinv[1];
    K.q2inv[0] = C->q2inv[0];
    K.q2inv[1] = C->q2inv[1];
    K.mask = xk->mask;
    K.XU = (uint64_t *)d_ws;
    K.p = prm->p;
    K.enroll = 0;
    K.Bk = prm->B;
    K.bit = 0;
    K.u0 = 0;
    const int64_t ch = expand_chunk_cts(prm, nq), qch = ch / prm->p;
    for (int64_t j0 = 0; j0 < nq && !rc; j0 += qch) {
        const int64_t nqc = nq - j0 < qch ? nq - j0 : qch;
        const unsigned ncb = (unsigned)(2 * nqc * prm->p);
        K.in = d_in + (size_t)j0 * 6 * N;
        K.out = d_out + (size_t)j0 * prm->p * 4 * N;
        K.gk = nullptr;
        K.g = 1;
        k_exp_mask<<<ncb, T, X1_SMEM_BYTES, s>>>(K);
        rc = launch_check();
        for (int t = 0; t < log_p && !rc; t++) {
            K.gk = xk->gk1 + (size_t)t * 12 * N;
            K.g = (uint32_t)powmod_d(5, (uint64_t)prm->s << t, 2 * N);
            k_rot1_digits<<<ncb, T, X2_SMEM_BYTES, s>>>(K);
            k_rot1_ks<<<ncb, T, X3_SMEM_BYTES, s>>>(K);
            rc = launch_check();
        }
    }
    return rc;
}

// ------------------------------------------------------------------ f4: server-side enrollment
static int64_t enroll_chunk_templates(const bm_params *prm, int64_t n)
{
    int64_t ch = 2048; // parts per launch: 10 N u64 of workspace each (W + XU, 1.25 GiB)
    if (const char *e = getenv("BM_EXPAND_CHUNK")) {
        long v = atol(e);
        if (v > 0) ch = v;
    }
    int64_t t = ch / prm->p;
    if (t < 1) t = 1;
    return n < t ? n : t;
}

size_t bm_enroll_ws_bytes(const bm_params *prm, int64_t n)
{
    if (!prm || n <= 0) return 0;
    return (size_t)enroll_chunk_templates(prm, n) * prm->p * (4 + XU_POLYS) * N * sizeof(uint64_t);
}

int bm_enroll(const bm_params *prm, const bm_xk_dev *xk, const uint64_t *d_in, int64_t n, int64_t first_template,
              uint64_t *d_db, int64_t n_sets, void *d_ws, size_t ws_bytes, void *stream)
{
    if (!prm || !xk || n < 0 || first_template < 0 || n_sets < 0) return BM_ERR_INVALID_ARG;
    if (memcmp(xk->digest, prm->digest, 32) || xk->p != prm->p || xk->d != prm->d) return BM_ERR_KEY_MISMATCH;
    int log_b = 0;
    while ((1 << log_b) < prm->B) log_b++;
    if (xk->n_rot < log_b) return BM_ERR_MISSING_ROTATION_KEY;
    if (!xk->emask) return BM_ERR_INVALID_ARG;
    if (n == 0) return BM_OK;
    if ((first_template + n + prm->B - 1) / prm->B > n_sets) return BM_ERR_CAPACITY;
    if (!d_in || !d_db || !d_ws) return BM_ERR_INVALID_ARG;
    if (ws_bytes < bm_enroll_ws_bytes(prm, n)) return BM_ERR_WORKSPACE;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t tch = enroll_chunk_templates(prm, n);
    uint64_t *W = (uint64_t *)d_ws;
    ExpK K;
    for (int i = 0; i < 4; i++) K.pr[i] = C->pr[i];
    K.pinv[0] = C->pinv[0];
    K.pinv[1] = C->pinv[1];
    K.q2inv[0] = C->q2inv[0];
    K.q2inv[1] = C->q2inv[1];
    K.mask = xk->emask;
    K.XU = W + (size_t)tch * prm->p * 4 * N;
    K.p = prm->p;
    K.out = W;
    K.Bk = prm->B;
    for (int64_t c0 = 0; c0 < n && !rc; c0 += tch) {
        const int64_t nc = n - c0 < tch ? n - c0 : tch;
        const unsigned ncb = (unsigned)(2 * nc * prm->p);
        K.in = d_in + (size_t)c0 * 6 * N;
        K.u0 = first_template + c0;
        K.enroll = 0;
        K.g = 1;
        K.gk = nullptr;
        K.bit = 0;
        k_exp_mask<<<ncb, T, X1_SMEM_BYTES, s>>>(K); // Res(Mul(P)(C_u, E_i)) for every part
        rc = launch_check();
        K.enroll = 1;
        for (int b = 0; b < log_b && !rc; b++) {     // right rotation by (k - i) s = left by m s, bit by bit
            K.bit = b;
            K.gk = xk->gk1 + (size_t)b * 12 * N;
            K.g = (uint32_t)powmod_d(5, (uint64_t)prm->s << b, 2 * N);
            k_rot1_digits<<<ncb, T, X2_SMEM_BYTES, s>>>(K);
            k_rot1_ks<<<ncb, T, X3_SMEM_BYTES, s>>>(K);
            rc = launch_check();
        }
        if (rc) break;
        const int64_t t0 = K.u0 / prm->B, t1 = (K.u0 + nc - 1) / prm->B;
        k_enroll_add<<<(unsigned)((t1 - t0 + 1) * prm->p * 4 * (N / 256)), 256, 0, s>>>(W, K.u0, nc, prm->p, prm->B, t0,
                                                                                         d_db);
        rc = launch_check();
    }
    return rc;
}

// ------------------------------------------------------------------ f1: compressed scan
int bm_ck_to_device(const bm_params *prm, const bm_ck *ck, const int64_t *h_mask, bm_ck_dev **out)
{
    if (!prm || !ck || !h_mask || !out) return BM_ERR_INVALID_ARG;
    if (memcmp(ck->digest, prm->digest, 32) || ck->d != prm->d || ck->p != prm->p) return BM_ERR_KEY_MISMATCH;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    bm_ck_dev *d = new bm_ck_dev;
    d->dev = C->dev;
    memcpy(d->digest, prm->digest, 32);
    d->d = prm->d;
    d->p = prm->p;
    d->s = prm->s;
    d->log_s = ck->log_s;
    d->rlk2 = d->gkl = d->gkc = d->mask = nullptr;
    const int l4[4] = {0, 1, 3, 2}, l3[3] = {0, 1, 2}, l0[2] = {0, 2}, lm[2] = {0, 1};
    const uint64_t s4[4] = {C->pinv[0].x, C->pinv[1].x, C->pinv2.x, 1}, s3[3] = {C->pinv[0].x, C->pinv[1].x, 1};
    const uint64_t s0[2] = {C->pinv[0].x, 1}, sm[2] = {C->q1inv.x, 1};
    rc = upload_key_polys(C, ck->rlk2.data(), 24, 4, l4, &d->rlk2, s4);
    if (!rc && ck->log_s > 0) rc = upload_key_polys(C, ck->gkl.data(), 12 * (int64_t)ck->log_s, 3, l3, &d->gkl, s3);
    if (!rc && prm->s > 1) rc = upload_key_polys(C, ck->gkc.data(), 4 * (int64_t)(prm->s - 1), 2, l0, &d->gkc, s0);
    if (!rc) {
        std::vector<uint64_t> m(2 * (size_t)N);
        for (int l = 0; l < 2; l++) {
            const uint64_t q = l ? Q1 : Q0;
            for (int k = 0; k < N; k++) {
                const int64_t x = h_mask[k];
                m[(size_t)l * N + k] = x >= 0 ? (uint64_t)x % q : q - 1 - (uint64_t)(-(x + 1)) % q;
            }
        }
        rc = upload_key_polys(C, m.data(), 2, 2, lm, &d->mask, sm);
    }
    if (rc) {
        cudaFree(d->rlk2);
        cudaFree(d->gkl);
        cudaFree(d->gkc);
        cudaFree(d->mask);
        cudaGetLastError();
        delete d;
        return rc;
    }
    *out = d;
    return BM_OK;
}

void bm_ck_dev_free(bm_ck_dev *d)
{
    if (!d) return;
    cudaFree(d->rlk2);
    cudaFree(d->gkl);
    cudaFree(d->gkc);
    cudaFree(d->mask);
    delete d;
}

// workspace per pair (u64 polynomials): D01 6, D2 3, XU 9, XC 4, XR 2, XO 2, scratch 2
constexpr int CMP_WS_POLYS = 28;
static int64_t cmp_chunk_pairs(int64_t total)
{
    int64_t ch = 4096;
    if (const char *e = getenv("BM_CHUNK_PAIRS")) {
        long v = atol(e);
        if (v > 0) ch = v;
    }
    return total < ch ? total : ch;
}

size_t bm_match_cmp_ws_bytes(const bm_params *prm, int64_t n_sets, int32_t nq)
{
    if (!prm || n_sets <= 0 || nq <= 0) return 0;
    return (size_t)cmp_chunk_pairs(n_sets * (int64_t)nq) * CMP_WS_POLYS * N * sizeof(uint64_t);
}

int bm_match_cmp(const bm_params *prm, const bm_ck_dev *ck, const uint64_t *d_db, int64_t n_sets, const uint64_t *d_q,
                 int32_t nq, uint64_t *d_out, void *d_ws, size_t ws_bytes, void *stream)
{
    if (!prm || !ck || n_sets < 0 || nq < 0) return BM_ERR_INVALID_ARG;
    if (memcmp(ck->digest, prm->digest, 32) || ck->p != prm->p || ck->d != prm->d) return BM_ERR_KEY_MISMATCH;
    if (ck->log_s < prm->log_s) return BM_ERR_MISSING_ROTATION_KEY;
    const int64_t total = n_sets * (int64_t)nq;
    if (total == 0) return BM_OK;
    if (!d_db || !d_q || !d_out || !d_ws) return BM_ERR_INVALID_ARG;
    if (ws_bytes < bm_match_cmp_ws_bytes(prm, n_sets, nq)) return BM_ERR_WORKSPACE;
    DevCtx *Cx;
    int rc = ctx_get(&Cx);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t ch = cmp_chunk_pairs(total), n_groups = (n_sets + prm->s - 1) / prm->s;
    CmpK C;
    MatchK &K = C.m;
    for (int i = 0; i < 4; i++) K.pr[i] = Cx->pr[i];
    K.pinv[0] = Cx->pinv[0];
    K.pinv[1] = Cx->pinv[1];
    K.q1inv = Cx->q1inv;
    K.db = d_db;
    K.qry = d_q;
    K.out = nullptr;
    K.n_sets = n_sets;
    K.p = prm->p;

    uint64_t *ws = (uint64_t *)d_ws;
    const size_t P1 = (size_t)ch * N;
    K.D01 = ws;
    K.D2 = K.D01 + 6 * P1;
    K.XU = K.D2 + 3 * P1;
    K.XC = K.XU + 9 * P1;
    K.XR = K.XC + 4 * P1;
    K.XO = K.XR + 2 * P1;
    K.ACC = nullptr;
    C.scr = K.XO + 2 * P1;
    C.pinv2 = Cx->pinv2;
    C.q2inv[0] = Cx->q2inv[0];
    C.q2inv[1] = Cx->q2inv[1];
    C.rlk2 = ck->rlk2;
    C.gkc = ck->gkc;
    C.mask = ck->mask;
    C.s = prm->s;
    ExpK X; // the level-1 ladder reuses f3's rotation kernels (C <- C + Rot(C, 2^i))
    for (int i = 0; i < 4; i++) X.pr[i] = Cx->pr[i];
    X.pinv[0] = Cx->pinv[0];
    X.pinv[1] = Cx->pinv[1];
    X.q2inv[0] = Cx->q2inv[0];
    X.q2inv[1] = Cx->q2inv[1];
    X.mask = nullptr;
    X.in = nullptr;
    X.out = K.XC;
    X.XU = K.XU;
    X.p = 1;
    X.enroll = 0;
    X.Bk = 1;
    X.bit = 0;
    X.u0 = 0;
    cudaMemsetAsync(d_out, 0, (size_t)nq * n_groups * 2 * N * sizeof(uint64_t), s);
    const int64_t ct_full = n_sets < ch ? n_sets : ch;
    const int64_t cq_full = ch / ct_full < nq ? ch / ct_full : nq;
    for (int64_t jq0 = 0; jq0 < nq && !rc; jq0 += cq_full)
        for (int64_t t0 = 0; t0 < n_sets && !rc; t0 += ct_full) {
            K.jq0 = jq0;
            K.t0 = t0;
            K.cq = (int32_t)(nq - jq0 < cq_full ? nq - jq0 : cq_full);
            K.ct = n_sets - t0 < ct_full ? n_sets - t0 : ct_full;
            const int64_t np = K.cq * K.ct;
            const unsigned npu = (unsigned)np;
            const unsigned ntiles = (unsigned)(((K.cq + TQB - 1) / TQB) * ((K.ct + TSB - 1) / TSB) * (N / CS / TSL));
            k_tensor<3><<<3 * ntiles, TT, TENSOR_SMEM_BYTES, s>>>(K, 0, prm->p);
            k_digits3<<<3 * npu, T, C1_SMEM_BYTES, s>>>(C);
            k_relin3<<<2 * npu, T, C2_SMEM_BYTES, s>>>(C);
            rc = launch_check();
            for (int i = 0; i < prm->log_s && !rc; i++) {
                X.gk = ck->gkl + (size_t)i * 12 * N;
                X.g = (uint32_t)powmod_d(5, (uint64_t)1 << i, 2 * N);
                k_rot1_digits<<<2 * npu, T, X2_SMEM_BYTES, s>>>(X);
                k_rot1_ks<<<2 * npu, T, X3_SMEM_BYTES, s>>>(X);
                rc = launch_check();
            }
            if (rc) break;
            k_cmp_mask<<<2 * npu, T, SMEM_BYTES, s>>>(C);
            k_cmp_rot<<<npu, T, C4_SMEM_BYTES, s>>>(C);
            const int64_t g0 = t0 / prm->s, g1 = (t0 + K.ct - 1) / prm->s, ng = g1 - g0 + 1;
            k_cmp_add<<<(unsigned)(K.cq * ng * 2 * (N / 256)), 256, 0, s>>>(C, d_out, n_groups, g0, ng);
            rc = launch_check();
        }
    return rc;
}

// ------------------------------------------------------------------ the scan
static int64_t chunk_pairs(int64_t total)
{
    int64_t ch = 16384; // large chunks: fewer launches and kernel tails (workspace 768 KiB per pair)
    if (const char *e = getenv("BM_CHUNK_PAIRS")) {
        long v = atol(e);
        if (v > 0) ch = v;
    }
    return total < ch ? total : ch;
}

size_t bm_match_ws_bytes(const bm_params *prm, int64_t n_sets, int32_t nq, int32_t order)
{
    if (!prm || n_sets <= 0 || nq <= 0) return 0;
    const int polys = order == BM_ORDER_PAPER ? WS_POLYS_PAPER : WS_POLYS;
    return (size_t)chunk_pairs(n_sets * (int64_t)nq) * polys * N * sizeof(uint64_t);
}

void bm_set_profiling(int32_t on)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.on = on != 0;
}
void bm_profile_reset(void)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    bool on = g_prof.on;
    g_prof = Prof();
    g_prof.on = on;
}
int bm_profile_read(double *ms, int64_t *launches, int64_t *units)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (int i = 0; i < 7; i++) {
        if (ms) ms[i] = g_prof.ms[i];
        if (launches) launches[i] = g_prof.launches[i];
        if (units) units[i] = g_prof.units[i];
    }
    return BM_OK;
}

int bm_match(const bm_params *prm, const bm_evk_dev *evk, const uint64_t *d_db, int64_t n_sets, const uint64_t *d_q,
             int32_t nq, uint64_t *d_out, void *d_ws, size_t ws_bytes, int32_t order, void *stream)
{
    if (!prm || !evk || n_sets < 0 || nq < 0 ||
        (order != BM_ORDER_HOISTED && order != BM_ORDER_PAPER && order != BM_ORDER_HOISTED_ROT))
        return BM_ERR_INVALID_ARG;
    if (memcmp(evk->digest, prm->digest, 32)) return BM_ERR_KEY_MISMATCH;
    if (order != BM_ORDER_HOISTED_ROT && evk->n_rot < prm->log_s) return BM_ERR_MISSING_ROTATION_KEY;
    if (order == BM_ORDER_HOISTED_ROT && evk->n_hrot < prm->s - 1) return BM_ERR_MISSING_ROTATION_KEY;
    const int64_t total = n_sets * (int64_t)nq;
    if (total == 0) return BM_OK;
    if (!d_db || !d_q || !d_out || !d_ws) return BM_ERR_INVALID_ARG;
    if (ws_bytes < bm_match_ws_bytes(prm, n_sets, nq, order)) return BM_ERR_WORKSPACE;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t ch = chunk_pairs(total);

    MatchK K;
    for (int i = 0; i < 4; i++) K.pr[i] = C->pr[i];
    K.pinv[0] = C->pinv[0];
    K.pinv[1] = C->pinv[1];
    K.q1inv = C->q1inv;
    K.pmod[0] = C->pmod[0];
    K.pmod[1] = C->pmod[1];
    K.rlk = reinterpret_cast<const uint64_t *>(evk->rlk);
    K.gk = reinterpret_cast<const uint64_t *>(evk->gk);
    K.db = d_db;
    K.qry = d_q;
    K.out = d_out;
    K.n_sets = n_sets;
    K.p = prm->p;
    uint64_t *ws = (uint64_t *)d_ws;
    const size_t P1 = (size_t)ch * N;
    K.D01 = ws;
    K.D2 = K.D01 + 4 * P1;
    K.XC = K.D2 + 2 * P1;
    K.XU = K.XC + 2 * P1;
    K.ACC = order == BM_ORDER_PAPER ? K.XU + 4 * P1 : nullptr;
    const CtBuf bufC = order == BM_ORDER_PAPER ? CtBuf{K.ACC, 2 * N} : CtBuf{K.XC, 2 * N};

    bool prof;
    {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        prof = g_prof.on;
    }
    std::vector<Rec> recs;
    auto beg = [&](int cls, int64_t units) {
        if (!prof) return;
        Rec r;
        r.cls = cls;
        r.units = units;
        cudaEventCreate(&r.a);
        cudaEventCreate(&r.b);
        cudaEventRecord(r.a, s);
        recs.push_back(r);
    };
    auto end = [&]() {
        if (prof) cudaEventRecord(recs.back().b, s);
    };

    const int log_s = prm->log_s;
    // chunks are rectangles of cq queries x ct sets (cq * ct <= ch pairs)
    const int64_t ct_full = n_sets < ch ? n_sets : ch;
    const int64_t cq_full = ch / ct_full < nq ? ch / ct_full : nq;
    for (int64_t jq0 = 0; jq0 < nq && !rc; jq0 += cq_full)
    for (int64_t t0 = 0; t0 < n_sets && !rc; t0 += ct_full) {
        K.jq0 = jq0;
        K.t0 = t0;
        K.cq = (int32_t)(nq - jq0 < cq_full ? nq - jq0 : cq_full);
        K.ct = n_sets - t0 < ct_full ? n_sets - t0 : ct_full;
        const int64_t np = K.cq * K.ct;
        const unsigned npu = (unsigned)np;
        const unsigned ntiles = (unsigned)(((K.cq + TQB - 1) / TQB) * ((K.ct + TSB - 1) / TSB) * (N / CS / TSL));
        const bool per_part = order == BM_ORDER_PAPER;
        const int n_rounds = per_part ? prm->p : 1;
        for (int r = 0; r < n_rounds && !rc; r++) {
            const int lo = per_part ? r : 0, hi = per_part ? r + 1 : prm->p;
            beg(0, 2 * np);
            k_tensor<2><<<2 * ntiles, TT, TENSOR_SMEM_BYTES, s>>>(K, lo, hi);
            end();
            beg(1, 6 * np);
            k_digits<<<2 * npu, T, K2_SMEM_BYTES, s>>>(K);
            end();
            beg(2, 6 * np);
            k_relin<<<2 * npu, T, K3_SMEM_BYTES, s>>>(K, bufC, r > 0 ? 1 : 0);
            end();
            rc = launch_check();
        }
        if (log_s > 0 && !rc && order == BM_ORDER_HOISTED_ROT) {
            beg(5, 6 * np);
            k_hrot<<<npu, T, HROT_SMEM_BYTES, s>>>(K, bufC, evk->hgk, prm->s);
            end();
            rc = launch_check();
        } else if (log_s > 0 && !rc) {
            beg(4, 6 * log_s * np);
            k_ladder<<<npu, T, LADDER_SMEM_BYTES, s>>>(K, bufC, log_s);
            end();
            rc = launch_check();
        }
        if (log_s == 0 && !rc) {
            beg(6, 2 * np);
            k_out_intt<<<2 * npu, T, SMEM_BYTES, s>>>(K, bufC);
            end();
            rc = launch_check();
        }
    }
    if (prof) {
        if (cudaStreamSynchronize(s) != cudaSuccess) rc = BM_ERR_CUDA;
        std::lock_guard<std::mutex> lk(g_prof_mu);
        for (Rec &r : recs) {
            float ms = 0;
            cudaEventElapsedTime(&ms, r.a, r.b);
            g_prof.ms[r.cls] += ms;
            g_prof.launches[r.cls] += 1;
            g_prof.units[r.cls] += r.units;
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
    }
    return rc;
}

// End-to-end scan from host buffers: the queries are processed in G groups.  Group g's query
// upload (copy stream), scan (one of two compute streams, alternating, so that one group's
// kernels fill the tails of the previous group's) and result download (second copy stream)
// overlap with the neighbouring groups through HOST_SLOTS device buffer slots and events.
constexpr int HOST_SLOTS = 4;
static int host_groups(int64_t n_sets, int32_t nq)
{
    // about 576 (query, set) pairs per group (a few waves of the ladder kernel), at least 4 groups
    int64_t g = (n_sets * (int64_t)nq + 575) / 576;
    g = g < 4 ? 4 : g;
    if (const char *e = getenv("BM_HOST_GROUPS")) g = atoi(e) > 0 ? atoi(e) : g;
    return (int)(nq < g ? nq : g);
}

size_t bm_match_host_ws_bytes(const bm_params *prm, int64_t n_sets, int32_t nq, int32_t order)
{
    if (!prm || n_sets <= 0 || nq <= 0) return 0;
    const int G = host_groups(n_sets, nq);
    const int64_t gq = (nq + G - 1) / G;
    const size_t qbytes = (size_t)gq * prm->p * 4 * N * 8, obytes = (size_t)gq * n_sets * 2 * N * 8;
    const size_t mws = (bm_match_ws_bytes(prm, n_sets, (int32_t)gq, order) + 255) & ~(size_t)255;
    return HOST_SLOTS * (qbytes + obytes) + 2 * mws;
}

int bm_match_host(const bm_params *prm, const bm_evk_dev *evk, const uint64_t *d_db, int64_t n_sets,
                  const uint64_t *h_q, int32_t nq, uint64_t *h_out, void *d_ws, size_t ws_bytes, int32_t order,
                  void *stream)
{
    if (!prm || n_sets < 0 || nq < 0) return BM_ERR_INVALID_ARG;
    if (n_sets == 0 || nq == 0) return BM_OK;
    if (!h_q || !h_out || !d_ws) return BM_ERR_INVALID_ARG;
    if (ws_bytes < bm_match_host_ws_bytes(prm, n_sets, nq, order)) return BM_ERR_WORKSPACE;
    const int G = host_groups(n_sets, nq);
    const int64_t gq = (nq + G - 1) / G;
    const size_t qrow = (size_t)prm->p * 4 * N, orow = (size_t)n_sets * 2 * N; // u64 per query
    uint64_t *dq[HOST_SLOTS], *dout[HOST_SLOTS];
    uint64_t *base = (uint64_t *)d_ws;
    for (int k = 0; k < HOST_SLOTS; k++) dq[k] = base + k * gq * qrow;
    base += HOST_SLOTS * gq * qrow;
    for (int k = 0; k < HOST_SLOTS; k++) dout[k] = base + k * gq * orow;
    base += HOST_SLOTS * gq * orow;
    const size_t mws = (bm_match_ws_bytes(prm, n_sets, (int32_t)gq, order) + 255) & ~(size_t)255;
    void *ws[2] = {base, (uint8_t *)base + mws};
    cudaStream_t sc[2], su, sd;
    sc[0] = (cudaStream_t)stream;
    if (cudaStreamCreateWithFlags(&sc[1], cudaStreamNonBlocking) != cudaSuccess) return BM_ERR_CUDA;
    cudaStreamCreateWithFlags(&su, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking);
    // half-size first and last groups: the pipeline's unoverlapped head (first upload) and tail
    // (last download) shrink; the middle groups are gq queries
    std::vector<int64_t> g0, gn;
    {
        const int64_t h = nq >= 4 ? (gq + 1) / 2 : nq;
        int64_t q = 0;
        g0.push_back(0), gn.push_back(h), q = h;
        const int64_t tail = nq - q > h ? h : 0;
        while (q < nq - tail) {
            const int64_t c = nq - tail - q < gq ? nq - tail - q : gq;
            g0.push_back(q), gn.push_back(c), q += c;
        }
        if (tail) g0.push_back(q), gn.push_back(tail);
    }
    const int ngroups = (int)g0.size();
    std::vector<cudaEvent_t> ev_up(ngroups), ev_done(ngroups), ev_down(ngroups);
    for (int g = 0; g < ngroups; g++) {
        cudaEventCreateWithFlags(&ev_up[g], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev_done[g], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev_down[g], cudaEventDisableTiming);
    }
    cudaEvent_t ev_start;
    cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming);
    cudaEventRecord(ev_start, sc[0]); // everything starts after the work already on the caller's stream
    cudaStreamWaitEvent(sc[1], ev_start, 0);
    cudaStreamWaitEvent(su, ev_start, 0);
    int rc = BM_OK;
    for (int g = 0; g < ngroups && !rc; g++) {
        const int slot = g % HOST_SLOTS;
        cudaStream_t cs = sc[g & 1];
        const int64_t q0 = g0[g], nqg = gn[g];
        // the query slot is free once the scan of group g - HOST_SLOTS has consumed it
        if (g >= HOST_SLOTS) cudaStreamWaitEvent(su, ev_done[g - HOST_SLOTS], 0);
        if (cudaMemcpyAsync(dq[slot], h_q + q0 * qrow, nqg * qrow * 8, cudaMemcpyHostToDevice, su) != cudaSuccess)
            rc = BM_ERR_CUDA;
        cudaEventRecord(ev_up[g], su);
        cudaStreamWaitEvent(cs, ev_up[g], 0);
        // the output slot is free once group g - HOST_SLOTS's results are downloaded
        if (g >= HOST_SLOTS) cudaStreamWaitEvent(cs, ev_down[g - HOST_SLOTS], 0);
        if (!rc)
            rc = bm_match(prm, evk, d_db, n_sets, dq[slot], (int32_t)nqg, dout[slot], ws[g & 1], mws, order, cs);
        cudaEventRecord(ev_done[g], cs);
        cudaStreamWaitEvent(sd, ev_done[g], 0);
        if (!rc && cudaMemcpyAsync(h_out + q0 * orow, dout[slot], nqg * orow * 8, cudaMemcpyDeviceToHost, sd) != cudaSuccess)
            rc = BM_ERR_CUDA;
        cudaEventRecord(ev_down[g], sd);
    }
    if (cudaStreamSynchronize(sd) != cudaSuccess || cudaStreamSynchronize(su) != cudaSuccess ||
        cudaStreamSynchronize(sc[1]) != cudaSuccess || cudaStreamSynchronize(sc[0]) != cudaSuccess)
        rc = rc ? rc : BM_ERR_CUDA;
    for (int g = 0; g < ngroups; g++) {
        cudaEventDestroy(ev_up[g]);
        cudaEventDestroy(ev_done[g]);
        cudaEventDestroy(ev_down[g]);
    }
    cudaEventDestroy(ev_start);
    cudaStreamDestroy(sc[1]);
    cudaStreamDestroy(su);
    cudaStreamDestroy(sd);
    return rc;
}

int bm_sync(void *stream)
{
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "blindmatch: %s\n", cudaGetErrorString(e));
        return BM_ERR_CUDA;
    }
    return BM_OK;
}

#define BM_STR2(x) #x
#define BM_STR(x) BM_STR2(x)
const char *bm_build_info(void) { return "libblindmatch sm_100a (nvcc " BM_STR(__CUDACC_VER_MAJOR__) "." BM_STR(__CUDACC_VER_MINOR__) ")"; }

} // extern "C"
