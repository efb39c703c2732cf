// k_match.cuh -- the bm_match kernels: K1 k_tensor, K2 k_digits, K3 k_relin, K4 k_ladder_t (with the
// TMEM scratch helpers), K5 k_out_intt, and f2's K6 k_hrot; the workspace layout MatchK / CtBuf.
// Included once, by device.cu (one translation unit: the kernels are launched from its host side).
#pragma once

// ================================================================== device constants
__constant__ uint64_t c_cdt[19];

// Component 0 split / P-scaled resident C of the throughput ladder (K3 and k_ladder_t<false, true>)
#ifdef BM_LADDER_NO_SPLIT_C0
constexpr bool LADDER_SPLIT_C0 = false;
#else
constexpr bool LADDER_SPLIT_C0 = true;
#endif
// The pairs K3 hands to the one-CTA throughput ladder (pi < split_lim) carry P C instead of C:
// every update of the ladder is linear mod q0, so with C' = P C
//   c'_c <- c'_c + [c = 0] sigma(c'_0) + sigma(c'_1) (P^-1 gk_r[c][q0]) - NTT_q0(y^c mod q0)
// (the same folded keys), the digit is INTT_q0 with N^-1 P^-1 folded into its last stage (pr0s; the
// exact integer x in [0, q0) as before), and the output leaves through the same constants -- the
// P^-1 y^c product of every step but the last disappears (K3 folds P into its q1^-1 constant).
#if defined(BM_LADDER_NO_PSCALE) || defined(BM_LADDER_NO_SPLIT_C0) || defined(BM_K3_NO_SPLIT)
constexpr bool LADDER_PSCALE = false;
#else
constexpr bool LADDER_PSCALE = true;
#endif

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
    // P-scaled throughput ladder (LADDER_PSCALE, below): q1^-1 P mod q0, and q0's constants with
    // N^-1 P^-1 in place of N^-1 (the inverse transform that leaves the scaled domain)
    ulonglong2 q1invP;
    PrimeK pr0s;
    uint64_t pmod[2];   // P mod q0, q1
    const uint64_t *rlk, *gk; // PLANAR Shoup keys: poly k at [2k N, 2k N + N) = w, [2k N + N, 2k N + 2N) = w'
    const uint64_t *db, *qry;
    uint64_t *out;
    int64_t n_sets;       // sets in the DB (output row length)
    int64_t jq0, t0, ct;  // chunk = queries [jq0, jq0+cq) x sets [t0, t0+ct); pair pi = a*ct + b
    int32_t cq;
    int32_t p;
    BM_D int64_t out_row(int64_t pi) const { return (jq0 + pi / ct) * n_sets + t0 + pi % ct; }
    // bm_match_rows: query j's results go to rows[j] (possibly a peer GPU's memory) at global set
    // set_off + t; otherwise to out [nq][n_sets][2][N]
    uint64_t *const *rows = nullptr;
    int64_t set_off = 0;
    int64_t pair0 = 0; // the ladder kernels' first pair (a launch may cover only the chunk's tail)
    int64_t nq_total = 0; // queries of the whole call (debug bounds checks)
    // pairs pi < split_lim leave K3 with component 0 split for the throughput ladder (coef_acc_update):
    // the NTT-domain part in the ciphertext buffer, the coefficient-domain part over D01[pi][0][q1]
    int64_t split_lim = 0;
    int64_t cap = 0; // pairs of the workspace (the chunk capacity): the D01 / D2 piece stride (dofs)
    BM_D uint64_t *out_at(int64_t pi, int c) const
    {
        BM_CHECK(pi >= 0 && pi < (int64_t)cq * ct && jq0 + pi / ct < nq_total && t0 + pi % ct < n_sets);
        if (rows) return rows[jq0 + pi / ct] + ((set_off + t0 + pi % ct) * 2 + c) * (int64_t)N;
        return out + (out_row(pi) * 2 + c) * (int64_t)N;
    }
    uint64_t *D01, *D2, *XC, *XU, *ACC;
    uint64_t *XR, *XO;  // f1: level-0 masked results (NTT), rotated results (coefficients)
};

// D01 (poly P = 2 c + l: d_c[q_l]) and D2 (P = l) of the level-1 scan: 16-coefficient pieces with the
// pairs interleaved -- piece stride cap * 16 u64, pair stride 16 u64 -- so the K1 epilogues' per-pair
// pieces of consecutive pairs are adjacent in HBM, while one pair's NTT-domain warp access (512 bytes,
// 64 coefficients) is still four whole 128-byte lines
#ifndef BM_DPIECE
#define BM_DPIECE 64
#endif
constexpr int DPIECE = BM_DPIECE; // coefficients per piece (16, 32, 64: A/B)
BM_D size_t dofs(const MatchK &K, int P, int64_t pi, int j)
{
    return ((size_t)(P * (N / DPIECE) + j / DPIECE) * (size_t)K.cap + (size_t)pi) * DPIECE + (j % DPIECE);
}

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

// an NTT-domain polynomial of the D01 / D2 piece layout into registers (M4, like load_eval)
BM_D void load_eval_d(uint64_t a[16], const uint64_t *base, const MatchK &K, int P, int64_t pi)
{
#pragma unroll
    for (int e = 0; e < 16; e += 2) {
        const int j = 1024 * (e >> 1) + 2 * (int)threadIdx.x; // pos_M4(tid, e)
        const ulonglong2 v = ld2(base + dofs(K, P, pi, j));
        a[e] = v.x;
        a[e + 1] = v.y;
    }
}

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

// u0 w0 + u1 w1 as a 128-bit value (the key-switch inner products: lazy [0, 2q) digits times canonical
// key residues, u < 2^61, w < 2^60).  BM_DOT_SPLIT (A/B variant): from 30-bit limbs,
// every partial product one IMAD.WIDE into a carry-free 64-bit sum (L < 2^61, M < 2^63, H < 2^62),
// then L + M 2^30 + H 2^60 -- fewer FMA-pipe slots, but K3 ran 3% slower than with the 128-bit form
BM_D u128 dot2(uint64_t u0, uint64_t w0, uint64_t u1, uint64_t w1)
{
#ifndef BM_DOT_SPLIT
    return (u128)u0 * w0 + (u128)u1 * w1; // the product default: the split form measured 3% slower in K3
#else
    constexpr uint32_t M30 = (1u << 30) - 1;
    const uint32_t a0 = (uint32_t)u0 & M30, b0 = (uint32_t)(u0 >> 30), c0 = (uint32_t)w0 & M30, d0 = (uint32_t)(w0 >> 30);
    const uint32_t a1 = (uint32_t)u1 & M30, b1 = (uint32_t)(u1 >> 30), c1 = (uint32_t)w1 & M30, d1 = (uint32_t)(w1 >> 30);
    const uint64_t L = (uint64_t)a0 * c0 + (uint64_t)a1 * c1;
    const uint64_t M = (uint64_t)a0 * d0 + (uint64_t)b0 * c0 + (uint64_t)a1 * d1 + (uint64_t)b1 * c1;
    const uint64_t H = (uint64_t)b0 * d0 + (uint64_t)b1 * d1;
    return (u128)L + ((u128)M << 30) + ((u128)H << 60);
#endif
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

// A/B variant (BM_TENSOR_ACC29; the tensor ran 7% SLOWER with it, so the product
// keeps the 128-bit multiply-accumulate): integer-limb accumulator with operands split into 29-bit limbs,
// x y = xl yl + (xl yh + xh yl) 2^29 + xh yh 2^58, every partial product ONE IMAD.WIDE into its own
// 64-bit sum -- no carry chains (a 128-bit multiply-accumulate costs ~13 instructions, a third of
// them IMAD.X carries on the FMA pipe).  Exact for up to 15 products of operands < 2^59 (the
// Karatsuba sums: xh < 2^30, so M grows by < 2^60 per product): the tile folds every PCH = 8 parts.
struct Acc29 {
    uint64_t L, M, H;
    BM_D void zero() { L = M = H = 0; }
    BM_D void set(uint64_t r) { L = r, M = 0, H = 0; }            // r < 2^60: L stays < 2^63
    BM_D void mac(uint32_t xl, uint32_t xh, uint32_t yl, uint32_t yh)
    {
        L += (uint64_t)xl * yl;
        M += (uint64_t)xl * yh;
        M += (uint64_t)xh * yl;
        H += (uint64_t)xh * yh;
    }
    BM_D u128 value() const { return (u128)L + ((u128)M << 29) + ((u128)H << 58); }
};
constexpr uint32_t M29 = (1u << 29) - 1;
// grid: ((qt * (N / CS) + slice) * nst + st) * 2 + l  (limbs alternate, so each SM holds one
// q0-limb CTA on the integer pipe and one q1-limb CTA on the FP64 pipe; set tiles next: the CTAs
// that share a query slice run together and the query data streams from HBM once)
// NL = limbs per ciphertext (2: level 1; 3: level 2, f1), L = limb index; L = 1 (q1) runs on the FP64
// pipe, L = 0 (q0) and L = 2 (q2, prime index 3) on the integer pipe
// stage the operands of one round (coefficient slice sl, parts i0 .. i0 + pc - 1) with cp.async
template <int L, int NL, bool SW> BM_D void tensor_stage(const MatchK &K, uint64_t *Qs, uint64_t *Ss, int qt, int sl, int st,
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
        // tile row tr: a query (or, swapped, a set) on the TQB side, a set (a query) on the TSB side
        const bool qside = (tr < TQB) != SW;
        int64_t a = tr < TQB ? (int64_t)qt * TQB + tr : (int64_t)st * TSB + (tr - TQB);
        if (qside) {
            a = a < K.cq ? a : K.cq - 1;
            src = K.qry + ((size_t)(K.jq0 + a) * K.p + i0 + part) * 2 * NL * N;
        } else {
            a = a < K.ct ? a : K.ct - 1;
            src = K.db + ((size_t)(K.t0 + a) * K.p + i0 + part) * 2 * NL * N;
        }
        dst = tr < TQB ? Qs + ((tr * PCH + part) * 2 + comp) * CS : Ss + (((tr - TQB) * PCH + part) * 2 + comp) * CS;
        cp_async16(dst + 2 * ch, src + (size_t)(NL * comp + L) * N + c0 + 2 * ch);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// NL = limbs per ciphertext (2: level 1; 3: level 2, f1), L = limb index; L = 1 (q1) runs on the FP64
// pipe, L = 0 (q0) and L = 2 (q2, prime index 3) on the integer pipe.  The CTA walks TSL consecutive
// coefficient slices; the rounds (slice, chunk of PCH parts) are double-buffered: round r + 1's
// operands are copied by cp.async while round r is computed.
template <int L, int NL, bool SW> BM_D void tensor_tile(const MatchK &K, uint64_t *stage, int qt, int sl0, int st, int part_lo,
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
    const int R = (SW ? 1 : TSL) * n_chunks; // the swapped (small-batch) tiles: one slice per CTA, more CTAs
    auto chunk_pc = [&](int j) { const int i0 = part_lo + j * PCH; return part_hi - i0 < PCH ? part_hi - i0 : PCH; };
    tensor_stage<L, NL, SW>(K, stage, stage + TQB * PCH * 2 * CS, qt, sl0, st, part_lo, chunk_pc(0));
#ifdef BM_TENSOR_ACC29
    Acc29 a0[2][2], a1[2][2], a2[2][2];    // q0, q2: split-limb integer sums (A/B variant)
#else
    u128 a0[2][2], a1[2][2], a2[2][2];     // q0, q2: 128-bit integer sums
#endif
    double f0[2][2], f1[2][2], f2[2][2];   // q1: exact FP64 sums of signed residues
#pragma unroll 1
    for (int r = 0; r < R; r++) {
        const int sl = sl0 + r / n_chunks, j = r % n_chunks, i0 = part_lo + j * PCH, pc = chunk_pc(j);
        if (r + 1 < R) {
            const int r1 = r + 1, j1 = r1 % n_chunks;
            uint64_t *b1 = stage + (size_t)(r1 & 1) * BUF;
            tensor_stage<L, NL, SW>(K, b1, b1 + TQB * PCH * 2 * CS, qt, sl0 + r1 / n_chunks, st, part_lo + j1 * PCH,
                                chunk_pc(j1));
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        BM_SYNCTHREADS();
        const uint64_t *Qs = stage + (size_t)(r & 1) * BUF, *Ss = Qs + TQB * PCH * 2 * CS;
        if (j == 0) {
#pragma unroll
            for (int u = 0; u < 2; u++)
#pragma unroll
                for (int v = 0; v < 2; v++) {
#ifdef BM_TENSOR_ACC29
                    if (INTL) a0[u][v].zero(), a1[u][v].zero(), a2[u][v].zero();
#else
                    if (INTL) a0[u][v] = a1[u][v] = a2[u][v] = 0;
#endif
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
#ifndef BM_TENSOR_ACC29
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
#else
            if (INTL) {
                uint32_t xl[3][2], xh[3][2], yl[3][2], yh[3][2]; // [x0, x1, x0 + x1] split at bit 29
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    const uint64_t xv[3] = {x0[u], x1[u], x0[u] + x1[u]}, yv[3] = {y0[u], y1[u], y0[u] + y1[u]};
#pragma unroll
                    for (int t = 0; t < 3; t++) {
                        xl[t][u] = (uint32_t)xv[t] & M29, xh[t][u] = (uint32_t)(xv[t] >> 29);
                        yl[t][u] = (uint32_t)yv[t] & M29, yh[t][u] = (uint32_t)(yv[t] >> 29);
                    }
                }
#pragma unroll
                for (int u = 0; u < 2; u++)
#pragma unroll
                    for (int v = 0; v < 2; v++) {
                        a0[u][v].mac(xl[0][u], xh[0][u], yl[0][v], yh[0][v]);
                        a2[u][v].mac(xl[1][u], xh[1][u], yl[1][v], yh[1][v]);
                        a1[u][v].mac(xl[2][u], xh[2][u], yl[2][v], yh[2][v]);
                    }
            } else {
#endif
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
        // folds: Acc29 every PCH = 8 parts (q0, q2: at most 15 products per sum) / 3 q1 per part below
        // 2^51 (q1): every 512 parts
#ifdef BM_TENSOR_ACC29
        constexpr bool FOLD8 = INTL;
#else
        constexpr bool FOLD8 = false;
#endif
        if ((FOLD8 || ((i0 + pc - part_lo) & 511) == 0) && i0 + pc < part_hi) {
#pragma unroll
            for (int u = 0; u < 2; u++)
#pragma unroll
                for (int v = 0; v < 2; v++) {
                    if (INTL) {
#ifdef BM_TENSOR_ACC29
                        a0[u][v].set(red128s<PI>(a0[u][v].value(), P.r64));
                        a1[u][v].set(red128s<PI>(a1[u][v].value(), P.r64));
                        a2[u][v].set(red128s<PI>(a2[u][v].value(), P.r64));
#else
                        a0[u][v] = red128s<PI>(a0[u][v], P.r64);
                        a1[u][v] = red128s<PI>(a1[u][v], P.r64);
                        a2[u][v] = red128s<PI>(a2[u][v], P.r64);
#endif
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
                    if (a >= (SW ? K.ct : K.cq) || bb >= (SW ? K.cq : K.ct)) continue;
                    const int64_t pi = SW ? bb * K.ct + a : a * K.ct + bb;
                    const int jj = sl * CS + c;
                    uint64_t d0, d2, kk;
                    if (INTL) {
#ifdef BM_TENSOR_ACC29
                        d0 = red128s<PI>(a0[u][v].value(), P.r64);
                        d2 = red128s<PI>(a2[u][v].value(), P.r64);
                        kk = red128s<PI>(a1[u][v].value(), P.r64);
#else
                        d0 = red128s<PI>(a0[u][v], P.r64);
                        d2 = red128s<PI>(a2[u][v], P.r64);
                        kk = red128s<PI>(a1[u][v], P.r64);
#endif
                    } else {
                        d0 = f64_mod_q1(f0[u][v]);
                        d2 = f64_mod_q1(f2[u][v]);
                        kk = f64_mod_q1(f1[u][v]);
                    }
                    const uint64_t d1 = submod_d(submod_d(kk, d0, q), d2, q);
                    if (NL == 2) { // the level-1 scan's piece layout (dofs)
                        K.D01[dofs(K, L, pi, jj)] = d0;
                        K.D01[dofs(K, 2 + L, pi, jj)] = d1;
                        K.D2[dofs(K, L, pi, jj)] = d2;
                    } else {
                        K.D01[((size_t)pi * 2 * NL + 0 + L) * N + jj] = d0;
                        K.D01[((size_t)pi * 2 * NL + NL + L) * N + jj] = d1;
                        K.D2[((size_t)pi * NL + L) * N + jj] = d2;
                    }
                }
        }
        BM_SYNCTHREADS(); // every read of buffer r & 1 is done before round r + 2 overwrites it
    }
}

template <int NL, bool SW> __global__ void __launch_bounds__(TT, 2) k_tensor(MatchK K, int part_lo, int part_hi)
{
    extern __shared__ uint64_t sm[];
    const int nst = (int)(((SW ? K.cq : K.ct) + TSB - 1) / TSB);
    int64_t b = blockIdx.x;
    const int l = (int)(b % NL);
    b /= NL;
    const int st = (int)(b % nst);
    b /= nst;
    constexpr int TS = SW ? 1 : TSL; // slices per CTA
    const int sg = (int)(b % (N / CS / TS));
    const int qt = (int)(b / (N / CS / TS));
    if (l == 0) tensor_tile<0, NL, SW>(K, sm, qt, sg * TS, st, part_lo, part_hi);
    else if (l == 1) tensor_tile<1, NL, SW>(K, sm, qt, sg * TS, st, part_lo, part_hi);
    else if (NL == 3) tensor_tile<2, NL, SW>(K, sm, qt, sg * TS, st, part_lo, part_hi);
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
    load_eval_d(a, K.D2, K, l, pi);
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
// L2 prefetch of a polynomial's 128-byte lines that this thread's later ld2 (pos_M4) reads: one lane in
// eight issues each line (16-byte vectors, eight lanes per line); the data move DRAM -> L2 while the
// CTA computes the current phase's transform
BM_D void prefetch_poly_l2(const uint64_t *p)
{
#ifdef BM_K3_PREFETCH
    if ((threadIdx.x & 7) == 0) {
#pragma unroll
        for (int e = 0; e < E; e += 2) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + pos_M4(threadIdx.x, e)));
    }
#endif
}
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
    // d2[q_l] = D2 poly l, d_c[q_l] = D01 poly 2 c + l (dofs)
    uint64_t a[E];
    // ---- P limb
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int j = pos_M4(tid, e);
        const ulonglong2 u = ld2(xu + 1 * N + j), v = ld2(xu + 3 * N + j);
        const ulonglong2 w0 = ld2(r0 + 2 * 2 * N + j), w1 = ld2(r1 + 2 * 2 * N + j);
        a[e] = red128s<2>(dot2(u.x, w0.x, v.x, w1.x), K.pr[2].r64);
        a[e + 1] = red128s<2>(dot2(u.y, w0.y, v.y, w1.y), K.pr[2].r64);
    }
    prefetch_poly_l2(xu + 0 * N); // the q1 phase's DRAM operands, during INTT_P
    inv<2>(a, sm, K.pr[2]);
#pragma unroll
    for (int e = 0; e < E; e++) ys[tid + T * e] = a[e]; // Y, canonical [0, P), coefficient j_M1(tid, e)
    // ---- q1 limb
    const ulonglong2 pinv1 = K.pinv[1];
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int j = pos_M4(tid, e);
        const ulonglong2 u = ld2(xu + 0 * N + j), v = ld2(K.D2 + dofs(K, 1, pi, j)), dd = ld2(K.D01 + dofs(K, 2 * c + 1, pi, j));
        const ulonglong2 w0 = ld2(r0 + 1 * 2 * N + j), w1 = ld2(r1 + 1 * 2 * N + j);
        const uint64_t ka = red128s<1>(dot2(u.x, w0.x, v.x, w1.x), K.pr[1].r64);
        const uint64_t kb = red128s<1>(dot2(u.y, w0.y, v.y, w1.y), K.pr[1].r64);
        a[e] = reduce_bnd<1>(dd.x + ka);
        a[e + 1] = reduce_bnd<1>(dd.y + kb);
    }
    prefetch_poly_l2(xu + 2 * N); // the q0 phase's DRAM operands, during INTT_q1 and NTT_q0
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
    // pairs of the throughput ladder leave P-scaled (LADDER_PSCALE): q1^-1 P in place of q1^-1
    const ulonglong2 q1inv = (LADDER_PSCALE && pi < K.split_lim) ? K.q1invP : K.q1inv;
    uint64_t *co = dst.at(pi, c);
    if (c == 0 && pi < K.split_lim) {
        // component 0 for the throughput ladder, split (k_ladder_t<false>, coef_acc_update): the NTT_q0 of
        // A is not needed -- C0 = q1^-1 (d0 + P^-1 KS0[q0]) (NTT domain) + q1^-1 (-A) (coefficient domain,
        // M1 order, lazily in [0, 2 q0)), the latter written over d_0[q1] (read only by this CTA, and
        // only before inv_f's barriers)
#pragma unroll
        for (int e = 0; e < E; e++) K.D01[dofs(K, 1, pi, j_M1(tid, e))] = reduce_lazy<0>(shoup4<0>(6 * Q0 - a[e], q1inv));
#pragma unroll
        for (int e = 0; e < E; e += 2) {
            const int j = pos_M4(tid, e);
            const ulonglong2 u = ld2(K.D2 + dofs(K, 0, pi, j)), v = ld2(xu + 2 * N + j), dd = ld2(K.D01 + dofs(K, 2 * c, pi, j));
            const ulonglong2 w0 = ld2(r0 + j), w1 = ld2(r1 + j);
            const uint64_t ka = red128s<0>(dot2(u.x, w0.x, v.x, w1.x), K.pr[0].r64);
            const uint64_t kb = red128s<0>(dot2(u.y, w0.y, v.y, w1.y), K.pr[0].r64);
            st2(co + j, reduce_bnd<0>(shoup4<0>(dd.x + ka, q1inv)), reduce_bnd<0>(shoup4<0>(dd.y + kb, q1inv)));
        }
        return;
    }
    fwd<0, false>(a, sm, K.pr[0]); // A, in [0, 2 q0)
    // ---- q0 limb and output
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int j = pos_M4(tid, e);
        const ulonglong2 u = ld2(K.D2 + dofs(K, 0, pi, j)), v = ld2(xu + 2 * N + j), dd = ld2(K.D01 + dofs(K, 2 * c, pi, j));
        const ulonglong2 w0 = ld2(r0 + j), w1 = ld2(r1 + j);
        const uint64_t ka = red128s<0>(dot2(u.x, w0.x, v.x, w1.x), K.pr[0].r64);
        const uint64_t kb = red128s<0>(dot2(u.y, w0.y, v.y, w1.y), K.pr[0].r64);
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
    BM_SYNCTHREADS();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    return *s_addr + ((uint32_t)(32 * (warp & 3)) << 16) + (COLS / 4) * (uint32_t)(warp >> 2);
}
template <uint32_t COLS> BM_D void tmem_free(uint32_t base) // all threads, after every TMEM access of the CTA
{
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    BM_SYNCTHREADS();
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
// the level-0 ciphertext C = (c0, c1) resident in shared memory (NTT domain, stored in natural
// order, ntt3.cuh nat_at: conflict-free automorphism gathers), so C never leaves the SM between
// steps.  Per step r = 2^i, g = 5^r mod 2N:
//   digit   x   = INTT_q0(sigma_g(c1)) in [0, q0), lifted to P as is (reading R4); XP = NTT_P(x)
//   comp c  y^c = centred_P(INTT_P(XP gk_r[c][P]))
//           c_c <- c_c + [c = 0] sigma_g(c0) + sigma_g(c1) (P^-1 gk_r[c][q0]) - NTT_q0(P^-1 y^c)
// (P^-1 is folded into the device Galois keys' q0 limb, and P^-1 y^c = P^-1 y - [y > P/2] needs
// no centring reduction)
// The last step leaves the NTT domain directly (INTT is linear, the rounding term y^c is already
// in coefficient form): out_c = INTT_q0(c_c + [c = 0] sigma(c0) + P^-1 sigma(c1) gk[c][q0])
// - P^-1 y^c, i.e. 6 transforms per step and none for the output conversion.  The throughput mode
// (k_ladder_t<false>) keeps c0 as two accumulators (coef_acc_update): 5 transforms per step, 6 in the
// last one.
constexpr size_t LADDER_SMEM_BYTES = 3 * SMEM_WORDS * sizeof(uint64_t);


// Latency mode (k_ladder_t<true>): when a launch has fewer pairs than half the SMs (a single query
// against a small DB: the paper's measurement shape), most SMs idle and the latency is one CTA's 6
// transforms per step.  Launched as 2-CTA clusters, the ladder runs one pair per cluster: rank c
// owns component c, both ranks compute the digit (INTT_q0 + NTT_P of sigma_g(c1); rank 0 copies c1
// from rank 1's shared memory over DSMEM first) and then ONLY their own component's INTT_P +
// NTT_q0 -- 4 transforms on the critical path per step instead of 6, identical residues.  Cluster
// barriers per step: (1) c1 of the previous step is complete before rank 0 copies it; (2) rank 0's
// copy is done before rank 1 overwrites c1 (split arrive / wait around the step's transforms).
BM_D uint32_t cluster_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
BM_D void cluster_arrive()
{
    bm_jitter();
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
BM_D void cluster_wait()
{
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    bm_jitter();
}
// generic address of the same shared-memory location in CTA `rank` of this cluster
BM_D const uint64_t *cluster_peer(const uint64_t *p, uint32_t rank)
{
    uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    uint64_t g;
    asm volatile("cvta.shared::cluster.u64 %0, %1;" : "=l"(g) : "l"((uint64_t)r));
    return reinterpret_cast<const uint64_t *>(g);
}

BM_D void tmem_ld8(uint32_t taddr, uint64_t v[8]) // 16 columns -> 8 u64 (waits)
{
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                 "%13, %14, %15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15])
                 : "r"(taddr)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15])
                 :
                 : "memory");
#pragma unroll
    for (int i = 0; i < 8; i++) v[i] = (uint64_t)r[2 * i] | ((uint64_t)r[2 * i + 1] << 32);
}

// Component 0's coefficient-domain accumulator of the throughput ladder (k_ladder_t<false>).  c0 never
// feeds the digit, and every operation on it is linear mod q0 and commutes with the NTT (sigma_g is a
// permutation of the evaluations and a signed permutation X^j -> +-X^(j g mod N) of the coefficients), so
//   c0_L = INTT_q0(S0) + A,  S0 <- S0 + sigma(S0) + sigma(c1) P^-1 gk0[q0]   (NTT domain, pointwise)
//                            A  <- A + sigma(A) - P^-1 y^0                  (coefficient domain)
// gives the same residues as c0 <- c0 + sigma(c0) + sigma(c1) P^-1 gk0[q0] - NTT_q0(P^-1 y^0) with
// one transform less per step (the NTT_q0 of P^-1 y^0; the output's INTT_q0 is needed anyway).
// A lives in TMEM (this thread's coefficients j_M1(tid, e), lazily in [0, 2 q0)); sigma(A) is a scatter
// through the exchange buffer.  py: P^-1 y^0 (< 5 q0) in M1 order; first: A = 0 before this step.
BM_D void coef_acc_update(const uint64_t py[E], uint64_t *XB, uint32_t tacc, uint32_t g, bool first)
{
    const int tid = threadIdx.x;
    uint64_t t[E];
    if (first) {
#pragma unroll
        for (int e = 0; e < E; e++) t[e] = reduce_lazy<0>(5 * Q0 - py[e]);
    } else {
        BM_SYNCTHREADS(); // the transform's last reads of XB are done
#pragma unroll
        for (int h = 0; h < 2; h++) {
            uint64_t v[8];
            tmem_ld8(tacc + 16 * h, v);
#pragma unroll
            for (int e = 0; e < 8; e++) {
                const uint32_t j = (uint32_t)j_M1(tid, 8 * h + e);
                const uint32_t u = (j * g) & (2 * N - 1); // X^j -> X^(j g mod 2N) = -X^(u - N) for u >= N
                BM_CHECK(pidx((int)(u & (N - 1))) < SMEM_WORDS);
                XB[pidx((int)(u & (N - 1)))] = (u & N) ? 2 * Q0 - v[e] : v[e]; // (0, 2 q0]
                t[8 * h + e] = v[e] + 5 * Q0 - py[8 * h + e];                  // < 7 q0
            }
        }
        BM_SYNCTHREADS();
#pragma unroll
        for (int e = 0; e < E; e++) t[e] = reduce_lazy<0>(t[e] + XB[pidx(j_M1(tid, e))]); // < 9 q0
    }
    tmem_st16(tacc, t);
}

// ACC (throughput mode only): every pair of the launch comes from K3 with component 0 split (pi < split_lim)
template <bool CL, bool ACC = false> __global__ void __launch_bounds__(T, 1) k_ladder_t(MatchK K, CtBuf cin, int L)
{
    extern __shared__ uint64_t sm[];
    uint64_t *XB = sm, *S0 = sm + SMEM_WORDS, *S1 = sm + 2 * SMEM_WORDS;
    const int tid = threadIdx.x;
    // CL (latency mode, launched as 2-CTA clusters): rank r runs only component r; rank 0 keeps c0 in
    // S0 and refreshes a copy of c1 in S1 from rank 1's S1 (DSMEM) every step
    const int rank = CL ? (int)cluster_rank() : 0;
    const int64_t pi = K.pair0 + (CL ? blockIdx.x >> 1 : blockIdx.x);
    __shared__ uint32_t s_tmem;
    const uint32_t tks1 = tmem_alloc<256>(&s_tmem), ttsc = tks1 + 32; // TMEM scratch (see tmem_alloc)
    // component 0's coefficient-domain accumulator (throughput mode); it shares ttsc's columns: ttsc is
    // written only by component 1 of the last step, after component 0 has read the accumulator
    const uint32_t tacc = ttsc;
    const ulonglong2 pinv = K.pinv[0];
    const int nt = nat_tid(tid); // S0, S1 in natural order (nat_at / nat_auto: conflict-free)
    if (!CL || rank == 0) stage_nat(S0, cin.at(pi, 0));
    if (!CL || rank == 1) stage_nat(S1, cin.at(pi, 1));
    const uint64_t *peer_c1 = CL && rank == 0 ? cluster_peer(S1, 1) : nullptr;
    uint64_t a[E];
    // component 0 split by K3 (coef_acc_update): its coefficient-domain part starts the accumulator
    static_assert(!(CL && ACC), "the cluster ladders take component 0 unsplit");
    constexpr bool have_acc = ACC;
    // PS: the resident C (and the accumulator) of these pairs is P C (LADDER_PSCALE, above): the
    // inverse q0 transforms divide by P as well, and y^c enters reduced mod q0 instead of as P^-1 y^c
    constexpr bool PS = ACC && LADDER_PSCALE;
    const PrimeK &pr0i = PS ? K.pr0s : K.pr[0];
    const uint64_t pneg = Q0 - K.pmod[0]; // -P mod q0
    BM_CHECK(!ACC || pi < K.split_lim);
    if (have_acc) {
#pragma unroll
        for (int e = 0; e < E; e++) a[e] = K.D01[dofs(K, 1, pi, j_M1(tid, e))];
        tmem_st16(tacc, a);
    }
    uint32_t g = 5; // 5^(2^i) mod 2N
#pragma unroll 1
    for (int i = 0; i < L; i++, g = (g * g) & (2 * N - 1)) {
        const bool last = i == L - 1;
        // [rot][c][q0|P] planar polys of 2N u64
        const uint64_t *gq0 = K.gk + (size_t)(i * 4 + 0) * 2 * N, *gp0 = gq0 + 2 * N;
        const uint64_t *gq1 = K.gk + (size_t)(i * 4 + 2) * 2 * N, *gp1 = gq1 + 2 * N;
        if (CL) {
            cluster_arrive(); // (1) both ranks' c_c of the previous step (or the staging) are complete
            cluster_wait();
            if (rank == 0) {
                const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(peer_c1);
                ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(S1);
                for (int k = tid; k < SMEM_WORDS / 2; k += T) dst[k] = src[k];
            }
            cluster_arrive(); // (2) arrive: rank 0's copy of c1 is done (waited for before c1 is rewritten)
        }
        BM_SYNCTHREADS(); // S0 / S1 of the previous step (or the initial staging) are complete
        // digit: sigma_g(c1) -> INTT_q0 -> NTT_P
#pragma unroll
        for (int e = 0; e < E; e++) a[e] = S1[nat_auto(nt, e, g)];
        inv<0>(a, XB, pr0i);
        fwd<2, false>(a, XB, K.pr[2]); // lazy [0, 2P): Shoup operand only
        // P-limb key-switch products for both components; component 1's waits in the workspace
        if (CL) { // this rank's component only
            const uint64_t *gp = rank ? gp1 : gp0;
#pragma unroll
            for (int e = 0; e < E; e += 2) {
                ulonglong2 w, wb;
                ldkey2(gp, pos_M4(tid, e), w, wb);
                a[e] = shoup4<2>(a[e], w);
                a[e + 1] = shoup4<2>(a[e + 1], wb);
            }
        } else {
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
        }
#pragma unroll 1
        for (int c = 0; c < 2; c++) {
            if (CL && c != rank) continue; // latency mode: this rank's component only
            if (!CL && c == 1) tmem_ld16(tks1, a); // component 1's P-limb product, parked in TMEM above
            inv<2>(a, XB, K.pr[2]);
            // P^-1 y^c mod q0 with y^c = y - [y > P/2] P:  P^-1 y - [y > P/2], < 5 q0
            // (PS: y^c mod q0 itself, lazily: (y mod q0) + [y > P/2] (-P mod q0) < 3 q0; only component
            // 1's last step, whose term leaves in coefficient form, takes the P^-1 product)
            if (PS && (c == 0 || !last)) {
#pragma unroll
                for (int e = 0; e < E; e++) a[e] = reduce_lazy<0>(a[e]) + (a[e] > (QP >> 1) ? pneg : 0);
            } else {
#pragma unroll
                for (int e = 0; e < E; e++) a[e] = shoup4<0>(a[e], pinv) + (a[e] > (QP >> 1) ? Q0 - 1 : 0);
            }
            uint64_t *S = c ? S1 : S0;
            const uint64_t *gq = c ? gq1 : gq0;
#ifndef BM_LADDER_NO_SPLIT_C0
            if (!CL && c == 0) {
                // component 0 in two accumulators (coef_acc_update): the coefficient-domain part takes
                // (1 + sigma_g) and - P^-1 y^0; the NTT-domain part S0 takes only the pointwise terms
                coef_acc_update(a, XB, tacc, g, i == 0 && !have_acc);
                ulonglong2 kk[2];
#pragma unroll
                for (int e = 0; e < E; e++) {
                    const int j = nat_at(nt, e), jp = nat_auto(nt, e, g);
                    if (!(e & 1)) ldkey2(gq, pos_M4(tid, e), kk[0], kk[1]);
                    const uint64_t ks = shoup4<0>(S1[jp], kk[e & 1]); // [0, 4 q0)
                    a[e] = reduce_lazy<0>(ks + S0[j] + S0[jp]);       // < 8 q0 -> [0, 2 q0)
                }
                if (!last) {
                    BM_SYNCTHREADS(); // every read of the old c0 is done
#pragma unroll
                    for (int e = 0; e < E; e++) S0[nat_at(nt, e)] = a[e];
                } else {
                    inv<0>(a, XB, pr0i); // canonical
                    uint64_t *o = K.out_at(pi, 0);
                    uint64_t t[E];
                    tmem_ld16(tacc, t); // [0, 2 q0)
                    if (PS) { // the accumulator is P A: its one P^-1 product
#pragma unroll
                        for (int e = 0; e < E; e++) t[e] = shoup4<0>(t[e], pinv); // [0, 4 q0)
                    }
#pragma unroll
                    for (int e = 0; e < E; e++) o[j_M1(tid, e)] = reduce_bnd<0>(a[e] + t[e]);
                }
                continue;
            }
#endif
            if (!last) {
                fwd<0, false>(a, XB, K.pr[0]); // NTT_q0(P^-1 y^c), lazy [0, 2 q0)
                ulonglong2 kk[2];
#pragma unroll
                for (int e = 0; e < E; e++) {
                    const int j = nat_at(nt, e), jp = nat_auto(nt, e, g);
                    if (!(e & 1)) ldkey2(gq, pos_M4(tid, e), kk[0], kk[1]);
                    // sigma(c1) P^-1 gk[c][q0] (P^-1 folded into the device key), [0, 4 q0)
                    const uint64_t ks = shoup4<0>(S1[jp], kk[e & 1]);
                    uint64_t v = ks + 2 * Q0 - a[e] + S[j]; // < 8 q0 (S in [0, 2 q0))
                    if (c == 0) v += S0[jp];           // < 10 q0
#ifdef BM_LADDER_CANON_S
                    a[e] = reduce_bnd<0>(v);
#else
                    a[e] = reduce_lazy<0>(v);          // [0, 2 q0): the resident C stays lazy (its readers:
                                                       // Shoup operands and inv<0>, which takes < 4 q0)
#endif
                }
                if (CL) cluster_wait(); // (2) wait: c1 may be rewritten now
                BM_SYNCTHREADS();        // every read of the old c_c is done
#pragma unroll
                for (int e = 0; e < E; e++) S[nat_at(nt, e)] = a[e];
            } else {
                tmem_st16(ttsc, a); // P^-1 y^c (coefficient j_M1(tid, e)), < 5 q0
                ulonglong2 kk[2];
#pragma unroll
                for (int e = 0; e < E; e++) {
                    const int j = nat_at(nt, e), jp = nat_auto(nt, e, g);
                    if (!(e & 1)) ldkey2(gq, pos_M4(tid, e), kk[0], kk[1]);
                    const uint64_t ks = shoup4<0>(S1[jp], kk[e & 1]);
                    uint64_t v = ks + S[j]; // < 6 q0
                    if (c == 0) v += S0[jp]; // < 8 q0
#ifdef BM_LADDER_CANON_S
                    a[e] = reduce_bnd<0>(v);
#else
                    a[e] = reduce_lazy<0>(v); // [0, 2 q0) < 4 q0: inv<0>'s input bound; its output is canonical
#endif
                }
                inv<0>(a, XB, pr0i);
                uint64_t *o = K.out_at(pi, c);
                uint64_t t[E];
                tmem_ld16(ttsc, t);
#pragma unroll
                for (int e = 0; e < E; e++) o[j_M1(tid, e)] = submod_d(a[e], reduce_bnd<0>(t[e]), Q0);
                if (CL) cluster_wait(); // (2) wait: rank 1 stays resident until rank 0's last copy is done
            }
        }
    }
    tmem_free<256>(s_tmem);
}

// ================================================================== latency mode, 3 ranks: the pipelined ladder
// For launches of at most n_SM / 3 pairs.  The c0 chain never feeds the c1 chain, and the c1 chain
// can run in two domains at once (exact by linearity mod q0):
//   c1coef_{i+1} = INTT_q0(c1_i + P^-1 sigma(c1_i) gk1[q0]) - P^-1 y^1_i,   digit_{i+1} = sigma_coef(c1coef_{i+1})
// so a 3-CTA cluster runs one pair with two transform levels per step on the critical path (k_ladder_t:
// 6 in one CTA, 4 on a pair):
//   rank A: digit_i (coefficient-domain automorphism gather) -> NTT_P -> products with gk0 / gk1[P];
//           INTT_P(XP gk1) -> t1 = P^-1 y^1 (to B)
//   rank B: c1_i = NTT_q0(c1coef_i); w = INTT_q0(c1_i + P^-1 sigma(c1_i) gk1[q0]); c1coef_{i+1} = w - t1
//           (to A's digit buffer; the last step's is output component 1)
//   rank C: one level behind: INTT_P(XP gk0) -> P^-1 y^0, NTT_q0, the c0 update of k_ladder_t (sigma(c1_i)
//           from a copy of B's c1_i); after the last step the output INTT of component 0.
// Residues are identical to k_ladder_t (test_latency_mode_cluster_ladder).  Three cluster barriers per
// step order the DSMEM traffic: XP gk0 (A -> C, read remotely), c1_i (B -> C copy), t1 (A -> B), c1coef (B -> A).
__global__ void __launch_bounds__(T, 1) k_ladder_c3(MatchK K, CtBuf cin, int L)
{
    extern __shared__ uint64_t sm[];
    uint64_t *XB = sm, *R1 = sm + SMEM_WORDS, *R2 = sm + 2 * SMEM_WORDS; // two role buffers of SMEM_WORDS
    const int tid = threadIdx.x;
    const int rank = (int)cluster_rank();
    const int64_t pi = K.pair0 + blockIdx.x / 3;
    const ulonglong2 pinv = K.pinv[0];
    const int nt = nat_tid(tid);
    __shared__ uint32_t s_tmem;
    const uint32_t ttsc = tmem_alloc<128>(&s_tmem); // C: the last step's P^-1 y^0
    auto csync = [] { cluster_arrive(); cluster_wait(); };
    // A: R1 = SD (c1coef, plain coefficient order), R2 = U0 (XP gk0[P], thread-private order)
    // B: R1 = S1 (c1_i, natural order), R2 = T1 (t1 from A, thread-private order)
    // C: R1 = S0 (c0, natural order), R2 = S1c (copy of B's S1)
    uint64_t a[E];
    if (rank == 0) load_eval(a, cin.at(pi, 1)), inv<0>(a, XB, K.pr[0]);
#pragma unroll
    for (int e = 0; e < E; e++)
        if (rank == 0) R1[j_M1(tid, e)] = a[e];
    if (rank == 1) stage_nat(R1, cin.at(pi, 1));
    if (rank == 2) stage_nat(R1, cin.at(pi, 0));
    uint64_t *peerU0 = rank == 2 ? const_cast<uint64_t *>(cluster_peer(R2, 0)) : nullptr; // A's U0
    uint64_t *peerS1 = rank == 2 ? const_cast<uint64_t *>(cluster_peer(R1, 1)) : nullptr; // B's S1
    uint64_t *peerT1 = rank == 0 ? const_cast<uint64_t *>(cluster_peer(R2, 1)) : nullptr; // B's T1
    uint64_t *peerSD = rank == 1 ? const_cast<uint64_t *>(cluster_peer(R1, 0)) : nullptr; // A's SD
    csync();
    uint32_t g = 5, gi = 3277, gprev = 5; // 5^(2^i), its inverse mod 2N (5 * 3277 = 16385), the previous g
#pragma unroll 1
    for (int i = 0; i < L; i++, g = (g * g) & (2 * N - 1), gi = (gi * gi) & (2 * N - 1)) {
        const bool last = i == L - 1;
        const uint64_t *gq0 = K.gk + (size_t)(i * 4 + 0) * 2 * N, *gp0 = gq0 + 2 * N;
        const uint64_t *gq1 = K.gk + (size_t)(i * 4 + 2) * 2 * N, *gp1 = gq1 + 2 * N;
        // ---------------- level 1
        if (rank == 0) { // digit_i = sigma_g(c1coef_i): coefficient k -> k g mod 2N, negated past N
#pragma unroll
            for (int e = 0; e < E; e++) {
                const uint32_t k0 = ((uint32_t)j_M1(tid, e) * gi) & (2 * N - 1);
                const uint64_t x = R1[k0 & (N - 1)];
                a[e] = k0 < (uint32_t)N ? x : (x ? Q0 - x : 0);
            }
            fwd<2, false>(a, XB, K.pr[2]); // XP, lazy [0, 2P)
#pragma unroll
            for (int e = 0; e < E; e += 2) {
                const int pos = pos_M4(tid, e);
                ulonglong2 w0, w0b, w1, w1b;
                ldkey2(gp0, pos, w0, w0b);
                ldkey2(gp1, pos, w1, w1b);
                R2[tid + T * e] = shoup4<2>(a[e], w0);
                R2[tid + T * (e + 1)] = shoup4<2>(a[e + 1], w0b);
                a[e] = shoup4<2>(a[e], w1);
                a[e + 1] = shoup4<2>(a[e + 1], w1b);
            }
        } else if (rank == 1) {
            if (i > 0) { // c1_i = NTT_q0(c1coef_i), canonical, natural order
                fwd<0>(a, XB, K.pr[0]);
                BM_SYNCTHREADS(); // every read of the old S1 (this CTA's gathers) is done
#pragma unroll
                for (int e = 0; e < E; e++) R1[nat_at(nt, e)] = a[e];
            }
        } else if (i > 0) { // C: the c0 update of step i - 1 (a = P^-1 y^0_{i-1}, coefficient order)
            const uint64_t *gqp = K.gk + (size_t)((i - 1) * 4 + 0) * 2 * N;
            fwd<0, false>(a, XB, K.pr[0]); // NTT_q0(P^-1 y^0), lazy [0, 2 q0)
            ulonglong2 kk[2];
#pragma unroll
            for (int e = 0; e < E; e++) {
                const int j = nat_at(nt, e), jp = nat_auto(nt, e, gprev);
                if (!(e & 1)) ldkey2(gqp, pos_M4(tid, e), kk[0], kk[1]);
                const uint64_t ks = shoup4<0>(R2[jp], kk[e & 1]);
                a[e] = reduce_bnd<0>(ks + 2 * Q0 - a[e] + R1[j] + R1[jp]);
            }
            BM_SYNCTHREADS();
#pragma unroll
            for (int e = 0; e < E; e++) R1[nat_at(nt, e)] = a[e];
        }
        csync(); // (1) XP gk0 in A's U0, c1_i in B's S1, c0_i in C's S0
        // ---------------- level 2
        if (rank == 0) { // t1 = P^-1 y^1 -> B's T1
            inv<2>(a, XB, K.pr[2]);
#pragma unroll
            for (int e = 0; e < E; e++)
                peerT1[tid + T * e] = shoup4<0>(a[e], pinv) + (a[e] > (QP >> 1) ? Q0 - 1 : 0); // < 5 q0
        } else if (rank == 1) { // w = INTT_q0(c1_i + P^-1 sigma(c1_i) gk1[q0])
            ulonglong2 kk[2];
#pragma unroll
            for (int e = 0; e < E; e++) {
                const int j = nat_at(nt, e), jp = nat_auto(nt, e, g);
                if (!(e & 1)) ldkey2(gq1, pos_M4(tid, e), kk[0], kk[1]);
                a[e] = reduce_bnd<0>(shoup4<0>(R1[jp], kk[e & 1]) + R1[j]);
            }
            inv<0>(a, XB, K.pr[0]); // w, canonical
        } else { // C: P^-1 y^0_i from A's XP gk0
#pragma unroll
            for (int e = 0; e < E; e++) a[e] = peerU0[tid + T * e];
            inv<2>(a, XB, K.pr[2]);
#pragma unroll
            for (int e = 0; e < E; e++) a[e] = shoup4<0>(a[e], pinv) + (a[e] > (QP >> 1) ? Q0 - 1 : 0); // P^-1 y^0
        }
        csync(); // (2) t1 in B's T1
        // ---------------- level 2b: c1coef_{i+1} = w - t1 (B); C copies c1_i before B overwrites it
        if (rank == 2) {
            const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(peerS1);
            ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(R2);
            for (int k = tid; k < SMEM_WORDS / 2; k += T) dst[k] = src[k];
        }
        if (rank == 1) {
#pragma unroll
            for (int e = 0; e < E; e++) a[e] = submod_d(a[e], reduce_bnd<0>(R2[tid + T * e]), Q0);
            if (last) {
                uint64_t *o = K.out_at(pi, 1);
#pragma unroll
                for (int e = 0; e < E; e++) o[j_M1(tid, e)] = a[e];
            } else {
#pragma unroll
                for (int e = 0; e < E; e++) peerSD[j_M1(tid, e)] = a[e];
            }
        }
        csync(); // (3) A's SD holds c1coef_{i+1}, C holds its copy of c1_i; every remote access is done
        gprev = g;
    }
    if (rank == 2) { // output component 0: INTT_q0(c0 + sigma(c0) + P^-1 sigma(c1) gk0[q0]) - P^-1 y^0
        const uint32_t gl = gprev;
        const uint64_t *gq = K.gk + (size_t)((L - 1) * 4 + 0) * 2 * N;
        tmem_st16(ttsc, a);
        ulonglong2 kk[2];
#pragma unroll
        for (int e = 0; e < E; e++) {
            const int j = nat_at(nt, e), jp = nat_auto(nt, e, gl);
            if (!(e & 1)) ldkey2(gq, pos_M4(tid, e), kk[0], kk[1]);
            a[e] = reduce_bnd<0>(shoup4<0>(R2[jp], kk[e & 1]) + R1[j] + R1[jp]);
        }
        inv<0>(a, XB, K.pr[0]);
        uint64_t *o = K.out_at(pi, 0);
        uint64_t t[E];
        tmem_ld16(ttsc, t);
#pragma unroll
        for (int e = 0; e < E; e++) o[j_M1(tid, e)] = submod_d(a[e], reduce_bnd<0>(t[e]), Q0);
    }
    tmem_free<128>(s_tmem);
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
// Generalised for the baby-step giant-step variant (BM_ORDER_BSGS): the n rotations by i * step,
// i < n (key of rotation r at hgk[r - 1]; g_step = 5^step mod 2N); NTT_OUT: the result stays in the
// NTT domain, canonical, in nout (the giant pass's input) -- per component
//   out_c = base_c + A[c][q0] - NTT_q0(P^-1 y^c)   (= NTT_q0 of the coefficient form, exactly)
// with the same transform count (NTT_q0 of P^-1 y^c in place of INTT_q0 of the sum).
constexpr size_t HROT_SMEM_BYTES = 3 * SMEM_WORDS * sizeof(uint64_t);

template <bool NTT_OUT>
__global__ void __launch_bounds__(T, 1) k_hrot(MatchK K, CtBuf cin, const uint64_t *hgk, int n, int step,
                                               uint32_t g_step, CtBuf nout)
{
    extern __shared__ uint64_t sm[];
    // XB: transform exchanges; SX: (c1, X~P) pairs in natural order (one 16-byte gather per rotation)
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
    const int nt = nat_tid(tid); // SX, SP in natural order (ntt3.cuh nat_at: conflict-free gathers)
    uint64_t a[E];
#pragma unroll 1
    for (int ph = 0; ph < 3; ph++) {
        const int c = ph - 1;
        if (ph == 0) { // (c1, .) staged in natural order; a = c1
            load_eval(a, cin.at(pi, 1));
#pragma unroll
            for (int e = 0; e < E; e++) SX[nat_at(nt, e)].x = a[e];
        } else {       // y^c = INTT_P(A[c][P]); a = base_c + A[c][q0]
            tmem_ld16(tA + 32 * (2 * c + 1), a); // A[c][P]
            inv<2>(a, XB, K.pr[2]); // y^c (canonical [0, P))
#pragma unroll
            for (int e = 0; e < E; e++) a[e] = shoup4<0>(a[e], pinv) + (a[e] > (QP >> 1) ? Q0 - 1 : 0);
            if (!NTT_OUT) {
                tmem_st16(tA + 32 * (2 * c + 1), a); // P^-1 y^c (coefficient j_M1(tid, e)) over A[c][P]
                const uint64_t *base = c ? cin.at(pi, 1) : b0s;
#pragma unroll
                for (int e = 0; e < E; e += 2) {
                    const int pos = pos_M4(tid, e);
                    const ulonglong2 bv = *reinterpret_cast<const ulonglong2 *>(base + pos);
                    a[e] = bv.x;
                    a[e + 1] = bv.y;
                }
                uint64_t av[E];
                tmem_ld16(tA + 32 * (2 * c), av); // A[c][q0]
#pragma unroll
                for (int e = 0; e < E; e++) a[e] = csub(a[e] + av[e], Q0);
            }
        }
        if (NTT_OUT && ph > 0) { // out_c = base_c + A[c][q0] - NTT_q0(P^-1 y^c), NTT domain, canonical
            fwd<0, false>(a, XB, K.pr[0]); // lazy [0, 2 q0)
            const uint64_t *base = c ? cin.at(pi, 1) : b0s;
            uint64_t *o = nout.at(pi, c);
            uint64_t av[E];
            tmem_ld16(tA + 32 * (2 * c), av); // A[c][q0]
#pragma unroll
            for (int e = 0; e < E; e += 2) {
                const int pos = pos_M4(tid, e);
                const ulonglong2 bv = *reinterpret_cast<const ulonglong2 *>(base + pos);
                const uint64_t x0 = csub(bv.x + av[e], Q0), x1 = csub(bv.y + av[e + 1], Q0);
                st2(o + pos, submod_d(x0, csub(a[e], Q0), Q0), submod_d(x1, csub(a[e + 1], Q0), Q0));
            }
            continue;
        }
        inv<0>(a, XB, K.pr[0]);
        if (ph > 0) { // out_c = INTT_q0(base_c + A[c][q0]) - P^-1 y^c
            uint64_t *o = K.out_at(pi, c);
            uint64_t t[E];
            tmem_ld16(tA + 32 * (2 * c + 1), t);
#pragma unroll
            for (int e = 0; e < E; e++) o[j_M1(tid, e)] = submod_d(a[e], reduce_bnd<0>(t[e]), Q0);
            continue;
        }
        // ---- digit: X~P = NTT_P(x), staged next to c1
        fwd<2, false>(a, XB, K.pr[2]); // lazy [0, 2P): Shoup / 128-bit product operand
#pragma unroll
        for (int e = 0; e < E; e++) SX[nat_at(nt, e)].y = a[e];
        BM_SYNCTHREADS();
        // ---- the s-1 rotations' key-switch products, two coefficients (one 16-byte key position) at a
        //      time, the next rotation's keys loaded while this one's are used
#pragma unroll 1
        for (int g2 = 0; g2 < E / 2; g2++) {
            const int e0 = 2 * g2, pos = pos_M4(tid, e0);
            const uint32_t i0 = nat_i(nt, e0), i1 = nat_i(nt, e0 + 1);
            u128 A[2][4]; // [coefficient][c * 2 + limb (q0, P)]
#pragma unroll
            for (int u = 0; u < 2; u++)
#pragma unroll
                for (int v = 0; v < 4; v++) A[u][v] = 0;
            ulonglong2 kc[4], kn[4];
#pragma unroll
            for (int v = 0; v < 4; v++) kc[v] = ld2(hgk + ((size_t)(step - 1) * 4 + v) * N + pos);
            uint32_t gr = 1;
#pragma unroll 1
            for (int r = 1; r < n; r++) {
                gr = (gr * g_step) & (2 * N - 1); // 5^(r step) mod 2N
                if (r + 1 < n) {
#pragma unroll
                    for (int v = 0; v < 4; v++) kn[v] = ld2(hgk + ((size_t)((r + 1) * step - 1) * 4 + v) * N + pos);
                }
                const ulonglong2 x0 = SX[nat_auto_i(i0, gr)], x1 = SX[nat_auto_i(i1, gr)];
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
        //      q0: the same residues as the term-by-term sum), c0 staged in natural order over X~P
        BM_SYNCTHREADS();
        stage_nat(SP, cin.at(pi, 0));
#pragma unroll 1
        for (uint32_t g = g_step, w = 1; w < (uint32_t)n; w <<= 1, g = (g * g) & (2 * N - 1)) {
            BM_SYNCTHREADS();
#pragma unroll
            for (int e = 0; e < E; e++) {
                a[e] = csub(SP[nat_at(nt, e)] + SP[nat_auto(nt, e, g)], Q0);
            }
            BM_SYNCTHREADS();
#pragma unroll
            for (int e = 0; e < E; e++) SP[nat_at(nt, e)] = a[e];
        }
        BM_SYNCTHREADS();
#pragma unroll
        for (int e = 0; e < E; e++) b0s[pos_M4(tid, e)] = SP[nat_at(nt, e)];
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
    store_coef(K.out_at(pi, c), a);
}

// ================================================================== f2 K7: relin-free degree-2 output
// BM_ORDER_DEG2 (p = d, s = 1, reading R32): the scan stops after the
// tensor, the result is the degree-2 ciphertext (d0, d1, d2) = sum_i tensor(C_u,i, C_s,i) rescaled by q1
// component by component -- no key switch, no rotations (s = 1: every slot is a score).  CTA (pair, c):
//   U = INTT_q1(d_c[q1]) (canonical);  z^ = centred_q1(U);  out_c = q1^-1 (INTT_q0(d_c[q0]) - z^) mod q0
// (PAPER.md:329 Res at level 1 -> 0 on each component; the same rescale K3 applies after its ModDown).
// Output [nq][n_sets][3][N] (coefficients, [0, q0)) or rows[j] + (set * 3 + c) N.
constexpr size_t K7_SMEM_BYTES = (SMEM_WORDS + (size_t)N) * sizeof(uint64_t);
__global__ void __launch_bounds__(T, 1) k_rescale_deg2(MatchK K)
{
    extern __shared__ uint64_t sm[];
    uint64_t *zs = sm + SMEM_WORDS;
    const int tid = threadIdx.x;
    const int64_t pi = blockIdx.x / 3;
    const int c = (int)(blockIdx.x - 3 * pi);
    const uint64_t *src = c < 2 ? K.D01 : K.D2; // poly P0 = [q0], P0 + 1 = [q1] (dofs)
    const int P0 = c < 2 ? 2 * c : 0;
    uint64_t a[E];
    load_eval_d(a, src, K, P0 + 1, pi);
    inv_f<1>(a, sm, K.pr[1].invf, K.pr[1].ninvf, K.pr[1].ninv_w1f); // canonical [0, q1)
#pragma unroll
    for (int e = 0; e < E; e++) zs[tid + T * e] = a[e] > (Q1 >> 1) ? a[e] + (Q0 - Q1) : a[e]; // z^ mod q0
    load_eval_d(a, src, K, P0, pi);
    inv<0>(a, sm, K.pr[0]); // canonical [0, q0)
    const ulonglong2 q1inv = K.q1inv;
#pragma unroll
    for (int e = 0; e < E; e++) a[e] = reduce_bnd<0>(shoup4<0>(a[e] + Q0 - zs[tid + T * e], q1inv));
    BM_CHECK(pi >= 0 && pi < (int64_t)K.cq * K.ct && K.jq0 + pi / K.ct < K.nq_total);
    const int64_t set = K.t0 + pi % K.ct;
    uint64_t *o = K.rows ? K.rows[K.jq0 + pi / K.ct] + ((K.set_off + set) * 3 + c) * (int64_t)N
                         : K.out + ((K.out_row(pi)) * 3 + c) * (int64_t)N;
    store_coef(o, a);
}
