// ntt2.cuh -- prime-specialised NTT core (v2).  Same layouts and transform as ntt.cuh
// (CT forward / GS inverse, bit-reversed evaluation order, L1 -> L3 and L3 -> L1), but:
//  * the prime is a template parameter (q0, q1, P), so q and 2q are immediates;
//  * the Shoup quotient is approximated from three 32-bit partial products
//    (a1 w1 + hi(a1 w0) + hi(a0 w1)), which under-estimates floor(a w' / 2^64) by at most 2,
//    so a w - Q q lies in [0, 4q) (instead of [0, 2q)) for any a < 2^64;
//  * lazy-reduction bounds are chosen per prime:
//      forward q0, q1: no reduction inside the transform (bound grows by 4q per stage;
//                      13 stages -> < 53q < 2^64 for q0), one final reduction;
//      forward P:      values kept in [0, 8q) with one conditional subtraction per butterfly;
//      inverse q1:     no reduction (the x-output bound doubles per stage: < 2^15 q < 2^55);
//      inverse q0, P:  values kept in [0, 4q) with one conditional subtraction per butterfly.
#pragma once
#include "ntt.cuh"

namespace bm {

template <int PI> struct PrimeC;
template <> struct PrimeC<0> { static constexpr uint64_t q = Q0; };
template <> struct PrimeC<1> { static constexpr uint64_t q = Q1; };
template <> struct PrimeC<2> { static constexpr uint64_t q = QP; };
template <> struct PrimeC<3> { static constexpr uint64_t q = Q2; }; // f3 only
// the 40-bit primes (q1, q2) share the lazy-reduction schedule: never reduced inside a transform
template <int PI> constexpr bool Q40 = (PI == 1 || PI == 3);

// Q q mod 2^64
template <int PI> BM_D uint64_t mul_q(uint64_t Q)
{
    return Q * PrimeC<PI>::q;
}

// a w mod q, lazily: result in [0, 4q) for any a < 2^64 (w < q, wp = floor(w 2^64 / q)).
// Q = a1 wp1 + hi(a0 wp1) + hi(a1 wp0) (32-bit halves) under-estimates floor(a wp / 2^64) by at
// most 2; the remainder a w - Q q is formed mod 2^64 as a w + Q (2^64 - q) in one multiply-add
// chain: 2 IMAD.HI + 3 IMAD.WIDE + 4 IMAD on the FMA-heavy pipe, one carry on the ALU pipe.
// (IMAD.WIDE / IMAD.HI issue at half the IMAD rate, tools/pipe_bench.cu.  Tried and dropped:
// forming Q q from shifts for q = 2^k - c (ptxas re-balances it back onto IMAD.X, slower), and
// the quotient's cross terms on the idle FP64 pipe (exact, but the u32 <-> f64 conversions cost
// more FMA/ALU issue than the two IMAD.HI they replace: 2.36 vs 2.75 butterflies/clk/SM).)
template <int PI> BM_D uint64_t shoup4(uint64_t a, uint64_t w, uint64_t wp)
{
#ifdef BM_SHOUP_C
    const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), w0 = (uint32_t)wp, w1 = (uint32_t)(wp >> 32);
    const uint64_t Q = (uint64_t)a1 * w1 + ((uint64_t)__umulhi(a1, w0) + __umulhi(a0, w1));
    return a * w - mul_q<PI>(Q);
#else
    constexpr uint64_t nq = 0ull - PrimeC<PI>::q;
    uint64_t r;
    asm("{\n\t"
        ".reg .u32 a0, a1, w0, w1, p0, p1, h, c, t0, t1, r0, r1;\n\t"
        ".reg .u64 Q, R;\n\t"
        "mov.b64 {a0, a1}, %1;\n\t"
        "mov.b64 {w0, w1}, %2;\n\t"
        "mov.b64 {p0, p1}, %3;\n\t"
        "mul.hi.u32 h, a0, p1;\n\t"
        "mad.hi.cc.u32 h, a1, p0, h;\n\t"
        "addc.u32 c, 0, 0;\n\t"
        "mov.b64 Q, {h, c};\n\t"
        "mad.wide.u32 Q, a1, p1, Q;\n\t"
        "mov.b64 {t0, t1}, Q;\n\t"
        "mul.wide.u32 R, a0, w0;\n\t"
        "mad.wide.u32 R, t0, %4, R;\n\t"
        "mov.b64 {r0, r1}, R;\n\t"
        "mad.lo.u32 r1, a0, w1, r1;\n\t"
        "mad.lo.u32 r1, a1, w0, r1;\n\t"
        "mad.lo.u32 r1, t0, %5, r1;\n\t"
        "mad.lo.u32 r1, t1, %4, r1;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "}"
        : "=l"(r)
        : "l"(a), "l"(w), "l"(wp), "n"((uint32_t)nq), "n"((uint32_t)(nq >> 32)));
    return r;
#endif
}
template <int PI> BM_D uint64_t shoup4(uint64_t a, ulonglong2 w) { return shoup4<PI>(a, w.x, w.y); }

// exact x mod q for any x < 2^64 (Shoup with w = 1 and a final correction)
template <int PI> BM_D uint64_t reduce_full(uint64_t x, uint64_t one_p)
{
    constexpr uint64_t q = PrimeC<PI>::q;
    uint64_t r = x - mul_q<PI>(__umul64hi(x, one_p)); // [0, 2q)
    return r >= q ? r - q : r;
}

// exact x mod q for the bounded x the NTT produces (any x < 2^64 for q0 and P, x < 2^62 for q1,
// x < 2^60 for q2): q = 2^k - c with 0 < c < 2^20, so Qe = x >> k under-estimates floor(x / q) by
// at most 1 (x / q - x / 2^k = x c / (2^k q) < 1 for these bounds) and x - Qe q lies in [0, 2q).
template <int PI> BM_D uint64_t reduce_bnd(uint64_t x)
{
    constexpr int k = PI == 0 ? 58 : Q40<PI> ? 40 : 60;
    constexpr uint64_t q = PrimeC<PI>::q;
    constexpr uint64_t c = (1ull << k) - q; // 835583, 147455, 16383, 737279
    const uint64_t Qe = x >> k;
    const uint64_t r = x - (Qe << k) + Qe * c;
    return r >= q ? r - q : r;
}

// x - floor(x / 2^k) q = (x mod 2^k) + floor(x / 2^k) c  in [0, 2q) for any x < 2^64 (q0, P):
// reduce_bnd without its final conditional subtraction (the lazy reductions of ntt3.cuh)
template <int PI> BM_D uint64_t reduce_lazy(uint64_t x)
{
    static_assert(!Q40<PI>, "q1 / q2 transforms never reduce inside");
    constexpr int k = PI == 0 ? 58 : 60;
    constexpr uint32_t c = (uint32_t)((1ull << k) - PrimeC<PI>::q); // 835583, 16383
    const uint32_t Qe = (uint32_t)(x >> k);                         // <= 63 / 15
    return (x & ((1ull << k) - 1)) + (uint64_t)(Qe * c);
}

// ------------------------------------------------------------------ forward (L1 -> L3)
template <int PI> BM_D void ct4(uint64_t &x, uint64_t &y, ulonglong2 w)
{
    constexpr uint64_t q = PrimeC<PI>::q;
    uint64_t X = x;
    if (PI == 2) X = X >= 4 * q ? X - 4 * q : X; // P: keep [0, 8q)
    const uint64_t T = shoup4<PI>(y, w);         // [0, 4q)
    x = X + T;
    y = X - T + 4 * q;
}

template <int PI> BM_D void ntt_fwd2(uint64_t a[32], uint64_t *sm, const PrimeK &P)
{
    const int tid = threadIdx.x;
#pragma unroll
    for (int s = 0; s < 5; s++) {
        const int half = 16 >> s;
#pragma unroll
        for (int k = 0; k < 32; k++) {
            if (k & half) continue;
            ct4<PI>(a[k], a[k + half], ldtw(P.fwd + (1 << s) + (k >> (5 - s))));
        }
    }
    exchange<1, 2>(a, sm);
#pragma unroll
    for (int s = 5; s < 9; s++) {
        const int half = 8 >> (s - 5);
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int B = (tid + 256 * h) >> 4;
#pragma unroll
            for (int k = 0; k < 16; k++) {
                if (k & half) continue;
                ct4<PI>(a[16 * h + k], a[16 * h + k + half], ldtw(P.fwd + (1 << s) + (B << (s - 5)) + (k >> (9 - s))));
            }
        }
    }
    exchange<2, 3>(a, sm);
#pragma unroll
    for (int s = 9; s < 13; s++) {
        const int half = 8 >> (s - 9);
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int G = tid + 256 * h;
#pragma unroll
            for (int k = 0; k < 16; k++) {
                if (k & half) continue;
                ct4<PI>(a[16 * h + k], a[16 * h + k + half], ldtw(P.fwd + (1 << s) + (G << (s - 9)) + (k >> (13 - s))));
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 32; e++) a[e] = reduce_full<PI>(a[e], P.one_p);
}

// Forward CT butterfly of stage s for ntt3.cuh.  q0, q1: never reduced (bound grows by 4q per
// stage, < 53 q < 2^64 after 13 stages).  P (16 P < 2^64): the unmultiplied input is reduced
// lazily to [0, 2q) on stages s = 0 (mod 3), so inputs stay < 14 q (2 + 3 x 4); one 5-instruction
// lazy reduction every third stage instead of a 6-instruction conditional subtraction each stage.
template <int PI> BM_D void ct4s(uint64_t &x, uint64_t &y, ulonglong2 w, int s)
{
    constexpr uint64_t q = PrimeC<PI>::q;
    uint64_t X = x;
    if (PI == 2 && s % 3 == 0) X = reduce_lazy<2>(X);
    const uint64_t T = shoup4<PI>(y, w); // [0, 4q)
    x = X + T;
    y = X - T + 4 * q;
}

// ------------------------------------------------------------------ inverse (L3 -> L1)
// GS butterfly of inverse stage number ST (0 = first executed) whose inputs are < B q with
// B = 4 (q0, P: reduced every stage) or 4 * 2^ST (q1: never reduced): x + y, (x - y + Bq) w
template <int PI, int ST> BM_D void gs4(uint64_t &x, uint64_t &y, ulonglong2 w)
{
    constexpr uint64_t q = PrimeC<PI>::q;
    constexpr uint64_t B = Q40<PI> ? (4ull << ST) : 4ull;
    uint64_t X = x + y;
    if (!Q40<PI>) X = X >= 4 * q ? X - 4 * q : X; // q0, P: keep [0, 4q)
    const uint64_t T = x - y + (uint64_t)B * q;
    x = X;
    y = shoup4<PI>(T, w);
}

// Inverse GS butterfly of stage ST (0 = first executed) for ntt3.cuh, inputs < B q: the x-side
// output x + y doubles the bound each stage, the y-side (a Shoup product) is < 4q.
//   q1: B = 4 << ST, never reduced (< 2^15 q1 after 12 stages);
//   q0: B = 4 << (ST mod 4), x + y reduced lazily to [0, 2q) when ST = 3 (mod 4) (64 q0 < 2^64);
//   P:  B = 4 << (ST mod 2), reduced when ST is odd (16 P < 2^64).
// So B = 4 again at ST = 12 (the last stage, N^-1 folded in, ntt3.cuh) for every prime but q1.
template <int PI, int ST> BM_D void gs4s(uint64_t &x, uint64_t &y, ulonglong2 w)
{
    constexpr uint64_t q = PrimeC<PI>::q;
    constexpr uint64_t B = Q40<PI> ? (4ull << ST) : PI == 0 ? (4ull << (ST % 4)) : (4ull << (ST % 2));
    constexpr bool RED = PI == 0 ? (ST % 4 == 3) : PI == 2 ? (ST % 2 == 1) : false;
    uint64_t X = x + y;
    if (RED) X = reduce_lazy<Q40<PI> ? 0 : PI>(X);
    const uint64_t T = x - y + B * q;
    x = X;
    y = shoup4<PI>(T, w);
}

template <int PI> BM_D void ntt_inv2(uint64_t a[32], uint64_t *sm, const PrimeK &P)
{
    const int tid = threadIdx.x;
#pragma unroll
    for (int s = 12; s >= 9; s--) {
        const int half = 8 >> (s - 9);
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int G = tid + 256 * h;
#pragma unroll
            for (int k = 0; k < 16; k++) {
                if (k & half) continue;
                const ulonglong2 w = ldtw(P.inv + (1 << s) + (G << (s - 9)) + (k >> (13 - s)));
                switch (12 - s) {
                case 0: gs4<PI, 0>(a[16 * h + k], a[16 * h + k + half], w); break;
                case 1: gs4<PI, 1>(a[16 * h + k], a[16 * h + k + half], w); break;
                case 2: gs4<PI, 2>(a[16 * h + k], a[16 * h + k + half], w); break;
                default: gs4<PI, 3>(a[16 * h + k], a[16 * h + k + half], w); break;
                }
            }
        }
    }
    exchange<3, 2>(a, sm);
#pragma unroll
    for (int s = 8; s >= 5; s--) {
        const int half = 8 >> (s - 5);
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int B = (tid + 256 * h) >> 4;
#pragma unroll
            for (int k = 0; k < 16; k++) {
                if (k & half) continue;
                const ulonglong2 w = ldtw(P.inv + (1 << s) + (B << (s - 5)) + (k >> (9 - s)));
                switch (12 - s) {
                case 4: gs4<PI, 4>(a[16 * h + k], a[16 * h + k + half], w); break;
                case 5: gs4<PI, 5>(a[16 * h + k], a[16 * h + k + half], w); break;
                case 6: gs4<PI, 6>(a[16 * h + k], a[16 * h + k + half], w); break;
                default: gs4<PI, 7>(a[16 * h + k], a[16 * h + k + half], w); break;
                }
            }
        }
    }
    exchange<2, 1>(a, sm);
#pragma unroll
    for (int s = 4; s >= 1; s--) {
        const int half = 16 >> s;
#pragma unroll
        for (int k = 0; k < 32; k++) {
            if (k & half) continue;
            const ulonglong2 w = ldtw(P.inv + (1 << s) + (k >> (5 - s)));
            switch (12 - s) {
            case 8: gs4<PI, 8>(a[k], a[k + half], w); break;
            case 9: gs4<PI, 9>(a[k], a[k + half], w); break;
            case 10: gs4<PI, 10>(a[k], a[k + half], w); break;
            default: gs4<PI, 11>(a[k], a[k + half], w); break;
            }
        }
    }
    // last stage (s = 0) with N^-1 folded in; inputs < inv_bound(12) q
    constexpr uint64_t q = PrimeC<PI>::q;
    constexpr uint64_t Bq = (Q40<PI> ? (4ull << 12) : 4ull) * q;
#pragma unroll
    for (int k = 0; k < 16; k++) {
        const uint64_t x = a[k], y = a[k + 16];
        a[k] = reduce_full<PI>(shoup4<PI>(x + y, P.ninv), P.one_p);
        a[k + 16] = reduce_full<PI>(shoup4<PI>(x - y + Bq, P.ninv_w1), P.one_p);
    }
}

// runtime prime dispatch (one code copy per prime at each call site)
BM_D void ntt_fwd_rt(uint64_t a[32], uint64_t *sm, const PrimeK &P, int pi)
{
    if (pi == 0) ntt_fwd2<0>(a, sm, P);
    else if (pi == 1) ntt_fwd2<1>(a, sm, P);
    else ntt_fwd2<2>(a, sm, P);
}
BM_D void ntt_inv_rt(uint64_t a[32], uint64_t *sm, const PrimeK &P, int pi)
{
    if (pi == 0) ntt_inv2<0>(a, sm, P);
    else if (pi == 1) ntt_inv2<1>(a, sm, P);
    else ntt_inv2<2>(a, sm, P);
}

} // namespace bm
