// ntt2.cuh -- prime-specialised modular arithmetic of the NTT core (ntt3.cuh) and the kernels.
// (The v2 transform core that first used it now lives in tools/ntt_legacy.cuh.)
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
#include "ntt_base.cuh"

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
// forming Q q from shifts for q = 2^k - c (ptxas re-balances it back onto IMAD.X, slower; for
// P = 2^60 - 2^14 + 1 the shift form takes 11 instead of 14 FMA-pipe slots but adds 5 ALU
// instructions, and the ladder ran 16.52 -> 16.56 ms: issue, not the FMA pipe alone, binds), and
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

// exact x mod q for the bounded x the NTT produces (any x < 2^64 for q0 and P, x < 2^62 for q1,
// x < 2^60 for q2): q = 2^k - c with 0 < c < 2^20, so Qe = x >> k under-estimates floor(x / q) by
// at most 1 (x / q - x / 2^k = x c / (2^k q) < 1 for these bounds) and x - Qe q lies in [0, 2q).
template <int PI> BM_D uint64_t reduce_bnd(uint64_t x)
{
    constexpr int k = PI == 0 ? 58 : Q40<PI> ? 40 : 60;
    constexpr uint64_t q = PrimeC<PI>::q;
    constexpr uint64_t c = (1ull << k) - q; // 835583, 147455, 16383, 737279
    uint64_t r;
#ifdef BM_RB64
    if (true) {
#else
    if (Q40<PI>) {
#endif
        const uint64_t Qe = x >> k; // < 2^22: Qe c needs 64 bits
        r = x - (Qe << k) + Qe * c;
    } else {
        // Qe < 64 and c < 2^20: one 32-bit IMAD (a 64-bit Qe c costs an IMAD.WIDE + a move)
        const uint32_t Qe = (uint32_t)(x >> k);
        r = (x & ((1ull << k) - 1)) + (uint64_t)(Qe * (uint32_t)c);
    }
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

// ------------------------------------------------------------------ forward butterfly
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

// ------------------------------------------------------------------ inverse butterfly
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

} // namespace bm
