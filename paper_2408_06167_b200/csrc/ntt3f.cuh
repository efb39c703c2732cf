// ntt3f.cuh -- the q1 and q2 transforms on the FP64 pipe (exact), templated on the prime index
// (PI = 1: q1, PI = 3: q2; the comments write q1 for either).  q1 < 2^40, so every residue, lazy
// value and product piece fits a double exactly; the data stay in the registers and the shared-
// memory exchanges of ntt3.cuh (same layouts M1..M4, same 512-thread CTA) as double bit patterns.
// The Shoup product becomes (tools/pipe_bench.cu: DFMA issues at the IMAD rate on its own pipe):
//   a w mod q1 for |a| < 2^46, 0 <= w < q1, wq = fl(w / q1):
//     hi = fl(a w), lo = a w - hi (one FMA, exact), qt = floor(fl(a wq)) (round-down magic add),
//     r = (hi - qt q1) + lo   -- the FMA's exact result is an integer below 2^44, nothing rounds.
//   |a wq - a w / q1| < 2^-6, so qt is the true quotient floor(a w / q1) or one off: |r| < 3 q1.
// 7 FP64 instructions per product instead of 2 IMAD.HI + 3 IMAD.WIDE + 4 IMAD on the FMA pipe.
// Values are signed integers: the forward bound grows by 3 q1 per stage (< 40 q1 < 2^46), the
// inverse x-side doubles per stage and is reduced to (-q1, 2 q1) every fifth stage.  Outputs are
// canonical u64 residues, like fwd<1> / inv<1>; inputs are canonical u64 residues.
#pragma once
#include "ntt3.cuh"

namespace bm {
namespace v3 {

template <int PI> BM_HD constexpr double f_q() { return PI == 1 ? (double)Q1 : (double)Q2; }
template <int PI> BM_HD constexpr double f_qinv() { return PI == 1 ? 1.0 / (double)Q1 : 1.0 / (double)Q2; }
constexpr double F_MAGIC = 6755399441055744.0; // 1.5 2^52: x + M has ulp 1 for |x| < 2^51
constexpr double F_2P52 = 4503599627370496.0;

BM_D double fl_floor(double x) { return __dadd_rd(x, F_MAGIC) - F_MAGIC; }
BM_D double as_d(uint64_t x) { return __longlong_as_double((long long)x); }
BM_D uint64_t as_u(double x) { return (uint64_t)__double_as_longlong(x); }
// twiddle entry: (w, wq) as double bit patterns
template <int PI> BM_D double mulw(double a, ulonglong2 t)
{
    const double w = as_d(t.x), wq = as_d(t.y);
    const double hi = a * w;
    const double lo = __fma_rn(a, w, -hi);
    const double qt = fl_floor(a * wq);
    return __fma_rn(-qt, f_q<PI>(), hi) + lo;
}
// (-q1, 2 q1) for |x| < 2^51
template <int PI> BM_D double red_f(double x) { return __fma_rn(-fl_floor(x * f_qinv<PI>()), f_q<PI>(), x); }
// canonical u64 residue of an integer-valued double |x| < 2^51
template <int PI> BM_D uint64_t canon_f(double x)
{
    double r = red_f<PI>(x);
    r = r < 0 ? r + f_q<PI>() : r;
    r = r >= f_q<PI>() ? r - f_q<PI>() : r;
    return as_u(r + F_2P52) & ((1ull << 52) - 1);
}
BM_D double from_u(uint64_t x) { return as_d(x | 0x4330000000000000ull) - F_2P52; } // x < 2^52

template <int PI> BM_D void ct_f(uint64_t &x, uint64_t &y, ulonglong2 w)
{
    const double X = as_d(x), T = mulw<PI>(as_d(y), w);
    x = as_u(X + T);
    y = as_u(X - T);
}
template <int PI, int ST> BM_D void gs_f(uint64_t &x, uint64_t &y, ulonglong2 w)
{
    const double a = as_d(x), b = as_d(y);
    double X = a + b;
    if (ST % 5 == 4) X = red_f<PI>(X);
    x = as_u(X);
    y = as_u(mulw<PI>(a - b, w));
}

// forward, M1 -> M4 (twiddles fwdf), canonical u64 in and out
template <int PI> BM_D void fwd_f(uint64_t a[E], uint64_t *sm, const ulonglong2 *tw)
{
    const int tid = threadIdx.x;
#pragma unroll
    for (int e = 0; e < E; e++) a[e] = as_u(from_u(a[e]));
#pragma unroll
    for (int s = 0; s < 4; s++) {
        const int half = 8 >> s;
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & half) continue;
            ct_f<PI>(a[k], a[k + half], ldtw(tw + (1 << s) + (k >> (4 - s))));
        }
    }
    xchg<1, 2>(a, sm);
    {
        const int B = tid >> 5;
#pragma unroll
        for (int s = 4; s < 8; s++) {
            const int half = 8 >> (s - 4);
#pragma unroll
            for (int k = 0; k < E; k++) {
                if (k & half) continue;
                ct_f<PI>(a[k], a[k + half], ldtw(tw + (1 << s) + (B << (s - 4)) + (k >> (8 - s))));
            }
        }
    }
    xchg<2, 3>(a, sm);
    const int G = tid >> 1, odd = tid & 1;
#pragma unroll
    for (int s = 8; s < 12; s++) {
        const int half = 8 >> (s - 8);
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & half) continue;
            ct_f<PI>(a[k], a[k + half], ldtw(tw + (1 << s) + ((k >> (12 - s)) << 8) + G));
        }
    }
#pragma unroll
    for (int m = 0; m < 8; m++) {
        const uint64_t r = shfl1(odd ? a[2 * m] : a[2 * m + 1]);
        uint64_t x = odd ? r : a[2 * m], y = odd ? a[2 * m + 1] : r;
        ct_f<PI>(x, y, ldtw(tw + 4096 + 512 * m + tid));
        a[2 * m] = canon_f<PI>(as_d(x));
        a[2 * m + 1] = canon_f<PI>(as_d(y));
    }
}

// inverse, M4 -> M1 (twiddles invf; N^-1 and N^-1 inv[1] as (w, wq) doubles), canonical in and out
template <int PI> BM_D void inv_f(uint64_t a[E], uint64_t *sm, const ulonglong2 *tw, ulonglong2 ninv, ulonglong2 ninv_w1)
{
    const int tid = threadIdx.x;
    const int G = tid >> 1, odd = tid & 1;
#pragma unroll
    for (int e = 0; e < E; e++) a[e] = as_u(from_u(a[e]));
#pragma unroll
    for (int m = 0; m < 8; m++) gs_f<PI, 0>(a[2 * m], a[2 * m + 1], ldtw(tw + 4096 + 512 * m + tid));
#pragma unroll
    for (int m = 0; m < 8; m++) {
        const uint64_t r = shfl1(odd ? a[2 * m] : a[2 * m + 1]);
        if (odd) a[2 * m] = r;
        else a[2 * m + 1] = r;
    }
#pragma unroll
    for (int s = 11; s >= 8; s--) {
        const int half = 8 >> (s - 8);
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & half) continue;
            const ulonglong2 w = ldtw(tw + (1 << s) + ((k >> (12 - s)) << 8) + G);
            switch (12 - s) {
            case 1: gs_f<PI, 1>(a[k], a[k + half], w); break;
            case 2: gs_f<PI, 2>(a[k], a[k + half], w); break;
            case 3: gs_f<PI, 3>(a[k], a[k + half], w); break;
            default: gs_f<PI, 4>(a[k], a[k + half], w); break;
            }
        }
    }
    xchg<3, 2>(a, sm);
    {
        const int B = tid >> 5;
#pragma unroll
        for (int s = 7; s >= 4; s--) {
            const int half = 8 >> (s - 4);
#pragma unroll
            for (int k = 0; k < E; k++) {
                if (k & half) continue;
                const ulonglong2 w = ldtw(tw + (1 << s) + (B << (s - 4)) + (k >> (8 - s)));
                switch (12 - s) {
                case 5: gs_f<PI, 5>(a[k], a[k + half], w); break;
                case 6: gs_f<PI, 6>(a[k], a[k + half], w); break;
                case 7: gs_f<PI, 7>(a[k], a[k + half], w); break;
                default: gs_f<PI, 8>(a[k], a[k + half], w); break;
                }
            }
        }
    }
    xchg<2, 1>(a, sm);
#pragma unroll
    for (int s = 3; s >= 1; s--) {
        const int half = 8 >> s;
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & half) continue;
            const ulonglong2 w = ldtw(tw + (1 << s) + (k >> (4 - s)));
            switch (12 - s) {
            case 9: gs_f<PI, 9>(a[k], a[k + half], w); break;
            case 10: gs_f<PI, 10>(a[k], a[k + half], w); break;
            default: gs_f<PI, 11>(a[k], a[k + half], w); break;
            }
        }
    }
    // s = 0 with N^-1 folded in (inputs |v| < 12 q1: reduced at ST 9, doubled twice since)
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const double x = as_d(a[k]), y = as_d(a[k + 8]);
        a[k] = canon_f<PI>(mulw<PI>(x + y, ninv));
        a[k + 8] = canon_f<PI>(mulw<PI>(x - y, ninv_w1));
    }
}

} // namespace v3
} // namespace bm
