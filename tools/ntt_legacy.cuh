// ntt_legacy.cuh -- DIAGNOSTIC ONLY (tools/ntt_bench.cu), not part of the library: the superseded
// v1 core (below) and v2 transforms (end of file) the library's ntt3.cuh replaced.
//
// v1: register-blocked negacyclic NTT / INTT of one 8192-coefficient u64 polynomial
// per 256-thread CTA (K1 in SURVEY.md sec. 2.2).
//
// Transform: forward = Cooley-Tukey with psi^brev twiddles (Harvey lazy butterflies in
// [0,4q)), output in bit-reversed evaluation order: NTT(a)[j] = a(psi^(2 brev13(j) + 1)).
// Inverse = Gentleman-Sande with psi^-brev twiddles, N^-1 folded into the last stage.
//
// Each thread owns 32 coefficients in registers; 13 stages = 3 register passes (5 + 4 + 4
// radix-2 stages) with 2 shared-memory transposes in between:
//   layout L1 ("coefficient"): a[k]        <-> j = tid + 256 k              (k < 32)
//   layout L2 (middle):        a[16h + k]  <-> j = 256 (c>>4) + 16 k + (c&15), c = tid + 256 h
//   layout L3 ("evaluation"):  a[16h + k]  <-> j = 16 (tid + 256 h) + k      (k < 16)
// Forward maps L1 -> L3, inverse L3 -> L1.  Shared memory is padded (one word per 16) so
// every transpose is bank-conflict free.
#pragma once
#include "../paper_2408_06167_b200/csrc/ntt2.cuh"

namespace bm {

constexpr int NTT_THREADS = 256;

// CT butterfly: x, y in [0,4q) -> x + w y, x - w y in [0,4q)
BM_D void ct_bfly(uint64_t &x, uint64_t &y, ulonglong2 w, uint64_t q, uint64_t q2)
{
    uint64_t X = x >= q2 ? x - q2 : x;
    uint64_t T = shoup(y, w, q);
    x = X + T;
    y = X - T + q2;
}
// GS butterfly: x, y in [0,2q) -> x + y, (x - y) w in [0,2q)
BM_D void gs_bfly(uint64_t &x, uint64_t &y, ulonglong2 w, uint64_t q, uint64_t q2)
{
    uint64_t X = x + y;
    X = X >= q2 ? X - q2 : X;
    uint64_t T = x - y + q2;
    x = X;
    y = shoup(T, w, q);
}

// ---------------------------------------------------------------- layout helpers
// j of element e (0..31) in each layout for thread tid
BM_D int j_L1(int tid, int e) { return tid + 256 * e; }
BM_D int j_L2(int tid, int e)
{
    int c = tid + 256 * (e >> 4);
    return 256 * (c >> 4) + 16 * (e & 15) + (c & 15);
}
BM_D int j_L3(int tid, int e) { return 16 * (tid + 256 * (e >> 4)) + (e & 15); }

// Device storage order of NTT-domain polynomials: the element thread tid holds in register e
// of layout L3 lives at pos_L3(tid, e) = 512 (e/2) + 2 tid + (e&1), so that every NTT-domain
// global access is one coalesced 16-byte vector per lane (512 contiguous bytes per warp) for
// the register pair (e, e+1).  j_of_pos inverts it (used by the automorphism gathers).
BM_D int pos_L3(int tid, int e) { return 512 * (e >> 1) + 2 * tid + (e & 1); }
BM_D int j_of_pos(int pos)
{
    const int tid = (pos >> 1) & 255, e = 2 * (pos >> 9) + (pos & 1);
    return j_L3(tid, e);
}

template <int FROM, int TO>
BM_D void exchange(uint64_t a[32], uint64_t *sm)
{
    const int tid = threadIdx.x;
    __syncthreads(); // previous readers of sm are done
#pragma unroll
    for (int e = 0; e < 32; e++) {
        int j = FROM == 1 ? j_L1(tid, e) : FROM == 2 ? j_L2(tid, e) : j_L3(tid, e);
        sm[pidx(j)] = a[e];
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 32; e++) {
        int j = TO == 1 ? j_L1(tid, e) : TO == 2 ? j_L2(tid, e) : j_L3(tid, e);
        a[e] = sm[pidx(j)];
    }
}

// ---------------------------------------------------------------- forward (L1 -> L3)
// input residues < 4q (canonical inputs are fine); output canonical [0,q)
BM_D void ntt_fwd(uint64_t a[32], uint64_t *sm, const PrimeK &P)
{
    const int tid = threadIdx.x;
    const uint64_t q = P.q, q2 = P.q2;
    // pass 1: stages s = 0..4 (t = 4096 .. 256); partner k + (16 >> s); twiddle index (1<<s) + (k >> (5-s))
#pragma unroll
    for (int s = 0; s < 5; s++) {
        const int half = 16 >> s;
#pragma unroll
        for (int k = 0; k < 32; k++) {
            if (k & half) continue;
            ulonglong2 w = ldtw(P.fwd + (1 << s) + (k >> (5 - s)));
            ct_bfly(a[k], a[k + half], w, q, q2);
        }
    }
    exchange<1, 2>(a, sm);
    // pass 2: stages s = 5..8 (t = 128 .. 16); element e = 16h + k, j = 256 B + 16 k + e_lo;
    // twiddle index (1<<s) + (j >> (13 - s)) = (1<<s) + (B << (s-5)) + (k >> (9 - s))
#pragma unroll
    for (int s = 5; s < 9; s++) {
        const int half = 8 >> (s - 5);
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int B = (tid + 256 * h) >> 4;
            ulonglong2 w[8];
#pragma unroll
            for (int i = 0; i < (1 << (s - 5)); i++) w[i] = ldtw(P.fwd + (1 << s) + (B << (s - 5)) + i);
#pragma unroll
            for (int k = 0; k < 16; k++) {
                if (k & half) continue;
                ct_bfly(a[16 * h + k], a[16 * h + k + half], w[k >> (9 - s)], q, q2);
            }
        }
    }
    exchange<2, 3>(a, sm);
    // pass 3: stages s = 9..12 (t = 8 .. 1); j = 16 G + k; twiddle (1<<s) + (G << (s-9)) + (k >> (13 - s))
#pragma unroll
    for (int s = 9; s < 13; s++) {
        const int half = 8 >> (s - 9);
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int G = tid + 256 * h;
            ulonglong2 w[8];
#pragma unroll
            for (int i = 0; i < (1 << (s - 9)); i++) w[i] = ldtw(P.fwd + (1 << s) + (G << (s - 9)) + i);
#pragma unroll
            for (int k = 0; k < 16; k++) {
                if (k & half) continue;
                ct_bfly(a[16 * h + k], a[16 * h + k + half], w[k >> (13 - s)], q, q2);
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 32; e++) a[e] = csub(csub(a[e], q2), q);
}

// ---------------------------------------------------------------- inverse (L3 -> L1)
// input residues < 2q; output canonical [0,q)
BM_D void ntt_inv(uint64_t a[32], uint64_t *sm, const PrimeK &P)
{
    const int tid = threadIdx.x;
    const uint64_t q = P.q, q2 = P.q2;
    // pass A: stages s = 12..9 on L3
#pragma unroll
    for (int s = 12; s >= 9; s--) {
        const int half = 8 >> (s - 9);
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int G = tid + 256 * h;
            ulonglong2 w[8];
#pragma unroll
            for (int i = 0; i < (1 << (s - 9)); i++) w[i] = ldtw(P.inv + (1 << s) + (G << (s - 9)) + i);
#pragma unroll
            for (int k = 0; k < 16; k++) {
                if (k & half) continue;
                gs_bfly(a[16 * h + k], a[16 * h + k + half], w[k >> (13 - s)], q, q2);
            }
        }
    }
    exchange<3, 2>(a, sm);
    // pass B: stages s = 8..5 on L2
#pragma unroll
    for (int s = 8; s >= 5; s--) {
        const int half = 8 >> (s - 5);
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int B = (tid + 256 * h) >> 4;
            ulonglong2 w[8];
#pragma unroll
            for (int i = 0; i < (1 << (s - 5)); i++) w[i] = ldtw(P.inv + (1 << s) + (B << (s - 5)) + i);
#pragma unroll
            for (int k = 0; k < 16; k++) {
                if (k & half) continue;
                gs_bfly(a[16 * h + k], a[16 * h + k + half], w[k >> (9 - s)], q, q2);
            }
        }
    }
    exchange<2, 1>(a, sm);
    // pass C: stages s = 4..1 on L1, then s = 0 with N^-1 folded in
#pragma unroll
    for (int s = 4; s >= 1; s--) {
        const int half = 16 >> s;
#pragma unroll
        for (int k = 0; k < 32; k++) {
            if (k & half) continue;
            ulonglong2 w = ldtw(P.inv + (1 << s) + (k >> (5 - s)));
            gs_bfly(a[k], a[k + half], w, q, q2);
        }
    }
#pragma unroll
    for (int k = 0; k < 16; k++) {
        uint64_t x = a[k], y = a[k + 16];
        a[k] = csub(shoup(x + y, P.ninv, q), q);
        a[k + 16] = csub(shoup(x - y + q2, P.ninv_w1, q), q);
    }
}

// NTT-domain automorphism sigma_g as an index map: NTT(sigma_g a)[j] = NTT(a)[perm_g(j)],
// perm_g(j) = brev13(((2 brev13(j) + 1) g mod 2N - 1) / 2).
BM_D int auto_perm(int j, uint32_t g)
{
    uint32_t e = 2u * (uint32_t)brev13(j) + 1u;
    e = (e * g) & (2u * N - 1u);
    return brev13((int)((e - 1u) >> 1));
}

// ================================================================== v2 (prime-specialised, 256 threads)
// exact x mod q for any x < 2^64 (Shoup with w = 1 and a final correction)
template <int PI> BM_D uint64_t reduce_full(uint64_t x, uint64_t one_p)
{
    constexpr uint64_t q = PrimeC<PI>::q;
    uint64_t r = x - mul_q<PI>(__umul64hi(x, one_p)); // [0, 2q)
    return r >= q ? r - q : r;
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
