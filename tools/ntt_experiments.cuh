// ntt_experiments.cuh -- DIAGNOSTIC ONLY (tools/ntt_bench.cu v5 / v6), not part of the
// library: the paired-transform cores measured this round and dropped.
//   v5 fwd2x / inv2x: two integer-prime polynomials interleaved stage by stage (shared twiddle loads, one
//      barrier per exchange for both): 3.03 vs 3.08 butterflies/clk/SM for q0 alone -- no gain.
//   v6 fwd_h / inv_h: an integer-prime transform interleaved with a q1 transform on the FP64 pipe:
//      3.45 butterflies/clk/SM over both, against 3.69 for the two run one after the other.
#pragma once
#include "../paper_2408_06167_b200/csrc/ntt3f.cuh"

namespace bm {
namespace v3 {

// ------------------------------------------------------------------ two polynomials at once
// The same transforms on two independent polynomials a, b of one prime (e.g. the ladder's two
// key-switch components): each twiddle is loaded once for both, each exchange writes both before one
// barrier, and the two butterfly streams interleave (one poly's shared-memory traffic overlaps the
// other's arithmetic).  Exchange buffers smA, smB (SMEM_WORDS each).
template <int FROM, int TO>
BM_D void xchg2(uint64_t a[E], uint64_t b[E], uint64_t *smA, uint64_t *smB)
{
    const int tid = threadIdx.x;
    constexpr bool local_w = (FROM != 1), local_r = (TO != 1);
    if (FROM == 1 || (FROM == 3 && TO == 2)) BM_SYNCTHREADS();
    else BM_SYNCWARP();
#pragma unroll
    for (int k = 0; k < E; k++) {
        const int j = FROM == 1 ? j_M1(tid, k) : FROM == 2 ? j_M2(tid, k) : j_M3(tid, k);
        smA[pidx(j)] = a[k];
        smB[pidx(j)] = b[k];
    }
    if (local_w && local_r) BM_SYNCWARP();
    else BM_SYNCTHREADS();
#pragma unroll
    for (int k = 0; k < E; k++) {
        const int j = TO == 1 ? j_M1(tid, k) : TO == 2 ? j_M2(tid, k) : j_M3(tid, k);
        a[k] = smA[pidx(j)];
        b[k] = smB[pidx(j)];
    }
}

template <int PI, bool CANON = true>
BM_D void fwd2x(uint64_t a[E], uint64_t b[E], uint64_t *smA, uint64_t *smB, const PrimeK &P)
{
    const int tid = threadIdx.x;
#pragma unroll
    for (int s = 0; s < 4; s++) {
        const int half = 8 >> s;
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & half) continue;
            const ulonglong2 w = ldtw(P.fwd + (1 << s) + (k >> (4 - s)));
            ct4s<PI>(a[k], a[k + half], w, s);
            ct4s<PI>(b[k], b[k + half], w, s);
        }
    }
    xchg2<1, 2>(a, b, smA, smB);
    {
        const int B = tid >> 5;
#pragma unroll
        for (int s = 4; s < 8; s++) {
            const int half = 8 >> (s - 4);
#pragma unroll
            for (int k = 0; k < E; k++) {
                if (k & half) continue;
                const ulonglong2 w = ldtw(P.fwd + (1 << s) + (B << (s - 4)) + (k >> (8 - s)));
                ct4s<PI>(a[k], a[k + half], w, s);
                ct4s<PI>(b[k], b[k + half], w, s);
            }
        }
    }
    xchg2<2, 3>(a, b, smA, smB);
    const int G = tid >> 1, odd = tid & 1;
#pragma unroll
    for (int s = 8; s < 12; s++) {
        const int half = 8 >> (s - 8);
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & half) continue;
            const ulonglong2 w = ldtw(P.fwd + (1 << s) + ((k >> (12 - s)) << 8) + G);
            ct4s<PI>(a[k], a[k + half], w, s);
            ct4s<PI>(b[k], b[k + half], w, s);
        }
    }
#pragma unroll
    for (int m = 0; m < 8; m++) {
        const ulonglong2 w = ldtw(P.fwd + 4096 + 512 * m + tid);
        const uint64_t ra = shfl1(odd ? a[2 * m] : a[2 * m + 1]), rb = shfl1(odd ? b[2 * m] : b[2 * m + 1]);
        uint64_t xa = odd ? ra : a[2 * m], ya = odd ? a[2 * m + 1] : ra;
        uint64_t xb = odd ? rb : b[2 * m], yb = odd ? b[2 * m + 1] : rb;
        ct4s<PI>(xa, ya, w, 12);
        ct4s<PI>(xb, yb, w, 12);
        if (CANON || Q40<PI>) {
            a[2 * m] = reduce_bnd<PI>(xa), a[2 * m + 1] = reduce_bnd<PI>(ya);
            b[2 * m] = reduce_bnd<PI>(xb), b[2 * m + 1] = reduce_bnd<PI>(yb);
        } else {
            a[2 * m] = reduce_lazy<Q40<PI> ? 0 : PI>(xa), a[2 * m + 1] = reduce_lazy<Q40<PI> ? 0 : PI>(ya);
            b[2 * m] = reduce_lazy<Q40<PI> ? 0 : PI>(xb), b[2 * m + 1] = reduce_lazy<Q40<PI> ? 0 : PI>(yb);
        }
    }
}

template <int PI> BM_D void inv2x(uint64_t a[E], uint64_t b[E], uint64_t *smA, uint64_t *smB, const PrimeK &P)
{
    const int tid = threadIdx.x;
    const int G = tid >> 1, odd = tid & 1;
#pragma unroll
    for (int m = 0; m < 8; m++) {
        const ulonglong2 w = ldtw(P.inv + 4096 + 512 * m + tid);
        gs4s<PI, 0>(a[2 * m], a[2 * m + 1], w);
        gs4s<PI, 0>(b[2 * m], b[2 * m + 1], w);
    }
#pragma unroll
    for (int m = 0; m < 8; m++) {
        const uint64_t ra = shfl1(odd ? a[2 * m] : a[2 * m + 1]), rb = shfl1(odd ? b[2 * m] : b[2 * m + 1]);
        if (odd) a[2 * m] = ra, b[2 * m] = rb;
        else a[2 * m + 1] = ra, b[2 * m + 1] = rb;
    }
#pragma unroll
    for (int s = 11; s >= 8; s--) {
        const int half = 8 >> (s - 8);
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & half) continue;
            const ulonglong2 w = ldtw(P.inv + (1 << s) + ((k >> (12 - s)) << 8) + G);
            switch (12 - s) {
            case 1: gs4s<PI, 1>(a[k], a[k + half], w); gs4s<PI, 1>(b[k], b[k + half], w); break;
            case 2: gs4s<PI, 2>(a[k], a[k + half], w); gs4s<PI, 2>(b[k], b[k + half], w); break;
            case 3: gs4s<PI, 3>(a[k], a[k + half], w); gs4s<PI, 3>(b[k], b[k + half], w); break;
            default: gs4s<PI, 4>(a[k], a[k + half], w); gs4s<PI, 4>(b[k], b[k + half], w); break;
            }
        }
    }
    xchg2<3, 2>(a, b, smA, smB);
    {
        const int B = tid >> 5;
#pragma unroll
        for (int s = 7; s >= 4; s--) {
            const int half = 8 >> (s - 4);
#pragma unroll
            for (int k = 0; k < E; k++) {
                if (k & half) continue;
                const ulonglong2 w = ldtw(P.inv + (1 << s) + (B << (s - 4)) + (k >> (8 - s)));
                switch (12 - s) {
                case 5: gs4s<PI, 5>(a[k], a[k + half], w); gs4s<PI, 5>(b[k], b[k + half], w); break;
                case 6: gs4s<PI, 6>(a[k], a[k + half], w); gs4s<PI, 6>(b[k], b[k + half], w); break;
                case 7: gs4s<PI, 7>(a[k], a[k + half], w); gs4s<PI, 7>(b[k], b[k + half], w); break;
                default: gs4s<PI, 8>(a[k], a[k + half], w); gs4s<PI, 8>(b[k], b[k + half], w); break;
                }
            }
        }
    }
    xchg2<2, 1>(a, b, smA, smB);
#pragma unroll
    for (int s = 3; s >= 1; s--) {
        const int half = 8 >> s;
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & half) continue;
            const ulonglong2 w = ldtw(P.inv + (1 << s) + (k >> (4 - s)));
            switch (12 - s) {
            case 9: gs4s<PI, 9>(a[k], a[k + half], w); gs4s<PI, 9>(b[k], b[k + half], w); break;
            case 10: gs4s<PI, 10>(a[k], a[k + half], w); gs4s<PI, 10>(b[k], b[k + half], w); break;
            default: gs4s<PI, 11>(a[k], a[k + half], w); gs4s<PI, 11>(b[k], b[k + half], w); break;
            }
        }
    }
    constexpr uint64_t Bq = (Q40<PI> ? (4ull << 12) : 4ull) * PrimeC<PI>::q;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const uint64_t xa = a[k], ya = a[k + 8], xb = b[k], yb = b[k + 8];
        a[k] = reduce_bnd<PI>(shoup4<PI>(xa + ya, P.ninv));
        a[k + 8] = reduce_bnd<PI>(shoup4<PI>(xa - ya + Bq, P.ninv_w1));
        b[k] = reduce_bnd<PI>(shoup4<PI>(xb + yb, P.ninv));
        b[k + 8] = reduce_bnd<PI>(shoup4<PI>(xb - yb + Bq, P.ninv_w1));
    }
}

// ------------------------------------------------------------------ hybrid pairs: an integer-prime transform
// (FMA pipe) interleaved with a q1/q2 transform on the FP64 pipe, stage by stage, one exchange barrier
// for both (ntt3.cuh xchg2): the two pipes work at once instead of one after the other.
// a: prime PI (ntt3.cuh arithmetic, tables P), b: prime PF on the FP64 pipe (tables twf, ninvf, ninv_w1f)
template <int PI, bool CANON, int PF>
BM_D void fwd_h(uint64_t a[E], uint64_t b[E], uint64_t *smA, uint64_t *smB, const PrimeK &P, const ulonglong2 *twf)
{
    const int tid = threadIdx.x;
#pragma unroll
    for (int e = 0; e < E; e++) b[e] = as_u(from_u(b[e]));
#pragma unroll
    for (int s = 0; s < 4; s++) {
        const int half = 8 >> s;
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & half) continue;
            ct4s<PI>(a[k], a[k + half], ldtw(P.fwd + (1 << s) + (k >> (4 - s))), s);
            ct_f<PF>(b[k], b[k + half], ldtw(twf + (1 << s) + (k >> (4 - s))));
        }
    }
    xchg2<1, 2>(a, b, smA, smB);
    {
        const int B = tid >> 5;
#pragma unroll
        for (int s = 4; s < 8; s++) {
            const int half = 8 >> (s - 4);
#pragma unroll
            for (int k = 0; k < E; k++) {
                if (k & half) continue;
                const int t = (1 << s) + (B << (s - 4)) + (k >> (8 - s));
                ct4s<PI>(a[k], a[k + half], ldtw(P.fwd + t), s);
                ct_f<PF>(b[k], b[k + half], ldtw(twf + t));
            }
        }
    }
    xchg2<2, 3>(a, b, smA, smB);
    const int G = tid >> 1, odd = tid & 1;
#pragma unroll
    for (int s = 8; s < 12; s++) {
        const int half = 8 >> (s - 8);
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & half) continue;
            const int t = (1 << s) + ((k >> (12 - s)) << 8) + G;
            ct4s<PI>(a[k], a[k + half], ldtw(P.fwd + t), s);
            ct_f<PF>(b[k], b[k + half], ldtw(twf + t));
        }
    }
#pragma unroll
    for (int m = 0; m < 8; m++) {
        const int t = 4096 + 512 * m + tid;
        const uint64_t ra = shfl1(odd ? a[2 * m] : a[2 * m + 1]), rb = shfl1(odd ? b[2 * m] : b[2 * m + 1]);
        uint64_t xa = odd ? ra : a[2 * m], ya = odd ? a[2 * m + 1] : ra;
        uint64_t xb = odd ? rb : b[2 * m], yb = odd ? b[2 * m + 1] : rb;
        ct4s<PI>(xa, ya, ldtw(P.fwd + t), 12);
        ct_f<PF>(xb, yb, ldtw(twf + t));
        if (CANON || Q40<PI>) {
            a[2 * m] = reduce_bnd<PI>(xa), a[2 * m + 1] = reduce_bnd<PI>(ya);
        } else {
            a[2 * m] = reduce_lazy<Q40<PI> ? 0 : PI>(xa), a[2 * m + 1] = reduce_lazy<Q40<PI> ? 0 : PI>(ya);
        }
        b[2 * m] = canon_f<PF>(as_d(xb)), b[2 * m + 1] = canon_f<PF>(as_d(yb));
    }
}

template <int PI, int PF>
BM_D void inv_h(uint64_t a[E], uint64_t b[E], uint64_t *smA, uint64_t *smB, const PrimeK &P, const ulonglong2 *twf,
                ulonglong2 ninvf, ulonglong2 ninv_w1f)
{
    const int tid = threadIdx.x;
    const int G = tid >> 1, odd = tid & 1;
#pragma unroll
    for (int e = 0; e < E; e++) b[e] = as_u(from_u(b[e]));
#pragma unroll
    for (int m = 0; m < 8; m++) {
        const int t = 4096 + 512 * m + tid;
        gs4s<PI, 0>(a[2 * m], a[2 * m + 1], ldtw(P.inv + t));
        gs_f<PF, 0>(b[2 * m], b[2 * m + 1], ldtw(twf + t));
    }
#pragma unroll
    for (int m = 0; m < 8; m++) {
        const uint64_t ra = shfl1(odd ? a[2 * m] : a[2 * m + 1]), rb = shfl1(odd ? b[2 * m] : b[2 * m + 1]);
        if (odd) a[2 * m] = ra, b[2 * m] = rb;
        else a[2 * m + 1] = ra, b[2 * m + 1] = rb;
    }
#pragma unroll
    for (int s = 11; s >= 8; s--) {
        const int half = 8 >> (s - 8);
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & half) continue;
            const int t = (1 << s) + ((k >> (12 - s)) << 8) + G;
            const ulonglong2 w = ldtw(P.inv + t), wf = ldtw(twf + t);
            switch (12 - s) {
            case 1: gs4s<PI, 1>(a[k], a[k + half], w); gs_f<PF, 1>(b[k], b[k + half], wf); break;
            case 2: gs4s<PI, 2>(a[k], a[k + half], w); gs_f<PF, 2>(b[k], b[k + half], wf); break;
            case 3: gs4s<PI, 3>(a[k], a[k + half], w); gs_f<PF, 3>(b[k], b[k + half], wf); break;
            default: gs4s<PI, 4>(a[k], a[k + half], w); gs_f<PF, 4>(b[k], b[k + half], wf); break;
            }
        }
    }
    xchg2<3, 2>(a, b, smA, smB);
    {
        const int B = tid >> 5;
#pragma unroll
        for (int s = 7; s >= 4; s--) {
            const int half = 8 >> (s - 4);
#pragma unroll
            for (int k = 0; k < E; k++) {
                if (k & half) continue;
                const int t = (1 << s) + (B << (s - 4)) + (k >> (8 - s));
                const ulonglong2 w = ldtw(P.inv + t), wf = ldtw(twf + t);
                switch (12 - s) {
                case 5: gs4s<PI, 5>(a[k], a[k + half], w); gs_f<PF, 5>(b[k], b[k + half], wf); break;
                case 6: gs4s<PI, 6>(a[k], a[k + half], w); gs_f<PF, 6>(b[k], b[k + half], wf); break;
                case 7: gs4s<PI, 7>(a[k], a[k + half], w); gs_f<PF, 7>(b[k], b[k + half], wf); break;
                default: gs4s<PI, 8>(a[k], a[k + half], w); gs_f<PF, 8>(b[k], b[k + half], wf); break;
                }
            }
        }
    }
    xchg2<2, 1>(a, b, smA, smB);
#pragma unroll
    for (int s = 3; s >= 1; s--) {
        const int half = 8 >> s;
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & half) continue;
            const int t = (1 << s) + (k >> (4 - s));
            const ulonglong2 w = ldtw(P.inv + t), wf = ldtw(twf + t);
            switch (12 - s) {
            case 9: gs4s<PI, 9>(a[k], a[k + half], w); gs_f<PF, 9>(b[k], b[k + half], wf); break;
            case 10: gs4s<PI, 10>(a[k], a[k + half], w); gs_f<PF, 10>(b[k], b[k + half], wf); break;
            default: gs4s<PI, 11>(a[k], a[k + half], w); gs_f<PF, 11>(b[k], b[k + half], wf); break;
            }
        }
    }
    constexpr uint64_t Bq = (Q40<PI> ? (4ull << 12) : 4ull) * PrimeC<PI>::q;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const uint64_t xa = a[k], ya = a[k + 8];
        const double xb = as_d(b[k]), yb = as_d(b[k + 8]);
        a[k] = reduce_bnd<PI>(shoup4<PI>(xa + ya, P.ninv));
        a[k + 8] = reduce_bnd<PI>(shoup4<PI>(xa - ya + Bq, P.ninv_w1));
        b[k] = canon_f<PF>(mulw<PF>(xb + yb, ninvf));
        b[k + 8] = canon_f<PF>(mulw<PF>(xb - yb, ninv_w1f));
    }
}


// ================================================================== v7: 1,024 threads x 8 coefficients (experiment)
// More warps per SM (32 instead of 16) at 8 coefficients per thread (fits 64 registers), for latency
// hiding; 3 register passes of 3 stages + one lane-pair shuffle stage, 3 exchanges per transform (two
// CTA-wide, one warp-local) against v3's 2.  Twiddles from NATURAL-order tables (index k at k).
// Layouts (w = warp, l = lane, k < 8):
//   J1: j = tid + 1024 k                                   (k <-> bits 10..12)
//   J2: j = (w & 3) | l << 2 | k << 7 | (w >> 2) << 10     (k <-> bits 7..9; warp region: bits 2..9)
//   J3: j = (w & 3) | (l & 3) << 2 | k << 4 | (l >> 2) << 7 | (w >> 2) << 10   (k <-> bits 4..6; same region)
//   J4: j = (l & 1) | k << 1 | (l >> 1) << 4 | w << 8      (k <-> bits 1..3)
//   J5 (after stage 12): a[2m + b] <-> j = b | (2m + (l & 1)) << 1 | (l >> 1) << 4 | w << 8
namespace x10 {
constexpr int T10 = 1024, E8 = 8;
BM_D int J1(int t, int k) { return t + 1024 * k; }
BM_D int J2(int t, int k) { const int w = t >> 5, l = t & 31; return (w & 3) | (l << 2) | (k << 7) | ((w >> 2) << 10); }
BM_D int J3(int t, int k)
{
    const int w = t >> 5, l = t & 31;
    return (w & 3) | ((l & 3) << 2) | (k << 4) | ((l >> 2) << 7) | ((w >> 2) << 10);
}
BM_D int J4(int t, int k) { const int w = t >> 5, l = t & 31; return (l & 1) | (k << 1) | ((l >> 1) << 4) | (w << 8); }
BM_D int J5(int t, int e)
{
    const int w = t >> 5, l = t & 31;
    return (e & 1) | ((2 * (e >> 1) + (l & 1)) << 1) | ((l >> 1) << 4) | (w << 8);
}
template <int L> BM_D int J(int t, int k) { return L == 1 ? J1(t, k) : L == 2 ? J2(t, k) : L == 3 ? J3(t, k) : J4(t, k); }

template <int FROM, int TO, bool WARP> BM_D void xch(uint64_t a[E8], uint64_t *sm)
{
    const int t = threadIdx.x;
    if (WARP) __syncwarp();
    else __syncthreads();
#pragma unroll
    for (int k = 0; k < E8; k++) sm[pidx(J<FROM>(t, k))] = a[k];
    if (WARP) __syncwarp();
    else __syncthreads();
#pragma unroll
    for (int k = 0; k < E8; k++) a[k] = sm[pidx(J<TO>(t, k))];
}

// one register pass of 3 forward stages s0, s0+1, s0+2 in layout L (stage s pairs bit 12 - s <-> k bit 2 - (s - s0))
template <int PI, int L, int S0> BM_D void fpass(uint64_t a[E8], const ulonglong2 *tw)
{
    const int t = threadIdx.x;
#pragma unroll
    for (int s = S0; s < S0 + 3; s++) {
        const int half = 4 >> (s - S0);
#pragma unroll
        for (int k = 0; k < E8; k++) {
            if (k & half) continue;
            const int jl = J<L>(t, k);
            ct4s<PI>(a[k], a[k + half], __ldg(tw + (1 << s) + (jl >> (13 - s))), s);
        }
    }
}
template <int PI, int L, int S0, int ST0> BM_D void ipass(uint64_t a[E8], const ulonglong2 *tw)
{
    const int t = threadIdx.x;
#pragma unroll
    for (int s = S0 + 2; s >= S0; s--) {
        const int half = 4 >> (s - S0);
#pragma unroll
        for (int k = 0; k < E8; k++) {
            if (k & half) continue;
            const int jl = J<L>(t, k);
            const ulonglong2 w = __ldg(tw + (1 << s) + (jl >> (13 - s)));
            constexpr int dummy = 0;
            (void)dummy;
            switch (12 - s) {
            case 1: gs4s<PI, 1>(a[k], a[k + half], w); break;
            case 2: gs4s<PI, 2>(a[k], a[k + half], w); break;
            case 3: gs4s<PI, 3>(a[k], a[k + half], w); break;
            case 4: gs4s<PI, 4>(a[k], a[k + half], w); break;
            case 5: gs4s<PI, 5>(a[k], a[k + half], w); break;
            case 6: gs4s<PI, 6>(a[k], a[k + half], w); break;
            case 7: gs4s<PI, 7>(a[k], a[k + half], w); break;
            case 8: gs4s<PI, 8>(a[k], a[k + half], w); break;
            case 9: gs4s<PI, 9>(a[k], a[k + half], w); break;
            case 10: gs4s<PI, 10>(a[k], a[k + half], w); break;
            default: gs4s<PI, 11>(a[k], a[k + half], w); break;
            }
        }
    }
}

template <int PI> BM_D void fwd10(uint64_t a[E8], uint64_t *sm, const ulonglong2 *tw)
{
    const int t = threadIdx.x, odd = t & 1;
    fpass<PI, 1, 0>(a, tw);
    xch<1, 2, false>(a, sm);
    fpass<PI, 2, 3>(a, tw);
    xch<2, 3, true>(a, sm);
    fpass<PI, 3, 6>(a, tw);
    xch<3, 4, false>(a, sm);
    fpass<PI, 4, 9>(a, tw);
#pragma unroll
    for (int m = 0; m < 4; m++) { // stage 12 on lane pairs: even lane k = 2m, odd lane k = 2m + 1
        const uint64_t r = __shfl_xor_sync(0xffffffffu, odd ? a[2 * m] : a[2 * m + 1], 1);
        uint64_t x = odd ? r : a[2 * m], y = odd ? a[2 * m + 1] : r;
        const int jl = J4(t, 2 * m + odd) & ~1;
        ct4s<PI>(x, y, __ldg(tw + 4096 + (jl >> 1)), 12);
        a[2 * m] = reduce_bnd<PI>(x);
        a[2 * m + 1] = reduce_bnd<PI>(y);
    }
}

template <int PI> BM_D void inv10(uint64_t a[E8], uint64_t *sm, const ulonglong2 *tw, ulonglong2 ninv, ulonglong2 ninv_w1)
{
    const int t = threadIdx.x, odd = t & 1;
#pragma unroll
    for (int m = 0; m < 4; m++) gs4s<PI, 0>(a[2 * m], a[2 * m + 1], __ldg(tw + 4096 + (J5(t, 2 * m) >> 1)));
#pragma unroll
    for (int m = 0; m < 4; m++) {
        const uint64_t r = __shfl_xor_sync(0xffffffffu, odd ? a[2 * m] : a[2 * m + 1], 1);
        if (odd) a[2 * m] = r;
        else a[2 * m + 1] = r;
    }
    ipass<PI, 4, 9, 1>(a, tw);
    xch<4, 3, false>(a, sm);
    ipass<PI, 3, 6, 4>(a, tw);
    xch<3, 2, true>(a, sm);
    ipass<PI, 2, 3, 7>(a, tw);
    xch<2, 1, false>(a, sm);
    // stages 2, 1 in J1 (k bits 1, 0), then stage 0 (k bit 2) with N^-1 folded in
#pragma unroll
    for (int s = 2; s >= 1; s--) {
        const int half = 4 >> s;
#pragma unroll
        for (int k = 0; k < E8; k++) {
            if (k & half) continue;
            const ulonglong2 w = __ldg(tw + (1 << s) + (J1(t, k) >> (13 - s)));
            if (s == 2) gs4s<PI, 10>(a[k], a[k + half], w);
            else gs4s<PI, 11>(a[k], a[k + half], w);
        }
    }
    constexpr uint64_t Bq = (Q40<PI> ? (4ull << 12) : 4ull) * PrimeC<PI>::q;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const uint64_t x = a[k], y = a[k + 4];
        a[k] = reduce_bnd<PI>(shoup4<PI>(x + y, ninv));
        a[k + 4] = reduce_bnd<PI>(shoup4<PI>(x - y + Bq, ninv_w1));
    }
}
} // namespace x10
} // namespace v3
} // namespace bm
