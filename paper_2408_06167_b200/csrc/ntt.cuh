// ntt.cuh -- register-blocked negacyclic NTT / INTT of one 8192-coefficient u64 polynomial
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
#include "bm_common.cuh"

namespace bm {

constexpr int NTT_THREADS = 256;
constexpr int SMEM_WORDS = N + N / 16; // 8704 u64 = 69,632 B

BM_D int pidx(int j) { return j + (j >> 4); }

BM_D ulonglong2 ldtw(const ulonglong2 *p) { return __ldg(p); }

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
BM_D int brev13(int x) { return (int)(__brev((unsigned)x) >> 19); }
BM_D int auto_perm(int j, uint32_t g)
{
    uint32_t e = 2u * (uint32_t)brev13(j) + 1u;
    e = (e * g) & (2u * N - 1u);
    return brev13((int)((e - 1u) >> 1));
}

} // namespace bm
