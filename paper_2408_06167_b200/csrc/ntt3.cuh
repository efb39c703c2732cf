// ntt3.cuh -- NTT core v3: one 8192-point negacyclic transform per 512-thread CTA, 16
// coefficients per thread (K1 in SURVEY.md sec. 2.2).  Same transform as ntt.cuh (CT forward
// with psi^brev twiddles, GS inverse with N^-1 folded in; NTT(a)[j] = a(psi^(2 brev13(j)+1)))
// and the prime-specialised lazy arithmetic of ntt2.cuh.
//
// 13 stages = 3 register passes of 4 stages (two shared-memory transposes) + 1 stage done on
// lane pairs with warp shuffles.  Layouts (tid < 512, register index e < 16):
//   M1 "coefficient": a[k]      <-> j = tid + 512 k
//   M2:               a[k]      <-> j = 512 (tid>>5) + 32 k + (tid&31)
//   M3:               a[k]      <-> j = 32 (tid>>1) + 2 k + (tid&1)
//   M4 "evaluation":  a[2m + b] <-> j = 32 (tid>>1) + 4 m + 2 (tid&1) + b      (m < 8, b < 2)
// Forward: M1 -> s0..3 -> M2 -> s4..7 -> M3 -> s8..11 -> shuffle stage s12 -> M4.
// Inverse: M4 -> s12 (in registers) -> shuffle -> M3 -> s11..8 -> M2 -> s7..4 -> M1 -> s3..0.
// NTT-domain polynomials are stored in M4 order at pos(tid, 2m+b) = 1024 m + 2 tid + b, so every
// NTT-domain global access is a coalesced 16-byte vector per lane.
#pragma once
#include "ntt2.cuh"

namespace bm {
namespace v3 {

constexpr int T = 512; // threads per CTA
constexpr int E = 16;  // coefficients per thread

BM_D int j_M1(int tid, int k) { return tid + 512 * k; }
BM_D int j_M2(int tid, int k) { return 512 * (tid >> 5) + 32 * k + (tid & 31); }
BM_D int j_M3(int tid, int k) { return 32 * (tid >> 1) + 2 * k + (tid & 1); }
BM_D int j_M4(int tid, int e) { return 32 * (tid >> 1) + 4 * (e >> 1) + 2 * (tid & 1) + (e & 1); }
BM_D int pos_M4(int tid, int e) { return 1024 * (e >> 1) + 2 * tid + (e & 1); }

// Storage position of twiddle index k (k = 2^s + r, stage s) in the device tables.  Stages 0..8 are
// stored as indexed (their loads are warp-uniform or lane-contiguous); stages 9..11 (r = G 2^(s-8) + kk,
// G = tid >> 1) and 12 (r = 16 G + 2 m + odd) are stored in the order the 512-thread CTA loads them,
// kk-major / m-major, so every twiddle load of a warp is one contiguous 256-512 B run instead of 16
// strided sectors.  A bijection on [2^s, 2^(s+1)) per stage.
BM_HD int tw_pos(int k)
{
    int s = 0;
    while ((2 << s) <= k) s++;
    const int r = k - (1 << s);
    if (s <= 8) return k;
    if (s <= 11) return (1 << s) + (r & ((1 << (s - 8)) - 1)) * 256 + (r >> (s - 8));
    return 4096 + 512 * ((r >> 1) & 7) + 2 * (r >> 4) + (r & 1);
}

// Layout exchange through shared memory.  M2 and M3 partition j into per-warp 512-point regions
// (warp w owns j in [512 w, 512 w + 512)), so an M2 <-> M3 exchange stays inside one warp and only
// needs __syncwarp; exchanges with M1 span the CTA.  Hazards on the shared buffer: a CTA-wide
// write must wait for every warp's previous reads (__syncthreads before it); a warp-local write
// into region w only races with other warps' reads of region w, which only CTA-wide (M1) reads
// do, so xchg<3,2> (the inverse's first exchange, which may follow an M1 read) starts with a
// CTA barrier while xchg<2,3> (which always follows xchg<1,2>'s region-local reads) does not.
template <int FROM, int TO>
BM_D void xchg(uint64_t a[E], uint64_t *sm)
{
#if defined(BM_DIAG_XCHG) // tools/ntt_bench.cu diagnostic builds only (wrong results): 1 = barriers, no data; 2 = nothing
    if (BM_DIAG_XCHG == 1) { BM_SYNCTHREADS(); BM_SYNCTHREADS(); }
    return;
#endif
    const int tid = threadIdx.x;
    constexpr bool local_w = (FROM != 1);          // writes stay in the warp's region
    constexpr bool local_r = (TO != 1);            // reads stay in the warp's region
    if (FROM == 1 || (FROM == 3 && TO == 2)) BM_SYNCTHREADS();
    else BM_SYNCWARP();
#pragma unroll
    for (int k = 0; k < E; k++) {
        const int j = FROM == 1 ? j_M1(tid, k) : FROM == 2 ? j_M2(tid, k) : j_M3(tid, k);
        BM_CHECK(pidx(j) < SMEM_WORDS);
        sm[pidx(j)] = a[k];
    }
    if (local_w && local_r) BM_SYNCWARP();
    else BM_SYNCTHREADS();
#pragma unroll
    for (int k = 0; k < E; k++) {
        const int j = TO == 1 ? j_M1(tid, k) : TO == 2 ? j_M2(tid, k) : j_M3(tid, k);
        a[k] = sm[pidx(j)];
    }
}

BM_D uint64_t shfl1(uint64_t v) { return __shfl_xor_sync(0xffffffffu, v, 1); }

// ------------------------------------------------------------------ forward (M1 -> M4)
// CANON = false: outputs only reduced to [0, 2q) (q0, P; q1 stays canonical) for consumers that
// take lazy operands (Shoup products, sums that are reduced afterwards)
template <int PI, bool CANON = true> BM_D void fwd(uint64_t a[E], uint64_t *sm, const PrimeK &P)
{
    const int tid = threadIdx.x;
    // pass 1: s = 0..3, t = 512 (8 >> s); partner k + (8 >> s); twiddle (1<<s) + (k >> (4-s))
#pragma unroll
    for (int s = 0; s < 4; s++) {
        const int half = 8 >> s;
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & half) continue;
            ct4s<PI>(a[k], a[k + half], ldtw(P.fwd + (1 << s) + (k >> (4 - s))), s);
        }
    }
    xchg<1, 2>(a, sm);
    // pass 2: s = 4..7; twiddle (1<<s) + (B << (s-4)) + (k >> (8-s)), B = warp index (uniform per warp)
    {
        const int B = tid >> 5;
#pragma unroll
        for (int s = 4; s < 8; s++) {
            const int half = 8 >> (s - 4);
#pragma unroll
            for (int k = 0; k < E; k++) {
                if (k & half) continue;
                ct4s<PI>(a[k], a[k + half], ldtw(P.fwd + (1 << s) + (B << (s - 4)) + (k >> (8 - s))), s);
            }
        }
    }
    xchg<2, 3>(a, sm);
    // pass 3: s = 8..11; twiddle index (1<<s) + (G << (s-8)) + (k >> (12-s)), G = tid >> 1, stored at
    // (1<<s) + (k >> (12-s)) 256 + G (tw_pos)
    const int G = tid >> 1, odd = tid & 1;
#pragma unroll
    for (int s = 8; s < 12; s++) {
        const int half = 8 >> (s - 8);
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & half) continue;
            ct4s<PI>(a[k], a[k + half], ldtw(P.fwd + (1 << s) + ((k >> (12 - s)) << 8) + G), s);
        }
    }
    // stage 12 (t = 1) on lane pairs: the even lane takes butterflies k = 2m, the odd lane k = 2m+1
#pragma unroll
    for (int m = 0; m < 8; m++) {
        const uint64_t r = shfl1(odd ? a[2 * m] : a[2 * m + 1]);
        uint64_t x = odd ? r : a[2 * m], y = odd ? a[2 * m + 1] : r;
        ct4s<PI>(x, y, ldtw(P.fwd + 4096 + 512 * m + tid), 12);
        if (CANON || Q40<PI>) {
            a[2 * m] = reduce_bnd<PI>(x);
            a[2 * m + 1] = reduce_bnd<PI>(y);
        } else {
            a[2 * m] = reduce_lazy<Q40<PI> ? 0 : PI>(x);
            a[2 * m + 1] = reduce_lazy<Q40<PI> ? 0 : PI>(y);
        }
    }
}

// ------------------------------------------------------------------ inverse (M4 -> M1)
template <int PI> BM_D void inv(uint64_t a[E], uint64_t *sm, const PrimeK &P)
{
    const int tid = threadIdx.x;
    const int G = tid >> 1, odd = tid & 1;
    // stage 12 (first executed, st = 0): in-register pairs (j, j+1)
#pragma unroll
    for (int m = 0; m < 8; m++) gs4s<PI, 0>(a[2 * m], a[2 * m + 1], ldtw(P.inv + 4096 + 512 * m + tid));
    // back to M3: even lane keeps a[2m] and receives a[2m+1]; odd lane keeps a[2m+1]
#pragma unroll
    for (int m = 0; m < 8; m++) {
        const uint64_t r = shfl1(odd ? a[2 * m] : a[2 * m + 1]);
        if (odd) a[2 * m] = r;
        else a[2 * m + 1] = r;
    }
    // pass 3: s = 11..8 (st = 1..4)
#pragma unroll
    for (int s = 11; s >= 8; s--) {
        const int half = 8 >> (s - 8);
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & half) continue;
            const ulonglong2 w = ldtw(P.inv + (1 << s) + ((k >> (12 - s)) << 8) + G);
            switch (12 - s) {
            case 1: gs4s<PI, 1>(a[k], a[k + half], w); break;
            case 2: gs4s<PI, 2>(a[k], a[k + half], w); break;
            case 3: gs4s<PI, 3>(a[k], a[k + half], w); break;
            default: gs4s<PI, 4>(a[k], a[k + half], w); break;
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
                const ulonglong2 w = ldtw(P.inv + (1 << s) + (B << (s - 4)) + (k >> (8 - s)));
                switch (12 - s) {
                case 5: gs4s<PI, 5>(a[k], a[k + half], w); break;
                case 6: gs4s<PI, 6>(a[k], a[k + half], w); break;
                case 7: gs4s<PI, 7>(a[k], a[k + half], w); break;
                default: gs4s<PI, 8>(a[k], a[k + half], w); break;
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
            const ulonglong2 w = ldtw(P.inv + (1 << s) + (k >> (4 - s)));
            switch (12 - s) {
            case 9: gs4s<PI, 9>(a[k], a[k + half], w); break;
            case 10: gs4s<PI, 10>(a[k], a[k + half], w); break;
            default: gs4s<PI, 11>(a[k], a[k + half], w); break;
            }
        }
    }
    // s = 0 with N^-1 folded in; inputs < B q with B of stage 12
    constexpr uint64_t Bq = (Q40<PI> ? (4ull << 12) : 4ull) * PrimeC<PI>::q;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const uint64_t x = a[k], y = a[k + 8];
        a[k] = reduce_bnd<PI>(shoup4<PI>(x + y, P.ninv));
        a[k + 8] = reduce_bnd<PI>(shoup4<PI>(x - y + Bq, P.ninv_w1));
    }
}

BM_D void fwd_rt(uint64_t a[E], uint64_t *sm, const PrimeK &P, int pi)
{
    if (pi == 0) fwd<0>(a, sm, P);
    else if (pi == 1) fwd<1>(a, sm, P);
    else if (pi == 2) fwd<2>(a, sm, P);
    else fwd<3>(a, sm, P);
}
BM_D void inv_rt(uint64_t a[E], uint64_t *sm, const PrimeK &P, int pi)
{
    if (pi == 0) inv<0>(a, sm, P);
    else if (pi == 1) inv<1>(a, sm, P);
    else if (pi == 2) inv<2>(a, sm, P);
    else inv<3>(a, sm, P);
}

// ------------------------------------------------------------------ global <-> register helpers
BM_D ulonglong2 ldv(const uint64_t *p) { return __ldg(reinterpret_cast<const ulonglong2 *>(p)); }
BM_D void stv(uint64_t *p, uint64_t x, uint64_t y) { *reinterpret_cast<ulonglong2 *>(p) = make_ulonglong2(x, y); }

// NTT-domain (M4, storage pos_M4): 8 coalesced 16-byte vectors per thread
BM_D void load_eval(uint64_t a[E], const uint64_t *p)
{
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const ulonglong2 v = ldv(p + pos_M4(threadIdx.x, e));
        a[e] = v.x;
        a[e + 1] = v.y;
    }
}
BM_D void store_eval(uint64_t *p, const uint64_t a[E])
{
#pragma unroll
    for (int e = 0; e < E; e += 2) stv(p + pos_M4(threadIdx.x, e), a[e], a[e + 1]);
}
// coefficient domain (M1): coalesced 8-byte accesses
BM_D void load_coef(uint64_t a[E], const uint64_t *p)
{
#pragma unroll
    for (int k = 0; k < E; k++) a[k] = p[j_M1(threadIdx.x, k)];
}
BM_D void store_coef(uint64_t *p, const uint64_t a[E])
{
#pragma unroll
    for (int k = 0; k < E; k++) p[j_M1(threadIdx.x, k)] = a[k];
}
// stage an NTT-domain polynomial into shared memory indexed by NTT index j
BM_D void stage_by_j(uint64_t *sm, const uint64_t *p)
{
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const ulonglong2 v = ldv(p + pos_M4(threadIdx.x, e));
        sm[pidx(j_M4(threadIdx.x, e))] = v.x;
        sm[pidx(j_M4(threadIdx.x, e + 1))] = v.y;
    }
}

// Natural-order shared-memory storage of an NTT-domain polynomial (the resident operands of the
// rotation kernels): NTT index j (bit-reversed evaluation order) is stored at word npad(i), i.e.
// i + (i >> 4) with bank bit 0 toggled by bit 11, i = brev13(j) the natural index of its
// evaluation point.  The
// automorphism sigma_g maps natural index i to i g + (g - 1) / 2 mod N (odd g).  A 64-bit warp access
// is served per half-warp (16 lanes x 8 B = one 128-byte wavefront when the lanes hit 16 distinct
// 8-byte bank pairs): a half-warp's M4 elements differ in natural-index bits 5, 6, 7 and 11, and the
// (i >> 4) padding spreads bits 5..7 over 8 bank pairs while the bit-11 toggle of the bank's low bit
// separates the two halves -- so the M4 accesses AND every sigma_g gather take the minimum 2
// wavefronts (a model over all 13 Galois elements 5^(2^k); the j + (j >> 4) padding of the exchange
// buffer gives 4 and 6-7, plain i + (i >> 4) gives 4 and 4).  The map is a bijection onto
// [0, N + N/16).  j_M4's thread bits (1, 5..12) and element bits (0, 2..4) are disjoint, so
// i = nat_tid | nat_e with nat_e a constant (and bit 11 a thread bit).
BM_HD constexpr int brev13c(int x)
{
    int r = 0;
    for (int b = 0; b < 13; b++) r |= ((x >> b) & 1) << (12 - b);
    return r;
}
BM_D int nat_tid(int tid) { return brev13(32 * (tid >> 1) + 2 * (tid & 1)); }
BM_HD constexpr int nat_e(int e) { return brev13c(4 * (e >> 1) + (e & 1)); }
// word(i) = pad(T) ^ bit11(T) + pad(E), T = the natural-index bits a thread owns (0..7, 11), E = the
// element bits (8, 9, 10, 12): additive in the element part, so nat_at is a per-thread base plus
// an immediate offset (an XOR after the sum cost the ladder 2% in address arithmetic)
BM_HD constexpr int npad(int i)
{
    const int t = i & 0x8FF, e = i & 0x1700;
    return ((t + (t >> 4)) ^ ((t >> 11) & 1)) + (e + (e >> 4));
}
// word of this thread's element e (M4) / of the element sigma_g moves there
BM_D int nat_at(int ntid, int e) { return npad(ntid) + npad(nat_e(e)); }
// npad for a runtime index: the thread / element split of npad is only for immediates, and
// ((t + (t >> 4)) ^ b) + (e + (e >> 4)) = (i + (i >> 4)) ^ b with b = bit 11 of i, because e + (e >> 4)
// has bit 0 clear (so the bank-bit toggle commutes with adding it): 5 instructions per gather
BM_D int npad_rt(uint32_t i) { return (int)((i + (i >> 4)) ^ ((i >> 11) & 1u)); }
BM_D int nat_auto_i(uint32_t i, uint32_t g)
{
#ifdef BM_NPAD_SPLIT
    const int w = npad((int)((i * g + ((g - 1) >> 1)) & (N - 1)));
#else
    const int w = npad_rt((i * g + ((g - 1) >> 1)) & (N - 1));
#endif
    BM_CHECK(w >= 0 && w < SMEM_WORDS && (g & 1));
    return w;
}
BM_D int nat_auto(int ntid, int e, uint32_t g) { return nat_auto_i((uint32_t)(ntid | nat_e(e)), g); }
// natural index of element e when e is not a compile-time constant
BM_D uint32_t nat_i(int ntid, int e) { return (uint32_t)(ntid | brev13(4 * (e >> 1) + (e & 1))); }
BM_D void stage_nat(uint64_t *sm, const uint64_t *p)
{
    const int nt = nat_tid(threadIdx.x);
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const ulonglong2 v = ldv(p + pos_M4(threadIdx.x, e));
        sm[nat_at(nt, e)] = v.x;
        sm[nat_at(nt, e + 1)] = v.y;
    }
}

} // namespace v3
} // namespace bm
