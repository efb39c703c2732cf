// bm_common.cuh -- product-side shared definitions (host + device).
// Nothing here is shared with oracle/; the oracle implements the same definitions
// independently and the tests compare the two.
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>
#include "blindmatch.h"

#define BM_HD __host__ __device__ __forceinline__
#define BM_D __device__ __forceinline__

// Debug builds (the sanitizer substitute; never the product):
//  BM_DEBUG_CHECKS: device-side bounds checks (shared-memory words, output rows, tables) that trap;
//  BM_DEBUG_JITTER: every CTA / warp barrier and cluster barrier is surrounded by a per-thread
//    pseudo-random spin of up to ~2000 cycles, so warps, lanes and cluster ranks reach each phase in
//    shuffled orders -- a missing barrier then shows up as a result that differs from the oracle.
#ifdef BM_DEBUG_CHECKS
#include <cstdio>
#define BM_CHECK(c)                                                                                   \
    do {                                                                                             \
        if (!(c)) {                                                                                  \
            printf("BM_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x, \
                   (int)threadIdx.x, #c);                                                            \
            __trap();                                                                                \
        }                                                                                            \
    } while (0)
#else
#define BM_CHECK(c) \
    do {            \
    } while (0)
#endif
#ifdef BM_DEBUG_JITTER
__device__ __forceinline__ void bm_jitter()
{
    unsigned x = (unsigned)clock64() ^ (threadIdx.x * 2654435761u) ^ (blockIdx.x * 40503u);
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    const long long t0 = clock64(), n = (long long)(x & 2047u);
    while (clock64() - t0 < n) {
    }
}
#define BM_SYNCTHREADS()  \
    do {                  \
        bm_jitter();      \
        __syncthreads();  \
        bm_jitter();      \
    } while (0)
#define BM_SYNCWARP()    \
    do {                 \
        bm_jitter();     \
        __syncwarp();    \
        bm_jitter();     \
    } while (0)
#else
#define bm_jitter() \
    do {            \
    } while (0)
#define BM_SYNCTHREADS() __syncthreads()
#define BM_SYNCWARP() __syncwarp()
#endif

namespace bm {

constexpr int N = BM_N;        // ring degree ("N = 8,192")
constexpr int LOGN = BM_LOGN;
constexpr int SLOTS = BM_SLOTS;

// BASELINE.json configs[0]: largest primes below 2^58, 2^40, 2^60 with q = 1 mod 2^14.
// bm_params_init re-verifies primality and the NTT condition at run time.
constexpr uint64_t Q0 = 288230376150876161ull;  // 2^58 - 835583
constexpr uint64_t Q1 = 1099511480321ull;       // 2^40 - 147455
constexpr uint64_t QP = 1152921504606830593ull; // 2^60 - 16383
// f3 (server-side query expansion): the chain extended by one level,
// q2 = the largest prime below q1 with q2 = 1 mod 2^14 (reading R24)
constexpr uint64_t Q2 = 1099510890497ull;       // 2^40 - 737279 = 2^40 - 45 2^14 + 1

// Purposes of the ChaCha20 random streams (reading R14).
enum : uint32_t {
    P_SK = 1, P_PK_A = 2, P_PK_E = 3, P_RLK_A = 4, P_RLK_E = 5, P_GK_A = 6, P_GK_E = 7,
    P_ENC_U = 8, P_ENC_E0 = 9, P_ENC_E1 = 10,
    P_GK1_A = 11, P_GK1_E = 12, // f3/f4/f1: level-1 Galois keys
    P_RLK2_A = 13, P_RLK2_E = 14 // f1: 3-digit relinearisation key at level 2
};

// ---------------------------------------------------------------- ChaCha20 (RFC 8439 sec. 2.3)
BM_HD uint32_t rotl32(uint32_t x, int n) { return (x << n) | (x >> (32 - n)); }

#define BM_QR(a, b, c, d)                      \
    a += b; d ^= a; d = rotl32(d, 16);         \
    c += d; b ^= c; b = rotl32(b, 12);         \
    a += b; d ^= a; d = rotl32(d, 8);          \
    c += d; b ^= c; b = rotl32(b, 7);

// Stream key/nonce of (seed, purpose, object, sub): key = {seed lo, seed hi, purpose, kx[0..4]},
// nonce = {obj lo, obj hi, sub}; the 32-bit block counter indexes 8 u64 draws per block.
// kx: 160 bits of key extension -- zero in the seeded (test / reproducibility) mode, where the
// streams are those of DESIGN.md reading R14 and the oracle; getrandom() output in the default
// OS-entropy mode (bm_rng_mode), so keys carry 224 bits of entropy and every encryption call is
// keyed afresh.
struct Stream {
    uint32_t k0, k1, k2, n0, n1, n2;
    uint32_t kx[5];
};
BM_HD Stream make_stream(uint64_t seed, uint32_t purpose, uint64_t obj, uint32_t sub, const uint32_t *kx = nullptr)
{
    Stream s;
    s.k0 = (uint32_t)seed; s.k1 = (uint32_t)(seed >> 32); s.k2 = purpose;
    s.n0 = (uint32_t)obj; s.n1 = (uint32_t)(obj >> 32); s.n2 = sub;
    for (int i = 0; i < 5; i++) s.kx[i] = kx ? kx[i] : 0u;
    return s;
}

// 8 u64 draws of block `ctr`: out[i] = word[2i] | word[2i+1] << 32
BM_HD void chacha_draws(const Stream &st, uint32_t ctr, uint64_t out[8])
{
    uint32_t x0 = 0x61707865u, x1 = 0x3320646eu, x2 = 0x79622d32u, x3 = 0x6b206574u;
    uint32_t x4 = st.k0, x5 = st.k1, x6 = st.k2, x7 = st.kx[0], x8 = st.kx[1], x9 = st.kx[2], x10 = st.kx[3],
             x11 = st.kx[4];
    uint32_t x12 = ctr, x13 = st.n0, x14 = st.n1, x15 = st.n2;
#pragma unroll
    for (int r = 0; r < 10; r++) {
        BM_QR(x0, x4, x8, x12) BM_QR(x1, x5, x9, x13) BM_QR(x2, x6, x10, x14) BM_QR(x3, x7, x11, x15)
        BM_QR(x0, x5, x10, x15) BM_QR(x1, x6, x11, x12) BM_QR(x2, x7, x8, x13) BM_QR(x3, x4, x9, x14)
    }
    x0 += 0x61707865u; x1 += 0x3320646eu; x2 += 0x79622d32u; x3 += 0x6b206574u;
    x4 += st.k0; x5 += st.k1; x6 += st.k2;
    x7 += st.kx[0]; x8 += st.kx[1]; x9 += st.kx[2]; x10 += st.kx[3]; x11 += st.kx[4];
    x12 += ctr; x13 += st.n0; x14 += st.n1; x15 += st.n2;
    out[0] = (uint64_t)x0 | ((uint64_t)x1 << 32);
    out[1] = (uint64_t)x2 | ((uint64_t)x3 << 32);
    out[2] = (uint64_t)x4 | ((uint64_t)x5 << 32);
    out[3] = (uint64_t)x6 | ((uint64_t)x7 << 32);
    out[4] = (uint64_t)x8 | ((uint64_t)x9 << 32);
    out[5] = (uint64_t)x10 | ((uint64_t)x11 << 32);
    out[6] = (uint64_t)x12 | ((uint64_t)x13 << 32);
    out[7] = (uint64_t)x14 | ((uint64_t)x15 << 32);
}
#undef BM_QR

// ---------------------------------------------------------------- samplers
// ternary: (x mod 3) - 1
BM_HD int ternary_of(uint64_t x) { return (int)(x % 3u) - 1; }
// discrete Gaussian sigma 3.2, |e| <= 19: magnitude = #{k : (x & (2^63-1)) >= cdt[k]}, sign = bit 63
BM_HD int gauss_of(uint64_t x, const uint64_t *cdt)
{
    uint64_t v = x & 0x7fffffffffffffffull;
    int mag = 0;
#pragma unroll
    for (int k = 0; k < 19; k++) mag += (v >= cdt[k]) ? 1 : 0;
    return (x >> 63) ? -mag : mag;
}

#ifdef __CUDACC__
// ---------------------------------------------------------------- modular arithmetic (device)
// Shoup product a*w mod q, lazy: any a < 2^64, w < q < 2^62, wp = floor(w 2^64 / q); result in [0, 2q).
BM_D uint64_t shoup(uint64_t a, uint64_t w, uint64_t wp, uint64_t q)
{
    return a * w - __umul64hi(a, wp) * q;
}
BM_D uint64_t shoup(uint64_t a, ulonglong2 w, uint64_t q) { return shoup(a, w.x, w.y, q); }
BM_D uint64_t csub(uint64_t a, uint64_t q) { return a >= q ? a - q : a; }

// x mod q for x < 2^64 via floor(2^64/q) (Shoup with w = 1): result in [0, q)
BM_D uint64_t reduce64(uint64_t x, uint64_t q, uint64_t one_p)
{
    return csub(x - __umul64hi(x, one_p) * q, q);
}

// 128-bit value (hi, lo) mod q, hi < 2^64: hi * (2^64 mod q) + lo; result in [0, q)
BM_D uint64_t reduce128(uint64_t hi, uint64_t lo, uint64_t q, ulonglong2 r64, uint64_t one_p)
{
    uint64_t t = shoup(hi, r64, q) + (lo - __umul64hi(lo, one_p) * q); // [0, 4q)
    t = csub(t, 2 * q);
    return csub(t, q);
}

// Per-prime constants used by the kernels.
struct PrimeK {
    uint64_t q, q2;            // q, 2q
    const ulonglong2 *fwd;     // psi_rev Shoup pairs [N]: psi^brev13(k)
    const ulonglong2 *inv;     // inverse twiddles [N]: psi^-brev13(k)
    ulonglong2 ninv;           // N^-1
    ulonglong2 ninv_w1;        // N^-1 * inv[1]  (folded into the last inverse stage)
    ulonglong2 r64;            // 2^64 mod q
    uint64_t one_p;            // floor(2^64 / q)
    // q1 only (ntt3f.cuh, the FP64-pipe transforms): (w, fl(w / q1)) as double bit patterns
    const ulonglong2 *fwdf, *invf;
    ulonglong2 ninvf, ninv_w1f;
};

#endif // __CUDACC__

} // namespace bm
