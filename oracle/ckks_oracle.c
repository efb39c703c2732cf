/*
 * ckks_oracle.c -- plain, slow, obviously-correct CPU oracle for the Blind-Match
 * encrypted 1:N cosine scan (HE-C^3, Algorithm 2).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load, call or execute anything under
 * oracle/.  The product library (paper_2408_06167_b200/) never includes, links
 * or imports this file, and this file includes nothing from the product.
 *
 * Everything is textbook: canonical residues in [0,q), modular products via
 * unsigned __int128 '%', polynomials kept in the COEFFICIENT domain, and a
 * negacyclic product built from the standard pre-twisted radix-2 cyclic NTT
 * (the only "library primitive" step; pinned against schoolbook
 * multiplication in tests/test_oracle_ring.py).  No blocking, no fusion, no
 * lazy reduction, no reordering beyond what the op definitions state.
 *
 * Scheme (RNS-CKKS, the paper's HE library setting, PAPER.md:155-170, 850-862;
 * parameters fixed by BASELINE.json configs / SURVEY.md Appendix A):
 *   ring   R = Z[X]/(X^N+1), N = 2^logN (8192 in every config; small N only in pins)
 *   primes q0 (58-bit), q1 (40-bit), special P (60-bit), each the largest prime
 *          below 2^k with q = 1 mod 16384 (BASELINE.json configs[0]).
 *   level 1 = {q0,q1}, level 0 = {q0}.  Key-switching uses one RNS digit per
 *   Q-prime and the special prime P (reading R3).
 *
 * Randomness: ChaCha20 block function (RFC 8439 sec. 2.3), addressed by
 * (seed, purpose, object, sub-stream, block counter); samplers in or_sample().
 * Both sides (oracle and product) implement this generator independently
 * (reading R14).
 *
 * Data layouts (all coefficient domain, u64 residues, limb-major):
 *   ct level 1   [2 comps][2 limbs q0,q1][N]
 *   ct level 0   [2 comps][1 limb  q0][N]
 *   pk           [2 comps (b,a)][2 limbs][N]
 *   rlk          [2 digits j][2 comps (b,a)][3 limbs q0,q1,P][N]
 *   gk           [n_rot][2 comps (b,a)][2 limbs q0,P][N]; entry i is rotation 2^i
 *   hgk          [s-1][2 comps][2 limbs q0,P][N]; entry r-1 is rotation r (f2 hoisted sum)
 *   sk           int8[N] in {-1,0,1}
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef unsigned __int128 u128;
typedef __int128 i128;

/* ------------------------------------------------------------------ */
/* scalar modular arithmetic (plain definitions)                        */
/* ------------------------------------------------------------------ */
static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }
static uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a + b) % q); }
static uint64_t submod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a + q - b) % q); }
static uint64_t powmod(uint64_t a, uint64_t e, uint64_t q)
{
    uint64_t r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = mulmod(r, a, q);
        a = mulmod(a, a, q);
        e >>= 1;
    }
    return r;
}
/* q prime: Fermat inverse */
static uint64_t invmod(uint64_t a, uint64_t q) { return powmod(a, q - 2, q); }
/* signed integer -> residue in [0,q) */
static uint64_t from_signed(int64_t x, uint64_t q)
{
    i128 r = (i128)x % (i128)q;
    if (r < 0) r += q;
    return (uint64_t)r;
}
/* residue in [0,q) -> centred representative in (-q/2, q/2]  (q odd) */
static int64_t centred(uint64_t x, uint64_t q) { return (x > q / 2) ? (int64_t)x - (int64_t)q : (int64_t)x; }

/* ------------------------------------------------------------------ */
/* primes (BASELINE.json configs[0]: "largest below 2^k with q=1 mod 16384") */
/* ------------------------------------------------------------------ */
/* deterministic Miller-Rabin; the first 12 prime bases are exact for n < 3.3e24 */
int or_is_prime(uint64_t n)
{
    static const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) {
        if (n == bases[i]) return 1;
        if (n % bases[i] == 0) return 0;
    }
    uint64_t d = n - 1;
    int r = 0;
    while ((d & 1) == 0) { d >>= 1; r++; }
    for (int i = 0; i < 12; i++) {
        uint64_t x = powmod(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int k = 1; k < r; k++) {
            x = mulmod(x, x, n);
            if (x == n - 1) { comp = 0; break; }
        }
        if (comp) return 0;
    }
    return 1;
}

/* largest prime q < 2^bits with q = 1 (mod m) */
uint64_t or_find_prime(int bits, uint64_t m)
{
    uint64_t q = ((uint64_t)1 << bits) - m + 1;   /* 2^bits = 0 mod m, so this is the largest candidate */
    while (!or_is_prime(q)) q -= m;
    return q;
}

/* fills {q0, q1, P} */
void or_primes(uint64_t out[3])
{
    out[0] = or_find_prime(58, 16384);
    out[1] = or_find_prime(40, 16384);
    out[2] = or_find_prime(60, 16384);
}

/* ------------------------------------------------------------------ */
/* ring: negacyclic product via pre-twisted cyclic NTT                 */
/* ------------------------------------------------------------------ */
typedef struct {
    int N, logN;
    uint64_t q;
    uint64_t psi;        /* primitive 2N-th root of unity mod q */
    uint64_t *psi_pow;   /* psi^k, k < N            */
    uint64_t *ipsi_pow;  /* psi^-k, k < N           */
    uint64_t *omega_pow; /* omega^k, omega = psi^2, k < N */
    uint64_t *iomega_pow;
    uint64_t n_inv;
} ring_t;

static void ring_init(ring_t *R, int logN, uint64_t q)
{
    R->logN = logN;
    R->N = 1 << logN;
    R->q = q;
    const uint64_t twoN = 2 * (uint64_t)R->N;
    /* psi = x^((q-1)/2N) has order dividing 2N; order is exactly 2N iff psi^N = -1 */
    for (uint64_t x = 2;; x++) {
        uint64_t c = powmod(x, (q - 1) / twoN, q);
        if (powmod(c, R->N, q) == q - 1) { R->psi = c; break; }
    }
    R->psi_pow = malloc(sizeof(uint64_t) * R->N);
    R->ipsi_pow = malloc(sizeof(uint64_t) * R->N);
    R->omega_pow = malloc(sizeof(uint64_t) * R->N);
    R->iomega_pow = malloc(sizeof(uint64_t) * R->N);
    uint64_t ipsi = invmod(R->psi, q), om = mulmod(R->psi, R->psi, q), iom = invmod(om, q);
    uint64_t a = 1, b = 1, c = 1, d = 1;
    for (int k = 0; k < R->N; k++) {
        R->psi_pow[k] = a; a = mulmod(a, R->psi, q);
        R->ipsi_pow[k] = b; b = mulmod(b, ipsi, q);
        R->omega_pow[k] = c; c = mulmod(c, om, q);
        R->iomega_pow[k] = d; d = mulmod(d, iom, q);
    }
    R->n_inv = invmod((uint64_t)R->N, q);
}

static void ring_free(ring_t *R)
{
    free(R->psi_pow); free(R->ipsi_pow); free(R->omega_pow); free(R->iomega_pow);
}

static unsigned bitrev(unsigned x, int bits)
{
    unsigned r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* textbook iterative radix-2 cyclic NTT (bit-reverse copy, then log N butterfly levels):
 * A_i = sum_k a_k w^(ik) with w = omega (forward) or omega^-1 (inverse, unscaled). */
static void cyclic_ntt(const ring_t *R, uint64_t *a, const uint64_t *wpow)
{
    const int N = R->N;
    const uint64_t q = R->q;
    for (int i = 0; i < N; i++) {
        unsigned j = bitrev((unsigned)i, R->logN);
        if (j > (unsigned)i) { uint64_t t = a[i]; a[i] = a[j]; a[j] = t; }
    }
    for (int len = 2; len <= N; len <<= 1) {
        int step = N / len; /* w_len = w^(N/len) */
        for (int start = 0; start < N; start += len) {
            for (int k = 0; k < len / 2; k++) {
                uint64_t w = wpow[k * step];
                uint64_t u = a[start + k];
                uint64_t v = mulmod(a[start + k + len / 2], w, q);
                a[start + k] = addmod(u, v, q);
                a[start + k + len / 2] = submod(u, v, q);
            }
        }
    }
}

/* c = a * b mod (X^N + 1, q).  Negacyclic convolution = cyclic convolution of the
 * psi-twisted inputs, untwisted by psi^-k.  c may alias a or b. */
static void poly_mul(const ring_t *R, const uint64_t *a, const uint64_t *b, uint64_t *c)
{
    const int N = R->N;
    const uint64_t q = R->q;
    uint64_t *A = malloc(sizeof(uint64_t) * N), *B = malloc(sizeof(uint64_t) * N);
    for (int k = 0; k < N; k++) {
        A[k] = mulmod(a[k], R->psi_pow[k], q);
        B[k] = mulmod(b[k], R->psi_pow[k], q);
    }
    cyclic_ntt(R, A, R->omega_pow);
    cyclic_ntt(R, B, R->omega_pow);
    for (int k = 0; k < N; k++) A[k] = mulmod(A[k], B[k], q);
    cyclic_ntt(R, A, R->iomega_pow);
    for (int k = 0; k < N; k++) c[k] = mulmod(mulmod(A[k], R->n_inv, q), R->ipsi_pow[k], q);
    free(A); free(B);
}

static void poly_add(uint64_t q, int N, const uint64_t *a, const uint64_t *b, uint64_t *c)
{
    for (int k = 0; k < N; k++) c[k] = addmod(a[k], b[k], q);
}
static void poly_sub(uint64_t q, int N, const uint64_t *a, const uint64_t *b, uint64_t *c)
{
    for (int k = 0; k < N; k++) c[k] = submod(a[k], b[k], q);
}
static void poly_scale(uint64_t q, int N, const uint64_t *a, uint64_t s, uint64_t *c)
{
    for (int k = 0; k < N; k++) c[k] = mulmod(a[k], s, q);
}

/* exported for the schoolbook pin: c = a*b mod (X^N+1, q) */
void or_poly_mul(int logN, uint64_t q, const uint64_t *a, const uint64_t *b, uint64_t *c)
{
    ring_t R;
    ring_init(&R, logN, q);
    poly_mul(&R, a, b, c);
    ring_free(&R);
}

/* Galois automorphism sigma_g: a(X) -> a(X^g), g odd.  Coefficient k moves to
 * t = k*g mod 2N; since X^N = -1 it lands at t-N with a sign flip when t >= N. */
static void automorphism(uint64_t q, int N, const uint64_t *a, uint64_t g, uint64_t *out)
{
    const uint64_t twoN = 2 * (uint64_t)N;
    for (int k = 0; k < N; k++) {
        uint64_t t = ((uint64_t)k * g) % twoN;
        if (t < (uint64_t)N) out[t] = a[k];
        else out[t - N] = submod(0, a[k], q);
    }
}

void or_automorphism(int logN, uint64_t q, const uint64_t *a, uint64_t g, uint64_t *out)
{
    automorphism(q, 1 << logN, a, g, out);
}

/* ------------------------------------------------------------------ */
/* ChaCha20 (RFC 8439 sec. 2.1-2.3) and samplers                       */
/* ------------------------------------------------------------------ */
static uint32_t rotl32(uint32_t x, int n) { return (x << n) | (x >> (32 - n)); }

void or_chacha_quarter(uint32_t *a, uint32_t *b, uint32_t *c, uint32_t *d)
{
    *a += *b; *d ^= *a; *d = rotl32(*d, 16);
    *c += *d; *b ^= *c; *b = rotl32(*b, 12);
    *a += *b; *d ^= *a; *d = rotl32(*d, 8);
    *c += *d; *b ^= *c; *b = rotl32(*b, 7);
}

void or_chacha20_block(const uint32_t key[8], uint32_t counter, const uint32_t nonce[3], uint32_t out[16])
{
    uint32_t s[16], x[16];
    s[0] = 0x61707865u; s[1] = 0x3320646eu; s[2] = 0x79622d32u; s[3] = 0x6b206574u;
    for (int i = 0; i < 8; i++) s[4 + i] = key[i];
    s[12] = counter;
    s[13] = nonce[0]; s[14] = nonce[1]; s[15] = nonce[2];
    memcpy(x, s, sizeof s);
    for (int r = 0; r < 10; r++) {
        or_chacha_quarter(&x[0], &x[4], &x[8], &x[12]);
        or_chacha_quarter(&x[1], &x[5], &x[9], &x[13]);
        or_chacha_quarter(&x[2], &x[6], &x[10], &x[14]);
        or_chacha_quarter(&x[3], &x[7], &x[11], &x[15]);
        or_chacha_quarter(&x[0], &x[5], &x[10], &x[15]);
        or_chacha_quarter(&x[1], &x[6], &x[11], &x[12]);
        or_chacha_quarter(&x[2], &x[7], &x[8], &x[13]);
        or_chacha_quarter(&x[3], &x[4], &x[9], &x[14]);
    }
    for (int i = 0; i < 16; i++) out[i] = x[i] + s[i];
}

/* Draw number n (u64) of stream (seed, purpose, obj, sub):
 * key = {seed lo, seed hi, purpose, 0,0,0,0,0}, nonce = {obj lo, obj hi, sub},
 * block counter = n / 8, u64 = word[2(n%8)] | word[2(n%8)+1] << 32. */
uint64_t or_draw(uint64_t seed, uint32_t purpose, uint64_t obj, uint32_t sub, uint64_t n)
{
    uint32_t key[8] = {(uint32_t)seed, (uint32_t)(seed >> 32), purpose, 0, 0, 0, 0, 0};
    uint32_t nonce[3] = {(uint32_t)obj, (uint32_t)(obj >> 32), sub};
    uint32_t blk[16];
    or_chacha20_block(key, (uint32_t)(n / 8), nonce, blk);
    int w = (int)(n % 8) * 2;
    return (uint64_t)blk[w] | ((uint64_t)blk[w + 1] << 32);
}

/* purposes of the random streams */
enum { P_SK = 1, P_PK_A = 2, P_PK_E = 3, P_RLK_A = 4, P_RLK_E = 5, P_GK_A = 6, P_GK_E = 7,
       P_ENC_U = 8, P_ENC_E0 = 9, P_ENC_E1 = 10 };

/* Discrete Gaussian CDT, sigma = 3.2, support |x| <= 19:
 * OR_CDT[k] = floor(2^63 * Pr(|X| <= k)), k = 0..18, generated exactly by
 * oracle/gen_cdt.py (Python Decimal, 60 digits). */
#include "cdt_table.h"

/* kind 0: uniform mod q from a 128-bit draw (draws 2k, 2k+1);
 * kind 1: ternary (draw k mod 3) - 1;
 * kind 2: Gaussian: v = low 63 bits of draw k, mag = #{j : v >= CDT[j]}, sign = top bit.
 * Output: residues mod q (q = 0 requests the signed integers cast to uint64). */
void or_sample(uint64_t seed, uint32_t purpose, uint64_t obj, uint32_t sub, int kind, int n, uint64_t q, uint64_t *out)
{
    for (int k = 0; k < n; k++) {
        int64_t v;
        if (kind == 0) {
            u128 x = ((u128)or_draw(seed, purpose, obj, sub, 2 * (uint64_t)k + 1) << 64) |
                     or_draw(seed, purpose, obj, sub, 2 * (uint64_t)k);
            out[k] = (uint64_t)(x % q);
            continue;
        } else if (kind == 1) {
            v = (int64_t)(or_draw(seed, purpose, obj, sub, (uint64_t)k) % 3) - 1;
        } else {
            uint64_t x = or_draw(seed, purpose, obj, sub, (uint64_t)k);
            uint64_t u = x & 0x7fffffffffffffffull;
            int mag = 0;
            for (int j = 0; j < 19; j++)
                if (u >= OR_CDT[j]) mag++;
            v = (x >> 63) ? -mag : mag;
        }
        out[k] = q ? from_signed(v, q) : (uint64_t)v;
    }
}

/* ------------------------------------------------------------------ */
/* parameter context                                                   */
/* ------------------------------------------------------------------ */
typedef struct {
    int logN, N;
    uint64_t q[3];      /* q0, q1, P */
    ring_t R[3];
    uint64_t P_mod[2];  /* P mod q0, P mod q1 */
    uint64_t P_inv[2];  /* P^-1 mod q0, q1   */
    uint64_t q1_inv_q0; /* q1^-1 mod q0      */
} ctx_t;

static void ctx_init(ctx_t *c, int logN)
{
    c->logN = logN;
    c->N = 1 << logN;
    or_primes(c->q);
    for (int k = 0; k < 3; k++) ring_init(&c->R[k], logN, c->q[k]);
    for (int k = 0; k < 2; k++) {
        c->P_mod[k] = c->q[2] % c->q[k];
        c->P_inv[k] = invmod(c->P_mod[k], c->q[k]);
    }
    c->q1_inv_q0 = invmod(c->q[1] % c->q[0], c->q[0]);
}
static void ctx_free(ctx_t *c)
{
    for (int k = 0; k < 3; k++) ring_free(&c->R[k]);
}

/* Galois element for a left slot rotation by r: g = 5^r mod 2N (reading R6) */
static uint64_t galois_elt(int N, uint64_t r) { return powmod(5, r, 2 * (uint64_t)N); }

/* ------------------------------------------------------------------ */
/* key generation (rows a0 of SURVEY.md sec. 8a)     */
/* ------------------------------------------------------------------ */
/* One Galois key for a left rotation by r (g = 5^r mod 2N), PRNG object obj, over {q0,P}:
 * b = -a s + e + (P mod q0) sigma_g(s) in q0; -a s + e in P; layout [2 comps (b,a)][2 limbs][N].
 * sv: the secret as signed integers. */
static void galois_key(const ctx_t *C, uint64_t seed, uint64_t r, uint64_t obj, int zero_error, const int64_t *sv,
                       uint64_t *gkr)
{
    const int N = C->N;
    uint64_t g = galois_elt(N, r);
    uint64_t *tmp = malloc(sizeof(uint64_t) * N), *e = malloc(sizeof(uint64_t) * N);
    uint64_t *s = malloc(sizeof(uint64_t) * N), *a = malloc(sizeof(uint64_t) * N);
    uint64_t *ss = malloc(sizeof(uint64_t) * N);
    int64_t *ev = malloc(sizeof(int64_t) * N);
    or_sample(seed, P_GK_E, obj, 0, 2, N, 0, (uint64_t *)ev);
    if (zero_error) memset(ev, 0, sizeof(int64_t) * N);
    for (int li = 0; li < 2; li++) {
        int l = li == 0 ? 0 : 2;
        uint64_t q = C->q[l];
        for (int k = 0; k < N; k++) { s[k] = from_signed(sv[k], q); e[k] = from_signed(ev[k], q); }
        or_sample(seed, P_GK_A, obj, (uint32_t)l, 0, N, q, a);
        uint64_t *b = gkr + (size_t)(0 * 2 + li) * N;
        uint64_t *aa = gkr + (size_t)(1 * 2 + li) * N;
        poly_mul(&C->R[l], a, s, tmp);
        poly_sub(q, N, e, tmp, b);
        if (l == 0) {
            automorphism(q, N, s, g, ss);
            poly_scale(q, N, ss, C->P_mod[0], tmp);
            poly_add(q, N, b, tmp, b);
        }
        memcpy(aa, a, sizeof(uint64_t) * N);
    }
    free(tmp); free(e); free(s); free(a); free(ss); free(ev);
}

/* sk: ternary s.  pk = (b, a) over {q0,q1}: b = -a s + e.
 * rlk_j (digit j in {0,1}) over {q0,q1,P}: b = -a s + e + [k==j] (P mod q_k) s^2, P-limb b = -a s + e.
 * gk_i (rotation 2^i) over {q0,P}: b = -a s + e + (P mod q0) sigma_g(s) in q0; -a s + e in P.
 * zero_error != 0 sets every key error to 0 (used only by the key-switch identity pin). */
int or_keygen(int logN, uint64_t seed, int n_rot, int zero_error,
              int8_t *sk, uint64_t *pk, uint64_t *rlk, uint64_t *gk)
{
    ctx_t C;
    ctx_init(&C, logN);
    const int N = C.N;
    uint64_t *tmp = malloc(sizeof(uint64_t) * N), *e = malloc(sizeof(uint64_t) * N);
    uint64_t *s = malloc(sizeof(uint64_t) * N), *a = malloc(sizeof(uint64_t) * N);
    uint64_t *s2 = malloc(sizeof(uint64_t) * N), *ss = malloc(sizeof(uint64_t) * N);
    int64_t *sv = malloc(sizeof(int64_t) * N), *ev = malloc(sizeof(int64_t) * N);

    or_sample(seed, P_SK, 0, 0, 1, N, 0, (uint64_t *)sv);
    for (int k = 0; k < N; k++) sk[k] = (int8_t)sv[k];

    /* public key */
    or_sample(seed, P_PK_E, 0, 0, 2, N, 0, (uint64_t *)ev);
    if (zero_error) memset(ev, 0, sizeof(int64_t) * N);
    for (int l = 0; l < 2; l++) {
        uint64_t q = C.q[l];
        for (int k = 0; k < N; k++) { s[k] = from_signed(sv[k], q); e[k] = from_signed(ev[k], q); }
        or_sample(seed, P_PK_A, 0, (uint32_t)l, 0, N, q, a);
        poly_mul(&C.R[l], a, s, tmp);
        uint64_t *b = pk + (size_t)(0 * 2 + l) * N, *aa = pk + (size_t)(1 * 2 + l) * N;
        poly_sub(q, N, e, tmp, b);
        memcpy(aa, a, sizeof(uint64_t) * N);
    }

    /* relinearization key: rlk[j][comp][limb][N] */
    for (int j = 0; j < 2; j++) {
        or_sample(seed, P_RLK_E, (uint64_t)j, 0, 2, N, 0, (uint64_t *)ev);
        if (zero_error) memset(ev, 0, sizeof(int64_t) * N);
        for (int l = 0; l < 3; l++) {
            uint64_t q = C.q[l];
            for (int k = 0; k < N; k++) { s[k] = from_signed(sv[k], q); e[k] = from_signed(ev[k], q); }
            or_sample(seed, P_RLK_A, (uint64_t)j, (uint32_t)l, 0, N, q, a);
            uint64_t *b = rlk + ((size_t)(j * 2 + 0) * 3 + l) * N;
            uint64_t *aa = rlk + ((size_t)(j * 2 + 1) * 3 + l) * N;
            poly_mul(&C.R[l], a, s, tmp);
            poly_sub(q, N, e, tmp, b);
            if (l == j) {
                poly_mul(&C.R[l], s, s, s2);
                poly_scale(q, N, s2, C.P_mod[l], tmp);
                poly_add(q, N, b, tmp, b);
            }
            memcpy(aa, a, sizeof(uint64_t) * N);
        }
    }

    /* Galois keys: gk[i][comp][limb in {q0,P}][N], rotation r = 2^i, PRNG object i */
    for (int i = 0; i < n_rot; i++)
        galois_key(&C, seed, (uint64_t)1 << i, (uint64_t)i, zero_error, sv, gk + (size_t)i * 4 * N);
    free(tmp); free(e); free(s); free(a); free(s2); free(ss); free(sv); free(ev);
    ctx_free(&C);
    return 0;
}

/* f2: Galois keys for EVERY rotation r = 1..s-1 (the hoisted rotation sum),
 * hgk[r-1][2 comps][2 limbs q0,P][N], PRNG object HROT_OBJ + r (disjoint from the ladder's i < 13). */
#define HROT_OBJ 64
int or_keygen_hoisted(int logN, uint64_t seed, int s, int zero_error, uint64_t *hgk)
{
    ctx_t C;
    ctx_init(&C, logN);
    const int N = C.N;
    int64_t *sv = malloc(sizeof(int64_t) * N);
    or_sample(seed, P_SK, 0, 0, 1, N, 0, (uint64_t *)sv);
    for (int r = 1; r < s; r++)
        galois_key(&C, seed, (uint64_t)r, (uint64_t)(HROT_OBJ + r), zero_error, sv, hgk + (size_t)(r - 1) * 4 * N);
    free(sv);
    ctx_free(&C);
    return 0;
}

/* ------------------------------------------------------------------ */
/* encryption / decryption                */
/* ------------------------------------------------------------------ */
/* Public-key encryption of integer plaintexts pt[n_cts][N] at level 1:
 * ct_o = (u*b + e0 + pt, u*a + e1) mod {q0,q1}, u ternary, e0/e1 Gaussian,
 * drawn from streams (seed, ENC_*, obj = first_obj + index, sub 0). */
void or_encrypt(int logN, const uint64_t *pk, const int64_t *pt, int64_t n_cts, uint64_t first_obj,
                uint64_t seed, uint64_t *out)
{
    ctx_t C;
    ctx_init(&C, logN);
    const int N = C.N;
    int64_t *uv = malloc(sizeof(int64_t) * N), *e0v = malloc(sizeof(int64_t) * N), *e1v = malloc(sizeof(int64_t) * N);
    uint64_t *u = malloc(sizeof(uint64_t) * N), *t = malloc(sizeof(uint64_t) * N), *x = malloc(sizeof(uint64_t) * N);
    for (int64_t c = 0; c < n_cts; c++) {
        uint64_t obj = first_obj + (uint64_t)c;
        or_sample(seed, P_ENC_U, obj, 0, 1, N, 0, (uint64_t *)uv);
        or_sample(seed, P_ENC_E0, obj, 0, 2, N, 0, (uint64_t *)e0v);
        or_sample(seed, P_ENC_E1, obj, 0, 2, N, 0, (uint64_t *)e1v);
        for (int l = 0; l < 2; l++) {
            uint64_t q = C.q[l];
            const uint64_t *b = pk + (size_t)(0 * 2 + l) * N, *a = pk + (size_t)(1 * 2 + l) * N;
            uint64_t *c0 = out + ((size_t)c * 4 + 0 * 2 + l) * N, *c1 = out + ((size_t)c * 4 + 1 * 2 + l) * N;
            for (int k = 0; k < N; k++) u[k] = from_signed(uv[k], q);
            poly_mul(&C.R[l], u, b, t);
            for (int k = 0; k < N; k++)
                x[k] = addmod(from_signed(e0v[k], q), from_signed(pt[(size_t)c * N + k], q), q);
            poly_add(q, N, t, x, c0);
            poly_mul(&C.R[l], u, a, t);
            for (int k = 0; k < N; k++) x[k] = from_signed(e1v[k], q);
            poly_add(q, N, t, x, c1);
        }
    }
    free(uv); free(e0v); free(e1v); free(u); free(t); free(x);
    ctx_free(&C);
}

/* m = c0 + c1*s mod q_l for each limb l < n_limbs; ct layout [2][n_limbs][N] */
void or_decrypt(int logN, const int8_t *sk, const uint64_t *ct, int n_limbs, uint64_t *m)
{
    ctx_t C;
    ctx_init(&C, logN);
    const int N = C.N;
    uint64_t *s = malloc(sizeof(uint64_t) * N), *t = malloc(sizeof(uint64_t) * N);
    for (int l = 0; l < n_limbs; l++) {
        uint64_t q = C.q[l];
        for (int k = 0; k < N; k++) s[k] = from_signed(sk[k], q);
        poly_mul(&C.R[l], ct + (size_t)(1 * n_limbs + l) * N, s, t);
        poly_add(q, N, ct + (size_t)(0 * n_limbs + l) * N, t, m + (size_t)l * N);
    }
    free(s); free(t);
    ctx_free(&C);
}

/* ------------------------------------------------------------------ */
/* evaluation ops                          */
/* ------------------------------------------------------------------ */
/* ModDown by P of a key-switch accumulator: out[k] = (KS[k] - centred_P(KS[P])) * P^-1 mod q_k,
 * for k < n_q (KS layout [n_q + 1 limbs][N], P limb last). */
static void moddown(const ctx_t *C, int n_q, const uint64_t *KS, uint64_t *out)
{
    const int N = C->N;
    const uint64_t P = C->q[2];
    const uint64_t *ksP = KS + (size_t)n_q * N;
    for (int l = 0; l < n_q; l++) {
        uint64_t q = C->q[l];
        for (int k = 0; k < N; k++) {
            uint64_t y = from_signed(centred(ksP[k], P), q);
            out[(size_t)l * N + k] = mulmod(submod(KS[(size_t)l * N + k], y, q), C->P_inv[l], q);
        }
    }
}

/* Relinearization (the "re-linearization" inside Mul):
 * (d0, d1, d2) at level 1 -> (d0 + KS'_0, d1 + KS'_1), digits x_j = [d2]_{q_j} lifted
 * non-centred to {q0,q1,P}; KS_c = sum_j x_j * rlk_j[c]; KS' = ModDown(KS).
 * d layout [3][2][N]; out layout [2][2][N]. */
static void relinearize(const ctx_t *C, const uint64_t *d, const uint64_t *rlk, uint64_t *out)
{
    const int N = C->N;
    uint64_t *KS = calloc((size_t)3 * N, sizeof(uint64_t));
    uint64_t *x = malloc(sizeof(uint64_t) * N), *t = malloc(sizeof(uint64_t) * N);
    uint64_t *ksd = malloc(sizeof(uint64_t) * 2 * N);
    for (int c = 0; c < 2; c++) {
        memset(KS, 0, sizeof(uint64_t) * 3 * N);
        for (int j = 0; j < 2; j++) {
            const uint64_t *xj = d + (size_t)(2 * 2 + j) * N; /* [d2]_{q_j}, entries in [0,q_j) */
            for (int l = 0; l < 3; l++) {
                uint64_t q = C->q[l];
                for (int k = 0; k < N; k++) x[k] = xj[k] % q;
                poly_mul(&C->R[l], x, rlk + ((size_t)(j * 2 + c) * 3 + l) * N, t);
                poly_add(q, N, KS + (size_t)l * N, t, KS + (size_t)l * N);
            }
        }
        moddown(C, 2, KS, ksd);
        for (int l = 0; l < 2; l++)
            poly_add(C->q[l], N, d + (size_t)(c * 2 + l) * N, ksd + (size_t)l * N, out + (size_t)(c * 2 + l) * N);
    }
    free(KS); free(x); free(t); free(ksd);
}

/* Rescale (Res): level 1 -> 0; c' = (c[q0] - centred_{q1}(c[q1])) * q1^-1 mod q0.
 * in [2][2][N] -> out [2][1][N] */
static void rescale(const ctx_t *C, const uint64_t *in, uint64_t *out)
{
    const int N = C->N;
    const uint64_t q0 = C->q[0], q1 = C->q[1];
    for (int c = 0; c < 2; c++)
        for (int k = 0; k < N; k++) {
            uint64_t z = from_signed(centred(in[(size_t)(c * 2 + 1) * N + k], q1), q0);
            out[(size_t)c * N + k] = mulmod(submod(in[(size_t)(c * 2 + 0) * N + k], z, q0), C->q1_inv_q0, q0);
        }
}

/* Rot (left rotation by r, reading R6) at level 0 with Galois key gk_r
 * ([2 comps][2 limbs q0,P][N]): (sigma_g(c0) + KS'_0, KS'_1), KS_c = x * gk[c], x = sigma_g(c1)
 * lifted non-centred to {q0,P}. in/out [2][1][N] (out may not alias in). */
static void rotate(const ctx_t *C, const uint64_t *in, uint64_t r, const uint64_t *gkr, uint64_t *out)
{
    const int N = C->N;
    const uint64_t q0 = C->q[0], P = C->q[2];
    const uint64_t g = galois_elt(N, r);
    uint64_t *a0 = malloc(sizeof(uint64_t) * N), *a1 = malloc(sizeof(uint64_t) * N);
    uint64_t *xP = malloc(sizeof(uint64_t) * N);
    uint64_t *KS = malloc(sizeof(uint64_t) * 2 * N), *ksd = malloc(sizeof(uint64_t) * N);
    automorphism(q0, N, in, g, a0);
    automorphism(q0, N, in + N, g, a1);
    for (int k = 0; k < N; k++) xP[k] = a1[k] % P;
    for (int c = 0; c < 2; c++) {
        /* KS layout for moddown: [q0][P] */
        poly_mul(&C->R[0], a1, gkr + (size_t)(c * 2 + 0) * N, KS);
        poly_mul(&C->R[2], xP, gkr + (size_t)(c * 2 + 1) * N, KS + N);
        moddown(C, 1, KS, ksd);
        if (c == 0) poly_add(q0, N, a0, ksd, out);
        else memcpy(out + N, ksd, sizeof(uint64_t) * N);
    }
    free(a0); free(a1); free(xP); free(KS); free(ksd);
}

/* f2 (NOT the paper's ladder): sum_{r=0}^{s-1} Rot(C, r) at level 0 with ONE
 * hoisted key switch (Halevi-Shoup hoisting): the digit x = c1 in coefficient form (integers in
 * [0, q0)) is lifted to {q0, P} once; each rotation applies sigma_{5^r} to the lifted digit in each
 * limb as a signed permutation (a negated coefficient becomes -x mod q in that limb), the products
 * KS_r[c] = sigma_r(x~) hgk_r[c] are summed over r in {q0, P} and ModDown'ed once:
 *   out_0 = sum_{r<s} sigma_r(c0) + ModDown(sum_{r>=1} KS_r[0]),  out_1 = c1 + ModDown(sum_{r>=1} KS_r[1]).
 * Slot k s of the result holds the same block sum as the ladder's (decrypts to the same scores up to
 * noise), but the residues differ: it has its own parity (order 2).  in/out [2][1][N]. */
/* (generalised for the baby-step giant-step variant below: the n rotations by i * step, i < n; the
 *  key of rotation r is hgk[r - 1]; step = 1, n = s is the sum above) */
static void hoisted_rot_sum_step(const ctx_t *C, int n, int step, const uint64_t *hgk, const uint64_t *in,
                                 uint64_t *out)
{
    const int N = C->N;
    const uint64_t q0 = C->q[0], P = C->q[2];
    const uint64_t *c0 = in, *c1 = in + N;
    uint64_t *xr0 = malloc(sizeof(uint64_t) * N), *xrP = malloc(sizeof(uint64_t) * N);
    uint64_t *t = malloc(sizeof(uint64_t) * N), *xP = malloc(sizeof(uint64_t) * N);
    uint64_t *acc = calloc((size_t)4 * N, sizeof(uint64_t)); /* [c][q0 | P][N] */
    uint64_t *c0sum = malloc(sizeof(uint64_t) * N), *ksd = malloc(sizeof(uint64_t) * N);
    for (int k = 0; k < N; k++) xP[k] = c1[k] % P; /* non-centred lift (reading R4): x < q0 < P */
    memcpy(c0sum, c0, sizeof(uint64_t) * N);
    for (int i = 1; i < n; i++) {
        const int r = i * step;
        const uint64_t g = galois_elt(N, (uint64_t)r);
        const uint64_t *key = hgk + (size_t)(r - 1) * 4 * N;
        automorphism(q0, N, c1, g, xr0);
        automorphism(P, N, xP, g, xrP);
        automorphism(q0, N, c0, g, t);
        poly_add(q0, N, c0sum, t, c0sum);
        for (int c = 0; c < 2; c++) {
            poly_mul(&C->R[0], xr0, key + (size_t)(c * 2 + 0) * N, t);
            poly_add(q0, N, acc + (size_t)(c * 2 + 0) * N, t, acc + (size_t)(c * 2 + 0) * N);
            poly_mul(&C->R[2], xrP, key + (size_t)(c * 2 + 1) * N, t);
            poly_add(P, N, acc + (size_t)(c * 2 + 1) * N, t, acc + (size_t)(c * 2 + 1) * N);
        }
    }
    for (int c = 0; c < 2; c++) {
        moddown(C, 1, acc + (size_t)c * 2 * N, ksd);
        poly_add(q0, N, c == 0 ? c0sum : c1, ksd, out + (size_t)c * N);
    }
    free(xr0); free(xrP); free(t); free(xP); free(acc); free(c0sum); free(ksd);
}

static void hoisted_rot_sum(const ctx_t *C, int s, const uint64_t *hgk, const uint64_t *in, uint64_t *out)
{
    hoisted_rot_sum_step(C, s, 1, hgk, in, out);
}

/* f2 baby-step giant-step rotation sum (NOT the paper's ladder): with
 * s = b g, b = 2^ceil(log2(s) / 2), g = s / b,
 *   sum_{r<s} Rot(C, r) = sum_{j<g} Rot( sum_{i<b} Rot(C, i), j b )
 * each of the two sums by one hoisted key switch (b - 1 and g - 1 key products, two ModDowns per
 * component instead of one): the baby steps use the keys of rotations 1..b-1, the giant steps those of
 * b, 2b, .., (g-1) b -- all among hgk[s-1].  Same decrypted scores as the ladder, its own residues. */
static void bsgs_rot_sum(const ctx_t *C, int s, const uint64_t *hgk, const uint64_t *in, uint64_t *out)
{
    int log_s = 0;
    while ((1 << log_s) < s) log_s++;
    const int b = 1 << ((log_s + 1) / 2), g = s / b;
    uint64_t *baby = malloc(sizeof(uint64_t) * 2 * C->N);
    hoisted_rot_sum_step(C, b, 1, hgk, in, baby);
    hoisted_rot_sum_step(C, g, b, hgk, baby, out);
    free(baby);
}

void or_hoisted_rot_sum(int logN, int s, const uint64_t *hgk, const uint64_t *in, uint64_t *out)
{
    ctx_t C; ctx_init(&C, logN); hoisted_rot_sum(&C, s, hgk, in, out); ctx_free(&C);
}
void or_bsgs_rot_sum(int logN, int s, const uint64_t *hgk, const uint64_t *in, uint64_t *out)
{
    ctx_t C; ctx_init(&C, logN); bsgs_rot_sum(&C, s, hgk, in, out); ctx_free(&C);
}

/* exported single-op entry points for the pins */
void or_relinearize(int logN, const uint64_t *d, const uint64_t *rlk, uint64_t *out)
{
    ctx_t C; ctx_init(&C, logN); relinearize(&C, d, rlk, out); ctx_free(&C);
}
void or_rescale(int logN, const uint64_t *in, uint64_t *out)
{
    ctx_t C; ctx_init(&C, logN); rescale(&C, in, out); ctx_free(&C);
}
void or_rotate(int logN, const uint64_t *in, uint64_t r, const uint64_t *gkr, uint64_t *out)
{
    ctx_t C; ctx_init(&C, logN); rotate(&C, in, r, gkr, out); ctx_free(&C);
}
void or_moddown(int logN, int n_q, const uint64_t *KS, uint64_t *out)
{
    ctx_t C; ctx_init(&C, logN); moddown(&C, n_q, KS, out); ctx_free(&C);
}

/* Mul(C) tensor part for one pair of level-1 ciphertexts, accumulated into d [3][2][N]:
 * d0 += a0 b0, d1 += a0 b1 + a1 b0, d2 += a1 b1 (negacyclic products per limb). */
static void tensor_acc(const ctx_t *C, const uint64_t *ca, const uint64_t *cb, uint64_t *d)
{
    const int N = C->N;
    uint64_t *t = malloc(sizeof(uint64_t) * N);
    for (int l = 0; l < 2; l++) {
        uint64_t q = C->q[l];
        const uint64_t *a0 = ca + (size_t)(0 * 2 + l) * N, *a1 = ca + (size_t)(1 * 2 + l) * N;
        const uint64_t *b0 = cb + (size_t)(0 * 2 + l) * N, *b1 = cb + (size_t)(1 * 2 + l) * N;
        uint64_t *d0 = d + (size_t)(0 * 2 + l) * N, *d1 = d + (size_t)(1 * 2 + l) * N, *d2 = d + (size_t)(2 * 2 + l) * N;
        poly_mul(&C->R[l], a0, b0, t); poly_add(q, N, d0, t, d0);
        poly_mul(&C->R[l], a0, b1, t); poly_add(q, N, d1, t, d1);
        poly_mul(&C->R[l], a1, b0, t); poly_add(q, N, d1, t, d1);
        poly_mul(&C->R[l], a1, b1, t); poly_add(q, N, d2, t, d2);
    }
    free(t);
}

/* ------------------------------------------------------------------ */
/* Algorithm 2, HE-C^3 for one (query, set) pair    */
/* ------------------------------------------------------------------ */
/* order 0 (HOISTED): C = Res(Relin(sum_i tensor(C_u,i, C_s,i)))
 * order 1 (PAPER):   C = sum_i Res(Relin(tensor(C_u,i, C_s,i))), C_out starting as the
 *                    trivial zero ciphertext (line 3; reading R9).
 * then for i = 1..log2(s): C = Add(Rot(C, 2^(i-1)), C)   (lines 7-9, reading R7).
 * order 2 (f2, not the paper's ladder): order 0's C, then hoisted_rot_sum (gk = hgk).
 * order 4 (f2, not the paper's ladder): order 0's C, then bsgs_rot_sum (gk = hgk).
 * qct, sct: [p][2][2][N]; out: [2][1][N]. */
static void he_c3_pair(const ctx_t *C, int p, int log_s, int order, const uint64_t *rlk, const uint64_t *gk,
                       const uint64_t *qct, const uint64_t *sct, uint64_t *out)
{
    const int N = C->N;
    const size_t ct1 = (size_t)4 * N;
    uint64_t *d = calloc((size_t)6 * N, sizeof(uint64_t));
    uint64_t *r1 = malloc(sizeof(uint64_t) * 4 * N);
    uint64_t *r0 = malloc(sizeof(uint64_t) * 2 * N);
    uint64_t *rot = malloc(sizeof(uint64_t) * 2 * N);
    const uint64_t q0 = C->q[0];
    memset(out, 0, sizeof(uint64_t) * 2 * N);
    if (order == 0 || order == 2 || order == 4) {
        for (int i = 0; i < p; i++) tensor_acc(C, qct + i * ct1, sct + i * ct1, d);
        relinearize(C, d, rlk, r1);
        rescale(C, r1, out);
    } else {
        for (int i = 0; i < p; i++) {
            memset(d, 0, sizeof(uint64_t) * 6 * N);
            tensor_acc(C, qct + i * ct1, sct + i * ct1, d);
            relinearize(C, d, rlk, r1);
            rescale(C, r1, r0);
            poly_add(q0, 2 * N, out, r0, out); /* Add at level 0, both components */
        }
    }
    if (order == 2 || order == 4) { /* f2: gk holds the hoisted keys hgk[s-1] */
        memcpy(r0, out, sizeof(uint64_t) * 2 * N);
        if (order == 2) hoisted_rot_sum(C, 1 << log_s, gk, r0, out);
        else bsgs_rot_sum(C, 1 << log_s, gk, r0, out);
    } else {
        for (int i = 1; i <= log_s; i++) {
            rotate(C, out, (uint64_t)1 << (i - 1), gk + (size_t)(i - 1) * 4 * N, rot);
            poly_add(q0, 2 * N, rot, out, out);
        }
    }
    free(d); free(r1); free(r0); free(rot);
}

typedef struct {
    const ctx_t *C;
    int p, log_s, order;
    const uint64_t *rlk, *gk, *db, *q;
    int64_t n_sets;
    const int64_t *pairs; /* [n_pairs][2] = (query, set) */
    int64_t n_pairs;
    uint64_t *out;        /* [n_pairs][2][N] */
    int64_t next;
    pthread_mutex_t mu;
} job_t;

static void *worker(void *arg)
{
    job_t *J = (job_t *)arg;
    const int N = J->C->N;
    const size_t set_stride = (size_t)J->p * 4 * N;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        int64_t i = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (i >= J->n_pairs) break;
        int64_t qi = J->pairs[2 * i], si = J->pairs[2 * i + 1];
        he_c3_pair(J->C, J->p, J->log_s, J->order, J->rlk, J->gk, J->q + (size_t)qi * set_stride,
                   J->db + (size_t)si * set_stride, J->out + (size_t)i * 2 * N);
    }
    return NULL;
}

/* The scan: for each listed (query, set) pair run HE-C^3.  db [n_sets][p][2][2][N],
 * q [nq][p][2][2][N], rlk/gk as in or_keygen, out [n_pairs][2][1][N].
 * Pairs are independent; they are spread over n_threads threads. */
int or_match(int logN, int d, int p, int order, const uint64_t *rlk, const uint64_t *gk,
             const uint64_t *db, int64_t n_sets, const uint64_t *q, int64_t nq,
             const int64_t *pairs, int64_t n_pairs, uint64_t *out, int n_threads)
{
    if (p <= 0 || d % p) return -1;
    int s = d / p, log_s = 0;
    while ((1 << log_s) < s) log_s++;
    if ((1 << log_s) != s) return -1;
    for (int64_t i = 0; i < n_pairs; i++)
        if (pairs[2 * i] < 0 || pairs[2 * i] >= nq || pairs[2 * i + 1] < 0 || pairs[2 * i + 1] >= n_sets) return -2;
    ctx_t C;
    ctx_init(&C, logN);
    job_t J;
    memset(&J, 0, sizeof J);
    J.C = &C; J.p = p; J.log_s = log_s; J.order = order; J.rlk = rlk; J.gk = gk; J.db = db; J.q = q;
    J.n_sets = n_sets; J.pairs = pairs; J.n_pairs = n_pairs; J.out = out; J.next = 0;
    pthread_mutex_init(&J.mu, NULL);
    if (n_threads < 1) n_threads = 1;
    pthread_t *th = malloc(sizeof(pthread_t) * n_threads);
    for (int t = 0; t < n_threads; t++) pthread_create(&th[t], NULL, worker, &J);
    for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&J.mu);
    ctx_free(&C);
    return 0;
}

/* ------------------------------------------------------------------ */
/* f2: the relin-free degree-2 output for p = d      */
/* (s = 1: no rotation, so no key switch needs a degree-1 ciphertext).  */
/* ------------------------------------------------------------------ */
/* C = sum_i tensor(C_u,i, C_s,i) = (d0, d1, d2) at level 1 (PAPER.md:328 without the relinearisation
 * inside Mul(C)), then Res of EACH component by q1 (the rescale formula above applied to
 * three polynomials); the client decrypts with (1, s, s^2).  qct, sct [p][2][2][N]; out [3][1][N]. */
static void deg2_pair(const ctx_t *C, int p, const uint64_t *qct, const uint64_t *sct, uint64_t *out)
{
    const int N = C->N;
    const size_t ct1 = (size_t)4 * N;
    const uint64_t q0 = C->q[0], q1 = C->q[1];
    uint64_t *d = calloc((size_t)6 * N, sizeof(uint64_t));
    for (int i = 0; i < p; i++) tensor_acc(C, qct + i * ct1, sct + i * ct1, d);
    for (int c = 0; c < 3; c++)
        for (int k = 0; k < N; k++) {
            uint64_t z = from_signed(centred(d[(size_t)(c * 2 + 1) * N + k], q1), q0);
            out[(size_t)c * N + k] = mulmod(submod(d[(size_t)(c * 2 + 0) * N + k], z, q0), C->q1_inv_q0, q0);
        }
    free(d);
}

typedef struct {
    const ctx_t *C;
    int p;
    const uint64_t *db, *q;
    const int64_t *pairs;
    int64_t n_pairs, next;
    uint64_t *out; /* [n_pairs][3][N] */
    pthread_mutex_t mu;
} job2_t;

static void *worker2(void *arg)
{
    job2_t *J = (job2_t *)arg;
    const int N = J->C->N;
    const size_t set_stride = (size_t)J->p * 4 * N;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        int64_t i = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (i >= J->n_pairs) break;
        deg2_pair(J->C, J->p, J->q + (size_t)J->pairs[2 * i] * set_stride, J->db + (size_t)J->pairs[2 * i + 1] * set_stride,
                  J->out + (size_t)i * 3 * N);
    }
    return NULL;
}

/* the degree-2 scan over listed pairs; requires d == p (s = 1).  out [n_pairs][3][1][N] */
int or_match_deg2(int logN, int d, int p, const uint64_t *db, int64_t n_sets, const uint64_t *q, int64_t nq,
                  const int64_t *pairs, int64_t n_pairs, uint64_t *out, int n_threads)
{
    if (p <= 0 || d != p) return -1;
    for (int64_t i = 0; i < n_pairs; i++)
        if (pairs[2 * i] < 0 || pairs[2 * i] >= nq || pairs[2 * i + 1] < 0 || pairs[2 * i + 1] >= n_sets) return -2;
    ctx_t C;
    ctx_init(&C, logN);
    job2_t J;
    memset(&J, 0, sizeof J);
    J.C = &C; J.p = p; J.db = db; J.q = q; J.pairs = pairs; J.n_pairs = n_pairs; J.out = out;
    pthread_mutex_init(&J.mu, NULL);
    if (n_threads < 1) n_threads = 1;
    pthread_t *th = malloc(sizeof(pthread_t) * n_threads);
    for (int t = 0; t < n_threads; t++) pthread_create(&th[t], NULL, worker2, &J);
    for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&J.mu);
    ctx_free(&C);
    return 0;
}

/* m = c0 + c1 s + c2 s^2 (mod q0) of a level-0 degree-2 ciphertext ct [3][N] */
void or_decrypt_deg2(int logN, const int8_t *sk, const uint64_t *ct, uint64_t *m)
{
    ctx_t C;
    ctx_init(&C, logN);
    const int N = C.N;
    const uint64_t q0 = C.q[0];
    uint64_t *s = calloc((size_t)N, sizeof(uint64_t)), *s2 = calloc((size_t)N, sizeof(uint64_t)), *t = calloc((size_t)N, sizeof(uint64_t));
    for (int k = 0; k < N; k++) s[k] = from_signed(sk[k], q0);
    poly_mul(&C.R[0], s, s, s2);
    memcpy(m, ct, sizeof(uint64_t) * N);
    poly_mul(&C.R[0], ct + N, s, t);
    poly_add(q0, N, m, t, m);
    poly_mul(&C.R[0], ct + 2 * (size_t)N, s2, t);
    poly_add(q0, N, m, t, m);
    free(s); free(s2); free(t);
    ctx_free(&C);
}

/* ================================================================== */
/* f3: server-side query expansion, Algorithm 1    */
/* "Input Ciphertext Expansion", on the chain        */
/* extended by one level: Q2 = {q0, q1, q2}, q2 = the largest prime     */
/* below q1 with q2 = 1 (mod 16384) (reading R24).            */
/* ================================================================== */
/* Layouts (coefficient domain):
 *   ct level 2   [2 comps][3 limbs q0,q1,q2][N]
 *   pk_q2        [2 comps (b,a)][N]: the q2 limb of the public key (its q0, q1 limbs are pk's)
 *   gk1          [n_rot][2 digits j][2 comps (b,a)][3 limbs q0,q1,P][N]; entry t is the
 *                level-1 Galois key of the left rotation by s 2^t (n_rot = log2 p for the
 *                expansion, log2 B for the enrollment, which uses the same family)
 *   masks        [p][N] int64 plaintexts of X_i at scale q2 (encoded by the caller)           */
enum { P_GK1_A = 11, P_GK1_E = 12 };

/* largest prime below `below` with q = 1 (mod m) */
uint64_t or_find_prime_below(uint64_t below, uint64_t m)
{
    uint64_t q = below - m;
    while (!or_is_prime(q)) q -= m;
    return q;
}
uint64_t or_q2(void)
{
    uint64_t q[3];
    or_primes(q);
    return or_find_prime_below(q[1], 16384);
}

typedef struct {
    ctx_t c;             /* q0, q1, P as everywhere else */
    uint64_t q2;
    ring_t R2;
    uint64_t q2_inv[2];  /* q2^-1 mod q0, q1 */
} ctx2_t;

static void ctx2_init(ctx2_t *x, int logN)
{
    ctx_init(&x->c, logN);
    x->q2 = or_find_prime_below(x->c.q[1], 16384);
    ring_init(&x->R2, logN, x->q2);
    for (int k = 0; k < 2; k++) x->q2_inv[k] = invmod(x->q2 % x->c.q[k], x->c.q[k]);
}
static void ctx2_free(ctx2_t *x)
{
    ring_free(&x->R2);
    ctx_free(&x->c);
}
/* modulus and ring of level-2 limb l (0: q0, 1: q1, 2: q2) */
static uint64_t l2_q(const ctx2_t *x, int l) { return l == 2 ? x->q2 : x->c.q[l]; }
static const ring_t *l2_R(const ctx2_t *x, int l) { return l == 2 ? &x->R2 : &x->c.R[l]; }

/* Expansion keys.  pk_q2 = (-a s + e, a) mod q2 with pk's error e (P_PK_E, object 0) and
 * a from (P_PK_A, object 0, sub-stream 3): the level-2 public key is pk extended by one limb.
 * gk1 for rotation r = s 2^t, digit j in {0,1}: over {q0,q1,P},
 *   b = -a s + e + [l = j] (P mod q_l) sigma_{5^r}(s) in limb q_l,   b = -a s + e in limb P,
 * a from (P_GK1_A, object 2r + j, sub-stream l), e from (P_GK1_E, object 2r + j). */
int or_keygen_exp(int logN, uint64_t seed, int d, int p, int n_rot, int zero_error, uint64_t *pk_q2, uint64_t *gk1)
{
    if (p <= 0 || d % p || n_rot < 0) return -1;
    ctx2_t X;
    ctx2_init(&X, logN);
    const ctx_t *C = &X.c;
    const int N = C->N, s = d / p;
    uint64_t *tmp = malloc(sizeof(uint64_t) * N), *e = malloc(sizeof(uint64_t) * N);
    uint64_t *sq = calloc((size_t)N, sizeof(uint64_t)), *a = malloc(sizeof(uint64_t) * N);
    uint64_t *ss = malloc(sizeof(uint64_t) * N);
    int64_t *sv = malloc(sizeof(int64_t) * N), *ev = malloc(sizeof(int64_t) * N);
    or_sample(seed, P_SK, 0, 0, 1, N, 0, (uint64_t *)sv);

    /* pk limb q2 */
    or_sample(seed, P_PK_E, 0, 0, 2, N, 0, (uint64_t *)ev);
    if (zero_error) memset(ev, 0, sizeof(int64_t) * N);
    for (int k = 0; k < N; k++) { sq[k] = from_signed(sv[k], X.q2); e[k] = from_signed(ev[k], X.q2); }
    or_sample(seed, P_PK_A, 0, 3, 0, N, X.q2, a);
    poly_mul(&X.R2, a, sq, tmp);
    poly_sub(X.q2, N, e, tmp, pk_q2);
    memcpy(pk_q2 + N, a, sizeof(uint64_t) * N);

    /* level-1 Galois keys of the strides s 2^t, t < n_rot (expansion: t < log2 p; enrollment:
     * t < log2 B, reading R27) */
    for (int t = 0; t < n_rot; t++) {
        const uint64_t r = (uint64_t)s << t, g = galois_elt(N, r);
        for (int j = 0; j < 2; j++) {
            const uint64_t obj = 2 * r + (uint64_t)j;
            or_sample(seed, P_GK1_E, obj, 0, 2, N, 0, (uint64_t *)ev);
            if (zero_error) memset(ev, 0, sizeof(int64_t) * N);
            for (int l = 0; l < 3; l++) {
                const uint64_t q = C->q[l];
                for (int k = 0; k < N; k++) { sq[k] = from_signed(sv[k], q); e[k] = from_signed(ev[k], q); }
                or_sample(seed, P_GK1_A, obj, (uint32_t)l, 0, N, q, a);
                uint64_t *b = gk1 + ((((size_t)t * 2 + j) * 2 + 0) * 3 + l) * N;
                uint64_t *aa = gk1 + ((((size_t)t * 2 + j) * 2 + 1) * 3 + l) * N;
                poly_mul(&C->R[l], a, sq, tmp);
                poly_sub(q, N, e, tmp, b);
                if (l == j) {
                    automorphism(q, N, sq, g, ss);
                    poly_scale(q, N, ss, C->P_mod[l], tmp);
                    poly_add(q, N, b, tmp, b);
                }
                memcpy(aa, a, sizeof(uint64_t) * N);
            }
        }
    }
    free(tmp); free(e); free(sq); free(a); free(ss); free(sv); free(ev);
    ctx2_free(&X);
    return 0;
}

/* Public-key encryption at level 2 ("a client encrypts the user's feature vector"):
 * ct_o = (u b + e0 + pt, u a + e1) over {q0,q1,q2}, the same streams as or_encrypt (object
 * first_obj + c), pk = [2][2][N] over {q0,q1} and pk_q2 = [2][N].  out [n_cts][2][3][N]. */
void or_encrypt_l2(int logN, const uint64_t *pk, const uint64_t *pk_q2, const int64_t *pt, int64_t n_cts,
                   uint64_t first_obj, uint64_t seed, uint64_t *out)
{
    ctx2_t X;
    ctx2_init(&X, logN);
    const int N = X.c.N;
    int64_t *uv = malloc(sizeof(int64_t) * N), *e0v = malloc(sizeof(int64_t) * N), *e1v = malloc(sizeof(int64_t) * N);
    uint64_t *u = malloc(sizeof(uint64_t) * N), *t = malloc(sizeof(uint64_t) * N), *x = malloc(sizeof(uint64_t) * N);
    for (int64_t c = 0; c < n_cts; c++) {
        uint64_t obj = first_obj + (uint64_t)c;
        or_sample(seed, P_ENC_U, obj, 0, 1, N, 0, (uint64_t *)uv);
        or_sample(seed, P_ENC_E0, obj, 0, 2, N, 0, (uint64_t *)e0v);
        or_sample(seed, P_ENC_E1, obj, 0, 2, N, 0, (uint64_t *)e1v);
        for (int l = 0; l < 3; l++) {
            const uint64_t q = l2_q(&X, l);
            const uint64_t *b = l == 2 ? pk_q2 : pk + (size_t)(0 * 2 + l) * N;
            const uint64_t *a = l == 2 ? pk_q2 + N : pk + (size_t)(1 * 2 + l) * N;
            uint64_t *c0 = out + ((size_t)c * 6 + 0 * 3 + l) * N, *c1 = out + ((size_t)c * 6 + 1 * 3 + l) * N;
            for (int k = 0; k < N; k++) u[k] = from_signed(uv[k], q);
            poly_mul(l2_R(&X, l), u, b, t);
            for (int k = 0; k < N; k++)
                x[k] = addmod(from_signed(e0v[k], q), from_signed(pt[(size_t)c * N + k], q), q);
            poly_add(q, N, t, x, c0);
            poly_mul(l2_R(&X, l), u, a, t);
            for (int k = 0; k < N; k++) x[k] = from_signed(e1v[k], q);
            poly_add(q, N, t, x, c1);
        }
    }
    free(uv); free(e0v); free(e1v); free(u); free(t); free(x);
    ctx2_free(&X);
}

/* m = c0 + c1 s mod q_l for the three level-2 limbs; ct [2][3][N] -> m [3][N] */
void or_decrypt_l2(int logN, const int8_t *sk, const uint64_t *ct, uint64_t *m)
{
    ctx2_t X;
    ctx2_init(&X, logN);
    const int N = X.c.N;
    uint64_t *s = malloc(sizeof(uint64_t) * N), *t = malloc(sizeof(uint64_t) * N);
    for (int l = 0; l < 3; l++) {
        const uint64_t q = l2_q(&X, l);
        for (int k = 0; k < N; k++) s[k] = from_signed(sk[k], q);
        poly_mul(l2_R(&X, l), ct + (size_t)(3 + l) * N, s, t);
        poly_add(q, N, ct + (size_t)l * N, t, m + (size_t)l * N);
    }
    free(s); free(t);
    ctx2_free(&X);
}

/* Mul(P) then Res (Algorithm 1 line 5): level 2 -> level 1,
 *   t_l = c_l * pt mod q_l (negacyclic, each comp),  out_k = (t_k - centred_{q2}(t_2)) q2^-1 mod q_k.
 * in [2][3][N], pt int64 [N], out [2][2][N]. */
static void mul_plain_rescale_q2(const ctx2_t *X, const uint64_t *in, const int64_t *pt, uint64_t *out)
{
    const int N = X->c.N;
    uint64_t *m = malloc(sizeof(uint64_t) * N), *t = malloc(sizeof(uint64_t) * 3 * N);
    for (int c = 0; c < 2; c++) {
        for (int l = 0; l < 3; l++) {
            const uint64_t q = l2_q(X, l);
            for (int k = 0; k < N; k++) m[k] = from_signed(pt[k], q);
            poly_mul(l2_R(X, l), in + (size_t)(c * 3 + l) * N, m, t + (size_t)l * N);
        }
        for (int l = 0; l < 2; l++) {
            const uint64_t q = X->c.q[l];
            for (int k = 0; k < N; k++) {
                uint64_t z = from_signed(centred(t[(size_t)2 * N + k], X->q2), q);
                out[(size_t)(c * 2 + l) * N + k] = mulmod(submod(t[(size_t)l * N + k], z, q), X->q2_inv[l], q);
            }
        }
    }
    free(m); free(t);
}
void or_mul_plain_rescale_q2(int logN, const uint64_t *in, const int64_t *pt, uint64_t *out)
{
    ctx2_t X; ctx2_init(&X, logN); mul_plain_rescale_q2(&X, in, pt, out); ctx2_free(&X);
}

/* Rot at level 1 (reading R6) with a 2-digit Galois key gkr [2 digits][2][3][N]:
 * a_c = sigma_g(c_c) per limb; digits x_j = [a_1]_{q_j} in [0, q_j) lifted non-centred to
 * {q0,q1,P} (reading R4); KS_c = sum_j x_j gkr[j][c]; out = (a_0 + ModDown(KS_0), ModDown(KS_1)).
 * in/out [2][2][N] (out may not alias in). */
static void rotate1(const ctx_t *C, const uint64_t *in, uint64_t r, const uint64_t *gkr, uint64_t *out)
{
    const int N = C->N;
    const uint64_t g = galois_elt(N, r);
    uint64_t *a = malloc(sizeof(uint64_t) * 4 * N), *x = malloc(sizeof(uint64_t) * N);
    uint64_t *t = malloc(sizeof(uint64_t) * N), *KS = malloc(sizeof(uint64_t) * 3 * N);
    uint64_t *ksd = malloc(sizeof(uint64_t) * 2 * N);
    for (int c = 0; c < 2; c++)
        for (int l = 0; l < 2; l++)
            automorphism(C->q[l], N, in + (size_t)(c * 2 + l) * N, g, a + (size_t)(c * 2 + l) * N);
    for (int c = 0; c < 2; c++) {
        memset(KS, 0, sizeof(uint64_t) * 3 * N);
        for (int j = 0; j < 2; j++) {
            const uint64_t *xj = a + (size_t)(1 * 2 + j) * N; /* [sigma(c1)]_{q_j}, in [0, q_j) */
            for (int l = 0; l < 3; l++) {
                const uint64_t q = C->q[l];
                for (int k = 0; k < N; k++) x[k] = xj[k] % q;
                poly_mul(&C->R[l], x, gkr + ((size_t)(j * 2 + c) * 3 + l) * N, t);
                poly_add(q, N, KS + (size_t)l * N, t, KS + (size_t)l * N);
            }
        }
        moddown(C, 2, KS, ksd);
        for (int l = 0; l < 2; l++) {
            uint64_t *o = out + (size_t)(c * 2 + l) * N;
            if (c == 0) poly_add(C->q[l], N, a + (size_t)l * N, ksd + (size_t)l * N, o);
            else memcpy(o, ksd + (size_t)l * N, sizeof(uint64_t) * N);
        }
    }
    free(a); free(x); free(t); free(KS); free(ksd);
}
void or_rotate1(int logN, const uint64_t *in, uint64_t r, const uint64_t *gkr, uint64_t *out)
{
    ctx_t C; ctx_init(&C, logN); rotate1(&C, in, r, gkr, out); ctx_free(&C);
}

/* Algorithm 1 with SPEC.md:297's post-condition (reading R25): for each
 * query ciphertext (level 2, tiled query) and part i < p:
 *   C_i = Res(Mul(P)(C_in, mask_i)),  then for t = 0 .. log2(p)-1:  C_i = Add(C_i, Rot(C_i, s 2^t)).
 * in [n][2][3][N], out [n][p][2][2][N] (level 1). */
int or_expand(int logN, int d, int p, const int64_t *masks, const uint64_t *gk1, const uint64_t *in, int64_t n,
              uint64_t *out)
{
    if (p <= 0 || d % p) return -1;
    int log_p = 0;
    while ((1 << log_p) < p) log_p++;
    if ((1 << log_p) != p) return -1;
    const int s = d / p;
    ctx2_t X;
    ctx2_init(&X, logN);
    const int N = X.c.N;
    uint64_t *rot = malloc(sizeof(uint64_t) * 4 * N);
    for (int64_t qi = 0; qi < n; qi++)
        for (int i = 0; i < p; i++) {
            uint64_t *Ci = out + ((size_t)qi * p + i) * 4 * N;
            mul_plain_rescale_q2(&X, in + (size_t)qi * 6 * N, masks + (size_t)i * N, Ci);
            for (int t = 0; t < log_p; t++) {
                rotate1(&X.c, Ci, (uint64_t)s << t, gk1 + (size_t)t * 12 * N, rot);
                for (int l = 0; l < 2; l++)
                    for (int c = 0; c < 2; c++)
                        poly_add(X.c.q[l], N, Ci + (size_t)(c * 2 + l) * N, rot + (size_t)(c * 2 + l) * N,
                                 Ci + (size_t)(c * 2 + l) * N);
            }
        }
    free(rot);
    ctx2_free(&X);
    return 0;
}

/* ================================================================== */
/* f4: server-side enrollment packing, Fig. 3 /    */
/* PAPER.md:251-269, on the same extended chain      */
/* ================================================================== */
/* The client encrypts the unit template in slots [0, d) (zeros elsewhere) at level 2.  For each
 * part i, with template index u = tB + k:
 *   C = Res(Mul(P)(C_u, E_i)),  E_i[x] = [x in [i s, (i+1) s)] at scale q2,
 *   C = Rot_right(C, (k - i) s) = Rot_left(C, m s), m = (i - k) mod B, done as the left rotations
 *       by s 2^t for the set bits t of m, ascending (reading R27),
 *   set[t][i] += C.
 * in [n][2][3][N] (templates first_u .. first_u + n - 1), emasks [p][N], gk1 [log2 B] keys,
 * db [n_sets][p][2][2][N] level 1 (accumulated; sets indexed from 0). */
int or_enroll(int logN, int d, int p, const int64_t *emasks, const uint64_t *gk1, const uint64_t *in, int64_t n,
              int64_t first_u, uint64_t *db, int64_t n_sets)
{
    if (p <= 0 || d % p) return -1;
    const int N = 1 << logN, S = N / 2, s = d / p, B = S / s;
    if (first_u < 0 || (first_u + n + B - 1) / B > n_sets) return -2;
    ctx2_t X;
    ctx2_init(&X, logN);
    uint64_t *C = malloc(sizeof(uint64_t) * 4 * N), *rot = malloc(sizeof(uint64_t) * 4 * N);
    for (int64_t c = 0; c < n; c++) {
        const int64_t u = first_u + c, t = u / B;
        const int k = (int)(u % B);
        for (int i = 0; i < p; i++) {
            mul_plain_rescale_q2(&X, in + (size_t)c * 6 * N, emasks + (size_t)i * N, C);
            const int m = ((i - k) % B + B) % B;
            for (int b = 0; (1 << b) < B; b++) {
                if (!((m >> b) & 1)) continue;
                rotate1(&X.c, C, (uint64_t)s << b, gk1 + (size_t)b * 12 * N, rot);
                memcpy(C, rot, sizeof(uint64_t) * 4 * N);
            }
            uint64_t *dst = db + ((size_t)t * p + i) * 4 * N;
            for (int cl = 0; cl < 4; cl++)
                poly_add(X.c.q[cl & 1], N, dst + (size_t)cl * N, C + (size_t)cl * N, dst + (size_t)cl * N);
        }
    }
    free(C); free(rot);
    ctx2_free(&X);
    return 0;
}

/* ================================================================== */
/* f1: output compression (PAPER.md:273, 343-345;  */
/* SPEC.md:321-329), on the same extended chain, so HE-C^3 runs one    */
/* level higher: level 2 -> (tensor, relin, Res by q2) -> level 1 ->   */
/* ladder at level 1 -> compression: Res_q1(Mul(P)(C_t, M)), right     */
/* rotation by (t mod s) at level 0, add (reading R28).      */
/* ================================================================== */
/* Layouts (coefficient domain):
 *   rlk2   [3 digits j][2 comps][4 limbs q0,q1,q2,P][N]
 *   gkl    [log2 s][2 digits][2 comps][3 limbs q0,q1,P][N]: level-1 Galois keys of the ladder's
 *          rotations 2^i (the gk1 family of f3, objects 2r + j)
 *   gkc    [s-1][2 comps][2 limbs q0,P][N]: level-0 Galois keys of the left rotations by S - u
 *          (right rotations by u), u = 1..s-1, PRNG objects CMP_OBJ + u
 *   mask   int64 [N]: M[x] = [x mod s = 0] at scale q1 (encoded by the caller)              */
enum { P_RLK2_A = 13, P_RLK2_E = 14 };
#define CMP_OBJ 4096

/* one level-1 Galois key (the f3 family): rotation r, digits j in {0,1}, over {q0,q1,P} */
static void galois_key1(const ctx_t *C, uint64_t seed, uint64_t r, int zero_error, const int64_t *sv, uint64_t *out)
{
    const int N = C->N;
    const uint64_t g = galois_elt(N, r);
    uint64_t *tmp = malloc(sizeof(uint64_t) * N), *e = malloc(sizeof(uint64_t) * N);
    uint64_t *sq = calloc((size_t)N, sizeof(uint64_t)), *a = malloc(sizeof(uint64_t) * N);
    uint64_t *ss = malloc(sizeof(uint64_t) * N);
    int64_t *ev = malloc(sizeof(int64_t) * N);
    for (int j = 0; j < 2; j++) {
        const uint64_t obj = 2 * r + (uint64_t)j;
        or_sample(seed, P_GK1_E, obj, 0, 2, N, 0, (uint64_t *)ev);
        if (zero_error) memset(ev, 0, sizeof(int64_t) * N);
        for (int l = 0; l < 3; l++) {
            const uint64_t q = C->q[l];
            for (int k = 0; k < N; k++) { sq[k] = from_signed(sv[k], q); e[k] = from_signed(ev[k], q); }
            or_sample(seed, P_GK1_A, obj, (uint32_t)l, 0, N, q, a);
            uint64_t *b = out + (((size_t)j * 2 + 0) * 3 + l) * N, *aa = out + (((size_t)j * 2 + 1) * 3 + l) * N;
            poly_mul(&C->R[l], a, sq, tmp);
            poly_sub(q, N, e, tmp, b);
            if (l == j) {
                automorphism(q, N, sq, g, ss);
                poly_scale(q, N, ss, C->P_mod[l], tmp);
                poly_add(q, N, b, tmp, b);
            }
            memcpy(aa, a, sizeof(uint64_t) * N);
        }
    }
    free(tmp); free(e); free(sq); free(a); free(ss); free(ev);
}

/* modulus / ring of a 4-limb key-switching limb (0 q0, 1 q1, 2 q2, 3 P) */
static uint64_t l4_q(const ctx2_t *x, int l) { return l == 3 ? x->c.q[2] : l2_q(x, l); }
static const ring_t *l4_R(const ctx2_t *x, int l) { return l == 3 ? &x->c.R[2] : l2_R(x, l); }

/* Compression keys: rlk2 (3 digits over {q0,q1,q2,P}: b = -a s + e + [l = j](P mod q_l) s^2, a from
 * (P_RLK2_A, object j, sub-stream l), e from (P_RLK2_E, object j)); the ladder's level-1 Galois keys;
 * the level-0 keys of the right rotations by u = 1..s-1. */
int or_keygen_cmp(int logN, uint64_t seed, int d, int p, int zero_error, uint64_t *rlk2, uint64_t *gkl, uint64_t *gkc)
{
    if (p <= 0 || d % p) return -1;
    ctx2_t X;
    ctx2_init(&X, logN);
    const ctx_t *C = &X.c;
    const int N = C->N, S = N / 2, s = d / p;
    uint64_t *tmp = malloc(sizeof(uint64_t) * N), *e = malloc(sizeof(uint64_t) * N);
    uint64_t *sq = calloc((size_t)N, sizeof(uint64_t)), *a = malloc(sizeof(uint64_t) * N);
    uint64_t *s2 = malloc(sizeof(uint64_t) * N);
    int64_t *sv = malloc(sizeof(int64_t) * N), *ev = malloc(sizeof(int64_t) * N);
    or_sample(seed, P_SK, 0, 0, 1, N, 0, (uint64_t *)sv);
    for (int j = 0; j < 3; j++) {
        or_sample(seed, P_RLK2_E, (uint64_t)j, 0, 2, N, 0, (uint64_t *)ev);
        if (zero_error) memset(ev, 0, sizeof(int64_t) * N);
        for (int l = 0; l < 4; l++) {
            const uint64_t q = l4_q(&X, l);
            for (int k = 0; k < N; k++) { sq[k] = from_signed(sv[k], q); e[k] = from_signed(ev[k], q); }
            or_sample(seed, P_RLK2_A, (uint64_t)j, (uint32_t)l, 0, N, q, a);
            uint64_t *b = rlk2 + (((size_t)j * 2 + 0) * 4 + l) * N, *aa = rlk2 + (((size_t)j * 2 + 1) * 4 + l) * N;
            poly_mul(l4_R(&X, l), a, sq, tmp);
            poly_sub(q, N, e, tmp, b);
            if (l == j) {
                poly_mul(l4_R(&X, l), sq, sq, s2);
                poly_scale(q, N, s2, C->q[2] % q, tmp);
                poly_add(q, N, b, tmp, b);
            }
            memcpy(aa, a, sizeof(uint64_t) * N);
        }
    }
    int log_s = 0;
    while ((1 << log_s) < s) log_s++;
    for (int i = 0; i < log_s; i++) galois_key1(C, seed, (uint64_t)1 << i, zero_error, sv, gkl + (size_t)i * 12 * N);
    for (int u = 1; u < s; u++)
        galois_key(C, seed, (uint64_t)(S - u), (uint64_t)(CMP_OBJ + u), zero_error, sv, gkc + (size_t)(u - 1) * 4 * N);
    free(tmp); free(e); free(sq); free(a); free(s2); free(sv); free(ev);
    ctx2_free(&X);
    return 0;
}

/* Relinearization at level 2 (3 digits) followed by Res by q2 (level 2 -> 1), the textbook way:
 * x_j = [d2]_{q_j} in [0, q_j) lifted to {q0,q1,q2,P}; KS_c = sum_j x_j rlk2_j[c]; ModDown by P to
 * {q0,q1,q2}; c_c = d_c + KS'_c; then (c_c[q_k] - centred_{q2}(c_c[q2])) q2^-1 mod q_k.
 * d [3][3][N] -> out [2][2][N]. */
static void relin_rescale_l2(const ctx2_t *X, const uint64_t *d, const uint64_t *rlk2, uint64_t *out)
{
    const int N = X->c.N;
    const uint64_t P = X->c.q[2];
    uint64_t *KS = malloc(sizeof(uint64_t) * 4 * N), *x = malloc(sizeof(uint64_t) * N);
    uint64_t *t = malloc(sizeof(uint64_t) * N), *cc = malloc(sizeof(uint64_t) * 3 * N);
    for (int c = 0; c < 2; c++) {
        memset(KS, 0, sizeof(uint64_t) * 4 * N);
        for (int j = 0; j < 3; j++) {
            const uint64_t *xj = d + (size_t)(2 * 3 + j) * N; /* [d2]_{q_j}, in [0, q_j) */
            for (int l = 0; l < 4; l++) {
                const uint64_t q = l4_q(X, l);
                for (int k = 0; k < N; k++) x[k] = xj[k] % q;
                poly_mul(l4_R(X, l), x, rlk2 + (((size_t)j * 2 + c) * 4 + l) * N, t);
                poly_add(q, N, KS + (size_t)l * N, t, KS + (size_t)l * N);
            }
        }
        /* ModDown by P to the three Q limbs, added to d_c */
        for (int l = 0; l < 3; l++) {
            const uint64_t q = l2_q(X, l), pinv = invmod(P % q, q);
            for (int k = 0; k < N; k++) {
                uint64_t y = from_signed(centred(KS[(size_t)3 * N + k], P), q);
                uint64_t ks = mulmod(submod(KS[(size_t)l * N + k], y, q), pinv, q);
                cc[(size_t)l * N + k] = addmod(d[(size_t)(c * 3 + l) * N + k], ks, q);
            }
        }
        /* Res by q2 */
        for (int l = 0; l < 2; l++) {
            const uint64_t q = X->c.q[l];
            for (int k = 0; k < N; k++) {
                uint64_t z = from_signed(centred(cc[(size_t)2 * N + k], X->q2), q);
                out[(size_t)(c * 2 + l) * N + k] = mulmod(submod(cc[(size_t)l * N + k], z, q), X->q2_inv[l], q);
            }
        }
    }
    free(KS); free(x); free(t); free(cc);
}
void or_relin_rescale_l2(int logN, const uint64_t *d, const uint64_t *rlk2, uint64_t *out)
{
    ctx2_t X; ctx2_init(&X, logN); relin_rescale_l2(&X, d, rlk2, out); ctx2_free(&X);
}

/* HE-C^3 of one (query, set) pair one level up (hoisted order, reading R8): level-2 inputs
 * qct, sct [p][2][3][N] -> tensor over 3 limbs -> relin_rescale_l2 -> log2(s) ladder steps
 * C = C + Rot(C, 2^(i-1)) at level 1 (rotate1, keys gkl).  out [2][2][N] (level 1). */
static void he_c3_pair_l2(const ctx2_t *X, int p, int log_s, const uint64_t *rlk2, const uint64_t *gkl,
                          const uint64_t *qct, const uint64_t *sct, uint64_t *out)
{
    const int N = X->c.N;
    uint64_t *d = calloc((size_t)9 * N, sizeof(uint64_t)), *t = malloc(sizeof(uint64_t) * N);
    uint64_t *rot = malloc(sizeof(uint64_t) * 4 * N);
    for (int i = 0; i < p; i++) {
        const uint64_t *ca = qct + (size_t)i * 6 * N, *cb = sct + (size_t)i * 6 * N;
        for (int l = 0; l < 3; l++) {
            const uint64_t q = l2_q(X, l);
            const ring_t *R = l2_R(X, l);
            const uint64_t *a0 = ca + (size_t)l * N, *a1 = ca + (size_t)(3 + l) * N;
            const uint64_t *b0 = cb + (size_t)l * N, *b1 = cb + (size_t)(3 + l) * N;
            uint64_t *d0 = d + (size_t)l * N, *d1 = d + (size_t)(3 + l) * N, *d2 = d + (size_t)(6 + l) * N;
            poly_mul(R, a0, b0, t); poly_add(q, N, d0, t, d0);
            poly_mul(R, a0, b1, t); poly_add(q, N, d1, t, d1);
            poly_mul(R, a1, b0, t); poly_add(q, N, d1, t, d1);
            poly_mul(R, a1, b1, t); poly_add(q, N, d2, t, d2);
        }
    }
    relin_rescale_l2(X, d, rlk2, out);
    for (int i = 1; i <= log_s; i++) {
        rotate1(&X->c, out, (uint64_t)1 << (i - 1), gkl + (size_t)(i - 1) * 12 * N, rot);
        for (int cl = 0; cl < 4; cl++)
            poly_add(X->c.q[cl & 1], N, out + (size_t)cl * N, rot + (size_t)cl * N, out + (size_t)cl * N);
    }
    free(d); free(t); free(rot);
}

/* Compression of one result: level 1 C_t -> Res_q1(Mul(P)(C_t, M)) (level 0), then the
 * right rotation by u = t mod s (left rotation by S - u, key gkc[u-1]); out [2][1][N] */
static void compress_one(const ctx2_t *X, int u, const int64_t *mask, const uint64_t *gkc, const uint64_t *in,
                         uint64_t *out)
{
    const int N = X->c.N;
    uint64_t *m = malloc(sizeof(uint64_t) * N), *t = malloc(sizeof(uint64_t) * 4 * N);
    uint64_t *r0 = malloc(sizeof(uint64_t) * 2 * N);
    for (int cl = 0; cl < 4; cl++) {
        const uint64_t q = X->c.q[cl & 1];
        for (int k = 0; k < N; k++) m[k] = from_signed(mask[k], q);
        poly_mul(&X->c.R[cl & 1], in + (size_t)cl * N, m, t + (size_t)cl * N);
    }
    rescale(&X->c, t, u ? r0 : out);
    if (u) rotate(&X->c, r0, (uint64_t)(N / 2 - u), gkc + (size_t)(u - 1) * 4 * N, out);
    free(m); free(t); free(r0);
}

typedef struct {
    const ctx2_t *X;
    int p, log_s, s;
    const uint64_t *rlk2, *gkl, *gkc, *db, *q;
    const int64_t *mask;
    int64_t n_sets, nq, n_groups;
    uint64_t *out;
    int64_t next;
    pthread_mutex_t mu;
} cjob_t;

static void *cworker(void *arg)
{
    cjob_t *J = (cjob_t *)arg;
    const int N = J->X->c.N, p = J->p, s = J->s;
    const size_t st = (size_t)p * 6 * N;
    uint64_t *C = malloc(sizeof(uint64_t) * 4 * N), *o = malloc(sizeof(uint64_t) * 2 * N);
    for (;;) {
        pthread_mutex_lock(&J->mu);
        int64_t w = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (w >= J->nq * J->n_groups) break;
        const int64_t qi = w / J->n_groups, g = w % J->n_groups;
        uint64_t *acc = J->out + (size_t)w * 2 * N;
        memset(acc, 0, sizeof(uint64_t) * 2 * N);
        for (int u = 0; u < s; u++) {
            const int64_t t = g * s + u;
            if (t >= J->n_sets) break;
            he_c3_pair_l2(J->X, p, J->log_s, J->rlk2, J->gkl, J->q + (size_t)qi * st, J->db + (size_t)t * st, C);
            compress_one(J->X, u, J->mask, J->gkc, C, o);
            poly_add(J->X->c.q[0], 2 * N, acc, o, acc);
        }
    }
    free(C); free(o);
    return NULL;
}

/* The compressed scan: db [n_sets][p][2][3][N] and q [nq][p][2][3][N] at level 2 ->
 * out [nq][ceil(n_sets / s)][2][1][N] (level 0): packed ciphertext g holds, at slot k s + u, the
 * score of set g s + u's block k. */
int or_match_cmp(int logN, int d, int p, const uint64_t *rlk2, const uint64_t *gkl, const uint64_t *gkc,
                 const int64_t *mask, const uint64_t *db, int64_t n_sets, const uint64_t *q, int64_t nq, uint64_t *out,
                 int n_threads)
{
    if (p <= 0 || d % p) return -1;
    const int s = d / p;
    int log_s = 0;
    while ((1 << log_s) < s) log_s++;
    if ((1 << log_s) != s) return -1;
    ctx2_t X;
    ctx2_init(&X, logN);
    cjob_t J;
    memset(&J, 0, sizeof J);
    J.X = &X; J.p = p; J.log_s = log_s; J.s = s; J.rlk2 = rlk2; J.gkl = gkl; J.gkc = gkc; J.db = db; J.q = q;
    J.mask = mask; J.n_sets = n_sets; J.nq = nq; J.n_groups = (n_sets + s - 1) / s; J.out = out;
    pthread_mutex_init(&J.mu, NULL);
    if (n_threads < 1) n_threads = 1;
    pthread_t *th = malloc(sizeof(pthread_t) * n_threads);
    for (int i = 0; i < n_threads; i++) pthread_create(&th[i], NULL, cworker, &J);
    for (int i = 0; i < n_threads; i++) pthread_join(th[i], NULL);
    free(th);
    pthread_mutex_destroy(&J.mu);
    ctx2_free(&X);
    return 0;
}
