// host.cpp -- host (client-side) part of libblindmatch: parameters, key generation,
// packing + encoding, decryption, argmax.  Compiled by g++ (needs libquadmath for the
// exact Gaussian CDT).  Device work lives in device.cu.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstring>
#include <mutex>
#include <new>
#include <thread>
#include <vector>
#include <quadmath.h>
#include <cerrno>
#include <cstdlib>
#include <sys/random.h>

#include "bm_common.cuh"
#include "bm_host.h"

using u128 = unsigned __int128;

namespace bm {

uint64_t mulmod_h(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)((u128)a * b % q); }
static uint64_t powmod_h(uint64_t a, uint64_t e, uint64_t q)
{
    uint64_t r = 1;
    a %= q;
    for (; e; e >>= 1, a = mulmod_h(a, a, q))
        if (e & 1) r = mulmod_h(r, a, q);
    return r;
}
static uint64_t inv_h(uint64_t a, uint64_t q) { return powmod_h(a, q - 2, q); }
uint64_t shoup_companion(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }

// Miller-Rabin with the 12 smallest prime bases (deterministic below 3.3e24)
static bool is_prime_h(uint64_t n)
{
    const uint64_t B[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return false;
    for (uint64_t b : B)
        if (n % b == 0) return n == b;
    uint64_t d = n - 1;
    int r = 0;
    while (!(d & 1)) d >>= 1, r++;
    for (uint64_t b : B) {
        uint64_t x = powmod_h(b, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int i = 1; i < r && comp; i++) {
            x = mulmod_h(x, x, n);
            if (x == n - 1) comp = false;
        }
        if (comp) return false;
    }
    return true;
}

static unsigned brev13_h(unsigned x)
{
    unsigned r = 0;
    for (int i = 0; i < LOGN; i++) r = (r << 1) | ((x >> i) & 1);
    return r;
}

static HostPrime g_primes[4];
static uint64_t g_cdt[19];
static std::once_flag g_once;

// discrete Gaussian CDT (sigma 3.2, |x| <= 19): floor(2^63 Pr(|X| <= k)) in binary128
static void make_cdt()
{
    __float128 sig2 = (__float128)32 / 10 * ((__float128)32 / 10), rho[20], Z = 0;
    for (int k = 0; k < 20; k++) rho[k] = expq(-(__float128)(k * k) / (2 * sig2));
    Z = rho[0];
    for (int k = 1; k < 20; k++) Z += 2 * rho[k];
    __float128 acc = 0, two63 = ldexpq((__float128)1, 63);
    for (int k = 0; k < 19; k++) {
        acc += (k == 0 ? rho[0] : 2 * rho[k]);
        g_cdt[k] = (uint64_t)floorq(two63 * acc / Z);
    }
}

static void init_tables()
{
    const uint64_t Qs[4] = {Q0, Q1, QP, Q2};
    for (int i = 0; i < 4; i++) {
        HostPrime &H = g_primes[i];
        H.q = Qs[i];
        // psi: the first g^((q-1)/2N), g = 3, 5, 7, ..., with psi^N = -1 (order exactly 2N)
        for (uint64_t g = 3;; g += 2) {
            uint64_t c = powmod_h(g, (H.q - 1) / (2 * N), H.q);
            if (powmod_h(c, N, H.q) == H.q - 1) { H.psi = c; break; }
        }
        H.fwd.resize(N);
        H.inv.resize(N);
        uint64_t ipsi = inv_h(H.psi, H.q);
        for (unsigned k = 0; k < (unsigned)N; k++) {
            unsigned e = brev13_h(k);
            H.fwd[k] = powmod_h(H.psi, e, H.q);
            H.inv[k] = powmod_h(ipsi, e, H.q);
        }
        H.ninv = inv_h(N, H.q);
    }
    make_cdt();
}

const HostPrime &host_prime(int i)
{
    std::call_once(g_once, init_tables);
    return g_primes[i];
}
const uint64_t *host_cdt()
{
    std::call_once(g_once, init_tables);
    return g_cdt;
}

// host negacyclic NTT, same orders as the device kernels (CT with psi^brev, GS inverse)
void host_ntt_fwd(uint64_t *a, int pi)
{
    const HostPrime &H = host_prime(pi);
    const uint64_t q = H.q;
    for (int m = 1, t = N / 2; m < N; m <<= 1, t >>= 1)
        for (int i = 0; i < m; i++) {
            uint64_t w = H.fwd[m + i];
            for (int j = 2 * i * t; j < 2 * i * t + t; j++) {
                uint64_t u = a[j], v = mulmod_h(a[j + t], w, q);
                a[j] = (u + v) % q;
                a[j + t] = (u + q - v) % q;
            }
        }
}
void host_ntt_inv(uint64_t *a, int pi)
{
    const HostPrime &H = host_prime(pi);
    const uint64_t q = H.q;
    for (int m = N / 2, t = 1; m >= 1; m >>= 1, t <<= 1)
        for (int i = 0; i < m; i++) {
            uint64_t w = H.inv[m + i];
            for (int j = 2 * i * t; j < 2 * i * t + t; j++) {
                uint64_t u = a[j], v = a[j + t];
                a[j] = (u + v) % q;
                a[j + t] = mulmod_h((u + q - v) % q, w, q);
            }
        }
    for (int j = 0; j < N; j++) a[j] = mulmod_h(a[j], H.ninv, q);
}

} // namespace bm

using namespace bm;

// ================================================================== helpers
static uint64_t to_res(int64_t x, uint64_t q)
{
    if (x >= 0) return (uint64_t)x % q;
    uint64_t r = (uint64_t)(-(x + 1)) % q; // -(x+1) >= 0 avoids INT64_MIN overflow
    return q - 1 - r;
}

// c = a * b mod (X^N+1, q_pi), all canonical
static void poly_mul_h(const uint64_t *a, const uint64_t *b, uint64_t *c, int pi)
{
    std::vector<uint64_t> A(a, a + N), B(b, b + N);
    host_ntt_fwd(A.data(), pi);
    host_ntt_fwd(B.data(), pi);
    const uint64_t q = host_prime(pi).q;
    for (int k = 0; k < N; k++) A[k] = mulmod_h(A[k], B[k], q);
    host_ntt_inv(A.data(), pi);
    memcpy(c, A.data(), sizeof(uint64_t) * N);
}

// ------------------------------------------------------------------ randomness mode
// BM_RNG_OS (default): the keygen family keys its ChaCha20 streams with the seed AND a 160-bit process
// key drawn once from getrandom() (224 bits of key entropy; the same seed gives the same secret within
// the process, so bm_evk_add_hoisted / bm_xk_keygen / bm_ck_keygen still match bm_keygen), and every
// encryption call draws a fresh 160-bit extension (two batches encrypted with the same seed and object
// numbers share no randomness).  BM_RNG_SEEDED: all-zero extensions, the reproducible streams of
// DESIGN.md reading R14 that the oracle implements (tests, bench).
static std::atomic<int> g_rng_mode(BM_RNG_OS);
static uint32_t g_proc_kx[5];
static std::once_flag g_proc_once;
static const uint32_t g_zero_kx[5] = {0, 0, 0, 0, 0};

static void os_random(void *buf, size_t n)
{
    uint8_t *p = (uint8_t *)buf;
    while (n) {
        const ssize_t r = getrandom(p, n, 0);
        if (r < 0) {
            if (errno == EINTR) continue;
            abort(); // no entropy source: refuse to produce keys or ciphertexts
        }
        p += r;
        n -= (size_t)r;
    }
}

namespace bm {
const uint32_t *rng_keygen_kx()
{
    if (g_rng_mode.load() == BM_RNG_SEEDED) return g_zero_kx;
    std::call_once(g_proc_once, [] { os_random(g_proc_kx, sizeof(g_proc_kx)); });
    return g_proc_kx;
}
void rng_encrypt_kx(uint32_t out[5])
{
    if (g_rng_mode.load() == BM_RNG_SEEDED) {
        memset(out, 0, 5 * sizeof(uint32_t));
        return;
    }
    os_random(out, 5 * sizeof(uint32_t));
}
} // namespace bm

// draws n u64 values of a stream, in order
static void stream_draws(uint64_t seed, uint32_t purpose, uint64_t obj, uint32_t sub, int n, uint64_t *out)
{
    Stream st = make_stream(seed, purpose, obj, sub, rng_keygen_kx());
    uint64_t d[8];
    for (int b = 0; b * 8 < n; b++) {
        chacha_draws(st, (uint32_t)b, d);
        for (int i = 0; i < 8 && b * 8 + i < n; i++) out[b * 8 + i] = d[i];
    }
}
static void sample_uniform(uint64_t seed, uint32_t purpose, uint64_t obj, uint32_t sub, uint64_t q, uint64_t *out)
{
    std::vector<uint64_t> d(2 * N);
    stream_draws(seed, purpose, obj, sub, 2 * N, d.data());
    for (int k = 0; k < N; k++) out[k] = (uint64_t)((((u128)d[2 * k + 1] << 64) | d[2 * k]) % q);
}
static void sample_small(uint64_t seed, uint32_t purpose, uint64_t obj, int gauss, int64_t *out)
{
    std::vector<uint64_t> d(N);
    stream_draws(seed, purpose, obj, 0, N, d.data());
    const uint64_t *cdt = host_cdt();
    for (int k = 0; k < N; k++) out[k] = gauss ? gauss_of(d[k], cdt) : ternary_of(d[k]);
}

static void make_digest(uint8_t out[32])
{
    // 4 x FNV-1a-64 over (N, q0, q1, P, scale bits)
    uint64_t words[5] = {(uint64_t)N, Q0, Q1, QP, 40};
    for (int h = 0; h < 4; h++) {
        uint64_t x = 0xcbf29ce484222325ull ^ (uint64_t)(h * 0x9e3779b97f4a7c15ull);
        for (int w = 0; w < 5; w++)
            for (int b = 0; b < 8; b++) {
                x ^= (words[w] >> (8 * b)) & 0xff;
                x *= 0x100000001b3ull;
            }
        memcpy(out + 8 * h, &x, 8);
    }
}

static bool pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

// ================================================================== C ABI (host part)
extern "C" {

int bm_rng_mode(int32_t mode)
{
    if (mode != BM_RNG_SEEDED && mode != BM_RNG_OS) return BM_ERR_INVALID_ARG;
    g_rng_mode.store(mode);
    return BM_OK;
}
int32_t bm_get_rng_mode(void) { return g_rng_mode.load(); }

int bm_params_init(bm_params *o, int32_t d, int32_t p)
{
    if (!o) return BM_ERR_INVALID_ARG;
    if (!pow2(d) || !pow2(p) || p > d || d > SLOTS) return BM_ERR_INVALID_LAYOUT;
    const uint64_t Qs[4] = {Q0, Q1, QP, Q2};
    for (uint64_t q : Qs)
        if (!is_prime_h(q) || (q - 1) % (2 * N) != 0) return BM_ERR_INVALID_PRIME;
    // HE-standard 128-bit classical bound at N = 8192: log2(PQ) <= 218
    double logpq = std::log2((double)Q0) + std::log2((double)Q1) + std::log2((double)QP);
    if (logpq > 218.0) return BM_ERR_INSECURE_PARAMS;
    memset(o, 0, sizeof *o);
    o->logN = LOGN;
    o->N = N;
    o->slots = SLOTS;
    o->d = d;
    o->p = p;
    o->s = d / p;
    o->B = SLOTS / o->s;
    o->log_s = 0;
    while ((1 << o->log_s) < o->s) o->log_s++;
    o->q[0] = Q0;
    o->q[1] = Q1;
    o->q[2] = QP;
    o->scale = std::ldexp(1.0, 40);
    o->out_scale = std::ldexp(1.0, 80) / (double)Q1;
    o->q2 = Q2;
    make_digest(o->digest);
    host_prime(0); // build tables once
    return BM_OK;
}

// Galois key of a left rotation by r (g = 5^r mod 2N) over {q0, P}, PRNG object obj:
// (-a s + e + (P mod q0) sigma_g(s) [q0], a) and (-a s + e [P], a); out [2 comps][2 limbs][N]
static void galois_key(uint64_t seed, const std::vector<int64_t> &sv, uint64_t r, uint64_t obj, uint64_t *out)
{
    const uint64_t Qs[3] = {Q0, Q1, QP};
    const uint64_t g = powmod_h(5, r, 2 * N);
    std::vector<int64_t> ev(N);
    std::vector<uint64_t> s(N), e(N), a(N), t(N), sg(N);
    sample_small(seed, P_GK_E, obj, 1, ev.data());
    for (int li = 0; li < 2; li++) {
        int l = li ? 2 : 0;
        uint64_t q = Qs[l];
        for (int k = 0; k < N; k++) s[k] = to_res(sv[k], q), e[k] = to_res(ev[k], q);
        sample_uniform(seed, P_GK_A, obj, (uint32_t)l, q, a.data());
        poly_mul_h(a.data(), s.data(), t.data(), l);
        uint64_t *b = out + (size_t)(0 * 2 + li) * N;
        uint64_t *aa = out + (size_t)(1 * 2 + li) * N;
        for (int k = 0; k < N; k++) b[k] = (e[k] + q - t[k]) % q, aa[k] = a[k];
        if (l == 0) {
            // sigma_g(s): coefficient k -> k g mod 2N, negated past N
            std::fill(sg.begin(), sg.end(), 0);
            for (int k = 0; k < N; k++) {
                uint64_t x = (uint64_t)k * g % (2 * N);
                if (x < (uint64_t)N) sg[x] = s[k];
                else sg[x - N] = (q - s[k]) % q;
            }
            uint64_t pm = QP % q;
            for (int k = 0; k < N; k++) b[k] = (b[k] + mulmod_h(sg[k], pm, q)) % q;
        }
    }
}

// f2: Galois keys of every rotation r = 1..s-1 for the hoisted rotation sum,
// PRNG object HROT_OBJ + r (disjoint from the ladder keys' objects i < 13)
constexpr uint64_t HROT_OBJ = 64;
int bm_evk_add_hoisted(const bm_params *prm, uint64_t seed, bm_evk *evk)
{
    if (!prm || !evk) return BM_ERR_INVALID_ARG;
    if (memcmp(evk->digest, prm->digest, 32)) return BM_ERR_KEY_MISMATCH;
    std::vector<int64_t> sv(N);
    sample_small(seed, P_SK, 0, 0, sv.data());
    const int n = prm->s - 1;
    evk->n_hrot = n;
    evk->hgk.assign((size_t)n * 4 * N, 0);
    for (int r = 1; r <= n; r++) galois_key(seed, sv, (uint64_t)r, HROT_OBJ + r, &evk->hgk[(size_t)(r - 1) * 4 * N]);
    return BM_OK;
}

int bm_keygen(const bm_params *prm, uint64_t seed, bm_sk **skp, bm_pk **pkp, bm_evk **evkp)
{
    if (!prm) return BM_ERR_INVALID_ARG;
    const uint64_t Qs[3] = {Q0, Q1, QP};
    std::vector<int64_t> sv(N), ev(N);
    std::vector<uint64_t> s(N), e(N), a(N), t(N), s2(N), sg(N);
    sample_small(seed, P_SK, 0, 0, sv.data());

    bm_sk *sk = new (std::nothrow) bm_sk;
    bm_pk *pk = new (std::nothrow) bm_pk;
    bm_evk *evk = new (std::nothrow) bm_evk;
    if (!sk || !pk || !evk) { delete sk; delete pk; delete evk; return BM_ERR_OOM; }
    memcpy(sk->digest, prm->digest, 32);
    memcpy(pk->digest, prm->digest, 32);
    memcpy(evk->digest, prm->digest, 32);
    sk->s.resize(N);
    for (int k = 0; k < N; k++) sk->s[k] = (int8_t)sv[k];

    // pk = (-a s + e, a) over {q0, q1}
    pk->v.assign(4 * (size_t)N, 0);
    sample_small(seed, P_PK_E, 0, 1, ev.data());
    for (int l = 0; l < 2; l++) {
        uint64_t q = Qs[l];
        for (int k = 0; k < N; k++) s[k] = to_res(sv[k], q), e[k] = to_res(ev[k], q);
        sample_uniform(seed, P_PK_A, 0, (uint32_t)l, q, a.data());
        poly_mul_h(a.data(), s.data(), t.data(), l);
        uint64_t *b = &pk->v[(size_t)(0 * 2 + l) * N], *aa = &pk->v[(size_t)(1 * 2 + l) * N];
        for (int k = 0; k < N; k++) b[k] = (e[k] + q - t[k]) % q, aa[k] = a[k];
    }

    // rlk_j over {q0, q1, P}: (-a s + e + [l == j] (P mod q_l) s^2, a)
    evk->rlk.assign(12 * (size_t)N, 0);
    for (int j = 0; j < 2; j++) {
        sample_small(seed, P_RLK_E, (uint64_t)j, 1, ev.data());
        for (int l = 0; l < 3; l++) {
            uint64_t q = Qs[l];
            for (int k = 0; k < N; k++) s[k] = to_res(sv[k], q), e[k] = to_res(ev[k], q);
            sample_uniform(seed, P_RLK_A, (uint64_t)j, (uint32_t)l, q, a.data());
            poly_mul_h(a.data(), s.data(), t.data(), l);
            uint64_t *b = &evk->rlk[((size_t)(j * 2 + 0) * 3 + l) * N];
            uint64_t *aa = &evk->rlk[((size_t)(j * 2 + 1) * 3 + l) * N];
            for (int k = 0; k < N; k++) b[k] = (e[k] + q - t[k]) % q, aa[k] = a[k];
            if (l == j) {
                poly_mul_h(s.data(), s.data(), s2.data(), l);
                uint64_t pm = QP % q;
                for (int k = 0; k < N; k++) b[k] = (b[k] + mulmod_h(s2[k], pm, q)) % q;
            }
        }
    }

    // gk_i (rotation r = 2^i), PRNG object i
    evk->n_rot = prm->log_s;
    evk->gk.assign((size_t)evk->n_rot * 4 * N, 0);
    for (int i = 0; i < evk->n_rot; i++) galois_key(seed, sv, (uint64_t)1 << i, (uint64_t)i, &evk->gk[(size_t)i * 4 * N]);
    if (skp) *skp = sk; else delete sk;
    if (pkp) *pkp = pk; else delete pk;
    if (evkp) *evkp = evk; else delete evk;
    return BM_OK;
}

static bool canonical(const uint64_t *v, size_t n_polys, const int *limb_primes, int n_limbs);

// Level-1 Galois key of the left rotation by r (f3/f4/f1), 2 digits j over {q0, q1, P}:
// (-a s + e + [l = j] (P mod q_l) sigma_{5^r}(s), a), a from (P_GK1_A, object 2r + j, sub-stream l),
// e from (P_GK1_E, object 2r + j); out [2 digits][2 comps][3 limbs][N]
static void galois_key1(uint64_t seed, const std::vector<int64_t> &sv, uint64_t r, uint64_t *out)
{
    const uint64_t Qs[3] = {Q0, Q1, QP};
    const uint64_t g = powmod_h(5, r, 2 * N);
    std::vector<int64_t> ev(N);
    std::vector<uint64_t> s(N), e(N), a(N), t(N), sg(N);
    for (int j = 0; j < 2; j++) {
        const uint64_t obj = 2 * r + (uint64_t)j;
        sample_small(seed, P_GK1_E, obj, 1, ev.data());
        for (int l = 0; l < 3; l++) {
            const uint64_t q = Qs[l];
            for (int k = 0; k < N; k++) s[k] = to_res(sv[k], q), e[k] = to_res(ev[k], q);
            sample_uniform(seed, P_GK1_A, obj, (uint32_t)l, q, a.data());
            poly_mul_h(a.data(), s.data(), t.data(), l);
            uint64_t *b = out + (((size_t)j * 2 + 0) * 3 + l) * N;
            uint64_t *aa = out + (((size_t)j * 2 + 1) * 3 + l) * N;
            for (int k = 0; k < N; k++) b[k] = (e[k] + q - t[k]) % q, aa[k] = a[k];
            if (l == j) {
                std::fill(sg.begin(), sg.end(), 0);
                for (int k = 0; k < N; k++) {
                    uint64_t y = (uint64_t)k * g % (2 * N);
                    if (y < (uint64_t)N) sg[y] = s[k];
                    else sg[y - N] = (q - s[k]) % q;
                }
                const uint64_t pm = QP % q;
                for (int k = 0; k < N; k++) b[k] = (b[k] + mulmod_h(sg[k], pm, q)) % q;
            }
        }
    }
}

// f1 (reading R28): 3-digit relinearisation key over {q0, q1, q2, P} (b = -a s + e + [l = j](P mod q_l) s^2,
// a from (P_RLK2_A, object j, sub-stream l), e from (P_RLK2_E, object j)), the ladder's level-1 Galois keys
// of 2^i (i < log2 s) and the level-0 keys of the right rotations by u = 1..s-1 (left by S - u, object
// CMP_OBJ + u)
constexpr uint64_t CMP_OBJ = 4096;
int bm_ck_keygen(const bm_params *prm, uint64_t seed, bm_ck **out)
{
    if (!prm || !out) return BM_ERR_INVALID_ARG;
    const uint64_t Q4[4] = {Q0, Q1, Q2, QP};
    const int pi4[4] = {0, 1, 3, 2};
    bm_ck *x = new (std::nothrow) bm_ck;
    if (!x) return BM_ERR_OOM;
    memcpy(x->digest, prm->digest, 32);
    x->d = prm->d;
    x->p = prm->p;
    x->log_s = prm->log_s;
    std::vector<int64_t> sv(N), ev(N);
    std::vector<uint64_t> s(N), e(N), a(N), t(N), s2(N);
    sample_small(seed, P_SK, 0, 0, sv.data());
    x->rlk2.assign(24 * (size_t)N, 0);
    for (int j = 0; j < 3; j++) {
        sample_small(seed, P_RLK2_E, (uint64_t)j, 1, ev.data());
        for (int l = 0; l < 4; l++) {
            const uint64_t q = Q4[l];
            for (int k = 0; k < N; k++) s[k] = to_res(sv[k], q), e[k] = to_res(ev[k], q);
            sample_uniform(seed, P_RLK2_A, (uint64_t)j, (uint32_t)l, q, a.data());
            poly_mul_h(a.data(), s.data(), t.data(), pi4[l]);
            uint64_t *b = &x->rlk2[(((size_t)j * 2 + 0) * 4 + l) * N], *aa = &x->rlk2[(((size_t)j * 2 + 1) * 4 + l) * N];
            for (int k = 0; k < N; k++) b[k] = (e[k] + q - t[k]) % q, aa[k] = a[k];
            if (l == j) {
                poly_mul_h(s.data(), s.data(), s2.data(), pi4[l]);
                const uint64_t pm = QP % q;
                for (int k = 0; k < N; k++) b[k] = (b[k] + mulmod_h(s2[k], pm, q)) % q;
            }
        }
    }
    x->gkl.assign((size_t)x->log_s * 12 * N, 0);
    for (int i = 0; i < x->log_s; i++) galois_key1(seed, sv, (uint64_t)1 << i, &x->gkl[(size_t)i * 12 * N]);
    const int s_ = prm->s;
    x->gkc.assign((size_t)(s_ - 1) * 4 * N, 0);
    for (int u = 1; u < s_; u++) galois_key(seed, sv, (uint64_t)(SLOTS - u), CMP_OBJ + u, &x->gkc[(size_t)(u - 1) * 4 * N]);
    *out = x;
    return BM_OK;
}
void bm_ck_free(bm_ck *x) { delete x; }
int bm_ck_export(const bm_ck *x, uint64_t *rlk2, uint64_t *gkl, uint64_t *gkc)
{
    if (!x) return BM_ERR_INVALID_ARG;
    if (rlk2) memcpy(rlk2, x->rlk2.data(), x->rlk2.size() * 8);
    if (gkl) memcpy(gkl, x->gkl.data(), x->gkl.size() * 8);
    if (gkc) memcpy(gkc, x->gkc.data(), x->gkc.size() * 8);
    return BM_OK;
}

// f3 expansion keys (reading R26).  pk limb q2: (-a s + e, a) with pk's error (P_PK_E,
// object 0) and a from (P_PK_A, object 0, sub-stream 3).  Level-1 Galois key of the left rotation
// by r = s 2^t, digit j: over {q0, q1, P}, (-a s + e + [l = j] (P mod q_l) sigma_{5^r}(s), a) with
// a from (P_GK1_A, object 2r + j, sub-stream l) and e from (P_GK1_E, object 2r + j).
int bm_xk_keygen(const bm_params *prm, uint64_t seed, bm_xk **out)
{
    if (!prm || !out) return BM_ERR_INVALID_ARG;
    bm_xk *x = new (std::nothrow) bm_xk;
    if (!x) return BM_ERR_OOM;
    memcpy(x->digest, prm->digest, 32);
    x->d = prm->d;
    x->p = prm->p;
    // strides s 2^t for t < log2 B: the expansion uses t < log2 p, the enrollment all of them
    x->n_rot = 0;
    while ((1 << x->n_rot) < prm->B) x->n_rot++;
    std::vector<int64_t> sv(N), ev(N);
    std::vector<uint64_t> s(N), e(N), a(N), t(N), sg(N);
    sample_small(seed, P_SK, 0, 0, sv.data());
    // pk limb q2
    x->pk_q2.assign(2 * (size_t)N, 0);
    sample_small(seed, P_PK_E, 0, 1, ev.data());
    for (int k = 0; k < N; k++) s[k] = to_res(sv[k], Q2), e[k] = to_res(ev[k], Q2);
    sample_uniform(seed, P_PK_A, 0, 3, Q2, a.data());
    poly_mul_h(a.data(), s.data(), t.data(), 3);
    for (int k = 0; k < N; k++) x->pk_q2[k] = (e[k] + Q2 - t[k]) % Q2, x->pk_q2[N + k] = a[k];
    // level-1 Galois keys
    x->gk1.assign((size_t)x->n_rot * 12 * N, 0);
    for (int tt = 0; tt < x->n_rot; tt++) galois_key1(seed, sv, (uint64_t)prm->s << tt, &x->gk1[(size_t)tt * 12 * N]);
    *out = x;
    return BM_OK;
}
void bm_xk_free(bm_xk *x) { delete x; }
int bm_xk_export(const bm_xk *x, uint64_t *pk_q2, uint64_t *gk1, int32_t *n_rot)
{
    if (!x) return BM_ERR_INVALID_ARG;
    if (pk_q2) memcpy(pk_q2, x->pk_q2.data(), x->pk_q2.size() * 8);
    if (gk1) memcpy(gk1, x->gk1.data(), x->gk1.size() * 8);
    if (n_rot) *n_rot = x->n_rot;
    return BM_OK;
}
int bm_xk_import(const bm_params *prm, const uint64_t *pk_q2, const uint64_t *gk1, int32_t n_rot, bm_xk **out)
{
    if (!prm || !pk_q2 || (!gk1 && n_rot > 0) || !out) return BM_ERR_INVALID_ARG;
    int log_p = 0, log_b = 0;
    while ((1 << log_p) < prm->p) log_p++;
    while ((1 << log_b) < prm->B) log_b++;
    if (n_rot < log_p || n_rot > log_b) return BM_ERR_MISSING_ROTATION_KEY;
    const int pq2[1] = {3}, pk3[3] = {0, 1, 2};
    if (!canonical(pk_q2, 2, pq2, 1) || (n_rot && !canonical(gk1, (size_t)n_rot * 12, pk3, 3)))
        return BM_ERR_INVALID_ARG;
    bm_xk *x = new (std::nothrow) bm_xk;
    if (!x) return BM_ERR_OOM;
    memcpy(x->digest, prm->digest, 32);
    x->d = prm->d;
    x->p = prm->p;
    x->n_rot = n_rot;
    x->pk_q2.assign(pk_q2, pk_q2 + 2 * (size_t)N);
    x->gk1.assign(gk1, gk1 + (size_t)n_rot * 12 * N);
    *out = x;
    return BM_OK;
}

void bm_sk_free(bm_sk *x) { delete x; }
void bm_pk_free(bm_pk *x) { delete x; }
void bm_evk_free(bm_evk *x) { delete x; }

int bm_sk_export(const bm_sk *sk, int8_t *out)
{
    if (!sk || !out) return BM_ERR_INVALID_ARG;
    memcpy(out, sk->s.data(), N);
    return BM_OK;
}
int bm_pk_export(const bm_pk *pk, uint64_t *out)
{
    if (!pk || !out) return BM_ERR_INVALID_ARG;
    memcpy(out, pk->v.data(), pk->v.size() * 8);
    return BM_OK;
}
int bm_evk_export(const bm_evk *evk, uint64_t *rlk, uint64_t *gk, int32_t *n_rot)
{
    if (!evk) return BM_ERR_INVALID_ARG;
    if (rlk) memcpy(rlk, evk->rlk.data(), evk->rlk.size() * 8);
    if (gk) memcpy(gk, evk->gk.data(), evk->gk.size() * 8);
    if (n_rot) *n_rot = evk->n_rot;
    return BM_OK;
}

static bool canonical(const uint64_t *v, size_t n_polys, const int *limb_primes, int n_limbs)
{
    for (size_t p = 0; p < n_polys; p++) {
        uint64_t q = host_prime(limb_primes[p % n_limbs]).q;
        for (int k = 0; k < N; k++)
            if (v[p * N + k] >= q) return false;
    }
    return true;
}

int bm_sk_import(const bm_params *prm, const int8_t *in, bm_sk **out)
{
    if (!prm || !in || !out) return BM_ERR_INVALID_ARG;
    for (int k = 0; k < N; k++)
        if (in[k] < -1 || in[k] > 1) return BM_ERR_INVALID_ARG;
    bm_sk *sk = new (std::nothrow) bm_sk;
    if (!sk) return BM_ERR_OOM;
    memcpy(sk->digest, prm->digest, 32);
    sk->s.assign(in, in + N);
    *out = sk;
    return BM_OK;
}
int bm_pk_import(const bm_params *prm, const uint64_t *in, bm_pk **out)
{
    if (!prm || !in || !out) return BM_ERR_INVALID_ARG;
    const int lp[2] = {0, 1};
    if (!canonical(in, 4, lp, 2)) return BM_ERR_INVALID_ARG;
    bm_pk *pk = new (std::nothrow) bm_pk;
    if (!pk) return BM_ERR_OOM;
    memcpy(pk->digest, prm->digest, 32);
    pk->v.assign(in, in + 4 * (size_t)N);
    *out = pk;
    return BM_OK;
}
int bm_evk_import(const bm_params *prm, const uint64_t *rlk, const uint64_t *gk, int32_t n_rot, bm_evk **out)
{
    if (!prm || !rlk || !out || n_rot < 0 || (n_rot > 0 && !gk)) return BM_ERR_INVALID_ARG;
    const int lr[3] = {0, 1, 2}, lg[2] = {0, 2};
    if (!canonical(rlk, 12, lr, 3) || (n_rot && !canonical(gk, 4 * (size_t)n_rot, lg, 2))) return BM_ERR_INVALID_ARG;
    bm_evk *e = new (std::nothrow) bm_evk;
    if (!e) return BM_ERR_OOM;
    memcpy(e->digest, prm->digest, 32);
    e->n_rot = n_rot;
    e->rlk.assign(rlk, rlk + 12 * (size_t)N);
    if (n_rot) e->gk.assign(gk, gk + (size_t)n_rot * 4 * N);
    *out = e;
    return BM_OK;
}

// ------------------------------------------------------------------ encoding
// pt_k = round(Delta * (2/N) Re(sum_t X[t] w^(k t))), X[5^j mod 2N] = z_j, w = exp(i pi / N):
// one 2N-point complex FFT (positive exponent) per plaintext.  The twiddles w^m, m < N, come from
// one table computed in long double (a configs[3] database is 32,768 plaintexts: per-butterfly
// cos / sin calls made the encoder the setup's bottleneck).
static const std::vector<std::complex<double>> &fft_twiddles()
{
    static std::vector<std::complex<double>> w;
    static std::once_flag f;
    std::call_once(f, [] {
        w.resize(N);
        for (int m = 0; m < N; m++) {
            const long double a = 3.141592653589793238462643383279502884L * m / N; // 2 pi m / 2N
            w[m] = std::complex<double>((double)cosl(a), (double)sinl(a));
        }
    });
    return w;
}

static void fft_pos(std::vector<std::complex<double>> &a)
{
    const int n = (int)a.size(); // 2N
    const std::vector<std::complex<double>> &W = fft_twiddles();
    for (int i = 1, j = 0; i < n; i++) {
        int bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    for (int len = 2; len <= n; len <<= 1) {
        const int step = n / len; // w_len^k = exp(2 pi i k / len) = W[k n / len]
        for (int i = 0; i < n; i += len)
            for (int k = 0; k < len / 2; k++) {
                const std::complex<double> u = a[i + k], v = a[i + k + len / 2] * W[k * step];
                a[i + k] = u + v;
                a[i + k + len / 2] = u - v;
            }
    }
}

// run f(i) for i < n on up to hardware_concurrency threads (encoding is per plaintext independent);
// returns the first nonzero status
extern "C++" {
template <typename F> static int parallel_for(int64_t n, F f)
{
    int nt = (int)std::min<int64_t>(n, std::max(1u, std::thread::hardware_concurrency()));
    if (nt <= 1) {
        for (int64_t i = 0; i < n; i++)
            if (int rc = f(i)) return rc;
        return BM_OK;
    }
    std::atomic<int64_t> next(0);
    std::atomic<int> status(BM_OK);
    std::vector<std::thread> th;
    for (int t = 0; t < nt; t++)
        th.emplace_back([&] {
            for (int64_t i; (i = next.fetch_add(1)) < n && status.load() == BM_OK;)
                if (int rc = f(i)) status.store(rc);
        });
    for (auto &x : th) x.join();
    return status.load();
}
} // extern "C++"

static const std::vector<int> &slot_exp()
{
    static std::vector<int> e;
    static std::once_flag f;
    std::call_once(f, [] {
        e.resize(SLOTS);
        uint64_t x = 1;
        for (int j = 0; j < SLOTS; j++) e[j] = (int)x, x = x * 5 % (2 * N);
    });
    return e;
}

static int encode_slots(const double *z, int64_t *pt, double delta = 1099511627776.0 /* 2^40 */)
{
    const std::vector<int> &e = slot_exp();
    std::vector<std::complex<double>> X(2 * N);
    for (int j = 0; j < SLOTS; j++) X[e[j]] = z[j];
    fft_pos(X);
    const double scale = delta * 2.0 / N;
    for (int k = 0; k < N; k++) {
        double v = scale * X[k].real();
        if (!std::isfinite(v) || std::fabs(v) > 9.0e18) return BM_ERR_MAGNITUDE;
        pt[k] = (int64_t)(v >= 0 ? std::floor(v + 0.5) : -std::floor(-v + 0.5));
    }
    return BM_OK;
}

static int unit_rows(const double *x, int64_t n, int d, std::vector<double> &out)
{
    out.resize((size_t)n * d);
    for (int64_t r = 0; r < n; r++) {
        double ss = 0;
        for (int i = 0; i < d; i++) {
            double v = x[r * d + i];
            if (!std::isfinite(v)) return BM_ERR_MAGNITUDE;
            ss += v * v;
        }
        if (!(ss > 0)) return BM_ERR_ZERO_VECTOR;
        double inv = 1.0 / std::sqrt(ss);
        for (int i = 0; i < d; i++) out[r * d + i] = x[r * d + i] * inv;
    }
    return BM_OK;
}

int bm_encode_db(const bm_params *prm, const double *tmpl, int64_t n, int64_t first_set, int64_t n_sets, int64_t *pt)
{
    if (!prm || (!tmpl && n > 0) || !pt || n < 0 || first_set < 0 || n_sets < 0) return BM_ERR_INVALID_ARG;
    const int d = prm->d, p = prm->p, s = prm->s, B = prm->B;
    int64_t lo = first_set * B, hi = std::min<int64_t>(n, (first_set + n_sets) * B);
    std::vector<double> unit;
    if (hi > lo) {
        int rc = unit_rows(tmpl + lo * d, hi - lo, d, unit);
        if (rc) return rc;
    }
    return parallel_for(n_sets * p, [&](int64_t ti) {
        const int64_t t = ti / p;
        const int i = (int)(ti % p);
        std::vector<double> z(SLOTS, 0.0);
        for (int k = 0; k < B; k++) {
            int64_t u = (first_set + t) * B + k;
            if (u >= n) break;
            const double *v = &unit[(u - lo) * d];
            for (int j = 0; j < s; j++) z[k * s + j] = v[i * s + j];
        }
        return encode_slots(z.data(), pt + ((size_t)t * p + i) * N);
    });
}

int bm_encode_query(const bm_params *prm, const double *q, int64_t nq, int64_t *pt)
{
    if (!prm || (!q && nq > 0) || !pt || nq < 0) return BM_ERR_INVALID_ARG;
    const int d = prm->d, p = prm->p, s = prm->s;
    std::vector<double> unit;
    if (nq) {
        int rc = unit_rows(q, nq, d, unit);
        if (rc) return rc;
    }
    return parallel_for(nq * p, [&](int64_t ji) {
        const int64_t j = ji / p;
        const int i = (int)(ji % p);
        std::vector<double> z(SLOTS);
        for (int x = 0; x < SLOTS; x++) z[x] = unit[j * d + i * s + (x % s)];
        return encode_slots(z.data(), pt + ((size_t)j * p + i) * N);
    });
}

// f3: the client's single query ciphertext holds the unit query tiled S/d times,
// encoded at 2^40; the expansion masks X_i[x] = [(x mod d) in [i s, (i+1) s)]
// are encoded at scale q2, so that Res by q2 leaves the expanded parts at scale exactly 2^40.
int bm_encode_query_tiled(const bm_params *prm, const double *q, int64_t nq, int64_t *pt)
{
    if (!prm || (!q && nq > 0) || !pt || nq < 0) return BM_ERR_INVALID_ARG;
    const int d = prm->d;
    std::vector<double> unit;
    if (nq) {
        int rc = unit_rows(q, nq, d, unit);
        if (rc) return rc;
    }
    std::vector<double> z(SLOTS);
    for (int64_t j = 0; j < nq; j++) {
        for (int x = 0; x < SLOTS; x++) z[x] = unit[j * d + (x % d)];
        int rc = encode_slots(z.data(), pt + (size_t)j * N);
        if (rc) return rc;
    }
    return BM_OK;
}
int bm_encode_masks(const bm_params *prm, int32_t kind, int64_t *pt)
{
    if (!prm || !pt || (kind != 0 && kind != 1)) return BM_ERR_INVALID_ARG;
    const int d = prm->d, s = prm->s;
    std::vector<double> z(SLOTS);
    for (int i = 0; i < prm->p; i++) {
        for (int x = 0; x < SLOTS; x++) {
            const int y = kind == 0 ? x % d : x; // X_i is d-periodic, E_i is one block
            z[x] = (y >= i * s && y < (i + 1) * s) ? 1.0 : 0.0;
        }
        int rc = encode_slots(z.data(), pt + (size_t)i * N, (double)Q2);
        if (rc) return rc;
    }
    return BM_OK;
}

// f1: the compression's score mask M[x] = [x mod s = 0] at scale q1 (Res by q1 restores the
// input's scale)
int bm_encode_cmp_mask(const bm_params *prm, int64_t *pt)
{
    if (!prm || !pt) return BM_ERR_INVALID_ARG;
    std::vector<double> z(SLOTS);
    for (int x = 0; x < SLOTS; x++) z[x] = (x % prm->s) == 0 ? 1.0 : 0.0;
    return encode_slots(z.data(), pt, (double)Q1);
}

// f4: the client's enrollment ciphertext holds the unit template in slots [0, d), zeros elsewhere
// ("occupies the initial slots ... padded with zeros")
int bm_encode_enroll(const bm_params *prm, const double *v, int64_t n, int64_t *pt)
{
    if (!prm || (!v && n > 0) || !pt || n < 0) return BM_ERR_INVALID_ARG;
    const int d = prm->d;
    std::vector<double> unit;
    if (n) {
        int rc = unit_rows(v, n, d, unit);
        if (rc) return rc;
    }
    std::vector<double> z(SLOTS, 0.0);
    for (int64_t j = 0; j < n; j++) {
        for (int x = 0; x < d; x++) z[x] = unit[j * d + x];
        int rc = encode_slots(z.data(), pt + (size_t)j * N);
        if (rc) return rc;
    }
    return BM_OK;
}

// ------------------------------------------------------------------ serialisation
// Frame: 64-byte header {char magic[4] = "BMCT", u32 version = 1, u8 digest[32], i32 level,
// i32 n_limbs, f64 scale, i64 n_cts} followed by n_cts x [2][n_limbs][N] u64 little-endian residues in
// [0, q) of the COEFFICIENT domain (device NTT-domain ciphertexts go through bm_ct_to_coeff first).
// Level 2 (f1/f3/f4: limbs q0, q1, q2), level 1 (q0, q1), level 0 (q0).
namespace {
struct CtHeader {
    char magic[4];
    uint32_t version;
    uint8_t digest[32];
    int32_t level, n_limbs;
    double scale;
    int64_t n_cts;
};
static_assert(sizeof(CtHeader) == 64, "frame header is 64 bytes");
const int LEVEL_PRIMES[3] = {0, 1, 3}; // host prime index of limb l
bool ct_canonical(const uint64_t *ct, int64_t n_cts, int n_limbs)
{
    for (int64_t c = 0; c < n_cts * 2; c++)
        for (int l = 0; l < n_limbs; l++) {
            const uint64_t q = host_prime(LEVEL_PRIMES[l]).q;
            const uint64_t *v = ct + ((size_t)c * n_limbs + l) * N;
            for (int k = 0; k < N; k++)
                if (v[k] >= q) return false;
        }
    return true;
}
} // namespace

int bm_ct_export(const bm_params *prm, const uint64_t *ct, int64_t n_cts, int32_t level, double scale, uint8_t *buf,
                 size_t *len)
{
    if (!prm || !len || n_cts < 0 || (n_cts > 0 && !ct)) return BM_ERR_INVALID_ARG;
    if (level < 0 || level > 2) return BM_ERR_LEVEL;
    const int nl = level + 1;
    const size_t need = sizeof(CtHeader) + (size_t)n_cts * 2 * nl * N * sizeof(uint64_t);
    if (!buf) {
        *len = need;
        return BM_OK;
    }
    if (*len < need) return BM_ERR_INVALID_ARG;
    if (!ct_canonical(ct, n_cts, nl)) return BM_ERR_INVALID_ARG;
    CtHeader h;
    memcpy(h.magic, "BMCT", 4);
    h.version = 1;
    memcpy(h.digest, prm->digest, 32);
    h.level = level;
    h.n_limbs = nl;
    h.scale = scale;
    h.n_cts = n_cts;
    memcpy(buf, &h, sizeof h); // the library runs on little-endian hosts only (x86-64 / aarch64)
    memcpy(buf + sizeof h, ct, need - sizeof h);
    *len = need;
    return BM_OK;
}

int bm_ct_import(const bm_params *prm, const uint8_t *buf, size_t len, uint64_t *ct, int64_t *n_cts, int32_t *level,
                 double *scale)
{
    if (!prm || !buf || len < sizeof(CtHeader)) return BM_ERR_INVALID_ARG;
    CtHeader h;
    memcpy(&h, buf, sizeof h);
    if (memcmp(h.magic, "BMCT", 4) || h.version != 1) return BM_ERR_INVALID_ARG;
    if (memcmp(h.digest, prm->digest, 32)) return BM_ERR_KEY_MISMATCH;
    if (h.level < 0 || h.level > 2 || h.n_limbs != h.level + 1 || h.n_cts < 0) return BM_ERR_LEVEL;
    const size_t need = sizeof h + (size_t)h.n_cts * 2 * h.n_limbs * N * sizeof(uint64_t);
    if (len != need) return BM_ERR_INVALID_ARG;
    if (n_cts) *n_cts = h.n_cts;
    if (level) *level = h.level;
    if (scale) *scale = h.scale;
    if (!ct) return BM_OK; // size query
    memcpy(ct, buf + sizeof h, need - sizeof h);
    return ct_canonical(ct, h.n_cts, h.n_limbs) ? BM_OK : BM_ERR_INVALID_ARG;
}

// ------------------------------------------------------------------ decryption
// m = c0 + c1 s (+ c2 s^2 when deg == 2) mod q0, centred
static int decrypt_m(const bm_params *prm, const bm_sk *sk, const uint64_t *ct, int64_t n, int deg, int64_t *m)
{
    if (!prm || !sk || (!ct && n) || (!m && n) || n < 0) return BM_ERR_INVALID_ARG;
    if (memcmp(sk->digest, prm->digest, 32)) return BM_ERR_KEY_MISMATCH;
    std::vector<uint64_t> s(N), s2(N);
    for (int k = 0; k < N; k++) s[k] = to_res(sk->s[k], Q0);
    host_ntt_fwd(s.data(), 0);
    for (int k = 0; k < N; k++) s2[k] = mulmod_h(s[k], s[k], Q0);
    return parallel_for(n, [&](int64_t c) {
        std::vector<uint64_t> t(N), t2(N);
        const uint64_t *c0 = ct + (size_t)c * (deg + 1) * N, *c1 = c0 + N, *c2 = c1 + N;
        for (int k = 0; k < N; k++)
            if (c0[k] >= Q0 || c1[k] >= Q0 || (deg == 2 && c2[k] >= Q0)) return (int)BM_ERR_INVALID_ARG;
        memcpy(t.data(), c1, 8 * N);
        host_ntt_fwd(t.data(), 0);
        for (int k = 0; k < N; k++) t[k] = mulmod_h(t[k], s[k], Q0);
        if (deg == 2) {
            memcpy(t2.data(), c2, 8 * N);
            host_ntt_fwd(t2.data(), 0);
            for (int k = 0; k < N; k++) t[k] = (t[k] + mulmod_h(t2[k], s2[k], Q0)) % Q0;
        }
        host_ntt_inv(t.data(), 0);
        for (int k = 0; k < N; k++) {
            uint64_t v = (c0[k] + t[k]) % Q0;
            m[(size_t)c * N + k] = v > Q0 / 2 ? (int64_t)v - (int64_t)Q0 : (int64_t)v;
        }
        return (int)BM_OK;
    });
}

int bm_decrypt_raw(const bm_params *prm, const bm_sk *sk, const uint64_t *ct, int64_t n, int64_t *m)
{
    return decrypt_m(prm, sk, ct, n, 1, m);
}

static int decrypt_scores(const bm_params *prm, const bm_sk *sk, const uint64_t *ct, int64_t n, int deg,
                          double *scores)
{
    if (!prm || !scores) return BM_ERR_INVALID_ARG;
    std::vector<int64_t> m((size_t)std::max<int64_t>(n, 0) * N);
    int rc = decrypt_m(prm, sk, ct, n, deg, m.data());
    if (rc) return rc;
    // score of block k = slot k*s:  z = sum_t m_t cos(pi t e / N) / out_scale, e = 5^(k s) mod 2N
    static std::vector<double> cosT;
    static std::once_flag f;
    std::call_once(f, [] {
        cosT.resize(2 * N);
        for (int i = 0; i < 2 * N; i++) cosT[i] = std::cos(M_PI * i / N);
    });
    const std::vector<int> &e = slot_exp();
    return parallel_for(n, [&](int64_t c) {
        for (int k = 0; k < prm->B; k++) {
            uint64_t ex = (uint64_t)e[(size_t)k * prm->s];
            double acc = 0;
            const int64_t *mm = &m[(size_t)c * N];
            for (int t = 0; t < N; t++) acc += (double)mm[t] * cosT[(ex * t) % (2 * N)];
            scores[(size_t)c * prm->B + k] = acc / prm->out_scale;
        }
        return (int)BM_OK;
    });
}

int bm_decrypt(const bm_params *prm, const bm_sk *sk, const uint64_t *ct, int64_t n, double *scores)
{
    return decrypt_scores(prm, sk, ct, n, 1, scores);
}

int bm_decrypt_deg2(const bm_params *prm, const bm_sk *sk, const uint64_t *ct, int64_t n, double *scores)
{
    return decrypt_scores(prm, sk, ct, n, 2, scores);
}

// f1: packed (compressed) results: every slot is a score -- slot k s + u of packed ciphertext g is set
// g s + u's block k; scale 2^80 / q2 (HE-C^3 one level up, reading R28)
int bm_decrypt_packed(const bm_params *prm, const bm_sk *sk, const uint64_t *ct, int64_t n, double *slots)
{
    if (!prm || !slots) return BM_ERR_INVALID_ARG;
    std::vector<int64_t> m((size_t)std::max<int64_t>(n, 0) * N);
    int rc = bm_decrypt_raw(prm, sk, ct, n, m.data());
    if (rc) return rc;
    std::vector<double> cosT(2 * N);
    for (int i = 0; i < 2 * N; i++) cosT[i] = std::cos(M_PI * i / N);
    const std::vector<int> &e = slot_exp();
    const double scale = std::ldexp(1.0, 80) / (double)Q2;
    for (int64_t c = 0; c < n; c++)
        for (int j = 0; j < SLOTS; j++) {
            const uint64_t ex = (uint64_t)e[j];
            double acc = 0;
            const int64_t *mm = &m[(size_t)c * N];
            for (int t = 0; t < N; t++) acc += (double)mm[t] * cosT[(ex * t) % (2 * N)];
            slots[(size_t)c * SLOTS + j] = acc / scale;
        }
    return BM_OK;
}

int bm_top1(const double *scores, int64_t n, int64_t *idx, double *best)
{
    if (!scores || !idx || n <= 0) return BM_ERR_INVALID_ARG;
    int64_t bi = 0;
    for (int64_t i = 1; i < n; i++)
        if (scores[i] > scores[bi]) bi = i; // strict: lowest index wins ties
    *idx = bi;
    if (best) *best = scores[bi];
    return BM_OK;
}

const char *bm_strerror(int s)
{
    switch (s) {
    case BM_OK: return "ok";
    case BM_ERR_INVALID_ARG: return "invalid argument";
    case BM_ERR_INVALID_LAYOUT: return "invalid layout (d, p must be powers of two, p <= d <= 4096)";
    case BM_ERR_INSECURE_PARAMS: return "parameters exceed the 128-bit security bound";
    case BM_ERR_INVALID_PRIME: return "modulus is not an NTT-friendly prime";
    case BM_ERR_CUDA: return "CUDA error (or no CUDA device)";
    case BM_ERR_OOM: return "out of memory";
    case BM_ERR_ZERO_VECTOR: return "zero-norm feature vector";
    case BM_ERR_MAGNITUDE: return "non-finite or too large input value";
    case BM_ERR_CAPACITY: return "templates exceed set capacity";
    case BM_ERR_LEVEL: return "wrong ciphertext level";
    case BM_ERR_MISSING_ROTATION_KEY: return "missing Galois (rotation) key";
    case BM_ERR_KEY_MISMATCH: return "key / parameter digest mismatch";
    case BM_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown error";
    }
}

} // extern "C"
