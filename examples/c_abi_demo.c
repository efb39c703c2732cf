/* c_abi_demo.c -- a plain C consumer of libblindmatch (include/blindmatch.h), no Python involved.
 *
 *   ./c_abi_demo host   client-side calls only (any machine): params, keygen, key export/import,
 *                       encoding, and decryption of a trivial level-0 ciphertext (m, 0) back to the
 *                       encoded slots; device calls must fail with BM_ERR_CUDA when no GPU is present
 *   ./c_abi_demo gpu    the whole path on cuda:0 (BASELINE.json configs[0] shape: d = 16, p = 1, 256
 *                       templates, 1 genuine query): keygen -> upload -> encrypt DB and query ->
 *                       bm_match -> copy back -> bm_decrypt -> bm_top1, scores vs plaintext dot products
 *
 * Build: gcc -O2 -I include -I /usr/local/cuda/include examples/c_abi_demo.c \
 *          -L paper_2408_06167_b200 -lblindmatch -L /usr/local/cuda/lib64 -lcudart -lm \
 *          -Wl,-rpath,$PWD/paper_2408_06167_b200 -o c_abi_demo
 * Exit status 0 on success.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "blindmatch.h"

#define CHECK(call)                                                                  \
    do {                                                                             \
        int rc_ = (call);                                                            \
        if (rc_ != BM_OK) {                                                          \
            fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #call, bm_strerror(rc_)); \
            return 1;                                                                \
        }                                                                            \
    } while (0)

static uint64_t lcg = 88172645463325252ull;
static double gauss(void) /* Box-Muller on a 64-bit LCG (demo data only) */
{
    lcg = lcg * 6364136223846793005ull + 1442695040888963407ull;
    double u1 = ((lcg >> 11) + 1.0) / 9007199254740993.0;
    lcg = lcg * 6364136223846793005ull + 1442695040888963407ull;
    double u2 = (lcg >> 11) / 9007199254740992.0;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
static void unit_rows(double *x, int n, int d)
{
    for (int r = 0; r < n; r++) {
        double ss = 0;
        for (int i = 0; i < d; i++) x[r * d + i] = gauss(), ss += x[r * d + i] * x[r * d + i];
        for (int i = 0; i < d; i++) x[r * d + i] /= sqrt(ss);
    }
}

static int host_mode(void)
{
    bm_params prm;
    CHECK(bm_rng_mode(BM_RNG_SEEDED));
    CHECK(bm_params_init(&prm, 16, 1));
    if (bm_params_init(&prm, 24, 1) != BM_ERR_INVALID_LAYOUT) return 1;
    CHECK(bm_params_init(&prm, 16, 1));
    bm_sk *sk;
    bm_pk *pk;
    bm_evk *evk;
    CHECK(bm_keygen(&prm, 7, &sk, &pk, &evk));
    int8_t *s = malloc(BM_N);
    CHECK(bm_sk_export(sk, s));
    bm_sk *sk2;
    CHECK(bm_sk_import(&prm, s, &sk2));
    /* encode a query, make the trivial level-0 ciphertext (pt mod q0, 0), decrypt it */
    double q[16];
    unit_rows(q, 1, 16);
    int64_t *pt = malloc(sizeof(int64_t) * BM_N);
    CHECK(bm_encode_query(&prm, q, 1, pt));
    uint64_t *ct = calloc(2 * BM_N, sizeof(uint64_t));
    for (int k = 0; k < BM_N; k++) ct[k] = pt[k] >= 0 ? (uint64_t)pt[k] % prm.q[0] : prm.q[0] - (uint64_t)(-pt[k]) % prm.q[0];
    double *scores = malloc(sizeof(double) * prm.B);
    CHECK(bm_decrypt(&prm, sk2, ct, 1, scores));
    /* slot k s holds q[(k s) mod s] = q[0] scaled by 2^40 / out_scale (the trivial ct sits at scale 2^40) */
    double err = 0;
    for (int k = 0; k < prm.B; k++) err = fmax(err, fabs(scores[k] * prm.out_scale / prm.scale - q[0]));
    printf("host: B = %d scores, max |slot - q[0]| = %.3g\n", prm.B, err);
    if (err > 1e-9) return 1;
    int64_t idx;
    double best;
    CHECK(bm_top1(scores, prm.B, &idx, &best));
    /* without a GPU every device call reports BM_ERR_CUDA (there is no CPU fallback) */
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0) {
        bm_evk_dev *ed;
        int rc = bm_evk_to_device(&prm, evk, &ed);
        printf("host: no GPU, bm_evk_to_device -> %s\n", bm_strerror(rc));
        if (rc != BM_ERR_CUDA) return 1;
    }
    bm_sk_free(sk), bm_sk_free(sk2), bm_pk_free(pk), bm_evk_free(evk);
    free(s), free(pt), free(ct), free(scores);
    printf("host: ok (%s)\n", bm_build_info());
    return 0;
}

static int gpu_mode(void)
{
    const int d = 16, p = 1, n = 256;
    bm_params prm;
    CHECK(bm_rng_mode(BM_RNG_OS)); /* the product default: OS-entropy keys and encryption randomness */
    CHECK(bm_params_init(&prm, d, p));
    bm_sk *sk;
    bm_pk *pk;
    bm_evk *evk;
    CHECK(bm_keygen(&prm, 1, &sk, &pk, &evk));
    bm_pk_dev *pkd;
    bm_evk_dev *evkd;
    CHECK(bm_pk_to_device(&prm, pk, &pkd));
    CHECK(bm_evk_to_device(&prm, evk, &evkd));
    double *T = malloc(sizeof(double) * n * d), Q[16];
    unit_rows(T, n, d);
    for (int i = 0; i < d; i++) Q[i] = T[17 * d + i] + 0.05 * gauss(); /* a genuine query of template 17 */
    const int64_t n_sets = (n + prm.B - 1) / prm.B;
    const size_t ct1 = (size_t)2 * 2 * BM_N * sizeof(uint64_t);
    uint64_t *d_db, *d_q, *d_out;
    void *d_ws;
    const size_t ws = bm_match_ws_bytes(&prm, n_sets, 1, BM_ORDER_HOISTED);
    if (cudaMalloc((void **)&d_db, n_sets * p * ct1) || cudaMalloc((void **)&d_q, p * ct1) ||
        cudaMalloc((void **)&d_out, n_sets * 2 * BM_N * sizeof(uint64_t)) || cudaMalloc(&d_ws, ws))
        return 1;
    CHECK(bm_encrypt_db(&prm, pkd, T, n, 0, n_sets, 2, d_db, 0));
    CHECK(bm_encrypt_query(&prm, pkd, Q, 1, 0, 3, d_q, 0));
    CHECK(bm_match(&prm, evkd, d_db, n_sets, d_q, 1, d_out, d_ws, ws, BM_ORDER_HOISTED, 0));
    CHECK(bm_sync(0));
    uint64_t *h_out = malloc(n_sets * 2 * BM_N * sizeof(uint64_t));
    cudaMemcpy(h_out, d_out, n_sets * 2 * BM_N * sizeof(uint64_t), cudaMemcpyDeviceToHost);
    double *scores = malloc(sizeof(double) * n_sets * prm.B);
    CHECK(bm_decrypt(&prm, sk, h_out, n_sets, scores));
    double qn = 0, err = 0;
    for (int i = 0; i < d; i++) qn += Q[i] * Q[i];
    for (int u = 0; u < n; u++) {
        double dot = 0;
        for (int i = 0; i < d; i++) dot += T[u * d + i] * Q[i];
        err = fmax(err, fabs(scores[u] - dot / sqrt(qn)));
    }
    int64_t idx;
    double best;
    CHECK(bm_top1(scores, n, &idx, &best));
    printf("gpu: %d templates, max |score - cos| = %.3g, top-1 = %lld (%.4f), launches %lld\n", n, err, (long long)idx,
           best, (long long)bm_launch_count());
    if (err > 1e-4 || idx != 17) return 1;
    cudaFree(d_db), cudaFree(d_q), cudaFree(d_out), cudaFree(d_ws);
    bm_pk_dev_free(pkd), bm_evk_dev_free(evkd), bm_sk_free(sk), bm_pk_free(pk), bm_evk_free(evk);
    free(T), free(h_out), free(scores);
    printf("gpu: ok\n");
    return 0;
}

int main(int argc, char **argv)
{
    if (argc > 1 && !strcmp(argv[1], "gpu")) return gpu_mode();
    return host_mode();
}
