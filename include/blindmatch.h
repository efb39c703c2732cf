/*
 * blindmatch.h -- C ABI of the B200-native Blind-Match encrypted 1:N cosine scan.
 *
 * The method is HE-C^3 (Algorithm 2) in RNS-CKKS with
 *   N = 8192 (S = N/2 = 4096 real slots, reading R1),
 *   q0 = 2^58-835583, q1 = 2^40-147455, special prime P = 2^60-16383
 *   (largest primes below 2^k with q = 1 mod 16384; BASELINE.json configs[0]),
 *   scale 2^40, ternary secret, discrete Gaussian errors sigma = 3.2.
 * The client packs/encrypts, the server scans,
 * the client decrypts and takes the argmax.
 *
 * Conventions (all functions):
 *  - return 0 (BM_OK) or a negative bm_status; bm_strerror() names it.
 *  - "host" pointers are ordinary CPU memory, "device" pointers are CUDA device memory
 *    of the current device (e.g. torch tensors' data_ptr()); all are caller-owned unless
 *    a function returns a library handle (free it with the matching *_free).
 *  - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).  Device
 *    functions are asynchronous and stream-ordered; kernel faults surface at bm_sync().
 *  - residues are uint64 in [0, q).  Coefficient-domain ("canonical") layouts are
 *    limb-major: a level-1 ciphertext is [2 comps][2 limbs q0,q1][N], a level-0 one
 *    [2][1][N].  NTT-domain ("device") layouts have the same shape, with the library's
 *    internal evaluation order; convert with bm_ct_to_coeff / bm_ct_from_coeff.
 *  - there is no CPU fallback: device functions fail with BM_ERR_CUDA without a GPU.
 */
#ifndef BLINDMATCH_H
#define BLINDMATCH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BM_LOGN 13
#define BM_N 8192
#define BM_SLOTS 4096

typedef enum {
    BM_OK = 0,
    BM_ERR_INVALID_ARG = -1,          /* null pointer, negative count, bad enum              */
    BM_ERR_INVALID_LAYOUT = -2,       /* d, p not powers of two, p > d, d > S  */
    BM_ERR_INSECURE_PARAMS = -3,      /* log2(q0 q1 P) above the 128-bit bound */
    BM_ERR_INVALID_PRIME = -4,        /* a modulus is not an NTT-friendly prime              */
    BM_ERR_CUDA = -5,                 /* CUDA runtime / kernel error, or no device           */
    BM_ERR_OOM = -6,                  /* device allocation failed                             */
    BM_ERR_ZERO_VECTOR = -7,          /* a template/query has zero norm        */
    BM_ERR_MAGNITUDE = -8,            /* non-finite input value                */
    BM_ERR_CAPACITY = -9,             /* templates do not fit in the given sets              */
    BM_ERR_LEVEL = -10,               /* wrong ciphertext level for the op      */
    BM_ERR_MISSING_ROTATION_KEY = -11,/* evk lacks a Galois key the layout needs */
    BM_ERR_KEY_MISMATCH = -12,        /* key / params digest mismatch          */
    BM_ERR_WORKSPACE = -13            /* workspace smaller than bm_match_ws_bytes()           */
} bm_status;

typedef enum {
    BM_ORDER_HOISTED = 0,     /* sum_i tensor_i, then one relin + one rescale (reading R8) */
    BM_ORDER_PAPER = 1,       /* per part Res(Mul(C_u,i, C_s,i)), then Add at level 0 */
    BM_ORDER_HOISTED_ROT = 2, /* f2, NOT the paper's ladder: BM_ORDER_HOISTED's C,
                                 then sum_{r<s} Rot(C, r) with ONE hoisted key switch (Halevi-Shoup):
                                 same decrypted scores, different residues; needs bm_evk_add_hoisted */
    BM_ORDER_DEG2 = 3,        /* f2, relin-free, p = d only (s = 1, no ladder):
                                 sum_i tensor_i rescaled by q1 component by component; the result is
                                 the DEGREE-2 ciphertext (d0, d1, d2) [nq][n_sets][3][N] (coefficients,
                                 scale out_scale), decrypted with (1, s, s^2) by bm_decrypt_deg2;
                                 evk unused (may be NULL); BM_ERR_INVALID_LAYOUT when p != d */
    BM_ORDER_BSGS = 4         /* f2, NOT the paper's ladder: BM_ORDER_HOISTED's C,
                                 then baby-step giant-step: sum_{j<g} Rot(sum_{i<b} Rot(C, i), j b),
                                 b = 2^ceil(log2(s)/2), g = s/b, each sum one hoisted key switch; same
                                 decrypted scores, its own residues; needs bm_evk_add_hoisted */
} bm_order;

/* Scheme parameters and the packing layout:
 * d = feature size (paper's m), p = parts (paper's N_in), s = d/p, B = S/s templates per set,
 * log_s = log2 s ladder steps, Galois keys for rotations 2^i, i < log_s. */
typedef struct bm_params {
    int32_t logN, N, slots;
    int32_t d, p, s, B, log_s;
    uint64_t q[3];          /* q0, q1, P                               */
    double scale;           /* 2^40                                    */
    double out_scale;       /* 2^80 / q1: scale of bm_match outputs    */
    uint8_t digest[32];     /* digest of (N, q0, q1, P, scale); not of the layout (d, p) */
    uint64_t q2;            /* f3 only: the extra 40-bit prime of level 2 (2^40 - 45 2^14 + 1) */
} bm_params;

typedef struct bm_sk bm_sk;           /* host: ternary secret (client only)              */
typedef struct bm_pk bm_pk;           /* host: public key (b, a) over {q0,q1}             */
typedef struct bm_evk bm_evk;         /* host: relinearization key + Galois keys          */
typedef struct bm_pk_dev bm_pk_dev;   /* device copy of pk (NTT domain)                   */
typedef struct bm_evk_dev bm_evk_dev; /* device copy of evk (NTT domain)                  */

/* Randomness (a seeded generator as a test mode, a cryptographic one otherwise).
 * Every draw comes from ChaCha20 (RFC 8439) keyed by the call's 64-bit seed, the draw's purpose and a
 * 160-bit key extension; objects / components / limbs are nonces (reading R14).
 *   BM_RNG_OS (the default): the keygen family (bm_keygen, bm_evk_add_hoisted, bm_xk_keygen,
 *     bm_ck_keygen) uses a 160-bit process key drawn once from getrandom() -- 224 bits of key entropy,
 *     and the same seed gives the same secret within the process, so the family stays consistent;
 *     keys outlive the process through bm_*_export / import -- and EVERY encryption call (bm_encrypt,
 *     bm_encrypt_db, bm_encrypt_query, bm_encrypt_l2) draws a fresh 160-bit extension, so two batches
 *     encrypted with the same seed and object numbers share no randomness.
 *   BM_RNG_SEEDED: all extensions zero -- deterministic in the seed (tests, benchmarks, the oracle's
 *     streams).  Never reuse a seed across encryptions in this mode.
 * bm_rng_mode returns BM_ERR_INVALID_ARG for another value.  Process-wide. */
#define BM_RNG_SEEDED 0
#define BM_RNG_OS 1
int bm_rng_mode(int32_t mode);
int32_t bm_get_rng_mode(void);

/* Fill *out for feature size d and part count p (both powers of two, 1 <= p <= d <= 4096).
 * Errors: BM_ERR_INVALID_ARG (out null), BM_ERR_INVALID_LAYOUT, BM_ERR_INVALID_PRIME,
 * BM_ERR_INSECURE_PARAMS. */
int bm_params_init(bm_params *out, int32_t d, int32_t p);

/* Key generation, host, deterministic in `seed`.
 * sk: s ternary.  pk = (-a s + e, a) over {q0,q1}.  rlk_j, j in {0,1}, over {q0,q1,P}:
 * (-a s + e + [k=j](P mod q_k) s^2, a).  gk_i (rotation 2^i, i < log_s) over {q0,P}:
 * (-a s + e + (P mod q0) sigma_{5^(2^i)}(s) [q0 limb only], a).  Any of sk/pk/evk may be
 * NULL to skip returning it.  Randomness: ChaCha20 streams (reading R14). */
int bm_keygen(const bm_params *prm, uint64_t seed, bm_sk **sk, bm_pk **pk, bm_evk **evk);
void bm_sk_free(bm_sk *);
void bm_pk_free(bm_pk *);
void bm_evk_free(bm_evk *);
/* f2: add to evk the Galois keys of every rotation r = 1..s-1 (same secret: pass keygen's seed;
 * PRNG object 64 + r), needed by BM_ORDER_HOISTED_ROT; upload with bm_evk_to_device afterwards.
 * Errors: BM_ERR_INVALID_ARG, BM_ERR_KEY_MISMATCH (evk made for other params). */
int bm_evk_add_hoisted(const bm_params *prm, uint64_t seed, bm_evk *evk);

/* Canonical (coefficient-domain) exports.  sk: int8[N].  pk: [2][2][N].
 * rlk: [2 digits][2 comps][3 limbs q0,q1,P][N].  gk: [log_s][2][2 limbs q0,P][N]
 * (gk may be NULL; *n_rot receives log_s when non-NULL). */
int bm_sk_export(const bm_sk *, int8_t *out);
int bm_pk_export(const bm_pk *, uint64_t *out);
int bm_evk_export(const bm_evk *, uint64_t *rlk, uint64_t *gk, int32_t *n_rot);
/* Build host keys from canonical arrays (e.g. keys received over the network). */
int bm_sk_import(const bm_params *, const int8_t *in, bm_sk **out);
int bm_pk_import(const bm_params *, const uint64_t *in, bm_pk **out);
int bm_evk_import(const bm_params *, const uint64_t *rlk, const uint64_t *gk, int32_t n_rot, bm_evk **out);

/* Upload keys to the current device (NTT domain + Shoup companions).  Synchronous.
 * Errors: BM_ERR_CUDA, BM_ERR_OOM, BM_ERR_KEY_MISMATCH (evk built for other params). */
int bm_pk_to_device(const bm_params *, const bm_pk *, bm_pk_dev **out);
int bm_evk_to_device(const bm_params *, const bm_evk *, bm_evk_dev **out);
void bm_pk_dev_free(bm_pk_dev *);
void bm_evk_dev_free(bm_evk_dev *);

/* Client-side packing + CKKS encoding (host, FP64).
 * bm_encode_db: templates tmpl[n][d] (host, row-major; each normalised to unit L2 norm)
 *   -> pt[n_sets][p][N] int64, for sets first_set .. first_set+n_sets-1 (global set t holds
 *   templates tB .. tB+B-1; template u = tB+k occupies slots k*s .. k*s+s-1 of part i with
 *   v[i*s .. i*s+s-1]; empty blocks are zero).  n counts ALL templates (global indexing).
 * bm_encode_query: q[nq][d] -> pt[nq][p][N], part i holds w_i[x] = q[i*s + (x mod s)].
 * Encoding: m_k = (2/N) sum_j z_j cos(pi k 5^j / N), pt_k = round(2^40 m_k) (reading R15).
 * Errors: BM_ERR_ZERO_VECTOR, BM_ERR_MAGNITUDE, BM_ERR_INVALID_ARG. */
int bm_encode_db(const bm_params *, const double *tmpl, int64_t n, int64_t first_set, int64_t n_sets, int64_t *pt);
int bm_encode_query(const bm_params *, const double *q, int64_t nq, int64_t *pt);

/* Public-key encryption on the device: for c < n_cts, object o = first_obj + c,
 * ct_o = (u b + e0 + pt_c, u a + e1) over {q0,q1} with u ternary, e0, e1 Gaussian drawn
 * from ChaCha20 streams (seed, purpose, o).  d_pt: device int64 [n_cts][N];
 * d_out: device uint64 [n_cts][2][2][N], NTT domain.  DB objects are numbered
 * set*p + part, query objects query*p + part, so shards encrypt bit-identically. */
int bm_encrypt(const bm_params *, const bm_pk_dev *, const int64_t *d_pt, int64_t n_cts, uint64_t first_obj,
               uint64_t seed, uint64_t *d_out, void *stream);
/* Convenience: bm_encode_db / bm_encode_query on the host, upload, bm_encrypt.
 * Blocks until the upload of the plaintexts is done. */
int bm_encrypt_db(const bm_params *, const bm_pk_dev *, const double *tmpl, int64_t n, int64_t first_set,
                  int64_t n_sets, uint64_t seed, uint64_t *d_out, void *stream);
int bm_encrypt_query(const bm_params *, const bm_pk_dev *, const double *q, int64_t nq, int64_t first_query,
                     uint64_t seed, uint64_t *d_out, void *stream);

/* Domain conversion of n_cts ciphertexts with n_limbs limbs (1, 2 or 3; limbs q0[,q1[,q2]]),
 * layout [n_cts][2][n_limbs][N], device in/out (may alias). */
int bm_ct_to_coeff(const bm_params *, const uint64_t *d_in, int64_t n_cts, int32_t n_limbs, uint64_t *d_out,
                   void *stream);
int bm_ct_from_coeff(const bm_params *, const uint64_t *d_in, int64_t n_cts, int32_t n_limbs, uint64_t *d_out,
                     void *stream);

/* Ciphertext (de)serialisation: a framed canonical byte form for
 * storage and the network.  64-byte header {"BMCT", version 1, the params digest, level, limbs, scale,
 * n_cts} + n_cts x [2][level+1 limbs][N] little-endian u64 residues in [0, q), COEFFICIENT domain
 * (convert device NTT-domain ciphertexts with bm_ct_to_coeff first).  Levels 0, 1 and 2 (the f1/f3/f4
 * chain, limbs q0, q1, q2).  bm_ct_export with buf = NULL returns the size in *len.  bm_ct_import with
 * ct = NULL returns n_cts / level / scale only.  Host memory.  Errors: BM_ERR_INVALID_ARG (bad frame,
 * short buffer, non-canonical residue), BM_ERR_KEY_MISMATCH (frame made for other params),
 * BM_ERR_LEVEL. */
int bm_ct_export(const bm_params *, const uint64_t *ct, int64_t n_cts, int32_t level, double scale, uint8_t *buf,
                 size_t *len);
int bm_ct_import(const bm_params *, const uint8_t *buf, size_t len, uint64_t *ct, int64_t *n_cts, int32_t *level,
                 double *scale);

/* THE HOT PATH: HE-C^3 scan of nq queries against n_sets sets.
 * d_db:  device [n_sets][p][2][2][N] level-1 NTT-domain DB (bm_encrypt output);
 * d_q:   device [nq][p][2][2][N] level-1 NTT-domain query parts (client-expanded, reading R10);
 * d_out: device [nq][n_sets][2][N] level-0 results, COEFFICIENT domain (canonical), scale
 *        prm->out_scale; slot k*s of (query j, set t) decrypts to cos(q_j, v_{tB+k}).
 * d_ws:  device workspace of at least bm_match_ws_bytes(prm, n_sets, nq, order) bytes.
 * Per (query, set): tensor + sum over parts (a4), relinearize (a5), rescale (a6), log2(s)
 * rotate-and-add steps (a7), all in sm_100a kernels on `stream`; allocates nothing.
 * BM_ORDER_DEG2 instead writes d_out [nq][n_sets][3][N] (the degree-2 result; see bm_order).
 * Errors: BM_ERR_INVALID_ARG, BM_ERR_MISSING_ROTATION_KEY, BM_ERR_KEY_MISMATCH,
 * BM_ERR_WORKSPACE, BM_ERR_CUDA (launch errors; faults at bm_sync). nq = 0 or n_sets = 0
 * is a no-op.  Kernel choice depends only on the launch size, never on the results: chunks of
 * fewer than 8 queries use the swapped tensor tiles and launches of at most n_SM / 2 (n_SM / 3)
 * pairs run the ladder on 2-CTA (3-CTA) clusters (latency mode, e.g. one query against a small DB);
 * the residues are identical either way. */
size_t bm_match_ws_bytes(const bm_params *, int64_t n_sets, int32_t nq, int32_t order);
int bm_match(const bm_params *, const bm_evk_dev *, const uint64_t *d_db, int64_t n_sets, const uint64_t *d_q,
             int32_t nq, uint64_t *d_out, void *d_ws, size_t ws_bytes, int32_t order, void *stream);

/* a8 fused into the scan ("the main server combines the returned
 * outputs"): the same scan, but every result is stored by the output kernels themselves straight into
 * its query's ROW on the query's root GPU -- over NVLink when the row lives on a peer (a pointer
 * obtained with bm_ipc_open), so the gather overlaps the scan pair by pair and needs no collective.
 * d_rows: DEVICE array of nq pointers; row j holds n_row_sets level-0 results [n_row_sets][2][N]
 *         (coefficient domain, as d_out of bm_match), and (query j, local set t) is written at
 *         d_rows[j] + ((set_offset + t) * 2 + c) * N, i.e. this rank's sets at their GLOBAL set
 *         numbers.  Rows are caller-owned; they must not overlap.
 * The caller orders the root's reads after every writer's scan (e.g. an NCCL all-reduce queued
 * on each writer's stream after this call).  Errors as bm_match; BM_ERR_INVALID_ARG if d_rows is
 * NULL or set_offset < 0. */
int bm_match_rows(const bm_params *, const bm_evk_dev *, const uint64_t *d_db, int64_t n_sets, const uint64_t *d_q,
                  int32_t nq, uint64_t *const *d_rows, int64_t set_offset, void *d_ws, size_t ws_bytes, int32_t order,
                  void *stream);

/* CUDA IPC for bm_match_rows across processes (one process per GPU): bm_ipc_handle returns the
 * 64-byte handle of the device allocation containing d_ptr and d_ptr's byte offset inside it;
 * another process opens it with bm_ipc_open (peer access enabled lazily; *d_base = the allocation's
 * base in this process, add the offset) and releases it with bm_ipc_close.  Errors: BM_ERR_CUDA,
 * BM_ERR_INVALID_ARG. */
int bm_ipc_handle(const void *d_ptr, uint8_t handle[64], uint64_t *offset);
int bm_ipc_open(const uint8_t handle[64], void **d_base);
int bm_ipc_close(void *d_base);

/* The same scan end to end from HOST buffers: h_q (host [nq][p][2][2][N], NTT domain) is
 * copied in and h_out (host [nq][n_sets][2][N]) copied out inside the call.  The queries are
 * processed in groups of max(576, min(16384, 4 n_sets)) (query, set) pairs (or BM_OPT_HOST_GROUPS groups): group g's
 * upload, scan and download overlap the neighbouring groups (four device slots, two internal
 * copy streams, the scans alternating between `stream` and an internal stream, all starting
 * after the work already queued on `stream`; the internal streams are created once per device and
 * the calls on one device are serialised by the library).
 * Pinned host memory is required for the overlap.  d_ws must hold bm_match_host_ws_bytes(...)
 * bytes.  Synchronous (returns after h_out is written). */
size_t bm_match_host_ws_bytes(const bm_params *, int64_t n_sets, int32_t nq, int32_t order);
int bm_match_host(const bm_params *, const bm_evk_dev *, const uint64_t *d_db, int64_t n_sets, const uint64_t *h_q,
                  int32_t nq, uint64_t *h_out, void *d_ws, size_t ws_bytes, int32_t order, void *stream);

/* Streaming variant for result sets larger than host memory (BASELINE.json configs[3]: 1,048,576
 * templates x 256 queries = 128 GiB of level-0 results per batch): query j's results are written to
 * host row (j mod ring_rows) of h_ring [ring_rows][n_sets][2][N], overwriting earlier queries' rows
 * (the caller consumes rows between calls, or -- a benchmark -- not at all).  ring_rows >= 1;
 * ring_rows >= nq is bm_match_host.  Same workspace, same scan, same errors. */
int bm_match_host_ring(const bm_params *, const bm_evk_dev *, const uint64_t *d_db, int64_t n_sets,
                       const uint64_t *h_q, int32_t nq, uint64_t *h_ring, int32_t ring_rows, void *d_ws,
                       size_t ws_bytes, int32_t order, void *stream);

/* The DB in the tensor-core layout (server-side enrollment step for K1 on the tcgen05 tensor cores,
 * DESIGN.md sec. 3 "K1 on the tensor cores"; the tensor of PAPER.md:327-328 as a u8 x u8 -> s32 GEMM per
 * coefficient).  bm_db_tc_register packs d_db [n_sets][p][2][2][N] (device storage order) into the
 * caller-owned device buffer d_packed (>= bm_db_tc_bytes bytes; 128-set tiles, per limb and coefficient one
 * contiguous 128 x 16 p-byte block) on `stream` and records the pair: from then on bm_match / bm_match_rows /
 * bm_match_host* calls with this d_db (same n_sets and p) compute the tensor on the tensor cores (results
 * identical).  The caller keeps d_db unchanged and d_packed allocated while registered (register again
 * after changing d_db; registering a d_db again replaces its entry); bm_db_tc_unregister forgets it
 * (BM_ERR_INVALID_ARG if it was not registered).  p must be 4 or 8 (BM_ERR_INVALID_ARG otherwise;
 * bm_db_tc_bytes returns 0); BM_ERR_WORKSPACE if bytes is too small. */
size_t bm_db_tc_bytes(const bm_params *, int64_t n_sets);
int bm_db_tc_register(const bm_params *, const uint64_t *d_db, int64_t n_sets, void *d_packed, size_t bytes,
                      void *stream);
int bm_db_tc_unregister(const uint64_t *d_db);

/* Library options (process-wide; the defaults are the product -- tests and tuning runs change them).
 * Changing BM_OPT_CHUNK_PAIRS / BM_OPT_EXPAND_CHUNK / BM_OPT_CMP_CHUNK changes the workspace size the
 * *_ws_bytes functions return: size the workspace after setting them.  Results never depend on them.
 * bm_set_option returns BM_ERR_INVALID_ARG for an unknown key or a value out of range. */
typedef enum {
    BM_OPT_CHUNK_PAIRS = 0,  /* (query, set) pairs per bm_match chunk, >= 1 (default 16384)          */
    BM_OPT_EXPAND_CHUNK = 1, /* (query, part) outputs per bm_expand / bm_enroll launch (2048)       */
    BM_OPT_HOST_GROUPS = 2,  /* bm_match_host query groups, 0 = automatic (see bm_match_host)      */
    BM_OPT_LADDER_C2 = 3,    /* 0/1: latency-mode ladder on 2-CTA clusters (1)                      */
    BM_OPT_LADDER_C3 = 4,    /* 0/1: latency-mode ladder on 3-CTA clusters (1)                      */
    BM_OPT_LADDER_TAIL = 5,  /* 0/1: a large launch's partial last wave on the cluster ladders (1)  */
    BM_OPT_CMP_CHUNK = 6,    /* pairs per bm_match_cmp chunk (4096)                                 */
    BM_OPT_TENSOR_MMA = 7,   /* 0/1: K1 on the tensor cores for registered DBs (bm_db_tc_*) (1)      */
    BM_OPT_COUNT_ = 8
} bm_option;
int bm_set_option(int32_t key, int64_t value);
int64_t bm_get_option(int32_t key);

/* Number of kernels the library has launched in this process (every launch site counts itself;
 * the bench's gpu_launches claim).  bm_launch_count_reset sets it to 0. */
int64_t bm_launch_count(void);
void bm_launch_count_reset(void);

/* Per-kernel-class device time of the last bm_match on this thread when profiling is
 * enabled (bm_set_profiling(1)); classes: 0 tensor, 1 digits + ModUp NTTs, 2 key switch +
 * ModDown + rescale, 3 unused, 4 rotate-and-add ladder (fused), 5 f2 hoisted rotation sum, 6 output
 * INTT (s = 1).  ms[7] and
 * launches[7] accumulate until bm_profile_reset(). */
void bm_set_profiling(int32_t on);
void bm_profile_reset(void);
int bm_profile_read(double *ms, int64_t *launches, int64_t *units);

/* Client side on the DEVICE (a9 at the scale of a 1:N batch).
 * bm_sk_to_device uploads the secret (NTT domain mod q0; synchronous; a client-side handle -- the
 * server never needs it).  bm_decrypt_dev decrypts n level-0 results d_ct [n][2][N] (device,
 * COEFFICIENT domain: bm_match's d_out) and decodes the B score slots k*s into d_scores [n][B]
 * (device float64): m = c0 + c1 s mod q0 (centred), slot j = Re m(zeta^(5^j)), zeta = exp(i pi / N),
 * evaluated for all odd powers by one N-point FP64 FFT per ciphertext, divided by prm->out_scale.
 * Same scores as bm_decrypt (the direct cosine sum) to ~1e-12.  Asynchronous on `stream`.
 * Errors: BM_ERR_INVALID_ARG, BM_ERR_KEY_MISMATCH, BM_ERR_CUDA, BM_ERR_OOM. */
typedef struct bm_sk_dev bm_sk_dev;
int bm_sk_to_device(const bm_params *, const bm_sk *, bm_sk_dev **out);
void bm_sk_dev_free(bm_sk_dev *);
int bm_decrypt_dev(const bm_params *, const bm_sk_dev *, const uint64_t *d_ct, int64_t n, double *d_scores,
                   void *stream);

/* Client side (host): decrypt level-0 results h_ct [n][2][1][N] (canonical) and decode the
 * B scores at slots k*s into scores[n][B].  bm_decrypt_raw returns the
 * centred message coefficients m = c0 + c1 s mod q0 as int64 [n][N]. */
int bm_decrypt(const bm_params *, const bm_sk *, const uint64_t *h_ct, int64_t n, double *scores);
int bm_decrypt_raw(const bm_params *, const bm_sk *, const uint64_t *h_ct, int64_t n, int64_t *m);
/* f2 degree-2 results (BM_ORDER_DEG2): h_ct [n][3][N] coefficient-domain (d0, d1, d2) over q0;
 * m = d0 + d1 s + d2 s^2 mod q0 (the decryption of a degree-2 ciphertext, PAPER.md:155-157 extended
 * to the tensor's third component), then scores[n][B] as bm_decrypt (s = 1: every slot).  Same errors. */
int bm_decrypt_deg2(const bm_params *, const bm_sk *, const uint64_t *h_ct, int64_t n, double *scores);
/* argmax with the lowest index winning ties. */
int bm_top1(const double *scores, int64_t n, int64_t *idx, double *best);

/* ---------------------------------------------------------------------------------------------
 * f3: SERVER-SIDE QUERY EXPANSION, Algorithm 1 "Input Ciphertext Expansion"
 * with SPEC.md:297's post-condition (readings R24-R26).  It needs one
 * more level than BASELINE.json's chain, so it runs on the chain extended by q2 = prm->q2:
 * level 2 = {q0, q1, q2}.  The client encrypts ONE ciphertext per query: the unit query tiled
 * S/d times at level 2, scale 2^40.  The server computes, for every part i < p,
 *   C_i = Res_q2(Mul(P)(C, X_i)),  X_i[x] = [(x mod d) in [i s, (i+1) s)] encoded at scale q2,
 *   then for t < log2 p:  C_i = C_i + Rot(C_i, s 2^t)   (level-1 rotations, 2-digit key switch),
 * so C_i is a level-1 ciphertext at scale exactly 2^40 with w_i[x] = q[i s + (x mod s)]: the
 * d_q input of bm_match.  The rest of the scan is unchanged.
 * ------------------------------------------------------------------------------------------- */
typedef struct bm_xk bm_xk;           /* host: pk limb q2 + level-1 Galois keys of strides s 2^t */
typedef struct bm_xk_dev bm_xk_dev;   /* device: level-2 pk, Galois keys, masks (NTT domain)      */

/* Expansion / enrollment keys for keygen(seed)'s secret (pass the same seed).  pk limb q2 =
 * (-a s + e, a) with pk's error e; gk1[t][j] (rotation r = s 2^t, t < log2 B, digit j) over
 * {q0,q1,P}: (-a s + e + [l = j](P mod q_l) sigma_{5^r}(s) [limb q_l], a).  The expansion uses
 * t < log2 p, the enrollment (f4) every t < log2 B.  Errors: BM_ERR_INVALID_ARG, BM_ERR_OOM. */
int bm_xk_keygen(const bm_params *, uint64_t seed, bm_xk **out);
void bm_xk_free(bm_xk *);
/* pk_q2 [2][N]; gk1 [n_rot][2 digits][2 comps][3 limbs q0,q1,P][N] (canonical).  Import accepts
 * log2 p <= n_rot <= log2 B (BM_ERR_MISSING_ROTATION_KEY otherwise). */
int bm_xk_export(const bm_xk *, uint64_t *pk_q2, uint64_t *gk1, int32_t *n_rot);
int bm_xk_import(const bm_params *, const uint64_t *pk_q2, const uint64_t *gk1, int32_t n_rot, bm_xk **out);
/* Upload (synchronous): the level-2 public key (pk's limbs + xk's q2 limb), the Galois keys, the
 * p expansion masks h_masks [p][N] and (optional, f4) the p enrollment masks h_emasks [p][N]
 * (int64 plaintexts, e.g. from bm_encode_masks), all to the NTT domain.
 * Errors: BM_ERR_KEY_MISMATCH, BM_ERR_CUDA, BM_ERR_OOM. */
int bm_xk_to_device(const bm_params *, const bm_pk *, const bm_xk *, const int64_t *h_masks, const int64_t *h_emasks,
                    bm_xk_dev **out);
void bm_xk_dev_free(bm_xk_dev *);
/* Client encoding (host): q[nq][d] -> pt[nq][N], the unit query tiled S/d times at scale 2^40;
 * bm_encode_enroll: v[n][d] -> pt[n][N], the unit template in slots [0, d), zeros elsewhere (f4);
 * masks: pt[p][N] at scale q2, kind 0 the expansion masks X_i[x] = [(x mod d) in [i s, (i+1) s)],
 * kind 1 the enrollment masks E_i[x] = [x in [i s, (i+1) s)].
 * Errors: BM_ERR_ZERO_VECTOR, BM_ERR_MAGNITUDE, BM_ERR_INVALID_ARG. */
int bm_encode_query_tiled(const bm_params *, const double *q, int64_t nq, int64_t *pt);
int bm_encode_enroll(const bm_params *, const double *v, int64_t n, int64_t *pt);
int bm_encode_masks(const bm_params *, int32_t kind, int64_t *pt);
/* Level-2 public-key encryption (device): ct_o = (u b + e0 + pt, u a + e1) over {q0,q1,q2}, the
 * streams of bm_encrypt (so limbs q0, q1 equal bm_encrypt's).  d_pt [n][N] int64 device;
 * d_out [n][2][3][N] NTT domain. */
int bm_encrypt_l2(const bm_params *, const bm_xk_dev *, const int64_t *d_pt, int64_t n_cts, uint64_t first_obj,
                  uint64_t seed, uint64_t *d_out, void *stream);
/* Algorithm 1 on the device: d_in [nq][2][3][N] level 2 (NTT) -> d_out [nq][p][2][2][N] level 1
 * (NTT), the layout bm_match takes as d_q.  d_ws of at least bm_expand_ws_bytes(prm, nq) bytes.
 * Asynchronous on `stream`, allocates nothing.  Errors: BM_ERR_INVALID_ARG, BM_ERR_KEY_MISMATCH,
 * BM_ERR_WORKSPACE, BM_ERR_CUDA. */
size_t bm_expand_ws_bytes(const bm_params *, int32_t nq);
int bm_expand(const bm_params *, const bm_xk_dev *, const uint64_t *d_in, int32_t nq, uint64_t *d_out, void *d_ws,
              size_t ws_bytes, void *stream);
/* f4: SERVER-SIDE ENROLLMENT PACKING, Fig. 3 (SPEC.md:282-293,
 * DESIGN.md reading R27), same extended chain.  d_in [n][2][3][N] (level 2, NTT): the level-2
 * encryptions of bm_encode_enroll's templates first_template .. first_template + n - 1.  For template
 * u = tB + k and part i:  set[t][i] += Rot_right(Res_q2(Mul(P)(C_u, E_i)), (k - i) s), the rotation
 * done as left rotations by s 2^b for the set bits b of (i - k) mod B.  d_db [n_sets][p][2][2][N]
 * (level 1, NTT; zero-filled for a fresh store) is accumulated in place -- the layout bm_encrypt_db
 * writes and bm_match reads.  Asynchronous on `stream`, allocates nothing; d_ws of at least
 * bm_enroll_ws_bytes(prm, n) bytes.  Errors: BM_ERR_INVALID_ARG (also: no enrollment masks
 * uploaded), BM_ERR_KEY_MISMATCH, BM_ERR_MISSING_ROTATION_KEY, BM_ERR_CAPACITY (a template beyond
 * n_sets), BM_ERR_WORKSPACE, BM_ERR_CUDA. */
size_t bm_enroll_ws_bytes(const bm_params *, int64_t n);
int bm_enroll(const bm_params *, const bm_xk_dev *, const uint64_t *d_in, int64_t n, int64_t first_template,
              uint64_t *d_db, int64_t n_sets, void *d_ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------------
 * f1: OUTPUT COMPRESSION (DESIGN.md
 * reading R28), on the same extended chain: HE-C^3 runs one level higher -- level-2 DB and query
 * parts (bm_encrypt_l2 of bm_encode_db / bm_encode_query plaintexts), tensor over three limbs,
 * 3-digit relinearisation and Res by q2, the ladder at level 1 -- and then every set's result C_t
 * is compressed: Res_q1(Mul(P)(C_t, M)), M[x] = [x mod s = 0] (the score slots), rotated right by
 * t mod s at level 0 and added into packed ciphertext t / s.  Packed ciphertext g holds, at slot
 * k s + u, the score of set g s + u's block k; every other slot of the uncompressed output (the
 * partial sums) is masked away, and the output is s times smaller.
 * ------------------------------------------------------------------------------------------- */
typedef struct bm_ck bm_ck;           /* host: rlk2 (3 digits), ladder keys at level 1, rotation keys */
typedef struct bm_ck_dev bm_ck_dev;

/* Keys for keygen(seed)'s secret: rlk2_j (j < 3) over {q0,q1,q2,P}: (-a s + e + [l = j](P mod q_l)
 * s^2, a); the level-1 Galois keys of 2^i, i < log2 s (the f3 family); the level-0 Galois keys of the
 * right rotations by u = 1..s-1 (left by S - u).  Export layouts: rlk2 [3][2][4 limbs q0,q1,q2,P][N],
 * gkl [log2 s][2][2][3 limbs q0,q1,P][N], gkc [s-1][2][2 limbs q0,P][N]. */
int bm_ck_keygen(const bm_params *, uint64_t seed, bm_ck **out);
void bm_ck_free(bm_ck *);
int bm_ck_export(const bm_ck *, uint64_t *rlk2, uint64_t *gkl, uint64_t *gkc);
/* The score mask M at scale q1 (int64 [N]). */
int bm_encode_cmp_mask(const bm_params *, int64_t *pt);
/* Upload keys and mask (synchronous).  Errors: BM_ERR_KEY_MISMATCH, BM_ERR_CUDA, BM_ERR_OOM. */
int bm_ck_to_device(const bm_params *, const bm_ck *, const int64_t *h_mask, bm_ck_dev **out);
void bm_ck_dev_free(bm_ck_dev *);
/* The compressed scan: d_db [n_sets][p][2][3][N], d_q [nq][p][2][3][N] (level 2, NTT) ->
 * d_out [nq][ceil(n_sets / s)][2][N] (level 0, COEFFICIENT domain, scale 2^80 / q2; overwritten).
 * Asynchronous, allocates nothing; d_ws of bm_match_cmp_ws_bytes(...) bytes.  Errors as bm_match. */
size_t bm_match_cmp_ws_bytes(const bm_params *, int64_t n_sets, int32_t nq);
int bm_match_cmp(const bm_params *, const bm_ck_dev *, const uint64_t *d_db, int64_t n_sets, const uint64_t *d_q,
                 int32_t nq, uint64_t *d_out, void *d_ws, size_t ws_bytes, void *stream);
/* Client: decrypt n packed results h_ct [n][2][1][N] and decode ALL S slots into slots [n][S]
 * (slot k s + u of packed ciphertext g = score of set g s + u, block k). */
int bm_decrypt_packed(const bm_params *, const bm_sk *, const uint64_t *h_ct, int64_t n, double *slots);

int bm_sync(void *stream);
const char *bm_strerror(int status);
/* Library build information ("sm_100a", git hash...) */
const char *bm_build_info(void);

#ifdef __cplusplus
}
#endif
#endif
