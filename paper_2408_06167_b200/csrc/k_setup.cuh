// k_setup.cuh -- setup kernels: k_encrypt (a1, a2, f3's level-2 encryption), k_convert
// (NTT <-> coefficient), k_key_ntt (key upload).
// Included once, by device.cu (one translation unit: the kernels are launched from its host side).
#pragma once

// ================================================================== encryption / conversion / keys
struct EncK {
    PrimeK pr[4];
    const ulonglong2 *pk; // [2][n_limbs][N]
    const int64_t *pt;    // [n][N]
    uint64_t *out;        // [n][2][n_limbs][N]
    uint64_t first_obj, seed;
    uint32_t kx[5];       // ChaCha20 key extension of this call (zeros when seeded, bm_rng_mode)
    int n_limbs;          // 2 (level 1: q0, q1) or 3 (f3 level 2: q0, q1, q2)
    int lp[3];            // prime index of each limb
};

// sample a small polynomial of stream st into sm (residues mod q), adding pt if given
BM_D void sample_to_smem(uint64_t *sm, const Stream &st, int gauss, uint64_t q, uint64_t one_p, const int64_t *pt)
{
    for (int r = 0; r < N / 8 / T; r++) {
        const int b = threadIdx.x + T * r;
        uint64_t d[8];
        chacha_draws(st, (uint32_t)b, d);
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int k = 8 * b + i;
            const int v = gauss ? gauss_of(d[i], c_cdt) : ternary_of(d[i]);
            uint64_t x = v >= 0 ? (uint64_t)v : q - (uint64_t)(-v);
            if (pt) {
                const int64_t m = pt[k];
                uint64_t mr = m >= 0 ? reduce64((uint64_t)m, q, one_p) : submod_d(0, reduce64((uint64_t)(-m), q, one_p), q);
                x = csub(x + mr, q);
            }
            sm[pidx(k)] = x;
        }
    }
}

__global__ void __launch_bounds__(T, 1) k_encrypt(EncK Ek)
{
    extern __shared__ uint64_t sm[];
    const int tid = threadIdx.x;
    const int nl = Ek.n_limbs;
    const int64_t ct = blockIdx.x / nl;
    const int l = (int)(blockIdx.x % nl), pi = Ek.lp[l];
    const uint64_t o = Ek.first_obj + (uint64_t)ct;
    const PrimeK P = Ek.pr[pi];
    const uint64_t q = P.q;
    uint64_t *c0 = Ek.out + ((size_t)ct * 2 * nl + 0 + l) * N;
    uint64_t *c1 = Ek.out + ((size_t)ct * 2 * nl + nl + l) * N;
    const ulonglong2 *pb = Ek.pk + (size_t)(0 + l) * N, *pa = Ek.pk + (size_t)(nl + l) * N;
    uint64_t a[E];
    // phase 0: NTT(u) -> kept in c0 until phase 2;  phase 1: c1 = u a + e1;  phase 2: c0 = u b + e0 + pt
    for (int ph = 0; ph < 3; ph++) {
        BM_SYNCTHREADS();
        const uint32_t purpose = ph == 0 ? P_ENC_U : ph == 1 ? P_ENC_E1 : P_ENC_E0;
        sample_to_smem(sm, make_stream(Ek.seed, purpose, o, 0, Ek.kx), ph != 0, q, P.one_p,
                       ph == 2 ? Ek.pt + (size_t)ct * N : nullptr);
        BM_SYNCTHREADS();
#pragma unroll
        for (int e = 0; e < E; e++) a[e] = sm[pidx(j_M1(tid, e))];
        fwd_rt(a, sm, P, pi);
        if (ph == 0) {
            store_eval(c0, a);
            continue;
        }
        uint64_t *dst = ph == 1 ? c1 : c0;
        const ulonglong2 *key = ph == 1 ? pa : pb;
#pragma unroll
        for (int e = 0; e < E; e++) {
            const int j = pos_M4(tid, e);
            dst[j] = csub(csub(shoup(c0[j], ldkey1(key, j), q) + a[e], 2 * q), q);
        }
    }
}

struct ConvK {
    PrimeK pr[4];
    const uint64_t *in;
    uint64_t *out;
    int n_limbs;
    int lp[4];          // prime index of each limb
    uint64_t scale[4];  // k_key_ntt: constant folded into each limb (canonical, < q)
    int planar;         // k_key_ntt: write (w, w') as two planes per polynomial (ldkey2) instead of pairs
};

// one block per polynomial; dir 0: coefficient -> NTT, 1: NTT -> coefficient
__global__ void __launch_bounds__(T, 1) k_convert(ConvK C, int dir)
{
    extern __shared__ uint64_t sm[];
    const int64_t poly = blockIdx.x;
    const int li = (int)(poly % C.n_limbs);
    const int pidx_ = C.lp[li];
    const PrimeK P = C.pr[pidx_];
    const uint64_t *in = C.in + (size_t)poly * N;
    uint64_t *out = C.out + (size_t)poly * N;
    uint64_t a[E];
    if (dir == 0) {
        load_coef(a, in);
        fwd_rt(a, sm, P, pidx_);
        BM_SYNCTHREADS(); // in may alias out
        store_eval(out, a);
    } else {
        load_eval(a, in);
        inv_rt(a, sm, P, pidx_);
        BM_SYNCTHREADS();
        store_coef(out, a);
    }
}

// keys: canonical coefficients -> NTT domain Shoup pairs (storage order pos_M4)
__global__ void __launch_bounds__(T, 1) k_key_ntt(ConvK C, ulonglong2 *dst)
{
    extern __shared__ uint64_t sm[];
    const int tid = threadIdx.x;
    const int64_t poly = blockIdx.x;
    const int li = (int)(poly % C.n_limbs);
    const int pidx_ = C.lp[li];
    const PrimeK P = C.pr[pidx_];
    uint64_t a[E];
    load_coef(a, C.in + (size_t)poly * N);
    fwd_rt(a, sm, P, pidx_);
    const uint64_t sc = C.scale[li];
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint64_t w = (uint64_t)((u128)a[e] * sc % P.q); // setup only: plain 128-bit remainder
        const uint64_t wp = (uint64_t)(((u128)w << 64) / P.q);
        if (C.planar) {
            uint64_t *d = reinterpret_cast<uint64_t *>(dst) + (size_t)poly * 2 * N;
            d[pos_M4(tid, e)] = w;
            d[N + pos_M4(tid, e)] = wp;
        } else {
            dst[(size_t)poly * N + pos_M4(tid, e)] = make_ulonglong2(w, wp);
        }
    }
}

// ================================================================== client-side decryption on the device (a9)
// PAPER.md:347-349 (the client decrypts the returned ciphertexts and reads the score slots), at the
// scale of a 1:N identification batch: one CTA per level-0 ciphertext (c0, c1) in the canonical
// coefficient domain (bm_match's output):
//   m = c0 + INTT_q0(NTT_q0(c1) * NTT_q0(s))  (mod q0), centred      -- 2 transforms
//   X[t] = sum_k m_k zeta^(k (2t + 1)), zeta = exp(i pi / N)          -- the canonical embedding at
//          the odd powers: y_k = m_k zeta^k, then an N-point FP64 FFT (positive exponent) in shared memory
//   score[b] = Re X[t(b s)] / out_scale, t(j) = (5^j mod 2N - 1) / 2   (slot j = b s holds template b)
// The host bm_decrypt evaluates the same slots by the direct O(N) cosine sum (the reference the GPU
// test compares against).
struct DecK {
    PrimeK pr0;
    const uint64_t *s;      // planar Shoup key of the secret, NTT domain mod q0 (2N u64)
    const uint64_t *ct;     // [n][2][N] level 0, coefficient domain
    double *scores;         // [n][B]
    const double2 *zeta;    // [N]: exp(i pi k / N)
    const int32_t *slot_t;  // [S]: t(j)
    int32_t B, s_len;
    double inv_scale;
};
constexpr size_t DEC_SMEM_BYTES = (size_t)N * sizeof(double2); // 128 KiB (also holds the NTT exchanges)

__global__ void __launch_bounds__(T, 1) k_decrypt(DecK K)
{
    extern __shared__ uint64_t sm[];
    double2 *X = reinterpret_cast<double2 *>(sm);
    const int tid = threadIdx.x;
    const int64_t c = blockIdx.x;
    const uint64_t *c0 = K.ct + (size_t)c * 2 * N, *c1 = c0 + N;
    uint64_t a[E];
    load_coef(a, c1);
    fwd<0, false>(a, sm, K.pr0); // [0, 2 q0)
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        ulonglong2 w, wb;
        ldkey2(K.s, pos_M4(tid, e), w, wb);
        a[e] = shoup4<0>(a[e], w);       // [0, 4 q0): the inverse transform's input bound
        a[e + 1] = shoup4<0>(a[e + 1], wb);
    }
    inv<0>(a, sm, K.pr0); // c1 s, canonical, coefficient j_M1(tid, e)
    BM_SYNCTHREADS();      // the exchange buffer becomes X
#pragma unroll
    for (int e = 0; e < E; e++) {
        const int k = j_M1(tid, e);
        uint64_t v = a[e] + c0[k];
        v = v >= Q0 ? v - Q0 : v;
        const double m = v > (Q0 >> 1) ? -(double)(Q0 - v) : (double)v; // centred, exact (< 2^53 in practice)
        const double2 z = K.zeta[k];
        X[brev13(k)] = make_double2(m * z.x, m * z.y);
    }
    BM_SYNCTHREADS();
    // iterative radix-2 DIT over bit-reversed input: block length len, twiddle exp(2 pi i k / len) = zeta[2 k N / len]
#pragma unroll 1
    for (int lg = 1; lg <= LOGN; lg++) {
        const int half = 1 << (lg - 1);
        for (int b = tid; b < N / 2; b += T) {
            const int k = b & (half - 1);
            const int i = ((b >> (lg - 1)) << lg) + k, j = i + half;
            const double2 w = K.zeta[(2 * k) << (LOGN - lg)];
            const double2 u = X[i], v = X[j];
            const double vr = v.x * w.x - v.y * w.y, vi = v.x * w.y + v.y * w.x;
            X[i] = make_double2(u.x + vr, u.y + vi);
            X[j] = make_double2(u.x - vr, u.y - vi);
        }
        BM_SYNCTHREADS();
    }
    for (int b = tid; b < K.B; b += T) {
        BM_CHECK(b * K.s_len < SLOTS && K.slot_t[b * K.s_len] < N);
        K.scores[(size_t)c * K.B + b] = X[K.slot_t[b * K.s_len]].x * K.inv_scale;
    }
}
