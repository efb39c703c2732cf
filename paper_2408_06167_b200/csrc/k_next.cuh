// k_next.cuh -- the NEXT-row kernels: f3 query expansion and f4 server-side
// enrollment (ExpK: k_exp_mask, k_rot1_digits, k_rot1_ks, k_enroll_add), f1 compressed scan (CmpK:
// k_digits3, k_relin3a, k_relin3b, k_cmp_mask, k_cmp_rot, k_cmp_add).
// Included once, by device.cu (one translation unit: the kernels are launched from its host side).
#pragma once

// ================================================================== f3: server-side query expansion
// Algorithm 1 "Input Ciphertext Expansion" on the chain
// extended by q2 (readings R24-R26).  Per query ciphertext (level 2 = {q0, q1, q2}, NTT
// domain) and part i < p -- a "ct" below is one (query, part) output:
//   X1 k_exp_mask   (ct, c)  C_i = Res_q2(C (.) X_i): the mask product in all three limbs, y = INTT_q2
//                            of the q2 limb, then per Q limb out = c X_i q2^-1 - NTT(q2^-1 y^) with
//                            q2^-1 y^ = q2^-1 y - [y > q2/2] (q2^-1 is folded into the device masks'
//                            Q limbs, like P^-1 into the key-switching keys): 3 transforms
//   for t < log2 p, r = s 2^t, g = 5^r:  C_i <- C_i + Rot(C_i, r) at level 1 (2-digit key switch):
//   X2 k_rot1_digits (ct, l) sigma_g(c1)[q_l] (an NTT-index gather), x_l = INTT_{q_l} of it, ModUp:
//                            x0 -> NTT_{q1}, NTT_P; x1 -> NTT_{q0}, NTT_P: 3 transforms
//   X3 k_rot1_ks    (ct, c)  KS_c over {q0, q1, P} with gk1 (P^-1 in its Q limbs), y = INTT_P(KS_c[P]),
//                            c_c <- c_c + [c = 0] sigma_g(c0) + P^-1 KS_c - NTT(P^-1 y^) per Q limb: 3
// XU per ct: [0] sigma(c1)[q0] (digit 0 in its own limb), [1] x0~[q1], [2] x0~[P], [3] x1~[q0],
//            [4] sigma(c1)[q1] (digit 1 in its own limb), [5] x1~[P]   (all NTT domain)
struct ExpK {
    PrimeK pr[4];            // q0, q1, P, q2
    ulonglong2 pinv[2];      // P^-1 mod q0, q1
    ulonglong2 q2inv[2];     // q2^-1 mod q0, q1
    const ulonglong2 *mask;  // [p][3 limbs q0,q1,q2][N]; the Q limbs carry q2^-1
    const ulonglong2 *gk;    // this step's level-1 Galois key [2 digits][2 comps][3 limbs q0,q1,P][N]
    const uint64_t *in;      // [n_q][2][3][N] level 2 (the chunk's first query)
    uint64_t *out;           // [n_q][p][2][2][N] level 1 (the chunk's first query)
    uint64_t *XU;            // [cts][6][N]
    int p;
    uint32_t g;              // Galois element of this step
    // f4 enrollment mode (enroll = 1): pure rotation C <- Rot(C) (no add), applied only to the parts
    // whose amount m = (i - k) mod B has bit `bit` set (template u = u0 + ct / p, k = u mod B)
    int enroll, Bk, bit;
    int64_t u0;
    BM_D bool skip(int64_t ct) const
    {
        if (!enroll) return false;
        const int64_t u = u0 + ct / p;
        const int i = (int)(ct % p), k = (int)(u % Bk);
        const int m = ((i - k) % Bk + Bk) % Bk;
        return !((m >> bit) & 1);
    }
};
constexpr int XU_POLYS = 6;
constexpr size_t X1_SMEM_BYTES = (SMEM_WORDS + (size_t)N) * sizeof(uint64_t);
constexpr size_t X2_SMEM_BYTES = 2 * SMEM_WORDS * sizeof(uint64_t);
constexpr size_t X3_SMEM_BYTES = (2 * SMEM_WORDS + (size_t)N) * sizeof(uint64_t);

__global__ void __launch_bounds__(T, 1) k_exp_mask(ExpK K)
{
    extern __shared__ uint64_t sm[];
    uint64_t *ys = sm + SMEM_WORDS;
    const int tid = threadIdx.x;
    const int64_t ct = blockIdx.x >> 1;
    const int c = blockIdx.x & 1;
    const int64_t jq = ct / K.p;
    const int i = (int)(ct % K.p);
    const uint64_t *cin = K.in + ((size_t)jq * 2 + c) * 3 * N; // [l][N]
    const ulonglong2 *mk = K.mask + (size_t)i * 3 * N;
    uint64_t *co = K.out + ((size_t)ct * 2 + c) * 2 * N;     // [l][N]
    uint64_t a[E];
    // q2 limb: y = INTT_q2(c[q2] X_i[q2]) (canonical)
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int pos = pos_M4(tid, e);
        const ulonglong2 v = ld2(cin + 2 * N + pos);
        ulonglong2 ma, mb;
        ldkey2(mk + 2 * N, pos, ma, mb);
        a[e] = reduce_bnd<3>(shoup4<3>(v.x, ma));
        a[e + 1] = reduce_bnd<3>(shoup4<3>(v.y, mb));
    }
    inv_f<3>(a, sm, K.pr[3].invf, K.pr[3].ninvf, K.pr[3].ninv_w1f); // canonical (FP64 pipe)
#pragma unroll
    for (int e = 0; e < E; e++) ys[tid + T * e] = a[e];
    // q1 limb (FP64-pipe transform): q2^-1 y^ mod q1 = q2^-1 y - [y > q2/2]
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint64_t y = a[e];
        a[e] = reduce_bnd<1>(shoup4<1>(y, K.q2inv[1]) + (y > (Q2 >> 1) ? Q1 - 1 : 0));
    }
    fwd_f<1>(a, sm, K.pr[1].fwdf);
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int pos = pos_M4(tid, e);
        const ulonglong2 v = ld2(cin + 1 * N + pos);
        ulonglong2 ma, mb;
        ldkey2(mk + 1 * N, pos, ma, mb);
        const uint64_t xa = shoup4<1>(v.x, ma), xb = shoup4<1>(v.y, mb);
        st2(co + 1 * N + pos, reduce_bnd<1>(xa + Q1 - a[e]), reduce_bnd<1>(xb + Q1 - a[e + 1]));
    }
    // q0 limb
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint64_t y = ys[tid + T * e];
        a[e] = shoup4<0>(y, K.q2inv[0]) + (y > (Q2 >> 1) ? Q0 - 1 : 0); // < 5 q0
    }
    fwd<0>(a, sm, K.pr[0]); // canonical
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int pos = pos_M4(tid, e);
        const ulonglong2 v = ld2(cin + pos);
        ulonglong2 ma, mb;
        ldkey2(mk, pos, ma, mb);
        const uint64_t xa = shoup4<0>(v.x, ma), xb = shoup4<0>(v.y, mb);
        st2(co + pos, reduce_bnd<0>(xa + Q0 - a[e]), reduce_bnd<0>(xb + Q0 - a[e + 1]));
    }
}

// X2: digits of sigma_g(c1) and their ModUp (the rotation's half of k_digits)
__global__ void __launch_bounds__(T, 1) k_rot1_digits(ExpK K)
{
    extern __shared__ uint64_t sm[];
    uint64_t *S = sm + SMEM_WORDS, *xs = S; // xs reuses S once the gather is done (the INTT's barriers)
    const int tid = threadIdx.x;
    const int64_t ct = blockIdx.x >> 1;
    const int l = blockIdx.x & 1;
    if (K.skip(ct)) return;
    const uint64_t *c1 = K.out + ((size_t)ct * 2 + 1) * 2 * N + (size_t)l * N;
    uint64_t *xu = K.XU + (size_t)ct * XU_POLYS * N;
    const int nt = nat_tid(tid);
    stage_nat(S, c1); // natural order: conflict-free gather (ntt3.cuh nat_at)
    BM_SYNCTHREADS();
    uint64_t a[E];
#pragma unroll
    for (int e = 0; e < E; e++) a[e] = S[nat_auto(nt, e, K.g)];
    store_eval(xu + (size_t)(l == 0 ? 0 : 4) * N, a); // the digit in its own limb: sigma(c1)[q_l]
    if (l == 0) {
        inv<0>(a, sm, K.pr[0]);
#pragma unroll
        for (int e = 0; e < E; e++) {
            xs[tid + T * e] = a[e];
            a[e] = reduce_bnd<1>(a[e]); // x0 < q0 < 2^58: x0 mod q1
        }
        fwd_f<1>(a, sm, K.pr[1].fwdf);
        store_eval(xu + 1 * N, a);
    } else {
        inv_f<1>(a, sm, K.pr[1].invf, K.pr[1].ninvf, K.pr[1].ninv_w1f);
#pragma unroll
        for (int e = 0; e < E; e++) xs[tid + T * e] = a[e];
        fwd<0, false>(a, sm, K.pr[0]); // x1 < q1 < q0; lazy [0, 2 q0): a Shoup operand only
        store_eval(xu + 3 * N, a);
    }
#pragma unroll
    for (int e = 0; e < E; e++) a[e] = xs[tid + T * e];
    fwd<2, false>(a, sm, K.pr[2]);
    store_eval(xu + (size_t)(l == 0 ? 2 : 5) * N, a);
}

// X3: key switch + ModDown + add, one CTA per (ct, component), c_c updated in place
__global__ void __launch_bounds__(T, 1) k_rot1_ks(ExpK K)
{
    extern __shared__ uint64_t sm[];
    uint64_t *S = sm + SMEM_WORDS, *ys = sm + 2 * SMEM_WORDS;
    const int tid = threadIdx.x;
    const int64_t ct = blockIdx.x >> 1;
    const int c = blockIdx.x & 1;
    if (K.skip(ct)) return;
    const uint64_t *xu = K.XU + (size_t)ct * XU_POLYS * N;
    uint64_t *cc = K.out + ((size_t)ct * 2 + c) * 2 * N; // [l][N]
    const uint64_t *c0 = K.out + (size_t)ct * 4 * N;
    const ulonglong2 *k0 = K.gk + (size_t)(0 * 2 + c) * 3 * N, *k1 = K.gk + (size_t)(1 * 2 + c) * 3 * N;
    uint64_t a[E];
    // P limb: y = INTT_P(x0~[P] gk[0][c][P] + x1~[P] gk[1][c][P])
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int pos = pos_M4(tid, e);
        const ulonglong2 u = ld2(xu + 2 * N + pos), v = ld2(xu + 5 * N + pos);
        // 8-byte keys (w planes), exact 128-bit inner products, one reduction (as K3)
        const ulonglong2 w0 = ld2(reinterpret_cast<const uint64_t *>(k0 + 2 * N) + pos);
        const ulonglong2 w1 = ld2(reinterpret_cast<const uint64_t *>(k1 + 2 * N) + pos);
        a[e] = red128s<2>(dot2(u.x, w0.x, v.x, w1.x), K.pr[2].r64);
        a[e + 1] = red128s<2>(dot2(u.y, w0.y, v.y, w1.y), K.pr[2].r64);
    }
    inv<2>(a, sm, K.pr[2]);
#pragma unroll
    for (int e = 0; e < E; e++) ys[tid + T * e] = a[e];
#pragma unroll 1
    for (int l = 1; l >= 0; l--) { // q1 (FP64-pipe transform), then q0
        // P^-1 y^ mod q_l = P^-1 y - [y > P/2]
        if (l == 1) {
#pragma unroll
            for (int e = 0; e < E; e++) {
                const uint64_t y = ys[tid + T * e];
                a[e] = reduce_bnd<1>(shoup4<1>(y, K.pinv[1]) + (y > (QP >> 1) ? Q1 - 1 : 0));
            }
            fwd_f<1>(a, sm, K.pr[1].fwdf);
        } else {
#pragma unroll
            for (int e = 0; e < E; e++) {
                const uint64_t y = ys[tid + T * e];
                a[e] = shoup4<0>(y, K.pinv[0]) + (y > (QP >> 1) ? Q0 - 1 : 0); // < 5 q0
            }
            fwd<0>(a, sm, K.pr[0]);
        }
        if (c == 0) { // sigma_g(c0)[q_l] by a gather (natural order; c0 is this CTA's to overwrite)
            BM_SYNCTHREADS(); // previous limb's gathers from S are done
            stage_nat(S, c0 + (size_t)l * N);
            BM_SYNCTHREADS();
        }
        const uint64_t q = l ? Q1 : Q0;
        const ulonglong2 *kl0 = k0 + (size_t)l * N, *kl1 = k1 + (size_t)l * N;
        const uint64_t *x0 = xu + (size_t)(l == 0 ? 0 : 1) * N, *x1 = xu + (size_t)(l == 0 ? 3 : 4) * N;
#pragma unroll
        for (int e = 0; e < E; e += 2) {
            const int pos = pos_M4(tid, e);
            const ulonglong2 u = ld2(x0 + pos), v = ld2(x1 + pos);
            // C + Rot(C) (expansion) or Rot(C) alone (enrollment)
            const ulonglong2 cv = K.enroll ? make_ulonglong2(0, 0)
                                           : *reinterpret_cast<const ulonglong2 *>(cc + (size_t)l * N + pos);
            uint64_t ka, kb;
            const ulonglong2 w0 = ld2(reinterpret_cast<const uint64_t *>(kl0) + pos);
            const ulonglong2 w1 = ld2(reinterpret_cast<const uint64_t *>(kl1) + pos);
            const u128 sa = (u128)u.x * w0.x + (u128)v.x * w1.x, sb = (u128)u.y * w0.y + (u128)v.y * w1.y;
            if (l) {
                ka = red128s<1>(sa, K.pr[1].r64);
                kb = red128s<1>(sb, K.pr[1].r64);
            } else {
                ka = red128s<0>(sa, K.pr[0].r64);
                kb = red128s<0>(sb, K.pr[0].r64);
            }
            uint64_t va = cv.x + ka + q - a[e], vb = cv.y + kb + q - a[e + 1]; // < 11 q
            if (c == 0) {
                va += S[nat_auto(nat_tid(tid), e, K.g)];
                vb += S[nat_auto(nat_tid(tid), e + 1, K.g)];
            }
            a[e] = l ? reduce_bnd<1>(va) : reduce_bnd<0>(va);
            a[e + 1] = l ? reduce_bnd<1>(vb) : reduce_bnd<0>(vb);
        }
        if (c == 0) BM_SYNCTHREADS(); // every gather of the old c0[q_l] is done before it is overwritten
#pragma unroll
        for (int e = 0; e < E; e += 2) st2(cc + (size_t)l * N + pos_M4(tid, e), a[e], a[e + 1]);
    }
}

// f4: set[t][i] += the rotated parts of its templates (elementwise in the NTT domain, canonical)
// grid: (local set, part, comp x limb, N / 256 slices); W [n][p][2][2][N] holds templates u0 .. u0+n-1
__global__ void __launch_bounds__(256) k_enroll_add(const uint64_t *W, int64_t u0, int64_t n, int p, int Bk,
                                                    int64_t t0, uint64_t *db)
{
    const int slice = blockIdx.x % (N / 256);
    int64_t b = blockIdx.x / (N / 256);
    const int cl = (int)(b % 4);
    b /= 4;
    const int i = (int)(b % p);
    const int64_t t = t0 + b / p;
    const uint64_t q = (cl & 1) ? Q1 : Q0;
    const int k = slice * 256 + threadIdx.x;
    const int64_t lo = t * Bk > u0 ? t * Bk : u0, hi = (t + 1) * Bk < u0 + n ? (t + 1) * Bk : u0 + n;
    uint64_t *dst = db + (((size_t)t * p + i) * 4 + cl) * N + k;
    uint64_t acc = *dst;
    for (int64_t u = lo; u < hi; u++) acc = csub(acc + W[(((size_t)(u - u0) * p + i) * 4 + cl) * N + k], q);
    *dst = acc;
}

// ================================================================== f1: output compression
// SURVEY.md sec. 8f row f1 (reading R28): HE-C^3 one
// level up on the extended chain, then the compression.  Per chunk of (query, set) pairs:
//   k_tensor<3>                        tensor + part sum over the three level-2 limbs
//   C1 k_digits3   (pair, digit j)     x_j = INTT_{q_j}(d2[q_j]), ModUp to the other two Q primes and P
//   C2 k_relin3a/b (pair, c[, l])      KS_c over {q0,q1,q2,P} (rlk2, P^-1 in its Q limbs), ModDown fused
//                                      with Res by q2 (the R22 rewriting with q2 in q1's role): level 1
//   ladder at level 1: log2 s x (k_rot1_digits, k_rot1_ks) with the ladder's level-1 Galois keys
//   C3 k_cmp_mask  (pair, c)           Res_q1(Mul(P)(C, M)): level 0 (q1^-1 folded into M's q0 limb)
//   C4 k_cmp_rot   (pair)              right rotation by u = t mod s (left by S - u) at level 0 and the
//                                      output INTT (u = 0: the INTT only); coefficient domain
//   C5 k_cmp_add                        packed[g] += the s rotated results of group g
constexpr int D2X_POLYS = 9; // XU at level 2: per digit j its 3 ModUp targets (other two Q limbs, P)
constexpr size_t C1_SMEM_BYTES = (SMEM_WORDS + (size_t)N) * sizeof(uint64_t);
constexpr size_t C4_SMEM_BYTES = 3 * SMEM_WORDS * sizeof(uint64_t);

BM_D uint32_t pow5_mod2n(uint32_t r) // 5^r mod 2N
{
    uint32_t x = 1, b = 5;
    for (; r; r >>= 1, b = (b * b) & (2 * N - 1))
        if (r & 1) x = (x * b) & (2 * N - 1);
    return x;
}

struct CmpK {
    MatchK m;                 // pr[4], pinv[2], q1inv, D01/D2/XU/XC/XR/XO, chunk geometry
    ulonglong2 pinv2;         // P^-1 mod q2
    ulonglong2 q2inv[2];      // q2^-1 mod q0, q1
    const ulonglong2 *rlk2;   // [3 j][2 c][4 limbs q0,q1,q2,P][N]
    const ulonglong2 *gkc;    // [s-1][2 c][2 limbs q0,P][N]
    const ulonglong2 *mask;   // [2 limbs q0,q1][N], q1^-1 in the q0 limb
    uint64_t *scr;            // [pairs][2][N] scratch of k_cmp_rot
    int s;
};

__global__ void __launch_bounds__(T, 1) k_digits3(CmpK C)
{
    extern __shared__ uint64_t sm[];
    uint64_t *xs = sm + SMEM_WORDS;
    const MatchK &K = C.m;
    const int tid = threadIdx.x;
    const int64_t pi = blockIdx.x / 3;
    const int j = (int)(blockIdx.x % 3);
    uint64_t a[E];
    load_eval(a, K.D2 + ((size_t)pi * 3 + j) * N);
    uint64_t *xu = K.XU + ((size_t)pi * D2X_POLYS + 3 * j) * N; // targets: other Q limbs ascending, then P
    if (j == 0) inv<0>(a, sm, K.pr[0]);
    else if (j == 1) inv_f<1>(a, sm, K.pr[1].invf, K.pr[1].ninvf, K.pr[1].ninv_w1f);
    else inv_f<3>(a, sm, K.pr[3].invf, K.pr[3].ninvf, K.pr[3].ninv_w1f);
#pragma unroll
    for (int e = 0; e < E; e++) xs[tid + T * e] = a[e]; // x_j in [0, q_j), non-centred (reading R4)
#pragma unroll 1
    for (int k = 0; k < 3; k++) {
        // target k: the other two Q limbs ascending, then P (prime indices: 0 q0, 1 q1, 2 P, 3 q2)
        const int tp = k == 2 ? 2 : j == 0 ? (k == 0 ? 1 : 3) : j == 1 ? (k == 0 ? 0 : 3) : (k == 0 ? 0 : 1);
#pragma unroll
        for (int e = 0; e < E; e++) {
            const uint64_t x = xs[tid + T * e];
            if (tp == 1) a[e] = j == 0 ? reduce_bnd<1>(x) : x;                 // q1: x0 < 2^58; x2 < q2 < q1
            else if (tp == 3) a[e] = j == 0 ? reduce_bnd<3>(x) : csub(x, Q2);  // q2: x0 < 2^58; x1 < q1 < 2 q2
            else a[e] = x;                                                     // q0 (x1, x2 < q0), P (x < P)
        }
        if (tp == 2) fwd<2, false>(a, sm, K.pr[2]);       // lazy [0, 2P): a Shoup operand only
        else if (tp == 1) fwd_f<1>(a, sm, K.pr[1].fwdf);   // canonical (FP64 pipe)
        else if (tp == 3) fwd_f<3>(a, sm, K.pr[3].fwdf);  // canonical (FP64 pipe)
        else fwd<0, false>(a, sm, K.pr[0]);               // lazy [0, 2 q0)
        store_eval(xu + (size_t)k * N, a);
    }
}

// the digit j's residue in limb tp (prime index) as stored by k_digits3 / k_tensor<3>
BM_D const uint64_t *digit_poly(const MatchK &K, int64_t pi, int j, int tp)
{
    const int lj = j == 2 ? 3 : j; // prime index of digit j's own limb
    if (tp == lj) return K.D2 + ((size_t)pi * 3 + j) * N;
    const int k = tp == 2 ? 2 : j == 0 ? (tp == 1 ? 0 : 1) : j == 1 ? (tp == 0 ? 0 : 1) : (tp == 0 ? 0 : 1);
    return K.XU + ((size_t)pi * D2X_POLYS + 3 * j + k) * N;
}

// C2: key switch with rlk2 + ModDown + Res by q2 (reading R28; the R22 rewriting), in two kernels so
// that each CTA runs at most two transform kinds (with all four in one kernel ncu's top stall was
// no_instruction: 6.4 warps per issue -- the unrolled transforms, ~40 KB of SASS each, overflow the
// instruction cache):
//   C2a (pair, c):     y = INTT_P(KS_c[P]);  U = INTT_q2(d_c[q2] + P^-1 KS_c[q2]);  R = U - P^-1 y^ (mod q2)
//                      -> y and R to the workspace (XR, XO: free until k_cmp_mask)
//   C2b (pair, c, l):  out_c[q_l] = q2^-1 (d_c[q_l] + P^-1 KS_c[q_l] - NTT_l(P^-1 y^ + z^)), z^ = c_q2(R)
constexpr size_t C2_SMEM_BYTES = (SMEM_WORDS + (size_t)N) * sizeof(uint64_t);
BM_D const ulonglong2 *rlk2_key(const CmpK &C, int j, int c, int l) // rlk2 [j][c][l][N], l: 0 q0, 1 q1, 2 q2, 3 P
{
    return C.rlk2 + (((size_t)j * 2 + c) * 4 + l) * N;
}
// 8-byte keys: the w plane of a planar poly (positions pos, pos + 1); exact 128-bit inner products
BM_D ulonglong2 rlk2_w(const ulonglong2 *k, int pos) { return ld2(reinterpret_cast<const uint64_t *>(k) + pos); }

__global__ void __launch_bounds__(T, 1) k_relin3a(CmpK C)
{
    extern __shared__ uint64_t sm[];
    uint64_t *ys = sm + SMEM_WORDS;
    const MatchK &K = C.m;
    const int tid = threadIdx.x;
    const int64_t pi = blockIdx.x >> 1;
    const int c = blockIdx.x & 1;
    const uint64_t *dc = K.D01 + ((size_t)pi * 6 + c * 3) * N; // d_c[q0], d_c[q1], d_c[q2]
    uint64_t *yg = K.XR + ((size_t)pi * 2 + c) * N, *rg = K.XO + ((size_t)pi * 2 + c) * N; // thread-private order
    uint64_t a[E];
    // ---- P limb
    {
        const uint64_t *x0 = digit_poly(K, pi, 0, 2), *x1 = digit_poly(K, pi, 1, 2), *x2 = digit_poly(K, pi, 2, 2);
        const ulonglong2 *r0 = rlk2_key(C, 0, c, 3), *r1 = rlk2_key(C, 1, c, 3), *r2 = rlk2_key(C, 2, c, 3);
#pragma unroll
        for (int e = 0; e < E; e += 2) {
            const int pos = pos_M4(tid, e);
            const ulonglong2 u = ld2(x0 + pos), v = ld2(x1 + pos), w = ld2(x2 + pos);
            const ulonglong2 k0 = rlk2_w(r0, pos), k1 = rlk2_w(r1, pos), k2 = rlk2_w(r2, pos);
            a[e] = red128s<2>((u128)u.x * k0.x + (u128)v.x * k1.x + (u128)w.x * k2.x, K.pr[2].r64);
            a[e + 1] = red128s<2>((u128)u.y * k0.y + (u128)v.y * k1.y + (u128)w.y * k2.y, K.pr[2].r64);
        }
    }
    inv<2>(a, sm, K.pr[2]);
#pragma unroll
    for (int e = 0; e < E; e++) ys[tid + T * e] = yg[tid + T * e] = a[e]; // y, canonical
    // ---- q2 limb
    {
        const uint64_t *x0 = digit_poly(K, pi, 0, 3), *x1 = digit_poly(K, pi, 1, 3), *x2 = digit_poly(K, pi, 2, 3);
        const ulonglong2 *r0 = rlk2_key(C, 0, c, 2), *r1 = rlk2_key(C, 1, c, 2), *r2 = rlk2_key(C, 2, c, 2);
#pragma unroll
        for (int e = 0; e < E; e += 2) {
            const int pos = pos_M4(tid, e);
            const ulonglong2 u = ld2(x0 + pos), v = ld2(x1 + pos), w = ld2(x2 + pos), dd = ld2(dc + 2 * N + pos);
            const ulonglong2 k0 = rlk2_w(r0, pos), k1 = rlk2_w(r1, pos), k2 = rlk2_w(r2, pos);
            a[e] = reduce_bnd<3>(dd.x + red128s<3>((u128)u.x * k0.x + (u128)v.x * k1.x + (u128)w.x * k2.x, K.pr[3].r64));
            a[e + 1] =
                reduce_bnd<3>(dd.y + red128s<3>((u128)u.y * k0.y + (u128)v.y * k1.y + (u128)w.y * k2.y, K.pr[3].r64));
        }
    }
    inv_f<3>(a, sm, K.pr[3].invf, K.pr[3].ninvf, K.pr[3].ninv_w1f); // U, canonical (FP64 pipe)
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint64_t y = ys[tid + T * e];
        const uint64_t f = y > (QP >> 1) ? 1 : 0;
        rg[tid + T * e] = reduce_bnd<3>(a[e] + f + 4 * Q2 - shoup4<3>(y, C.pinv2)); // R = U - P^-1 y^ (mod q2)
    }
}

__global__ void __launch_bounds__(T, 1) k_relin3b(CmpK C)
{
    extern __shared__ uint64_t sm[];
    const MatchK &K = C.m;
    const int tid = threadIdx.x;
    const int64_t pi = blockIdx.x >> 2;
    const int c = (blockIdx.x >> 1) & 1, l = blockIdx.x & 1; // l = 1: q1 (FP64-pipe transform), 0: q0
    const uint64_t *dc = K.D01 + ((size_t)pi * 6 + c * 3) * N;
    const uint64_t *yg = K.XR + ((size_t)pi * 2 + c) * N, *rg = K.XO + ((size_t)pi * 2 + c) * N;
    const uint64_t q = l ? Q1 : Q0;
    uint64_t a[E];
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint64_t y = yg[tid + T * e], R = rg[tid + T * e]; // written by the same thread index in C2a
        const uint64_t f = y > (QP >> 1) ? 1 : 0;
        const uint64_t z = R > (Q2 >> 1) ? R + (q - Q2) : R; // z^ mod q_l
        if (l) a[e] = reduce_bnd<1>(shoup4<1>(y, K.pinv[1]) + (f ? Q1 - 1 : 0) + z);
        else a[e] = shoup4<0>(y, K.pinv[0]) + (f ? Q0 - 1 : 0) + z; // < 6 q0
    }
    if (l) fwd_f<1>(a, sm, K.pr[1].fwdf); // canonical
    else fwd<0, false>(a, sm, K.pr[0]);  // [0, 2 q0)
    const uint64_t *x0 = digit_poly(K, pi, 0, l), *x1 = digit_poly(K, pi, 1, l), *x2 = digit_poly(K, pi, 2, l);
    const ulonglong2 *r0 = rlk2_key(C, 0, c, l), *r1 = rlk2_key(C, 1, c, l), *r2 = rlk2_key(C, 2, c, l);
    uint64_t *co = K.XC + ((size_t)pi * 2 + c) * 2 * N + (size_t)l * N;
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int pos = pos_M4(tid, e);
        const ulonglong2 u = ld2(x0 + pos), v = ld2(x1 + pos), w = ld2(x2 + pos), dd = ld2(dc + (size_t)l * N + pos);
        const ulonglong2 k0 = rlk2_w(r0, pos), k1 = rlk2_w(r1, pos), k2 = rlk2_w(r2, pos);
        const u128 sa = (u128)u.x * k0.x + (u128)v.x * k1.x + (u128)w.x * k2.x;
        const u128 sb = (u128)u.y * k0.y + (u128)v.y * k1.y + (u128)w.y * k2.y;
        if (l) {
            const uint64_t va = dd.x + red128s<1>(sa, K.pr[1].r64) + Q1 - a[e];
            const uint64_t vb = dd.y + red128s<1>(sb, K.pr[1].r64) + Q1 - a[e + 1];
            st2(co + pos, reduce_bnd<1>(shoup4<1>(va, C.q2inv[1])), reduce_bnd<1>(shoup4<1>(vb, C.q2inv[1])));
        } else {
            const uint64_t va = dd.x + red128s<0>(sa, K.pr[0].r64) + 2 * Q0 - a[e];
            const uint64_t vb = dd.y + red128s<0>(sb, K.pr[0].r64) + 2 * Q0 - a[e + 1];
            st2(co + pos, reduce_bnd<0>(shoup4<0>(va, C.q2inv[0])), reduce_bnd<0>(shoup4<0>(vb, C.q2inv[0])));
        }
    }
}

// C3: Res_q1(Mul(P)(C, M)) per (pair, c): y = INTT_q1(c[q1] M[q1]); out = c[q0] M'[q0] - NTT_q0(q1^-1 y^)
__global__ void __launch_bounds__(T, 1) k_cmp_mask(CmpK C)
{
    extern __shared__ uint64_t sm[];
    const MatchK &K = C.m;
    const int tid = threadIdx.x;
    const int64_t pi = blockIdx.x >> 1;
    const int c = blockIdx.x & 1;
    const uint64_t *ci = K.XC + ((size_t)pi * 2 + c) * 2 * N;
    uint64_t a[E];
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int pos = pos_M4(tid, e);
        const ulonglong2 v = ld2(ci + N + pos);
        ulonglong2 ma, mb;
        ldkey2(C.mask + N, pos, ma, mb);
        a[e] = reduce_bnd<1>(shoup4<1>(v.x, ma));
        a[e + 1] = reduce_bnd<1>(shoup4<1>(v.y, mb));
    }
    inv_f<1>(a, sm, K.pr[1].invf, K.pr[1].ninvf, K.pr[1].ninv_w1f); // y, canonical
#pragma unroll
    for (int e = 0; e < E; e++) a[e] = shoup4<0>(a[e], K.q1inv) + (a[e] > (Q1 >> 1) ? Q0 - 1 : 0); // < 5 q0
    fwd<0>(a, sm, K.pr[0]); // canonical
    uint64_t *co = K.XR + ((size_t)pi * 2 + c) * N;
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int pos = pos_M4(tid, e);
        const ulonglong2 v = ld2(ci + pos);
        ulonglong2 ma, mb;
        ldkey2(C.mask, pos, ma, mb);
        st2(co + pos, reduce_bnd<0>(shoup4<0>(v.x, ma) + Q0 - a[e]), reduce_bnd<0>(shoup4<0>(v.y, mb) + Q0 - a[e + 1]));
    }
}

// C4: right rotation by u = t mod s of the level-0 ciphertext XR (left rotation by S - u with key gkc[u-1]),
// straight to the coefficient domain:  out_0 = INTT_q0(sigma(c0) + sigma(c1) P^-1 gk[0][q0]) - P^-1 y^0,
// out_1 = INTT_q0(sigma(c1) P^-1 gk[1][q0]) - P^-1 y^1;  u = 0: out_c = INTT_q0(c_c).
__global__ void __launch_bounds__(T, 1) k_cmp_rot(CmpK C)
{
    extern __shared__ uint64_t sm[];
    uint64_t *XB = sm, *S0 = sm + SMEM_WORDS, *S1 = sm + 2 * SMEM_WORDS;
    const MatchK &K = C.m;
    const int tid = threadIdx.x;
    const int64_t pi = blockIdx.x;
    const int u = (int)((K.t0 + pi % K.ct) % C.s);
    const uint64_t *ci = K.XR + (size_t)pi * 2 * N;
    uint64_t *co = K.XO + (size_t)pi * 2 * N;
    uint64_t a[E];
    if (u == 0) {
#pragma unroll 1
        for (int c = 0; c < 2; c++) {
            load_eval(a, ci + (size_t)c * N);
            inv<0>(a, XB, K.pr[0]);
            store_coef(co + (size_t)c * N, a);
        }
        return;
    }
    const uint32_t g = (uint32_t)pow5_mod2n(SLOTS - u);
    const ulonglong2 *gk = C.gkc + (size_t)(u - 1) * 4 * N; // [c][q0 | P][N]
    uint64_t *ks1 = C.scr + (size_t)pi * 2 * N, *tsc = ks1 + N;
    const int nt = nat_tid(tid);
    stage_nat(S0, ci); // natural order: conflict-free gathers (ntt3.cuh nat_at)
    stage_nat(S1, ci + N);
    BM_SYNCTHREADS();
#pragma unroll
    for (int e = 0; e < E; e++) a[e] = S1[nat_auto(nt, e, g)];
    inv<0>(a, XB, K.pr[0]);
    fwd<2, false>(a, XB, K.pr[2]); // lazy [0, 2P): Shoup operand only
#pragma unroll
    for (int e = 0; e < E; e += 2) {
        const int pos = pos_M4(tid, e);
        ulonglong2 w0, w0b, w1, w1b;
        ldkey2(gk + N, pos, w0, w0b);
        ldkey2(gk + 3 * N, pos, w1, w1b);
        st2(ks1 + pos, shoup4<2>(a[e], w1), shoup4<2>(a[e + 1], w1b));
        a[e] = shoup4<2>(a[e], w0);
        a[e + 1] = shoup4<2>(a[e + 1], w0b);
    }
#pragma unroll 1
    for (int c = 0; c < 2; c++) {
        if (c == 1) { // written by this thread above: coherent loads
#pragma unroll
            for (int e = 0; e < E; e += 2) {
                const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(ks1 + pos_M4(tid, e));
                a[e] = v.x;
                a[e + 1] = v.y;
            }
        }
        inv<2>(a, XB, K.pr[2]);
#pragma unroll
        for (int e = 0; e < E; e++) tsc[j_M1(tid, e)] = shoup4<0>(a[e], K.pinv[0]) + (a[e] > (QP >> 1) ? Q0 - 1 : 0);
        const ulonglong2 *gq = gk + (size_t)(2 * c) * N;
#pragma unroll
        for (int e = 0; e < E; e++) {
            const int jp = nat_auto(nt, e, g);
            uint64_t v = shoup4<0>(S1[jp], ldkey1(gq, pos_M4(tid, e))); // [0, 4 q0)
            if (c == 0) v += S0[jp];
            a[e] = reduce_bnd<0>(v);
        }
        inv<0>(a, XB, K.pr[0]);
        uint64_t *o = co + (size_t)c * N;
#pragma unroll
        for (int e = 0; e < E; e++) {
            const int j = j_M1(tid, e);
            o[j] = submod_d(a[e], reduce_bnd<0>(tsc[j]), Q0);
        }
    }
}

// C5: d_out[query][group] += sum of its rotated results in this chunk (coefficient domain, canonical)
__global__ void __launch_bounds__(256) k_cmp_add(CmpK C, uint64_t *out, int64_t n_groups, int64_t g0, int64_t ng)
{
    const MatchK &K = C.m;
    const int slice = blockIdx.x % (N / 256);
    int64_t b = blockIdx.x / (N / 256);
    const int c = (int)(b & 1);
    b >>= 1;
    const int64_t g = g0 + b % ng, a = b / ng;
    const int k = slice * 256 + threadIdx.x;
    const int64_t tlo = g * C.s > K.t0 ? g * C.s : K.t0;
    const int64_t thi = (g + 1) * C.s < K.t0 + K.ct ? (g + 1) * C.s : K.t0 + K.ct;
    uint64_t *dst = out + (((size_t)(K.jq0 + a) * n_groups + g) * 2 + c) * N + k;
    uint64_t acc = *dst;
    for (int64_t t = tlo; t < thi; t++) acc = csub(acc + K.XO[(((size_t)a * K.ct + (t - K.t0)) * 2 + c) * N + k], Q0);
    *dst = acc;
}
