// pair_kernels.cuh -- RECORD OF A DROPPED EXPERIMENT, not compiled into the library:
// K2 / K3 as one CTA per (query, set) pair with paired transforms (tools/ntt_experiments.cuh).  Bit-exact
// against the two-CTA kernels (tested while it lived in k_match.cuh), but slower on configs[1]:
// digits 3.18 -> 3.40 ms, relin 5.80 -> 9.04 ms (profiles/r02_ab_pair_kernels.txt).
// ================================================================== K2 / K3 as pair kernels (two transforms at a time)
// One CTA per (query, set) pair runs the work of K2's two CTAs (or K3's two), with the independent
// transforms paired: an integer-prime transform interleaved stage by stage with a q1 transform on the
// FP64 pipe (ntt3f.cuh fwd_h / inv_h), or two integer transforms sharing twiddle loads and exchange
// barriers (ntt3.cuh fwd2x / inv2x).  Two exchange buffers; the values a phase parks for later live in
// tensor memory.  Same residues as k_digits / k_relin (the arithmetic is the same, only interleaved).
constexpr size_t PAIR_SMEM_BYTES = 2 * SMEM_WORDS * sizeof(uint64_t);

// K2h: x0 = INTT_q0(d2[q0]) || x1 = INTT_q1(d2[q1]);  NTT_q0(x1) || NTT_q1(x0 mod q1);  NTT_P(x0) || NTT_P(x1)
__global__ void __launch_bounds__(T, 1) k_digits_h(MatchK K)
{
    extern __shared__ uint64_t sm[];
    uint64_t *XA = sm, *XB = sm + SMEM_WORDS;
    const int64_t pi = blockIdx.x;
    __shared__ uint32_t s_tmem;
    const uint32_t tx = tmem_alloc<256>(&s_tmem); // x0 at +0, x1 at +32 columns
    uint64_t a[E], b[E];
    load_eval(a, K.D2 + ((size_t)pi * 2 + 0) * N);
    load_eval(b, K.D2 + ((size_t)pi * 2 + 1) * N);
    inv_h<0, 1>(a, b, XA, XB, K.pr[0], K.pr[1].invf, K.pr[1].ninvf, K.pr[1].ninv_w1f); // x0, x1 canonical
    tmem_st16(tx, a);
    tmem_st16(tx + 32, b);
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint64_t x0 = a[e];
        a[e] = b[e];                  // x1 (< q1 < q0) -> q0
        b[e] = reduce_bnd<1>(x0);     // x0 mod q1
    }
    fwd_h<0, false, 1>(a, b, XA, XB, K.pr[0], K.pr[1].fwdf);
    uint64_t *xu = K.XU + (size_t)pi * 4 * N;
    store_eval(xu + 2 * N, a); // x1~[q0] (lazy [0, 2 q0): a Shoup operand only)
    store_eval(xu + 0 * N, b); // x0~[q1]
    tmem_ld16(tx, a);
    tmem_ld16(tx + 32, b);
    fwd2x<2, false>(a, b, XA, XB, K.pr[2]);
    store_eval(xu + 1 * N, a); // x0~[P]
    store_eval(xu + 3 * N, b); // x1~[P]
    tmem_free<256>(s_tmem);
}

// K3h, both components of a pair: per component c, INTT_P(KS_c[P]) || INTT_q1(d_c[q1] + P^-1 KS_c[q1])
// (hybrid), the rescale terms, parked; then NTT_q0 of both at once, and the q0-limb outputs (k_relin's
// arithmetic, R22).
__global__ void __launch_bounds__(T, 1) k_relin_h(MatchK K, CtBuf dst, int accumulate)
{
    extern __shared__ uint64_t sm[];
    uint64_t *XA = sm, *XB = sm + SMEM_WORDS;
    const int tid = threadIdx.x;
    const int64_t pi = blockIdx.x;
    __shared__ uint32_t s_tmem;
    const uint32_t tt = tmem_alloc<256>(&s_tmem); // component 0's rescale term at +0
    const uint64_t *xu = K.XU + (size_t)pi * 4 * N;
    const uint64_t *d2 = K.D2 + (size_t)pi * 2 * N;
    const ulonglong2 pinv0 = K.pinv[0], pinv1 = K.pinv[1];
    uint64_t a[E], b[E];
#pragma unroll 1
    for (int c = 0; c < 2; c++) {
        const uint64_t *r0 = K.rlk + (size_t)(0 * 2 + c) * 3 * 2 * N, *r1 = K.rlk + (size_t)(1 * 2 + c) * 3 * 2 * N;
        const uint64_t *dc = K.D01 + ((size_t)pi * 4 + c * 2) * N;
#pragma unroll
        for (int e = 0; e < E; e += 2) {
            const int j = pos_M4(tid, e);
            const ulonglong2 u = ld2(xu + 1 * N + j), v = ld2(xu + 3 * N + j);
            const ulonglong2 w0 = ld2(r0 + 2 * 2 * N + j), w1 = ld2(r1 + 2 * 2 * N + j);
            a[e] = red128s<2>(dot2(u.x, w0.x, v.x, w1.x), K.pr[2].r64);
            a[e + 1] = red128s<2>(dot2(u.y, w0.y, v.y, w1.y), K.pr[2].r64);
            const ulonglong2 u1 = ld2(xu + 0 * N + j), v1 = ld2(d2 + 1 * N + j), dd = ld2(dc + 1 * N + j);
            const ulonglong2 k0 = ld2(r0 + 1 * 2 * N + j), k1 = ld2(r1 + 1 * 2 * N + j);
            b[e] = reduce_bnd<1>(dd.x + red128s<1>(dot2(u1.x, k0.x, v1.x, k1.x), K.pr[1].r64));
            b[e + 1] = reduce_bnd<1>(dd.y + red128s<1>(dot2(u1.y, k0.y, v1.y, k1.y), K.pr[1].r64));
        }
        inv_h<2, 1>(a, b, XA, XB, K.pr[2], K.pr[1].invf, K.pr[1].ninvf, K.pr[1].ninv_w1f); // Y, U canonical
#pragma unroll
        for (int e = 0; e < E; e++) {
            const uint64_t y = a[e];
            const uint64_t f = y > (QP >> 1) ? 1 : 0;
            const uint64_t R = reduce_bnd<1>(b[e] + f + 4 * Q1 - shoup4<1>(y, pinv1)); // U - P^-1 y^
            const uint64_t z = R > (Q1 >> 1) ? R + (Q0 - Q1) : R;                      // centred, in q0
            a[e] = shoup4<0>(y, pinv0) + z + (f ? Q0 - 1 : 0);                         // < 6 q0
        }
        if (c == 0) tmem_st16(tt, a);
    }
    tmem_ld16(tt, b); // b = component 0's term, a = component 1's
    fwd2x<0, false>(b, a, XA, XB, K.pr[0]);
    const ulonglong2 q1inv = K.q1inv;
#pragma unroll 1
    for (int c = 0; c < 2; c++) {
        const uint64_t *r0 = K.rlk + (size_t)(0 * 2 + c) * 3 * 2 * N, *r1 = K.rlk + (size_t)(1 * 2 + c) * 3 * 2 * N;
        const uint64_t *dc = K.D01 + ((size_t)pi * 4 + c * 2) * N;
        uint64_t *co = dst.at(pi, c);
        const uint64_t *A = c ? a : b;
#pragma unroll
        for (int e = 0; e < E; e += 2) {
            const int j = pos_M4(tid, e);
            const ulonglong2 u = ld2(d2 + 0 * N + j), v = ld2(xu + 2 * N + j), dd = ld2(dc + j);
            const ulonglong2 w0 = ld2(r0 + j), w1 = ld2(r1 + j);
            const uint64_t ka = red128s<0>(dot2(u.x, w0.x, v.x, w1.x), K.pr[0].r64);
            const uint64_t kb = red128s<0>(dot2(u.y, w0.y, v.y, w1.y), K.pr[0].r64);
            uint64_t oa = reduce_bnd<0>(shoup4<0>(dd.x + ka + 2 * Q0 - A[e], q1inv));
            uint64_t ob = reduce_bnd<0>(shoup4<0>(dd.y + kb + 2 * Q0 - A[e + 1], q1inv));
            if (accumulate) {
                const ulonglong2 cc = *reinterpret_cast<const ulonglong2 *>(co + j);
                oa = csub(oa + cc.x, Q0);
                ob = csub(ob + cc.y, Q0);
            }
            st2(co + j, oa, ob);
        }
    }
    tmem_free<256>(s_tmem);
}

