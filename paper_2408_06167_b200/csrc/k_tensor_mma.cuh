// k_tensor_mma.cuh -- K1 (a4, the tensor + part sum) on the 5th-generation tensor
// cores: tcgen05.mma kind::i8 (u8 x u8 -> s32, exact), accumulators in TMEM.
//
// For one coefficient c and one limb q_l the tensor is a contraction over the parts:
//   d0[q][s] = sum_i x0_i y0_i,  d2 = sum_i x1_i y1_i,  d1 = sum_i (x0_i y1_i + x1_i y0_i)     (mod q_l)
// with x the query's and y the template set's NTT-domain residues.  Splitting each set residue into
// its bytes, y = sum_v y_v 2^(8v), and premultiplying the query residue, X_v = 2^(8v) x mod q_l, gives
//   sum_i x_i y_i == sum_u 2^(8u) sum_{i,v} y_{i,v} byte_u(X_{i,v})          (mod q_l)
// i.e. a u8 GEMM per coefficient: A = set bytes [sets x (i, v)] (the DB as stored: the bytes of a
// u64 residue ARE its y_v), B = query bytes [(i, v) x (q, u)], and 8 s32 columns (u) per query that
// the epilogue folds as sum_u 2^(8u) out_u (< 2^79) and reduces mod q_l.  Every partial sum is an exact
// integer (at most 16 p products of two bytes < 2^23 for p <= 8), so d0, d1, d2 are the same canonical
// residues the CUDA-core K1 (k_tensor) produces -- the GPU parity tests compare them end to end.
//
// Tile: 128 sets (MMA M = TMEM lanes) x 8 queries (MMA N = 64 = 8 queries x 8 bytes) x one limb x a
// block of TM_CB coefficients, TM_CG = 4 per iteration.  The set operand comes from the DB packed once
// into this layout (k_tm_dbpack, bm_db_tc_register: one contiguous 128 x 16 p-byte block per tile, limb
// and coefficient), the query operand from k_tm_qexp; both stream into shared memory by cp.async one
// iteration ahead.  Per coefficient: 8 MMAs of K = 32 bytes for p = 8 (d0: 2, d2: 2, d1: 4) into one of
// two TMEM accumulator sets of 192 columns (the MMAs of one overlap the epilogue of the other); each
// thread then stores 32 bytes (4 coefficients) per (pair, output) into D01 / D2 (dofs piece layout).
// Shared-memory operands are in the canonical K-major SWIZZLE_NONE layout: 8-row x 16-byte core
// matrices, LBO = the next core matrix along K, SBO = the next 8-row group (tools/probe/umma_i8_probe.cu
// checked this encoding bit for bit on the B200).
#pragma once
#include "k_match.cuh"

namespace bm {

constexpr int TM_M = 128;        // sets per tile (MMA M)
constexpr int TM_Q = 8;          // queries per tile
constexpr int TM_N = TM_Q * 8;   // MMA N: (query, byte u)
#ifndef BM_TM_CB
#define BM_TM_CB 64
#endif
constexpr int TM_CB = BM_TM_CB;  // coefficients per CTA

// bytes of the expanded query operand per (limb, query tile, coefficient): [comp][g 8][kc P/2][8][16]
BM_HD constexpr size_t tm_b_bytes(int P) { return (size_t)1024 * P; }

// constants: X_v = 2^(8v) x mod q_l (Shoup pairs), and 2^40 mod q0 for the q0 epilogue fold
struct TmConst {
    ulonglong2 w[2][8];
    ulonglong2 c40;
};

// ---------------------------------------------------------------- the query operand (B)
// one thread per (limb l, query tile qt, coefficient c, comp, query g of the tile, core column kc):
// the core matrix (g, kc) of comp-block comp = 8 rows u of 16 bytes: byte u of X_v(x_{2kc}) (v = 0..7),
// then of X_v(x_{2kc+1}).  Queries past the chunk's cq are zero rows.
template <int P> __global__ void __launch_bounds__(256) k_tm_qexp(MatchK K, uint8_t *XB, int n_qt, TmConst tc)
{
    int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
    const int kc = (int)(t % (P / 2));
    t /= P / 2;
    const int g = (int)(t % 8);
    t /= 8;
    const int comp = (int)(t % 2);
    t /= 2;
    const int c = (int)(t % N);
    t /= N;
    const int qt = (int)(t % n_qt);
    const int l = (int)(t / n_qt);
    if (l >= 2) return;
    const int q = qt * TM_Q + g;
    uint4 *dst = reinterpret_cast<uint4 *>(XB + ((size_t)(l * n_qt + qt) * N + c) * tm_b_bytes(P) +
                                           (size_t)comp * 512 * P + (size_t)(g * (P / 2) + kc) * 128);
    if (q >= K.cq) {
#pragma unroll
        for (int u = 0; u < 8; u++) dst[u] = make_uint4(0, 0, 0, 0);
        return;
    }
    uint64_t X[16];
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int i = 2 * kc + h;
        const uint64_t x = K.qry[((((size_t)(K.jq0 + q) * K.p + i) * 2 + comp) * 2 + l) * N + c];
#pragma unroll
        for (int v = 0; v < 8; v++)
            X[8 * h + v] = l == 0 ? reduce_bnd<0>(shoup4<0>(x, tc.w[0][v])) : reduce_bnd<1>(shoup4<1>(x, tc.w[1][v]));
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
        uint32_t wd[4];
#pragma unroll
        for (int w4 = 0; w4 < 4; w4++) {
            uint32_t a = 0;
#pragma unroll
            for (int b = 0; b < 4; b++) a |= ((uint32_t)(X[4 * w4 + b] >> (8 * u)) & 0xFFu) << (8 * b);
            wd[w4] = a;
        }
        dst[u] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    }
}

// ---------------------------------------------------------------- tcgen05 helpers
BM_D uint64_t tm_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46); // version 1, SWIZZLE_NONE
}
// u8 x u8 -> s32, M = 128, N = 64, both operands K-major
constexpr uint32_t TM_IDESC = (2u << 4) | ((uint32_t)(TM_N >> 3) << 17) | ((uint32_t)(TM_M >> 4) << 24);
BM_D void tm_mma(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t acc)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                 "l"(ad), "l"(bd), "r"(TM_IDESC), "r"(acc));
}
BM_D void tm_commit(uint64_t *mbar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(mbar))
                 : "memory");
}
BM_D void tm_wait(uint64_t *mbar, uint32_t phase)
{
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done)
                     : "r"((uint32_t)__cvta_generic_to_shared(mbar)), "r"(phase)
                     : "memory");
    }
}
BM_D void tm_ld32(uint32_t taddr, uint32_t r[32])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                 "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
                 "[%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                   "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                   "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                   "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                   "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
                 :
                 : "memory");
}

// ---------------------------------------------------------------- the DB in the tensor-core layout
// The set operand (A) of every coefficient as one contiguous 128-set x 16 p-byte block in the canonical
// K-major layout: packed[((st * 2 + l) * N + c) * 2048 p + (grp * p + kc) * 128 + r * 16 + b], set
// 128 st + 8 grp + r, K byte 16 kc + b = (comp, part i, byte v) with kc = comp p / 2 + i / 2.  Sets past
// n_sets are zero.  One thread per (st, l, grp, kc, c), c fastest: the DB reads are coalesced along
// the coefficients, every thread writes one 128-byte core matrix.
BM_HD constexpr size_t tm_a_bytes(int P) { return (size_t)TM_M * 16 * P; }
template <int P> __global__ void __launch_bounds__(256) k_tm_dbpack(const uint64_t *db, int64_t n_sets, int64_t n_st,
                                                                    uint8_t *packed)
{
    int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
    const int c = (int)(t % N);
    t /= N;
    const int kc = (int)(t % P);
    t /= P;
    const int grp = (int)(t % 16);
    t /= 16;
    const int l = (int)(t % 2);
    const int64_t st = t / 2;
    if (st >= n_st) return;
    const int comp = kc / (P / 2), i0 = 2 * (kc % (P / 2));
    uint4 *dst = reinterpret_cast<uint4 *>(packed + ((size_t)(st * 2 + l) * N + c) * tm_a_bytes(P) + (size_t)(grp * P + kc) * 128);
#pragma unroll
    for (int r = 0; r < 8; r++) {
        const int64_t set = st * TM_M + 8 * grp + r;
        uint64_t x = 0, y = 0;
        if (set < n_sets) {
            x = db[((((size_t)set * P + i0) * 2 + comp) * 2 + l) * N + c];
            y = db[((((size_t)set * P + i0 + 1) * 2 + comp) * 2 + l) * N + c];
        }
        dst[r] = make_uint4((uint32_t)x, (uint32_t)(x >> 32), (uint32_t)y, (uint32_t)(y >> 32));
    }
}

// ---------------------------------------------------------------- the tensor kernel
BM_D void cp_async16_cg(void *smem, const void *gmem)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem));
}
// one 32-byte store (STG.E.ENL2.256): a whole sector per (pair, output) and iteration
BM_D void tm_st4(uint64_t *p, uint64_t a, uint64_t b, uint64_t c, uint64_t d)
{
#ifdef BM_TM_ST2
    st2(p, a, b);
    st2(p + 2, c, d);
#else
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
#endif
}
BM_D void tm_ld16(uint32_t taddr, uint32_t r[16])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                 "%13, %14, %15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15])
                 : "r"(taddr)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15])
                 :
                 : "memory");
}
constexpr int TM_T = 512;         // 16 warps: warp w reads TMEM lanes 32 (w & 3) .. (sets), queries 2 (w >> 2) + {0, 1}
constexpr int TM_CG = 4;          // coefficients per iteration (a full 32-byte sector per (pair, output) store)
constexpr uint32_t TM_COLS = 512; // two accumulator sets of 192 columns (d0, d2, d1): MMA of one overlaps the
                                  // epilogue of the other
template <int P> constexpr size_t tm_smem_bytes() { return 2 * (size_t)TM_CG * (tm_a_bytes(P) + tm_b_bytes(P)); }

// the MMAs of one coefficient: d0 = A[comp 0] B[comp 0], d2 = A[1] B[1], d1 = A[0] B[1] + A[1] B[0]
template <int P> BM_D void tm_mma_coef(uint32_t acc, const uint8_t *sa, const uint8_t *sb)
{
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sa), b0 = (uint32_t)__cvta_generic_to_shared(sb);
    const uint32_t b1 = b0 + 512 * P; // comp-block 1
    constexpr uint32_t ALBO = 128, ASBO = 128 * P, BLBO = 128, BSBO = 64 * P;
#pragma unroll
    for (int kk = 0; kk < P / 4; kk++) {
        const uint32_t ak0 = a0 + kk * 256, ak1 = a0 + (P / 2) * 128 + kk * 256;
        tm_mma(acc + 0, tm_sdesc(ak0, ALBO, ASBO), tm_sdesc(b0 + kk * 256, BLBO, BSBO), kk);   // d0
        tm_mma(acc + 64, tm_sdesc(ak1, ALBO, ASBO), tm_sdesc(b1 + kk * 256, BLBO, BSBO), kk);  // d2
        tm_mma(acc + 128, tm_sdesc(ak0, ALBO, ASBO), tm_sdesc(b1 + kk * 256, BLBO, BSBO), kk); // d1
    }
#pragma unroll
    for (int kk = 0; kk < P / 4; kk++)
        tm_mma(acc + 128, tm_sdesc(a0 + (P / 2) * 128 + kk * 256, ALBO, ASBO), tm_sdesc(b0 + kk * 256, BLBO, BSBO), 1);
}

// one accumulator set -> this thread's 6 residues (outputs d0, d2, d1 of its set and 2 queries); the three
// TMEM loads are issued back to back and waited for once
#define TM_R16(b) "=r"(r[b + 0]), "=r"(r[b + 1]), "=r"(r[b + 2]), "=r"(r[b + 3]), "=r"(r[b + 4]), "=r"(r[b + 5]), \
    "=r"(r[b + 6]), "=r"(r[b + 7]), "=r"(r[b + 8]), "=r"(r[b + 9]), "=r"(r[b + 10]), "=r"(r[b + 11]),          \
    "=r"(r[b + 12]), "=r"(r[b + 13]), "=r"(r[b + 14]), "=r"(r[b + 15])
#define TM_W16(b) "+r"(r[b + 0]), "+r"(r[b + 1]), "+r"(r[b + 2]), "+r"(r[b + 3]), "+r"(r[b + 4]), "+r"(r[b + 5]), \
    "+r"(r[b + 6]), "+r"(r[b + 7]), "+r"(r[b + 8]), "+r"(r[b + 9]), "+r"(r[b + 10]), "+r"(r[b + 11]),          \
    "+r"(r[b + 12]), "+r"(r[b + 13]), "+r"(r[b + 14]), "+r"(r[b + 15])
#define TM_LD16_ASM "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
template <int L> BM_D void tm_epilogue(uint32_t t_ep, const TmConst &tc, uint64_t val[6])
{
    uint32_t r[48];
    asm volatile(TM_LD16_ASM : TM_R16(0) : "r"(t_ep) : "memory");
    asm volatile(TM_LD16_ASM : TM_R16(16) : "r"(t_ep + 64) : "memory");
    asm volatile(TM_LD16_ASM : TM_R16(32) : "r"(t_ep + 128) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" : TM_W16(0), TM_W16(16), TM_W16(32) : : "memory");
#pragma unroll
    for (int o = 0; o < 3; o++) {
#pragma unroll
        for (int j = 0; j < 2; j++) {
            const uint32_t *v = r + 16 * o + 8 * j;
            const uint64_t lo = (uint64_t)v[0] + ((uint64_t)v[1] << 8) + ((uint64_t)v[2] << 16) + ((uint64_t)v[3] << 24) +
                                ((uint64_t)v[4] << 32); // < 2^56
            if (L == 0) {
                const uint64_t hi = (uint64_t)v[5] + ((uint64_t)v[6] << 8) + ((uint64_t)v[7] << 16); // < 2^40
                val[2 * o + j] = reduce_bnd<0>(shoup4<0>(hi, tc.c40) + lo);                        // < 4 q0 + 2^56
            } else {
                val[2 * o + j] = reduce_bnd<1>(lo); // X_v < q1 < 2^40: bytes 5..7 of the query operand are 0
            }
        }
    }
}

// grid: ((cb * n_st + st) * n_qt + qt) * 2 + l, st counted from the chunk's first set tile (K.t0 / 128).
// Per iteration TM_CG = 4 coefficients: their operands (contiguous blocks of the packed DB and of the
// expanded queries) arrive by cp.async one iteration ahead; the MMAs of coefficients 0, 1 go to the two
// accumulator sets, 2 and 3 follow as soon as the epilogue has drained a set; every thread then writes
// 32 bytes (4 coefficients) per (pair, output).
template <int P, int L> BM_D void tm_tile(const MatchK &K, const uint8_t *DBP, const uint8_t *XB, int n_qt, int qt, int st,
                                          int c_lo, const TmConst &tc, uint8_t *tsm, uint64_t *mbar, uint32_t tmem)
{
    constexpr int A_BYTES = (int)tm_a_bytes(P), B_BYTES = (int)tm_b_bytes(P);
    constexpr int STAGE = TM_CG * (A_BYTES + B_BYTES); // A_c .. A_c+3, then B_c .. B_c+3
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint8_t *ag = DBP + ((size_t)((K.t0 / TM_M + st) * 2 + L) * N) * A_BYTES;
    const uint8_t *bg = XB + ((size_t)L * n_qt + qt) * N * B_BYTES;
    auto load = [&](int c, int buf) {
        uint8_t *sb = tsm + buf * STAGE;
#pragma unroll
        for (int k = 0; k < TM_CG * A_BYTES / 16 / TM_T; k++)
            cp_async16_cg(sb + 16 * (k * TM_T + tid), ag + (size_t)c * A_BYTES + 16 * (k * TM_T + tid));
#pragma unroll
        for (int k = 0; k < TM_CG * B_BYTES / 16 / TM_T; k++)
            cp_async16_cg(sb + TM_CG * A_BYTES + 16 * (k * TM_T + tid), bg + (size_t)c * B_BYTES + 16 * (k * TM_T + tid));
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int s_ep = 32 * (warp & 3) + lane, g = warp >> 2;
    const int64_t set_ep = (int64_t)st * TM_M + s_ep;
    const uint32_t t_ep = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 16 * g;
    // outputs of this thread: pairs (query 8 qt + 2 g + j, set), d0, d2, d1 at D01 poly L, D2 poly L,
    // D01 poly 2 + L (dofs: the 4 coefficients of an iteration are one 32-byte piece, and the warp's 32
    // consecutive sets write 32 adjacent pieces)
    int64_t pij[2];
    bool ok[2];
#pragma unroll
    for (int j = 0; j < 2; j++) {
        const int64_t q = (int64_t)qt * TM_Q + 2 * g + j;
        ok[j] = q < K.cq && set_ep < K.ct;
        pij[j] = ok[j] ? q * K.ct + set_ep : 0;
    }
    uint32_t ph0 = 0, ph1 = 0;
    load(c_lo, 0);
#pragma unroll 1
    for (int c = c_lo, buf = 0; c < c_lo + TM_CB; c += TM_CG, buf ^= 1) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        BM_SYNCTHREADS(); // operands in shared memory; the previous iteration's TMEM reads are done
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint8_t *sa = tsm + buf * STAGE, *sb = sa + TM_CG * A_BYTES;
        if (tid == 0) {
            tm_mma_coef<P>(tmem, sa, sb);
            tm_commit(mbar + 0);
            tm_mma_coef<P>(tmem + 256, sa + A_BYTES, sb + B_BYTES);
            tm_commit(mbar + 1);
        }
        if (c + TM_CG < c_lo + TM_CB) load(c + TM_CG, buf ^ 1); // the other buffer: its MMAs completed
        uint64_t val[TM_CG][6];
#pragma unroll
        for (int k = 0; k < TM_CG; k++) {
            const int a = k & 1;
            tm_wait(mbar + a, a ? ph1 : ph0);
            if (a) ph1 ^= 1; else ph0 ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            tm_epilogue<L>(t_ep + 256 * a, tc, val[k]);
            if (k + 2 < TM_CG) {
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                BM_SYNCTHREADS(); // accumulator set a drained
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (tid == 0) {
                    tm_mma_coef<P>(tmem + 256 * a, sa + (k + 2) * A_BYTES, sb + (k + 2) * B_BYTES);
                    tm_commit(mbar + a);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < 3; o++)
#pragma unroll
            for (int j = 0; j < 2; j++)
                if (ok[j]) {
                    uint64_t *d = (o == 1 ? K.D2 : K.D01) + dofs(K, o == 2 ? 2 + L : L, pij[j], c);
                    tm_st4(d, val[0][2 * o + j], val[1][2 * o + j], val[2][2 * o + j], val[3][2 * o + j]);
                }
    }
}

template <int P> __global__ void __launch_bounds__(TM_T, 1) k_tensor_mma(MatchK K, const uint8_t *DBP, const uint8_t *XB,
                                                                      int n_qt, int n_st, TmConst tc)
{
    static_assert(P == 4 || P == 8, "k_tensor_mma: p = 4 or 8");
    extern __shared__ __align__(1024) uint8_t tsm[];
    __shared__ __align__(8) uint64_t mbar[2];
    __shared__ uint32_t s_tmem;
    const int tid = threadIdx.x, warp = tid >> 5;
    int64_t b = blockIdx.x;
    const int l = (int)(b & 1);
    b >>= 1;
    const int qt = (int)(b % n_qt);
    b /= n_qt;
    const int st = (int)(b % n_st);
    const int cb = (int)(b / n_st);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&s_tmem)),
                     "n"(TM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(mbar + 0)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(mbar + 1)));
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    BM_SYNCTHREADS();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    if (l == 0) tm_tile<P, 0>(K, DBP, XB, n_qt, qt, st, cb * TM_CB, tc, tsm, mbar, tmem);
    else tm_tile<P, 1>(K, DBP, XB, n_qt, qt, st, cb * TM_CB, tc, tsm, mbar, tmem);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    BM_SYNCTHREADS();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TM_COLS) : "memory");
}

} // namespace bm
