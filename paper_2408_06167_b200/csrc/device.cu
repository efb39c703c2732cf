// device.cu -- the device-facing C ABI of libblindmatch and, through the three headers it
// includes (k_match.cuh, k_next.cuh, k_setup.cuh), its sm_100a kernels.
//
// Hot path (bm_match, HE-C^3) per (query, set) pair, hoisted order
// (reading R8); every transform is one 8192-point NTT held by a 512-thread CTA (ntt3.cuh):
//   K1 k_tensor  (tile of pairs, limb)   a4: d0, d1, d2 = sum_i tensor(C_u,i, C_s,i) (Karatsuba),
//                                        a contraction over the parts tiled through shared memory
//   K2 k_digits  (pair, digit l)         a5: x_l = INTT_{q_l}(d2[q_l]); ModUp: x0 -> NTT_{q1,P},
//                                        x1 -> NTT_{q0,P}  (3 transforms)
//   K3 k_relin   (pair, component c)     a5+a6: KS_c = sum_j x_j rlk_j over {q0,q1,P}; ModDown fused
//                                        with the rescale by q1 (exact, R22):
//                                        INTT_P, INTT_q1, NTT_q0 (3 transforms) -> C_c (level 0)
//   K4 k_ladder_t<false> (pair)          a7+a8: the log2(s) rotate-and-add steps with C resident in
//                                        shared memory and per-thread scratch in TMEM, 6 transforms
//                                        per step, coefficient-domain output
//      k_ladder_t<true> (2-CTA cluster per pair, latency mode: <= n_SM / 2 pairs): rank c runs
//                                        component c, 4 transforms per step on the critical path
//   K5 k_out_intt (pair, c)              a8 when s = 1 (no ladder): INTT_q0 of C
// Also here: K6 k_hrot (f2, the hoisted rotation sum), the f3/f4 kernels (query expansion and
// server-side enrollment: k_exp_mask, k_rot1_digits, k_rot1_ks, k_enroll_add) and the f1 kernels
// (compressed scan one level up: k_tensor<3>, k_digits3, k_relin3a/b, k_cmp_mask, k_cmp_rot,
// k_cmp_add), encryption / conversion / key upload, and the host side of the device C ABI.
// Memory-access conventions: NTT-domain data in the pair-coalesced M4 order,
// twiddles in load order (tw_pos), Shoup keys planar (ldkey2).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <algorithm>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h> // header-only NVTX v3: named ranges for Nsight timelines (no-ops without a tool)

#include "bm_common.cuh"
#include "bm_host.h"
#include "ntt3.cuh"
#include "ntt3f.cuh"
using namespace bm::v3;

using namespace bm;
typedef unsigned __int128 u128;

#include "k_match.cuh"
#include "k_tensor_mma.cuh"
#include "k_next.cuh"
#include "k_setup.cuh"

// ================================================================== host side: device context
namespace {

struct DevCtx {
    int dev = -1;
    ulonglong2 *tw = nullptr;  // [4][2][N]: q0, q1, P, q2 (f3)
    ulonglong2 *twf = nullptr; // [q1, q2][fwd, inv][N], FP64 form
    PrimeK pr[4] = {};
    ulonglong2 pinv[2], q1inv;
    ulonglong2 q1invP;         // q1^-1 P mod q0 (LADDER_PSCALE)
    PrimeK pr0s = {};          // pr[0] with N^-1 P^-1 for N^-1 (LADDER_PSCALE)
    ulonglong2 q2inv[2];       // f3: q2^-1 mod q0, q1
    ulonglong2 pinv2;          // f1: P^-1 mod q2
    uint64_t pmod[2];
    int n_sm = 148;
    double2 *zeta = nullptr;    // [N] exp(i pi k / N) (device decryption's canonical embedding)
    int32_t *slot_t = nullptr;  // [S] (5^j mod 2N - 1) / 2
    int max_cl[4] = {0, 0, 0, 0}; // cudaOccupancyMaxActiveClusters of the cluster ladders (index: cluster size)
    TmConst tmc;                  // k_tensor_mma: 2^(8v) mod q0, q1 and 2^40 mod q0 (Shoup pairs)
    // bm_match_host's extra streams (created once per device, reused by every call under host_mu)
    std::mutex host_mu;
    cudaStream_t hs[3] = {nullptr, nullptr, nullptr}; // second compute stream, upload, download
    std::vector<cudaEvent_t> hev;                      // bm_match_host's events, grown on demand, reused
};

std::mutex g_mu;
std::vector<DevCtx *> g_ctx;

// DBs registered in the tensor-core layout (bm_db_tc_register): bm_match runs K1 on the tensor cores
// for them (k_tensor_mma)
struct TcDb {
    const uint64_t *db;
    int64_t n_sets;
    int32_t p;
    const uint8_t *packed;
};
std::mutex g_tc_mu;
std::vector<TcDb> g_tc;
const uint8_t *tc_lookup(const uint64_t *db, int64_t n_sets, int32_t p)
{
    std::lock_guard<std::mutex> lk(g_tc_mu);
    for (const TcDb &e : g_tc)
        if (e.db == db && e.n_sets == n_sets && e.p == p) return e.packed;
    return nullptr;
}

ulonglong2 shoup_pair(uint64_t w, uint64_t q) { return make_ulonglong2(w, shoup_companion(w, q)); }
uint64_t powmod_d(uint64_t a, uint64_t e, uint64_t q)
{
    uint64_t r = 1;
    a %= q;
    for (; e; e >>= 1, a = mulmod_h(a, a, q))
        if (e & 1) r = mulmod_h(r, a, q);
    return r;
}

const size_t SMEM_BYTES = SMEM_WORDS * sizeof(uint64_t);

template <typename F> void set_smem(F f) { cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES); }

int ctx_get(DevCtx **out)
{
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) {
        cudaGetLastError();
        return BM_ERR_CUDA;
    }
    std::lock_guard<std::mutex> lk(g_mu);
    if ((int)g_ctx.size() <= dev) g_ctx.resize(dev + 1, nullptr);
    if (g_ctx[dev]) {
        *out = g_ctx[dev];
        return BM_OK;
    }
    DevCtx *C = new DevCtx;
    C->dev = dev;
    cudaDeviceGetAttribute(&C->n_sm, cudaDevAttrMultiProcessorCount, dev);
    std::vector<ulonglong2> h(8 * (size_t)N);
    for (int i = 0; i < 4; i++) {
        const HostPrime &H = host_prime(i);
        for (int k = 0; k < N; k++) {
            h[(size_t)(2 * i) * N + tw_pos(k)] = shoup_pair(H.fwd[k], H.q);     // load-order storage
            h[(size_t)(2 * i + 1) * N + tw_pos(k)] = shoup_pair(H.inv[k], H.q);
        }
    }
    if (cudaMalloc(&C->tw, h.size() * sizeof(ulonglong2)) != cudaSuccess) {
        delete C;
        cudaGetLastError();
        return BM_ERR_OOM;
    }
    cudaMemcpy(C->tw, h.data(), h.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice);
    // q1 and q2 twiddles for the FP64-pipe transforms (ntt3f.cuh): (w, fl(w / q)) as double bit patterns
    auto fpair = [](uint64_t w, uint64_t q) {
        const double dw = (double)w, dq = dw / (double)q;
        uint64_t a, b;
        memcpy(&a, &dw, 8);
        memcpy(&b, &dq, 8);
        return make_ulonglong2(a, b);
    };
    {
        const int fp[2] = {1, 3};
        std::vector<ulonglong2> hf(4 * (size_t)N);
        for (int f = 0; f < 2; f++) {
            const HostPrime &H = host_prime(fp[f]);
            for (int k = 0; k < N; k++)
                hf[(size_t)(2 * f) * N + tw_pos(k)] = fpair(H.fwd[k], H.q),
                                       hf[(size_t)(2 * f + 1) * N + tw_pos(k)] = fpair(H.inv[k], H.q);
        }
        if (cudaMalloc(&C->twf, hf.size() * sizeof(ulonglong2)) != cudaSuccess) {
            cudaFree(C->tw);
            delete C;
            cudaGetLastError();
            return BM_ERR_OOM;
        }
        cudaMemcpy(C->twf, hf.data(), hf.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice);
        for (int f = 0; f < 2; f++) {
            const HostPrime &H = host_prime(fp[f]);
            PrimeK &P = C->pr[fp[f]];
            P.fwdf = C->twf + (size_t)(2 * f) * N;
            P.invf = C->twf + (size_t)(2 * f + 1) * N;
            P.ninvf = fpair(H.ninv, H.q);
            P.ninv_w1f = fpair(mulmod_h(H.ninv, H.inv[1], H.q), H.q);
        }
    }
    for (int i = 0; i < 4; i++) {
        const HostPrime &H = host_prime(i);
        PrimeK &P = C->pr[i];
        P.q = H.q;
        P.q2 = 2 * H.q;
        P.fwd = C->tw + (size_t)(2 * i) * N;
        P.inv = C->tw + (size_t)(2 * i + 1) * N;
        P.ninv = shoup_pair(H.ninv, H.q);
        P.ninv_w1 = shoup_pair(mulmod_h(H.ninv, H.inv[1], H.q), H.q);
        uint64_t r64 = (uint64_t)(((u128)1 << 64) % H.q);
        P.r64 = shoup_pair(r64, H.q);
        P.one_p = (uint64_t)((((u128)1) << 64) / H.q);
    }
    for (int l = 0; l < 2; l++) {
        uint64_t q = C->pr[l].q;
        C->pmod[l] = QP % q;
        C->pinv[l] = shoup_pair(powmod_d(QP % q, q - 2, q), q);
    }
    C->q1inv = shoup_pair(powmod_d(Q1 % Q0, Q0 - 2, Q0), Q0);
    {
        const HostPrime &H = host_prime(0);
        const uint64_t pi0 = C->pinv[0].x, nip = mulmod_h(H.ninv, pi0, Q0);
        C->q1invP = shoup_pair(mulmod_h(C->q1inv.x, QP % Q0, Q0), Q0);
        C->pr0s = C->pr[0];
        C->pr0s.ninv = shoup_pair(nip, Q0);
        C->pr0s.ninv_w1 = shoup_pair(mulmod_h(nip, H.inv[1], Q0), Q0);
    }
    for (int v = 0; v < 8; v++) {
        C->tmc.w[0][v] = shoup_pair(powmod_d(2, 8 * v, Q0), Q0);
        C->tmc.w[1][v] = shoup_pair(powmod_d(2, 8 * v, Q1), Q1);
    }
    C->tmc.c40 = shoup_pair(powmod_d(2, 40, Q0), Q0);
    for (int l = 0; l < 2; l++) C->q2inv[l] = shoup_pair(powmod_d(Q2 % C->pr[l].q, C->pr[l].q - 2, C->pr[l].q), C->pr[l].q);
    C->pinv2 = shoup_pair(powmod_d(QP % Q2, Q2 - 2, Q2), Q2);
    cudaMemcpyToSymbol(c_cdt, host_cdt(), sizeof(uint64_t) * 19);
    cudaFuncSetAttribute(k_tensor<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TENSOR_SMEM_BYTES);
    cudaFuncSetAttribute(k_tensor<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TENSOR_SMEM_BYTES);
    cudaFuncSetAttribute(k_tensor<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TENSOR_SMEM_BYTES);
    cudaFuncSetAttribute(k_digits, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K2_SMEM_BYTES);
    cudaFuncSetAttribute(k_tensor_mma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tm_smem_bytes<4>());
    cudaFuncSetAttribute(k_tensor_mma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tm_smem_bytes<8>());
    cudaFuncSetAttribute(k_relin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K3_SMEM_BYTES);
    set_smem(k_out_intt);
    cudaFuncSetAttribute(k_rescale_deg2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K7_SMEM_BYTES);
    cudaFuncSetAttribute(k_ladder_t<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LADDER_SMEM_BYTES);
    cudaFuncSetAttribute(k_ladder_t<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LADDER_SMEM_BYTES);
    cudaFuncSetAttribute(k_ladder_t<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LADDER_SMEM_BYTES);
    cudaFuncSetAttribute(k_ladder_c3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LADDER_SMEM_BYTES);
    cudaFuncSetAttribute(k_hrot<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HROT_SMEM_BYTES);
    cudaFuncSetAttribute(k_hrot<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HROT_SMEM_BYTES);
    set_smem(k_encrypt);
    cudaFuncSetAttribute(k_exp_mask, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)X1_SMEM_BYTES);
    cudaFuncSetAttribute(k_rot1_digits, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)X2_SMEM_BYTES);
    cudaFuncSetAttribute(k_rot1_ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)X3_SMEM_BYTES);
    cudaFuncSetAttribute(k_digits3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C1_SMEM_BYTES);
    cudaFuncSetAttribute(k_relin3a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C2_SMEM_BYTES);
    set_smem(k_relin3b);
    set_smem(k_cmp_mask);
    cudaFuncSetAttribute(k_cmp_rot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C4_SMEM_BYTES);
    set_smem(k_convert);
    set_smem(k_key_ntt);
    cudaFuncSetAttribute(k_decrypt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DEC_SMEM_BYTES);
    {   // device decryption tables: zeta^k = exp(i pi k / N) (long double, rounded once), slot -> FFT index
        std::vector<double2> z(N);
        for (int k = 0; k < N; k++) {
            const long double a = 3.141592653589793238462643383279502884L * k / N;
            z[k] = make_double2((double)cosl(a), (double)sinl(a));
        }
        std::vector<int32_t> t(SLOTS);
        uint64_t x = 1;
        for (int j = 0; j < SLOTS; j++, x = x * 5 % (2 * N)) t[j] = (int32_t)((x - 1) / 2);
        if (cudaMalloc(&C->zeta, N * sizeof(double2)) != cudaSuccess ||
            cudaMalloc(&C->slot_t, SLOTS * sizeof(int32_t)) != cudaSuccess) {
            cudaGetLastError();
            return BM_ERR_OOM;
        }
        cudaMemcpy(C->zeta, z.data(), N * sizeof(double2), cudaMemcpyHostToDevice);
        cudaMemcpy(C->slot_t, t.data(), SLOTS * sizeof(int32_t), cudaMemcpyHostToDevice);
    }
    // how many 2- / 3-CTA ladder clusters can be resident at once (MPS, green contexts or partitioned
    // SMs can make this smaller than n_SM / size): the cluster ladders are used only within it
    for (int cs = 2; cs <= 3; cs++) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3((unsigned)(cs * 16));
        cfg.blockDim = dim3(T);
        cfg.dynamicSmemBytes = LADDER_SMEM_BYTES;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        const cudaError_t e = cs == 3 ? cudaOccupancyMaxActiveClusters(&n, (void *)k_ladder_c3, &cfg)
                                      : cudaOccupancyMaxActiveClusters(&n, (void *)k_ladder_t<true>, &cfg);
        C->max_cl[cs] = e == cudaSuccess ? n : 0;
        cudaGetLastError();
    }
    if (cudaDeviceSynchronize() != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        cudaFree(C->tw);
        delete C;
        return BM_ERR_CUDA;
    }
    g_ctx[dev] = C;
    *out = C;
    return BM_OK;
}

int launch_check()
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "blindmatch: CUDA error %s\n", cudaGetErrorString(e));
        return BM_ERR_CUDA;
    }
    return BM_OK;
}

// NVTX range for the life of a scope (Nsight Systems timelines; a no-op without a tool attached)
struct NvtxRange {
    explicit NvtxRange(const char *m) { nvtxRangePushA(m); }
    ~NvtxRange() { nvtxRangePop(); }
};

// ------------------------------------------------------------------ options (bm_set_option)
// Process-wide tuning / test switches of the library (explicit, no environment lookups on the hot
// path); the defaults are the product.
std::atomic<int64_t> g_opt[BM_OPT_COUNT_] = {};
struct OptInit {
    OptInit()
    {
        g_opt[BM_OPT_CHUNK_PAIRS] = 16384; // pairs per bm_match chunk (workspace 768 KiB per pair)
        g_opt[BM_OPT_EXPAND_CHUNK] = 2048; // (query, part) outputs per bm_expand / bm_enroll launch
        g_opt[BM_OPT_HOST_GROUPS] = 0;     // bm_match_host query groups (0: about 576 pairs each)
        g_opt[BM_OPT_LADDER_C2] = 1;       // latency-mode ladder on 2-CTA clusters
        g_opt[BM_OPT_LADDER_C3] = 1;       // latency-mode ladder on 3-CTA clusters
        g_opt[BM_OPT_LADDER_TAIL] = 1;     // a large launch's partial last wave on the cluster ladders
        g_opt[BM_OPT_CMP_CHUNK] = 4096;    // pairs per bm_match_cmp chunk
        g_opt[BM_OPT_TENSOR_MMA] = 1;      // K1 on the tensor cores where it applies (k_tensor_mma)
    }
} g_opt_init;
int64_t opt(int k) { return g_opt[k].load(std::memory_order_relaxed); }

// kernels launched by the library (bm_launch_count): the bench's gpu_launches claim
std::atomic<int64_t> g_launches(0);
inline void counted(int64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ------------------------------------------------------------------ profiling
struct Prof {
    bool on = false;
    double ms[7] = {0};
    int64_t launches[7] = {0};
    int64_t units[7] = {0};
};
Prof g_prof;
std::mutex g_prof_mu;

struct Rec {
    int cls;
    int64_t units;
    cudaEvent_t a, b;
};

} // namespace

struct bm_pk_dev {
    int dev;
    uint8_t digest[32];
    ulonglong2 *pk;
};
struct bm_xk_dev {
    int dev;
    uint8_t digest[32];
    int32_t d, p, s, n_rot;
    ulonglong2 *pk2;   // [2][3 limbs q0,q1,q2][N] level-2 public key
    ulonglong2 *gk1;   // [n_rot][2][2][3 limbs q0,q1,P][N], P^-1 in the Q limbs
    ulonglong2 *mask;  // [p][3 limbs q0,q1,q2][N] expansion masks X_i, q2^-1 in the Q limbs
    ulonglong2 *emask; // [p][3][N] enrollment masks E_i (f4; nullptr if not uploaded)
};
struct bm_ck_dev {
    int dev;
    uint8_t digest[32];
    int32_t d, p, s, log_s;
    ulonglong2 *rlk2; // [3][2][4 limbs q0,q1,q2,P][N], P^-1 in the Q limbs
    ulonglong2 *gkl;  // [log_s][2][2][3 limbs q0,q1,P][N], P^-1 in the Q limbs
    ulonglong2 *gkc;  // [s-1][2][2 limbs q0,P][N], P^-1 in the q0 limb
    ulonglong2 *mask; // [2 limbs q0,q1][N], q1^-1 in the q0 limb
};
struct bm_evk_dev {
    int dev;
    uint8_t digest[32];
    int32_t n_rot;
    ulonglong2 *rlk; // [2][2][3] planar polys (ldkey2): 2N u64 each
    ulonglong2 *gk;  // [n_rot][2][2] planar polys
    int32_t n_hrot;  // f2 hoisted rotation keys (0: none)
    uint64_t *hgk;   // [n_hrot][2][2][N], NTT domain, plain residues (no Shoup companion), P^-1 in q0
};

struct bm_sk_dev {
    int dev;
    uint8_t digest[32];
    ulonglong2 *s; // planar Shoup key of the secret mod q0 (NTT domain)
};

// keys -> device NTT-domain Shoup pairs; limb li is multiplied by scale[li] (nullptr: 1); planar
// (default): per polynomial the w plane then the w' plane (read with ldkey2 / ldkey1)
static int upload_key_polys(DevCtx *C, const uint64_t *h, int64_t n_polys, int n_limbs, const int *lp, ulonglong2 **out,
                            const uint64_t *scale = nullptr, bool planar = true)
{
    uint64_t *tmp = nullptr;
    ulonglong2 *dst = nullptr;
    if (cudaMalloc(&tmp, (size_t)n_polys * N * 8) != cudaSuccess ||
        cudaMalloc(&dst, (size_t)n_polys * N * sizeof(ulonglong2)) != cudaSuccess) {
        cudaFree(tmp);
        cudaGetLastError();
        return BM_ERR_OOM;
    }
    cudaMemcpy(tmp, h, (size_t)n_polys * N * 8, cudaMemcpyHostToDevice);
    ConvK K;
    for (int i = 0; i < 4; i++) K.pr[i] = C->pr[i];
    K.in = tmp;
    K.out = nullptr;
    K.n_limbs = n_limbs;
    for (int i = 0; i < 4; i++) K.lp[i] = i < n_limbs ? lp[i] : 0;
    for (int i = 0; i < 4; i++) K.scale[i] = scale && i < n_limbs ? scale[i] : 1;
    K.planar = planar ? 1 : 0;
    k_key_ntt<<<(unsigned)n_polys, T, SMEM_BYTES>>>(K, dst);
    counted();
    int rc = launch_check();
    if (!rc && cudaDeviceSynchronize() != cudaSuccess) rc = BM_ERR_CUDA;
    cudaFree(tmp);
    if (rc) {
        cudaFree(dst);
        return rc;
    }
    *out = dst;
    return BM_OK;
}

extern "C" {

int bm_pk_to_device(const bm_params *prm, const bm_pk *pk, bm_pk_dev **out)
{
    if (!prm || !pk || !out) return BM_ERR_INVALID_ARG;
    if (memcmp(pk->digest, prm->digest, 32)) return BM_ERR_KEY_MISMATCH;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    bm_pk_dev *d = new bm_pk_dev;
    d->dev = C->dev;
    memcpy(d->digest, prm->digest, 32);
    const int lp[2] = {0, 1};
    rc = upload_key_polys(C, pk->v.data(), 4, 2, lp, &d->pk);
    if (rc) {
        delete d;
        return rc;
    }
    *out = d;
    return BM_OK;
}

int bm_evk_to_device(const bm_params *prm, const bm_evk *evk, bm_evk_dev **out)
{
    if (!prm || !evk || !out) return BM_ERR_INVALID_ARG;
    if (memcmp(evk->digest, prm->digest, 32)) return BM_ERR_KEY_MISMATCH;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    bm_evk_dev *d = new bm_evk_dev;
    d->dev = C->dev;
    memcpy(d->digest, prm->digest, 32);
    d->n_rot = evk->n_rot;
    d->gk = nullptr;
    d->n_hrot = 0;
    d->hgk = nullptr;
    const int lr[3] = {0, 1, 2}, lg[2] = {0, 2};
    // device convention: P^-1 is folded into the Q limbs of the key-switching keys (the ModDown
    // multiplies every Q-limb inner product by P^-1 anyway; exact mod q, saves one product)
    const uint64_t sr[3] = {C->pinv[0].x, C->pinv[1].x, 1}, sg[2] = {C->pinv[0].x, 1};
    rc = upload_key_polys(C, evk->rlk.data(), 12, 3, lr, &d->rlk, sr, true);
    if (!rc && evk->n_rot > 0)
        rc = upload_key_polys(C, evk->gk.data(), 4 * (int64_t)evk->n_rot, 2, lg, &d->gk, sg, true);
    if (!rc && evk->n_hrot > 0) { // f2 keys: keep only the residues (the hoisted sum accumulates in 128 bits)
        ulonglong2 *pairs = nullptr;
        const int64_t np = 4 * (int64_t)evk->n_hrot;
        rc = upload_key_polys(C, evk->hgk.data(), np, 2, lg, &pairs, sg, false); // interleaved: w at +0
        if (!rc && cudaMalloc(&d->hgk, (size_t)np * N * 8) != cudaSuccess) rc = BM_ERR_OOM;
        if (!rc && cudaMemcpy2D(d->hgk, 8, pairs, 16, 8, (size_t)np * N, cudaMemcpyDeviceToDevice) != cudaSuccess)
            rc = BM_ERR_CUDA;
        cudaFree(pairs);
        if (!rc) d->n_hrot = evk->n_hrot;
    }
    if (rc) {
        cudaFree(d->rlk);
        cudaFree(d->gk);
        cudaFree(d->hgk);
        cudaGetLastError();
        delete d;
        return rc;
    }
    *out = d;
    return BM_OK;
}

int bm_sk_to_device(const bm_params *prm, const bm_sk *sk, bm_sk_dev **out)
{
    if (!prm || !sk || !out) return BM_ERR_INVALID_ARG;
    if (memcmp(sk->digest, prm->digest, 32)) return BM_ERR_KEY_MISMATCH;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    std::vector<uint64_t> h(N);
    for (int k = 0; k < N; k++) h[k] = sk->s[k] >= 0 ? (uint64_t)sk->s[k] : Q0 - (uint64_t)(-sk->s[k]);
    bm_sk_dev *d = new bm_sk_dev;
    d->dev = C->dev;
    memcpy(d->digest, prm->digest, 32);
    const int lp[1] = {0};
    rc = upload_key_polys(C, h.data(), 1, 1, lp, &d->s);
    if (rc) {
        delete d;
        return rc;
    }
    *out = d;
    return BM_OK;
}

void bm_sk_dev_free(bm_sk_dev *d)
{
    if (!d) return;
    cudaFree(d->s);
    delete d;
}

int bm_decrypt_dev(const bm_params *prm, const bm_sk_dev *sk, const uint64_t *d_ct, int64_t n, double *d_scores,
                   void *stream)
{
    if (!prm || !sk || n < 0) return BM_ERR_INVALID_ARG;
    if (memcmp(sk->digest, prm->digest, 32)) return BM_ERR_KEY_MISMATCH;
    if (n == 0) return BM_OK;
    if (!d_ct || !d_scores) return BM_ERR_INVALID_ARG;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    DecK K;
    K.pr0 = C->pr[0];
    K.s = reinterpret_cast<const uint64_t *>(sk->s);
    K.ct = d_ct;
    K.scores = d_scores;
    K.zeta = C->zeta;
    K.slot_t = C->slot_t;
    K.B = prm->B;
    K.s_len = prm->s;
    K.inv_scale = 1.0 / prm->out_scale;
    for (int64_t c0 = 0; c0 < n && !rc; c0 += 1 << 30) { // grid.x limit
        DecK Kc = K;
        const int64_t nc = n - c0 < (1 << 30) ? n - c0 : (1 << 30);
        Kc.ct = d_ct + (size_t)c0 * 2 * N;
        Kc.scores = d_scores + (size_t)c0 * prm->B;
        k_decrypt<<<(unsigned)nc, T, DEC_SMEM_BYTES, (cudaStream_t)stream>>>(Kc);
        counted();
        rc = launch_check();
    }
    return rc;
}

void bm_pk_dev_free(bm_pk_dev *d)
{
    if (!d) return;
    cudaFree(d->pk);
    delete d;
}
void bm_evk_dev_free(bm_evk_dev *d)
{
    if (!d) return;
    cudaFree(d->rlk);
    cudaFree(d->gk);
    cudaFree(d->hgk);
    delete d;
}

int bm_encrypt(const bm_params *prm, const bm_pk_dev *pk, const int64_t *d_pt, int64_t n_cts, uint64_t first_obj,
               uint64_t seed, uint64_t *d_out, void *stream)
{
    if (!prm || !pk || n_cts < 0 || (n_cts > 0 && (!d_pt || !d_out))) return BM_ERR_INVALID_ARG;
    if (memcmp(pk->digest, prm->digest, 32)) return BM_ERR_KEY_MISMATCH;
    if (n_cts == 0) return BM_OK;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    EncK Ek;
    for (int i = 0; i < 4; i++) Ek.pr[i] = C->pr[i];
    Ek.pk = pk->pk;
    Ek.pt = d_pt;
    Ek.out = d_out;
    Ek.first_obj = first_obj;
    Ek.seed = seed;
    rng_encrypt_kx(Ek.kx); // fresh per call unless seeded (bm_rng_mode)
    Ek.n_limbs = 2;
    Ek.lp[0] = 0;
    Ek.lp[1] = 1;
    Ek.lp[2] = 3;
    k_encrypt<<<(unsigned)(2 * n_cts), T, SMEM_BYTES, (cudaStream_t)stream>>>(Ek);
    counted();
    return launch_check();
}

static int encrypt_host_pt(const bm_params *prm, const bm_pk_dev *pk, const std::vector<int64_t> &pt, int64_t n_cts,
                           uint64_t first_obj, uint64_t seed, uint64_t *d_out, void *stream)
{
    int64_t *d_pt = nullptr;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMallocAsync(&d_pt, pt.size() * 8, s) != cudaSuccess) {
        cudaGetLastError();
        return BM_ERR_OOM;
    }
    cudaMemcpyAsync(d_pt, pt.data(), pt.size() * 8, cudaMemcpyHostToDevice, s);
    int rc = bm_encrypt(prm, pk, d_pt, n_cts, first_obj, seed, d_out, stream);
    cudaFreeAsync(d_pt, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) rc = BM_ERR_CUDA;
    return rc;
}

int bm_encrypt_db(const bm_params *prm, const bm_pk_dev *pk, const double *tmpl, int64_t n, int64_t first_set,
                  int64_t n_sets, uint64_t seed, uint64_t *d_out, void *stream)
{
    if (!prm || !pk || n_sets < 0) return BM_ERR_INVALID_ARG;
    if (n_sets == 0) return BM_OK;
    std::vector<int64_t> pt((size_t)n_sets * prm->p * N);
    int rc = bm_encode_db(prm, tmpl, n, first_set, n_sets, pt.data());
    if (rc) return rc;
    return encrypt_host_pt(prm, pk, pt, n_sets * prm->p, (uint64_t)first_set * prm->p, seed, d_out, stream);
}

int bm_encrypt_query(const bm_params *prm, const bm_pk_dev *pk, const double *q, int64_t nq, int64_t first_query,
                     uint64_t seed, uint64_t *d_out, void *stream)
{
    if (!prm || !pk || nq < 0 || first_query < 0) return BM_ERR_INVALID_ARG;
    if (nq == 0) return BM_OK;
    std::vector<int64_t> pt((size_t)nq * prm->p * N);
    int rc = bm_encode_query(prm, q, nq, pt.data());
    if (rc) return rc;
    return encrypt_host_pt(prm, pk, pt, nq * prm->p, (uint64_t)first_query * prm->p, seed, d_out, stream);
}

static int convert(const bm_params *prm, const uint64_t *in, int64_t n_cts, int32_t n_limbs, uint64_t *out,
                   void *stream, int dir)
{
    if (!prm || n_cts < 0 || n_limbs < 1 || n_limbs > 3 || (n_cts && (!in || !out))) return BM_ERR_INVALID_ARG;
    if (n_cts == 0) return BM_OK;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    ConvK K;
    for (int i = 0; i < 4; i++) K.pr[i] = C->pr[i];
    K.in = in;
    K.out = out;
    K.n_limbs = n_limbs;
    K.lp[0] = 0;
    K.lp[1] = 1;
    K.lp[2] = 3; // level-2 limb q2 (f3)
    k_convert<<<(unsigned)(n_cts * 2 * n_limbs), T, SMEM_BYTES, (cudaStream_t)stream>>>(K, dir);
    counted();
    return launch_check();
}

int bm_ct_to_coeff(const bm_params *prm, const uint64_t *d_in, int64_t n_cts, int32_t n_limbs, uint64_t *d_out,
                   void *stream)
{
    return convert(prm, d_in, n_cts, n_limbs, d_out, stream, 1);
}
int bm_ct_from_coeff(const bm_params *prm, const uint64_t *d_in, int64_t n_cts, int32_t n_limbs, uint64_t *d_out,
                     void *stream)
{
    return convert(prm, d_in, n_cts, n_limbs, d_out, stream, 0);
}

// ------------------------------------------------------------------ f3: query expansion
static int upload_masks(DevCtx *C, const bm_params *prm, const int64_t *h_masks, ulonglong2 **out)
{
    // integer plaintexts -> residues per limb (q0, q1, q2), q2^-1 folded into the Q limbs
    std::vector<uint64_t> m(3 * (size_t)prm->p * N);
    const uint64_t qs[3] = {Q0, Q1, Q2};
    for (int i = 0; i < prm->p; i++)
        for (int l = 0; l < 3; l++)
            for (int k = 0; k < N; k++) {
                const int64_t x = h_masks[(size_t)i * N + k];
                const uint64_t q = qs[l];
                m[((size_t)i * 3 + l) * N + k] = x >= 0 ? (uint64_t)x % q : q - 1 - (uint64_t)(-(x + 1)) % q;
            }
    const uint64_t sm[3] = {C->q2inv[0].x, C->q2inv[1].x, 1};
    const int l2[3] = {0, 1, 3};
    return upload_key_polys(C, m.data(), 3 * (int64_t)prm->p, 3, l2, out, sm);
}

int bm_xk_to_device(const bm_params *prm, const bm_pk *pk, const bm_xk *xk, const int64_t *h_masks,
                    const int64_t *h_emasks, bm_xk_dev **out)
{
    if (!prm || !pk || !xk || !h_masks || !out) return BM_ERR_INVALID_ARG;
    if (memcmp(pk->digest, prm->digest, 32) || memcmp(xk->digest, prm->digest, 32) || xk->d != prm->d ||
        xk->p != prm->p)
        return BM_ERR_KEY_MISMATCH;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    bm_xk_dev *d = new bm_xk_dev;
    d->dev = C->dev;
    memcpy(d->digest, prm->digest, 32);
    d->d = prm->d;
    d->p = prm->p;
    d->s = prm->s;
    d->n_rot = xk->n_rot;
    d->pk2 = d->gk1 = d->mask = d->emask = nullptr;
    // level-2 pk: pk's limbs q0, q1 and xk's q2 limb
    std::vector<uint64_t> h(6 * (size_t)N);
    for (int c = 0; c < 2; c++) {
        memcpy(&h[(size_t)(c * 3 + 0) * N], &pk->v[(size_t)(c * 2 + 0) * N], 8 * (size_t)N);
        memcpy(&h[(size_t)(c * 3 + 1) * N], &pk->v[(size_t)(c * 2 + 1) * N], 8 * (size_t)N);
        memcpy(&h[(size_t)(c * 3 + 2) * N], &xk->pk_q2[(size_t)c * N], 8 * (size_t)N);
    }
    const int l2[3] = {0, 1, 3}, lk[3] = {0, 1, 2};
    rc = upload_key_polys(C, h.data(), 6, 3, l2, &d->pk2);
    // Galois keys: P^-1 folded into the Q limbs (the ModDown multiplies by it anyway)
    const uint64_t sk[3] = {C->pinv[0].x, C->pinv[1].x, 1};
    if (!rc && xk->n_rot > 0) rc = upload_key_polys(C, xk->gk1.data(), 12 * (int64_t)xk->n_rot, 3, lk, &d->gk1, sk);
    if (!rc) rc = upload_masks(C, prm, h_masks, &d->mask);
    if (!rc && h_emasks) rc = upload_masks(C, prm, h_emasks, &d->emask);
    if (rc) {
        cudaFree(d->pk2);
        cudaFree(d->gk1);
        cudaFree(d->mask);
        cudaFree(d->emask);
        cudaGetLastError();
        delete d;
        return rc;
    }
    *out = d;
    return BM_OK;
}

void bm_xk_dev_free(bm_xk_dev *d)
{
    if (!d) return;
    cudaFree(d->pk2);
    cudaFree(d->gk1);
    cudaFree(d->mask);
    cudaFree(d->emask);
    delete d;
}

int bm_encrypt_l2(const bm_params *prm, const bm_xk_dev *xk, const int64_t *d_pt, int64_t n_cts, uint64_t first_obj,
                  uint64_t seed, uint64_t *d_out, void *stream)
{
    if (!prm || !xk || n_cts < 0 || (n_cts > 0 && (!d_pt || !d_out))) return BM_ERR_INVALID_ARG;
    if (memcmp(xk->digest, prm->digest, 32)) return BM_ERR_KEY_MISMATCH;
    if (n_cts == 0) return BM_OK;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    EncK Ek;
    for (int i = 0; i < 4; i++) Ek.pr[i] = C->pr[i];
    Ek.pk = xk->pk2;
    Ek.pt = d_pt;
    Ek.out = d_out;
    Ek.first_obj = first_obj;
    Ek.seed = seed;
    rng_encrypt_kx(Ek.kx); // fresh per call unless seeded (bm_rng_mode)
    Ek.n_limbs = 3;
    Ek.lp[0] = 0;
    Ek.lp[1] = 1;
    Ek.lp[2] = 3;
    k_encrypt<<<(unsigned)(3 * n_cts), T, SMEM_BYTES, (cudaStream_t)stream>>>(Ek);
    counted();
    return launch_check();
}

static int64_t expand_chunk_cts(const bm_params *prm, int32_t nq)
{
    int64_t ch = opt(BM_OPT_EXPAND_CHUNK); // (query, part) outputs per launch: 6 N u64 of workspace each
    ch = ch / prm->p * prm->p; // whole queries
    if (ch < prm->p) ch = prm->p;
    const int64_t total = (int64_t)nq * prm->p;
    return total < ch ? total : ch;
}

size_t bm_expand_ws_bytes(const bm_params *prm, int32_t nq)
{
    if (!prm || nq <= 0) return 0;
    return (size_t)expand_chunk_cts(prm, nq) * XU_POLYS * N * sizeof(uint64_t);
}

int bm_expand(const bm_params *prm, const bm_xk_dev *xk, const uint64_t *d_in, int32_t nq, uint64_t *d_out, void *d_ws,
              size_t ws_bytes, void *stream)
{
    if (!prm || !xk || nq < 0) return BM_ERR_INVALID_ARG;
    if (memcmp(xk->digest, prm->digest, 32) || xk->p != prm->p || xk->d != prm->d) return BM_ERR_KEY_MISMATCH;
    int log_p = 0;
    while ((1 << log_p) < prm->p) log_p++;
    if (xk->n_rot < log_p) return BM_ERR_MISSING_ROTATION_KEY;
    if (nq == 0) return BM_OK;
    if (!d_in || !d_out || !d_ws) return BM_ERR_INVALID_ARG;
    if (ws_bytes < bm_expand_ws_bytes(prm, nq)) return BM_ERR_WORKSPACE;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    ExpK K;
    for (int i = 0; i < 4; i++) K.pr[i] = C->pr[i];
    K.pinv[0] = C->pinv[0];
    K.pinv[1] = C->pinv[1];
    K.q2inv[0] = C->q2inv[0];
    K.q2inv[1] = C->q2inv[1];
    K.mask = xk->mask;
    K.XU = (uint64_t *)d_ws;
    K.p = prm->p;
    K.enroll = 0;
    K.Bk = prm->B;
    K.bit = 0;
    K.u0 = 0;
    const int64_t ch = expand_chunk_cts(prm, nq), qch = ch / prm->p;
    for (int64_t j0 = 0; j0 < nq && !rc; j0 += qch) {
        const int64_t nqc = nq - j0 < qch ? nq - j0 : qch;
        const unsigned ncb = (unsigned)(2 * nqc * prm->p);
        K.in = d_in + (size_t)j0 * 6 * N;
        K.out = d_out + (size_t)j0 * prm->p * 4 * N;
        K.gk = nullptr;
        K.g = 1;
        k_exp_mask<<<ncb, T, X1_SMEM_BYTES, s>>>(K);
        counted();
        rc = launch_check();
        for (int t = 0; t < log_p && !rc; t++) {
            K.gk = xk->gk1 + (size_t)t * 12 * N;
            K.g = (uint32_t)powmod_d(5, (uint64_t)prm->s << t, 2 * N);
            k_rot1_digits<<<ncb, T, X2_SMEM_BYTES, s>>>(K);
            counted();
            k_rot1_ks<<<ncb, T, X3_SMEM_BYTES, s>>>(K);
            counted();
            rc = launch_check();
        }
    }
    return rc;
}

// ------------------------------------------------------------------ f4: server-side enrollment
static int64_t enroll_chunk_templates(const bm_params *prm, int64_t n)
{
    int64_t ch = opt(BM_OPT_EXPAND_CHUNK); // parts per launch: 10 N u64 of workspace each (W + XU)
    int64_t t = ch / prm->p;
    if (t < 1) t = 1;
    return n < t ? n : t;
}

size_t bm_enroll_ws_bytes(const bm_params *prm, int64_t n)
{
    if (!prm || n <= 0) return 0;
    return (size_t)enroll_chunk_templates(prm, n) * prm->p * (4 + XU_POLYS) * N * sizeof(uint64_t);
}

int bm_enroll(const bm_params *prm, const bm_xk_dev *xk, const uint64_t *d_in, int64_t n, int64_t first_template,
              uint64_t *d_db, int64_t n_sets, void *d_ws, size_t ws_bytes, void *stream)
{
    if (!prm || !xk || n < 0 || first_template < 0 || n_sets < 0) return BM_ERR_INVALID_ARG;
    if (memcmp(xk->digest, prm->digest, 32) || xk->p != prm->p || xk->d != prm->d) return BM_ERR_KEY_MISMATCH;
    int log_b = 0;
    while ((1 << log_b) < prm->B) log_b++;
    if (xk->n_rot < log_b) return BM_ERR_MISSING_ROTATION_KEY;
    if (!xk->emask) return BM_ERR_INVALID_ARG;
    if (n == 0) return BM_OK;
    if ((first_template + n + prm->B - 1) / prm->B > n_sets) return BM_ERR_CAPACITY;
    if (!d_in || !d_db || !d_ws) return BM_ERR_INVALID_ARG;
    if (ws_bytes < bm_enroll_ws_bytes(prm, n)) return BM_ERR_WORKSPACE;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t tch = enroll_chunk_templates(prm, n);
    uint64_t *W = (uint64_t *)d_ws;
    ExpK K;
    for (int i = 0; i < 4; i++) K.pr[i] = C->pr[i];
    K.pinv[0] = C->pinv[0];
    K.pinv[1] = C->pinv[1];
    K.q2inv[0] = C->q2inv[0];
    K.q2inv[1] = C->q2inv[1];
    K.mask = xk->emask;
    K.XU = W + (size_t)tch * prm->p * 4 * N;
    K.p = prm->p;
    K.out = W;
    K.Bk = prm->B;
    for (int64_t c0 = 0; c0 < n && !rc; c0 += tch) {
        const int64_t nc = n - c0 < tch ? n - c0 : tch;
        const unsigned ncb = (unsigned)(2 * nc * prm->p);
        K.in = d_in + (size_t)c0 * 6 * N;
        K.u0 = first_template + c0;
        K.enroll = 0;
        K.g = 1;
        K.gk = nullptr;
        K.bit = 0;
        k_exp_mask<<<ncb, T, X1_SMEM_BYTES, s>>>(K); // Res(Mul(P)(C_u, E_i)) for every part
        rc = launch_check();
        K.enroll = 1;
        for (int b = 0; b < log_b && !rc; b++) {     // right rotation by (k - i) s = left by m s, bit by bit
            K.bit = b;
            K.gk = xk->gk1 + (size_t)b * 12 * N;
            K.g = (uint32_t)powmod_d(5, (uint64_t)prm->s << b, 2 * N);
            k_rot1_digits<<<ncb, T, X2_SMEM_BYTES, s>>>(K);
            counted();
            k_rot1_ks<<<ncb, T, X3_SMEM_BYTES, s>>>(K);
            counted();
            rc = launch_check();
        }
        if (rc) break;
        const int64_t t0 = K.u0 / prm->B, t1 = (K.u0 + nc - 1) / prm->B;
        k_enroll_add<<<(unsigned)((t1 - t0 + 1) * prm->p * 4 * (N / 256)), 256, 0, s>>>(W, K.u0, nc, prm->p, prm->B, t0,
                                                                                         d_db);
        counted();
        rc = launch_check();
    }
    return rc;
}

// ------------------------------------------------------------------ f1: compressed scan
int bm_ck_to_device(const bm_params *prm, const bm_ck *ck, const int64_t *h_mask, bm_ck_dev **out)
{
    if (!prm || !ck || !h_mask || !out) return BM_ERR_INVALID_ARG;
    if (memcmp(ck->digest, prm->digest, 32) || ck->d != prm->d || ck->p != prm->p) return BM_ERR_KEY_MISMATCH;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    bm_ck_dev *d = new bm_ck_dev;
    d->dev = C->dev;
    memcpy(d->digest, prm->digest, 32);
    d->d = prm->d;
    d->p = prm->p;
    d->s = prm->s;
    d->log_s = ck->log_s;
    d->rlk2 = d->gkl = d->gkc = d->mask = nullptr;
    const int l4[4] = {0, 1, 3, 2}, l3[3] = {0, 1, 2}, l0[2] = {0, 2}, lm[2] = {0, 1};
    const uint64_t s4[4] = {C->pinv[0].x, C->pinv[1].x, C->pinv2.x, 1}, s3[3] = {C->pinv[0].x, C->pinv[1].x, 1};
    const uint64_t s0[2] = {C->pinv[0].x, 1}, sm[2] = {C->q1inv.x, 1};
    rc = upload_key_polys(C, ck->rlk2.data(), 24, 4, l4, &d->rlk2, s4);
    if (!rc && ck->log_s > 0) rc = upload_key_polys(C, ck->gkl.data(), 12 * (int64_t)ck->log_s, 3, l3, &d->gkl, s3);
    if (!rc && prm->s > 1) rc = upload_key_polys(C, ck->gkc.data(), 4 * (int64_t)(prm->s - 1), 2, l0, &d->gkc, s0);
    if (!rc) {
        std::vector<uint64_t> m(2 * (size_t)N);
        for (int l = 0; l < 2; l++) {
            const uint64_t q = l ? Q1 : Q0;
            for (int k = 0; k < N; k++) {
                const int64_t x = h_mask[k];
                m[(size_t)l * N + k] = x >= 0 ? (uint64_t)x % q : q - 1 - (uint64_t)(-(x + 1)) % q;
            }
        }
        rc = upload_key_polys(C, m.data(), 2, 2, lm, &d->mask, sm);
    }
    if (rc) {
        cudaFree(d->rlk2);
        cudaFree(d->gkl);
        cudaFree(d->gkc);
        cudaFree(d->mask);
        cudaGetLastError();
        delete d;
        return rc;
    }
    *out = d;
    return BM_OK;
}

void bm_ck_dev_free(bm_ck_dev *d)
{
    if (!d) return;
    cudaFree(d->rlk2);
    cudaFree(d->gkl);
    cudaFree(d->gkc);
    cudaFree(d->mask);
    delete d;
}

// workspace per pair (u64 polynomials): D01 6, D2 3, XU 9, XC 4, XR 2, XO 2, scratch 2
constexpr int CMP_WS_POLYS = 28;
static int64_t cmp_chunk_pairs(int64_t total)
{
    int64_t ch = opt(BM_OPT_CMP_CHUNK);
    return total < ch ? total : ch;
}

size_t bm_match_cmp_ws_bytes(const bm_params *prm, int64_t n_sets, int32_t nq)
{
    if (!prm || n_sets <= 0 || nq <= 0) return 0;
    return (size_t)cmp_chunk_pairs(n_sets * (int64_t)nq) * CMP_WS_POLYS * N * sizeof(uint64_t);
}

int bm_match_cmp(const bm_params *prm, const bm_ck_dev *ck, const uint64_t *d_db, int64_t n_sets, const uint64_t *d_q,
                 int32_t nq, uint64_t *d_out, void *d_ws, size_t ws_bytes, void *stream)
{
    if (!prm || !ck || n_sets < 0 || nq < 0) return BM_ERR_INVALID_ARG;
    if (memcmp(ck->digest, prm->digest, 32) || ck->p != prm->p || ck->d != prm->d) return BM_ERR_KEY_MISMATCH;
    if (ck->log_s < prm->log_s) return BM_ERR_MISSING_ROTATION_KEY;
    const int64_t total = n_sets * (int64_t)nq;
    if (total == 0) return BM_OK;
    if (!d_db || !d_q || !d_out || !d_ws) return BM_ERR_INVALID_ARG;
    if (ws_bytes < bm_match_cmp_ws_bytes(prm, n_sets, nq)) return BM_ERR_WORKSPACE;
    DevCtx *Cx;
    int rc = ctx_get(&Cx);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t ch = cmp_chunk_pairs(total), n_groups = (n_sets + prm->s - 1) / prm->s;
    CmpK C;
    MatchK &K = C.m;
    for (int i = 0; i < 4; i++) K.pr[i] = Cx->pr[i];
    K.pinv[0] = Cx->pinv[0];
    K.pinv[1] = Cx->pinv[1];
    K.q1inv = Cx->q1inv;
    K.db = d_db;
    K.qry = d_q;
    K.out = nullptr;
    K.nq_total = nq;
    K.n_sets = n_sets;
    K.p = prm->p;

    uint64_t *ws = (uint64_t *)d_ws;
    const size_t P1 = (size_t)ch * N;
    K.D01 = ws;
    K.D2 = K.D01 + 6 * P1;
    K.XU = K.D2 + 3 * P1;
    K.XC = K.XU + 9 * P1;
    K.XR = K.XC + 4 * P1;
    K.XO = K.XR + 2 * P1;
    K.ACC = nullptr;
    C.scr = K.XO + 2 * P1;
    C.pinv2 = Cx->pinv2;
    C.q2inv[0] = Cx->q2inv[0];
    C.q2inv[1] = Cx->q2inv[1];
    C.rlk2 = ck->rlk2;
    C.gkc = ck->gkc;
    C.mask = ck->mask;
    C.s = prm->s;
    ExpK X; // the level-1 ladder reuses f3's rotation kernels (C <- C + Rot(C, 2^i))
    for (int i = 0; i < 4; i++) X.pr[i] = Cx->pr[i];
    X.pinv[0] = Cx->pinv[0];
    X.pinv[1] = Cx->pinv[1];
    X.q2inv[0] = Cx->q2inv[0];
    X.q2inv[1] = Cx->q2inv[1];
    X.mask = nullptr;
    X.in = nullptr;
    X.out = K.XC;
    X.XU = K.XU;
    X.p = 1;
    X.enroll = 0;
    X.Bk = 1;
    X.bit = 0;
    X.u0 = 0;
    cudaMemsetAsync(d_out, 0, (size_t)nq * n_groups * 2 * N * sizeof(uint64_t), s);
    const int64_t ct_full = n_sets < ch ? n_sets : ch;
    const int64_t cq_full = ch / ct_full < nq ? ch / ct_full : nq;
    for (int64_t jq0 = 0; jq0 < nq && !rc; jq0 += cq_full)
        for (int64_t t0 = 0; t0 < n_sets && !rc; t0 += ct_full) {
            K.jq0 = jq0;
            K.t0 = t0;
            K.cq = (int32_t)(nq - jq0 < cq_full ? nq - jq0 : cq_full);
            K.ct = n_sets - t0 < ct_full ? n_sets - t0 : ct_full;
            const int64_t np = K.cq * K.ct;
            const unsigned npu = (unsigned)np;
            const unsigned ntiles = (unsigned)(((K.cq + TQB - 1) / TQB) * ((K.ct + TSB - 1) / TSB) * (N / CS / TSL));
            k_tensor<3, false><<<3 * ntiles, TT, TENSOR_SMEM_BYTES, s>>>(K, 0, prm->p);
            counted();
            k_digits3<<<3 * npu, T, C1_SMEM_BYTES, s>>>(C);
            counted();
            k_relin3a<<<2 * npu, T, C2_SMEM_BYTES, s>>>(C);
            counted();
            k_relin3b<<<4 * npu, T, SMEM_BYTES, s>>>(C);
            counted();
            rc = launch_check();
            for (int i = 0; i < prm->log_s && !rc; i++) {
                X.gk = ck->gkl + (size_t)i * 12 * N;
                X.g = (uint32_t)powmod_d(5, (uint64_t)1 << i, 2 * N);
                k_rot1_digits<<<2 * npu, T, X2_SMEM_BYTES, s>>>(X);
                counted();
                k_rot1_ks<<<2 * npu, T, X3_SMEM_BYTES, s>>>(X);
                counted();
                rc = launch_check();
            }
            if (rc) break;
            k_cmp_mask<<<2 * npu, T, SMEM_BYTES, s>>>(C);
            counted();
            k_cmp_rot<<<npu, T, C4_SMEM_BYTES, s>>>(C);
            counted();
            const int64_t g0 = t0 / prm->s, g1 = (t0 + K.ct - 1) / prm->s, ng = g1 - g0 + 1;
            k_cmp_add<<<(unsigned)(K.cq * ng * 2 * (N / 256)), 256, 0, s>>>(C, d_out, n_groups, g0, ng);
            counted();
            rc = launch_check();
        }
    return rc;
}

// ------------------------------------------------------------------ the scan
static int64_t chunk_pairs(int64_t total)
{
    int64_t ch = opt(BM_OPT_CHUNK_PAIRS); // large chunks: fewer launches and kernel tails (768 KiB of workspace per pair)
    return total < ch ? total : ch;
}

size_t bm_match_ws_bytes(const bm_params *prm, int64_t n_sets, int32_t nq, int32_t order)
{
    if (!prm || n_sets <= 0 || nq <= 0) return 0;
    const int polys = order == BM_ORDER_PAPER ? WS_POLYS_PAPER : WS_POLYS;
    return (size_t)chunk_pairs(n_sets * (int64_t)nq) * polys * N * sizeof(uint64_t);
}

void bm_set_profiling(int32_t on)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.on = on != 0;
}
void bm_profile_reset(void)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    bool on = g_prof.on;
    g_prof = Prof();
    g_prof.on = on;
}
int bm_profile_read(double *ms, int64_t *launches, int64_t *units)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (int i = 0; i < 7; i++) {
        if (ms) ms[i] = g_prof.ms[i];
        if (launches) launches[i] = g_prof.launches[i];
        if (units) units[i] = g_prof.units[i];
    }
    return BM_OK;
}

static int match_impl(const bm_params *prm, const bm_evk_dev *evk, const uint64_t *d_db, int64_t n_sets,
                      const uint64_t *d_q, int32_t nq, uint64_t *d_out, uint64_t *const *d_rows, int64_t set_offset,
                      void *d_ws, size_t ws_bytes, int32_t order, void *stream)
{
    const bool deg2 = order == BM_ORDER_DEG2;
    if (!prm || (!evk && !deg2) || n_sets < 0 || nq < 0 ||
        (order != BM_ORDER_HOISTED && order != BM_ORDER_PAPER && order != BM_ORDER_HOISTED_ROT &&
         order != BM_ORDER_BSGS && !deg2))
        return BM_ERR_INVALID_ARG;
    if (deg2 && prm->s != 1) return BM_ERR_INVALID_LAYOUT; // the degree-2 output has no ladder: p = d only
    if (evk && memcmp(evk->digest, prm->digest, 32)) return BM_ERR_KEY_MISMATCH;
    const bool hoisted_rot = order == BM_ORDER_HOISTED_ROT || order == BM_ORDER_BSGS;
    if (!deg2 && !hoisted_rot && evk->n_rot < prm->log_s) return BM_ERR_MISSING_ROTATION_KEY;
    if (hoisted_rot && evk->n_hrot < prm->s - 1) return BM_ERR_MISSING_ROTATION_KEY;
    const int64_t total = n_sets * (int64_t)nq;
    if (total == 0) return BM_OK;
    if (!d_db || !d_q || (!d_out && !d_rows) || !d_ws || set_offset < 0) return BM_ERR_INVALID_ARG;
    if (ws_bytes < bm_match_ws_bytes(prm, n_sets, nq, order)) return BM_ERR_WORKSPACE;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t ch = chunk_pairs(total);

    MatchK K;
    for (int i = 0; i < 4; i++) K.pr[i] = C->pr[i];
    K.pinv[0] = C->pinv[0];
    K.pinv[1] = C->pinv[1];
    K.q1inv = C->q1inv;
    K.q1invP = C->q1invP;
    K.pr0s = C->pr0s;
    K.pmod[0] = C->pmod[0];
    K.pmod[1] = C->pmod[1];
    K.rlk = evk ? reinterpret_cast<const uint64_t *>(evk->rlk) : nullptr;
    K.gk = evk ? reinterpret_cast<const uint64_t *>(evk->gk) : nullptr;
    K.db = d_db;
    K.qry = d_q;
    K.out = d_out;
    K.rows = d_rows;
    K.nq_total = nq;
    K.set_off = set_offset;
    K.n_sets = n_sets;
    K.p = prm->p;
    uint64_t *ws = (uint64_t *)d_ws;
    const size_t P1 = (size_t)ch * N;
    K.D01 = ws;
    K.D2 = K.D01 + 4 * P1;
    K.cap = ch; // the D01 / D2 piece layout's pair stride (dofs)
    K.XC = K.D2 + 2 * P1;
    K.XU = K.XC + 2 * P1;
    K.ACC = order == BM_ORDER_PAPER ? K.XU + 4 * P1 : nullptr;
    const CtBuf bufC = order == BM_ORDER_PAPER ? CtBuf{K.ACC, 2 * N} : CtBuf{K.XC, 2 * N};
    const uint8_t *dbp = tc_lookup(d_db, n_sets, prm->p); // the DB in the tensor-core layout, if registered

    bool prof;
    {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        prof = g_prof.on;
    }
    std::vector<Rec> recs;
    auto beg = [&](int cls, int64_t units) {
        if (!prof) return;
        Rec r;
        r.cls = cls;
        r.units = units;
        cudaEventCreate(&r.a);
        cudaEventCreate(&r.b);
        cudaEventRecord(r.a, s);
        recs.push_back(r);
    };
    auto end = [&]() {
        if (prof) cudaEventRecord(recs.back().b, s);
    };

    const int log_s = prm->log_s;
    NvtxRange nvtx_call(d_rows ? "bm_match_rows" : "bm_match");
    // chunks are rectangles of cq queries x ct sets (cq * ct <= ch pairs); at least TQB queries per chunk
    // when the call has them (the tensor's full, double-buffered tiles instead of the swapped ones)
    const int64_t cq_full = std::min<int64_t>(nq, std::max<int64_t>(ch / n_sets, std::min<int64_t>(TQB, ch)));
    const int64_t ct_full = std::min<int64_t>(n_sets, std::max<int64_t>(1, ch / cq_full));
    for (int64_t jq0 = 0; jq0 < nq && !rc; jq0 += cq_full)
    for (int64_t t0 = 0; t0 < n_sets && !rc; t0 += ct_full) {
        K.jq0 = jq0;
        K.t0 = t0;
        K.cq = (int32_t)(nq - jq0 < cq_full ? nq - jq0 : cq_full);
        K.ct = n_sets - t0 < ct_full ? n_sets - t0 : ct_full;
        const int64_t np = K.cq * K.ct;
        const unsigned npu = (unsigned)np;
        NvtxRange nvtx_chunk("bm_match chunk (tensor, digits, relin, ladder)");
        // few queries: k_tensor<2, true> puts the sets on the tile's wide (TQB) side and the queries
        // on the TSB side -- less of the tile wasted, identical residues (the products are symmetric)
        const bool tswap = K.cq < TQB && K.ct >= TQB;
        const int64_t na = tswap ? K.ct : K.cq, nb = tswap ? K.cq : K.ct;
        const unsigned ntiles = (unsigned)(((na + TQB - 1) / TQB) * ((nb + TSB - 1) / TSB) * (N / CS / (tswap ? 1 : TSL)));
        const bool per_part = order == BM_ORDER_PAPER;
        const int n_rounds = per_part ? prm->p : 1;
        // K1 on the tensor cores (k_tensor_mma): all parts at once (p = 4 or 8), at least half a 128-set
        // tile, and the query operand (16 p MiB per query tile) inside the XC / XU region (6 N u64 per pair
        // of the chunk capacity), which K1 does not otherwise use
        const int64_t n_qt = (K.cq + TM_Q - 1) / TM_Q, n_st = (K.ct + TM_M - 1) / TM_M;
        const bool use_mma = dbp && opt(BM_OPT_TENSOR_MMA) && !per_part && (prm->p == 4 || prm->p == 8) &&
                             K.t0 % TM_M == 0 && K.ct >= TM_M / 2 && K.cq >= TM_Q / 2 &&
                             (size_t)2 * n_qt * N * tm_b_bytes(prm->p) <= (size_t)6 * ch * N * sizeof(uint64_t);
        // the ladder's launch plan (see below): pairs [0, n_one) on the one-CTA kernel, the rest on clusters
        const bool c2ok = opt(BM_OPT_LADDER_C2) != 0, c3ok = opt(BM_OPT_LADDER_C3) != 0;
        const int64_t tail = np % C->n_sm;
        const bool fits = c2ok && C->max_cl[2] > 0;
        const bool all_cl = fits && np <= C->max_cl[2] && 2 * np <= C->n_sm;
        const bool tail_cl = !all_cl && fits && opt(BM_OPT_LADDER_TAIL) && np > C->n_sm && tail > 0 &&
                             2 * tail <= C->n_sm && tail <= C->max_cl[2];
        const int64_t n_one = all_cl ? 0 : tail_cl ? np - tail : np;
        // K3 leaves component 0 split (two accumulators) for the pairs the one-CTA ladder takes
#ifdef BM_K3_NO_SPLIT
        K.split_lim = 0;
#else
        K.split_lim = (LADDER_SPLIT_C0 && log_s > 0 && !hoisted_rot && !per_part && !deg2) ? n_one : 0;
#endif
        for (int r = 0; r < n_rounds && !rc; r++) {
            const int lo = per_part ? r : 0, hi = per_part ? r + 1 : prm->p;
            beg(0, 2 * np);
            if (use_mma) {
                // K1 on the tensor cores: the query operand (B) into the XC / XU region (free until K3)
                uint8_t *XB = reinterpret_cast<uint8_t *>(K.XC);
                const int64_t nthr = 2 * n_qt * (int64_t)N * 2 * TM_Q * (prm->p / 2);
                const unsigned nblk = (unsigned)((nthr + 255) / 256);
                const unsigned nmma = (unsigned)(2 * n_qt * n_st * (N / TM_CB));
                if (prm->p == 8) {
                    k_tm_qexp<8><<<nblk, 256, 0, s>>>(K, XB, (int)n_qt, C->tmc);
                    k_tensor_mma<8><<<nmma, TM_T, tm_smem_bytes<8>(), s>>>(K, dbp, XB, (int)n_qt, (int)n_st, C->tmc);
                } else {
                    k_tm_qexp<4><<<nblk, 256, 0, s>>>(K, XB, (int)n_qt, C->tmc);
                    k_tensor_mma<4><<<nmma, TM_T, tm_smem_bytes<4>(), s>>>(K, dbp, XB, (int)n_qt, (int)n_st, C->tmc);
                }
                counted(2);
            } else if (tswap) {
                k_tensor<2, true><<<2 * ntiles, TT, TENSOR_SMEM_BYTES, s>>>(K, lo, hi);
                counted();
            } else {
                k_tensor<2, false><<<2 * ntiles, TT, TENSOR_SMEM_BYTES, s>>>(K, lo, hi);
                counted();
            }
            end();
            if (deg2) {
                beg(6, 3 * np);
                k_rescale_deg2<<<3 * npu, T, K7_SMEM_BYTES, s>>>(K);
                counted();
                end();
                rc = launch_check();
                break;
            }
            beg(1, 6 * np);
            k_digits<<<2 * npu, T, K2_SMEM_BYTES, s>>>(K);
            counted();
            end();
            beg(2, 6 * np - K.split_lim); // transforms: one fewer for each split component 0
            k_relin<<<2 * npu, T, K3_SMEM_BYTES, s>>>(K, bufC, r > 0 ? 1 : 0);
            counted();
            end();
            rc = launch_check();
        }
        if (log_s > 0 && !rc && hoisted_rot) {
            // BM_ORDER_HOISTED_ROT: one hoisted sum of s rotations; BM_ORDER_BSGS: b = 2^ceil(log2(s)/2)
            // baby rotations (NTT-domain result in XU) then g = s / b giant ones by b (the oracle's
            // bsgs_rot_sum; g = 1 is the plain hoisted sum)
            const int b = order == BM_ORDER_BSGS ? 1 << ((log_s + 1) / 2) : prm->s, g = prm->s / b;
            const CtBuf bufU{K.XU, 4 * N};
            uint32_t gb = 1;
            for (int i = 0; i < b; i++) gb = (gb * 5u) & (2 * N - 1);
            beg(5, 6 * np * (g > 1 ? 2 : 1));
            if (g > 1) {
                k_hrot<true><<<npu, T, HROT_SMEM_BYTES, s>>>(K, bufC, evk->hgk, b, 1, 5u, bufU);
                counted();
                k_hrot<false><<<npu, T, HROT_SMEM_BYTES, s>>>(K, bufU, evk->hgk, g, b, gb, bufC);
            } else {
                k_hrot<false><<<npu, T, HROT_SMEM_BYTES, s>>>(K, bufC, evk->hgk, b, 1, 5u, bufC);
            }
            counted();
            end();
            rc = launch_check();
        } else if (log_s > 0 && !rc) {
            // transforms: 6 per step, 5 in the one-CTA kernel's steps but the last (component 0 split)
            beg(4, 6 * log_s * np - (LADDER_SPLIT_C0 ? (log_s - 1) * n_one : 0));
            // latency mode: at most n_SM / 2 pairs -> a 2-CTA cluster per pair (k_ladder_t<true>),
            // at most n_SM / 3 -> the 3-rank pipelined ladder (k_ladder_c3).  A large launch whose pair
            // count is not a multiple of n_SM runs its partial last wave the same way: the one-CTA
            // kernel takes floor(np / n_SM) full waves, the cluster kernels the remaining pairs.
            // the cluster paths are used only while their clusters fit the device at once
            // (DevCtx::max_cl, from cudaOccupancyMaxActiveClusters); a failed cluster launch falls
            // back to the one-CTA ladder for the same pairs (identical residues)
            auto one_cta = [&](int64_t p0, int64_t n) {
                MatchK Kt = K;
                Kt.pair0 = p0;
                if (p0 + n <= K.split_lim) k_ladder_t<false, true><<<(unsigned)n, T, LADDER_SMEM_BYTES, s>>>(Kt, bufC, log_s);
                else k_ladder_t<false><<<(unsigned)n, T, LADDER_SMEM_BYTES, s>>>(Kt, bufC, log_s);
                counted();
            };
            auto cluster_ladder = [&](int64_t p0, int64_t n) {
                const int cs = (c3ok && n <= C->max_cl[3]) ? 3 : 2;
                cudaLaunchConfig_t cfg = {};
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = cs;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.gridDim = dim3((unsigned)(cs * n));
                cfg.blockDim = dim3(T);
                cfg.dynamicSmemBytes = LADDER_SMEM_BYTES;
                cfg.stream = s;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                MatchK Kt = K;
                Kt.pair0 = p0;
                const cudaError_t e = cs == 3 ? cudaLaunchKernelEx(&cfg, k_ladder_c3, Kt, bufC, (int)log_s)
                                              : cudaLaunchKernelEx(&cfg, k_ladder_t<true>, Kt, bufC, (int)log_s);
                if (e != cudaSuccess) {
                    cudaGetLastError(); // not sticky: a launch-configuration error
                    one_cta(p0, n);
                    if (prof && LADDER_SPLIT_C0) recs.back().units -= (log_s - 1) * n;
                } else {
                    counted();
                }
            };
            if (all_cl) {
                cluster_ladder(0, np);
            } else if (tail_cl) {
                one_cta(0, n_one);
                cluster_ladder(n_one, tail);
            } else {
                one_cta(0, np);
            }
            end();
            rc = launch_check();
        }
        if (log_s == 0 && !rc && !deg2) {
            beg(6, 2 * np);
            k_out_intt<<<2 * npu, T, SMEM_BYTES, s>>>(K, bufC);
            counted();
            end();
            rc = launch_check();
        }
    }
    if (prof) {
        if (cudaStreamSynchronize(s) != cudaSuccess) rc = BM_ERR_CUDA;
        std::lock_guard<std::mutex> lk(g_prof_mu);
        for (Rec &r : recs) {
            float ms = 0;
            cudaEventElapsedTime(&ms, r.a, r.b);
            g_prof.ms[r.cls] += ms;
            g_prof.launches[r.cls] += 1;
            g_prof.units[r.cls] += r.units;
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
    }
    return rc;
}

int bm_match(const bm_params *prm, const bm_evk_dev *evk, const uint64_t *d_db, int64_t n_sets, const uint64_t *d_q,
             int32_t nq, uint64_t *d_out, void *d_ws, size_t ws_bytes, int32_t order, void *stream)
{
    if (!d_out && n_sets > 0 && nq > 0) return BM_ERR_INVALID_ARG;
    return match_impl(prm, evk, d_db, n_sets, d_q, nq, d_out, nullptr, 0, d_ws, ws_bytes, order, stream);
}

int bm_match_rows(const bm_params *prm, const bm_evk_dev *evk, const uint64_t *d_db, int64_t n_sets,
                  const uint64_t *d_q, int32_t nq, uint64_t *const *d_rows, int64_t set_offset, void *d_ws,
                  size_t ws_bytes, int32_t order, void *stream)
{
    if (!d_rows && n_sets > 0 && nq > 0) return BM_ERR_INVALID_ARG;
    return match_impl(prm, evk, d_db, n_sets, d_q, nq, nullptr, d_rows, set_offset, d_ws, ws_bytes, order, stream);
}

int bm_ipc_handle(const void *d_ptr, uint8_t handle[64], uint64_t *offset)
{
    if (!d_ptr || !handle || !offset) return BM_ERR_INVALID_ARG;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, const_cast<void *>(d_ptr)) != cudaSuccess) {
        cudaGetLastError();
        return BM_ERR_CUDA;
    }
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(handle, &h, 64);
    // the handle names the whole allocation: d_ptr's offset inside it (driver cuMemGetAddressRange,
    // reached through the runtime so the library does not link libcuda)
    typedef int (*range_fn)(unsigned long long *, size_t *, unsigned long long);
    static range_fn range = nullptr;
    if (!range) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
            cudaGetLastError();
            return BM_ERR_CUDA;
        }
        range = (range_fn)fn;
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (range(&base, &size, (unsigned long long)(uintptr_t)d_ptr) != 0) return BM_ERR_CUDA;
    *offset = (uint64_t)((uintptr_t)d_ptr - base);
    return BM_OK;
}

int bm_ipc_open(const uint8_t handle[64], void **d_base)
{
    if (!handle || !d_base) return BM_ERR_INVALID_ARG;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    if (cudaIpcOpenMemHandle(d_base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return BM_ERR_CUDA;
    }
    return BM_OK;
}

int bm_ipc_close(void *d_base)
{
    if (!d_base) return BM_ERR_INVALID_ARG;
    if (cudaIpcCloseMemHandle(d_base) != cudaSuccess) {
        cudaGetLastError();
        return BM_ERR_CUDA;
    }
    return BM_OK;
}

// End-to-end scan from host buffers: the queries are processed in G groups.  Group g's query
// upload (copy stream), scan (one of two compute streams, alternating, so that one group's
// kernels fill the tails of the previous group's) and result download (second copy stream)
// overlap with the neighbouring groups through HOST_SLOTS device buffer slots and events.
constexpr int HOST_SLOTS = 4;
static int host_groups(int64_t n_sets, int32_t nq)
{
    // about max(576, min(16384, 4 n_sets)) (query, set) pairs per group (a few waves of the ladder for
    // small databases; whole chunks of several queries for large ones, where one query's group would
    // stream the whole DB through the tensor per query), at least 4 groups
    const int64_t target = std::max<int64_t>(576, std::min<int64_t>(16384, 4 * n_sets));
    int64_t g = (n_sets * (int64_t)nq + target - 1) / target;
    g = g < 4 ? 4 : g;
    if (opt(BM_OPT_HOST_GROUPS) > 0) g = opt(BM_OPT_HOST_GROUPS);
    return (int)(nq < g ? nq : g);
}

size_t bm_match_host_ws_bytes(const bm_params *prm, int64_t n_sets, int32_t nq, int32_t order)
{
    if (!prm || n_sets <= 0 || nq <= 0) return 0;
    const int G = host_groups(n_sets, nq);
    const int64_t gq = (nq + G - 1) / G;
    const int nc = order == BM_ORDER_DEG2 ? 3 : 2; // result components
    const size_t qbytes = (size_t)gq * prm->p * 4 * N * 8, obytes = (size_t)gq * n_sets * nc * N * 8;
    const size_t mws = (bm_match_ws_bytes(prm, n_sets, (int32_t)gq, order) + 255) & ~(size_t)255;
    return HOST_SLOTS * (qbytes + obytes) + 2 * mws;
}

static int match_host_impl(const bm_params *prm, const bm_evk_dev *evk, const uint64_t *d_db, int64_t n_sets,
                           const uint64_t *h_q, int32_t nq, uint64_t *h_out, int32_t ring_rows, void *d_ws,
                           size_t ws_bytes, int32_t order, void *stream)
{
    if (!prm || n_sets < 0 || nq < 0 || ring_rows < 1) return BM_ERR_INVALID_ARG;
    if (n_sets == 0 || nq == 0) return BM_OK;
    if (!h_q || !h_out || !d_ws) return BM_ERR_INVALID_ARG;
    if (ws_bytes < bm_match_host_ws_bytes(prm, n_sets, nq, order)) return BM_ERR_WORKSPACE;
    DevCtx *Cx;
    int rc = ctx_get(&Cx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(Cx->host_mu); // the internal streams are shared by the calls on this device
    NvtxRange nvtx_call("bm_match_host");
    if (!Cx->hs[0])
        for (int k = 0; k < 3; k++)
            if (cudaStreamCreateWithFlags(&Cx->hs[k], cudaStreamNonBlocking) != cudaSuccess) {
                cudaGetLastError();
                return BM_ERR_CUDA;
            }
    const int G = host_groups(n_sets, nq);
    const int64_t gq = (nq + G - 1) / G;
    const size_t qrow = (size_t)prm->p * 4 * N, orow = (size_t)n_sets * (order == BM_ORDER_DEG2 ? 3 : 2) * N; // u64 per query
    uint64_t *dq[HOST_SLOTS], *dout[HOST_SLOTS];
    uint64_t *base = (uint64_t *)d_ws;
    for (int k = 0; k < HOST_SLOTS; k++) dq[k] = base + k * gq * qrow;
    base += HOST_SLOTS * gq * qrow;
    for (int k = 0; k < HOST_SLOTS; k++) dout[k] = base + k * gq * orow;
    base += HOST_SLOTS * gq * orow;
    const size_t mws = (bm_match_ws_bytes(prm, n_sets, (int32_t)gq, order) + 255) & ~(size_t)255;
    void *ws[2] = {base, (uint8_t *)base + mws};
    cudaStream_t sc[2] = {(cudaStream_t)stream, Cx->hs[0]}, su = Cx->hs[1], sd = Cx->hs[2];
    // half-size first and last groups: the pipeline's unoverlapped head (first upload) and tail
    // (last download) shrink; the middle groups are gq queries
    std::vector<int64_t> g0, gn;
    {
        const int64_t h = nq >= 4 ? (gq + 1) / 2 : gq; // (fewer queries: groups of gq, the slot size)
        int64_t q = 0;
        g0.push_back(0), gn.push_back(h), q = h;
        const int64_t tail = nq - q > h ? h : 0;
        while (q < nq - tail) {
            const int64_t c = nq - tail - q < gq ? nq - tail - q : gq;
            g0.push_back(q), gn.push_back(c), q += c;
        }
        if (tail) g0.push_back(q), gn.push_back(tail);
    }
    const int ngroups = (int)g0.size();
    // events: ev[g][0] upload done, [1] scan done, [2] download done, then the start event and the three
    // completion events; owned by the device context (created once, reused: the call synchronises before
    // returning, so every event is idle again)
    const size_t n_ev = 3 * (size_t)ngroups + 4;
    while (Cx->hev.size() < n_ev) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            return BM_ERR_CUDA;
        }
        Cx->hev.push_back(e);
    }
    cudaEvent_t *ev = Cx->hev.data();
    cudaEvent_t ev_start = ev[3 * (size_t)ngroups];
    cudaEventRecord(ev_start, sc[0]); // everything starts after the work already on the caller's stream
    cudaStreamWaitEvent(sc[1], ev_start, 0);
    cudaStreamWaitEvent(su, ev_start, 0);
    cudaStreamWaitEvent(sd, ev_start, 0);
    for (int g = 0; g < ngroups && !rc; g++) {
        cudaEvent_t *E = ev + 3 * (size_t)g;
        const int slot = g % HOST_SLOTS;
        cudaStream_t cs = sc[g & 1];
        const int64_t q0 = g0[g], nqg = gn[g];
        // the query slot is free once the scan of group g - HOST_SLOTS has consumed it
        if (g >= HOST_SLOTS) cudaStreamWaitEvent(su, ev[3 * (size_t)(g - HOST_SLOTS) + 1], 0);
        if (cudaMemcpyAsync(dq[slot], h_q + q0 * qrow, nqg * qrow * 8, cudaMemcpyHostToDevice, su) != cudaSuccess)
            rc = BM_ERR_CUDA;
        cudaEventRecord(E[0], su);
        cudaStreamWaitEvent(cs, E[0], 0);
        // the output slot is free once group g - HOST_SLOTS's results are downloaded
        if (g >= HOST_SLOTS) cudaStreamWaitEvent(cs, ev[3 * (size_t)(g - HOST_SLOTS) + 2], 0);
        if (!rc)
            rc = bm_match(prm, evk, d_db, n_sets, dq[slot], (int32_t)nqg, dout[slot], ws[g & 1], mws, order, cs);
        cudaEventRecord(E[1], cs);
        cudaStreamWaitEvent(sd, E[1], 0);
        // rows q0 .. q0 + nqg - 1 land at ring rows (q mod ring_rows): at most two contiguous runs
        for (int64_t q = q0; q < q0 + nqg && !rc;) {
            const int64_t r = q % ring_rows, run = std::min<int64_t>(q0 + nqg - q, ring_rows - r);
            if (cudaMemcpyAsync(h_out + r * orow, dout[slot] + (q - q0) * orow, run * orow * 8, cudaMemcpyDeviceToHost,
                                sd) != cudaSuccess)
                rc = BM_ERR_CUDA;
            q += run;
        }
        cudaEventRecord(E[2], sd);
    }
    // the caller's stream waits for the internal streams (stream-ordered completion), then the call blocks
    cudaEvent_t *fin = ev + 3 * (size_t)ngroups + 1;
    for (int k = 0; k < 3; k++) {
        cudaEventRecord(fin[k], k == 0 ? sc[1] : k == 1 ? su : sd);
        cudaStreamWaitEvent(sc[0], fin[k], 0);
    }
    if (cudaStreamSynchronize(sc[0]) != cudaSuccess) rc = rc ? rc : BM_ERR_CUDA;
    return rc;
}

int bm_match_host(const bm_params *prm, const bm_evk_dev *evk, const uint64_t *d_db, int64_t n_sets,
                  const uint64_t *h_q, int32_t nq, uint64_t *h_out, void *d_ws, size_t ws_bytes, int32_t order,
                  void *stream)
{
    return match_host_impl(prm, evk, d_db, n_sets, h_q, nq, h_out, nq > 0 ? nq : 1, d_ws, ws_bytes, order, stream);
}

int bm_match_host_ring(const bm_params *prm, const bm_evk_dev *evk, const uint64_t *d_db, int64_t n_sets,
                       const uint64_t *h_q, int32_t nq, uint64_t *h_ring, int32_t ring_rows, void *d_ws,
                       size_t ws_bytes, int32_t order, void *stream)
{
    return match_host_impl(prm, evk, d_db, n_sets, h_q, nq, h_ring, ring_rows, d_ws, ws_bytes, order, stream);
}

size_t bm_db_tc_bytes(const bm_params *prm, int64_t n_sets)
{
    if (!prm || n_sets <= 0 || (prm->p != 4 && prm->p != 8)) return 0;
    return (size_t)((n_sets + TM_M - 1) / TM_M) * 2 * N * tm_a_bytes(prm->p);
}
int bm_db_tc_register(const bm_params *prm, const uint64_t *d_db, int64_t n_sets, void *d_packed, size_t bytes,
                      void *stream)
{
    if (!prm || !d_db || !d_packed || n_sets <= 0) return BM_ERR_INVALID_ARG;
    if (prm->p != 4 && prm->p != 8) return BM_ERR_INVALID_ARG;
    if (bytes < bm_db_tc_bytes(prm, n_sets)) return BM_ERR_WORKSPACE;
    DevCtx *C;
    int rc = ctx_get(&C);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n_st = (n_sets + TM_M - 1) / TM_M;
    const int64_t nthr = n_st * 2 * 16 * prm->p * (int64_t)N;
    const unsigned nblk = (unsigned)((nthr + 255) / 256);
    uint8_t *pk = reinterpret_cast<uint8_t *>(d_packed);
    if (prm->p == 8) k_tm_dbpack<8><<<nblk, 256, 0, s>>>(d_db, n_sets, n_st, pk);
    else k_tm_dbpack<4><<<nblk, 256, 0, s>>>(d_db, n_sets, n_st, pk);
    counted();
    rc = launch_check();
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g_tc_mu);
    for (TcDb &e : g_tc)
        if (e.db == d_db) {
            e = TcDb{d_db, n_sets, prm->p, pk};
            return BM_OK;
        }
    g_tc.push_back(TcDb{d_db, n_sets, prm->p, pk});
    return BM_OK;
}
int bm_db_tc_unregister(const uint64_t *d_db)
{
    std::lock_guard<std::mutex> lk(g_tc_mu);
    for (size_t i = 0; i < g_tc.size(); i++)
        if (g_tc[i].db == d_db) {
            g_tc.erase(g_tc.begin() + (long)i);
            return BM_OK;
        }
    return BM_ERR_INVALID_ARG;
}

int bm_set_option(int32_t key, int64_t value)
{
    if (key < 0 || key >= BM_OPT_COUNT_) return BM_ERR_INVALID_ARG;
    const bool flag = key == BM_OPT_LADDER_C2 || key == BM_OPT_LADDER_C3 || key == BM_OPT_LADDER_TAIL ||
                      key == BM_OPT_TENSOR_MMA;
    if (flag ? (value != 0 && value != 1) : key == BM_OPT_HOST_GROUPS ? value < 0 : value < 1) return BM_ERR_INVALID_ARG;
    g_opt[key].store(value);
    return BM_OK;
}
int64_t bm_get_option(int32_t key)
{
    if (key < 0 || key >= BM_OPT_COUNT_) return BM_ERR_INVALID_ARG;
    return opt(key);
}
int64_t bm_launch_count(void) { return g_launches.load(); }
void bm_launch_count_reset(void) { g_launches.store(0); }

int bm_sync(void *stream)
{
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "blindmatch: %s\n", cudaGetErrorString(e));
        return BM_ERR_CUDA;
    }
    return BM_OK;
}

#define BM_STR2(x) #x
#define BM_STR(x) BM_STR2(x)
// "... ; ladder: split_c0 pscale" names the throughput ladder's exact rewritings this build uses (the
// bench's algorithmic modmul count depends on them)
const char *bm_build_info(void)
{
    static const std::string info = std::string("libblindmatch sm_100a (nvcc " BM_STR(__CUDACC_VER_MAJOR__) "." BM_STR(
                                        __CUDACC_VER_MINOR__) "); ladder:") +
                                    (LADDER_SPLIT_C0 ? " split_c0" : "") + (LADDER_PSCALE ? " pscale" : "");
    return info.c_str();
}

} // extern "C"
