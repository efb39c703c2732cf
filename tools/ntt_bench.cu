// NTT throughput microbenchmark (diagnostic, not part of the library):
// each CTA runs `iters` x (forward + inverse) 8192-point transforms on one polynomial held in
// registers/shared memory, for each of the three primes; checks the round trip is the identity.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../paper_2408_06167_b200/csrc/bm_common.cuh"
#include "../paper_2408_06167_b200/csrc/bm_host.h"
#include "../paper_2408_06167_b200/csrc/ntt3.cuh"
#include "../paper_2408_06167_b200/csrc/ntt3f.cuh"
#include "ntt_legacy.cuh"
#include "ntt_experiments.cuh"
using namespace bm;
typedef unsigned __int128 u128;

#ifndef MINB
#define MINB 2
#endif
template <int V, int PI>
__global__ void __launch_bounds__(256, MINB) k_bench(PrimeK P, uint64_t *data, int iters)
{
    extern __shared__ uint64_t sm[];
    uint64_t a[32];
    uint64_t *d = data + (size_t)blockIdx.x * N;
#pragma unroll
    for (int e = 0; e < 32; e++) a[e] = d[j_L1(threadIdx.x, e)];
    for (int it = 0; it < iters; it++) {
        if (V == 1) {
            ntt_fwd(a, sm, P);
            ntt_inv(a, sm, P);
        } else {
            ntt_fwd2<PI>(a, sm, P);
            ntt_inv2<PI>(a, sm, P);
        }
    }
#pragma unroll
    for (int e = 0; e < 32; e++) d[j_L1(threadIdx.x, e)] = a[e];
}

#ifndef MINB3
#define MINB3 2
#endif
template <int PI>
__global__ void __launch_bounds__(512, MINB3) k_bench3(PrimeK P, uint64_t *data, int iters)
{
    extern __shared__ uint64_t sm[];
    uint64_t a[16];
    uint64_t *d = data + (size_t)blockIdx.x * N;
    v3::load_coef(a, d);
    for (int it = 0; it < iters; it++) {
        if constexpr (PI == 3) { // q1 on the FP64 pipe (ntt3f.cuh)
            v3::fwd_f<1>(a, sm, P.fwdf);
            v3::inv_f<1>(a, sm, P.invf, P.ninvf, P.ninv_w1f);
        } else {
            v3::fwd<PI>(a, sm, P);
            v3::inv<PI>(a, sm, P);
        }
    }
    v3::store_coef(d, a);
}

// two polynomials per CTA through the dual transforms (ntt3.cuh fwd2x / inv2x); the butterfly count
// of one launch is 2x that of k_bench3 with the same grid
template <int PI>
__global__ void __launch_bounds__(512, 1) k_bench3x2(PrimeK P, uint64_t *data, int iters)
{
    extern __shared__ uint64_t sm[];
    uint64_t a[16], b[16];
    uint64_t *d = data + (size_t)blockIdx.x * 2 * N;
    v3::load_coef(a, d);
    v3::load_coef(b, d + N);
    for (int it = 0; it < iters; it++) {
        v3::fwd2x<PI>(a, b, sm, sm + SMEM_WORDS, P);
        v3::inv2x<PI>(a, b, sm, sm + SMEM_WORDS, P);
    }
    v3::store_coef(d, a);
    v3::store_coef(d + N, b);
}

// hybrid: one integer-prime polynomial (PI) and one q1 polynomial on the FP64 pipe per CTA (fwd_h / inv_h)
template <int PI>
__global__ void __launch_bounds__(512, 1) k_bench3h(PrimeK P, PrimeK P1, uint64_t *data, int iters)
{
    extern __shared__ uint64_t sm[];
    uint64_t a[16], b[16];
    uint64_t *d = data + (size_t)blockIdx.x * 2 * N;
    v3::load_coef(a, d);
    v3::load_coef(b, d + N);
    for (int it = 0; it < iters; it++) {
        v3::fwd_h<PI, true, 1>(a, b, sm, sm + SMEM_WORDS, P, P1.fwdf);
        v3::inv_h<PI, 1>(a, b, sm, sm + SMEM_WORDS, P, P1.invf, P1.ninvf, P1.ninv_w1f);
    }
    v3::store_coef(d, a);
    v3::store_coef(d + N, b);
}

// v7: 1,024 threads x 8 coefficients (tools/ntt_experiments.cuh x10), natural-order twiddle tables
template <int PI>
__global__ void __launch_bounds__(1024, 1) k_bench10(PrimeK P, uint64_t *data, int iters)
{
    extern __shared__ uint64_t sm[];
    uint64_t a[8];
    uint64_t *d = data + (size_t)blockIdx.x * N;
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = d[threadIdx.x + 1024 * k];
    for (int it = 0; it < iters; it++) {
        v3::x10::fwd10<PI>(a, sm, P.fwd);
        v3::x10::inv10<PI>(a, sm, P.inv, P.ninv, P.ninv_w1);
    }
#pragma unroll
    for (int k = 0; k < 8; k++) d[threadIdx.x + 1024 * k] = a[k];
}

static ulonglong2 sp(uint64_t w, uint64_t q) { return make_ulonglong2(w, shoup_companion(w, q)); }

int main(int argc, char **argv)
{
    int blocks = argc > 1 ? atoi(argv[1]) : 296 * 4;
    int iters = argc > 2 ? atoi(argv[2]) : 20;
    const size_t SM_BYTES = argc > 3 ? (size_t)atoi(argv[3]) : SMEM_WORDS * 8; // larger: less L1 left for twiddles
    typedef void (*KF)(PrimeK, uint64_t *, int);
    KF kf[4][3] = {{k_bench<1, 0>, k_bench<1, 1>, k_bench<1, 2>}, {k_bench<2, 0>, k_bench<2, 1>, k_bench<2, 2>},
                   {k_bench3<0>, k_bench3<1>, k_bench3<2>}, {k_bench3<3>, k_bench3<3>, k_bench3<3>}};
    for (int v = 0; v < 4; v++)
        for (int i = 0; i < 3; i++) cudaFuncSetAttribute(kf[v][i], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_BYTES);
    KF kx2[3] = {k_bench3x2<0>, k_bench3x2<1>, k_bench3x2<2>};
    for (int i = 0; i < 3; i++) cudaFuncSetAttribute(kx2[i], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * SMEM_WORDS * 8));
    for (int v = 1; v < 5; v++)
    for (int pi = 0; pi < 3; pi++) {
        if (v == 3 && pi != 1) continue; // v4 = q1 on the FP64 pipe
        if (v == 4 && pi == 1) continue; // v5 = dual transforms (q0, P)
        const HostPrime &H = host_prime(pi);
        std::vector<ulonglong2> tw(2 * N);
        // v1/v2 cores index the tables directly; the v3 cores (ntt3.cuh) read them in load order (tw_pos)
        for (int k = 0; k < N; k++) {
            const int pos = v >= 2 ? v3::tw_pos(k) : k;
            tw[pos] = sp(H.fwd[k], H.q), tw[N + pos] = sp(H.inv[k], H.q);
        }
        ulonglong2 *dtw;
        cudaMalloc(&dtw, tw.size() * 16);
        cudaMemcpy(dtw, tw.data(), tw.size() * 16, cudaMemcpyHostToDevice);
        PrimeK P;
        P.q = H.q; P.q2 = 2 * H.q; P.fwd = dtw; P.inv = dtw + N;
        P.ninv = sp(H.ninv, H.q);
        P.ninv_w1 = sp(mulmod_h(H.ninv, H.inv[1], H.q), H.q);
        P.r64 = sp((uint64_t)(((u128)1 << 64) % H.q), H.q);
        P.one_p = (uint64_t)(((u128)1 << 64) / H.q);
        ulonglong2 *dtwf = nullptr;
        if (v == 3) { // (w, fl(w / q1)) as doubles
            auto fp = [](uint64_t w) { double a = (double)w, b = a / (double)Q1; uint64_t x, y;
                                       memcpy(&x, &a, 8); memcpy(&y, &b, 8); return make_ulonglong2(x, y); };
            std::vector<ulonglong2> tf(2 * N);
            for (int k = 0; k < N; k++) tf[v3::tw_pos(k)] = fp(H.fwd[k]), tf[N + v3::tw_pos(k)] = fp(H.inv[k]);
            cudaMalloc(&dtwf, tf.size() * 16);
            cudaMemcpy(dtwf, tf.data(), tf.size() * 16, cudaMemcpyHostToDevice);
            P.fwdf = dtwf; P.invf = dtwf + N;
            P.ninvf = fp(H.ninv); P.ninv_w1f = fp(mulmod_h(H.ninv, H.inv[1], H.q));
        }
        const int per = v == 4 ? 2 : 1;                  // polynomials per CTA
        std::vector<uint64_t> h((size_t)blocks * N * per);
        srand(pi + 1);
        for (auto &x : h) x = (((uint64_t)rand() << 40) ^ ((uint64_t)rand() << 20) ^ rand()) % H.q;
        uint64_t *dd;
        cudaMalloc(&dd, h.size() * 8);
        cudaMemcpy(dd, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        KF k = v == 4 ? kx2[pi] : kf[v][pi];
        const int thr = v >= 2 ? 512 : 256;
        const size_t smb = v == 4 ? 2 * SMEM_WORDS * 8 : SM_BYTES;
        k<<<blocks, thr, smb>>>(P, dd, 1); // warm-up (+ round trip)
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<blocks, thr, smb>>>(P, dd, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        std::vector<uint64_t> back(h.size());
        cudaMemcpy(back.data(), dd, h.size() * 8, cudaMemcpyDeviceToHost);
        bool ok = back == h;
        double bfly = (double)blocks * per * iters * 2 * (N / 2) * LOGN;
        int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        printf("v%d prime %d: %s  %.3f ms  %.1f Gbfly/s  %.2f bfly/clk/SM (at %d MHz)  err=%s\n", v + 1, pi, ok ? "ok" : "MISMATCH", ms,
               bfly / ms / 1e6, bfly / (ms * 1e-3) / (148.0 * clk * 1e3), clk / 1000, cudaGetErrorString(cudaGetLastError()));
        cudaFree(dd); cudaFree(dtw); cudaFree(dtwf);
    }
    // v6: hybrid pairs (an integer-prime transform interleaved with a q1 transform on the FP64 pipe)
    auto mk = [&](int pi, bool fp) {
        const HostPrime &H = host_prime(pi);
        std::vector<ulonglong2> tw(2 * N);
        for (int k = 0; k < N; k++) tw[v3::tw_pos(k)] = sp(H.fwd[k], H.q), tw[N + v3::tw_pos(k)] = sp(H.inv[k], H.q);
        ulonglong2 *dtw;
        cudaMalloc(&dtw, tw.size() * 16);
        cudaMemcpy(dtw, tw.data(), tw.size() * 16, cudaMemcpyHostToDevice);
        PrimeK P;
        P.q = H.q; P.q2 = 2 * H.q; P.fwd = dtw; P.inv = dtw + N;
        P.ninv = sp(H.ninv, H.q);
        P.ninv_w1 = sp(mulmod_h(H.ninv, H.inv[1], H.q), H.q);
        P.r64 = sp((uint64_t)(((u128)1 << 64) % H.q), H.q);
        P.one_p = (uint64_t)(((u128)1 << 64) / H.q);
        if (fp) {
            auto fpp = [&](uint64_t w) { double a = (double)w, b = a / (double)H.q; uint64_t x, y;
                                         memcpy(&x, &a, 8); memcpy(&y, &b, 8); return make_ulonglong2(x, y); };
            std::vector<ulonglong2> tf(2 * N);
            for (int k = 0; k < N; k++) tf[v3::tw_pos(k)] = fpp(H.fwd[k]), tf[N + v3::tw_pos(k)] = fpp(H.inv[k]);
            ulonglong2 *dtwf;
            cudaMalloc(&dtwf, tf.size() * 16);
            cudaMemcpy(dtwf, tf.data(), tf.size() * 16, cudaMemcpyHostToDevice);
            P.fwdf = dtwf; P.invf = dtwf + N;
            P.ninvf = fpp(H.ninv); P.ninv_w1f = fpp(mulmod_h(H.ninv, H.inv[1], H.q));
        }
        return P;
    };
    const PrimeK P1 = mk(1, true);
    typedef void (*KH)(PrimeK, PrimeK, uint64_t *, int);
    KH kh[2] = {k_bench3h<0>, k_bench3h<2>};
    for (int i = 0; i < 2; i++) {
        cudaFuncSetAttribute(kh[i], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * SMEM_WORDS * 8));
        const int pi = i ? 2 : 0;
        const PrimeK P = mk(pi, false);
        std::vector<uint64_t> h((size_t)blocks * 2 * N);
        srand(pi + 7);
        for (size_t b = 0; b < (size_t)blocks; b++)
            for (int k = 0; k < 2 * N; k++)
                h[b * 2 * N + k] = (((uint64_t)rand() << 40) ^ ((uint64_t)rand() << 20) ^ rand()) % (k < N ? P.q : Q1);
        uint64_t *dd;
        cudaMalloc(&dd, h.size() * 8);
        cudaMemcpy(dd, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        kh[i]<<<blocks, 512, 2 * SMEM_WORDS * 8>>>(P, P1, dd, 1);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        kh[i]<<<blocks, 512, 2 * SMEM_WORDS * 8>>>(P, P1, dd, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        std::vector<uint64_t> back(h.size());
        cudaMemcpy(back.data(), dd, h.size() * 8, cudaMemcpyDeviceToHost);
        const bool ok = back == h;
        const double bfly = (double)blocks * 2 * iters * 2 * (N / 2) * LOGN;
        int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        printf("v6 hybrid prime %d + q1 fp64: %s  %.3f ms  %.1f Gbfly/s  %.2f bfly/clk/SM (at %d MHz)  err=%s\n", pi,
               ok ? "ok" : "MISMATCH", ms, bfly / ms / 1e6, bfly / (ms * 1e-3) / (148.0 * clk * 1e3), clk / 1000,
               cudaGetErrorString(cudaGetLastError()));
        cudaFree(dd);
    }
    // v7: 1,024-thread core, natural-order twiddles
    typedef void (*KT)(PrimeK, uint64_t *, int);
    KT k10[3] = {k_bench10<0>, k_bench10<1>, k_bench10<2>};
    for (int pi = 0; pi < 3; pi++) {
        cudaFuncSetAttribute(k10[pi], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(SMEM_WORDS * 8));
        const HostPrime &H = host_prime(pi);
        std::vector<ulonglong2> tw(2 * N);
        for (int k = 0; k < N; k++) tw[k] = sp(H.fwd[k], H.q), tw[N + k] = sp(H.inv[k], H.q);
        ulonglong2 *dtw;
        cudaMalloc(&dtw, tw.size() * 16);
        cudaMemcpy(dtw, tw.data(), tw.size() * 16, cudaMemcpyHostToDevice);
        PrimeK P;
        P.q = H.q; P.q2 = 2 * H.q; P.fwd = dtw; P.inv = dtw + N;
        P.ninv = sp(H.ninv, H.q);
        P.ninv_w1 = sp(mulmod_h(H.ninv, H.inv[1], H.q), H.q);
        std::vector<uint64_t> h((size_t)blocks * N);
        srand(pi + 11);
        for (auto &x : h) x = (((uint64_t)rand() << 40) ^ ((uint64_t)rand() << 20) ^ rand()) % H.q;
        uint64_t *dd;
        cudaMalloc(&dd, h.size() * 8);
        cudaMemcpy(dd, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        k10[pi]<<<blocks, 1024, SMEM_WORDS * 8>>>(P, dd, 1);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k10[pi]<<<blocks, 1024, SMEM_WORDS * 8>>>(P, dd, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        std::vector<uint64_t> back(h.size());
        cudaMemcpy(back.data(), dd, h.size() * 8, cudaMemcpyDeviceToHost);
        const bool ok = back == h;
        const double bfly = (double)blocks * iters * 2 * (N / 2) * LOGN;
        int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        printf("v7 1024x8 prime %d: %s  %.3f ms  %.1f Gbfly/s  %.2f bfly/clk/SM (at %d MHz)  err=%s\n", pi,
               ok ? "ok" : "MISMATCH", ms, bfly / ms / 1e6, bfly / (ms * 1e-3) / (148.0 * clk * 1e3), clk / 1000,
               cudaGetErrorString(cudaGetLastError()));
        cudaFree(dd); cudaFree(dtw);
    }
    return 0;
}
