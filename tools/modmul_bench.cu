// Modular-multiplication throughput microbenchmark (diagnostic, not part of the library;
// SURVEY.md sec. 8d "Integer-roofline microbenchmarks" 2-3): the library's own lazy Shoup product
// (ntt2.cuh shoup4<PI>, the multiply of every NTT butterfly and key-switch product) on q0, q1 and
// P, the FP64-pipe q1 product (k_match.cuh mulmod_q1_f64's arithmetic), and one forward radix-2
// butterfly (ct4s) per prime, in modmul/s over the whole GPU.  Register-resident: 8 independent
// dependency chains per thread, 2 CTAs x 512 threads per SM, every SM, ~0.2 s per kernel.
// Build: tools/build_micro.sh.  Output: one human line per kernel, then one JSON object.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2408_06167_b200/csrc/ntt2.cuh"
using namespace bm;

#define CH 8

template <int PI> __global__ void __launch_bounds__(512, 2) k_shoup(uint64_t *out, int iters, uint64_t w, uint64_t wp)
{
    uint64_t x[CH];
#pragma unroll
    for (int i = 0; i < CH; i++) x[i] = (uint64_t)(threadIdx.x * 7919 + blockIdx.x * 104729 + i) * 0x9e3779b97f4a7c15ull;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < CH; i++) x[i] = shoup4<PI>(x[i], w, wp); // any a < 2^64 -> [0, 4q)
    }
    uint64_t acc = 0;
#pragma unroll
    for (int i = 0; i < CH; i++) acc ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// forward CT butterfly of a stage that does not reduce (q0 / q1 schedule; P: the lazy schedule of
// stage 0) -- outputs fed back reduced so the chain never overflows: x + T, x - T + 4q
template <int PI> __global__ void __launch_bounds__(512, 2) k_bfly(uint64_t *out, int iters, uint64_t w, uint64_t wp)
{
    uint64_t x[CH], y[CH];
    constexpr uint64_t q = PrimeC<PI>::q;
#pragma unroll
    for (int i = 0; i < CH; i++) {
        x[i] = (uint64_t)(threadIdx.x * 31 + i) % q;
        y[i] = (uint64_t)(blockIdx.x * 17 + i * 3) % q;
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < CH; i++) {
            ct4s<PI>(x[i], y[i], make_ulonglong2(w, wp), 0);
            x[i] = reduce_lazy<PI == 1 ? 0 : PI>(x[i]);     // keep the chain bounded (an ALU op)
            y[i] = reduce_lazy<PI == 1 ? 0 : PI>(y[i]);
        }
    }
    uint64_t acc = 0;
#pragma unroll
    for (int i = 0; i < CH; i++) acc ^= x[i] ^ y[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// q1 on the FP64 pipe: hi = fl(a b), lo = fma(a, b, -hi), quotient floor by a round-down add of
// 1.5 2^52, r = fma(-qt, q1, hi) + lo (k_match.cuh mulmod_q1_f64)
__global__ void __launch_bounds__(512, 2) k_q1f(double *out, int iters, double b)
{
    constexpr double q = (double)Q1, qinv = 1.0 / (double)Q1, M = 6755399441055744.0;
    double x[CH];
#pragma unroll
    for (int i = 0; i < CH; i++) x[i] = (double)((threadIdx.x * 7919ull + i * 104729ull) % Q1);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < CH; i++) {
            const double hi = x[i] * b;
            const double lo = __fma_rn(x[i], b, -hi);
            const double qt = __dadd_rd(hi * qinv, M) - M;
            double r = __fma_rn(-qt, q, hi) + lo;        // (-3 q1, 3 q1)
            r = r < 0 ? r + q : r;                         // keep the chain in [0, 3 q1)
            x[i] = r;
        }
    }
    double acc = 0;
#pragma unroll
    for (int i = 0; i < CH; i++) acc += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

static uint64_t wp_of(uint64_t w, uint64_t q) { return (uint64_t)(((unsigned __int128)w << 64) / q); }

int main()
{
    int dev = 0, n_sm = 0, clk_khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    const int blocks = 2 * n_sm, threads = 512, iters = 1 << 14;
    uint64_t *out;
    cudaMalloc(&out, (size_t)blocks * threads * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double ops = (double)blocks * threads * CH * iters;
    double rate[8] = {0};
    const char *names[8] = {"shoup q0", "shoup q1", "shoup P", "bfly q0", "bfly q1", "bfly P", "q1 fp64", ""};
    const uint64_t Qs[3] = {Q0, Q1, QP};
    for (int k = 0; k < 7; k++) {
        const uint64_t q = Qs[k % 3], w = q / 3 + 12345, wp = wp_of(w, q);
        float best = 1e30f;
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(a);
            switch (k) {
            case 0: k_shoup<0><<<blocks, threads>>>(out, iters, w, wp); break;
            case 1: k_shoup<1><<<blocks, threads>>>(out, iters, w, wp); break;
            case 2: k_shoup<2><<<blocks, threads>>>(out, iters, w, wp); break;
            case 3: k_bfly<0><<<blocks, threads>>>(out, iters, w, wp); break;
            case 4: k_bfly<1><<<blocks, threads>>>(out, iters, w, wp); break;
            case 5: k_bfly<2><<<blocks, threads>>>(out, iters, w, wp); break;
            case 6: k_q1f<<<blocks, threads>>>((double *)out, iters, (double)(Q1 / 3 + 12345)); break;
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        cudaError_t e = cudaGetLastError();
        rate[k] = ops / (best / 1e3) / 1e9;
        printf("%-10s %8.3f ms  %8.1f G/s  (%.2f per clk per SM at %d MHz)  %s\n", names[k], best, rate[k],
               rate[k] * 1e9 / (n_sm * clk_khz * 1e3), clk_khz / 1000, cudaGetErrorString(e));
    }
    // the integer roofline of the hot path: the slowest 64-bit prime's Shoup product (q0 / P limbs
    // carry every transform of the ladder and the key switches)
    double peak = rate[0] < rate[2] ? rate[0] : rate[2];
    printf("{\"gmodmul_s\": %.1f, \"shoup_q0\": %.1f, \"shoup_q1\": %.1f, \"shoup_P\": %.1f, \"bfly_q0\": %.1f, "
           "\"bfly_q1\": %.1f, \"bfly_P\": %.1f, \"q1_fp64\": %.1f, \"n_sm\": %d, \"clock_mhz\": %d, "
           "\"basis\": \"tools/modmul_bench.cu: min(Shoup q0, Shoup P) lazy modmul/s, register-resident, 8 chains x "
           "512 threads x 2 CTAs per SM, all SMs, best of 3\"}\n",
           peak, rate[0], rate[1], rate[2], rate[3], rate[4], rate[5], rate[6], n_sm, clk_khz / 1000);
    return 0;
}
