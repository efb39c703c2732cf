// Probe of tcgen05.mma kind::i8 (u8 x u8 -> s32) with K-major SWIZZLE_NONE shared-memory operands:
// checks the descriptor encoding (LBO = K-adjacent core matrices, SBO = M/N-adjacent 8-row groups)
// against a CPU reference.  nvcc -gencode arch=compute_100a,code=sm_100a -o umma_i8_probe umma_i8_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

constexpr int M = 128, KB = 128; // K bytes
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46; // version (sm100)
    return d;               // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}
// core-matrix offset of (row, k) in a [rows/8][KB/16][8][16] byte layout
__host__ __device__ inline int coff(int row, int k) { return ((row >> 3) * (KB / 16) + (k >> 4)) * 128 + (row & 7) * 16 + (k & 15); }

__global__ void probe(const uint8_t *A, const uint8_t *B, int32_t *out, int variant, int N)
{
    __shared__ __align__(1024) uint8_t sA[M * KB];
    __shared__ __align__(1024) uint8_t sB[256 * KB - 1024];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t s_tmem;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < M * KB; i += blockDim.x) sA[coff(i / KB, i % KB)] = A[i];
    for (int i = tid; i < N * KB; i += blockDim.x) sB[coff(i / KB, i % KB)] = B[i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    const uint32_t lbo = variant == 0 ? 128 : (KB / 16) * 128, sbo = variant == 0 ? (KB / 16) * 128 : 128;
    if (tid == 0) {
        const uint32_t idesc = (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sA), b0 = (uint32_t)__cvta_generic_to_shared(sB);
        for (int kk = 0; kk < KB / 32; kk++) {
            const uint64_t ad = sdesc(a0 + kk * 2 * 128, lbo, sbo), bd = sdesc(b0 + kk * 2 * 128, lbo, sbo);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                         "l"(ad), "l"(bd), "r"(idesc), "r"(kk));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&mbar)) : "memory");
    }
    // wait for the MMAs (phase 0)
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(&mbar)) : "memory");
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // TMEM -> registers: warp w reads lanes 32 w .. 32 w + 31, 8 columns at a time
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(tmem + ((uint32_t)(32 * warp) << 16) + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 8; j++) out[tid * N + c0 + j] = (int32_t)r[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main()
{
    std::vector<uint8_t> A(M * KB), B(256 * KB);
    srand(1);
    for (auto &x : A) x = rand() & 255;
    for (auto &x : B) x = rand() & 255;
    uint8_t *dA, *dB;
    int32_t *dO;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, B.size());
    cudaMalloc(&dO, M * 256 * 4);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    for (int N : {64, 240})
    for (int variant = 0; variant < 2; variant++) {
        cudaMemset(dO, 0, M * 256 * 4);
        probe<<<1, 128>>>(dA, dB, dO, variant, N);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<int32_t> O(M * N);
        cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int m = 0; m < M; m++)
            for (int n = 0; n < N; n++) {
                int64_t s = 0;
                for (int k = 0; k < KB; k++) s += (int)A[m * KB + k] * (int)B[n * KB + k];
                if (s != O[m * N + n]) bad++;
            }
        printf("N=%d variant %d (%s): %s, %d / %d mismatches, out[0]=%d\n", N, variant, variant == 0 ? "LBO=K-adjacent" : "swapped",
               cudaGetErrorString(e), bad, M * N, O[0]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
