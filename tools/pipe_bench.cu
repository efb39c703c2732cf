// Pipe-throughput microbenchmark (diagnostic): warp instructions per clock per SM for the integer
// and FP64 instructions the modular arithmetic can use, alone and mixed, on sm_100a.
// Each thread runs 8 independent dependency chains; 2 CTAs x 512 threads per SM.
#include <cstdio>
#include <cstdint>

#define ITERS 4096
#define CH 8

template <int OP>
__global__ void __launch_bounds__(512) k(uint64_t *out, uint32_t s0)
{
    uint32_t a[CH], b[CH];
    double f[CH], g[CH];
#pragma unroll
    for (int i = 0; i < CH; i++) {
        a[i] = s0 + threadIdx.x * 7 + i;
        b[i] = a[i] * 3 + 1;
        f[i] = (double)a[i] * 1.0000001;
        g[i] = 0.999999;
    }
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int i = 0; i < CH; i++) {
            if (OP == 0) asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(a[i]) : "r"(b[i]));
            if (OP == 1) {
                uint64_t w;
                asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "=l"(w) : "r"(a[i]), "r"(b[i]));
                a[i] ^= (uint32_t)w;
            }
            if (OP == 2) asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(a[i]) : "r"(b[i]));
            if (OP == 3) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i]));
            if (OP == 4) asm volatile("fma.rn.f64 %0, %0, %1, %0;" : "+d"(f[i]) : "d"(g[i]));
            if (OP == 5) { // IMAD + DFMA interleaved
                asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(a[i]) : "r"(b[i]));
                asm volatile("fma.rn.f64 %0, %0, %1, %0;" : "+d"(f[i]) : "d"(g[i]));
            }
            if (OP == 6) { // IMAD + IADD interleaved
                asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(a[i]) : "r"(b[i]));
                asm volatile("add.u32 %0, %0, %1;" : "+r"(b[i]) : "r"(a[i]));
            }
            if (OP == 7) { // DFMA + IADD
                asm volatile("fma.rn.f64 %0, %0, %1, %0;" : "+d"(f[i]) : "d"(g[i]));
                asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i]));
            }
            if (OP == 8) { // 3-way: IMAD + DFMA + IADD
                asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(a[i]) : "r"(b[i]));
                asm volatile("fma.rn.f64 %0, %0, %1, %0;" : "+d"(f[i]) : "d"(g[i]));
                asm volatile("add.u32 %0, %0, %1;" : "+r"(b[i]) : "r"(a[i]));
            }
            if (OP == 9) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(f[i]) : "d"(g[i]));
            if (OP == 10) { // cvt u64 -> f64
                double t;
                asm volatile("cvt.rn.f64.u64 %0, %1;" : "=d"(t) : "l"((uint64_t)a[i] << 20));
                f[i] += t;
            }
            if (OP == 11) asm volatile("cvt.rmi.f64.f64 %0, %0;" : "+d"(f[i]));
            if (OP == 13) { // 64-bit add with carry: IADD3 + IADD3.X
                uint64_t t = ((uint64_t)b[i] << 32) | a[i];
                asm volatile("add.u64 %0, %0, %1;" : "+l"(t) : "l"(((uint64_t)a[i] << 32) | b[i]));
                a[i] = (uint32_t)t; b[i] = (uint32_t)(t >> 32);
            }
            if (OP == 14) asm volatile("shf.l.wrap.b32 %0, %0, %1, 13;" : "+r"(a[i]) : "r"(b[i]));
            if (OP == 15) asm volatile("lop3.b32 %0, %0, %1, %0, 0x96;" : "+r"(a[i]) : "r"(b[i]));
            if (OP == 16) { // setp + selp
                uint32_t t;
                asm volatile("{.reg .pred p; setp.gt.u32 p, %1, %2; selp.u32 %0, %1, %2, p;}" : "=r"(t) : "r"(a[i]), "r"(b[i]));
                a[i] = t + 1;
            }
            if (OP == 17) { // IMAD.WIDE alone (chain through the 64-bit accumulator)
                asm volatile("{.reg .u64 w; mov.b64 w, {%0, %1}; mad.wide.u32 w, %0, %1, w; mov.b64 {%0, %1}, w;}" : "+r"(a[i]), "+r"(b[i]));
            }
            if (OP == 18) { // I2F.F64.U32 (+DADD to consume)
                double t;
                asm volatile("cvt.rn.f64.u32 %0, %1;" : "=d"(t) : "r"(a[i]));
                f[i] += t; a[i] += 1;
            }
            if (OP == 19) { // F2I.S64.F64 floor (+IADD)
                uint64_t t;
                asm volatile("cvt.rmi.s64.f64 %0, %1;" : "=l"(t) : "d"(f[i]));
                a[i] += (uint32_t)t; f[i] += 1.0;
            }
            if (OP == 20) { // DADD.RM (magic floor)
                asm volatile("add.rm.f64 %0, %0, %1;" : "+d"(f[i]) : "d"(g[i]));
            }
            if (OP == 12) { // f64 -> u64
                uint64_t t;
                asm volatile("cvt.rzi.u64.f64 %0, %1;" : "=l"(t) : "d"(f[i]));
                a[i] += (uint32_t)t;
            }
        }
    }
    uint64_t r = 0;
#pragma unroll
    for (int i = 0; i < CH; i++) r += a[i] + b[i] + (uint64_t)f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int OP> void run(const char *name, int ninst, uint64_t *d)
{
    const int blocks = 148 * 2 * 4;
    k<OP><<<blocks, 512>>>(d, 1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<OP><<<blocks, 512>>>(d, 2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double warp_inst = (double)blocks * 16 * ITERS * CH * ninst;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-28s %7.3f ms  %6.3f warp-inst/clk/SM (%5.1f lanes/clk/SM)  %s\n", name, ms, warp_inst / cyc / 148,
           warp_inst / cyc / 148 * 32, cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    uint64_t *d;
    cudaMalloc(&d, 148 * 8 * 512 * 8);
    run<0>("IMAD (mad.lo.u32)", 1, d);
    run<1>("IMAD.WIDE (+LOP)", 1, d);
    run<2>("IMAD.HI", 1, d);
    run<3>("IADD", 1, d);
    run<4>("DFMA", 1, d);
    run<9>("DMUL", 1, d);
    run<5>("IMAD + DFMA", 2, d);
    run<6>("IMAD + IADD", 2, d);
    run<7>("DFMA + IADD", 2, d);
    run<8>("IMAD + DFMA + IADD", 3, d);
    run<13>("u64 add (IADD3+IADD3.X)", 2, d);
    run<14>("SHF funnel", 1, d);
    run<15>("LOP3", 1, d);
    run<16>("ISETP+SEL(+IADD)", 3, d);
    run<17>("IMAD.WIDE (acc chain)", 1, d);
    run<10>("cvt f64<-u64 (+DADD)", 1, d);
    run<11>("cvt.rmi f64 (floor)", 1, d);
    run<12>("cvt u64<-f64 (+IADD)", 1, d);
    run<18>("I2F.F64.U32 (+DADD +IADD)", 1, d);
    run<19>("F2I.S64.F64 floor (+IADD +DADD)", 1, d);
    run<20>("DADD.RM", 1, d);
    return 0;
}
