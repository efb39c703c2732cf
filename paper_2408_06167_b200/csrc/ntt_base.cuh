// ntt_base.cuh -- definitions shared by the NTT cores of the library (ntt3.cuh, ntt3f.cuh) and
// its kernels: the padded shared-memory exchange buffer, the twiddle load, the 13-bit bit reversal.
// (The superseded v1 / v2 transform cores live in tools/ntt_legacy.cuh, used only by the
// tools/ntt_bench.cu microbenchmark.)
#pragma once
#include "bm_common.cuh"

namespace bm {

constexpr int SMEM_WORDS = N + N / 16; // 8704 u64 = 69,632 B: one word of padding per 16

BM_D int pidx(int j) { return j + (j >> 4); }

#if defined(BM_DIAG_TW) // tools/ntt_bench.cu diagnostic builds only (wrong results): twiddles as constant-bank operands, no loads
__constant__ ulonglong2 c_diag_tw;
BM_D ulonglong2 ldtw(const ulonglong2 *) { return c_diag_tw; }
#else
BM_D ulonglong2 ldtw(const ulonglong2 *p) { return __ldg(p); }
#endif

BM_D int brev13(int x) { return (int)(__brev((unsigned)x) >> 19); }

} // namespace bm
