// bm_host.h -- internal interface between the host C++ part (host.cpp) and the CUDA part
// (device.cu) of libblindmatch.  Not installed, not part of the C ABI.
#pragma once
#include <stdint.h>
#include <vector>
#include "blindmatch.h"

namespace bm {

// Host-side NTT tables of the product (its own choice of psi; the oracle picks its own).
struct HostPrime {
    uint64_t q;
    uint64_t psi;                 // primitive 2N-th root of unity
    std::vector<uint64_t> fwd;    // psi^brev13(k), k < N
    std::vector<uint64_t> inv;    // psi^-brev13(k)
    uint64_t ninv;                // N^-1 mod q
};
const HostPrime &host_prime(int i); // 0: q0, 1: q1, 2: P, 3: q2 (f3)
const uint64_t *host_cdt();          // 19 Gaussian CDT thresholds

uint64_t mulmod_h(uint64_t a, uint64_t b, uint64_t q);
uint64_t shoup_companion(uint64_t w, uint64_t q); // floor(w 2^64 / q)

// randomness mode (bm_rng_mode): the key extension of the keygen family (the process key in the
// OS-entropy mode, zeros when seeded) and a fresh one for an encryption call
const uint32_t *rng_keygen_kx();
void rng_encrypt_kx(uint32_t out[5]);

// host negacyclic NTT (same ordering as the device kernels)
void host_ntt_fwd(uint64_t *a, int prime);
void host_ntt_inv(uint64_t *a, int prime);

} // namespace bm

struct bm_sk {
    uint8_t digest[32];
    std::vector<int8_t> s;
};
struct bm_pk {
    uint8_t digest[32];
    std::vector<uint64_t> v; // [2][2][N]
};
struct bm_evk {
    uint8_t digest[32];
    int32_t n_rot;
    std::vector<uint64_t> rlk; // [2][2][3][N]
    std::vector<uint64_t> gk;  // [n_rot][2][2][N]
    int32_t n_hrot = 0;        // f2 hoisted rotation keys (s - 1 of them, 0 if not generated)
    std::vector<uint64_t> hgk; // [n_hrot][2][2][N], entry r-1 = rotation r
};
// f3/f4 keys: the q2 limb of pk and the level-1 Galois keys of rotations s 2^t, t < n_rot
// (log2 p for the expansion; keygen makes log2 B, which the enrollment needs)
struct bm_xk {
    uint8_t digest[32];
    int32_t d, p, n_rot;
    std::vector<uint64_t> pk_q2; // [2][N]
    std::vector<uint64_t> gk1;   // [n_rot][2 digits][2 comps][3 limbs q0,q1,P][N]
};
// f1 compression keys (reading R28)
struct bm_ck {
    uint8_t digest[32];
    int32_t d, p, log_s;
    std::vector<uint64_t> rlk2; // [3 digits][2 comps][4 limbs q0,q1,q2,P][N]
    std::vector<uint64_t> gkl;  // [log_s][2 digits][2 comps][3 limbs q0,q1,P][N]
    std::vector<uint64_t> gkc;  // [s-1][2 comps][2 limbs q0,P][N]
};
