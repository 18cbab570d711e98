// Internal declarations shared by the host engine math (rs_host.cpp) and the
// CUDA fill path (rs_fill.cu). Not part of the C ABI.
#pragma once
#include <cstdint>
#include <string>

#include "../../include/randstream_b200.h"

namespace rs {

typedef unsigned __int128 u128;

// ---- error slot (rng.py:38-52 semantics: success clears, failure records)
void set_error(const std::string &msg);
void clear_error();

// ---- engine metadata (engines/*.py class attributes)
int state_words(int eng);
int seed_words(int eng);
int chunk(int eng);
bool known_engine(int eng);
bool simd_engine(int eng);
void engine_simd_from_base(int eng, uint64_t *state);  // lanes 1..7 from lane 0
bool device_engine(int eng);

// ---- GF(2) 256x256 matrices for the xoshiro256 linear step (jumps.py:93-126 restated
// as matrix powers). Column-major: col[j] = M * e_j (4 x u64).
struct Mat256 {
    uint64_t col[256][4];
};
const Mat256 &x256_pow2(int k);  // T^(2^k), 0 <= k < 256
void mat_vec(const Mat256 &m, const uint64_t in[4], uint64_t out[4]);
void mat_mul(const Mat256 &a, const Mat256 &b, Mat256 &out);  // out = a*b
void x256_advance(uint64_t s[4], u128 n);                      // n steps
void x256_step_host(uint64_t s[4]);
// xorshift128+ / xoroshiro128: T^(2^k) as 256-bit matrices with words 2, 3 zero (k < 128)
const Mat256 &x128_pow2(int engine, int k);
void x128_advance(int engine, uint64_t s[2], u128 n);

// ---- PCG64-DXSM LCG (pcg.py:41-55)
static const uint64_t PCG_MULT = 0xDA942042E4DD58B5ULL;
void pcg_affine(u128 inc, u128 n, u128 &mul, u128 &add);  // state' = mul*state + add after n steps
void pcg_advance(uint64_t s[4], u128 n);

// ---- Philox-4x64 counter (counter.py:108-121)
void philox_add(uint64_t ctr[4], u128 blocks);

// ---- ranlux++ 576-bit LCG (ranlux.py:16-61)
void rlx_mulmod(const uint64_t *x, const uint64_t *y, uint64_t *out);
void rlx_pow_A(u128 e, uint64_t *out);         // A^e mod m
void rlx_pow2k_A(int k, uint64_t *out);        // A^(2^k) mod m
const uint64_t *rlx_modulus();
void rlx_reduce_seed(const uint64_t *w, uint64_t *out);

// ---- generic
void engine_generate(int eng, uint64_t *state, uint64_t *out, int n);
// advance the engine by `words` output words (words % chunk == 0)
bool engine_advance_words(int eng, uint64_t *state, u128 words);
void seed_words_fe128(const uint64_t *ent, int nent, const uint64_t *spawn, int nspawn,
                      uint64_t *out, int nout);
void engine_seed_from(int eng, const uint64_t *w, uint64_t *state);

}  // namespace rs
