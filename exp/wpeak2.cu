// store-pattern probes for per-lane segmented output (8 GiB): no generation, values = index
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64; typedef unsigned int u32;
// per-lane segments of L words (aligned to C); chunk of C words per lane written as
// whole-warp instructions: each instruction writes 512 B = 32 lanes x 16 B covering
// 512/(8C) lanes' chunks (C=64: one lane's chunk; C=16: four lanes' chunks)
template <int C>
__global__ void k_tile(u64 *o, u64 n, u64 L) {
  u32 lane = threadIdx.x & 31;
  u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  u64 a = t * L, b = a + L < n ? a + L : n;
  if (a > n) a = n;
  u64 nch = (b - a) / C;
  u64 maxc = nch;
  for (int s = 16; s; s >>= 1) { u64 v = __shfl_xor_sync(~0u, maxc, s); maxc = v > maxc ? v : maxc; }
  constexpr int LPI = 64 / C;  // lanes' chunks per instruction (C*8 B each, 512 B per instruction)
  constexpr int TPL = 32 / LPI;  // threads per chunk
  for (u64 k = 0; k < maxc; k++) {
    u64 dst = k < nch ? (u64)(uintptr_t)(o + a + k * C) : 0;
#pragma unroll
    for (int g = 0; g < 32 / LPI; g++) {
      u32 r = LPI * g + lane / TPL, c = lane % TPL;
      u64 d = __shfl_sync(~0u, dst, r);
      if (d) asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(d + 16 * c), "l"(d), "l"(d) : "memory");
    }
  }
}
// warp-contiguous lockstep: lane i writes word i*Ls + k of its warp region (Ls words per lane)
__global__ void k_lock(u64 *o, u64 n, u64 Ls) {
  u32 lane = threadIdx.x & 31;
  u64 w = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 base = w * 32 * Ls; base < n; base += nw * 32 * Ls)
    for (u64 k = 0; k < Ls; k += 4) {
      u64 i = base + lane * Ls + k;
      if (i + 4 <= n) asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(o + i), "l"(i), "l"(i), "l"(i), "l"(i) : "memory");
    }
}
int main() {
  u64 n = 1ULL << 30; u64 *o; cudaMalloc(&o, n * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char *name, auto f) {
    float best = 1e9;
    for (int r = 0; r < 8; r++) { cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms; }
    printf("%-34s %.3f ms  %.1f GB/s  (%s)\n", name, best, n * 8 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  for (u64 T : {18944ULL, 37888ULL, 75776ULL, 151552ULL}) {
    char nm[64];
    u64 L16 = ((n + T - 1) / T + 15) / 16 * 16, L64 = ((n + T - 1) / T + 63) / 64 * 64;
    sprintf(nm, "tile C=16 T=%llu", T); run(nm, [&] { k_tile<16><<<(T + 255) / 256, 256>>>(o, n, L16); });
    sprintf(nm, "tile C=32 T=%llu", T); run(nm, [&] { k_tile<32><<<(T + 255) / 256, 256>>>(o, n, L64); });
    sprintf(nm, "tile C=64 T=%llu", T); run(nm, [&] { k_tile<64><<<(T + 255) / 256, 256>>>(o, n, L64); });
  }
  for (u64 Ls : {4ULL, 16ULL, 64ULL, 256ULL, 1024ULL}) {
    for (int bpsm : {4, 8}) {
      char nm[64]; sprintf(nm, "lock Ls=%llu grid=%dx%d", Ls, sms, bpsm);
      run(nm, [&] { k_lock<<<sms * bpsm, 256>>>(o, n, Ls); });
    }
  }
  return 0;
}
