// store-only bandwidth probes (8 GiB), CUDA events, best of 10
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__global__ void k_v2(u64 *o, u64 n) {  // 16 B per lane, coalesced grid-stride
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x, st = (u64)gridDim.x * blockDim.x;
  for (; 2 * i < n; i += st) asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(o + 2 * i), "l"(i), "l"(i) : "memory");
}
__global__ void k_v4(u64 *o, u64 n) {  // 32 B per lane
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x, st = (u64)gridDim.x * blockDim.x;
  for (; 4 * i < n; i += st) asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(o + 4 * i), "l"(i), "l"(i), "l"(i), "l"(i) : "memory");
}
__global__ void k_v4cs(u64 *o, u64 n) {  // 32 B per lane, streaming hint
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x, st = (u64)gridDim.x * blockDim.x;
  for (; 4 * i < n; i += st) asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(o + 4 * i), "l"(i), "l"(i), "l"(i), "l"(i) : "memory");
}
__global__ void k_seg(u64 *o, u64 n, u64 L) {  // per-thread contiguous segment, 32 B per store (like emit)
  u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  u64 a = t * L, b = a + L < n ? a + L : n;
  for (u64 i = a; i + 4 <= b; i += 4) asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(o + i), "l"(i), "l"(i), "l"(i), "l"(i) : "memory");
}
__global__ void k_seg8(u64 *o, u64 n, u64 L) {  // per-thread contiguous segment, 8 B stores
  u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  u64 a = t * L, b = a + L < n ? a + L : n;
  for (u64 i = a; i < b; i++) o[i] = i;
}
int main() {
  u64 n = 1ULL << 30; u64 *o; cudaMalloc(&o, n * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char *name, auto f) {
    float best = 1e9;
    for (int r = 0; r < 10; r++) { cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms; }
    printf("%-28s %.3f ms  %.1f GB/s  (%s)\n", name, best, n * 8 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  run("memset", [&] { cudaMemsetAsync(o, 1, n * 8); });
  for (int bpsm : {2, 4, 8, 16}) {
    char nm[64];
    sprintf(nm, "v2 grid=%dx%d", sms, bpsm); run(nm, [&] { k_v2<<<sms * bpsm, 256>>>(o, n); });
    sprintf(nm, "v4 grid=%dx%d", sms, bpsm); run(nm, [&] { k_v4<<<sms * bpsm, 256>>>(o, n); });
    sprintf(nm, "v4cs grid=%dx%d", sms, bpsm); run(nm, [&] { k_v4cs<<<sms * bpsm, 256>>>(o, n); });
  }
  for (u64 T : {75776ULL, 151552ULL, 303104ULL}) {
    char nm[64]; u64 L = ((n + T - 1) / T + 3) / 4 * 4;
    sprintf(nm, "seg32B T=%llu", T); run(nm, [&] { k_seg<<<(T + 255) / 256, 256>>>(o, n, L); });
    sprintf(nm, "seg8B T=%llu", T); run(nm, [&] { k_seg8<<<(T + 255) / 256, 256>>>(o, n, L); });
  }
  return 0;
}
