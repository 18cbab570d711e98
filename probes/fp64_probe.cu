// FP64 throughput probe (B200): DMMA shapes vs DFMA, all from registers.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>  // 0: m8n8k4, 1: m16n8k4, 2: m16n8k8, 3: m16n8k16
__global__ void k_dmma(double *out, int iters) {
    double a[8], b[4], c[4][4];
    for (int i = 0; i < 8; i++) a[i] = 1.0 + threadIdx.x * 1e-9 + i;
    for (int i = 0; i < 4; i++) b[i] = 1.0 - threadIdx.x * 1e-9 + i;
    for (int j = 0; j < 4; j++)
        for (int i = 0; i < 4; i++) c[j][i] = 0.0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int j = 0; j < 4; j++) {
            if constexpr (SHAPE == 0) {
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a[0]), "d"(b[0]));
            } else if constexpr (SHAPE == 1) {
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
            } else if constexpr (SHAPE == 2) {
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
            } else {
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                             : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                               "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
            }
        }
    }
    double s = 0;
    for (int j = 0; j < 4; j++)
        for (int i = 0; i < 4; i++) s += c[j][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double *out, int iters) {
    double x[8], y = 1.0 + threadIdx.x * 1e-9, z = 0.999999;
    for (int i = 0; i < 8; i++) x[i] = i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = fma(x[k], z, y);
    }
    double s = 0;
    for (int i = 0; i < 8; i++) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F>
double time_it(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 1 << 26);
    const int iters = 4096;
    const double fma_per_mma[4] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 16 * 8 * 16};
    const char *names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
    for (int wpb : {4, 8, 16}) {
        for (int bps : {1, 2, 4}) {
            int grid = sms * bps, block = 32 * wpb;
            for (int s = 0; s < 4; s++) {
                double ms = time_it([&] {
                    if (s == 0) k_dmma<0><<<grid, block>>>(out, iters);
                    if (s == 1) k_dmma<1><<<grid, block>>>(out, iters);
                    if (s == 2) k_dmma<2><<<grid, block>>>(out, iters);
                    if (s == 3) k_dmma<3><<<grid, block>>>(out, iters);
                });
                double fl = 2.0 * fma_per_mma[s] * 4 * iters * (double)grid * wpb;
                printf("dmma %-9s warps/blk %2d blk/SM %d: %.2f TF/s\n", names[s], wpb, bps, fl / ms / 1e9);
            }
            double ms = time_it([&] { k_dfma<<<grid, block>>>(out, iters); });
            double fl = 2.0 * 8 * iters * (double)grid * block;
            printf("dfma            warps/blk %2d blk/SM %d: %.2f TF/s\n", wpb, bps, fl / ms / 1e9);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
