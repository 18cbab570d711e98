// The multivariate-normal contraction X = mean + z L^T on the FP64 tensor cores
// (continuous.py:312-336: `mean + z @ factor.T`), z = n x d row-major standard normals,
// L = d x d row-major factor (a Cholesky factor is lower triangular; the pivoted
// semidefinite factor of continuous.py:293-309 is not).
//
// GEMM view: M = n samples, N = d output coordinates r, K = d inputs c;
// A = z (row-major M x K), B[c][r] = L[r][c] -- i.e. B "column-major" is L itself, rows
// of L contiguous along K, exactly what mma.sync .row.col wants for both operands.
//
//  * mma.sync.m8n8k4 .f64 = one DMMA.8x8x4 (the FP64 tensor pipe). Block tile 128 x 64
//    (4 warps, 2 x 2, warp tile 64 x 32 = 8 x 4 tiles), K staged 16 at a time through a
//    4-deep cp.async pipeline (24 KB per stage, 2 blocks per SM). The 32 DMMAs of a k4 step
//    are independent; the next step's DMMA on the same accumulator comes 32 issues later
//    (m16n8k8 chained two dependent DMMAs per tile: ncu showed "wait" as the top stall).
//  * k is permuted inside each group of 8: the first k4 step takes physical k = 2t from
//    thread t, the second 2t + 1, for A and B alike. The dot product is the same set of
//    products, and each thread's pair of operands is one 16-byte LDS.128.
//    Rows of a stage are 128 B; chunk c of row r sits at c ^ 4 (r & 1), so the 8 lanes of
//    a quarter-warp (rows g, g + 1) hit 8 distinct 16-byte bank groups.
//  * Lower-triangular L: L[r][c] = 0 for c > r, so the block for columns [n0, n0 + 64)
//    stops its K loop at n0 + 64, and inside it each 8-column mma tile skips the k8 steps
//    past its last column (warp-uniform). Work done ~ d (d + 8) / 2 products per vector
//    (d (d + 1) flops per vector is the algorithmic minimum).
//  * Epilogue: + mean[r], 16-byte stores (layout n_d) or the transposed d x n layout.
#include "rs_kernels.cuh"

namespace {

constexpr int MV_BM = 128, MV_BN = 64, MV_BK = 16, MV_STAGES = 4, MV_THREADS = 128;
constexpr int MV_STAGE_DBL = (MV_BM + MV_BN) * MV_BK;  // doubles per stage
constexpr size_t MV_SMEM = (size_t)MV_STAGES * MV_STAGE_DBL * 8;

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

// V doubles (8 V bytes) from global to shared; src_bytes = 0 zero-fills (out of range)
template <int V>
__device__ __forceinline__ void cp_async(void *dst, const double *src, bool ok) {
    const unsigned d = smem_u32(dst);
    const int sz = ok ? 8 * V : 0;
    if constexpr (V == 2)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// element (row r, col k) of a [rows][MV_BK] stage tile with the 16-byte-chunk swizzle
__device__ __forceinline__ int sw(int r, int k) { return r * MV_BK + ((((k >> 1) ^ ((r & 1) << 2))) << 1) + (k & 1); }

// one DMMA.8x8x4: c0, c1 = C[g][2t], C[g][2t+1] += sum_k A[g][k] B[k][2t..2t+1], thread t
// supplying A[g][k_t] and B[k_t][g] for its k slot
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

// V: doubles per cp.async (2 when d is even and the pointers 16-byte aligned, else 1).
// LAYOUT 0: X is n x d row-major (n_d); 1: X^T, d x ldx row-major (d_n: a block of n rows
// of a larger fill writes columns [0, n) of rows of length ldx).
template <int V, int LAYOUT>
__global__ void __launch_bounds__(MV_THREADS, 2) k_mvn_dmma(const double *__restrict__ z, const double *__restrict__ L,
                                                           const double *__restrict__ mean, double *__restrict__ X,
                                                           long long n, int d, int lower, int ntn, long long ldx) {
    extern __shared__ __align__(128) double mv_smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp >> 1, wn = warp & 1;
    // column tiles fastest: the d/64 blocks of one row panel run together and share its
    // z rows through L2 (z is read from HBM about once)
    const int nt = blockIdx.x % ntn;
    const long long m0 = (long long)(blockIdx.x / ntn) * MV_BM;
    const int n0 = nt * MV_BN;
    const int kend = lower ? min(d, n0 + MV_BN) : d;
    const int ktiles = (kend + MV_BK - 1) / MV_BK;

    auto load_stage = [&](int kt, int slot) {
        double *sa = mv_smem + (size_t)slot * MV_STAGE_DBL;
        double *sb = sa + MV_BM * MV_BK;
        const int k0 = kt * MV_BK;
        constexpr int CPR = MV_BK / V;  // copies per tile row
        for (int i = tid; i < MV_BM * CPR; i += MV_THREADS) {
            const int r = i / CPR, k = (i % CPR) * V;
            const long long row = m0 + r;
            const bool ok = row < n && k0 + k < d;
            cp_async<V>(sa + sw(r, k), ok ? z + row * d + k0 + k : z, ok);
        }
        for (int i = tid; i < MV_BN * CPR; i += MV_THREADS) {
            const int r = i / CPR, k = (i % CPR) * V;
            const int col = n0 + r;
            const bool ok = col < d && k0 + k < d;
            cp_async<V>(sb + sw(r, k), ok ? L + (size_t)col * d + k0 + k : L, ok);
        }
    };

    // warp tile 64 x 32 = 8 x 4 tiles of 8 x 8; acc[i][j] = C[8i + g][8j + 2t, +1]
    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < MV_STAGES - 1; s++) {
        if (s < ktiles) load_stage(s, s);
        cp_commit();
    }
    // the first column of this warp's tiles (triangular skip: tile j needs k < wcol + 8 j + 8)
    const int wcol = n0 + 32 * wn;
    for (int kt = 0; kt < ktiles; kt++) {
        cp_wait<MV_STAGES - 2>();
        __syncthreads();
        {
            const int nk = kt + MV_STAGES - 1;
            if (nk < ktiles) load_stage(nk, nk % MV_STAGES);
            cp_commit();
        }
        const double *sa = mv_smem + (size_t)(kt % MV_STAGES) * MV_STAGE_DBL;
        const double *sb = sa + MV_BM * MV_BK;
#pragma unroll
        for (int ks = 0; ks < MV_BK / 8; ks++) {
            const int kg = kt * MV_BK + 8 * ks;  // global k of this group of 8
            const int kk = 8 * ks + 2 * t;       // this thread's physical k pair in the stage
            // each k8 group runs as two k4 DMMA steps: step 0 takes physical k = 2t (.x),
            // step 1 k = 2t + 1 (.y) -- one LDS.128 per operand pair, and the 32 tiles of a
            // step are independent, so no DMMA waits on the previous one's accumulator
            double2 b[4], a[8];
#pragma unroll
            for (int j = 0; j < 4; j++) b[j] = *(const double2 *)(sb + sw(32 * wn + 8 * j + g, kk));
#pragma unroll
            for (int i = 0; i < 8; i++) a[i] = *(const double2 *)(sa + sw(64 * wm + 8 * i + g, kk));
#pragma unroll
            for (int j = 0; j < 4; j++) {
                if (lower && kg >= wcol + 8 * j + 8) continue;  // warp-uniform: L[r][c] = 0 for c > r
#pragma unroll
                for (int i = 0; i < 8; i++) dmma(acc[i][j], a[i].x, b[j].x);
            }
#pragma unroll
            for (int j = 0; j < 4; j++) {
                if (lower && kg >= wcol + 8 * j + 8) continue;
#pragma unroll
                for (int i = 0; i < 8; i++) dmma(acc[i][j], a[i].y, b[j].y);
            }
        }
    }
    cp_wait<0>();

    // epilogue: acc[i][j] = C[8i + g][8j + 2t, 8j + 2t + 1] (+ mean), 16-byte stores (n_d)
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const int col = n0 + 32 * wn + 8 * j + 2 * t;
        if (col >= d) continue;
        const bool two = col + 1 < d;
        const double mu0 = __ldg(mean + col), mu1 = two ? __ldg(mean + col + 1) : 0.0;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const long long row = m0 + 64 * wm + 8 * i + g;
            if (row >= n) continue;
            const double x0 = mu0 + acc[i][j][0], x1 = mu1 + acc[i][j][1];
            if constexpr (LAYOUT == 0) {
                double *p = X + row * d + col;
                if (V == 2 && two) {
                    *(double2 *)p = make_double2(x0, x1);
                } else {
                    p[0] = x0;
                    if (two) p[1] = x1;
                }
            } else {
                X[(long long)col * ldx + row] = x0;
                if (two) X[(long long)(col + 1) * ldx + row] = x1;
            }
        }
    }
}

}  // namespace

namespace rsk {
MvnLaunch mvn_kernel(int vec16, int layout) {
    const void *fn;
    if (vec16) fn = layout ? (const void *)k_mvn_dmma<2, 1> : (const void *)k_mvn_dmma<2, 0>;
    else fn = layout ? (const void *)k_mvn_dmma<1, 1> : (const void *)k_mvn_dmma<1, 0>;
    return MvnLaunch{fn, MV_SMEM, MV_THREADS, MV_BM, MV_BN};
}
}  // namespace rsk
