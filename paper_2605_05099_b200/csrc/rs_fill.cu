// B200 bulk stream-fill: kernels + orchestration behind the C ABI (include/randstream_b200.h).
//
// One logical word stream (the WordBuffer remainder followed by the engine's
// words, buffer.py:29-49) is cut into T contiguous segments of L engine words;
// thread t owns segment t and starts from an exact skip-ahead of the engine:
//   x256**/++ : GF(2) matrices T^(L*2^j) (block start: warp-cooperative mat-vec,
//               in-block: log-depth doubling in shared memory)   [A6]
//   pcg64     : affine LCG powers (mul, add) for L*2^j            [A7]
//   philox    : counter + t*L/4                                  [A9]
//   ranlux++  : x * A^((L/9)*2^j)                                [A8]
// Fixed-consumption fills (raw, u01, u01f, power-of-two bounds) map word i to
// output i and are written in one pass with 256-bit stores. Variable-consumption
// fills (ziggurat normal/exponential, gamma, beta, Lemire) keep the reference's
// exact draw order with a two-pass parse:
//   count  : each thread parses its segment from its start, counting samples that
//            start inside it and recording its exit (first boundary >= end);
//   fixup  : thread t's true entry is thread t-1's exit; the few threads whose
//            entry is not 0 re-parse in lockstep with their entry-0 parse until the
//            two meet at a common boundary (parses of these grammars converge within
//            a few words) -> exact per-thread counts;
//   scan   : exclusive prefix sum of the counts (stream compaction offsets);
//   emit   : each thread re-parses from its true entry and writes its samples at
//            their global offsets.
// Non-convergence inside a segment is detected and iterated to a fixed point.

#include "rs_kernels.cuh"

namespace {
// ----------------------------------------------------------------------------- host side
#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t _e = (x);                                                                  \
        if (_e != cudaSuccess) {                                                               \
            rs::set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " #x);  \
            return RS_ERR_CUDA;                                                                \
        }                                                                                      \
    } while (0)

struct DevCtx {
    bool ready = false;
    int sms = 0;
    RsZigSlow *zslow[2] = {nullptr, nullptr};
    ZigFast *zfast[2] = {nullptr, nullptr};
    RsZigSlowF *zslowf[2] = {nullptr, nullptr};
    ZigFastF *zfastf[2] = {nullptr, nullptr};
    u64 *rlxA = nullptr;
    // scratch
    size_t cap_T = 0;
    u64 *states = nullptr, *cnt0 = nullptr, *cnt1 = nullptr, *cnt = nullptr, *bsum = nullptr;  // bsum: per-block count sums (k_fixup -> k_emit)
    u32 *ex0 = nullptr, *ex1 = nullptr, *exA = nullptr, *exB = nullptr, *entry = nullptr;
    u32 *bm = nullptr;  // [2][bmw][T] boundary bitmaps
    size_t bm_bytes = 0;
    DevResult *res = nullptr;
    DevResult *res_host = nullptr;
    std::map<std::tuple<int, u64, int>, u64 *> x256_ml;  // (family, L, levels) -> matrices
    void *stage = nullptr;
    size_t stage_bytes = 0;
    double *mvn_z = nullptr;
    size_t mvn_bytes = 0;
    u64 *words = nullptr;  // materialized engine words for parse-from-memory
    size_t words_bytes = 0;
    u32 *overrun = nullptr;  // device flag: a parse read past the materialized words
    // gamma speculative store (FillPlan::spec ...): grown on demand
    void *spec = nullptr;
    size_t spec_bytes = 0;
    void *pre = nullptr;
    size_t pre_bytes = 0;
    // single-pass tile parse: one record per tile (+ the prefix record), tagged with a launch epoch
    u64 *tile_rec = nullptr;
    size_t tile_rec_n = 0;
    u32 tile_epoch = 0;
    // the counted slice of rs_range_count, waiting for rs_range_emit (its plan refers to
    // the scratch above, so any other fill on this device invalidates it)
    struct Range {
        bool valid = false;
        FillPlan p;
        rsk::VarKernels K;
        u32 *ex = nullptr;
        u64 count = 0;
        int unit = 1;
        bool mem = false;
        u64 origin = 0;  // units from the plan start to the slice start (warm-up segments)
        u64 entry = 0;   // the slice's entry (units from the slice start)
    } range;
};

std::mutex g_mu;
std::map<int, DevCtx> g_dev;

rs_status init_dev(int dev, DevCtx **out) {
    DevCtx &c = g_dev[dev];
    *out = &c;
    if (c.ready) return RS_OK;
    CK(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev));
    for (int k = 0; k < 2; k++) {
        RsZigSlow zs;
        RsZigFastHost zf[256];
        rs_build_zig(k, &zs, zf);
        CK(cudaMalloc(&c.zslow[k], sizeof(RsZigSlow)));
        CK(cudaMalloc(&c.zfast[k], sizeof(zf)));
        CK(cudaMemcpy(c.zslow[k], &zs, sizeof(RsZigSlow), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c.zfast[k], zf, sizeof(zf), cudaMemcpyHostToDevice));
    }
    for (int k = 0; k < 2; k++) {  // f32 tables (zigtables.py:1563-3116)
        RsZigSlowF zs;
        ZigFastF zf[256];
        for (int i = 0; i < 256; i++) {
            uint32_t fb = k ? RS_FE_F_BITS[i] : RS_FI_F_BITS[i], wb = k ? RS_WE_F_BITS[i] : RS_WI_F_BITS[i];
            memcpy(&zs.f[i], &fb, 4);
            zf[i].k = k ? RS_KE_F[i] : RS_KI_F[i];
            memcpy(&zf[i].w, &wb, 4);
        }
        CK(cudaMalloc(&c.zslowf[k], sizeof(RsZigSlowF)));
        CK(cudaMalloc(&c.zfastf[k], sizeof(zf)));
        CK(cudaMemcpy(c.zslowf[k], &zs, sizeof(RsZigSlowF), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c.zfastf[k], zf, sizeof(zf), cudaMemcpyHostToDevice));
    }
    u64 A[9];
    rs::rlx_pow2k_A(0, A);
    CK(cudaMalloc(&c.rlxA, sizeof(A)));
    CK(cudaMemcpy(c.rlxA, A, sizeof(A), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&c.res, sizeof(DevResult)));
    CK(cudaMalloc(&c.overrun, sizeof(u32)));
    CK(cudaMemset(c.overrun, 0, sizeof(u32)));
    CK(cudaMallocHost(&c.res_host, sizeof(DevResult)));
    c.ready = true;
    return RS_OK;
}

rs_status ensure_scratch(DevCtx &c, size_t T) {
    if (T <= c.cap_T) return RS_OK;
    size_t nT = T + T / 4;
    cudaFree(c.states); cudaFree(c.cnt0); cudaFree(c.cnt1); cudaFree(c.cnt); cudaFree(c.bsum);
    cudaFree(c.ex0); cudaFree(c.ex1); cudaFree(c.exA); cudaFree(c.exB); cudaFree(c.entry);
    CK(cudaMalloc(&c.states, nT * 32));
    CK(cudaMalloc(&c.cnt0, nT * 8));
    CK(cudaMalloc(&c.cnt1, nT * 8));
    CK(cudaMalloc(&c.ex1, nT * 4));
    CK(cudaMalloc(&c.cnt, nT * 8));
    CK(cudaMalloc(&c.bsum, (nT / BLOCK + 2) * 8));
    CK(cudaMalloc(&c.ex0, nT * 4));
    CK(cudaMalloc(&c.exA, nT * 4));
    CK(cudaMalloc(&c.exB, nT * 4));
    CK(cudaMalloc(&c.entry, nT * 4));
    c.cap_T = nT;
    return RS_OK;
}

// x256: ML[0] = T^L, ML[1 + k] = T^(32 L 2^k) for k < levels; cached per (L, levels) on the device
rs_status x256_mats(DevCtx &c, int engine, u64 L, int levels, u64 **out) {
    // x256 family, or the 128-bit xorshift128+ / xoroshiro128 matrices padded to 256 bits
    const bool narrow = engine == RS_ENG_X128P || engine == RS_ENG_XORO;
    auto pow2 = [&](int k) -> const rs::Mat256 & { return narrow ? rs::x128_pow2(engine, k) : rs::x256_pow2(k); };
    auto key = std::make_tuple(narrow ? engine : 0, L, levels);
    auto it = c.x256_ml.find(key);
    if (it != c.x256_ml.end()) { *out = it->second; return RS_OK; }
    std::vector<rs::Mat256> m(1 + levels);
    bool init = false;
    for (int k = 0; k < 64; k++)
        if ((L >> k) & 1) {
            if (!init) { m[0] = pow2(k); init = true; }
            else rs::mat_mul(pow2(k), m[0], m[0]);
        }
    if (levels > 0) {
        rs::Mat256 *t = new rs::Mat256(m[0]);
        for (int i = 0; i < 5; i++) rs::mat_mul(*t, *t, *t);  // T^(32 L)
        m[1] = *t;
        delete t;
        for (int k = 1; k < levels; k++) rs::mat_mul(m[k], m[k], m[k + 1]);
    }
    u64 *d;
    CK(cudaMalloc(&d, (size_t)(1 + levels) * sizeof(rs::Mat256)));
    CK(cudaMemcpy(d, m.data(), (size_t)(1 + levels) * sizeof(rs::Mat256), cudaMemcpyHostToDevice));
    if (c.x256_ml.size() > 16) {  // bound the cache
        for (auto &kv : c.x256_ml) cudaFree(kv.second);
        c.x256_ml.clear();
    }
    c.x256_ml[key] = d;
    *out = d;
    return RS_OK;
}

// resident blocks per SM; a kernel with dynamic shared memory gets its opt-in limit set
// here first (per device), so call this before launching it
int occupancy(const void *fn, size_t smem = 0) {
    static std::map<std::tuple<int, const void *, size_t>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    auto key = std::make_tuple(dev, fn, smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    if (smem > 0) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, BLOCK, smem) != cudaSuccess || nb < 1) {
        cudaGetLastError();
        nb = 1;
    }
    cache[key] = nb;
    return nb;
}

bool is_device_ptr(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

size_t elem_size(int dist) {
    switch (dist) {
    case RS_DIST_U01F: case RS_DIST_UNIFF: case RS_DIST_NORMF: case RS_DIST_EXPF: case RS_DIST_UINT32:
    case RS_DIST_INT32: return 4;
    default: return 8;
    }
}

// ---- dispatch (the kernels themselves live in the k_*.cu units)
using rsk::VarKernels;
// Engines whose parse passes read materialized words: the expensive ones (Philox,
// ranlux++, ChaCha20), the interleaved ones, and the registry's other skip-ahead
// engines (x128+, xoro++, squares), which thereby need no parse-kernel instantiations.
bool parse_from_memory(int e) {
    return e == RS_ENG_PHILOX || e == RS_ENG_RANLUX || e == RS_ENG_X256PP_SIMD || e == RS_ENG_X256SS_SIMD ||
           e == RS_ENG_CHACHA20 || e == RS_ENG_X128P || e == RS_ENG_XORO || e == RS_ENG_SQUARES;
}
// no skip-ahead: one device thread replays the stream (sfc64 rng.py:162-163; cwg128 likewise)
bool is_serial(int e) { return e == RS_ENG_SFC64 || e == RS_ENG_SFC64_SIMD || e == RS_ENG_CWG128; }
VarKernels var_kernels(int e, int fam) {
    switch (e) {
    case RS_ENG_X256SS: return rsk::var_kernels_x256ss(fam);
    case RS_ENG_X256PP: return rsk::var_kernels_x256pp(fam);
    case RS_ENG_PCG64: return rsk::var_kernels_pcg(fam);
    default: return rsk::var_kernels_mem(fam);  // words materialized first
    }
}
using rsk::fixed_kernel;
using rsk::philox_kernel;
using rsk::serial_kernel;
using rsk::simd_kernel;

rs_status launch(const void *fn, dim3 g, dim3 b, void **args, cudaStream_t st, size_t smem = 0) {
    CK(cudaLaunchKernel(fn, g, b, args, smem, st));
    return RS_OK;
}

// ---- parameter resolution (validated values)
struct Resolved {
    int dist;          // RS_DIST_* as requested
    int fixed_mode;    // FX_* or -1 for a variable-consumption family
    int family;        // FAM_*
    int kind;          // law within the family / fixed map
    int unit;          // 1 words, 2 halves
    double fp[4];
    u64 ip[4];
    GammaPrm ga, gb;
    int raw_norm;
    double words_per_sample;
    int table;         // 0 normal, 1 exponential, 2 normal f32, 3 exponential f32, -1 none
};

GammaPrm gamma_prm(double alpha, double theta) {
    // continuous.py:183-199; alpha < 1 runs gamma(alpha + 1, 1) then the boost
    GammaPrm g;
    g.alpha = alpha;
    g.theta = theta;
    g.boost = alpha < 1.0;
    double a = g.boost ? alpha + 1.0 : alpha;
    double th = g.boost ? 1.0 : theta;
    g.d = a - 1.0 / 3.0;
    g.cc = 1.0 / std::sqrt(9.0 * g.d);
    g.td = th * g.d;
    return g;
}
double gamma_words(const GammaPrm &g) { return 2.2 + (g.boost ? 1.0 : 0.0); }

#define RS_FAIL(msg)                \
    do {                            \
        rs::set_error(msg);         \
        return RS_ERR_VALUE;        \
    } while (0)

// fp / ip layouts per distribution: include/randstream_b200.h
rs_status resolve(int dist, const double *fp, const u64 *ip, Resolved &r) {
    memset(&r, 0, sizeof r);
    r.dist = dist;
    r.fixed_mode = -1;
    r.family = -1;
    r.unit = 1;
    r.table = -1;
    r.words_per_sample = 1.0;
    switch (dist) {
    case RS_DIST_UINT64: {
        u64 b = ip[0];
        bool b64 = ip[1] != 0;
        if (b == 0 || b64) { r.fixed_mode = FX_RAW; }
        else if ((b & (b - 1)) == 0) { r.fixed_mode = FX_POW2; r.ip[0] = b; }
        else {
            r.family = FAM_LEMIRE;
            r.ip[0] = b;
            r.ip[1] = (0 - b) % b;  // discrete.py:34
            r.words_per_sample = 1.0 / (1.0 - (double)r.ip[1] * 5.421010862427522e-20);
        }
        return RS_OK;
    }
    case RS_DIST_INT64: {  // bounded_int(m, n, 64): ip = {span, 64, m, full}
        if (ip[3]) { r.fixed_mode = FX_WMAP; r.kind = WK_I64; r.ip[2] = ip[2]; return RS_OK; }
        u64 b = ip[0];
        if (b == 0) RS_FAIL("bad signed range");
        r.family = FAM_LEMIRE;
        r.ip[0] = b;
        r.ip[1] = (0 - b) % b;
        r.ip[2] = ip[2];
        r.words_per_sample = 1.0 / (1.0 - (double)r.ip[1] * 5.421010862427522e-20);
        return RS_OK;
    }
    case RS_DIST_UINT32: case RS_DIST_INT32: {  // halves; ip = {b, width} | {span, 32, m, full}
        int width = dist == RS_DIST_INT32 ? 32 : (int)ip[1];
        if (width != 8 && width != 16 && width != 32) RS_FAIL("bounded width must be 8, 16, or 32");
        u64 full = 1ULL << width, mask = full - 1;
        u64 b = ip[0];
        r.unit = 2;
        if (dist == RS_DIST_INT32 && ip[3]) { r.fixed_mode = FX_HMAP; r.kind = HK_I32; r.ip[2] = ip[2]; return RS_OK; }
        if (b > full) RS_FAIL("bound out of range");
        if (dist == RS_DIST_UINT32 && (b == 0 || b == full)) {
            r.fixed_mode = FX_HMAP; r.kind = HK_MASK; r.ip[3] = mask; return RS_OK;
        }
        if (dist == RS_DIST_UINT32 && (b & (b - 1)) == 0) {
            r.fixed_mode = FX_HMAP; r.kind = HK_POW2; r.ip[0] = b; r.ip[1] = (u64)width; r.ip[3] = mask; return RS_OK;
        }
        if (b == 0) RS_FAIL("bad signed range");
        r.family = FAM_U32;
        r.ip[0] = b;
        r.ip[1] = (full - b) % b;
        r.ip[2] = dist == RS_DIST_INT32 ? ip[2] : 0;
        r.ip[3] = (u64)width;
        r.words_per_sample = 0.5 / (1.0 - (double)r.ip[1] / (double)full);
        return RS_OK;
    }
    case RS_DIST_U01: r.fixed_mode = FX_U01; return RS_OK;
    case RS_DIST_U01F: r.fixed_mode = FX_U01F; r.unit = 2; return RS_OK;
    case RS_DIST_UNIF:
        if (!(fp[1] > fp[0])) RS_FAIL("unif needs b > a");
        r.fixed_mode = FX_WMAP; r.kind = WK_UNIF; r.fp[0] = fp[0]; r.fp[1] = fp[1];
        return RS_OK;
    case RS_DIST_UNIFF:
        if (!(fp[1] > fp[0])) RS_FAIL("uniff needs b > a");
        r.fixed_mode = FX_HMAP; r.kind = HK_UNIFF; r.unit = 2; r.fp[0] = fp[0]; r.fp[1] = fp[1];
        return RS_OK;
    case RS_DIST_GUMBEL:
        if (!(fp[1] > 0.0)) RS_FAIL("gumbel scale must be > 0");
        r.fixed_mode = FX_WMAP; r.kind = WK_GUMBEL; r.fp[0] = fp[0]; r.fp[1] = fp[1];
        return RS_OK;
    case RS_DIST_NORM: case RS_DIST_STDNORM: case RS_DIST_LOGNORMAL:
        r.family = FAM_NORM;
        r.table = 0;
        r.words_per_sample = 1.03;
        if (dist == RS_DIST_STDNORM) { r.kind = NK_STD; r.raw_norm = 1; return RS_OK; }
        if (!(fp[1] >= 0.0)) RS_FAIL(dist == RS_DIST_NORM ? "normal variance must be >= 0" : "lognormal variance must be >= 0");
        r.kind = dist == RS_DIST_NORM ? NK_NORM : NK_LOGNORMAL;
        r.fp[0] = fp[0];
        r.fp[1] = std::sqrt(fp[1]);
        return RS_OK;
    case RS_DIST_SKEW_NORMAL: {  // fp = {alpha, mu, sigma}
        if (!(fp[2] > 0.0)) RS_FAIL("skew_normal scale must be > 0");
        double delta = fp[0] / std::sqrt(1.0 + fp[0] * fp[0]);
        r.family = FAM_NORM; r.kind = NK_SKEW; r.table = 0; r.words_per_sample = 2.06;
        r.fp[0] = delta; r.fp[1] = std::sqrt(1.0 - delta * delta); r.fp[2] = fp[1]; r.fp[3] = fp[2];
        return RS_OK;
    }
    case RS_DIST_EXP:
        if (!(fp[0] > 0.0)) RS_FAIL("exponential scale must be > 0");
        r.family = FAM_EXP; r.kind = EK_EXP; r.table = 1; r.fp[0] = fp[0]; r.words_per_sample = 1.04;
        return RS_OK;
    case RS_DIST_PARETO:
        if (!(fp[0] > 0.0 && fp[1] > 0.0)) RS_FAIL("pareto needs alpha > 0 and xm > 0");
        r.family = FAM_EXP; r.kind = EK_PARETO; r.table = 1; r.fp[0] = fp[0]; r.fp[1] = fp[1];
        r.words_per_sample = 1.04;
        return RS_OK;
    case RS_DIST_GPD:
        if (!(fp[2] > 0.0)) RS_FAIL("gpd scale must be > 0");
        r.family = FAM_EXP; r.kind = EK_GPD; r.table = 1; r.fp[0] = fp[0]; r.fp[1] = fp[1]; r.fp[2] = fp[2];
        r.words_per_sample = 1.04;
        return RS_OK;
    case RS_DIST_WEIBULL:
        if (!(fp[0] > 0.0 && fp[1] > 0.0)) RS_FAIL("weibull needs k > 0 and lambda > 0");
        r.family = FAM_EXP; r.kind = EK_WEIBULL; r.table = 1; r.fp[0] = fp[0]; r.fp[1] = fp[1];
        r.words_per_sample = 1.04;
        return RS_OK;
    case RS_DIST_GAMMA:
        if (!(fp[0] > 0.0)) RS_FAIL("gamma shape must be > 0");
        if (!(fp[1] > 0.0)) RS_FAIL("gamma scale must be > 0");
        r.family = FAM_GAMMA; r.kind = GK_GAMMA; r.table = 0;
        r.ga = gamma_prm(fp[0], fp[1]);
        r.words_per_sample = gamma_words(r.ga);
        return RS_OK;
    case RS_DIST_CHI2:
        if (!(fp[0] > 0.0)) RS_FAIL("chi2 degrees of freedom must be > 0");
        r.family = FAM_GAMMA; r.kind = GK_GAMMA; r.table = 0;
        r.ga = gamma_prm(fp[0] / 2.0, 2.0);
        r.words_per_sample = gamma_words(r.ga);
        return RS_OK;
    case RS_DIST_T:
        if (!(fp[0] > 0.0)) RS_FAIL("t degrees of freedom must be > 0");
        r.family = FAM_GAMMA; r.kind = GK_T; r.table = 0; r.fp[0] = fp[0];
        r.ga = gamma_prm(fp[0] / 2.0, 2.0);
        r.words_per_sample = 1.03 + gamma_words(r.ga);
        return RS_OK;
    case RS_DIST_F:
        if (!(fp[0] > 0.0 && fp[1] > 0.0)) RS_FAIL("f degrees of freedom must be > 0");
        r.family = FAM_GAMMA; r.kind = GK_F; r.table = 0; r.fp[0] = fp[0]; r.fp[1] = fp[1];
        r.ga = gamma_prm(fp[0] / 2.0, 1.0);
        r.gb = gamma_prm(fp[1] / 2.0, 1.0);
        r.words_per_sample = gamma_words(r.ga) + gamma_words(r.gb);
        return RS_OK;
    case RS_DIST_BETA:
        if (!(fp[0] > 0.0) || !(fp[1] > 0.0)) RS_FAIL("gamma shape must be > 0");
        r.family = FAM_GAMMA; r.kind = GK_BETA; r.table = 0;
        r.ga = gamma_prm(fp[0], 1.0);
        r.gb = gamma_prm(fp[1], 1.0);
        r.words_per_sample = gamma_words(r.ga) + gamma_words(r.gb);
        return RS_OK;
    case RS_DIST_NORMF:
        if (!(fp[1] >= 0.0)) RS_FAIL("normf variance must be >= 0");
        r.family = FAM_F32; r.kind = FK_NORMF; r.unit = 2; r.table = 2; r.fp[0] = fp[0]; r.fp[1] = std::sqrt(fp[1]);
        r.words_per_sample = 0.52;
        return RS_OK;
    case RS_DIST_EXPF:
        if (!(fp[0] > 0.0)) RS_FAIL("expf scale must be > 0");
        r.family = FAM_F32; r.kind = FK_EXPF; r.unit = 2; r.table = 3; r.fp[0] = fp[0];
        r.words_per_sample = 0.53;
        return RS_OK;
    }
    RS_FAIL("unknown distribution id");
}

void fill_plan_common(FillPlan &p, DevCtx &c, const Resolved &r, int engine, int fm) {
    p.engine = engine;
    p.dist = r.dist;
    p.fm = fm;
    memcpy(p.fp, r.fp, sizeof p.fp);
    memcpy(p.ip, r.ip, sizeof p.ip);
    p.ga = r.ga;
    p.gb = r.gb;
    p.raw_norm = r.raw_norm;
    p.kind = r.kind;
    p.unit = r.unit;
    p.fmode = r.fixed_mode;
    p.zslow = (r.table == 0 || r.table == 1) ? c.zslow[r.table] : nullptr;
    p.zfast = (r.table == 0 || r.table == 1) ? c.zfast[r.table] : nullptr;
    p.zslowf = (r.table == 2 || r.table == 3) ? c.zslowf[r.table - 2] : nullptr;
    p.zfastf = (r.table == 2 || r.table == 3) ? c.zfastf[r.table - 2] : nullptr;
    p.rlx_A = c.rlxA;
}

// Segment geometry + per-engine jump tables for stride L (engine origin = p.base)
rs_status plan_segments(DevCtx &c, FillPlan &p, u64 words, u64 Lmin, int occ, cudaStream_t st, bool tables = true,
                        u64 align = 36, u64 force_L = 0, u64 force_T = 0) {
    u64 L, T;
    if (force_L) {  // explicit geometry (rs_range_count: every rank's slice has the same shape)
        L = force_L;
        T = force_T;
    } else {
        // exactly one wave of resident threads: equal segments finish together
        u64 Tfull = (u64)c.sms * (u64)occ * BLOCK;
        L = (words + Tfull - 1) / Tfull;
        if (L < Lmin) L = Lmin;
        // a whole number of philox blocks (4) and ranlux chunks (9); fixed fills pass
        // align = 144 (also 16-word lines): every thread then has the same alignment
        // prologue, so the lanes stay in phase (ranlux mulmods convergent)
        L = (L + align - 1) / align * align;
        T = (words + L - 1) / L;
        if (T < 1) T = 1;
        T = (T + BLOCK - 1) / BLOCK * BLOCK;
    }
    p.L = L;
    p.T = (u32)T;
    int levels = 1;
    while ((1ULL << levels) < T) levels++;
    if (levels > MAXLEV) { rs::set_error("fill too large for one plan"); return RS_ERR_INTERNAL; }
    rs_status s = ensure_scratch(c, T);
    if (s) return s;
    if (!tables) return RS_OK;
    if (p.engine == RS_ENG_PCG64) {
        u128 inc = ((u128)p.base[3] << 64) | p.base[2];
        for (int j = 0; j < levels; j++) {
            u128 m, a;
            rs::pcg_affine(inc, (u128)L << j, m, a);
            p.pcg_m[j][0] = (u64)m; p.pcg_m[j][1] = (u64)(m >> 64);
            p.pcg_a[j][0] = (u64)a; p.pcg_a[j][1] = (u64)(a >> 64);
        }
    } else if (p.engine == RS_ENG_RANLUX) {
        for (int j = 0; j < levels; j++) rs::rlx_pow_A((u128)(L / 9) << j, p.rlx[j]);
    } else if (p.engine == RS_ENG_CHACHA20) {
        if ((p.base[5] >> 32) + (u128)T * (L / 8) > ((u128)1 << 32)) {
            rs::set_error("chacha20 stream exhausted");  // counter.py:212-213
            return RS_ERR_VALUE;
        }
    } else if (p.engine == RS_ENG_X256SS || p.engine == RS_ENG_X256PP || p.engine == RS_ENG_X128P ||
               p.engine == RS_ENG_XORO) {
        int lv = 0;  // bits of the warp index
        while ((1ULL << lv) < T / 32) lv++;
        u64 *ml;
        if (p.engine == RS_ENG_X128P || p.engine == RS_ENG_XORO) {  // padded 4-word states
            p.base[2] = p.base[3] = 0;
        }
        s = x256_mats(c, p.engine, L, lv, &ml);
        if (s) return s;
        p.x256_states = c.states;
        void *args[] = {&p, &ml, &c.states};
        s = launch(rsk::setup_kernel(), dim3((unsigned)(T / BLOCK)), dim3(BLOCK), args, st);
        if (s) return s;
    }
    return RS_OK;
}

// logical stream of `s`: buffer remainder then engine words
void stream_prefix(const rs_stream *s, FillPlan &p) {
    int P = s->fill - s->cursor;
    if (P < 0) P = 0;
    p.P = P;
    for (int i = 0; i < P; i++) p.prefix[i] = s->buf[s->cursor + i];
}

// post-fill position (buffer.py:29-49): E logical words consumed
rs_status apply_consumption(rs_stream *s, u64 E, const DevResult *sr) {
    int P = s->fill - s->cursor;
    if (P < 0) P = 0;
    if (E <= (u64)P) {
        s->cursor += (int)E;
        return RS_OK;
    }
    u64 ep = E - P;
    u64 R = (ep + CAP - 1) / CAP;
    if (is_serial(s->engine)) {  // rebuilt on the device by k_serial
        if (!sr || sr->serial_consumed != ep) {
            rs::set_error("serial fill bookkeeping mismatch");
            return RS_ERR_INTERNAL;
        }
        memcpy(s->state, sr->serial_state, 8 * rs::state_words(s->engine));
        memcpy(s->buf, sr->serial_buf, CAP * 8);
    } else {
        if (!rs::engine_advance_words(s->engine, s->state, (u128)(R - 1) * CAP)) {
            rs::set_error("cannot advance engine");
            return RS_ERR_INTERNAL;
        }
        rs::engine_generate(s->engine, s->state, s->buf, CAP);
    }
    s->fill = CAP;
    s->cursor = (int)(ep - (R - 1) * CAP);
    return RS_OK;
}

struct Staging {
    void *dptr = nullptr;
    bool host = false;
};

rs_status get_out(DevCtx &c, void *out, size_t bytes, Staging &sg) {
    if (is_device_ptr(out)) { sg.dptr = out; sg.host = false; return RS_OK; }
    sg.host = true;
    if (bytes > c.stage_bytes) {
        cudaFree(c.stage);
        c.stage = nullptr;
        CK(cudaMalloc(&c.stage, bytes));
        c.stage_bytes = bytes;
    }
    sg.dptr = c.stage;
    return RS_OK;
}

// k_fixed launch
rs_status launch_fixed(DevCtx &, FillPlan &p, const void *fn, cudaStream_t st) {
    void *args[] = {&p};
    return launch(fn, dim3(p.T / BLOCK), dim3(BLOCK), args, st, FX_SMEM);
}

// interleaved xoshiro fixed fill: lane states jumped per step group on the device
rs_status launch_simd(DevCtx &c, FillPlan &p, int mode, cudaStream_t st) {
    const void *fn = simd_kernel(p.engine, mode);
    u64 steps = (p.weng + 7) / 8;
    if (steps == 0) steps = 1;
    // Lane-thread groups: >= 128 steps per thread amortise the per-thread GF(2) setup
    // (k_x256_setup), capped at ONE block per SM: 148 x 32 groups, each a stream of 256-byte
    // runs, measured faster than 2, 3, 4 or 6 blocks per SM at every size from 2^26 up
    // (raw 2^30: 1.37 / 1.39 / 1.82 / 1.47 / 1.48 ms), and than the earlier 96 blocks, which
    // left a third of the SMs idle (1.83 ms).
    u64 blocks = ((steps + 127) / 128 + 31) / 32;
    if (blocks > (u64)c.sms) blocks = c.sms;
    u64 G = blocks * (BLOCK / 8);
    u64 Ls = (steps + G - 1) / G;
    if (Ls < 16) Ls = 16;
    Ls = (Ls + 3) / 4 * 4;  // whole 4-step batches (256-byte runs)
    G = (steps + Ls - 1) / Ls;
    u64 Gpad = (G + BLOCK - 1) / BLOCK * BLOCK;
    p.L = Ls;
    p.G = G;
    p.Gpad = Gpad;
    {   // 256-byte runs need the group's first word 32-byte aligned and every sample to exist
        // as a whole element (half modes: an even count after the pending half)
        const bool half = mode == FX_U01F || mode == FX_HMAP;
        uintptr_t a0 = (uintptr_t)p.out + (half ? 4 * ((u64)p.pending_used + 2ULL * p.P) : 8ULL * p.P);
        const u64 need = half ? (u64)p.pending_used + 2ULL * ((u64)p.P + p.weng / 8 * 8) : (u64)p.P + p.weng / 8 * 8;
        p.vec_ok = (a0 & 31) == 0 && need <= p.n;
    }
    rs_status rc = ensure_scratch(c, 8 * Gpad);
    if (rc) return rc;
    int lv = 0;
    while ((1ULL << lv) < Gpad / 32) lv++;
    u64 *ml;
    if ((rc = x256_mats(c, RS_ENG_X256PP, Ls, lv, &ml))) return rc;
    p.x256_states = c.states;
    void *sargs[] = {&p, &ml, &c.states};
    if ((rc = launch(rsk::setup_kernel(), dim3((unsigned)(Gpad / BLOCK), 8), dim3(BLOCK), sargs, st))) return rc;
    void *args[] = {&p};
    return launch(fn, dim3((unsigned)(8 * Gpad / BLOCK)), dim3(BLOCK), args, st);
}

// engine words [0, m.weng) of m.base into m.out (raw u64) with the fixed-fill kernels
rs_status launch_raw_words(DevCtx &c, FillPlan &m, cudaStream_t st) {
    rs_status rc;
    if (rs::simd_engine(m.engine)) return launch_simd(c, m, FX_RAW, st);
    if (m.engine == RS_ENG_PHILOX) {
        const void *fn = philox_kernel(FX_RAW);
        for (int i = 0; i < 10; i++) {
            m.rk0[i] = m.base[4] + (u64)i * 0x9E3779B97F4A7C15ULL;
            m.rk1[i] = m.base[5] + (u64)i * 0xBB67AE8584CAA73BULL;
        }
        m.vec_ok = (((uintptr_t)m.out) & 31) == 0;
        u64 nblk = (m.weng + 3) / 4;
        u64 g = (u64)c.sms * occupancy(fn);
        u64 need = (nblk + BLOCK - 1) / BLOCK;
        if (need < g) g = need;
        if (g < 1) g = 1;
        void *args[] = {&m};
        return launch(fn, dim3((unsigned)g), dim3(BLOCK), args, st);
    }
    const void *fn = fixed_kernel(m.engine, FX_RAW);
    if ((rc = plan_segments(c, m, m.weng, 64, occupancy(fn, FX_SMEM), st, true, 144))) return rc;
    return launch_fixed(c, m, fn, st);
}

// shortest segment of a variable-consumption plan (gamma-family resync distances)
u64 var_lmin(const Resolved &r) { return r.family == FAM_GAMMA ? (r.kind == GK_GAMMA ? 1024 : 2048) : 128; }
// shortest segment of a range slice (multiple of RS_RANGE_ALIGN): a slice is 1/N of a fill,
// so its segments are shorter than a whole fill's; resolution rounds absorb the rare
// segment that a re-parse crosses without meeting its speculative parse
u64 range_lmin(const Resolved &r) { return r.family == FAM_GAMMA ? 288 : 144; }

// Per-chunk device inputs of the parse passes: the materialized engine words
// (parse-from-memory engines) and the gamma family's boundary bitmaps.
rs_status prep_chunk(DevCtx &c, FillPlan &p, const Resolved &r, bool mem, cudaStream_t st) {
    rs_status rc;
    if (mem) {
        // materialize the chunk's engine words (+ slack for the parses that run past the
        // last segment end) with the coalesced fixed-fill kernel
        u64 nw = (u64)p.T * p.L + std::max<u64>(1ULL << 16, (u64)p.T * p.L / 64);
        nw = (nw + 143) / 144 * 144;
        if (nw * 8 > c.words_bytes) {
            cudaFree(c.words);
            c.words = nullptr;
            CK(cudaMalloc(&c.words, nw * 8));
            c.words_bytes = nw * 8;
        }
        FillPlan m = p;
        m.P = 0;
        m.lp0 = 0;
        m.n = nw;
        m.weng = nw;
        m.out = c.words;
        m.out0 = 0;
        m.pending_used = 0;
        m.unit = 1;
        m.fmode = FX_RAW;
        if ((rc = launch_raw_words(c, m, st))) return rc;
        p.words = c.words;
        p.overrun = c.overrun;
        p.nwords = nw;
    }
    p.bm = nullptr;
    if (r.family == FAM_GAMMA) {
        // the count pass's boundary bitmaps cover the whole segment (+ the exit overshoot
        // of 32 units): a fixup then never falls back to re-parsing from the start
        p.bmw = (u32)((p.L * (u64)r.unit + 63) / 32);
        size_t need = (size_t)p.T * 4 * 2 * p.bmw;
        if (need > c.bm_bytes) {
            cudaFree(c.bm);
            c.bm = nullptr;
            CK(cudaMalloc(&c.bm, need));
            c.bm_bytes = need;
        }
        p.bm = c.bm;
    }
    p.spec = nullptr;
    // the store costs ~36 bytes per provisioned sample slot; past 16 GiB (a 2^29-sample
    // gamma fill) the three-parse path keeps the scratch bounded
    const size_t spec_est = (size_t)p.T * ((p.L + (u64)CAP + 1) / (r.kind != GK_GAMMA ? 4 : 2) + 8) * 36;
    if (r.family == FAM_GAMMA && r.kind != GK_T && !getenv("RS_NO_SPEC") && spec_est <= (16ULL << 30)) {
        // an attempt draws 2 words, so a segment of L words starts <= L/2 + 1 samples
        // (<= L/4 + 1 for the paired laws: two gamma sub-samples per sample)
        const bool paired = r.kind != GK_GAMMA;
        // (+ the samples the buffered prefix can start in segment 0: without it every fill that
        // begins mid-buffer with P >= 16 words overflowed segment 0 and lost the store --
        // chained gamma(10) fills 2^26 ran 2.75 ms instead of 2.02)
        const u64 div = paired ? 4 : 2;
        const u64 cap = ((p.L + (u64)CAP + 1) / div + 8 + 3) / 4 * 4;  // (the full buffer: one size for every start position)
        const size_t T = p.T;
        size_t need = T * cap * 12 * (paired ? 2 : 1);
        if (need > c.spec_bytes) {
            cudaFree(c.spec);
            c.spec = nullptr;
            CK(cudaMalloc(&c.spec, need));
            c.spec_bytes = need;
        }
        size_t pneed = T * cap * 12 + T * 20 + 16;
        if (pneed > c.pre_bytes) {
            cudaFree(c.pre);
            c.pre = nullptr;
            CK(cudaMalloc(&c.pre, pneed));
            c.pre_bytes = pneed;
        }
        p.spec_cap = cap;
        p.spec = (double *)c.spec;
        p.spec_tal = (u32 *)((char *)c.spec + T * cap * 8);
        p.pre = (double *)c.pre;
        p.pre_tal = (u32 *)((char *)c.pre + T * cap * 8);
        p.cmode = p.pre_tal + T * cap;
        p.pre_n = p.cmode + T;
        p.spec_from = p.pre_n + T;
        p.c1own = p.spec_from + T;
        p.mrank0 = p.c1own + T;
        p.spec_over = p.mrank0 + T;
        p.spec1 = paired ? (double *)((char *)c.spec + T * cap * 12) : nullptr;
        p.spec1_tal = paired ? (u32 *)((char *)c.spec + T * cap * 20) : nullptr;
        CK(cudaMemsetAsync(p.spec_over, 0, 4, st));
    }
    return RS_OK;
}

// One chunk through the single-pass tile parse: `words` engine words from the chunk's origin
// (p.base), the buffered prefix ahead of them (p.P, first chunk) or p.lp0 words to skip.
// On return c.res_host holds the result record; fell_back = the chunk left the tile model
// (or the grid could not be made co-resident) and must be redone by the two-pass path.
constexpr u64 TILE_MIN_N = 1ULL << 16;  // far above the 144-word prefix: sample n - 1 lies in a tile
rs_status run_tile_chunk(DevCtx &c, FillPlan &p, const void *fn, u64 words, cudaStream_t st, bool &fell_back) {
    static std::map<std::pair<int, const void *>, int> occ_cache;
    int dev = 0;
    cudaGetDevice(&dev);
    auto key = std::make_pair(dev, fn);
    auto it = occ_cache.find(key);
    int occ;
    if (it == occ_cache.end()) {
        occ = 0;
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TL_SMEM) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, TL_T, TL_SMEM) != cudaSuccess) {
            cudaGetLastError();
            occ = 0;
        }
        occ_cache[key] = occ;
    } else {
        occ = it->second;
    }
    fell_back = true;
    if (occ < 1) return RS_OK;
    const u64 TW = (u64)TL_T * TL_W;
    const u64 NT = (words + TW - 1) / TW;
    if (NT >= (1ULL << 31)) return RS_OK;
    u64 G = (u64)c.sms * (u64)occ;
    if (G > (u64)TL_T) G = TL_T;  // one record load per thread in the finish
    if (G > NT) G = NT;
    rs_status rc = plan_segments(c, p, 0, 0, 0, st, true, 36, TL_W, (G * TL_T + BLOCK - 1) / BLOCK * BLOCK);
    if (rc) return rc;
    if (p.engine == RS_ENG_PCG64) {
        u128 inc = ((u128)p.base[3] << 64) | p.base[2], m, a;
        rs::pcg_affine(inc, (u128)G * TW, m, a);
        p.tile_m[0] = (u64)m; p.tile_m[1] = (u64)(m >> 64);
        p.tile_a[0] = (u64)a; p.tile_a[1] = (u64)(a >> 64);
    } else if (p.engine == RS_ENG_PHILOX) {
        for (int i = 0; i < 10; i++) {  // round keys k + r*W (counter.py:95-96)
            p.rk0[i] = p.base[4] + (u64)i * 0x9E3779B97F4A7C15ULL;
            p.rk1[i] = p.base[5] + (u64)i * 0xBB67AE8584CAA73BULL;
        }
    }
    if (NT + 1 > c.tile_rec_n) {
        cudaFree(c.tile_rec);
        c.tile_rec = nullptr;
        c.tile_rec_n = 0;
        const size_t cap = (size_t)(NT + 1) + (NT + 1) / 8 + 1024;
        CK(cudaMalloc(&c.tile_rec, cap * 8));
        CK(cudaMemsetAsync(c.tile_rec, 0, cap * 8, st));
        c.tile_rec_n = cap;
        c.tile_epoch = 0;
    }
    if (++c.tile_epoch == 0) {  // the epoch wrapped: clear the records once
        CK(cudaMemsetAsync(c.tile_rec, 0, c.tile_rec_n * 8, st));
        c.tile_epoch = 1;
    }
    p.tile_rec = c.tile_rec;
    p.tile_nt = (u32)NT;
    p.tile_epoch = c.tile_epoch;
    CK(cudaMemsetAsync(c.res, 0, offsetof(DevResult, serial_state), st));
    DevResult *res = c.res;
    void *args[] = {&p, &res};
    if ((rc = launch(fn, dim3((unsigned)G), dim3(TL_T), args, st, TL_SMEM))) return rc;
    CK(cudaMemcpyAsync(c.res_host, c.res, offsetof(DevResult, serial_state), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    fell_back = c.res_host->pad != 0;
    if (getenv("RS_TILE_DEBUG"))
        fprintf(stderr, "[tile] NT=%llu G=%llu P=%d lp0=%llu n=%llu total=%llu end=%llu next=%llu pad=%u\n", (unsigned long long)NT,
                (unsigned long long)G, p.P, (unsigned long long)p.lp0, (unsigned long long)p.n,
                (unsigned long long)c.res_host->total, (unsigned long long)c.res_host->end_pos,
                (unsigned long long)c.res_host->next_start, c.res_host->pad);
    return RS_OK;
}

// The device part of one fill. On return (sync=true) `E` holds the stream units
// consumed (64-bit words, or 32-bit halves incl. a used pending half when r.unit == 2)
// and `tal` the tallies.
rs_status run_fill(DevCtx &c, const rs_stream *s, const Resolved &r, u64 n, void *dout, cudaStream_t st, bool sync,
                   u64 &E, u64 *tal, int &rounds, u64 &chunks) {
    E = 0;
    rounds = 0;
    chunks = 0;
    c.range.valid = false;
    for (int i = 0; i < 6; i++) tal[i] = 0;
    if (n == 0) return RS_OK;
    FillPlan p;
    memset(&p, 0, sizeof p);
    fill_plan_common(p, c, r, s->engine, s->full_mantissa);
    stream_prefix(s, p);
    p.out = dout;
    p.out0 = 0;
    memcpy(p.base, s->state, sizeof p.base);
    memcpy(p.lanes, s->state, sizeof p.lanes);
    const u64 u = (u64)r.unit;
    p.pending_used = (u == 2 && s->has_pending) ? 1 : 0;
    p.pending_val = (u32)s->pending;
    rs_status rc;

    if (is_serial(s->engine)) {  // sfc64 / sfc64simd single stream: no skip-ahead, serial
        p.n = n;
        if (s->engine == RS_ENG_SFC64_SIMD) memcpy(p.lanes, s->state, sizeof p.lanes);
        DevResult *res = c.res;
        void *args[] = {&p, &res};
        rc = launch(serial_kernel(s->engine, r.family, r.fixed_mode), dim3(1), dim3(32), args, st);
        if (rc) return rc;
        if (sync) {
            CK(cudaMemcpyAsync(c.res_host, c.res, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            E = c.res_host->end_pos;
            for (int i = 0; i < 6; i++) tal[i] = c.res_host->tally[i];
        }
        chunks = 1;
        return RS_OK;
    }

    if (r.fixed_mode >= 0) {
        // fixed consumption: sample i <- logical unit i
        u64 words = u == 2 ? (n - p.pending_used + 1) / 2 : n;
        p.n = n;
        p.weng = words > (u64)p.P ? words - p.P : 0;
        if (s->engine == RS_ENG_PHILOX) {
            const void *fn = philox_kernel(r.fixed_mode);
            // round keys k + r*W (counter.py:95-96) live in the constant bank
            for (int i = 0; i < 10; i++) {
                p.rk0[i] = p.base[4] + (u64)i * 0x9E3779B97F4A7C15ULL;
                p.rk1[i] = p.base[5] + (u64)i * 0xBB67AE8584CAA73BULL;
            }
            uintptr_t a = (uintptr_t)dout;
            if (u == 2)
                p.vec_ok = ((a + 4 * ((u64)p.pending_used + 2ULL * p.P)) & 31) == 0;
            else
                p.vec_ok = ((a + 8ULL * p.P) & 31) == 0;
            u64 nblk = (p.weng + 3) / 4;
            u64 g = (u64)c.sms * occupancy(fn);
            u64 need = (nblk + BLOCK - 1) / BLOCK;
            if (need < g) g = need;
            if (g < 1) g = 1;
            void *args[] = {&p};
            rc = launch(fn, dim3((unsigned)g), dim3(BLOCK), args, st);
            if (rc) return rc;
            E = n;
            chunks = 1;
            return RS_OK;
        }
        if (rs::simd_engine(s->engine)) {
            if ((rc = launch_simd(c, p, r.fixed_mode, st))) return rc;
            E = n;
            chunks = 1;
            return RS_OK;
        }
        const void *fn = fixed_kernel(s->engine, r.fixed_mode);
        int focc = occupancy(fn, FX_SMEM);
        if (s->engine == RS_ENG_X256SS || s->engine == RS_ENG_X256PP || s->engine == RS_ENG_X128P || s->engine == RS_ENG_XORO) {
            // the GF(2) jump setup costs per thread: below ~1500 words per thread fewer resident
            // blocks win (x256** raw 2^26: 0.240 ms at 3 blocks/SM, 0.183 at 1; 2^30 keeps 3)
            const u64 k = p.weng / ((u64)c.sms * BLOCK * 1536);
            focc = (int)std::max<u64>(1, std::min<u64>((u64)focc, k));
        }
        rc = plan_segments(c, p, p.weng ? p.weng : 1, 64, focc, st, true, 144);
        if (rc) return rc;
        if ((rc = launch_fixed(c, p, fn, st))) return rc;
        E = n;
        chunks = 1;
        return RS_OK;
    }

    // variable consumption: chunks of provisioned words until n samples exist.
    // Chunk coordinates: chunk-local position lp in units; chunk 1 starts with the
    // pending half (u = 2) and the P buffered words, then the engine; a later chunk
    // has neither and lp counts engine units from its origin (thread 0 starts at lp0).
    VarKernels K = var_kernels(s->engine, r.family);
    const void *tile_fn = nullptr;
    if (sync && u == 1 && (r.family == FAM_NORM || r.family == FAM_EXP) && !(r.family == FAM_NORM && r.kind == NK_SKEW) &&
        getenv("RS_TILE"))  // (opt-in until it beats the two-pass path)
        tile_fn = rsk::tile_kernel(s->engine, r.family);
    const u64 P1 = (u64)p.P, pp1 = (u64)p.pending_used;
    u64 done = 0;    // samples produced so far
    u64 origin = 0;  // engine words from s->state to this chunk's origin (multiple of 36)
    u64 lp0 = 0;
    u64 Lmin = var_lmin(r);
    bool first = true;
    while (done < n) {
        u64 need = n - done;
        double ww = (double)need * r.words_per_sample;
        u64 words = (u64)(ww * 1.01 + 12.0 * std::sqrt(ww) + 2048.0);
        if (!first) {
            p.P = 0;
            p.pending_used = 0;
            u64 st32[32];
            memcpy(st32, s->state, sizeof st32);
            if (!rs::engine_advance_words(s->engine, st32, (u128)origin)) {
                rs::set_error("cannot position engine");
                return RS_ERR_INTERNAL;
            }
            memcpy(p.base, st32, sizeof p.base);
            memcpy(p.lanes, st32, sizeof p.lanes);
        }
        p.lp0 = lp0;
        p.n = need;
        p.out0 = done;
        if (tile_fn && need >= TILE_MIN_N) {
            // single-pass tile parse (rs_tile.cuh); a chunk outside its model (flag) is redone below
            bool fell_back = false;
            if ((rc = run_tile_chunk(c, p, tile_fn, words + lp0, st, fell_back))) return rc;
            if (!fell_back) {
                chunks++;
                for (int i = 0; i < 6; i++) tal[i] += c.res_host->tally[i];
                const u64 total = c.res_host->total;
                const u64 to_engine = first ? (u64)0 - (u * P1 + pp1) : u * origin;
                if (done + total >= n) {
                    E = u * P1 + pp1 + (c.res_host->end_pos + to_engine);
                    break;
                }
                done += total;
                const u64 resume = c.res_host->next_start + to_engine;
                origin = resume / u / 72 * 72;
                lp0 = resume - u * origin;
                first = false;
                continue;
            }
        }
        int occ = std::min(occupancy(K.count), std::min(occupancy(K.fixup), occupancy(K.emit)));
        const bool mem = parse_from_memory(s->engine);
        rc = plan_segments(c, p, words + (lp0 + u - 1) / u, Lmin, occ, st, !mem);
        if (rc) return rc;
        if ((rc = prep_chunk(c, p, r, mem, st))) return rc;
        CK(cudaMemsetAsync(c.res, 0, offsetof(DevResult, serial_state), st));
        unsigned g = p.T / BLOCK;
        int round = 0;
        DevResult *res = c.res;
        {
            void *a1[] = {&p, &c.cnt0, &c.ex0, &c.cnt1, &c.ex1};
            if ((rc = launch(K.count, dim3(g), dim3(BLOCK), a1, st))) return rc;
            const u32 *prev = c.ex0;
            void *a2[] = {&p, &c.cnt0, &c.ex0, &c.cnt1, &c.ex1, &prev, &c.entry, &c.cnt, &c.exA, &round, &res, &c.bsum};
            if ((rc = launch(K.fixup, dim3(g), dim3(BLOCK), a2, st))) return rc;
        }
        u32 *ex_cur = c.exA, *ex_other = c.exB;
        for (;;) {
            // (no scan launch: the fixup left per-block count sums, the emit blocks finish the offsets)
            void *a3[] = {&p, &c.entry, &c.cnt, &c.bsum, &ex_cur, &res};
            if ((rc = launch(K.emit, dim3(g), dim3(BLOCK), a3, st))) return rc;
            if (!sync) { chunks++; return RS_OK; }
            CK(cudaMemcpyAsync(c.res_host, c.res, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (!c.res_host->flag) break;
            // entries not at a fixed point: iterate the resolution (SURVEY 7.2#1 fallback)
            // after round k threads 0..k have final exits, so p.T rounds always suffice
            if (++round > (int)p.T) { rs::set_error("segment entry resolution did not converge"); return RS_ERR_INTERNAL; }
            rounds++;
            CK(cudaMemsetAsync(c.res, 0, offsetof(DevResult, serial_state), st));
            const u32 *prev = ex_cur;
            void *a2[] = {&p, &c.cnt0, &c.ex0, &c.cnt1, &c.ex1, &prev, &c.entry, &c.cnt, &ex_other, &round, &res, &c.bsum};
            if ((rc = launch(K.fixup, dim3(g), dim3(BLOCK), a2, st))) return rc;
            u32 *tmp = ex_cur; ex_cur = ex_other; ex_other = tmp;
        }
        chunks++;
        if (mem) {
            u32 over = 0, zero = 0;
            CK(cudaMemcpy(&over, c.overrun, sizeof over, cudaMemcpyDeviceToHost));
            if (over) {
                CK(cudaMemcpy(c.overrun, &zero, sizeof zero, cudaMemcpyHostToDevice));
                rs::set_error("parse ran past the materialized words (raise the slack)");
                return RS_ERR_INTERNAL;
            }
        }
        for (int i = 0; i < 6; i++) tal[i] += c.res_host->tally[i];
        u64 total = c.res_host->total;
        // chunk-local units -> engine units (from s->state) and whole-fill units
        u64 to_engine = first ? (u64)0 - (u * P1 + pp1) : u * origin;
        if (done + total >= n) {
            E = u * P1 + pp1 + (c.res_host->end_pos + to_engine);
            break;
        }
        done += total;
        u64 resume = c.res_host->next_start + to_engine;  // engine unit of the next boundary
        origin = resume / u / 72 * 72;  // whole Philox / ranlux / 8-word blocks
        lp0 = resume - u * origin;
        first = false;
    }
    return RS_OK;
}

// which reference tallies a fill touches (continuous.py:32-33: std_norm, std_exp, gamma)
void tally_seen(const Resolved &r, int32_t *seen) {
    seen[0] = seen[1] = seen[2] = 0;
    if (r.family == FAM_NORM) seen[0] = 1;
    if (r.family == FAM_EXP) seen[1] = 1;
    if (r.family == FAM_GAMMA) { seen[0] = 1; seen[2] = 1; }
}

// Restores the caller's current device on every return path: the entry points switch to
// the output pointer's device, and a Python caller's torch current device must not move.
struct DeviceGuard {
    int prev = -1;
    DeviceGuard() {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

rs_status check_stream(const rs_stream *s) {
    if (!s) { rs::set_error("null stream"); return RS_ERR_VALUE; }
    if (!rs::device_engine(s->engine)) { rs::set_error("engine not on the B200 fill path"); return RS_ERR_UNSUPPORTED; }
    if (s->fill < 0 || s->fill > CAP || s->cursor < 0 || s->cursor > s->fill) {
        rs::set_error("buffer cursor out of range");
        return RS_ERR_VALUE;
    }
    return RS_OK;
}

}  // namespace

// ============================================================================= C ABI
extern "C" {

rs_status rs_init_device(int32_t device) {
    std::lock_guard<std::mutex> g(g_mu);
    DeviceGuard dg;
    CK(cudaSetDevice(device));
    DevCtx *c;
    rs_status s = init_dev(device, &c);
    if (s == RS_OK) rs::clear_error();
    return s;
}

// rs_fill with g_mu already held by the caller (rs_fill, mvn_core)
static rs_status fill_locked(rs_stream *s, int32_t dist, const double *fparams, const uint64_t *iparams, uint64_t n,
                             void *out, rs_fill_result *result, void *cuda_stream) {
    DeviceGuard dg;
    rs_status rc = check_stream(s);
    if (rc) return rc;
    double fz[4] = {0, 0, 0, 0};
    u64 iz[4] = {0, 0, 0, 0};
    Resolved r;
    rc = resolve(dist, fparams ? fparams : fz, iparams ? iparams : iz, r);
    if (rc) return rc;
    if (result) memset(result, 0, sizeof *result);
    if (n == 0) { rs::clear_error(); return RS_OK; }  // the reference consumes nothing for n == 0
    if (!out) { rs::set_error("null output"); return RS_ERR_VALUE; }
    int dev;
    if (is_device_ptr(out)) {
        cudaPointerAttributes a;
        CK(cudaPointerGetAttributes(&a, out));
        dev = a.device;
        CK(cudaSetDevice(dev));
    } else {
        CK(cudaGetDevice(&dev));
    }
    DevCtx *c;
    if ((rc = init_dev(dev, &c))) return rc;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    size_t bytes = (size_t)n * elem_size(dist);
    Staging sg;
    if ((rc = get_out(*c, out, bytes, sg))) return rc;
    u64 Eu, tal[6];
    int rounds;
    u64 chunks;
    if ((rc = run_fill(*c, s, r, n, sg.dptr, st, true, Eu, tal, rounds, chunks))) return rc;
    if (sg.host) {
        CK(cudaMemcpyAsync(out, sg.dptr, bytes, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    // stream position after the fill (buffer.py:29-49)
    int P = s->fill - s->cursor;
    u64 pre_words[CAP];
    for (int i = 0; i < P; i++) pre_words[i] = s->buf[s->cursor + i];
    u64 E;            // 64-bit words taken from the buffer / engine
    bool odd = false; // a u32 consumer ended on a low half: the high half stays pending
    if (r.unit == 2) {
        u64 pp = s->has_pending ? 1 : 0;
        u64 rel = Eu > pp ? Eu - pp : 0;
        E = (rel + 1) / 2;
        odd = rel & 1;
    } else {
        E = Eu;
    }
    if ((rc = apply_consumption(s, E, is_serial(s->engine) ? c->res_host : nullptr))) return rc;
    if (odd) {
        u64 last = E - 1;
        u64 w = last < (u64)P ? pre_words[last] : s->buf[s->cursor - 1];
        s->has_pending = 1;
        s->pending = w >> 32;
    } else {
        s->has_pending = 0;
        s->pending = 0;
    }
    if (result) {
        result->words_consumed = E;
        for (int i = 0; i < 6; i++) result->tally[i] = tal[i];
        tally_seen(r, result->tally_seen);
        result->resync_rounds = rounds;
        result->chunks = chunks;
    }
    rs::clear_error();
    return RS_OK;
}

rs_status rs_fill(rs_stream *s, int32_t dist, const double *fparams, const uint64_t *iparams, uint64_t n, void *out,
                  rs_fill_result *result, void *cuda_stream) {
    std::lock_guard<std::mutex> g(g_mu);
    return fill_locked(s, dist, fparams, iparams, n, out, result, cuda_stream);
}

rs_status rs_fill_async(const rs_stream *s, int32_t dist, const double *fparams, const uint64_t *iparams, uint64_t n,
                        void *out_device, void *cuda_stream) {
    std::lock_guard<std::mutex> g(g_mu);
    rs_status rc = check_stream(s);
    if (rc) return rc;
    double fz[4] = {0, 0, 0, 0};
    u64 iz[4] = {0, 0, 0, 0};
    Resolved r;
    rc = resolve(dist, fparams ? fparams : fz, iparams ? iparams : iz, r);
    if (rc) return rc;
    // A variable-consumption fill needs host round trips (the resolution flag, further
    // fixup rounds, a second provisioning chunk, the overrun check): rs_fill only.
    if (r.fixed_mode < 0 || is_serial(s->engine)) {
        rs::set_error("rs_fill_async covers fixed-consumption laws on skip-ahead engines; use rs_fill");
        return RS_ERR_UNSUPPORTED;
    }
    if (n == 0) return RS_OK;
    int dev;
    CK(cudaGetDevice(&dev));
    DevCtx *c;
    if ((rc = init_dev(dev, &c))) return rc;
    u64 E, tal[6];
    int rounds;
    u64 chunks;
    rc = run_fill(*c, s, r, n, out_device, (cudaStream_t)cuda_stream, false, E, tal, rounds, chunks);
    if (rc == RS_OK) rs::clear_error();
    return rc;
}

rs_status rs_fill_streams(int32_t engine, const uint64_t *seed, int32_t n_seed, const uint64_t *spawn_prefix,
                          int32_t n_prefix, uint64_t j0, uint64_t n_streams, int32_t dist, const double *fparams,
                          const uint64_t *iparams, uint64_t n_per_stream, void *out, void *cuda_stream) {
    std::lock_guard<std::mutex> g(g_mu);
    DeviceGuard dg;
    if (engine != RS_ENG_SFC64 && engine != RS_ENG_PCG64 && engine != RS_ENG_PHILOX && engine != RS_ENG_X256SS &&
        engine != RS_ENG_X256PP && engine != RS_ENG_X128P && engine != RS_ENG_XORO && engine != RS_ENG_SQUARES &&
        engine != RS_ENG_CHACHA20 && engine != RS_ENG_CWG128) {
        rs::set_error("per-stream mode supports sfc64, pcg64, philox, x256**, x256++, x128+, xoro++, squares, chacha20, cwg128");
        return RS_ERR_UNSUPPORTED;
    }
    if (n_seed < 0 || n_seed > 16 || n_prefix < 0 || n_prefix > 7) {
        rs::set_error("seed / spawn key too long");
        return RS_ERR_VALUE;
    }
    double fz[4] = {0, 0, 0, 0};
    u64 iz[4] = {0, 0, 0, 0};
    Resolved r;
    rs_status rc = resolve(dist, fparams ? fparams : fz, iparams ? iparams : iz, r);
    if (rc) return rc;
    if (n_streams == 0 || n_per_stream == 0) { rs::clear_error(); return RS_OK; }
    int dev;
    if (is_device_ptr(out)) {
        cudaPointerAttributes a;
        CK(cudaPointerGetAttributes(&a, out));
        dev = a.device;
        CK(cudaSetDevice(dev));
    } else {
        CK(cudaGetDevice(&dev));
    }
    DevCtx *c;
    if ((rc = init_dev(dev, &c))) return rc;
    c->range.valid = false;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    size_t bytes = (size_t)n_streams * n_per_stream * elem_size(dist);
    Staging sg;
    if ((rc = get_out(*c, out, bytes, sg))) return rc;
    StreamArgs a;
    memset(&a, 0, sizeof a);
    a.engine = engine;
    a.nseed = n_seed;
    a.nprefix = n_prefix;
    for (int i = 0; i < n_seed; i++) a.seed[i] = seed[i];
    for (int i = 0; i < n_prefix; i++) a.prefix[i] = spawn_prefix[i];
    a.j0 = j0;
    a.nstreams = n_streams;
    a.nper = n_per_stream;
    a.dist = r.dist;
    a.fm = 0;
    memcpy(a.fp, r.fp, sizeof a.fp);
    memcpy(a.ip, r.ip, sizeof a.ip);
    a.ga = r.ga;
    a.gb = r.gb;
    a.kind = r.kind;
    a.zslow = (r.table == 0 || r.table == 1) ? c->zslow[r.table] : nullptr;
    a.zfast = (r.table == 0 || r.table == 1) ? c->zfast[r.table] : nullptr;
    a.zslowf = (r.table == 2 || r.table == 3) ? c->zslowf[r.table - 2] : nullptr;
    a.zfastf = (r.table == 2 || r.table == 3) ? c->zfastf[r.table - 2] : nullptr;
    a.rlx_A = c->rlxA;
    a.out = sg.dptr;
    int d = r.family;
    if (r.fixed_mode == FX_POW2) {  // b = 2^k: Lemire without a rejection zone
        d = FAM_LEMIRE;
        a.ip[0] = r.ip[0];
        a.ip[1] = 0;
        a.ip[2] = 0;
    } else if (r.fixed_mode == FX_HMAP && r.kind == HK_POW2) {
        d = FAM_U32;
        a.ip[0] = r.ip[0];
        a.ip[1] = 0;
        a.ip[2] = 0;
        a.ip[3] = r.ip[1];
    } else if (r.fixed_mode >= 0) {  // raw / u01 / u01f / unif / gumbel / masks / full spans
        d = FAM_FIXED;
        a.fmode = r.fixed_mode;
        memcpy(a.ip, r.ip, sizeof a.ip);
    }
    // Lemire with a rejection zone above 1/16 of the words (b close above a power of two,
    // e.g. 2^63+1): the word-level chunk ring; otherwise the unrolled 32-sample chunks, whose
    // smaller tile keeps 2^16 streams in one wave
    if (d == FAM_LEMIRE && a.ip[1] > (1ULL << 60)) d = FAM_LEMIRE_RING;
    const void *fn = rsk::streams_kernel(engine, d);
    void *args[] = {&a};
    unsigned g2 = (unsigned)((n_streams + STR_BLOCK - 1) / STR_BLOCK);
    if ((rc = launch(fn, dim3(g2), dim3(STR_BLOCK), args, st, d == FAM_LEMIRE_RING ? ST_SMEM_RING : ST_SMEM)))
        return rc;
    if (sg.host) {
        CK(cudaMemcpyAsync(out, sg.dptr, bytes, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    CK(cudaGetLastError());
    rs::clear_error();
    return RS_OK;
}

// rs_mvn (zext == nullptr: z drawn here from `s`) and rs_mvn_apply (z given, on the device).
// One lock from the scratch sizing to the final synchronisation: the per-device scratch
// (z, the factor, the mean, the staging buffer) is shared by every caller on the device.
// One launch of the contraction for `rows` samples: X = mean + z L^T, z rows x d
// (row-major), X rows x d (layout 0) or columns [0, rows) of a d x ldx matrix (layout 1).
static rs_status mvn_contract(const double *z, const double *Ld, const double *md, double *X, u64 rows, int64_t d,
                              int32_t layout, long long ldx, int lower, cudaStream_t st) {
    // 16-byte copies need an even d (rows 16-byte aligned) and aligned bases
    const bool vec16 = d % 2 == 0 && (((uintptr_t)z | (uintptr_t)Ld | (uintptr_t)X) & 15) == 0;
    rsk::MvnLaunch ml = rsk::mvn_kernel(vec16 ? 1 : 0, layout);
    CK(cudaFuncSetAttribute(ml.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ml.smem));
    long long nn = (long long)rows;
    int dd = (int)d;
    int ntn = (dd + ml.bn - 1) / ml.bn;
    unsigned long long blocks = (unsigned long long)((rows + ml.bm - 1) / ml.bm) * (unsigned long long)ntn;
    if (blocks > 0x7FFFFFFFULL) { rs::set_error("mvn too large for one launch"); return RS_ERR_VALUE; }
    void *args[] = {&z, &Ld, &md, &X, &nn, &dd, &lower, &ntn, &ldx};
    return launch(ml.fn, dim3((unsigned)blocks), dim3(ml.threads), args, st, ml.smem);
}

// A Cholesky factor is lower triangular (exact zeros above the diagonal): the kernel
// skips the zero products. The pivoted semidefinite factor (continuous.py:293-309) is
// not, and takes the full product.
static int host_lower(const double *Lh, int64_t d) {
    for (int64_t r = 0; r < d; r++)
        for (int64_t q = r + 1; q < d; q++)
            if (Lh[r * d + q] != 0.0) return 0;
    return 1;
}

static rs_status mvn_core(rs_stream *s, const double *L, const double *mean, int64_t d, uint64_t n, int32_t layout,
                          const double *zext, double *out, rs_fill_result *result, void *cuda_stream) {
    if (d < 1 || n < 1) { rs::set_error("mvn needs n >= 1"); return RS_ERR_VALUE; }
    if (layout != 0 && layout != 1) { rs::set_error("mvn layout must be 'n_d' or 'd_n'"); return RS_ERR_VALUE; }
    if (d > (1 << 20)) { rs::set_error("mvn dimension too large"); return RS_ERR_VALUE; }
    std::lock_guard<std::mutex> g(g_mu);
    DeviceGuard dg;
    rs_status rc;
    if (!zext && (rc = check_stream(s))) return rc;
    if (zext && !is_device_ptr(zext)) { rs::set_error("mvn z must be device memory"); return RS_ERR_VALUE; }
    int dev;
    if (is_device_ptr(out)) {
        cudaPointerAttributes a;
        CK(cudaPointerGetAttributes(&a, out));
        dev = a.device;
        CK(cudaSetDevice(dev));
    } else {
        CK(cudaGetDevice(&dev));
    }
    DevCtx *c;
    if ((rc = init_dev(dev, &c))) return rc;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const size_t nz = (size_t)n * (size_t)d;
    // z (unless given), the factor and the mean in device memory; offsets keep 16-byte alignment
    const size_t zb = zext ? 0 : (nz * 8 + 15) / 16 * 16, lb = ((size_t)d * d * 8 + 15) / 16 * 16;
    const size_t need = zb + lb + (size_t)d * 8;
    if (need > c->mvn_bytes) {
        cudaFree(c->mvn_z);
        c->mvn_z = nullptr;
        c->mvn_bytes = 0;
        CK(cudaMalloc(&c->mvn_z, need));
        c->mvn_bytes = need;
    }
    double *zbuf = c->mvn_z, *Ld = (double *)((char *)c->mvn_z + zb), *md = (double *)((char *)c->mvn_z + zb + lb);
    int lower;
    if (is_device_ptr(L)) {
        std::vector<double> hl((size_t)d * d);
        CK(cudaMemcpyAsync(hl.data(), L, (size_t)d * d * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        lower = host_lower(hl.data(), d);
    } else {
        lower = host_lower(L, d);
    }
    CK(cudaMemcpyAsync(Ld, L, (size_t)d * d * 8, cudaMemcpyDefault, st));
    CK(cudaMemcpyAsync(md, mean, (size_t)d * 8, cudaMemcpyDefault, st));
    const bool host_out = !is_device_ptr(out);
    double *X;
    if (host_out) {
        if (nz * 8 > c->stage_bytes) {
            cudaFree(c->stage);
            c->stage = nullptr;
            c->stage_bytes = 0;
            CK(cudaMalloc(&c->stage, nz * 8));
            c->stage_bytes = nz * 8;
        }
        X = (double *)c->stage;
    } else {
        X = out;
    }
    rs_fill_result fr;
    memset(&fr, 0, sizeof fr);
    // (A z fill does not overlap the contraction: at 2 blocks/SM the contraction holds the
    // whole register file, so no parse block can be co-resident; measured with
    // tools/mvn_overlap.py, the two on separate streams take the sum of their times.)
    if (!zext && (rc = fill_locked(s, RS_DIST_STDNORM, nullptr, nullptr, nz, zbuf, &fr, cuda_stream))) return rc;
    if ((rc = mvn_contract(zext ? zext : zbuf, Ld, md, X, n, d, layout, (long long)n, lower, st))) return rc;
    if (host_out) CK(cudaMemcpyAsync(out, X, nz * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    if (result) *result = fr;
    rs::clear_error();
    return RS_OK;
}

rs_status rs_mvn(rs_stream *s, const double *L, const double *mean, int64_t d, uint64_t n, int32_t layout,
                 double *out, rs_fill_result *result, void *cuda_stream) {
    return mvn_core(s, L, mean, d, n, layout, nullptr, out, result, cuda_stream);
}

rs_status rs_mvn_apply(const double *L, const double *mean, int64_t d, uint64_t n, int32_t layout,
                       const double *z_device, double *out, void *cuda_stream) {
    return mvn_core(nullptr, L, mean, d, n, layout, z_device, out, nullptr, cuda_stream);
}

rs_status rs_mvn_apply_rows(const double *L_device, const double *mean_device, int64_t d, int32_t lower,
                            uint64_t rows, const double *z_device, int32_t layout, double *out_device,
                            int64_t ld_out, void *cuda_stream) {
    if (d < 1 || d > (1 << 20)) { rs::set_error("mvn dimension out of range"); return RS_ERR_VALUE; }
    if (layout != 0 && layout != 1) { rs::set_error("mvn layout must be 'n_d' or 'd_n'"); return RS_ERR_VALUE; }
    if (rows == 0) { rs::clear_error(); return RS_OK; }
    if (!is_device_ptr(L_device) || !is_device_ptr(mean_device) || !is_device_ptr(z_device) ||
        !is_device_ptr(out_device)) {
        rs::set_error("rs_mvn_apply_rows takes device pointers");
        return RS_ERR_VALUE;
    }
    if (layout == 1 && ld_out < (int64_t)rows) { rs::set_error("mvn ld_out < rows"); return RS_ERR_VALUE; }
    DeviceGuard dg;
    cudaPointerAttributes a;
    CK(cudaPointerGetAttributes(&a, out_device));
    CK(cudaSetDevice(a.device));
    rs_status rc = mvn_contract(z_device, L_device, mean_device, out_device, rows, d, layout,
                                layout == 1 ? (long long)ld_out : (long long)rows, lower ? 1 : 0,
                                (cudaStream_t)cuda_stream);
    if (rc) return rc;
    CK(cudaGetLastError());
    rs::clear_error();
    return RS_OK;
}

// ----------------------------------------------------------------------------- sharded fills
// One rank's slice of a variable-consumption fill. The stream is at the
// slice start (fresh: no buffered words, no pending half); the slice is seg_len * n_seg
// engine words, parsed as n_seg segments; its samples are those that START in
// [entry, units(slice)). rs_range_count runs count + fixup (+ resolution rounds) + scan
// and reports the count and the exit; rs_range_emit writes the first `keep` samples.

rs_status rs_dist_info(int32_t dist, const double *fparams, const uint64_t *iparams, rs_dist_info_t *info) {
    double fz[4] = {0, 0, 0, 0};
    u64 iz[4] = {0, 0, 0, 0};
    Resolved r;
    rs_status rc = resolve(dist, fparams ? fparams : fz, iparams ? iparams : iz, r);
    if (rc) return rc;
    info->unit = r.unit;
    info->variable = r.fixed_mode < 0 ? 1 : 0;
    info->words_per_sample = r.words_per_sample;
    info->min_seg_len = r.fixed_mode < 0 ? range_lmin(r) : RS_RANGE_ALIGN;
    tally_seen(r, info->tally_seen);
    info->pad = 0;
    rs::clear_error();
    return RS_OK;
}

rs_status rs_range_geometry(int32_t engine, int32_t dist, const double *fparams, const uint64_t *iparams,
                            uint64_t words, uint64_t *seg_len, uint32_t *n_seg) {
    std::lock_guard<std::mutex> g(g_mu);
    double fz[4] = {0, 0, 0, 0};
    u64 iz[4] = {0, 0, 0, 0};
    Resolved r;
    rs_status rc = resolve(dist, fparams ? fparams : fz, iparams ? iparams : iz, r);
    if (rc) return rc;
    if (r.fixed_mode >= 0 || is_serial(engine) || !rs_engine_supported(engine)) {
        rs::set_error("range fills cover variable-consumption laws on skip-ahead engines");
        return RS_ERR_UNSUPPORTED;
    }
    int dev;
    CK(cudaGetDevice(&dev));
    DevCtx *c;
    if ((rc = init_dev(dev, &c))) return rc;
    VarKernels K = var_kernels(engine, r.family);
    int occ = std::min(occupancy(K.count), std::min(occupancy(K.fixup), occupancy(K.emit)));
    u64 Tfull = (u64)c->sms * (u64)occ * BLOCK;  // one wave, as plan_segments
    u64 L = (words + Tfull - 1) / Tfull;
    if (L < range_lmin(r)) L = range_lmin(r);
    L = (L + RS_RANGE_ALIGN - 1) / RS_RANGE_ALIGN * RS_RANGE_ALIGN;
    u64 T = (words + L - 1) / L;
    T = (T + BLOCK - 1) / BLOCK * BLOCK;
    if (T < BLOCK) T = BLOCK;
    if (T > 0xFFFFFFFFULL) { rs::set_error("slice too large"); return RS_ERR_VALUE; }
    *seg_len = L;
    *n_seg = (uint32_t)T;
    rs::clear_error();
    return RS_OK;
}

// count + exit of a slice of n_seg segments that follows n_warm warm-up segments (n_warm = 0:
// the slice alone, entering at `entry`; n_warm > 0: the plan starts at the warm-up window,
// whose first segment is assumed to start a sample, and the count / fixup passes resolve
// the slice's entry from the window's exit in the same launches)
static rs_status range_count_core(const rs_stream *s, int32_t dist, const double *fparams, const uint64_t *iparams,
                                  uint64_t entry, uint32_t n_warm, uint64_t seg_len, uint32_t n_seg, rs_range_info *info,
                                  void *cuda_stream) {
    rs_status rc = check_stream(s);
    if (rc) return rc;
    double fz[4] = {0, 0, 0, 0};
    u64 iz[4] = {0, 0, 0, 0};
    Resolved r;
    if ((rc = resolve(dist, fparams ? fparams : fz, iparams ? iparams : iz, r))) return rc;
    if (r.fixed_mode >= 0 || is_serial(s->engine)) {
        rs::set_error("range fills cover variable-consumption laws on skip-ahead engines");
        return RS_ERR_UNSUPPORTED;
    }
    if (s->cursor < s->fill || s->has_pending) {
        rs::set_error("a range fill starts at a fresh stream position (no buffered words)");
        return RS_ERR_VALUE;
    }
    if (seg_len == 0 || seg_len % RS_RANGE_ALIGN || n_seg == 0 || n_seg % BLOCK || n_warm % BLOCK ||
        (u64)n_warm + n_seg > 0xFFFFFFFFULL) {
        rs::set_error("range geometry: seg_len must be a multiple of 72 and n_seg, n_warm of 256");
        return RS_ERR_VALUE;
    }
    const u64 u = (u64)r.unit;
    if (entry >= u * seg_len) { rs::set_error("range entry beyond the first segment"); return RS_ERR_VALUE; }
    int dev;
    CK(cudaGetDevice(&dev));
    DevCtx *c;
    if ((rc = init_dev(dev, &c))) return rc;
    c->range.valid = false;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    FillPlan p;
    memset(&p, 0, sizeof p);
    fill_plan_common(p, *c, r, s->engine, s->full_mantissa);
    memcpy(p.base, s->state, sizeof p.base);
    memcpy(p.lanes, s->state, sizeof p.lanes);
    p.lp0 = n_warm ? 0 : entry;
    p.n = 0;
    p.n_warm = n_warm;
    const u32 Tall = n_warm + n_seg;
    VarKernels K = var_kernels(s->engine, r.family);
    const bool mem = parse_from_memory(s->engine);
    if ((rc = plan_segments(*c, p, seg_len * Tall, 0, 0, st, !mem, RS_RANGE_ALIGN, seg_len, Tall))) return rc;
    if ((rc = prep_chunk(*c, p, r, mem, st))) return rc;
    CK(cudaMemsetAsync(c->res, 0, offsetof(DevResult, serial_state), st));
    unsigned gdim = p.T / BLOCK;
    int round = 0;
    DevResult *res = c->res;
    void *a1[] = {&p, &c->cnt0, &c->ex0, &c->cnt1, &c->ex1};
    if ((rc = launch(K.count, dim3(gdim), dim3(BLOCK), a1, st))) return rc;
    const u32 *prev = c->ex0;
    u32 *ex_cur = c->exA, *ex_other = c->exB;
    void *a2[] = {&p, &c->cnt0, &c->ex0, &c->cnt1, &c->ex1, &prev, &c->entry, &c->cnt, &ex_cur, &round, &res, &c->bsum};
    if ((rc = launch(K.fixup, dim3(gdim), dim3(BLOCK), a2, st))) return rc;
    int rounds = 0;
    // The fixup zeroes the warm-up segments' counts and accumulates the slice's total, so
    // one read-back per round carries everything: the flag, the total, the last exit and
    // the window's exit (the slice's entry).
    u32 last_ex = 0, e32 = 0;
    for (;;) {  // entry resolution to a fixed point (as run_fill)
        CK(cudaMemcpyAsync(c->res_host, c->res, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&last_ex, ex_cur + (p.T - 1), 4, cudaMemcpyDeviceToHost, st));
        if (n_warm) CK(cudaMemcpyAsync(&e32, ex_cur + (n_warm - 1), 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (!c->res_host->flag) break;
        if (++round > (int)p.T) { rs::set_error("segment entry resolution did not converge"); return RS_ERR_INTERNAL; }
        rounds++;
        CK(cudaMemsetAsync(c->res, 0, offsetof(DevResult, serial_state), st));
        prev = ex_cur;
        void *a3[] = {&p, &c->cnt0, &c->ex0, &c->cnt1, &c->ex1, &prev, &c->entry, &c->cnt, &ex_other, &round, &res, &c->bsum};
        if ((rc = launch(K.fixup, dim3(gdim), dim3(BLOCK), a3, st))) return rc;
        u32 *tmp = ex_cur; ex_cur = ex_other; ex_other = tmp;
    }
    const u64 wentry = n_warm ? (u64)e32 : entry;  // the slice enters at the window's exit
    const u64 total = c->res_host->total;
    if (mem) {
        u32 over = 0, zero = 0;
        CK(cudaMemcpy(&over, c->overrun, sizeof over, cudaMemcpyDeviceToHost));
        if (over) {
            CK(cudaMemcpy(c->overrun, &zero, sizeof zero, cudaMemcpyHostToDevice));
            rs::set_error("parse ran past the materialized words (raise the slack)");
            return RS_ERR_INTERNAL;
        }
    }
    c->range.p = p;
    c->range.K = K;
    c->range.ex = ex_cur;
    c->range.count = total;
    c->range.unit = r.unit;
    c->range.mem = mem;
    c->range.origin = u * seg_len * (u64)n_warm;
    c->range.entry = wentry;
    c->range.valid = true;
    if (info) {
        memset(info, 0, sizeof *info);
        info->count = total;
        info->exit = last_ex;  // seg_end(T-1) == units(slice): the exit is past the slice end
        info->end_pos = wentry;
        info->unit = r.unit;
        info->resync_rounds = rounds;
    }
    rs::clear_error();
    return RS_OK;
}

rs_status rs_range_count(const rs_stream *s, int32_t dist, const double *fparams, const uint64_t *iparams,
                         uint64_t entry, uint64_t seg_len, uint32_t n_seg, rs_range_info *info, void *cuda_stream) {
    std::lock_guard<std::mutex> g(g_mu);
    return range_count_core(s, dist, fparams, iparams, entry, 0, seg_len, n_seg, info, cuda_stream);
}

rs_status rs_range_count_warm(const rs_stream *window_start, int32_t dist, const double *fparams,
                              const uint64_t *iparams, uint32_t n_warm, uint64_t seg_len, uint32_t n_seg,
                              rs_range_info *info, void *cuda_stream) {
    std::lock_guard<std::mutex> g(g_mu);
    if (n_warm == 0) { rs::set_error("rs_range_count_warm needs n_warm > 0 (else rs_range_count)"); return RS_ERR_VALUE; }
    return range_count_core(window_start, dist, fparams, iparams, 0, n_warm, seg_len, n_seg, info, cuda_stream);
}

rs_status rs_range_emit(uint64_t keep, void *out_device, rs_range_info *info, void *cuda_stream) {
    std::lock_guard<std::mutex> g(g_mu);
    int dev;
    CK(cudaGetDevice(&dev));
    DevCtx *c;
    rs_status rc;
    if ((rc = init_dev(dev, &c))) return rc;
    DevCtx::Range &R = c->range;
    if (!R.valid) { rs::set_error("no counted range on this device (another fill ran in between?)"); return RS_ERR_VALUE; }
    if (keep > R.count) { rs::set_error("keep exceeds the range's sample count"); return RS_ERR_VALUE; }
    if (info) {
        info->count = R.count;
        info->end_pos = R.entry;
        for (int i = 0; i < 6; i++) info->tally[i] = 0;
    }
    if (keep == 0) { rs::clear_error(); return RS_OK; }
    if (!out_device || !is_device_ptr(out_device)) { rs::set_error("range output must be device memory"); return RS_ERR_VALUE; }
    cudaStream_t st = (cudaStream_t)cuda_stream;
    FillPlan p = R.p;
    p.n = keep;
    p.out = out_device;
    p.out0 = 0;
    CK(cudaMemsetAsync(c->res, 0, offsetof(DevResult, serial_state), st));
    DevResult *res = c->res;
    void *a[] = {&p, &c->entry, &c->cnt, &c->bsum, &R.ex, &res};
    if ((rc = launch(R.K.emit, dim3(p.T / BLOCK), dim3(BLOCK), a, st))) return rc;
    CK(cudaMemcpyAsync(c->res_host, c->res, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    if (info) {
        info->end_pos = c->res_host->end_pos - R.origin;  // from the slice start
        for (int i = 0; i < 6; i++) info->tally[i] = c->res_host->tally[i];
    }
    rs::clear_error();
    return RS_OK;
}

}  // extern "C"
