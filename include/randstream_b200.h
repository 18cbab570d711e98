/*
 * randstream_b200.h -- C ABI of the B200-native bulk stream-fill library
 * (paper_2605_05099_b200/librandstream_b200.so).
 *
 * The reference (`randstream`, pure Python) has no FFI of its own; these entry
 * points replace the Python operator it exposes for this path and are what a
 * ctypes / cffi binding of that operator binds (INTEGRATION.md shows the stub):
 *
 *   rs_fill          replaces Rng.fill(dist, params, n)
 *                    /root/reference/pkg/src/randstream/rng.py:223-241
 *                    -> continuous.fill  continuous.py:413-431
 *                    -> discrete.fill    discrete.py:103-111
 *   rs_fill_streams  replaces the per-stream loop
 *                    `create(engine, seed, spawn_key=(j,)).fill(...)` over j
 *                    (state_io.py:13-19 + rng.py:223-241; spawn keys seeding.py:51-61)
 *   rs_mvn           replaces Rng.mvn(mean, cov, n, layout)  rng.py:273-275,
 *                    continuous.py:312-336 (the factor L is computed by the caller)
 *   rs_engine_*      the engine protocol used for stream positioning and the
 *                    144-word buffer refills: generate (engines/<name>.py generate),
 *                    seed (seeding.py:115-116 + engines seed_from), jump/advance
 *                    (rng.py:135-171, jumps.py:116-126, pcg.py:41-55, ranlux.py:90-93)
 *   rs_last_error    replaces the per-handle error slot (rng.py:38-52, state_io.py:45-47)
 *
 * Conventions: plain pointers and sizes only. `cuda_stream` is a cudaStream_t
 * passed as void* (NULL = legacy default stream). Output pointers may be
 * device memory (written in place, stream-ordered) or host memory (the
 * library stages through device scratch and copies back before returning).
 * All validation happens before any state change; on error the stream is
 * untouched and rs_last_error() describes the failure.
 */
#ifndef RANDSTREAM_B200_H
#define RANDSTREAM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 1
#define RS_BUFFER_CAPACITY 144 /* buffer.py:12 */

typedef enum {
    RS_OK = 0,
    RS_ERR_VALUE = 1,       /* ValueError in the reference */
    RS_ERR_UNSUPPORTED = 2, /* engine/dist not on the device path */
    RS_ERR_CUDA = 3,
    RS_ERR_INTERNAL = 4
} rs_status;

/* engine ids: the reference registry order, engines/__init__.py:11-26 */
typedef enum {
    RS_ENG_X256PP = 1,
    RS_ENG_X256SS = 2,
    RS_ENG_X128P = 3,
    RS_ENG_XORO = 4,
    RS_ENG_PCG64 = 5,
    RS_ENG_PHILOX = 6,
    RS_ENG_SQUARES = 7,
    RS_ENG_SFC64 = 8,
    RS_ENG_CWG128 = 9,
    RS_ENG_RANLUX = 10,
    RS_ENG_CHACHA20 = 11,
    RS_ENG_X256PP_SIMD = 12,
    RS_ENG_X256SS_SIMD = 13,
    RS_ENG_SFC64_SIMD = 14
} rs_engine;

/* distribution ids (continuous.py:339-359 / discrete.py:95-100 names) */
typedef enum {
    RS_DIST_UINT64 = 1,  /* "uint64": iparams[0]=b (0 = raw word), iparams[1]=1 means b = 2^64 */
    RS_DIST_U01 = 2,     /* "u01"   : f64, mapping per full_mantissa (rng.py:98-106) */
    RS_DIST_U01F = 3,    /* "u01f"  : f32 from u32 halves, low half first (rng.py:108-115) */
    RS_DIST_NORM = 4,    /* "norm"  : fparams {mu, var} */
    RS_DIST_EXP = 5,     /* "exp"   : fparams {beta} */
    RS_DIST_GAMMA = 6,   /* "gamma" : fparams {alpha, theta} */
    RS_DIST_BETA = 7,    /* "beta"  : fparams {a, b} */
    RS_DIST_STDNORM = 8, /* std_norm without the norm epilogue (the mvn z draws, continuous.py:332) */
    /* derived laws and transforms (continuous.py:136-290), bit-exact to the reference's
       bitexact mode (det_exp/det_log); within 4 ulp of its default numpy-vectorised mode */
    RS_DIST_UNIF = 9,         /* {a, b}                      f64 */
    RS_DIST_UNIFF = 10,       /* {a, b}                      f32, 32-bit halves */
    RS_DIST_NORMF = 11,       /* {mu, var}                   f32, 32-bit halves */
    RS_DIST_EXPF = 12,        /* {beta}                      f32, 32-bit halves */
    RS_DIST_LOGNORMAL = 13,   /* {mu, var} */
    RS_DIST_CHI2 = 14,        /* {nu} */
    RS_DIST_T = 15,           /* {nu} */
    RS_DIST_F = 16,           /* {nu1, nu2} */
    RS_DIST_GUMBEL = 17,      /* {mu, beta} */
    RS_DIST_PARETO = 18,      /* {alpha, xm} */
    RS_DIST_GPD = 19,         /* {xi, mu, sigma} */
    RS_DIST_WEIBULL = 20,     /* {k, lam} */
    RS_DIST_SKEW_NORMAL = 21, /* {alpha, mu, sigma} */
    /* integers (discrete.py:20-55): */
    RS_DIST_UINT32 = 22,      /* "uint8|16|32": iparams {b, width}           -> u32 on 32-bit halves */
    RS_DIST_INT32 = 23,       /* "int": iparams {span, 32, m, full_span}      -> i32 on 32-bit halves */
    RS_DIST_INT64 = 24        /* "long_long": iparams {span, 64, m, full_span} -> i64 */
} rs_dist;

/* A generator's full logical position (engine words + WordBuffer, buffer.py:17-60).
 * rs_fill reads it and writes back the post-fill position. */
typedef struct rs_stream {
    int32_t engine;         /* rs_engine */
    int32_t full_mantissa;  /* Rng.full_mantissa (rng.py:59-60) */
    int32_t bitexact;       /* Rng.bitexact (only affects transform families) */
    int32_t has_pending;    /* WordBuffer.pending is not None */
    uint64_t pending;       /* the buffered high half (u32) */
    uint64_t state[32];     /* engine.get_state() words (32 for the interleaved engines) */
    uint64_t buf[RS_BUFFER_CAPACITY];
    int32_t fill;           /* len(WordBuffer.words): 0 or 144 */
    int32_t cursor;         /* WordBuffer.cursor */
} rs_stream;

typedef struct rs_fill_result {
    uint64_t words_consumed;  /* logical 64-bit words taken from the stream */
    uint64_t tally[6];        /* norm attempts, norm pdf_evals, exp attempts, exp pdf_evals,
                                 gamma attempts, gamma pdf_evals (continuous.py:32-33) */
    int32_t tally_seen[3];    /* which of norm/exp/gamma the fill touched */
    int32_t resync_rounds;    /* extra segment-entry resolution rounds (0 normally) */
    uint64_t chunks;          /* provisioning rounds used */
} rs_fill_result;

/* library */
int32_t rs_abi_version(void);
const char *rs_last_error(void);                  /* thread-local, "" after a success */
rs_status rs_init_device(int32_t device);         /* upload constant tables once per device */
int32_t rs_engine_supported(int32_t engine);      /* 1 if rs_fill runs this engine on the GPU */

/* engine protocol (host-side state bookkeeping; the reference's L1/L1' layer) */
int32_t rs_engine_state_words(int32_t engine);
int32_t rs_engine_seed_words(int32_t engine);
int32_t rs_engine_chunk(int32_t engine);
rs_status rs_seed_words(const uint64_t *entropy, int32_t n_entropy, const uint64_t *spawn_key,
                        int32_t n_spawn, uint64_t *out, int32_t n_out);
rs_status rs_engine_seed(int32_t engine, const uint64_t *entropy, int32_t n_entropy,
                         const uint64_t *spawn_key, int32_t n_spawn, uint64_t *state_out);
rs_status rs_engine_seed_from(int32_t engine, const uint64_t *words, uint64_t *state_out);
rs_status rs_engine_check_state(int32_t engine, const uint64_t *words);
rs_status rs_engine_generate(int32_t engine, uint64_t *state, uint64_t *out, int32_t n);
rs_status rs_engine_jump(int32_t engine, uint64_t *state, int32_t k);
rs_status rs_engine_advance_words(int32_t engine, uint64_t *state, uint64_t words_lo, uint64_t words_hi);
rs_status rs_pcg_advance(uint64_t *state, uint64_t delta_lo, uint64_t delta_hi);

/* the hot path */
rs_status rs_fill(rs_stream *stream, int32_t dist, const double *fparams, const uint64_t *iparams,
                  uint64_t n, void *out, rs_fill_result *result, void *cuda_stream);

/* Launch-only variant for benchmarking/graph capture: same kernels, no host
 * synchronisation, `stream` is NOT advanced (each call recomputes the same fill). */
rs_status rs_fill_async(const rs_stream *stream, int32_t dist, const double *fparams,
                        const uint64_t *iparams, uint64_t n, void *out_device, void *cuda_stream);

/* per-stream mode: out[s][i] = create(engine, seed, spawn_key = prefix + (j0 + s,)).fill(...)[i] */
rs_status rs_fill_streams(int32_t engine, const uint64_t *seed, int32_t n_seed,
                          const uint64_t *spawn_prefix, int32_t n_prefix, uint64_t j0,
                          uint64_t n_streams, int32_t dist, const double *fparams,
                          const uint64_t *iparams, uint64_t n_per_stream, void *out,
                          void *cuda_stream);

/* x = mean + z @ L^T with z = n*d std_norm draws from `stream` (row-major (n, d)).
 * L: d x d row-major (device or host), mean: d (host). layout 0 = "n_d", 1 = "d_n". */
rs_status rs_mvn(rs_stream *stream, const double *L, const double *mean, int64_t d, uint64_t n,
                 int32_t layout, double *out, rs_fill_result *result, void *cuda_stream);

/* The contraction half of rs_mvn, for a caller that drew z itself (rs_fill of
 * RS_DIST_STDNORM, n*d values, device memory): x = mean + z @ L^T. It lets the
 * host factorise the covariance while the z fill runs (the reference computes
 * L first, continuous.py:312-336; the Python layer restores the stream if the
 * factorisation fails, so the observable order is the same). */
rs_status rs_mvn_apply(const double *L, const double *mean, int64_t d, uint64_t n, int32_t layout,
                       const double *z_device, double *out, void *cuda_stream);

/* The contraction for a block of `rows` samples, asynchronous and stream-ordered (no host
 * synchronisation), device pointers only: out = mean + z @ L^T for z rows x d row-major
 * (continuous.py:332-336 for those rows). layout 0: out is rows x d row-major; layout 1
 * ("d_n"): out points at column 0 of this block inside a d x ld_out row-major matrix
 * (ld_out = the whole fill's n). `lower` != 0 asserts that L is lower triangular (exact
 * zeros above the diagonal; the kernel then skips those products). The Python Rng.mvn
 * uses it with L and mean uploaded once; a caller may also split a large fill by rows. */
rs_status rs_mvn_apply_rows(const double *L_device, const double *mean_device, int64_t d, int32_t lower,
                            uint64_t rows, const double *z_device, int32_t layout, double *out_device,
                            int64_t ld_out, void *cuda_stream);

/* ---- multi-GPU sharding of variable-consumption fills ----
 * Replaces nothing one-for-one in the reference: it is the rank-local half of
 * `Rng.fill(dist, params, n)` (rng.py:223-241) when one logical stream is split
 * into contiguous word slices, one per GPU (paper_2605_05099_b200/shard.py runs
 * the protocol: warm-up entry guess, count, exchange of (entry, exit, count),
 * re-count on a mismatch, prefix offsets, emit). A slice is seg_len * n_seg
 * engine words of a stream positioned at its start (fresh: no buffered words,
 * no pending half); its samples are those that START at a unit position in
 * [entry, units(slice)), units = words, or 32-bit halves for the f32 laws. */
#define RS_RANGE_ALIGN 72 /* seg_len multiple: Philox blocks (4), ranlux chunks (9), 8-lane interleave */

typedef struct rs_dist_info_t {
    int32_t unit;              /* 1: 64-bit words, 2: 32-bit halves */
    int32_t variable;          /* 1: variable consumption (rejection samplers), 0: one unit per sample */
    double words_per_sample;   /* provisioning estimate (64-bit words per sample) */
    uint64_t min_seg_len;      /* shortest segment a range plan uses (multiple of RS_RANGE_ALIGN) */
    int32_t tally_seen[3];     /* which of the norm/exp/gamma tallies the law touches */
    int32_t pad;
} rs_dist_info_t;

typedef struct rs_range_info {
    uint64_t count;            /* samples starting in [entry, units(slice)) */
    uint64_t exit;             /* first sample boundary at or past the slice end, in units past it */
    uint64_t end_pos;          /* after rs_range_emit(keep > 0): unit position (from the slice start)
                                  right after sample keep-1; else the slice's entry */
    uint64_t tally[6];         /* emitted samples' tallies (rs_fill_result layout) */
    int32_t unit;
    int32_t resync_rounds;
} rs_range_info;

/* validated law description (host only, no device needed) */
rs_status rs_dist_info(int32_t dist, const double *fparams, const uint64_t *iparams, rs_dist_info_t *info);
/* slice shape for >= `words` engine words on the current device: one wave of segments */
rs_status rs_range_geometry(int32_t engine, int32_t dist, const double *fparams, const uint64_t *iparams,
                            uint64_t words, uint64_t *seg_len, uint32_t *n_seg);
/* count + exit of one slice (synchronous); keeps the plan for rs_range_emit on this device */
rs_status rs_range_count(const rs_stream *stream, int32_t dist, const double *fparams,
                         const uint64_t *iparams, uint64_t entry, uint64_t seg_len, uint32_t n_seg,
                         rs_range_info *info, void *cuda_stream);
/* rs_range_count with the entry guess folded in: `window_start` is positioned n_warm segments
 * (n_warm a multiple of 256) before the slice; the plan parses window + slice in the same
 * launches, assuming a sample starts at the window start, and the slice enters at the
 * window's exit (returned in info->end_pos). Saves the separate warm-up count's launches and
 * host round trip. The emitted samples and positions are those of rs_range_count(entry). */
rs_status rs_range_count_warm(const rs_stream *window_start, int32_t dist, const double *fparams,
                              const uint64_t *iparams, uint32_t n_warm, uint64_t seg_len, uint32_t n_seg,
                              rs_range_info *info, void *cuda_stream);
/* write the first `keep` samples of the counted slice into device memory (synchronous).
 * Any other fill on the device between count and emit invalidates the slice (RS_ERR_VALUE). */
rs_status rs_range_emit(uint64_t keep, void *out_device, rs_range_info *info, void *cuda_stream);

#ifdef __cplusplus
}
#endif
#endif
