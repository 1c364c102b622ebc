/*
 * vmt19937_b200.h -- C ABI of the B200-native VMT19937 generator.
 *
 * Drop-in boundary for the reference's generation path.
 * The reference exposes a C++ surface only (no C ABI, no FFI); each entry point
 * below names the reference interface it replaces. All functions return a
 * vmt_status (0 = success) and never throw; the three reference exception
 * classes map to VMT_EINVAL (std::invalid_argument), VMT_ESTATE
 * (std::logic_error) and VMT_EIO (std::runtime_error), plus VMT_ECUDA.
 *
 * Threading: one owner per handle, like VmtEngine; distinct
 * handles are independent. Buffers are caller-owned; every fill takes an
 * explicit length (the reference's sizes are implicit, engine.hpp:77,92).
 * Destination pointers may be device memory or host memory (pinned or
 * pageable); host destinations are filled through device staging.
 * Streams are cudaStream_t passed as void* (NULL = the handle's own stream).
 */
#ifndef VMT19937_B200_H
#define VMT19937_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vmt_generator* vmt_handle;

enum vmt_status {
    VMT_OK = 0,
    VMT_EINVAL = -1, /* std::invalid_argument (engine.hpp:29-32, jump.cpp:9-10) */
    VMT_ESTATE = -2, /* std::logic_error (engine.hpp:93-94, jump.cpp:30-31)     */
    VMT_EIO = -3,    /* std::runtime_error (jump_file.cpp:76-88)                */
    VMT_ECUDA = -4,  /* CUDA runtime failure (no device, launch error, OOM)     */
    VMT_ENOMEM = -5
};

/* QueryMode (engine.hpp:15) -- accepted for API parity; every mode emits the
 * same stream (test_engine.cpp:81-109). */
enum vmt_query_mode { VMT_QUERY_SINGLE = 0, VMT_QUERY_BLOCK16 = 1, VMT_QUERY_STATE_BLOCK = 2 };

/* Floating-point conversion rules (the reference has none: SURVEY.md G2/A16).
 * All are exact in IEEE arithmetic, so GPU and CPU agree bit for bit. */
enum vmt_real_rule {
    VMT_F32_24 = 0,    /* float  (x >> 8) * 2^-24            in [0,1)                      */
    VMT_F64_32 = 1,    /* double x * 2^-32                   in [0,1)  (genrand_real2)      */
    VMT_F64_REAL3 = 2, /* double (x + 0.5) * 2^-32           in (0,1)  (stats.cpp:118)      */
    VMT_F64_RES53 = 3  /* double ((a>>5)*2^26+(b>>6))*2^-53  in [0,1), 2 words per value    */
};

/* Pass as jump_exponent to get the library default (JumpSpec::full_period_exponent). */
#define VMT_FULL_PERIOD 0xFFFFFFFFu

/* JumpSpec::full_period_exponent (jump.cpp:13-15): 19937 - log2(lanes). */
unsigned vmt_full_period_exponent(unsigned lanes);

/* VmtEngine<M>(seed, F^(2^q), q) (engine.hpp:54-63) / VmtGenerator
 * (engine.hpp:162-167): seeds MT19937 (mt19937.cpp:22-27) and de-phases lane
 * t by t*2^q steps (make_dephased_states, jump.cpp:35-53) with a polynomial
 * jump on the GPU. lanes in {1,2,4,8,16,32} (32 lifts engine.hpp:43, G1).
 * jump_exponent: any q, or VMT_FULL_PERIOD. device: CUDA ordinal. */
int vmt_create(uint32_t seed, unsigned lanes, unsigned jump_exponent, int device, vmt_handle* out);

/* Adopts caller-supplied boundary lane states (lanes x 624 words, lane-major,
 * Mt19937::from_words semantics, mt19937.cpp:29-34) as the generator's start. */
int vmt_create_from_states(const uint32_t* lane_states, unsigned lanes, int device, vmt_handle* out);

/* Copy of a generator (VmtEngine's value semantics, engine.hpp:41-158): an
 * independent handle with the same lanes, de-phasing and stream position;
 * both continue with identical words. Waits for src's pending work. */
int vmt_clone(vmt_handle src, vmt_handle* out);

int vmt_destroy(vmt_handle h);

unsigned vmt_lanes(vmt_handle h);              /* VmtEngine::lanes (engine.hpp:47)          */
uint64_t vmt_state_words(vmt_handle h);        /* VmtEngine::state_words (engine.hpp:48)    */
unsigned vmt_jump_exponent(vmt_handle h);      /* VmtEngine::jump_exponent (engine.hpp:100) */
uint64_t vmt_position(vmt_handle h);           /* words consumed so far                     */

/* VmtEngine::next_u32 (engine.hpp:70-74). */
int vmt_next_u32(vmt_handle h, uint32_t* out);
/* VmtEngine::next_block16 (engine.hpp:77-87): exactly 16 words. */
int vmt_next_block16(vmt_handle h, uint32_t* out16);
/* VmtEngine::next_block_state (engine.hpp:92-98): exactly 624*lanes words;
 * VMT_ESTATE off a state-block boundary (engine.hpp:93-94). */
int vmt_next_block_state(vmt_handle h, uint32_t* out);

/* Next n stream words (any n; next_u32 continuation semantics). */
int vmt_fill_u32(vmt_handle h, uint32_t* dst, uint64_t n, void* stream);
/* Next n values converted by rule (VMT_F32_24). */
int vmt_fill_f32(vmt_handle h, float* dst, uint64_t n, int rule, void* stream);
/* Next n values converted by rule (VMT_F64_32 / VMT_F64_REAL3 / VMT_F64_RES53;
 * RES53 consumes 2n words and needs an even stream position). */
int vmt_fill_f64(vmt_handle h, double* dst, uint64_t n, int rule, void* stream);
/* XOR fold of the next n words without storing them (bench.cpp:13-18 fold;
 * fused no-store consumer). */
int vmt_checksum_xor(vmt_handle h, uint64_t n, uint32_t* out, void* stream);

/* Waits for all work this handle enqueued (device fills are asynchronous). */
int vmt_synchronize(vmt_handle h);

/* Advances the position by d words (new; arbitrary 64-bit distance). */
int vmt_skip(vmt_handle h, uint64_t d);
/* Sets the absolute stream position (forward or backward; new). */
int vmt_seek(vmt_handle h, uint64_t pos);

/* VmtEngine::interleaved_state (engine.hpp:100): 624*lanes words, state of
 * the most recently regenerated block (the de-phased seed states before the
 * first query). */
int vmt_export_state(vmt_handle h, uint32_t* out);

/* Batch of ngen independent generators with seeds seed0..seed0+ngen-1 (config
 * 3): dst[g*n_per_gen + i] = word i of generator g (generator-major). */
int vmt_batch_fill_u32(uint32_t seed0, unsigned ngen, unsigned lanes, unsigned jump_exponent,
                       uint64_t n_per_gen, uint32_t* dst, int device, void* stream);

/* A batch of ngen independent generators (seeds seed0..seed0+ngen-1, each a
 * VmtEngine<lanes> with the same de-phasing; config 3) advancing in lockstep:
 * vmt_batch_fill writes the next n_per_gen words of every generator,
 * dst[g*n_per_gen + i] (generator-major), continuing across calls like
 * next_u32; vmt_batch_skip advances every generator by d words. */
typedef struct vmt_batch* vmt_batch_handle;
int vmt_batch_create(uint32_t seed0, unsigned ngen, unsigned lanes, unsigned jump_exponent, int device,
                     vmt_batch_handle* out);
int vmt_batch_fill(vmt_batch_handle h, uint32_t* dst, uint64_t n_per_gen, void* stream);
int vmt_batch_skip(vmt_batch_handle h, uint64_t d);
uint64_t vmt_batch_position(vmt_batch_handle h);
/* ngen x 624*lanes interleaved states (VMT_ESTATE off a block boundary). */
int vmt_batch_export_state(vmt_batch_handle h, uint32_t* out);
int vmt_batch_destroy(vmt_batch_handle h);

/* Config 4 in one process: the stream's words [0, n) partitioned into ngpus
 * contiguous ranges (n/ngpus words each, the remainder one word each to the
 * first devices), each device positioned by one jump, no data exchange.
 * mode 0 stores into dsts[k] (device k memory), mode 1 only XOR-folds; the
 * global XOR checksum (bench.cpp:13-18 fold) goes to *checksum when non-NULL
 * (store mode computes it with a second, fused pass). The multi-process form
 * (one rank per GPU, torch.distributed) is bench.py / dist.py. */
int vmt_multi_gpu_fill(uint32_t seed, unsigned lanes, unsigned jump_exponent, uint64_t n, int ngpus,
                       const int* devices, uint32_t* const* dsts, int mode, uint32_t* checksum);

/* jump_state (jump.cpp:27-33) generalised to arbitrary 64-bit distances, for
 * n boundary states (n x 624 words, lane-major; host or device memory):
 * dst_i = src_i advanced by distances[i] steps (config 5). */
int vmt_jump_states(const uint32_t* src, uint64_t n, const uint64_t* distances, uint32_t* dst,
                    int device, void* stream);

/* Seeds n MT19937 states (init_genrand) into dst (n x 624, lane-major). */
int vmt_seed_states(const uint32_t* seeds, uint64_t n, uint32_t* dst, int device, void* stream);

/* Jump polynomials (host): x^d mod P and x^(2^q) mod P as 312 little-endian
 * u64 words; the characteristic polynomial P as 313 words. */
int vmt_jump_poly(uint64_t d_lo, uint64_t d_hi, uint64_t* out312);
int vmt_jump_poly_pow2(unsigned q, uint64_t* out312);
int vmt_charpoly(uint64_t* out313);

/* ---- GF(2) jump matrices (f2_matrix.hpp, jump_file.hpp) -------------------
 * A matrix is 19937 rows x 312 little-endian u64 (F2Matrix row-major payload,
 * f2_matrix.hpp:13-21 and 49-51; row i = image of basis vector i in the
 * effective layout, mt19937.cpp:57-101). Row/vector buffers may be host or
 * device memory. */
#define VMT_MATRIX_DIM 19937u
#define VMT_MATRIX_ROW_WORDS 312u
#define VMT_MATRIX_WORDS (19937ull * 312ull)

/* F^d for d = d_hi*2^64 + d_lo, computed on the GPU as 19937 polynomial jumps
 * of the basis states. vmt_jump_matrix_pow2(q) equals the reference's
 * mat_pow2(build_transition_matrix(), q) (f2_matrix.cpp:138-177,179-228)
 * byte for byte, for every q including the full-period exponents. */
int vmt_jump_matrix(uint64_t d_lo, uint64_t d_hi, uint64_t* rows, int device, void* stream);
int vmt_jump_matrix_pow2(unsigned q, uint64_t* rows, int device, void* stream);

/* write_jump_matrix_file / read_jump_matrix_file (jump_file.hpp:37,
 * jump_file.cpp:117-137): the 20-byte "VMTJ" header (version 1, dimension,
 * exponent, reserved 0) plus the payload, written through a temporary file.
 * The reader applies the reference's checks (magic, version, reserved,
 * zero dimension, payload size, padding bits -> VMT_EIO); a well-formed file
 * of another dimension is VMT_EINVAL. rows == NULL validates without
 * reading the payload. */
int vmt_write_jump_matrix_file(const char* path, const uint64_t* rows, unsigned exponent);
int vmt_read_jump_matrix_file(const char* path, uint64_t* rows, unsigned* exponent);

/* compute_jump_matrix (jump_file.cpp:171-209; the CLI `jump` command): writes
 * the file for F^(2^exponent) -- milliseconds on the GPU instead of
 * `exponent` CPU squarings (~50 h at the full period). */
int vmt_compute_jump_matrix_file(const char* path, unsigned exponent, int device);

/* vec_mat_mul (f2_matrix.cpp:119-136) for n effective vectors (n x 312 u64):
 * out_i = vecs_i * M, the XOR of the rows at the set bits of vecs_i. */
int vmt_vec_mat_mul(const uint64_t* vecs, uint64_t n, const uint64_t* rows, uint64_t* out, int device,
                    void* stream);

/* jump_state (jump.cpp:27-33) with a caller matrix, for n boundary states
 * (n x 624 words): dst_i = effective_to_state(state_to_effective(src_i) * M);
 * the dead low bits of word 0 come out zero (mt19937.cpp:79). */
int vmt_jump_states_matrix(const uint32_t* src, uint64_t n, const uint64_t* rows, uint32_t* dst, int device,
                           void* stream);

/* VmtEngine<M>(seed, jump_matrix, jump_exponent) (engine.hpp:54-63) with the
 * matrix de-phasing of make_dephased_states (jump.cpp:35-53): lane t = lane
 * t-1 * B on the GPU. rows may be NULL for lanes == 1 (engine.hpp:66-68).
 * vmt_create_from_file reads a .vmtj file and adopts its exponent (the CLI's
 * resolve_jump with an explicit file, vmt19937_main.cpp:30-37). */
int vmt_create_from_matrix(uint32_t seed, unsigned lanes, const uint64_t* rows, unsigned exponent, int device,
                           vmt_handle* out);
int vmt_create_from_file(uint32_t seed, unsigned lanes, const char* path, int device, vmt_handle* out);

/* Kernel tuning for the generation path: chunks per fill (0 = auto), and
 * the CTA shape variant (0 = auto). Returns VMT_EINVAL for unknown variants. */
int vmt_set_tuning(vmt_handle h, unsigned max_chunks, int variant);
/* Steady-state positioning prefetch: while a fill of >= 2^24 words
 * generates, the chunk start states of the predicted next fill (same size,
 * same gap) are computed on a side stream; a matching next fill skips its
 * positioning. Results are identical in every mode.
 *   VMT_PREFETCH_OFF     none
 *   VMT_PREFETCH_JUMPS   polynomial jumps on the side stream (with the
 *                        generation kernel ALU-saturated they slow it by as
 *                        much as they save)
 *   VMT_PREFETCH_TENSOR  default: one tcgen05 GEMM with the cached positioning
 *                        matrix, co-resident with the generation kernel on the
 *                        idle tensor cores (once the fill shape repeats and the
 *                        generation kernel leaves room on every SM; otherwise
 *                        the fill is positioned as without prefetch)
 * Returns VMT_EINVAL for other values. */
#define VMT_PREFETCH_OFF 0
#define VMT_PREFETCH_JUMPS 1
#define VMT_PREFETCH_TENSOR 2
int vmt_set_prefetch(vmt_handle h, int enable);

/* Chunk positioning of consecutive fills: mode 0 =
 * auto (one FP4 tensor-core GEMM -- our tcgen05 kernel -- maps the previous
 * fill's chunk states to the next fill's when the
 * fill shape and block delta repeat and there are at least 256 lane states;
 * polynomial jumps otherwise), 1 = polynomial jumps only, 2 = GEMM whenever
 * the shape repeats. Results are identical. */
int vmt_set_positioning(vmt_handle h, int mode);
int vmt_positioning_stats(vmt_handle h, uint64_t* gemm_positionings, uint64_t* cached_matrices);
/* Prefetch counters: tcgen05 prefetch launches (VMT_PREFETCH_TENSOR) and
 * fills that used prefetched chunk states (any mode). */
int vmt_prefetch_stats(vmt_handle h, uint64_t* tensor_prefetches, uint64_t* used);
/* De-phasing of many generators at once (vmt_batch_*, >= 4096 lane states)
 * runs as log2(lanes) FP4 GEMMs with a process-wide cache of the jump
 * matrices F^(s 2^q) per device (200 MB each, at most 8); this frees it,
 * and the process-wide host caches of the seed-independent polynomials
 * (de-phasing polynomials per (q, lanes), chunk polynomials per chunk size). */
int vmt_release_caches(int device);

/* Profiling: when enabled, each fill records CUDA events on its stream around
 * the chunk-positioning jumps and the generation kernel; vmt_last_timings
 * returns both durations (ms) of the most recent fill. */
int vmt_set_profiling(vmt_handle h, int enable);
int vmt_last_timings(vmt_handle h, float* jump_ms, float* gen_ms);
/* Sums over every fill recorded since profiling was enabled or since the
 * previous call (which resets them): fills, positioning-jump ms, generation ms. */
int vmt_profile_totals(vmt_handle h, uint64_t* fills, double* jump_ms, double* gen_ms);

/* Counters: kernels launched by this handle so far (generation, jump, seed,
 * reduce), and the number of lane-state jumps performed. */
int vmt_stats(vmt_handle h, uint64_t* gen_launches, uint64_t* jump_launches, uint64_t* other_launches,
              uint64_t* lane_jumps);

/* ---- fused statistics consumer (stats.hpp, stats.cpp) ---------------------
 * StatReport (stats.hpp:13-20). */
typedef struct {
    const char* name; /* static string */
    uint64_t samples;
    double statistic;
    double p_value;
    int pass;
} vmt_stat_report;

/* Consumes the next n words of the stream (like a fill, nothing stored: the
 * generation kernel counts in shared memory): out257[0] = one bits,
 * out257[1 + b] = occurrences of byte value b over the 4 bytes of each word. */
int vmt_stat_counts(vmt_handle h, uint64_t n, uint64_t* out257, void* stream);
/* monobit (stats.cpp:65-81) and chi2_bytes (stats.cpp:83-107) over the next
 * `count` words, the counts from vmt_stat_counts and the statistic, p-value
 * and pass flag by the reference's formulas. Undersized samples are
 * VMT_EINVAL like the reference's std::invalid_argument. */
int vmt_monobit(vmt_handle h, uint64_t count, vmt_stat_report* out);
int vmt_chi2_bytes(vmt_handle h, uint64_t count, vmt_stat_report* out);
/* The same reports from counts taken elsewhere (bins256 = byte-value counts). */
int vmt_monobit_from_counts(uint64_t count, uint64_t ones, vmt_stat_report* out);
int vmt_chi2_bytes_from_counts(uint64_t count, const uint64_t* bins256, vmt_stat_report* out);
/* lane_cross_correlation (stats.cpp:109-150) over the next count*lanes words:
 * lane t's sequence is column t of the combined stream. Needs lanes >= 2
 * (VMT_EINVAL). Floating point: equal to the reference within 1e-12. */
int vmt_lane_cross_correlation(vmt_handle h, uint64_t count, vmt_stat_report* out);
/* The same statistic over caller-supplied words, combined-stream order
 * (lane t's i-th word at words[i*lanes + t]); host arithmetic. Serves the
 * reference's lane_cross_correlation(std::vector<WordSource>, count). */
int vmt_lane_cross_correlation_from_words(const uint32_t* words, unsigned lanes, uint64_t count,
                                          vmt_stat_report* out);
/* detail::regularized_gamma_q (stats.hpp:47-50, stats.cpp:52-60). */
int vmt_regularized_gamma_q(double a, double x, double* out);

/* Measurement only: GB/s of a pure 16-byte-store kernel over `bytes` of HBM,
 * pattern 0 = grid-stride, 1 = one contiguous chunk per CTA (the generation
 * kernel's output pattern), 2 = as 1 with random-looking words (HBM interface
 * power depends on the bits toggled); grid = SMs x ctas_per_sm. The second
 * roofline denominator next to MEASURED_PEAKS.json's copy bandwidth. */
int vmt_store_bandwidth(int device, uint64_t bytes, int pattern, int ctas_per_sm, double* gbs);

const char* vmt_status_string(int status);
/* Message of the last failure on this thread. */
const char* vmt_last_error(void);
int vmt_version(void);

#ifdef __cplusplus
}
#endif

#endif /* VMT19937_B200_H */
