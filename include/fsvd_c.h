/*
 * fsvd_c.h -- C ABI of the B200-native FlashSVD runtime (libfsvd_b200.so).
 *
 * This is the drop-in boundary for the north-star path: the factorized
 * checkpoint loader and the prefill()/decode_step()/generate() entry points
 * that SPEC.md specifies for the reference (runtime module)
 * and that the reference C++ API exposes as headers under
 * proj/include/fsvd/ (loader: checkpoint.hpp:58-61 read_checkpoint(_file),
 * canonical.hpp:79-80 normalize<T>). Plain pointers and sizes only; no torch,
 * no C++ types, no exceptions across the boundary: every C++ error type of
 * the reference maps to one status code (tensor.hpp:17-31, checkpoint.hpp:21,
 * canonical.hpp:21, compress.hpp:18) and the message is kept in a
 * thread-local buffer read by fsvd_last_error().
 *
 * Threading: a model is immutable after load and may back
 * any number of sessions; a session is used by one host thread at a time.
 */
#ifndef FSVD_C_H
#define FSVD_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fsvd_status {
    FSVD_OK = 0,
    FSVD_ERR_SHAPE = 1,       /* fsvd::ShapeError        tensor.hpp:17      */
    FSVD_ERR_RANK = 2,        /* fsvd::RankError         tensor.hpp:20      */
    FSVD_ERR_NUMERIC = 3,     /* fsvd::NumericError      tensor.hpp:23      */
    FSVD_ERR_CAPACITY = 4,    /* fsvd::CapacityError     tensor.hpp:26      */
    FSVD_ERR_CONFIG = 5,      /* fsvd::ConfigError       tensor.hpp:29      */
    FSVD_ERR_FORMAT = 6,      /* fsvd::FormatError       checkpoint.hpp:21  */
    FSVD_ERR_NORMALIZE = 7,   /* fsvd::NormalizeError    canonical.hpp:21   */
    FSVD_ERR_CALIBRATION = 8, /* fsvd::CalibrationError  compress.hpp:18    */
    FSVD_ERR_CUDA = 9,        /* CUDA runtime / driver failure              */
    FSVD_ERR_OOM = 10,        /* device or host allocation failure          */
    FSVD_ERR_INVALID = 11,    /* null handle / bad enum / bad argument      */
    FSVD_ERR_INTERNAL = 12
} fsvd_status;

typedef enum fsvd_dtype { FSVD_DTYPE_F32 = 0, FSVD_DTYPE_BF16 = 1 } fsvd_dtype;

/* SPEC.md:294 Session.ffn_backend, route_ffn_auto SPEC.md:419-427 */
typedef enum fsvd_ffn_backend {
    FSVD_FFN_AUTO = 0,
    FSVD_FFN_NO_MERGE = 1,
    FSVD_FFN_PACKED = 2
} fsvd_ffn_backend;

/* SPEC.md:294 Session.plan_mode. PER_LAYER = one CUDA graph per decoder layer
 * (SPEC.md:401-418 full_layer plans); FULL_STEP = one graph per decode step
 * (extension; same kernels, same order); SPLIT = two graphs per layer
 * (attention body, MLP body) with an explicit boundary copy between them
 * (SPEC.md:404-418 split plans). */
typedef enum fsvd_plan_mode {
    FSVD_PLAN_EAGER = 0,
    FSVD_PLAN_PER_LAYER = 1,
    FSVD_PLAN_FULL_STEP = 2,
    FSVD_PLAN_SPLIT = 3
} fsvd_plan_mode;

/* SPEC.md:294 Session.attn_route. LOWRANK_HISTORY (ablation)
 * keeps the rank-space K/V history and reconstructs dense K, V (+ RoPE) for
 * every cached position at every decode step; eager plan only. */
typedef enum fsvd_attn_route {
    FSVD_ATTN_DENSE_KV = 0,
    FSVD_ATTN_LOWRANK_HISTORY = 1
} fsvd_attn_route;

typedef struct fsvd_config {
    uint64_t n_layers, d_model, n_heads, d_head, d_ff, vocab;
    double rope_base, norm_eps;
} fsvd_config;

/* Synthetic random-init factorized checkpoint (include/fsvd/synth.hpp). */
typedef struct fsvd_synth_spec {
    fsvd_config config;
    uint64_t capacity;
    char family;          /* 'A' | 'B' | 'C' | 'D' */
    double rho;           /* retained parameter ratio, (0, 1] */
    uint64_t group_size;  /* family C */
    uint64_t seed;
    int32_t conditioned;  /* gammas ~ 1 + U(+-0.1) */
    double rank_jitter;   /* families B / D */
} fsvd_synth_spec;

typedef struct fsvd_session_opts {
    uint32_t batch;           /* independent sequences advanced in lock step */
    uint64_t capacity;        /* KV positions per sequence; 0 = model capacity */
    fsvd_ffn_backend ffn;
    fsvd_plan_mode plan;
    fsvd_attn_route attn_route;
} fsvd_session_opts;

/* SPEC.md:299-302 StepStats, plus device-side counters. */
typedef struct fsvd_step_stats {
    uint64_t steps;            /* decode steps since create/reset */
    uint64_t dispatches;       /* host-visible launch boundaries (kernels + graph launches) */
    uint64_t kernel_launches;  /* kernels issued eagerly */
    uint64_t graph_launches;   /* cudaGraphLaunch calls */
    uint64_t allocs;           /* device allocations after session create */
    uint64_t copy_bytes;       /* host<->device bytes moved by the API calls */
    uint64_t last_dispatches;  /* dispatches of the last decode step */
    uint64_t recon_flops;      /* K/V reconstruction FLOPs of the lowrank_history route (0 for dense_kv) */
} fsvd_step_stats;

typedef struct fsvd_canonical fsvd_canonical; /* host CanonicalModel<float> */
typedef struct fsvd_model fsvd_model;         /* device-resident model      */
typedef struct fsvd_session fsvd_session;     /* KV cache + workspace + plans */

const char* fsvd_last_error(void);
const char* fsvd_version(void);

/* ---- host loader: read_checkpoint_file -> normalize<float> (CPU only) ---- */
fsvd_status fsvd_canonical_load_file(const char* path, fsvd_canonical** out);
fsvd_status fsvd_canonical_load_bytes(const uint8_t* bytes, size_t len, fsvd_canonical** out);
fsvd_status fsvd_canonical_synthetic(const fsvd_synth_spec* spec, fsvd_canonical** out);
fsvd_status fsvd_canonical_config(const fsvd_canonical* c, fsvd_config* cfg, uint64_t* capacity);
/* proj: 0..6 = q,k,v,o,up,gate,down (model.hpp kProjNames) */
fsvd_status fsvd_canonical_rank(const fsvd_canonical* c, uint64_t layer, uint32_t proj, uint64_t* rank);
/* Copy a canonical tensor as f32. Names: embedding, head, final_gamma,
 * layers.{i}.{q|k|v|o|up|gate|down}.{A|B}, layers.{i}.a_ug,
 * layers.{i}.attn_gamma, layers.{i}.mlp_gamma. count must match exactly. */
fsvd_status fsvd_canonical_copy(const fsvd_canonical* c, const char* name, float* out, uint64_t count);
/* Number of distinct shared-basis storage instances (family C). */
fsvd_status fsvd_canonical_shared_count(const fsvd_canonical* c, uint64_t* n);
/* 1 if layers (l0, l1) alias the same A storage for projection proj. */
fsvd_status fsvd_canonical_aliased(const fsvd_canonical* c, uint64_t l0, uint64_t l1, uint32_t proj, int32_t* out);
fsvd_status fsvd_canonical_destroy(fsvd_canonical* c);
/* Write a normalized model as a family-A FSVD15 file (the CLI's `normalize`). */
fsvd_status fsvd_canonical_write_file(const fsvd_canonical* c, const char* path);
/* Materialize a synthetic checkpoint as an FSVD15 file. */
fsvd_status fsvd_synthetic_write_file(const fsvd_synth_spec* spec, const char* path);

/* ---- device model ---- */
fsvd_status fsvd_model_load(const char* path, fsvd_dtype dtype, int32_t device, fsvd_model** out);
/* Statistics of this thread's last fsvd_model_load (streaming loader): wall
 * seconds, payload bytes read, host pinned staging held at once. */
fsvd_status fsvd_last_load_stats(double* seconds, uint64_t* payload_bytes, uint64_t* pinned_bytes);
fsvd_status fsvd_model_from_canonical(const fsvd_canonical* c, fsvd_dtype dtype, int32_t device, fsvd_model** out);
/* Device-side generation of a synthetic checkpoint: bit-identical weights to
 * fsvd_canonical_synthetic(spec) without a host copy (LLaMA-13B shape). */
fsvd_status fsvd_model_synthetic(const fsvd_synth_spec* spec, fsvd_dtype dtype, int32_t device, fsvd_model** out);
fsvd_status fsvd_model_info(const fsvd_model* m, fsvd_config* cfg, uint64_t* capacity, uint64_t* weight_bytes,
                            uint64_t* decode_weight_bytes);
/* Read back one canonical factor from the device as f32 (A: d_in x r, B: r x d_out). */
fsvd_status fsvd_model_copy_factor(const fsvd_model* m, uint64_t layer, uint32_t proj, int32_t which_b,
                                   float* out, uint64_t count);
fsvd_status fsvd_model_destroy(fsvd_model* m);

/* ---- sessions ---- */
fsvd_status fsvd_route_ffn_auto(fsvd_plan_mode plan, fsvd_ffn_backend requested, fsvd_ffn_backend* out);
fsvd_status fsvd_session_create(fsvd_model* m, const fsvd_session_opts* opts, fsvd_session** out);
/* tokens: [batch][T] host; logits_out: [batch][vocab] host, last position only. */
fsvd_status fsvd_prefill(fsvd_session* s, const int32_t* tokens, uint64_t T, float* logits_out);
/* tokens: [batch]; logits_out: [batch][vocab]. */
fsvd_status fsvd_decode_step(fsvd_session* s, const int32_t* tokens, float* logits_out);
/* prefill + max_new greedy steps (argmax on device, ties -> lowest index);
 * out: [batch][max_new]. */
fsvd_status fsvd_generate(fsvd_session* s, const int32_t* prompt, uint64_t T, uint64_t max_new, int32_t* out);
/* Device-pointer variants: asynchronous on the session stream. */
fsvd_status fsvd_prefill_device(fsvd_session* s, const int32_t* d_tokens, uint64_t T, float* d_logits);
fsvd_status fsvd_decode_step_device(fsvd_session* s, const int32_t* d_tokens, float* d_logits);
fsvd_status fsvd_generate_device(fsvd_session* s, const int32_t* d_prompt, uint64_t T, uint64_t max_new,
                                 int32_t* d_out);
/* n greedy decode steps continuing from the last argmax (no host round trip);
 * d_out: [batch][n] generated tokens or NULL; logits of the last step stay on the
 * session. Extension of SPEC.md:341-349 generate for a serving loop. */
fsvd_status fsvd_decode_steps_device(fsvd_session* s, uint64_t n, int32_t* d_out);
fsvd_status fsvd_session_sync(fsvd_session* s);
fsvd_status fsvd_session_stream(fsvd_session* s, void** cuda_stream);
fsvd_status fsvd_session_position(const fsvd_session* s, uint64_t* position);
fsvd_status fsvd_session_reset(fsvd_session* s);
fsvd_status fsvd_session_stats(const fsvd_session* s, fsvd_step_stats* st);
fsvd_status fsvd_session_resolved(const fsvd_session* s, fsvd_ffn_backend* ffn, fsvd_plan_mode* plan);
/* Decode engine: megakernel = 1 when the persistent decode megakernel runs the
 * step (else one kernel per op); ring stage bytes / stage count / attention
 * splits of the megakernel. */
fsvd_status fsvd_session_engine(const fsvd_session* s, int32_t* megakernel, int32_t* stage_bytes, int32_t* nstage,
                                int32_t* attn_splits);
/* Profiling (FSVD_TRACE=1 at session creation): per-CTA per-phase
 * %globaltimer stamps of the last full-step megakernel launch,
 * out = [grid][phases][4] (wait start, barrier passed, input staged, done). */
fsvd_status fsvd_session_trace(fsvd_session* s, uint64_t* out, uint64_t count, int32_t* phases, int32_t* grid);
/* Read cached K (which=0) or V (which=1) rows [pos0, pos0+npos) of sequence b
 * at layer l as f32, [npos][d_model] (head-major within a row, like the dense
 * reference K = rmsnorm(x)·W_k). */
fsvd_status fsvd_session_read_kv(fsvd_session* s, uint64_t layer, uint64_t b, int32_t which, uint64_t pos0,
                                 uint64_t npos, float* out);
fsvd_status fsvd_session_destroy(fsvd_session* s);

#ifdef __cplusplus
}
#endif
#endif /* FSVD_C_H */
