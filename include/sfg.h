/* sfg.h — C ABI of the B200-native splitf lookahead engine (libsfg.so).
 *
 * The engine is a drop-in for the compute hot path of the reference splitf
 * artifact (/root/reference/proj): the untrusted-side middle-layer forward of
 * one lookahead step and the trusted-side unembed -> greedy argmax -> n-gram
 * verify that follows it.  Two seams are exported:
 *
 *   Seam 1 (server, frame level):  sfg_server_*  replaces
 *       splitf::ServerEngine                      (server.hpp:28-77)
 *       and plugs in as a splitf::FrameHandler    (transport.hpp:44)
 *   Seam 2 (compute level):        sfg_bank_*, sfg_forward_layers,
 *       sfg_embed_at, sfg_finalize*   replace
 *       CacheBank / forward_layers / embed_at / finalize / argmax_row
 *                                                 (tinyformer.hpp:131-179)
 *   Local side (trusted):          sfg_client_*, sfg_decode, sfg_pool_*
 *       replace SplitClient::prefill/decode_step  (client.hpp:41-59) and
 *       decode_sequential / decode_lookahead_with_pool / NGramPool
 *                                                 (decoding.hpp:35-104)
 *
 * Conventions (mirroring the reference):
 *   - every call returns int32 status: 0 = ok, else (splitf::ErrorKind ordinal
 *     + 1) (error.hpp:10-21); sfg_last_error() gives the thread-local
 *     "category: message" string, exactly the text the reference would throw;
 *   - all pointers are caller-owned host memory borrowed for the call;
 *   - calls are synchronous (they return after the device result is on the
 *     host), like the reference's CPU calls;
 *   - weights are stored on device as bf16 (or f32) in the reference layout
 *     [in x out]; no host copy is kept.
 *
 * No torch types cross this boundary: plain pointers and sizes only.
 */
#ifndef SFG_H
#define SFG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes = splitf::ErrorKind ordinal + 1 (error.hpp:10-21) */
enum {
    SFG_OK = 0,
    SFG_ERR_CONFIG = 1,
    SFG_ERR_INPUT = 2,
    SFG_ERR_PROTOCOL = 3,
    SFG_ERR_TRANSPORT = 4,
    SFG_ERR_CAPACITY = 5,
    SFG_ERR_SESSION = 6,
    SFG_ERR_NUMERIC = 7,
    SFG_ERR_TRAINING = 8,
    SFG_ERR_DECOMPOSITION = 9,
    SFG_ERR_INTERNAL = 10
};

/* splitf::ModelConfig (tinyformer.hpp:15-33) */
typedef struct {
    int32_t vocab_size;
    int32_t n_layers;
    int32_t hidden_dim;
    int32_t n_heads;
    int32_t n_kv_heads;
    int32_t head_dim;
    int32_t ffn_dim;
    int32_t max_seq_len;
    float rope_base;
    float rms_eps;
    uint64_t seed;
} sfg_model_config;

/* Arithmetic of the layer executor.
 *  EXACT: CUDA-core kernels that reproduce the reference's fp32 operation
 *         order bit for bit (serial K accumulation, no FMA, glibc expf port):
 *         hidden states / logits / tokens bitwise equal to the CPU reference.
 *  FAST:  tcgen05 weight-streaming GEMMs (bf16 weights x 3-way bf16-split fp32
 *         activations, fp32 TMEM accumulation); batch-invariant, within the
 *         stated tolerance of the reference.                                */
enum { SFG_MATH_EXACT = 0, SFG_MATH_FAST = 1 };
enum { SFG_WEIGHTS_BF16 = 0, SFG_WEIGHTS_F32 = 1 };
enum { SFG_WIRE_F16 = 0, SFG_WIRE_F32 = 1 };

typedef struct {
    int32_t device;         /* CUDA device ordinal */
    int32_t math;           /* SFG_MATH_* */
    int32_t weight_dtype;   /* SFG_WEIGHTS_* (device storage; values rounded RNE) */
    int32_t layer_begin;    /* hosted decoder layers [layer_begin, layer_end)     */
    int32_t layer_end;
    int32_t with_embedding; /* local side: embedding table                        */
    int32_t with_head;      /* local side: final_norm + lm_head                   */
    int32_t extended_shapes;/* 1: also accept n_heads * head_dim != hidden_dim,
                               i.e. q_dim != hidden (Mistral NeMo 12B: 32 x 128 =
                               4096 vs 5120).  The reference's validate() rejects
                               such configs (tinyformer.cpp:109-111) although its
                               arithmetic uses q_dim() throughout (:405-406, :444,
                               :491); 0 keeps the reference's config errors.     */
} sfg_engine_options;

typedef struct sfg_engine sfg_engine;
typedef struct sfg_bank sfg_bank;
typedef struct sfg_server sfg_server;
typedef struct sfg_client sfg_client;
typedef struct sfg_pool sfg_pool;

const char* sfg_last_error(void);
const char* sfg_version(void);

/* ── engine (weights resident on one B200) ─────────────────────────────── */
/* Weights from the reference init stream: init_weights (tinyformer.cpp:123-152),
 * generated on the host tensor by tensor and uploaded; non-hosted tensors are
 * skipped in the stream.                                                      */
int32_t sfg_engine_create_seeded(const sfg_model_config* cfg, const sfg_engine_options* opt,
                                 sfg_engine** out);
/* Weights from a flat fp32 parameter array in snapshot declaration order
 * (PROTOCOL.md "Weight snapshots"; tinyformer.cpp:83-98).                    */
int32_t sfg_engine_create_from_params(const sfg_model_config* cfg, const sfg_engine_options* opt,
                                      const float* params, sfg_engine** out);
/* Tensor parallelism (configs[3]: NeMo-12B at TP=2): `tp_size`
 * engines, one process and GPU each, every engine holding 1/tp_size of each
 * layer's heads (QKV, O) and FFN columns (gate|up, down).  Row-parallel
 * outputs are summed with an NCCL all-reduce over NVLink (2 per layer).
 * Rank 0 creates the group id with sfg_tp_unique_id and shares its
 * SFG_TP_ID_BYTES with the other ranks (e.g. torch.distributed broadcast).
 * FAST math only; every rank must run the same calls in the same order.     */
enum { SFG_TP_ID_BYTES = 128 };
int32_t sfg_tp_unique_id(uint8_t* out /* SFG_TP_ID_BYTES */);
int32_t sfg_engine_create_tp(const sfg_model_config* cfg, const sfg_engine_options* opt, int32_t tp_size,
                             int32_t tp_rank, const uint8_t* tp_unique_id, sfg_engine** out);
void sfg_engine_destroy(sfg_engine* eng);
/* bytes of device memory held by the engine's weights */
int64_t sfg_engine_weight_bytes(const sfg_engine* eng);

/* ── seam 2: CacheBank + forward_layers (tinyformer.hpp:131-179) ─────────── */
int32_t sfg_bank_create(sfg_engine* eng, int32_t layer_begin, int32_t layer_end, sfg_bank** out);
void sfg_bank_destroy(sfg_bank* b);
int32_t sfg_bank_resolve(sfg_bank* b, const int32_t* keep, int32_t n);   /* tinyformer.cpp:282 */
int32_t sfg_bank_crop(sfg_bank* b, int32_t pos);                         /* tinyformer.cpp:310 */
void sfg_bank_mark_committed(sfg_bank* b, int32_t committed);            /* tinyformer.hpp:145 */
void sfg_bank_reset(sfg_bank* b);                                        /* tinyformer.cpp:324 */
void sfg_bank_state(const sfg_bank* b, int32_t* len, int32_t* committed);
int32_t sfg_bank_read_kv(sfg_bank* b, int32_t layer, int32_t kv_head, int32_t pos, float* k,
                         float* v);

/* forward_layers (tinyformer.cpp:375-508).  hidden/out: [seq x hidden_dim]
 * fp32; mask: [seq x (len+seq)] fp32 {0,-inf} or NULL for the causal prefix
 * law (build_attention_mask, tinyformer.cpp:229-241).                        */
int32_t sfg_forward_layers(sfg_engine* eng, sfg_bank* b, int32_t layer_begin, int32_t layer_end,
                           int32_t seq, const float* hidden, const int32_t* positions,
                           const float* mask, float* out);
int32_t sfg_embed_at(sfg_engine* eng, int32_t seq, const int32_t* ids, const int32_t* positions,
                     float* out);                                        /* tinyformer.cpp:348 */
int32_t sfg_finalize(sfg_engine* eng, int32_t seq, const float* hidden, float* logits);
int32_t sfg_finalize_argmax(sfg_engine* eng, int32_t seq, const float* hidden, int32_t* argmax);

/* ── seam 1: ServerEngine (server.hpp:28-77) ──────────────────────────── */
typedef struct {
    int32_t layer_begin;       /* ServerConfig (server.hpp:15-22) */
    int32_t layer_end;
    double session_expiry_s;
    int32_t max_sessions;
    int32_t response_dtype;    /* -1 mirror request, SFG_WIRE_F16, SFG_WIRE_F32 */
} sfg_server_config;

int32_t sfg_server_create(sfg_engine* eng, const sfg_server_config* cfg, sfg_server** out);
void sfg_server_destroy(sfg_server* s);
/* ServerEngine::handle over encoded frames (PROTOCOL.md).  Never fails for
 * bad requests: those yield encoded error frames.  *resp points into a
 * thread-local buffer valid until the next call on the same thread.        */
int32_t sfg_server_handle(sfg_server* s, const uint8_t* req, size_t req_len, const uint8_t** resp,
                          size_t* resp_len);
/* handle() over n frames, in order, with the same responses handle() gives
 * frame by frame.  Step frames of distinct sessions whose rows fit one pass
 * (<= 32 rows total, <= 16 per session, masks within the layer-stack
 * contract) share ONE weight pass: cross-session batching of concurrent
 * decoders; two sessions' full 16-row lookahead batches
 * share a pass.
 * resps[i] point into thread-local buffers valid until the next call.
 * Replaces a loop of ServerEngine::handle (server.hpp:49) over the frames a
 * transport has queued.                                                     */
int32_t sfg_server_handle_batch(sfg_server* s, int32_t n, const uint8_t* const* reqs, const size_t* req_lens,
                                const uint8_t** resps, size_t* resp_lens);
/* How many weight passes sfg_server_handle_batch shared between sessions.  */
uint64_t sfg_server_shared_passes(sfg_server* s);
size_t sfg_server_expire_sessions(sfg_server* s);
size_t sfg_server_session_count(sfg_server* s);
int32_t sfg_server_session_view(sfg_server* s, const char* session_id, int32_t* cache_len,
                                int32_t* committed_len, int32_t* provisional);
void sfg_server_set_clock(sfg_server* s, double (*now_s)(void* ctx), void* ctx);

/* ── local side: SplitClient + decode loops (client.hpp, decoding.hpp) ── */
typedef int32_t (*sfg_frame_handler)(void* ctx, const uint8_t* req, size_t req_len,
                                     const uint8_t** resp, size_t* resp_len);

/* ── multi-device serving front end ─────────────────
 * The reference binds ONE ServerEngine behind a FrameServer that runs a
 * thread per connection (transport.cpp:531, :565-581).  A router is the
 * FrameHandler over one server per device (or any frame handlers): a
 * session is placed on the least-loaded backend when its prompt frame
 * arrives and stays there (sticky); frames of an unplaced session get the
 * server's "session: unknown or expired session" error frame.  No
 * cross-device state, no collective on the data path.                      */
typedef struct sfg_router sfg_router;
int32_t sfg_router_create(sfg_server* const* servers, int32_t n, double session_expiry_s, sfg_router** out);
int32_t sfg_router_create_handlers(const sfg_frame_handler* fns, void* const* ctxs, int32_t n,
                                   double session_expiry_s, sfg_router** out);
void sfg_router_destroy(sfg_router* r);
/* FrameHandler (thread safe); *resp as for sfg_server_handle               */
int32_t sfg_router_handle(sfg_router* r, const uint8_t* req, size_t req_len, const uint8_t** resp,
                          size_t* resp_len);
/* backend index of a session, -1 if not placed                             */
int32_t sfg_router_session_device(sfg_router* r, const char* session_id);
/* sessions placed per backend into sessions[0..n); returns n              */
int32_t sfg_router_load(sfg_router* r, int32_t* sessions);
void sfg_router_set_clock(sfg_router* r, double (*now_s)(void* ctx), void* ctx);
/* Cross-session batching queue: a FrameHandler for many concurrent
 * connection threads.  Frames queue per backend; one worker per backend
 * drains whatever is queued through sfg_server_handle_batch (steps of
 * distinct sessions share one weight pass; each response is the one
 * handle() gives).  A call blocks until its own response is ready.        */
typedef struct sfg_batcher sfg_batcher;
int32_t sfg_batcher_create(sfg_router* r, int32_t max_frames /* 0: unlimited */, sfg_batcher** out);
void sfg_batcher_destroy(sfg_batcher* b);
int32_t sfg_batcher_handle(sfg_batcher* b, const uint8_t* req, size_t req_len, const uint8_t** resp,
                           size_t* resp_len);
void sfg_batcher_stats(sfg_batcher* b, uint64_t* batches, uint64_t* frames, uint64_t* max_batch);

typedef struct {
    int32_t prefix_layers;     /* SplitConfig (client.hpp:14-20) */
    int32_t suffix_layers;
    int32_t wire_dtype;        /* SFG_WIRE_* */
    double one_way_delay_ms;   /* SimChannel latency (transport.hpp:16-21) */
} sfg_client_config;

/* Frame-level client: every exchange is an encoded frame through `handler`
 * (e.g. sfg_server_handle, or the reference's ServerEngine).                 */
int32_t sfg_client_create(sfg_engine* local, const sfg_client_config* cfg, sfg_frame_handler handler,
                          void* handler_ctx, const char* session_id, sfg_client** out);
/* Device-linked client: the server runs in this process on the same device;
 * hidden rows cross as device buffers with the wire dtype's quantisation
 * applied on device (no host copies) — the HBM-resident measurement path.  */
int32_t sfg_client_create_linked(sfg_engine* local, const sfg_client_config* cfg, sfg_server* server,
                                 const char* session_id, sfg_client** out);
void sfg_client_destroy(sfg_client* c);
int32_t sfg_client_prefill(sfg_client* c, const int32_t* prompt, int32_t n, int32_t* first_token,
                           float* logits /* nullable [vocab] */);
/* decode_step (client.cpp:169-228); mask NULL => causal; crop < 0 => none.
 * logits [seq x vocab] and argmax [seq] are optional outputs.               */
int32_t sfg_client_decode_step(sfg_client* c, int32_t seq, const int32_t* tokens,
                               const int32_t* positions, const float* mask, const int32_t* keep,
                               int32_t n_keep, int32_t crop, float* logits, int32_t* argmax);

typedef struct {
    int32_t mode;              /* 0 sequential, 2 lookahead (DecodeMode) */
    int32_t window_w;          /* LookaheadConfig (decoding.hpp:25-30) */
    int32_t ngram_n;
    int32_t max_candidates_g;
    int32_t pool_capacity;
} sfg_decode_config;

typedef struct {
    int32_t steps;
    int32_t tokens_committed;
    double wall_seconds;
    double match_rate;
    uint64_t clamped;          /* wire CodecStats::clamped, both directions */
} sfg_decode_stats;

/* decode_sequential / decode_lookahead_with_pool (decoding.cpp:111-355); the
 * per-step unembed + argmax + verify + keep/window refresh runs as one fused
 * device kernel tail; the n-gram pool LRU stays on the host.               */
int32_t sfg_decode(sfg_client* c, const sfg_decode_config* cfg, sfg_pool* pool_or_null,
                   const int32_t* prompt, int32_t n, int32_t max_new, int32_t* out_tokens,
                   float* committed_logits /* nullable [max_new x vocab] */,
                   int32_t* step_batch /* nullable [max_new] */,
                   int32_t* step_accepted /* nullable [max_new] */, sfg_decode_stats* stats);

/* The same loop, resumable one step at a time (bench.py's unit of work):
 * create runs prefill; each step is one lookahead iteration and returns the
 * tokens it committed (<= window_w + 1) and its batch size.               */
typedef struct sfg_decoder sfg_decoder;
int32_t sfg_decoder_create(sfg_client* c, const sfg_decode_config* cfg, sfg_pool* pool_or_null,
                           const int32_t* prompt, int32_t n, int32_t max_new, sfg_decoder** out);
int32_t sfg_decoder_step(sfg_decoder* d, int32_t* committed /* nullable */, int32_t* n_committed,
                         int32_t* batch);
int32_t sfg_decoder_done(const sfg_decoder* d);
void sfg_decoder_destroy(sfg_decoder* d);

/* NGramPool (decoding.hpp:35-60) */
int32_t sfg_pool_create(int32_t ngram_n, size_t capacity, sfg_pool** out);
void sfg_pool_destroy(sfg_pool* p);
int32_t sfg_pool_update(sfg_pool* p, const int32_t* previous, const int32_t* current, int32_t w);
int32_t sfg_pool_lookup(sfg_pool* p, int32_t key, int32_t max_candidates, int32_t* out);
size_t sfg_pool_size(const sfg_pool* p);

/* ── wire codec (wire.cpp:83-187), host reference implementation ───────── */
uint16_t sfg_f32_to_f16(float v, uint64_t* clamped);
/* self-test: device f32 -> binary16 -> f32 round trip of n host values */
int32_t sfg_selftest_wire_roundtrip(const float* in, float* out, int32_t n, uint64_t* clamped);
float sfg_f16_to_f32(uint16_t bits);

/* ── measurement hooks (bench.py) ──────────────────────────────────────── */
typedef struct {
    double step_ms;            /* device time of the last step (CUDA events) */
    double server_ms;          /* device time of the middle-layer forward */
    double local_ms;           /* device time of prefix + suffix + head */
    int32_t launches;          /* kernels launched by the last step */
    int32_t batch;             /* rows of the last step */
} sfg_step_profile;
int32_t sfg_client_last_profile(sfg_client* c, sfg_step_profile* out);
/* Cumulative host->device / device->host bytes moved by the library's own
 * copies since process start (bench.py measures e2e bytes per step).      */
void sfg_copy_bytes(uint64_t* h2d, uint64_t* d2h);
/* Capture / replay the device part of steps as CUDA graphs (default on). */
void sfg_set_graphs(int32_t enabled);
/* Per-kernel-class CUDA-event timing on the launching stream (bench.py's
 * roofline).  Classes: 0 QKV, 1 attention, 2 O-proj, 3 gate|up, 4 down,
 * 5 RMSNorm, 6 LM head, 7 other.  bytes/flops are ALGORITHMIC per launch,
 * summed.                                                                 */
void sfg_profiler_enable(int32_t on);
/* debugging hooks: FAST megakernel on/off; copy a bank workspace buffer
 * (0 hidden rows, 1 q, 2 attention output, 3 SwiGLU activation) to host.  */
void sfg_debug_set_mega(int32_t on);
/* megakernel phase timeline: per CTA x barrier id, globaltimer stamps of
 * {input-barrier passed, activation image done, phase done, -}           */
void sfg_debug_mega_trace(int32_t on);
int32_t sfg_debug_mega_trace_read(sfg_bank* b, uint64_t* out, size_t n);
int32_t sfg_debug_bank_buffer(sfg_bank* b, int32_t which, float* out, int32_t n);
/* the server's frame-mask parser (mask_from_frame, server.cpp:148-171): f16
 * mask [q x kv] -> per-row visible runs [start, end) in row_off / starts /
 * ends (capacity max_runs); returns 0, or the protocol status for an entry
 * other than 0 / -0 / -inf; any_empty_row flags a row with no visible
 * position (host code, no device needed: CPU tests).                      */
int32_t sfg_debug_mask_runs(const uint16_t* mask, int32_t q, int32_t kv, int32_t* row_off, int32_t* starts,
                            int32_t* ends, int32_t max_runs, int32_t* n_runs, int32_t* any_empty_row);
void sfg_profiler_reset(void);
int32_t sfg_profiler_stats(int32_t cls, int64_t* count, double* ms, double* bytes, double* flops);

#ifdef __cplusplus
}
#endif
#endif
