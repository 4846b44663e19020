/* TEST INFRASTRUCTURE ONLY — the checker, never the product.
 *
 * Plain-C restatement ("port") of the reference splitf hot path
 * (/root/reference/proj/src/{tinyformer,decoding,server,client,wire}.cpp),
 * used by tests/ and bench.py's cpu_baseline leg as the CPU oracle.  The
 * product (paper_2602_16760_b200/, libsfg.so) never links or calls this.
 *
 * Parity of this port is PINNED against (1) the reference's own golden
 * vectors (frozen stream test_tinyformer.cpp:205-213, f16 constants
 * test_wire.cpp:61-105, verify/pool known answers test_decoding.cpp:33-96)
 * and (2) the unmodified reference compiled from its sources into
 * oracle/_ref/libsplitf_ref.so (see tests/test_oracle.py).
 *
 * Arithmetic contract: fp32, serial accumulation in the reference's loop
 * order, no FMA contraction (-ffp-contract=off, no -march), glibc libm for
 * expf/powf/sincosf — identical bits to the reference built the same way.
 */
#ifndef SPLITF_ORACLE_H
#define SPLITF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int vocab_size, n_layers, hidden_dim, n_heads, n_kv_heads, head_dim, ffn_dim, max_seq_len;
    float rope_base, rms_eps;
    uint64_t seed;
} orc_cfg;

typedef struct orc_model orc_model;
typedef struct orc_bank orc_bank;
typedef struct orc_pool orc_pool;

/* status: 0 ok, else ErrorKind ordinal + 1 (error.hpp:10-21) */
const char* orc_last_error(void);

int orc_model_new(const orc_cfg* c, int bf16_round, orc_model** out);
/* only decoder layers [lo, hi) of the init stream (no embedding / head) */
int orc_model_new_layers(const orc_cfg* c, int bf16_round, int lo, int hi, orc_model** out);
/* test switch: accept q_dim != hidden_dim (NeMo-12B), see splitf_oracle.c */
void orc_set_relaxed_validate(int on);
int orc_model_from_params(const orc_cfg* c, const float* params, orc_model** out);
void orc_model_free(orc_model* m);
int64_t orc_param_count(const orc_cfg* c);
int64_t orc_model_params(const orc_model* m, float* out);

int orc_bank_new(const orc_model* m, int lb, int le, orc_bank** out);
void orc_bank_free(orc_bank* b);
void orc_bank_state(const orc_bank* b, int* len, int* committed);
void orc_bank_mark_committed(orc_bank* b, int c);
int orc_bank_resolve(orc_bank* b, const int* keep, int n);
int orc_bank_crop(orc_bank* b, int pos);
int orc_bank_kv(const orc_bank* b, int layer, int head, int pos, float* k, float* v);

int orc_embed_at(const orc_model* m, int seq, const int* ids, const int* pos, float* out);
int orc_forward(const orc_model* m, orc_bank* b, int lb, int le, int seq, const float* h,
                const int* pos, const float* mask, float* out);
int orc_finalize(const orc_model* m, int seq, const float* h, float* logits);
int orc_argmax(const float* row, int vocab);
void orc_build_causal_mask(int k, int committed, float* out);

int orc_generate(const orc_model* m, const int* prompt, int n, int max_new, int* out_tokens,
                 float* out_logits);

/* wire.cpp:83-160 */
uint16_t orc_f32_to_f16(float v, uint64_t* clamped);
float orc_f16_to_f32(uint16_t b);

/* decoding.cpp:99-109; committed must hold n+1 ints */
int orc_verify_greedy(const float* logits, int vocab, int row_begin, const int* guesses, int n,
                      int anchor, int* committed);
int orc_verify_greedy_ids(const int* row_argmax, int row_begin, const int* guesses, int n,
                          int anchor, int* committed);

/* decoding.cpp:61-97 */
int orc_pool_new(int ngram_n, size_t capacity, orc_pool** out);
void orc_pool_free(orc_pool* p);
int orc_pool_update(orc_pool* p, const int* prev, const int* cur, int w);
int orc_pool_lookup(const orc_pool* p, int key, int max_c, int* out);
size_t orc_pool_size(const orc_pool* p);

typedef struct {
    int mode; /* 0 sequential, 2 lookahead */
    int prefix_layers, suffix_layers;
    int wire_f32;
    int server_dtype; /* -1 mirror, 0 f16, 1 f32 */
    int window_w, ngram_n, max_candidates_g;
    int pool_capacity;
} orc_decode_cfg;

typedef struct {
    int steps;
    int tokens_committed;
    uint64_t clamped;
} orc_decode_stats;

/* Split pipeline decode (client.cpp + server.cpp + decoding.cpp semantics,
 * in-process, wire quantisation applied). step_* arrays hold >= max_new. */
int orc_decode(const orc_model* m, const orc_decode_cfg* dc, orc_pool* pool_or_null,
               const int* prompt, int n, int max_new, int* out_tokens, float* out_logits,
               int* step_batch, int* step_accepted, orc_decode_stats* stats);

#ifdef __cplusplus
}
#endif
#endif
