// TEST INFRASTRUCTURE ONLY — the checker, never the product.
//
// extern "C" shim over the UNMODIFIED reference splitf library
// (/root/reference/proj/src/*.cpp), compiled by oracle/Makefile into
// oracle/_ref/libsplitf_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load it.
//
// Every entry point wraps a reference symbol; the citations name the symbol
// it exercises.  Errors: 0 = ok, otherwise (ErrorKind ordinal + 1) with the
// message available from ref_last_error() (error.hpp:10-21).
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "splitf/client.hpp"
#include "splitf/decoding.hpp"
#include "splitf/metrics.hpp"
#include "splitf/server.hpp"
#include "splitf/tinyformer.hpp"
#include "splitf/transport.hpp"
#include "splitf/wire.hpp"

using namespace splitf;

namespace {

thread_local std::string g_err;
thread_local std::vector<std::byte> g_resp;

int fail(const SplitError& e) {
    g_err = e.what();
    return static_cast<int>(e.kind()) + 1;
}
int fail_other(const std::exception& e) {
    g_err = std::string("internal: ") + e.what();
    return static_cast<int>(ErrorKind::internal) + 1;
}

#define GUARD(...)                                    \
    try {                                             \
        __VA_ARGS__;                                       \
        return 0;                                     \
    } catch (const SplitError& e) {                   \
        return fail(e);                               \
    } catch (const std::exception& e) {               \
        return fail_other(e);                         \
    }

// bf16 round-to-nearest-even of an fp32 value (the shared-weights protocol,
// SURVEY §8(c) row "Parity protocol" step 1).
float bf16_round(float v) {
    uint32_t u;
    std::memcpy(&u, &v, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return v;
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    u &= 0xffff0000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
}

void round_all(Weights& w) {
    auto rd = [](std::vector<float>& v) {
        for (auto& x : v) x = bf16_round(x);
    };
    rd(w.embedding);
    for (auto& l : w.layers) {
        rd(l.attn_norm); rd(l.wq); rd(l.wk); rd(l.wv); rd(l.wo);
        rd(l.ffn_norm); rd(l.w_gate); rd(l.w_up); rd(l.w_down);
    }
    rd(w.final_norm);
    rd(w.lm_head);
}

// Partial materialisation of init_weights (tinyformer.cpp:123-152): the same
// single mt19937_64 stream in declaration order, but only the tensors of the
// requested layers are filled; the rest of the stream is discarded.  Used to
// time one 7B-wide layer without allocating 29 GB.
bool g_timing_only = false;  // skipped tensors do not advance the stream

void fill_or_skip(std::vector<float>& dst, size_t n, float a, std::mt19937_64& rng, bool keep) {
    if (!keep) {
        if (!g_timing_only) rng.discard(n);
        return;
    }
    dst.resize(n);
    for (size_t i = 0; i < n; ++i) {
        const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
        dst[i] = a * static_cast<float>(2.0 * u - 1.0);
    }
}

bool g_unchecked = false;  // skip ModelConfig::validate (q_dim != hidden shapes)

Weights partial_weights(const ModelConfig& c, int lo, int hi, bool head) {
    if (!g_unchecked) c.validate();
    Weights w;
    w.config = c;
    w.layers.resize(c.n_layers);
    const float a = 1.0f / std::sqrt(static_cast<float>(c.hidden_dim));
    std::mt19937_64 rng(c.seed);
    const size_t h = c.hidden_dim, qd = c.q_dim(), kvd = c.kv_dim(), f = c.ffn_dim;
    fill_or_skip(w.embedding, c.vocab_size * h, a, rng, head);
    for (int i = 0; i < c.n_layers; ++i) {
        auto& l = w.layers[i];
        const bool k = i >= lo && i < hi;
        fill_or_skip(l.attn_norm, h, a, rng, k);
        fill_or_skip(l.wq, h * qd, a, rng, k);
        fill_or_skip(l.wk, h * kvd, a, rng, k);
        fill_or_skip(l.wv, h * kvd, a, rng, k);
        fill_or_skip(l.wo, qd * h, a, rng, k);
        fill_or_skip(l.ffn_norm, h, a, rng, k);
        fill_or_skip(l.w_gate, h * f, a, rng, k);
        fill_or_skip(l.w_up, h * f, a, rng, k);
        fill_or_skip(l.w_down, f * h, a, rng, k);
    }
    fill_or_skip(w.final_norm, h, a, rng, head);
    fill_or_skip(w.lm_head, h * c.vocab_size, a, rng, head);
    return w;
}

}  // namespace

extern "C" {

typedef struct {
    int vocab_size, n_layers, hidden_dim, n_heads, n_kv_heads, head_dim, ffn_dim, max_seq_len;
    float rope_base, rms_eps;
    uint64_t seed;
} ref_model_cfg;

typedef int32_t (*ref_frame_handler)(void* ctx, const uint8_t* req, size_t req_len,
                                     const uint8_t** resp, size_t* resp_len);

typedef struct {
    int mode;           // 0 sequential, 1 jacobi, 2 lookahead
    int prefix_layers;
    int suffix_layers;
    int wire_f32;       // SplitConfig::dtype
    int server_dtype;   // -1 mirror, 0 f16, 1 f32 (ServerConfig::response_dtype)
    int window_w, ngram_n, max_candidates_g;
    int pool_capacity;
    int block_k;
    double rtt_ms;
} ref_decode_cfg;

typedef struct {
    int steps;
    int tokens_committed;
    double wall_seconds;
    double acceptance_rate;
    double match_rate;
    double prefill_ms;
} ref_decode_stats;

const char* ref_last_error(void) { return g_err.c_str(); }

static ModelConfig to_cfg(const ref_model_cfg* c) {
    ModelConfig m;
    m.vocab_size = c->vocab_size;
    m.n_layers = c->n_layers;
    m.hidden_dim = c->hidden_dim;
    m.n_heads = c->n_heads;
    m.n_kv_heads = c->n_kv_heads;
    m.head_dim = c->head_dim;
    m.ffn_dim = c->ffn_dim;
    m.max_seq_len = c->max_seq_len;
    m.rope_base = c->rope_base;
    m.rms_eps = c->rms_eps;
    m.seed = c->seed;
    return m;
}

// init_weights (tinyformer.cpp:123) [+ bf16 RNE rounding in place].
// layer_lo/layer_hi < 0 => full reference init_weights; otherwise partial.
int ref_model_new(const ref_model_cfg* c, int bf16, int layer_lo, int layer_hi, int with_head,
                  void** out) {
    GUARD({
        auto* w = new Weights(layer_lo < 0 ? init_weights(to_cfg(c))
                                           : partial_weights(to_cfg(c), layer_lo, layer_hi,
                                                             with_head != 0));
        if (bf16) round_all(*w);
        *out = w;
    })
}

// The same partial init without ModelConfig::validate: q_dim != hidden_dim
// (Mistral NeMo 12B, 32 x 128 = 4096 vs 5120).  init_weights / ServerEngine /
// SplitClient reject that shape (tinyformer.cpp:109-111), but forward_layers
// and CacheBank never validate and use q_dim() throughout (:405-406, :444,
// :491), so the reference's own forward_layers runs on it unmodified.
int ref_model_new_unchecked(const ref_model_cfg* c, int bf16, int layer_lo, int layer_hi, int with_head,
                            void** out) {
    GUARD({
        g_unchecked = true;
        try {
            auto* w = new Weights(partial_weights(to_cfg(c), layer_lo, layer_hi, with_head != 0));
            if (bf16) round_all(*w);
            *out = w;
        } catch (...) {
            g_unchecked = false;
            throw;
        }
        g_unchecked = false;
    })
}

// Timing-only model for the CPU baseline: the requested tensors get
// U[-a, a] values (same distribution, NOT the reference stream positions)
// without walking the 7.25 G-draw stream; arithmetic cost is identical.
int ref_model_new_timing(const ref_model_cfg* c, int layer_lo, int layer_hi, int with_head, void** out) {
    GUARD({
        g_timing_only = true;
        g_unchecked = true;  // timing only: the NeMo-12B true shape (q_dim != hidden) too
        try {
            *out = new Weights(partial_weights(to_cfg(c), layer_lo, layer_hi, with_head != 0));
        } catch (...) {
            g_timing_only = false;
            g_unchecked = false;
            throw;
        }
        g_timing_only = false;
        g_unchecked = false;
    })
}

void ref_model_free(void* m) { delete static_cast<Weights*>(m); }

// Flat parameter dump in snapshot declaration order (PROTOCOL.md "Weight
// snapshots"); returns the parameter count, copies when out != NULL.
int64_t ref_model_params(void* m, float* out) {
    auto& w = *static_cast<Weights*>(m);
    int64_t n = 0;
    auto put = [&](const std::vector<float>& v) {
        if (out) std::memcpy(out + n, v.data(), v.size() * sizeof(float));
        n += static_cast<int64_t>(v.size());
    };
    put(w.embedding);
    for (auto& l : w.layers) {
        put(l.attn_norm); put(l.wq); put(l.wk); put(l.wv); put(l.wo);
        put(l.ffn_norm); put(l.w_gate); put(l.w_up); put(l.w_down);
    }
    put(w.final_norm);
    put(w.lm_head);
    return n;
}

// generate_monolithic_traced (tinyformer.cpp:534-573)
int ref_generate(void* m, const int* prompt, int n, int max_new, int* out_tokens,
                 float* out_logits) {
    GUARD({
        auto& w = *static_cast<Weights*>(m);
        MonolithicTrace t = generate_monolithic_traced(w, std::span<const int>(prompt, n), max_new);
        std::memcpy(out_tokens, t.tokens.data(), t.tokens.size() * sizeof(int));
        if (out_logits) std::memcpy(out_logits, t.step_logits.data.data(),
                                    t.step_logits.data.size() * sizeof(float));
    })
}

// Split pipeline (metrics.cpp:165-185 pieces) + run_decode (decoding.cpp:357).
// With handler == NULL the server side is the reference ServerEngine; with a
// handler, every request frame is encoded (wire.cpp:189) and handed to the
// C callback — this is how the GPU engine is dropped in behind the
// reference's own client and decode loop.
int ref_decode(void* m, const ref_decode_cfg* dc, const int* prompt, int n, int max_new,
               ref_frame_handler handler, void* hctx, int* out_tokens, float* out_logits,
               int* step_batch, int* step_accepted, ref_decode_stats* stats) {
    GUARD({
        auto& w = *static_cast<Weights*>(m);
        SplitConfig split;
        split.prefix_layers = dc->prefix_layers;
        split.suffix_layers = dc->suffix_layers;
        split.dtype = dc->wire_f32 ? wire::WireDtype::f32 : wire::WireDtype::f16;
        LatencyProfile link;
        link.one_way_delay_ms = dc->rtt_ms / 2.0;

        std::unique_ptr<ServerEngine> engine;
        FrameHandler fh;
        if (handler == nullptr) {
            ServerConfig sc;
            sc.layer_begin = split.prefix_layers;
            sc.layer_end = w.config.n_layers - split.suffix_layers;
            if (dc->server_dtype == 0) sc.response_dtype = wire::WireDtype::f16;
            if (dc->server_dtype == 1) sc.response_dtype = wire::WireDtype::f32;
            engine = std::make_unique<ServerEngine>(w, sc);
            ServerEngine* e = engine.get();
            fh = [e](const wire::Frame& f) { return e->handle(f); };
        } else {
            fh = [handler, hctx](const wire::Frame& f) {
                const auto bytes = wire::encode_frame(f);
                const uint8_t* resp = nullptr;
                size_t rlen = 0;
                const int32_t rc = handler(hctx, reinterpret_cast<const uint8_t*>(bytes.data()),
                                           bytes.size(), &resp, &rlen);
                if (rc != 0) throw SplitError(ErrorKind::transport, "handler failed");
                return wire::decode_frame(
                    std::span<const std::byte>(reinterpret_cast<const std::byte*>(resp), rlen));
            };
        }
        auto channel = open_sim_channel(link, fh);
        SplitClient client(w, split, *channel);
        JacobiConfig jc;
        jc.block_k = dc->block_k > 0 ? dc->block_k : 4;
        LookaheadConfig lc;
        lc.ngram_n = dc->ngram_n;
        lc.window_w = dc->window_w;
        lc.max_candidates_g = dc->max_candidates_g;
        lc.pool_capacity = static_cast<size_t>(dc->pool_capacity);
        const auto mode = dc->mode == 0   ? DecodeMode::sequential
                          : dc->mode == 1 ? DecodeMode::jacobi
                                          : DecodeMode::lookahead;
        DecodeResult r = run_decode(mode, client, std::span<const int>(prompt, n), max_new, jc, lc);
        std::memcpy(out_tokens, r.tokens.data(), r.tokens.size() * sizeof(int));
        if (out_logits) std::memcpy(out_logits, r.committed_logits.data.data(),
                                    r.committed_logits.data.size() * sizeof(float));
        for (size_t i = 0; i < r.stats.step_timings.size(); ++i) {
            if (step_batch) step_batch[i] = r.stats.step_timings[i].batch_len;
            if (step_accepted) step_accepted[i] = r.stats.step_timings[i].accepted;
        }
        if (stats) {
            stats->steps = r.stats.steps;
            stats->tokens_committed = r.stats.tokens_committed;
            stats->wall_seconds = r.stats.wall_seconds;
            stats->acceptance_rate = r.stats.acceptance_rate;
            stats->match_rate = r.stats.match_rate;
            stats->prefill_ms = r.stats.prefill_ms;
        }
    })
}

// ── CacheBank / forward_layers / finalize (tinyformer.hpp:131-179) ───────

int ref_bank_new(void* m, int lb, int le, void** out) {
    GUARD({ *out = new CacheBank(static_cast<Weights*>(m)->config, lb, le); })
}
void ref_bank_free(void* b) { delete static_cast<CacheBank*>(b); }

// forward_layers (tinyformer.cpp:375-508); mask == NULL => causal
// build_attention_mask(seq, bank.len()) (tinyformer.cpp:229-241).
int ref_forward(void* m, void* bank, int lb, int le, int seq, const float* h, const int* pos,
                const float* mask, float* out) {
    GUARD({
        auto& w = *static_cast<Weights*>(m);
        auto& b = *static_cast<CacheBank*>(bank);
        HiddenStates hs;
        hs.seq = seq;
        hs.dim = w.config.hidden_dim;
        hs.data.assign(h, h + static_cast<size_t>(seq) * hs.dim);
        hs.positions.assign(pos, pos + seq);
        AttentionMask am;
        if (mask) {
            am.q_len = seq;
            am.kv_len = b.len() + seq;
            am.data.assign(mask, mask + static_cast<size_t>(am.q_len) * am.kv_len);
        } else {
            am = build_attention_mask(seq, b.len());
        }
        HiddenStates o = forward_layers(w, lb, le, hs, b, am);
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
    })
}

int ref_bank_resolve(void* bank, const int* keep, int n) {
    GUARD({ static_cast<CacheBank*>(bank)->resolve(std::span<const int>(keep, n)); })
}
int ref_bank_crop(void* bank, int pos) { GUARD({ static_cast<CacheBank*>(bank)->crop(pos); }) }
void ref_bank_mark_committed(void* bank, int c) { static_cast<CacheBank*>(bank)->mark_committed(c); }
void ref_bank_state(void* bank, int* len, int* committed) {
    auto& b = *static_cast<CacheBank*>(bank);
    *len = b.len();
    *committed = b.committed_len();
}
int ref_bank_kv(void* bank, int layer, int head, int pos, float* k, float* v) {
    GUARD({
        auto& c = static_cast<CacheBank*>(bank)->layer(layer);
        std::memcpy(k, c.key_at(head, pos), sizeof(float) * c.head_dim);
        std::memcpy(v, c.value_at(head, pos), sizeof(float) * c.head_dim);
    })
}

// Test hook: install a whole layer's K/V slabs [n_kv_heads x max_len x
// head_dim] (e.g. read back from the GPU bank) and set its length, so a
// long-context step can be checked without a CPU prefill of the context.
int ref_bank_load_layer(void* bank, int layer, const float* k, const float* v, int len) {
    GUARD({
        auto& c = static_cast<CacheBank*>(bank)->layer(layer);
        std::memcpy(c.keys.data(), k, c.keys.size() * sizeof(float));
        std::memcpy(c.values.data(), v, c.values.size() * sizeof(float));
        c.len = len;
    })
}

int ref_embed_at(void* m, int seq, const int* ids, const int* pos, float* out) {
    GUARD({
        HiddenStates h = embed_at(*static_cast<Weights*>(m), std::span<const int>(ids, seq),
                                  std::span<const int>(pos, seq));
        std::memcpy(out, h.data.data(), h.data.size() * sizeof(float));
    })
}

int ref_finalize(void* m, int seq, const float* h, float* logits) {
    GUARD({
        auto& w = *static_cast<Weights*>(m);
        HiddenStates hs;
        hs.seq = seq;
        hs.dim = w.config.hidden_dim;
        hs.data.assign(h, h + static_cast<size_t>(seq) * hs.dim);
        hs.positions.assign(seq, 0);
        Logits l = finalize(w, hs);
        std::memcpy(logits, l.data.data(), l.data.size() * sizeof(float));
    })
}

int ref_argmax(int vocab, const float* row) {
    Logits l;
    l.seq = 1;
    l.vocab = vocab;
    l.data.assign(row, row + vocab);
    return argmax_row(l, 0);
}

// verify_greedy (decoding.cpp:99-109); committed has room for n+1.
int ref_verify_greedy(int seq, int vocab, const float* logits, int row_begin, const int* guesses,
                      int n, int anchor, int* accepted, int* committed) {
    GUARD({
        Logits l;
        l.seq = seq;
        l.vocab = vocab;
        l.data.assign(logits, logits + static_cast<size_t>(seq) * vocab);
        VerifyResult vr = verify_greedy(l, row_begin, std::span<const int>(guesses, n), anchor);
        *accepted = vr.accepted;
        std::memcpy(committed, vr.committed.data(), vr.committed.size() * sizeof(int));
    })
}

// ── NGramPool (decoding.cpp:61-97) ───────────────────────────────────────
int ref_pool_new(int n, size_t cap, void** out) { GUARD({ *out = new NGramPool(n, cap); }) }
void ref_pool_free(void* p) { delete static_cast<NGramPool*>(p); }
// Copy of a pool (NGramPool is a value type): a junk pool seeded once is
// handed to several concurrent decodes.
int ref_pool_clone(void* p, void** out) { GUARD({ *out = new NGramPool(*static_cast<NGramPool*>(p)); }) }
int ref_pool_update(void* p, const int* prev, const int* cur, int w) {
    GUARD({
        static_cast<NGramPool*>(p)->update(std::span<const int>(prev, w),
                                           std::span<const int>(cur, w));
    })
}
// Writes up to max_c continuations of (n-1) tokens each; returns the count.
int ref_pool_lookup(void* p, int key, int max_c, int* out) {
    auto* pool = static_cast<NGramPool*>(p);
    auto hits = pool->lookup(key, max_c);
    int off = 0;
    for (auto& c : hits)
        for (int t : c) out[off++] = t;
    return static_cast<int>(hits.size());
}
size_t ref_pool_size(void* p) { return static_cast<NGramPool*>(p)->size(); }

// ── ServerEngine (server.hpp:28-77) ──────────────────────────────────────
struct RefServer {
    std::unique_ptr<ServerEngine> engine;
    const double* clock = nullptr;
};

int ref_server_new(void* m, int lb, int le, double expiry_s, int max_sessions, int response_dtype,
                   void** out) {
    GUARD({
        ServerConfig sc;
        sc.layer_begin = lb;
        sc.layer_end = le;
        sc.session_expiry_s = expiry_s;
        sc.max_sessions = max_sessions;
        if (response_dtype == 0) sc.response_dtype = wire::WireDtype::f16;
        if (response_dtype == 1) sc.response_dtype = wire::WireDtype::f32;
        auto* s = new RefServer;
        s->engine = std::make_unique<ServerEngine>(*static_cast<Weights*>(m), sc);
        *out = s;
    })
}
void ref_server_free(void* s) { delete static_cast<RefServer*>(s); }

// decode_frame → ServerEngine::handle → encode_frame (server.cpp:173-191).
int32_t ref_server_handle(void* s, const uint8_t* req, size_t n, const uint8_t** resp,
                          size_t* resp_n) {
    GUARD({
        auto* rs = static_cast<RefServer*>(s);
        wire::Frame f;
        try {
            f = wire::decode_frame(
                std::span<const std::byte>(reinterpret_cast<const std::byte*>(req), n));
        } catch (const SplitError& e) {
            wire::Frame err;
            err.header.kind = wire::FrameKind::error;
            err.header.tensor_shape = {0};
            err.header.error_msg = e.what();
            g_resp = wire::encode_frame(err);
            *resp = reinterpret_cast<const uint8_t*>(g_resp.data());
            *resp_n = g_resp.size();
            return 0;
        }
        g_resp = wire::encode_frame(rs->engine->handle(f));
        *resp = reinterpret_cast<const uint8_t*>(g_resp.data());
        *resp_n = g_resp.size();
    })
}
void ref_server_set_clock(void* s, const double* now) {
    auto* rs = static_cast<RefServer*>(s);
    rs->clock = now;
    rs->engine->set_clock([rs] { return *rs->clock; });
}
int ref_server_session_view(void* s, const char* sid, int* len, int* committed, int* prov) {
    auto v = static_cast<RefServer*>(s)->engine->session_view(sid);
    if (!v) return 0;
    *len = v->cache_len;
    *committed = v->committed_len;
    *prov = v->provisional;
    return 1;
}
size_t ref_server_expire(void* s) { return static_cast<RefServer*>(s)->engine->expire_sessions(); }
size_t ref_server_count(void* s) { return static_cast<RefServer*>(s)->engine->session_count(); }

// ── wire (wire.cpp:83-187) ───────────────────────────────────────────────
uint16_t ref_f32_to_f16(float v, uint64_t* clamped) {
    wire::CodecStats st;
    const uint16_t b = wire::f32_to_f16_bits(v, &st);
    if (clamped) *clamped += st.clamped;
    return b;
}
float ref_f16_to_f32(uint16_t b) { return wire::f16_bits_to_f32(b); }

// Corpora (metrics.cpp:107-134): kind 0 repetitive, 1 random.
int ref_corpus(int kind, int vocab, int n_prompts, int prompt_len, uint64_t seed, int* out) {
    GUARD({
        ModelConfig c;
        c.vocab_size = vocab;
        Corpus k = kind == 0 ? make_repetitive_corpus(c, n_prompts, prompt_len, seed)
                             : make_random_corpus(c, n_prompts, prompt_len, seed);
        int off = 0;
        for (auto& p : k.prompts)
            for (int t : p) out[off++] = t;
    })
}

// CPU-baseline timing helper: runs forward_layers over [lb, le) for `seq`
// rows on `threads` independent banks concurrently (one session per host
// thread, which is how the reference scales: server.cpp sessions + one
// FrameServer thread each).  Returns wall seconds.
double ref_time_forward(void* m, int lb, int le, int seq, int ctx, int threads) {
    auto& w = *static_cast<Weights*>(m);
    const int hidden = w.config.hidden_dim;
    std::vector<std::thread> ts;
    const auto t0 = std::chrono::steady_clock::now();
    for (int t = 0; t < threads; ++t) {
        ts.emplace_back([&, t] {
            CacheBank bank(w.config, lb, le);
            std::mt19937_64 rng(99 + t);
            if (ctx > 0) {
                for (int l = lb; l < le; ++l) {
                    auto& c = bank.layer(l);
                    for (auto& x : c.keys) x = static_cast<float>((rng() >> 40) * 0x1.0p-24) - 0.5f;
                    for (auto& x : c.values) x = static_cast<float>((rng() >> 40) * 0x1.0p-24) - 0.5f;
                    c.len = ctx;
                }
                bank.mark_committed(ctx);
            }
            HiddenStates h;
            h.seq = seq;
            h.dim = hidden;
            h.data.resize(static_cast<size_t>(seq) * hidden);
            for (auto& x : h.data) x = static_cast<float>((rng() >> 40) * 0x1.0p-24) - 0.5f;
            for (int i = 0; i < seq; ++i) h.positions.push_back(ctx + i);
            forward_layers(w, lb, le, h, bank, build_attention_mask(seq, ctx));
        });
    }
    for (auto& th : ts) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

double ref_time_finalize(void* m, int seq, int threads) {
    auto& w = *static_cast<Weights*>(m);
    std::vector<std::thread> ts;
    const auto t0 = std::chrono::steady_clock::now();
    for (int t = 0; t < threads; ++t) {
        ts.emplace_back([&, t] {
            HiddenStates h;
            h.seq = seq;
            h.dim = w.config.hidden_dim;
            h.data.assign(static_cast<size_t>(seq) * h.dim, 0.25f + 0.01f * t);
            h.positions.assign(seq, 0);
            finalize(w, h);
        });
    }
    for (auto& th : ts) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}


// ── 7B-shape golden generation (tests/golden/make_golden_7b.py) ──────────
// The reference ServerEngine takes its Weights by value and the client keeps a
// reference, so a full 7B split pipeline would hold 2 x 29 GB fp32.  Here ONE
// walk of the init_weights stream (tinyformer.cpp:123-152) fills two disjoint
// Weights objects: the client's (embedding, prefix + suffix layers, final
// norm, lm_head) and the server's (middle layers only).  Each reference
// function then touches only the tensors it owns (forward_layers over
// [begin, end), embed_at, finalize), so results are those of the full model.
int ref_split_models(const ref_model_cfg* cc, int bf16, int prefix, int suffix, void** client_out,
                     void** server_out) {
    GUARD({
        const ModelConfig c = to_cfg(cc);
        c.validate();
        auto cw = std::make_unique<Weights>();
        auto sw = std::make_unique<Weights>();
        cw->config = sw->config = c;
        cw->layers.resize(c.n_layers);
        sw->layers.resize(c.n_layers);
        const float a = 1.0f / std::sqrt(static_cast<float>(c.hidden_dim));
        std::mt19937_64 rng(c.seed);
        const size_t h = c.hidden_dim, qd = c.q_dim(), kvd = c.kv_dim(), f = c.ffn_dim;
        fill_or_skip(cw->embedding, c.vocab_size * h, a, rng, true);
        for (int i = 0; i < c.n_layers; ++i) {
            const bool local = i < prefix || i >= c.n_layers - suffix;
            auto& l = local ? cw->layers[i] : sw->layers[i];
            fill_or_skip(l.attn_norm, h, a, rng, true);
            fill_or_skip(l.wq, h * qd, a, rng, true);
            fill_or_skip(l.wk, h * kvd, a, rng, true);
            fill_or_skip(l.wv, h * kvd, a, rng, true);
            fill_or_skip(l.wo, qd * h, a, rng, true);
            fill_or_skip(l.ffn_norm, h, a, rng, true);
            fill_or_skip(l.w_gate, h * f, a, rng, true);
            fill_or_skip(l.w_up, h * f, a, rng, true);
            fill_or_skip(l.w_down, f * h, a, rng, true);
        }
        fill_or_skip(cw->final_norm, h, a, rng, true);
        fill_or_skip(cw->lm_head, h * c.vocab_size, a, rng, true);
        if (bf16) {
            round_all(*cw);
            round_all(*sw);
        }
        *client_out = cw.release();
        *server_out = sw.release();
    })
}

// ServerEngine over a Weights object that is MOVED in (server.cpp:27-28);
// `weights` is consumed (freed) on success.
int ref_server_new_move(void* weights, int lb, int le, int max_sessions, void** out) {
    GUARD({
        ServerConfig sc;
        sc.layer_begin = lb;
        sc.layer_end = le;
        sc.max_sessions = max_sessions;
        auto* w = static_cast<Weights*>(weights);
        auto* s = new RefServer;
        s->engine = std::make_unique<ServerEngine>(std::move(*w), sc);
        delete w;
        *out = s;
    })
}

// One decode through the reference client + decode loop against a shared
// reference ServerEngine (thread safe across sessions, server.hpp:53-57).
// mode 0 = decode_sequential, 2 = decode_lookahead_with_pool(pool) when pool
// != NULL else decode_lookahead.  The first `rec_frames` exchanges record the
// boundary rows as the reference saw them: the request rows decoded from the
// wire (prefix output) and the response rows (middle-layer output), each
// [rec_frames x max_rows x hidden] fp32, rows per frame in rec_rows.
int ref_decode_on(void* client_w, void* server, const ref_decode_cfg* dc, void* pool,
                  const char* session_id, const int* prompt, int n, int max_new, int rec_frames,
                  int max_rows, float* rec_req, float* rec_resp, int* rec_rows, int* out_tokens,
                  int* step_batch, int* step_accepted, ref_decode_stats* stats) {
    GUARD({
        auto& w = *static_cast<Weights*>(client_w);
        auto* rs = static_cast<RefServer*>(server);
        SplitConfig split;
        split.prefix_layers = dc->prefix_layers;
        split.suffix_layers = dc->suffix_layers;
        split.dtype = dc->wire_f32 ? wire::WireDtype::f32 : wire::WireDtype::f16;
        const int hd = w.config.hidden_dim;
        int frame_no = 0;
        FrameHandler fh = [&](const wire::Frame& f) {
            wire::Frame r = rs->engine->handle(f);
            if (frame_no < rec_frames && r.header.kind == wire::FrameKind::response) {
                const int rows = f.header.tensor_shape.empty() ? 0 : f.header.tensor_shape[0];
                const int take = rows < max_rows ? rows : max_rows;
                const auto in = wire::decode_values(f.tensor_bytes, f.header.dtype);
                const auto outv = wire::decode_values(r.tensor_bytes, r.header.dtype);
                const size_t base = static_cast<size_t>(frame_no) * max_rows * hd;
                std::memcpy(rec_req + base, in.data(), sizeof(float) * take * hd);
                std::memcpy(rec_resp + base, outv.data(), sizeof(float) * take * hd);
                rec_rows[frame_no] = take;
            }
            ++frame_no;
            return r;
        };
        LatencyProfile link;
        auto channel = open_sim_channel(link, fh);
        SplitClient client(w, split, *channel, session_id ? std::string(session_id) : std::string());
        LookaheadConfig lc;
        lc.ngram_n = dc->ngram_n;
        lc.window_w = dc->window_w;
        lc.max_candidates_g = dc->max_candidates_g;
        lc.pool_capacity = static_cast<size_t>(dc->pool_capacity);
        const std::span<const int> ps(prompt, n);
        DecodeResult r = dc->mode == 0 ? decode_sequential(client, ps, max_new)
                         : pool      ? decode_lookahead_with_pool(client, ps, max_new, lc,
                                                                  *static_cast<NGramPool*>(pool))
                                     : decode_lookahead(client, ps, max_new, lc);
        std::memcpy(out_tokens, r.tokens.data(), r.tokens.size() * sizeof(int));
        for (size_t i = 0; i < r.stats.step_timings.size(); ++i) {
            if (step_batch) step_batch[i] = r.stats.step_timings[i].batch_len;
            if (step_accepted) step_accepted[i] = r.stats.step_timings[i].accepted;
        }
        if (stats) {
            stats->steps = r.stats.steps;
            stats->tokens_committed = r.stats.tokens_committed;
            stats->wall_seconds = r.stats.wall_seconds;
            stats->acceptance_rate = r.stats.acceptance_rate;
            stats->match_rate = r.stats.match_rate;
            stats->prefill_ms = r.stats.prefill_ms;
        }
    })
}

}  // extern "C"
