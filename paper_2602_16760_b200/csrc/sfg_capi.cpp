// extern "C" boundary (include/sfg.h): status codes = ErrorKind + 1, the
// thread-local message is the exact text the reference would throw.
#include <cstring>
#include <memory>
#include <string>

#include "../../include/sfg.h"
#include "sfg_client.h"
#include "sfg_engine.h"
#include "sfg_prof.h"
#include "sfg_router.h"
#include "sfg_server.h"
#include "sfg_wire.h"

using namespace sfg;

namespace {
thread_local std::string g_err;
thread_local std::vector<uint8_t> g_resp;

int32_t fail(const Error& e) {
    g_err = e.what();
    return static_cast<int32_t>(e.kind());
}
int32_t fail_other(const std::exception& e) {
    g_err = std::string("internal: ") + e.what();
    return SFG_ERR_INTERNAL;
}
}  // namespace

#define SFG_GUARD(...)                      \
    try {                                   \
        __VA_ARGS__;                        \
        return SFG_OK;                      \
    } catch (const Error& e) {              \
        return fail(e);                     \
    } catch (const std::exception& e) {     \
        return fail_other(e);               \
    }

struct sfg_engine { std::unique_ptr<Engine> e; };
struct sfg_bank { std::unique_ptr<Bank> b; sfg_engine* eng; };
struct sfg_server { std::unique_ptr<Server> s; double (*clock)(void*) = nullptr; void* clock_ctx = nullptr; };
struct sfg_client { std::unique_ptr<Client> c; };
struct sfg_pool { std::unique_ptr<Pool> p; };
struct sfg_router { std::unique_ptr<Router> r; double (*clock)(void*) = nullptr; void* clock_ctx = nullptr; };
struct sfg_batcher { std::unique_ptr<Batcher> b; };

extern "C" {

const char* sfg_last_error(void) { return g_err.c_str(); }
const char* sfg_version(void) { return "sfg 0.1 (sm_100a)"; }

static int32_t make_engine(const sfg_model_config* cfg, const sfg_engine_options* opt, const float* params,
                           sfg_engine** out, const TpConfig& tp = TpConfig{}) {
    SFG_GUARD({
        if (!cfg || !opt || !out) throw Error(Kind::input, "null argument");
        auto* h = new sfg_engine;
        try {
            h->e = std::make_unique<Engine>(ModelCfg::from_c(*cfg), *opt, params, tp);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    })
}

int32_t sfg_engine_create_seeded(const sfg_model_config* cfg, const sfg_engine_options* opt, sfg_engine** out) {
    return make_engine(cfg, opt, nullptr, out);
}
int32_t sfg_engine_create_from_params(const sfg_model_config* cfg, const sfg_engine_options* opt,
                                      const float* params, sfg_engine** out) {
    if (!params) {
        g_err = "input: null parameter array";
        return SFG_ERR_INPUT;
    }
    return make_engine(cfg, opt, params, out);
}
int32_t sfg_tp_unique_id(uint8_t* out) {
    SFG_GUARD({
        if (!out) throw Error(Kind::input, "null argument");
        tp_unique_id(out, SFG_TP_ID_BYTES);
    })
}
int32_t sfg_engine_create_tp(const sfg_model_config* cfg, const sfg_engine_options* opt, int32_t tp_size,
                             int32_t tp_rank, const uint8_t* tp_unique_id, sfg_engine** out) {
    TpConfig tp;
    tp.size = tp_size;
    tp.rank = tp_rank;
    tp.unique_id = tp_unique_id;
    return make_engine(cfg, opt, nullptr, out, tp);
}
void sfg_engine_destroy(sfg_engine* eng) { delete eng; }
int64_t sfg_engine_weight_bytes(const sfg_engine* eng) { return eng ? eng->e->weight_bytes() : 0; }

int32_t sfg_bank_create(sfg_engine* eng, int32_t lb, int32_t le, sfg_bank** out) {
    SFG_GUARD({
        auto* b = new sfg_bank;
        b->eng = eng;
        try {
            b->b = std::make_unique<Bank>(*eng->e, lb, le);
        } catch (...) {
            delete b;
            throw;
        }
        *out = b;
    })
}
void sfg_bank_destroy(sfg_bank* b) { delete b; }
int32_t sfg_bank_resolve(sfg_bank* b, const int32_t* keep, int32_t n) { SFG_GUARD(b->b->resolve(keep, n)) }
int32_t sfg_bank_crop(sfg_bank* b, int32_t pos) { SFG_GUARD(b->b->crop(pos)) }
void sfg_bank_mark_committed(sfg_bank* b, int32_t c) { b->b->mark_committed(c); }
void sfg_bank_reset(sfg_bank* b) { b->b->reset(); }
void sfg_bank_state(const sfg_bank* b, int32_t* len, int32_t* committed) {
    *len = b->b->len();
    *committed = b->b->committed_len();
}
int32_t sfg_bank_read_kv(sfg_bank* b, int32_t layer, int32_t head, int32_t pos, float* k, float* v) {
    SFG_GUARD(b->b->read_kv(layer, head, pos, k, v))
}

int32_t sfg_forward_layers(sfg_engine* eng, sfg_bank* b, int32_t lb, int32_t le, int32_t seq, const float* hidden,
                           const int32_t* positions, const float* mask, float* out) {
    SFG_GUARD(eng->e->forward_host(*b->b, lb, le, seq, hidden, positions, mask, out))
}
int32_t sfg_embed_at(sfg_engine* eng, int32_t seq, const int32_t* ids, const int32_t* positions, float* out) {
    SFG_GUARD(eng->e->embed_host(seq, ids, positions, out))
}
int32_t sfg_finalize(sfg_engine* eng, int32_t seq, const float* hidden, float* logits) {
    SFG_GUARD(eng->e->finalize_host(seq, hidden, logits, nullptr))
}
int32_t sfg_finalize_argmax(sfg_engine* eng, int32_t seq, const float* hidden, int32_t* argmax) {
    SFG_GUARD(eng->e->finalize_host(seq, hidden, nullptr, argmax))
}

int32_t sfg_server_create(sfg_engine* eng, const sfg_server_config* cfg, sfg_server** out) {
    SFG_GUARD({
        ServerCfg sc;
        sc.layer_begin = cfg->layer_begin;
        sc.layer_end = cfg->layer_end;
        sc.session_expiry_s = cfg->session_expiry_s;
        sc.max_sessions = cfg->max_sessions;
        sc.response_dtype = cfg->response_dtype;
        auto* s = new sfg_server;
        try {
            s->s = std::make_unique<Server>(*eng->e, sc);
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    })
}
void sfg_server_destroy(sfg_server* s) { delete s; }
int32_t sfg_server_handle(sfg_server* s, const uint8_t* req, size_t n, const uint8_t** resp, size_t* resp_len) {
    SFG_GUARD({
        s->s->handle(req, n, g_resp);
        *resp = g_resp.data();
        *resp_len = g_resp.size();
    })
}
int32_t sfg_server_handle_batch(sfg_server* s, int32_t n, const uint8_t* const* reqs, const size_t* req_lens,
                                const uint8_t** resps, size_t* resp_lens) {
    SFG_GUARD({
        if (n < 0) throw sfg::Error(sfg::Kind::input, "negative frame count");
        thread_local std::vector<std::vector<uint8_t>> out;
        s->s->handle_batch(n, reqs, req_lens, out);
        for (int32_t i = 0; i < n; ++i) {
            resps[i] = out[i].data();
            resp_lens[i] = out[i].size();
        }
    })
}
uint64_t sfg_server_shared_passes(sfg_server* s) { return s->s->shared_passes(); }
size_t sfg_server_expire_sessions(sfg_server* s) { return s->s->expire_sessions(); }
size_t sfg_server_session_count(sfg_server* s) { return s->s->session_count(); }
int32_t sfg_server_session_view(sfg_server* s, const char* sid, int32_t* len, int32_t* committed, int32_t* prov) {
    int a = 0, b = 0, c = 0;
    if (!s->s->session_view(sid, &a, &b, &c)) return 0;
    *len = a;
    *committed = b;
    *prov = c;
    return 1;
}
// ── router / batching queue (sfg_router.h) ─────────────────────────────
int32_t sfg_router_create(sfg_server* const* servers, int32_t n, double session_expiry_s, sfg_router** out) {
    SFG_GUARD({
        if (n < 1 || !servers) throw sfg::Error(sfg::Kind::config, "router needs at least one backend");
        std::vector<Backend> bs(static_cast<size_t>(n));
        for (int32_t i = 0; i < n; ++i) {
            if (!servers[i]) throw sfg::Error(sfg::Kind::config, "null server");
            bs[i].server = servers[i]->s.get();
        }
        auto r = std::make_unique<sfg_router>();
        r->r = std::make_unique<Router>(std::move(bs), session_expiry_s);
        *out = r.release();
    })
}
int32_t sfg_router_create_handlers(const sfg_frame_handler* fns, void* const* ctxs, int32_t n, double session_expiry_s,
                                   sfg_router** out) {
    SFG_GUARD({
        if (n < 1 || !fns) throw sfg::Error(sfg::Kind::config, "router needs at least one backend");
        std::vector<Backend> bs(static_cast<size_t>(n));
        for (int32_t i = 0; i < n; ++i) {
            bs[i].fn = fns[i];
            bs[i].ctx = ctxs ? ctxs[i] : nullptr;
        }
        auto r = std::make_unique<sfg_router>();
        r->r = std::make_unique<Router>(std::move(bs), session_expiry_s);
        *out = r.release();
    })
}
void sfg_router_destroy(sfg_router* r) { delete r; }
int32_t sfg_router_handle(sfg_router* r, const uint8_t* req, size_t n, const uint8_t** resp, size_t* resp_len) {
    SFG_GUARD({
        r->r->handle(req, n, g_resp);
        *resp = g_resp.data();
        *resp_len = g_resp.size();
    })
}
int32_t sfg_router_session_device(sfg_router* r, const char* session_id) { return r->r->device_of(session_id); }
int32_t sfg_router_load(sfg_router* r, int32_t* sessions) {
    const std::vector<int> l = r->r->load();
    for (size_t i = 0; i < l.size(); ++i) sessions[i] = l[i];
    return static_cast<int32_t>(l.size());
}
void sfg_router_set_clock(sfg_router* r, double (*now_s)(void*), void* ctx) {
    r->clock = now_s;
    r->clock_ctx = ctx;
    r->r->set_clock([r] { return r->clock(r->clock_ctx); });
}
int32_t sfg_batcher_create(sfg_router* r, int32_t max_frames, sfg_batcher** out) {
    SFG_GUARD({
        auto b = std::make_unique<sfg_batcher>();
        b->b = std::make_unique<Batcher>(*r->r, max_frames);
        *out = b.release();
    })
}
void sfg_batcher_destroy(sfg_batcher* b) { delete b; }
int32_t sfg_batcher_handle(sfg_batcher* b, const uint8_t* req, size_t n, const uint8_t** resp, size_t* resp_len) {
    SFG_GUARD({
        b->b->handle(req, n, g_resp);
        *resp = g_resp.data();
        *resp_len = g_resp.size();
    })
}
void sfg_batcher_stats(sfg_batcher* b, uint64_t* batches, uint64_t* frames, uint64_t* max_batch) {
    if (batches) *batches = b->b->batches();
    if (frames) *frames = b->b->frames();
    if (max_batch) *max_batch = b->b->max_batch();
}

void sfg_server_set_clock(sfg_server* s, double (*now_s)(void*), void* ctx) {
    s->clock = now_s;
    s->clock_ctx = ctx;
    s->s->set_clock([s] { return s->clock(s->clock_ctx); });
}

static ClientCfg to_client_cfg(const sfg_client_config* cfg) {
    ClientCfg cc;
    cc.prefix_layers = cfg->prefix_layers;
    cc.suffix_layers = cfg->suffix_layers;
    cc.wire_dtype = cfg->wire_dtype;
    cc.one_way_delay_ms = cfg->one_way_delay_ms;
    return cc;
}

int32_t sfg_client_create(sfg_engine* local, const sfg_client_config* cfg, sfg_frame_handler handler, void* ctx,
                          const char* sid, sfg_client** out) {
    SFG_GUARD({
        auto* c = new sfg_client;
        try {
            c->c = std::make_unique<Client>(*local->e, to_client_cfg(cfg), handler, ctx, nullptr, sid ? sid : "");
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    })
}
int32_t sfg_client_create_linked(sfg_engine* local, const sfg_client_config* cfg, sfg_server* server,
                                 const char* sid, sfg_client** out) {
    SFG_GUARD({
        auto* c = new sfg_client;
        try {
            c->c = std::make_unique<Client>(*local->e, to_client_cfg(cfg), nullptr, nullptr, server->s.get(),
                                            sid ? sid : "");
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    })
}
void sfg_client_destroy(sfg_client* c) { delete c; }

int32_t sfg_client_prefill(sfg_client* c, const int32_t* prompt, int32_t n, int32_t* first, float* logits) {
    SFG_GUARD({
        const int t = c->c->prefill(prompt, n, logits);
        if (first) *first = t;
    })
}

int32_t sfg_client_decode_step(sfg_client* c, int32_t seq, const int32_t* tokens, const int32_t* positions,
                               const float* mask, const int32_t* keep, int32_t n_keep, int32_t crop, float* logits,
                               int32_t* argmax) {
    SFG_GUARD({
        std::optional<int> cr;
        if (crop >= 0) cr = crop;
        MaskRuns mr;
        const MaskRuns* mp = nullptr;
        if (mask) {
            // the kv extent the mask must cover is known only after keep/crop
            // are applied on the local banks; mirror that computation here.
            Bank& pb = c->c->prefix();
            int len = pb.len(), committed = pb.committed_len();
            if (n_keep > 0 || len - committed > 0) len = committed + n_keep;
            if (cr) len = *cr;
            mr = runs_from_dense(mask, seq, len + seq);
            mp = &mr;
        }
        c->c->decode_step(seq, tokens, positions, mp, keep, n_keep, cr, logits, argmax, nullptr, nullptr);
    })
}

static Decoder::Cfg to_decoder_cfg(const sfg_decode_config* cfg) {
    Decoder::Cfg dc;
    dc.mode = cfg->mode;
    dc.window_w = cfg->window_w;
    dc.ngram_n = cfg->ngram_n;
    dc.max_candidates_g = cfg->max_candidates_g;
    dc.pool_capacity = static_cast<size_t>(cfg->pool_capacity);
    return dc;
}

int32_t sfg_decode(sfg_client* c, const sfg_decode_config* cfg, sfg_pool* pool, const int32_t* prompt, int32_t n,
                   int32_t max_new, int32_t* out_tokens, float* committed_logits, int32_t* step_batch,
                   int32_t* step_accepted, sfg_decode_stats* stats) {
    SFG_GUARD({
        Decoder d(*c->c, to_decoder_cfg(cfg), pool ? pool->p.get() : nullptr, prompt, n, max_new,
                  committed_logits != nullptr);
        while (!d.done()) d.step();
        std::memcpy(out_tokens, d.tokens.data(), sizeof(int32_t) * d.tokens.size());
        if (committed_logits) std::memcpy(committed_logits, d.logits.data(), sizeof(float) * d.logits.size());
        if (step_batch) std::memcpy(step_batch, d.step_batch.data(), sizeof(int32_t) * d.step_batch.size());
        if (step_accepted) std::memcpy(step_accepted, d.step_accepted.data(), sizeof(int32_t) * d.step_accepted.size());
        if (stats) {
            stats->steps = d.steps;
            stats->tokens_committed = d.committed;
            stats->wall_seconds = d.wall_s;
            stats->match_rate = d.steps > 0 ? static_cast<double>(d.hits) / d.steps : 0.0;
            stats->clamped = c->c->clamped();
        }
    })
}

struct sfg_decoder { std::unique_ptr<Decoder> d; };

int32_t sfg_decoder_create(sfg_client* c, const sfg_decode_config* cfg, sfg_pool* pool, const int32_t* prompt,
                           int32_t n, int32_t max_new, sfg_decoder** out) {
    SFG_GUARD({
        auto* h = new sfg_decoder;
        try {
            h->d = std::make_unique<Decoder>(*c->c, to_decoder_cfg(cfg), pool ? pool->p.get() : nullptr, prompt, n,
                                             max_new, false);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    })
}

int32_t sfg_decoder_step(sfg_decoder* d, int32_t* committed, int32_t* n_committed, int32_t* batch) {
    SFG_GUARD({
        if (d->d->done()) throw Error(Kind::input, "decoder finished");
        const size_t before = d->d->tokens.size();
        const int k = d->d->step();
        if (committed) std::memcpy(committed, d->d->tokens.data() + before, sizeof(int32_t) * k);
        if (n_committed) *n_committed = k;
        if (batch) *batch = d->d->step_batch.back();
    })
}

int32_t sfg_decoder_done(const sfg_decoder* d) { return d->d->done() ? 1 : 0; }
void sfg_decoder_destroy(sfg_decoder* d) { delete d; }

int32_t sfg_client_last_profile(sfg_client* c, sfg_step_profile* out) {
    const StepProfile& p = c->c->last_profile();
    out->step_ms = p.step_ms;
    out->server_ms = p.server_ms;
    out->local_ms = p.local_ms;
    out->launches = p.launches;
    out->batch = p.batch;
    return SFG_OK;
}

void sfg_set_graphs(int32_t enabled) { graphs_enabled() = enabled != 0; }

void sfg_copy_bytes(uint64_t* h2d, uint64_t* d2h) {
    if (h2d) *h2d = copy_counters().h2d.load();
    if (d2h) *d2h = copy_counters().d2h.load();
}

void sfg_debug_set_mega(int32_t on) { mega_mode() = on ? 1 : 0; }
void sfg_debug_mega_trace(int32_t on) { mega_trace_enabled() = on != 0; }
int32_t sfg_debug_mega_trace_read(sfg_bank* b, uint64_t* out, size_t n) {
    return mega_trace_read(*b->b, reinterpret_cast<unsigned long long*>(out), n);
}

int32_t sfg_debug_mask_runs(const uint16_t* mask, int32_t q, int32_t kv, int32_t* row_off, int32_t* starts,
                            int32_t* ends, int32_t max_runs, int32_t* n_runs, int32_t* any_empty_row) {
    SFG_GUARD({
        const MaskRuns r = runs_from_f16_mask(mask, q, kv);
        if (static_cast<int>(r.runs.size()) > max_runs) throw Error(Kind::capacity, "run buffer too small");
        for (int i = 0; i <= q; ++i) row_off[i] = r.row_off[i];
        for (size_t i = 0; i < r.runs.size(); ++i) {
            starts[i] = r.runs[i].start;
            ends[i] = r.runs[i].end;
        }
        *n_runs = static_cast<int32_t>(r.runs.size());
        *any_empty_row = r.any_empty_row ? 1 : 0;
    });
}

int32_t sfg_debug_bank_buffer(sfg_bank* b, int32_t which, float* out, int32_t n) {
    SFG_GUARD({
        Workspace& ws = b->b->ws();
        const int tilesH = (b->eng->e->cfg().hidden_dim + 127) / 128;
        const float* src = which == 0 ? ws.h : which == 1 ? ws.q : which == 2 ? ws.att : which == 3 ? ws.act
                                                                                    : mega_ss(*b->b, which - 4, tilesH);
        if (!src) throw Error(Kind::input, "buffer not allocated");
        SFG_CUDA(cudaDeviceSynchronize());
        SFG_CUDA(cudaMemcpy(out, src, sizeof(float) * n, cudaMemcpyDeviceToHost));
    })
}

void sfg_profiler_enable(int32_t on) { KernelProfiler::get().enable(on != 0); }
void sfg_profiler_reset(void) { KernelProfiler::get().reset(); }
int32_t sfg_profiler_stats(int32_t cls, int64_t* count, double* ms, double* bytes, double* flops) {
    SFG_GUARD({
        cudaDeviceSynchronize();
        KernelProfiler::get().stats(cls, count, ms, bytes, flops);
    })
}

int32_t sfg_pool_create(int32_t n, size_t cap, sfg_pool** out) {
    SFG_GUARD({
        auto* p = new sfg_pool;
        try {
            p->p = std::make_unique<Pool>(n, cap);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    })
}
void sfg_pool_destroy(sfg_pool* p) { delete p; }
int32_t sfg_pool_update(sfg_pool* p, const int32_t* prev, const int32_t* cur, int32_t w) {
    SFG_GUARD(p->p->update(prev, cur, w))
}
int32_t sfg_pool_lookup(sfg_pool* p, int32_t key, int32_t max_c, int32_t* out) {
    std::vector<std::vector<int32_t>> hits;
    const int n = p->p->lookup(key, max_c, hits);
    int off = 0;
    for (auto& h : hits)
        for (int32_t t : h) out[off++] = t;
    return n;
}
size_t sfg_pool_size(const sfg_pool* p) { return p->p->size(); }

// Self-test hook: runs the device wire round trip (f32 -> binary16 -> f32)
// on n host values; used by the GPU tests to pin the device codec.
int32_t sfg_selftest_wire_roundtrip(const float* in, float* out, int32_t n, uint64_t* clamped) {
    SFG_GUARD({
        float* d = nullptr;
        unsigned long long* c = nullptr;
        SFG_CUDA(cudaMalloc(&d, sizeof(float) * (n > 0 ? n : 1)));
        SFG_CUDA(cudaMalloc(&c, sizeof(unsigned long long)));
        SFG_CUDA(cudaMemset(c, 0, sizeof(unsigned long long)));
        SFG_CUDA(cudaMemcpy(d, in, sizeof(float) * n, cudaMemcpyHostToDevice));
        launch_wire_roundtrip(d, 0, n, c, 0);
        SFG_CUDA(cudaGetLastError());
        SFG_CUDA(cudaMemcpy(out, d, sizeof(float) * n, cudaMemcpyDeviceToHost));
        unsigned long long hc = 0;
        SFG_CUDA(cudaMemcpy(&hc, c, sizeof(hc), cudaMemcpyDeviceToHost));
        if (clamped) *clamped = hc;
        cudaFree(d);
        cudaFree(c);
    })
}

uint16_t sfg_f32_to_f16(float v, uint64_t* clamped) { return wire::f32_to_f16_bits(v, clamped); }
float sfg_f16_to_f32(uint16_t b) { return wire::f16_bits_to_f32(b); }

}  // extern "C"
