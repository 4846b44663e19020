// Mode-independent device kernels: wire codec (pack/unpack), embedding
// gather, in-place KV-cache commit/rollback, argmax, weight conversion.
// Integer / bit work only (no floating-point rounding decisions except the
// bit-exact binary16 codec), so these are exact in every mode.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "sfg_engine.h"
#include "sfg_kernels.h"

namespace sfg {

namespace {
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, size_t>& attr_sizes() {
    static std::map<std::pair<int, const void*>, size_t> m;
    return m;
}
}  // namespace

void ensure_smem_attr(const void* fn, size_t smem) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(g_attr_mu);
    size_t& have = attr_sizes()[{dev, fn}];
    if (smem <= have) return;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) cuda_fail(e, "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)", __FILE__, __LINE__);
    have = smem;
}

int device_sm_count() {
    static int nsm[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!nsm[dev]) cudaDeviceGetAttribute(&nsm[dev], cudaDevAttrMultiProcessorCount, dev);
    return nsm[dev];
}

namespace {

// binary16 encode, bit-exact port of wire.cpp:83-135 (RNE, finite overflow
// clamps to +-65504 and counts, +-inf passes, NaN -> 0x7e00|sign).
__device__ __forceinline__ uint16_t f32_to_f16_bits(float v, unsigned* clamped) {
    const uint32_t bits = __float_as_uint(v);
    const uint16_t sign = (uint16_t)((bits >> 16) & 0x8000u);
    const uint32_t a = bits & 0x7fffffffu;
    if (a > 0x7f800000u) return sign | 0x7e00u;
    if (a == 0x7f800000u) return sign | 0x7c00u;
    if (__uint_as_float(a) > 65504.0f) {
        ++*clamped;
        return sign | 0x7bffu;
    }
    const int e = (int)((a >> 23) & 0xffu) - 127;
    uint32_t mant = a & 0x7fffffu;
    if (e < -25) return sign;
    if (e == -25) return mant == 0 ? sign : (uint16_t)(sign | 1u);
    if (e < -14) {
        mant |= 0x800000u;
        const int sh = -e - 1;
        const uint32_t hv = mant >> sh, rem = mant & ((1u << sh) - 1u), half = 1u << (sh - 1);
        return (uint16_t)(sign | (hv + ((rem > half || (rem == half && (hv & 1u))) ? 1u : 0u)));
    }
    uint32_t he = (uint32_t)(e + 15), hm = mant >> 13;
    const uint32_t rem = mant & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (hm & 1u))) {
        if (++hm == 0x400u) {
            hm = 0;
            ++he;
        }
    }
    if (he >= 31) {
        ++*clamped;
        return sign | 0x7bffu;
    }
    return (uint16_t)(sign | (he << 10) | hm);
}

// binary16 decode, wire.cpp:137-160 (exact; subnormals normalised).
__device__ __forceinline__ float f16_bits_to_f32(uint16_t b) {
    const uint32_t sign = (uint32_t)(b & 0x8000u) << 16, e = (b >> 10) & 0x1fu, mant = b & 0x3ffu;
    uint32_t o;
    if (e == 0) {
        if (mant == 0) {
            o = sign;
        } else {
            const int lz = __clz(mant) - 21;  // shifts until bit 10 is set
            o = sign | ((uint32_t)(113 - lz) << 23) | (((mant << lz) & 0x3ffu) << 13);
        }
    } else if (e == 31) {
        o = sign | 0x7f800000u | (mant << 13);
    } else {
        o = sign | ((e + 112) << 23) | (mant << 13);
    }
    return __uint_as_float(o);
}

__global__ void unpack_kernel(const void* __restrict__ wire, int f32, int n, float* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = f32 ? reinterpret_cast<const float*>(wire)[i]
                     : f16_bits_to_f32(reinterpret_cast<const uint16_t*>(wire)[i]);
}

__global__ void pack_kernel(const float* __restrict__ in, int f32, int n, void* __restrict__ wire,
                            unsigned long long* clamped) {
    unsigned c = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (f32)
            reinterpret_cast<float*>(wire)[i] = in[i];
        else
            reinterpret_cast<uint16_t*>(wire)[i] = f32_to_f16_bits(in[i], &c);
    }
    if (c && clamped) atomicAdd(clamped, (unsigned long long)c);
}

// f32 -> wire dtype -> f32 in place: the device-linked path's stand-in for
// encode_values + decode_values (same values the frame would carry).
__global__ void roundtrip_kernel(float* __restrict__ x, int f32, int n, unsigned long long* clamped) {
    unsigned c = 0;
    if (!f32)
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
            x[i] = f16_bits_to_f32(f32_to_f16_bits(x[i], &c));
    if (c && clamped) atomicAdd(clamped, (unsigned long long)c);
}

// Simulated one-way link delay on the device timeline (SimChannel's sleep,
// transport.cpp:235-243): one thread spins on %globaltimer, so the delay
// sits between the producing and consuming kernels of a captured graph.
__global__ void link_delay_kernel(unsigned long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        __nanosleep(2000);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
}

// embed_at (tinyformer.cpp:348-373): row gather, bf16/f32 -> f32 exact.
__global__ void embed_kernel(const void* __restrict__ table, int wt, const int32_t* __restrict__ ids,
                             int H, float* __restrict__ out) {
    const size_t src = (size_t)ids[blockIdx.x] * H;
    float* o = out + (size_t)blockIdx.x * H;
    for (int i = threadIdx.x; i < H; i += blockDim.x)
        o[i] = wt == W_BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(table)[src + i])
                            : reinterpret_cast<const float*>(table)[src + i];
}

// CacheBank::resolve compaction (tinyformer.cpp:291-306), in place on device.
// One CTA per (layer, kv head, K|V) slab.  Kept row i moves from committed +
// keep[i] to committed + i.  Within a chunk of rows all sources are gathered
// into shared memory before any destination is written (a kept row's
// destination may be another kept row's source: keep=[1,2]).  Chunks run in
// ascending order, which is safe because keep is strictly increasing:
// keep[j] >= j, so every later source committed + keep[j] (j > i) lies above
// the destination committed + i — the reference's serial loop relies on the
// same order.  Any keep length works with kCompactChunk rows of smem.
constexpr int kCompactChunk = 64;

__device__ __forceinline__ void compact_slab(float* __restrict__ base, int hd, int committed,
                                             const int32_t* __restrict__ keep, int n_keep, float* buf) {
    for (int c0 = 0; c0 < n_keep; c0 += kCompactChunk) {
        const int cn = min(kCompactChunk, n_keep - c0);
        for (int t = threadIdx.x; t < cn * hd; t += blockDim.x) {
            const int i = t / hd, dd = t - i * hd;
            buf[t] = base[(size_t)(committed + keep[c0 + i]) * hd + dd];
        }
        __syncthreads();
        for (int t = threadIdx.x; t < cn * hd; t += blockDim.x) {
            const int i = t / hd, dd = t - i * hd;
            base[(size_t)(committed + c0 + i) * hd + dd] = buf[t];
        }
        __syncthreads();
    }
}

__global__ void kv_compact_kernel(float* __restrict__ kc, float* __restrict__ vc, int n_kv,
                                  int max_len, int hd, int committed, const int32_t* __restrict__ keep,
                                  int n_keep) {
    extern __shared__ float buf[];  // [min(n_keep, kCompactChunk)][hd]
    const int slab = blockIdx.x;     // (layer * n_kv + head) * 2 + {0:K,1:V}
    float* base = ((slab & 1) ? vc : kc) + (size_t)(slab >> 1) * max_len * hd;
    compact_slab(base, hd, committed, keep, n_keep, buf);
}

// Same compaction, parameters from the step meta block (meta[1] committed,
// meta[2] n_keep, meta[3..] keep) so a captured graph replays it every step.
__global__ void kv_compact_meta_kernel(float* __restrict__ kc, float* __restrict__ vc, int max_len, int hd,
                                       const int32_t* __restrict__ meta) {
    extern __shared__ float buf[];
    const int committed = meta[1], n_keep = meta[2];
    if (n_keep <= 0) return;
    const int slab = blockIdx.x;
    float* base = ((slab & 1) ? vc : kc) + (size_t)(slab >> 1) * max_len * hd;
    compact_slab(base, hd, committed, meta + 3, n_keep, buf);
}

// argmax_row (tinyformer.cpp:329-340): first maximum wins == (max value,
// smallest index).  One CTA per row, fixed-shape tree; exact.
__device__ __forceinline__ void better(float& v, int& i, float v2, int i2) {
    if (v2 > v || (v2 == v && i2 < i)) {
        v = v2;
        i = i2;
    }
}

__global__ void argmax_kernel(const float* __restrict__ logits, int V, int32_t* __restrict__ out) {
    const float* r = logits + (size_t)blockIdx.x * V;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < V; i += blockDim.x) better(bv, bi, r[i], i);
    for (int o = 16; o > 0; o >>= 1) {
        const float v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        better(bv, bi, v2, i2);
    }
    __shared__ float sv[32];
    __shared__ int si[32];
    if ((threadIdx.x & 31) == 0) {
        sv[threadIdx.x >> 5] = bv;
        si[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) better(bv, bi, sv[w], si[w]);
        out[blockIdx.x] = bi == 0x7fffffff ? 0 : bi;
    }
}

// fp32 parameters -> device storage dtype (bf16 RNE or f32 copy).
__global__ void convert_kernel(const float* __restrict__ src, void* __restrict__ dst, int wt, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        if (wt == W_BF16)
            reinterpret_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(src[i]);
        else
            reinterpret_cast<float*>(dst)[i] = src[i];
    }
}

inline int blocks_for(size_t n, int t) {
    size_t b = (n + t - 1) / t;
    return (int)(b > 4096 ? 4096 : (b == 0 ? 1 : b));
}

}  // namespace

int launch_unpack_rows(const void* wire, int f32, int n, float* out, cudaStream_t s) {
    unpack_kernel<<<blocks_for(n, 256), 256, 0, s>>>(wire, f32, n, out);
    return 1;
}

int launch_pack_rows(const float* in, int f32, int n, void* wire, unsigned long long* clamped,
                     cudaStream_t s) {
    pack_kernel<<<blocks_for(n, 256), 256, 0, s>>>(in, f32, n, wire, clamped);
    return 1;
}

int launch_wire_roundtrip(float* x, int f32, int n, unsigned long long* clamped, cudaStream_t s) {
    if (f32) return 0;
    roundtrip_kernel<<<blocks_for(n, 256), 256, 0, s>>>(x, f32, n, clamped);
    return 1;
}

int launch_link_delay(double ms, cudaStream_t s) {
    if (ms <= 0.0) return 0;
    link_delay_kernel<<<1, 1, 0, s>>>(static_cast<unsigned long long>(ms * 1e6));
    return 1;
}

int launch_embed(const void* table, int wt, const int32_t* ids, int rows, int H, float* out,
                 cudaStream_t s) {
    embed_kernel<<<rows, 256, 0, s>>>(table, wt, ids, H, out);
    return 1;
}

int launch_kv_compact(float* kcache, float* vcache, int layers, int n_kv, int max_len, int hd,
                      int committed, const int32_t* keep, int n_keep, cudaStream_t s) {
    if (n_keep <= 0 || layers <= 0) return 0;
    const size_t smem = sizeof(float) * (size_t)std::min(n_keep, kCompactChunk) * hd;
    ensure_smem_attr(reinterpret_cast<const void*>(kv_compact_kernel), smem);
    kv_compact_kernel<<<layers * n_kv * 2, 256, smem, s>>>(
        kcache, vcache, n_kv, max_len, hd, committed, keep, n_keep);
    return 1;
}

int launch_kv_compact_meta(float* kcache, float* vcache, int layers, int n_kv, int max_len, int hd,
                           const int32_t* meta, int max_keep, cudaStream_t s) {
    if (layers <= 0) return 0;
    const size_t smem = sizeof(float) * (size_t)std::min(max_keep, kCompactChunk) * hd;
    ensure_smem_attr(reinterpret_cast<const void*>(kv_compact_meta_kernel), smem);
    kv_compact_meta_kernel<<<layers * n_kv * 2, 256, smem, s>>>(kcache, vcache, max_len, hd, meta);
    return 1;
}

int launch_argmax(const float* logits, int rows, int V, int32_t* out, cudaStream_t s) {
    argmax_kernel<<<rows, 1024, 0, s>>>(logits, V, out);
    return 1;
}

int launch_convert_weights(const float* src, void* dst, int wt, size_t n, cudaStream_t s) {
    convert_kernel<<<blocks_for(n, 256), 256, 0, s>>>(src, dst, wt, n);
    return 1;
}

}  // namespace sfg

namespace sfg {
namespace {

// verify_greedy (decoding.cpp:99-109) on device-resident argmaxes.
__device__ int verify_ids(const int32_t* amax, int row_begin, const int32_t* g, int n, int anchor,
                          int32_t* committed) {
    int k = 0;
    committed[0] = anchor;
    while (k < n && g[k] == committed[k]) {
        committed[k + 1] = amax[row_begin + k];
        ++k;
    }
    return k;
}

// Branch selection of decode_lookahead_with_pool (decoding.cpp:296-309):
// window first, candidates in recency order, strict '>' so ties keep the
// earlier branch.  Single thread: B <= a few dozen rows.
__global__ void verify_kernel(const int32_t* __restrict__ amax, const VerifyIn* __restrict__ in,
                              VerifyOut* __restrict__ out) {
    if (threadIdx.x != 0) return;
    const int B = in->rows;
    for (int i = 0; i < B && i < kMaxWindow + 1 + kMaxCand * kMaxCont; ++i) out->argmax[i] = amax[i];
    const int anchor = amax[0];
    out->anchor = anchor;
    if (in->mode != 2) {
        out->best = 0;
        out->committed[0] = anchor;
        return;
    }
    int32_t best_c[kMaxWindow + 1];
    int best = verify_ids(amax, 1, in->window, in->active_w, anchor, best_c);
    for (int i = 1; i <= best; ++i) out->best_rows[i - 1] = i;
    for (int b = 0; b < in->ncand; ++b) {
        int32_t vc[kMaxCont + 1];
        const int acc = verify_ids(amax, in->cand_begin[b], in->cands + b * in->cont, in->cont, anchor, vc);
        if (acc > best) {
            best = acc;
            for (int j = 0; j <= acc; ++j) best_c[j] = vc[j];
            for (int j = 0; j < acc; ++j) out->best_rows[j] = in->cand_begin[b] + j;
        }
    }
    out->best = best;
    for (int j = 0; j <= best; ++j) out->committed[j] = best_c[j];
}

}  // namespace

int launch_verify(const int32_t* argmax, const VerifyIn* in, VerifyOut* out, cudaStream_t s) {
    verify_kernel<<<1, 32, 0, s>>>(argmax, in, out);
    return 1;
}

}  // namespace sfg
