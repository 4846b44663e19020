// Frame codec (PROTOCOL.md); see sfg_wire.h.
#include "sfg_wire.h"

#include <cstring>
#include <nlohmann/json.hpp>

#include "sfg_engine.h"

namespace sfg::wire {

using nlohmann::json;

[[noreturn]] static void bad(const std::string& m) { throw Error(Kind::protocol, m); }

const char* to_string(FrameKind k) {
    switch (k) {
        case FrameKind::prompt: return "prompt";
        case FrameKind::step: return "step";
        case FrameKind::accept_and_step: return "accept_and_step";
        case FrameKind::response: return "response";
        case FrameKind::error: return "error";
        case FrameKind::ping: return "ping";
    }
    return "unknown";
}

static FrameKind kind_of(const std::string& s) {
    static const std::pair<const char*, FrameKind> names[] = {
        {"prompt", FrameKind::prompt}, {"step", FrameKind::step},
        {"accept_and_step", FrameKind::accept_and_step}, {"response", FrameKind::response},
        {"error", FrameKind::error}, {"ping", FrameKind::ping}};
    for (auto& [n, k] : names)
        if (s == n) return k;
    bad("unknown frame kind: " + s);
}

static Dtype dtype_of(const std::string& s) {
    if (s == "f16") return Dtype::f16;
    if (s == "f32") return Dtype::f32;
    bad("unknown dtype: " + s);
}

static int64_t elements(const std::vector<int64_t>& shape) {
    int64_t n = 1;
    for (int64_t d : shape) {
        if (d < 0) bad("negative dimension in shape");
        n *= d;
    }
    return n;
}

static std::vector<int64_t> int_array(const json& j, const char* field) {
    const json& v = j.at(field);
    if (!v.is_array()) bad(std::string("header field '") + field + "' must be an array");
    std::vector<int64_t> out;
    out.reserve(v.size());
    for (const json& e : v) {
        if (!e.is_number_integer()) bad(std::string("header field '") + field + "' must hold integers");
        out.push_back(e.get<int64_t>());
    }
    return out;
}

FrameView decode(const uint8_t* b, size_t n) {
    if (n < 4) bad("frame shorter than length prefix");
    const uint32_t hlen = uint32_t(b[0]) | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) | (uint32_t(b[3]) << 24);
    if (hlen > n - 4) bad("header length prefix exceeds available bytes");
    json j;
    try {
        j = json::parse(reinterpret_cast<const char*>(b) + 4, reinterpret_cast<const char*>(b) + 4 + hlen);
    } catch (const json::exception& e) {
        bad(std::string("invalid JSON header: ") + e.what());
    }
    if (!j.is_object()) bad("JSON header must be an object");
    FrameView f;
    Header& h = f.h;
    try {
        h.kind = kind_of(j.at("kind").get<std::string>());
        h.session_id = j.value("session_id", std::string{});
        h.shape = int_array(j, "shape");
        h.dtype = dtype_of(j.at("dtype").get<std::string>());
        if (j.contains("pos")) h.pos = int_array(j, "pos");
        if (j.contains("crop")) {
            if (!j["crop"].is_number_integer()) bad("'crop' must be an integer");
            h.crop = j["crop"].get<int64_t>();
        }
        if (j.contains("keep")) h.keep = int_array(j, "keep");
        if (j.contains("mask_shape")) h.mask_shape = int_array(j, "mask_shape");
        if (j.contains("err")) {
            if (!j["err"].is_string()) bad("'err' must be a string");
            h.err = j["err"].get<std::string>();
        }
        if (j.contains("srv_ms")) {
            if (!j["srv_ms"].is_number()) bad("'srv_ms' must be a number");
            h.srv_ms = j["srv_ms"].get<double>();
        }
    } catch (const json::exception& e) {
        bad(std::string("malformed header field: ") + e.what());
    }
    constexpr int64_t kMax = int64_t{1} << 30;
    const int64_t te = elements(h.shape);
    if (te > kMax) bad("declared tensor too large");
    f.tensor_len = static_cast<size_t>(te) * width(h.dtype);
    if (h.mask_shape) {
        const int64_t me = elements(*h.mask_shape);
        if (me > kMax) bad("declared mask too large");
        f.mask_len = static_cast<size_t>(me) * 2;
    }
    const size_t off = 4 + hlen, total = off + f.tensor_len + f.mask_len;
    if (n < total) bad("payload truncated");
    if (n > total) bad("trailing bytes after declared payload");
    f.tensor = b + off;
    f.mask = b + off + f.tensor_len;
    return f;
}

void encode(const Header& h, const uint8_t* tensor, size_t tensor_len, const uint8_t* mask,
            size_t mask_len, std::vector<uint8_t>& out) {
    if (tensor_len != static_cast<size_t>(elements(h.shape)) * width(h.dtype))
        bad("tensor payload does not match declared shape");
    if (h.mask_shape) {
        if (mask_len != static_cast<size_t>(elements(*h.mask_shape)) * 2)
            bad("mask payload does not match declared mask_shape");
    } else if (mask_len != 0) {
        bad("mask bytes present without mask_shape");
    }
    json j;
    j["kind"] = to_string(h.kind);
    j["session_id"] = h.session_id;
    j["shape"] = h.shape;
    j["dtype"] = h.dtype == Dtype::f16 ? "f16" : "f32";
    if (!h.pos.empty()) j["pos"] = h.pos;
    if (h.crop) j["crop"] = *h.crop;
    if (h.keep) j["keep"] = *h.keep;
    if (h.mask_shape) j["mask_shape"] = *h.mask_shape;
    if (h.err) j["err"] = *h.err;
    if (h.srv_ms) j["srv_ms"] = *h.srv_ms;
    const std::string hdr = j.dump();
    const uint32_t hl = static_cast<uint32_t>(hdr.size());
    out.resize(4 + hdr.size() + tensor_len + mask_len);
    out[0] = hl & 0xff;
    out[1] = (hl >> 8) & 0xff;
    out[2] = (hl >> 16) & 0xff;
    out[3] = (hl >> 24) & 0xff;
    std::memcpy(out.data() + 4, hdr.data(), hdr.size());
    if (tensor_len) std::memcpy(out.data() + 4 + hdr.size(), tensor, tensor_len);
    if (mask_len) std::memcpy(out.data() + 4 + hdr.size() + tensor_len, mask, mask_len);
}

// Host binary16 codec: the same algorithm the device pack/unpack kernels run
// (sfg_common.cu); used for the mask path and the exported ABI helpers.
uint16_t f32_to_f16_bits(float v, uint64_t* clamped) {
    uint32_t u;
    std::memcpy(&u, &v, 4);
    const uint16_t sign = static_cast<uint16_t>((u >> 16) & 0x8000u);
    const uint32_t a = u & 0x7fffffffu;
    if (a > 0x7f800000u) return sign | 0x7e00u;
    if (a == 0x7f800000u) return sign | 0x7c00u;
    float av;
    std::memcpy(&av, &a, 4);
    if (av > 65504.0f) {
        if (clamped) ++*clamped;
        return sign | 0x7bffu;
    }
    const int e = static_cast<int>((a >> 23) & 0xff) - 127;
    uint32_t mant = a & 0x7fffffu;
    if (e < -25) return sign;
    if (e == -25) return mant == 0 ? sign : static_cast<uint16_t>(sign | 1u);
    if (e < -14) {
        mant |= 0x800000u;
        const int sh = -e - 1;
        const uint32_t hv = mant >> sh, rem = mant & ((1u << sh) - 1u), half = 1u << (sh - 1);
        return static_cast<uint16_t>(sign | (hv + ((rem > half || (rem == half && (hv & 1u))) ? 1u : 0u)));
    }
    uint32_t he = static_cast<uint32_t>(e + 15), hm = mant >> 13;
    const uint32_t rem = mant & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (hm & 1u))) {
        if (++hm == 0x400u) {
            hm = 0;
            ++he;
        }
    }
    if (he >= 31) {
        if (clamped) ++*clamped;
        return sign | 0x7bffu;
    }
    return static_cast<uint16_t>(sign | (he << 10) | hm);
}

float f16_bits_to_f32(uint16_t b) {
    const uint32_t sign = static_cast<uint32_t>(b & 0x8000u) << 16, e = (b >> 10) & 0x1fu, mant = b & 0x3ffu;
    uint32_t o;
    if (e == 0) {
        if (mant == 0) {
            o = sign;
        } else {
            const int lz = __builtin_clz(mant) - 21;
            o = sign | (static_cast<uint32_t>(113 - lz) << 23) | (((mant << lz) & 0x3ffu) << 13);
        }
    } else if (e == 31) {
        o = sign | 0x7f800000u | (mant << 13);
    } else {
        o = sign | ((e + 112) << 23) | (mant << 13);
    }
    float f;
    std::memcpy(&f, &o, 4);
    return f;
}

}  // namespace sfg::wire
