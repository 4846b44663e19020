// Frame codec of the splitf wire protocol (PROTOCOL.md), host side.
// Byte-identical to the reference encoder/decoder (wire.cpp:189-302): the
// JSON header is serialised with sorted keys by nlohmann::json, payloads are
// raw little-endian binary16/binary32.  Only framing lives here; value
// packing/unpacking of hidden rows runs on the device (sfg_common.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <optional>
#include <string>
#include <vector>

namespace sfg::wire {

enum class FrameKind { prompt, step, accept_and_step, response, error, ping };
enum class Dtype { f16 = 0, f32 = 1 };

const char* to_string(FrameKind k);
inline size_t width(Dtype d) { return d == Dtype::f16 ? 2 : 4; }

struct Header {
    FrameKind kind = FrameKind::ping;
    std::string session_id;
    std::vector<int64_t> shape;
    Dtype dtype = Dtype::f16;
    std::vector<int64_t> pos;
    std::optional<int64_t> crop;
    std::optional<std::vector<int64_t>> keep;
    std::optional<std::vector<int64_t>> mask_shape;
    std::optional<std::string> err;
    std::optional<double> srv_ms;
};

// A decoded frame that borrows its payloads from the request buffer.
struct FrameView {
    Header h;
    const uint8_t* tensor = nullptr;
    size_t tensor_len = 0;
    const uint8_t* mask = nullptr;
    size_t mask_len = 0;
};

// decode_frame (wire.cpp:233-302); throws sfg::Error(protocol) on malformed input.
FrameView decode(const uint8_t* bytes, size_t n);
// encode_frame (wire.cpp:189-231) into `out` (cleared first).
void encode(const Header& h, const uint8_t* tensor, size_t tensor_len, const uint8_t* mask,
            size_t mask_len, std::vector<uint8_t>& out);

uint16_t f32_to_f16_bits(float v, uint64_t* clamped);  // wire.cpp:83-135
float f16_bits_to_f32(uint16_t b);                     // wire.cpp:137-160

}  // namespace sfg::wire
