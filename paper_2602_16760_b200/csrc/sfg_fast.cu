// FAST-mode layer executor (tcgen05 weight-streaming GEMMs) — placeholder
// until the tcgen05 path lands; engines created with SFG_MATH_FAST fail loudly.
#include "sfg_engine.h"

namespace sfg {

size_t fast_workspace_bytes(const ModelCfg&, int) { return 16; }

void fast_build_layer(Engine&, LayerWeights&, cudaStream_t) {
    throw Error(Kind::config, "FAST math is not built in this library version");
}

int fast_forward_layer(Engine&, Bank&, int, int, Workspace&, int, cudaStream_t) {
    throw Error(Kind::internal, "FAST math is not built in this library version");
}

}  // namespace sfg
