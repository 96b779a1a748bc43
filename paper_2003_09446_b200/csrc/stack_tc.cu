// stack_tc.cu -- K2-TC: tcgen05 3xTF32 fused layer stack (in progress).
#include "engine.hpp"

namespace detnet {

int tc_prepare() { return 0; }

int tc_pack(TcModel &tc, int K, int Z, int V, int L, const double *, const double *) {
    tc.ready = false;
    tc.K = K; tc.Z = Z; tc.V = V; tc.L = L;
    return 0;
}

int tc_launch(const TcModel &, const TcArgs &, cudaStream_t) {
    return fail(DETNET_ERR_UNSUPPORTED, "tcgen05 path not available");
}

void tc_release(TcModel &tc) { tc.w.release(); tc.ready = false; }

} // namespace detnet
