// kernels_f32.cu -- fp32 instantiations of the record-stream kernel (see stream_kernel.cuh).
#include "stream_dispatch.cuh"

namespace arrow {

int launch_stream_f32(const StreamArgs &a, const StreamCfg &c, cudaStream_t st) {
    using namespace ks;
    if (c.lpe == -1) {
        const int r = kr::run_rec<float>(a, st);
        if (r >= 0) return r;
        return (int)cudaErrorInvalidConfiguration;
    }
    if (c.lpe == 0) {
        const int r = kt::run_tma<float>(a, st);
        if (r >= 0) return r;
        return (int)cudaErrorInvalidConfiguration;
    }
#define ARROW_CFG(L, N, B, DD) \
    if (c.lpe == L && c.nv == N && c.vb == B && c.d == DD) return run_cfg<float, L, N, B, DD>(a, st);
    ARROW_CFG(8, 4, 16, 4)
    ARROW_CFG(16, 2, 16, 6)
    ARROW_CFG(8, 4, 16, 6)
    ARROW_CFG(4, 4, 16, 4)
    ARROW_CFG(2, 4, 16, 4)
    ARROW_CFG(1, 4, 16, 4)
    ARROW_CFG(8, 1, 16, 8)
    ARROW_CFG(32, 1, 16, 8)
    ARROW_CFG(32, 1, 16, 16)
    ARROW_CFG(16, 2, 16, 8)
    ARROW_CFG(1, 1, 16, 8)
    ARROW_CFG(32, 1, 8, 8)
    ARROW_CFG(8, 1, 8, 8)
    ARROW_CFG(1, 1, 8, 8)
    ARROW_CFG(32, 1, 4, 8)
    ARROW_CFG(8, 1, 4, 8)
    ARROW_CFG(1, 1, 4, 8)
#undef ARROW_CFG
    return (int)cudaErrorInvalidConfiguration;
}

}  // namespace arrow
