// scan_ws_kernel instantiations for the f32 LUT (see scan_ws.cuh).
#include "ws_launch.cuh"

namespace ivfpq {
cudaError_t ws_launch_f32(int layout, int logn, int sub_d, const WsArgs& w, size_t smem, int grid,
                           cudaStream_t st) {
    return ws_launch_dt<LUT_F32>(layout, logn, sub_d, w, smem, grid, st);
}
}  // namespace ivfpq
