// scan_ws_kernel instantiations for the e4m4 LUT (see scan_ws.cuh).
#include "ws_launch.cuh"

namespace ivfpq {
cudaError_t ws_launch_e4m4(int layout, int logn, int sub_d, const WsArgs& w, size_t smem, int grid,
                           cudaStream_t st) {
    return ws_launch_dt<LUT_E4M4>(layout, logn, sub_d, w, smem, grid, st);
}
}  // namespace ivfpq
