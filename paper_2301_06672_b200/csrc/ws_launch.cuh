// Launchers for scan_ws_kernel, one translation unit per LUT dtype
// (ws_f32.cu, ws_f16.cu, ws_e5m3.cu, ws_e4m4.cu) so they compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include "scan_ws.cuh"

namespace ivfpq {

template <int DT, int LOGN, int SUB_D, bool GMEM>
cudaError_t ws_launch_g(const WsArgs& w, size_t smem, int grid, cudaStream_t st) {
    static int ok = -1;
    if (ok < 0) {
        cudaError_t e = cudaFuncSetAttribute(scan_ws_kernel<DT, LOGN, SUB_D, GMEM>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        ok = 1;
    }
    if (!ok) return cudaErrorNotSupported;
    scan_ws_kernel<DT, LOGN, SUB_D, GMEM><<<grid, WS_THREADS, smem, st>>>(w);
    return cudaGetLastError();
}

// GMEM: the builders read the codebook from global memory (it does not fit
// TMEM); a separate instantiation keeps the common TMEM kernel's code as is.
template <int DT, int LOGN, int SUB_D>
cudaError_t ws_launch_t(const WsArgs& w, size_t smem, int grid, cudaStream_t st) {
    return w.gmem ? ws_launch_g<DT, LOGN, SUB_D, true>(w, smem, grid, st)
                  : ws_launch_g<DT, LOGN, SUB_D, false>(w, smem, grid, st);
}

template <int DT, int LOGN>
cudaError_t ws_launch_l(int sub_d, const WsArgs& w, size_t smem, int grid, cudaStream_t st) {
    switch (sub_d) {
        case 1: return ws_launch_t<DT, LOGN, 1>(w, smem, grid, st);
        case 2: return ws_launch_t<DT, LOGN, 2>(w, smem, grid, st);
        case 3: return ws_launch_t<DT, LOGN, 3>(w, smem, grid, st);
        case 4: return ws_launch_t<DT, LOGN, 4>(w, smem, grid, st);
    }
    return cudaErrorInvalidValue;
}

template <int DT>
cudaError_t ws_launch_dt(int logn, int sub_d, const WsArgs& w, size_t smem, int grid, cudaStream_t st) {
    switch (logn) {
        case 2: return ws_launch_l<DT, 2>(sub_d, w, smem, grid, st);
        case 3: return ws_launch_l<DT, 3>(sub_d, w, smem, grid, st);
        case 4: return ws_launch_l<DT, 4>(sub_d, w, smem, grid, st);
        case 5: return ws_launch_l<DT, 5>(sub_d, w, smem, grid, st);
        case 6: return ws_launch_l<DT, 6>(sub_d, w, smem, grid, st);
        case 7: return ws_launch_l<DT, 7>(sub_d, w, smem, grid, st);
        case 8: return ws_launch_l<DT, 8>(sub_d, w, smem, grid, st);
    }
    return cudaErrorInvalidValue;
}

// defined in ws_<dtype>.cu
cudaError_t ws_launch_f32(int logn, int sub_d, const WsArgs& w, size_t smem, int grid, cudaStream_t st);
cudaError_t ws_launch_f16(int logn, int sub_d, const WsArgs& w, size_t smem, int grid, cudaStream_t st);
cudaError_t ws_launch_e5m3(int logn, int sub_d, const WsArgs& w, size_t smem, int grid, cudaStream_t st);
cudaError_t ws_launch_e4m4(int logn, int sub_d, const WsArgs& w, size_t smem, int grid, cudaStream_t st);

}  // namespace ivfpq
