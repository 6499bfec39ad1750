// Launchers for scan_ws_kernel, one translation unit per LUT dtype
// (ws_f32.cu, ws_f16.cu, ws_e5m3.cu, ws_e4m4.cu) so they compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

#include "scan_ws.cuh"

namespace ivfpq {

// The dynamic-smem attribute is per device context, so it is set before every
// launch (cheap) instead of once per process.
template <class C, int DT, int LOGN, int SUB_D, bool GMEM, int NCH, bool CH = false, bool SMALLK = true>
cudaError_t ws_launch_k(const WsArgs& w, size_t smem, int grid, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(scan_ws_kernel<C, DT, LOGN, SUB_D, GMEM, NCH, CH, SMALLK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    scan_ws_kernel<C, DT, LOGN, SUB_D, GMEM, NCH, CH, SMALLK><<<grid, C::THREADS, smem, st>>>(w);
    return cudaGetLastError();
}

// Chunk count (s_pad / 16) as a compile-time constant for the BASELINE shapes
// (straight-line chunk loop), a runtime loop for every other shape:
//   cfg1/cfg2 s=64, cfg4 s=48 (p=8, sub_d=2); cfg5 s=32 (sub_d=3);
//   cfg3 s=240 (sub_d=4): p=8 with the codebook in global memory, p=5 in TMEM.
// Layout B (4 builder + 15 scanner warps) is built for the scan-heavy shapes
// only (cfg4, cfg5, cfg3 p5); any other shape reports NotSupported and the
// host falls back to layout A.
template <class C, int DT, int LOGN, int SUB_D, bool GMEM>
cudaError_t ws_launch_g(const WsArgs& w, size_t smem, int grid, cudaStream_t st) {
    const int nch = w.a.s_pad >> 4;
    // k > 32 (cfg4: k = 100): runtime top-k geometry, built for layout A only,
    // the cfg4 shape specialised, every other shape the generic chunk loop
    if (w.a.K > 32) {
        if constexpr (std::is_same_v<C, WsCfgB>) {
            return cudaErrorNotSupported;
        } else {
            if (w.nh > 1) {
                if constexpr (LOGN >= 5) return ws_launch_k<C, DT, LOGN, SUB_D, GMEM, 0, true, false>(w, smem, grid, st);
                return cudaErrorNotSupported;
            }
            if constexpr (LOGN == 8 && SUB_D == 2 && !GMEM)
                if (nch == 3) return ws_launch_k<C, DT, LOGN, SUB_D, GMEM, 3, false, false>(w, smem, grid, st);
            return ws_launch_k<C, DT, LOGN, SUB_D, GMEM, 0, false, false>(w, smem, grid, st);
        }
    }
    if constexpr (std::is_same_v<C, WsCfgB>) {
        if (w.nh == 1) {
            if constexpr (LOGN == 8 && SUB_D == 2 && !GMEM)
                if (nch == 3) return ws_launch_k<C, DT, LOGN, SUB_D, GMEM, 3>(w, smem, grid, st);
            if constexpr (LOGN == 8 && SUB_D == 3 && !GMEM)
                if (nch == 2) return ws_launch_k<C, DT, LOGN, SUB_D, GMEM, 2>(w, smem, grid, st);
            if constexpr (LOGN == 5 && SUB_D == 4 && !GMEM)
                if (nch == 15) return ws_launch_k<C, DT, LOGN, SUB_D, GMEM, 15>(w, smem, grid, st);
        }
        return cudaErrorNotSupported;
    } else {
        // row-chunked LUT jobs (tables beyond the shared-memory budget, only with
        // 2^p >= 32 codes): runtime chunk count per job
        if (w.nh > 1) {
            if constexpr (LOGN >= 5) return ws_launch_k<C, DT, LOGN, SUB_D, GMEM, 0, true>(w, smem, grid, st);
            return cudaErrorNotSupported;
        }
        if constexpr (LOGN == 8 && SUB_D == 2 && !GMEM) {
            if (nch == 4) return ws_launch_k<C, DT, LOGN, SUB_D, GMEM, 4>(w, smem, grid, st);
            if (nch == 3) return ws_launch_k<C, DT, LOGN, SUB_D, GMEM, 3>(w, smem, grid, st);
        }
        if constexpr (LOGN == 8 && SUB_D == 3 && !GMEM) {
            if (nch == 2) return ws_launch_k<C, DT, LOGN, SUB_D, GMEM, 2>(w, smem, grid, st);
        }
        if constexpr (SUB_D == 4 && ((LOGN == 8 && GMEM) || (LOGN == 5 && !GMEM))) {
            if (nch == 15) return ws_launch_k<C, DT, LOGN, SUB_D, GMEM, 15>(w, smem, grid, st);
        }
        return ws_launch_k<C, DT, LOGN, SUB_D, GMEM, 0>(w, smem, grid, st);
    }
}

// GMEM: the builders read the codebook from global memory (it does not fit
// TMEM); a separate instantiation keeps the common TMEM kernel's code as is.
template <class C, int DT, int LOGN, int SUB_D>
cudaError_t ws_launch_t(const WsArgs& w, size_t smem, int grid, cudaStream_t st) {
    return w.gmem ? ws_launch_g<C, DT, LOGN, SUB_D, true>(w, smem, grid, st)
                  : ws_launch_g<C, DT, LOGN, SUB_D, false>(w, smem, grid, st);
}

template <class C, int DT, int LOGN>
cudaError_t ws_launch_l(int sub_d, const WsArgs& w, size_t smem, int grid, cudaStream_t st) {
    switch (sub_d) {
        case 1: return ws_launch_t<C, DT, LOGN, 1>(w, smem, grid, st);
        case 2: return ws_launch_t<C, DT, LOGN, 2>(w, smem, grid, st);
        case 3: return ws_launch_t<C, DT, LOGN, 3>(w, smem, grid, st);
        case 4: return ws_launch_t<C, DT, LOGN, 4>(w, smem, grid, st);
    }
    return cudaErrorInvalidValue;
}

template <class C, int DT>
cudaError_t ws_launch_c(int logn, int sub_d, const WsArgs& w, size_t smem, int grid, cudaStream_t st) {
    switch (logn) {
        case 2: return ws_launch_l<C, DT, 2>(sub_d, w, smem, grid, st);
        case 3: return ws_launch_l<C, DT, 3>(sub_d, w, smem, grid, st);
        case 4: return ws_launch_l<C, DT, 4>(sub_d, w, smem, grid, st);
        case 5: return ws_launch_l<C, DT, 5>(sub_d, w, smem, grid, st);
        case 6: return ws_launch_l<C, DT, 6>(sub_d, w, smem, grid, st);
        case 7: return ws_launch_l<C, DT, 7>(sub_d, w, smem, grid, st);
        case 8: return ws_launch_l<C, DT, 8>(sub_d, w, smem, grid, st);
    }
    return cudaErrorInvalidValue;
}

// layout 0 = WsCfgA, 1 = WsCfgB
template <int DT>
cudaError_t ws_launch_dt(int layout, int logn, int sub_d, const WsArgs& w, size_t smem, int grid, cudaStream_t st) {
    return layout == 1 ? ws_launch_c<WsCfgB, DT>(logn, sub_d, w, smem, grid, st)
                       : ws_launch_c<WsCfgA, DT>(logn, sub_d, w, smem, grid, st);
}

// defined in ws_<dtype>.cu
cudaError_t ws_launch_f32(int layout, int logn, int sub_d, const WsArgs& w, size_t smem, int grid, cudaStream_t st);
cudaError_t ws_launch_f16(int layout, int logn, int sub_d, const WsArgs& w, size_t smem, int grid, cudaStream_t st);
cudaError_t ws_launch_e5m3(int layout, int logn, int sub_d, const WsArgs& w, size_t smem, int grid, cudaStream_t st);
cudaError_t ws_launch_e4m4(int layout, int logn, int sub_d, const WsArgs& w, size_t smem, int grid, cudaStream_t st);

}  // namespace ivfpq
