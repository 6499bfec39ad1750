// K1 -- coarse cluster selection (reference search.py:91-97 `select_clusters`
// with datasets.py:166-176 `squared_l2_to_all`).
//
// d2[c] = sum_t fl(acc + fl(fl(coarse[c][t] - q[t])^2)), sequential in t,
// no FMA: each term is an explicit __fsub_rn/__fmul_rn/__fadd_rn, so the
// distances are bit-identical to the reference's and the selected probe set
// (ascending d2, ties -> lower cluster id) is exactly the reference's.
//
// Two kernels:
//  * coarse_l2_kernel: a register-tiled exact distance "GEMM" (64 queries x
//    64 centroids per block, 4x4 outputs per thread, d staged through smem in
//    slices of 16).  Zero-padded tail dims add fl(acc + 0) = acc, exact.
//  * select_probes_kernel: one block per query, block top-nprobe over the
//    distance row with keys (d2 bits << 32 | global cluster id).
#pragma once
#include <stdint.h>

#include "topk.cuh"

namespace ivfpq {

constexpr int CL_BQ = 64, CL_BC = 64, CL_BK = 16;

__global__ void __launch_bounds__(256)
coarse_l2_kernel(const float* __restrict__ Q, int nq, const float* __restrict__ C, int nc, int d,
                 float* __restrict__ D) {
    __shared__ __align__(16) float Qs[CL_BK][CL_BQ + 4];
    __shared__ __align__(16) float Cs[CL_BK][CL_BC + 4];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int q0 = blockIdx.y * CL_BQ, c0 = blockIdx.x * CL_BC;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

    for (int k0 = 0; k0 < d; k0 += CL_BK) {
        for (int i = threadIdx.x; i < CL_BQ * CL_BK; i += 256) {
            int r = i / CL_BK, kk = i % CL_BK;
            int qr = q0 + r, kd = k0 + kk;
            Qs[kk][r] = (qr < nq && kd < d) ? Q[(size_t)qr * d + kd] : 0.0f;
            int cr = c0 + r;
            Cs[kk][r] = (cr < nc && kd < d) ? C[(size_t)cr * d + kd] : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < CL_BK; ++kk) {
            float4 qv = *reinterpret_cast<const float4*>(&Qs[kk][ty * 4]);
            float4 cv = *reinterpret_cast<const float4*>(&Cs[kk][tx * 4]);
            float qa[4] = {qv.x, qv.y, qv.z, qv.w}, ca[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float df = __fsub_rn(ca[j], qa[i]);
                    acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(df, df));
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int qr = q0 + ty * 4 + i;
        if (qr >= nq) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int cr = c0 + tx * 4 + j;
            if (cr < nc) D[(size_t)qr * nc + cr] = acc[i][j];
        }
    }
}

// One block per query: keys (d2 bits << 32 | global id), block top-P.
__global__ void __launch_bounds__(TK_BLOCK)
select_probes_kernel(const float* __restrict__ D, int nc, const int32_t* __restrict__ l2g, int P,
                     uint64_t* __restrict__ out_keys) {
    extern __shared__ __align__(16) uint8_t smem[];
    BlockTopK tk;
    tk.bind(smem, P);
    tk.init();
    const float* row = D + (size_t)blockIdx.x * nc;
    for (int base = 0; base < nc; base += TK_BLOCK) {
        int c = base + threadIdx.x;
        uint64_t key = ~0ull;
        if (c < nc) key = ((uint64_t)__float_as_uint(row[c]) << 32) | (uint32_t)l2g[c];
        tk.offer(key, key < tk.tau());
        if (base + TK_BLOCK < nc) tk.maybe_merge();
    }
    tk.merge();
    const uint64_t* r = tk.result();
    for (int i = threadIdx.x; i < P; i += TK_BLOCK) out_keys[(size_t)blockIdx.x * P + i] = r[i];
}

}  // namespace ivfpq
