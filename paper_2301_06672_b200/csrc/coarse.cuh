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

// packed f32x2 sub / mul: two IEEE ops with one rounding each, as the scalar
// __fsub_rn / __fmul_rn; the adds stay scalar so nothing can be contracted
__device__ __forceinline__ unsigned long long cl_pk2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void cl_upk2(unsigned long long v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long cl_sub2(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long cl_mul2(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

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
            const float qa[4] = {qv.x, qv.y, qv.z, qv.w};
            // 2 instructions per element (packed sub + mul, scalar add) instead of 3
            const unsigned long long c01 = cl_pk2(cv.x, cv.y), c23 = cl_pk2(cv.z, cv.w);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const unsigned long long qq = cl_pk2(qa[i], qa[i]);
                const unsigned long long d01 = cl_sub2(c01, qq), d23 = cl_sub2(c23, qq);
                float s0, s1, s2, s3;
                cl_upk2(cl_mul2(d01, d01), s0, s1);
                cl_upk2(cl_mul2(d23, d23), s2, s3);
                acc[i][0] = __fadd_rn(acc[i][0], s0);
                acc[i][1] = __fadd_rn(acc[i][1], s1);
                acc[i][2] = __fadd_rn(acc[i][2], s2);
                acc[i][3] = __fadd_rn(acc[i][3], s3);
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

namespace ivfpq {

// ---------------------------------------------------------------------------
// Fused K1: exact distances + per-query top-P in one kernel (P <= CT_MAXP).
//
// CTA = 64 queries x one slice of centroids, walked in tiles of 64.  Per tile
// a thread computes a 4x4 micro-tile with packed f32x2 sub/mul (one rounding
// each, as numpy) and scalar adds (sequential in t; scalar so that ptxas
// cannot contract the f32x2 multiply into an FFMA2).  Keys
// (d2 bits << 32 | global id) under the query's running P-th key are
// appended to the query's buffer; after each tile one warp per query
// rank-sorts the buffer and merges it into the query's sorted list.  Slices
// are merged by merge_keys_kernel.  No distance matrix touches HBM.
constexpr int CT_BQ = 64, CT_BC = 64, CT_BK = 16, CT_MAXP = 64;

struct CoarseTopkArgs {
    const float* Q;
    const float* C;
    const int32_t* l2g;
    uint64_t* out;  // [nslices][nq][P]
    int nq, nc, d, P, slice;
    // optional indirection (exact re-do of guard failures): row i of this
    // launch is query qlist[i], i < *qcount; outputs stay at row i
    const int* qlist = nullptr;
    const int* qcount = nullptr;
};

__host__ __device__ inline size_t coarse_topk_smem(int P, int d) {
    const int dk = (d + CT_BK - 1) / CT_BK * CT_BK;
    return (size_t)dk * (CT_BQ + 4) * 4 + (size_t)CT_BQ * (2 * P + CT_BC) * 8 + (size_t)CT_BQ * 16;
}

__device__ __forceinline__ unsigned long long ct_pk2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void ct_upk2(unsigned long long v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long ct_sub2(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long ct_mul2(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

__global__ void __launch_bounds__(256) coarse_topk_kernel(const CoarseTopkArgs a) {
    __shared__ __align__(16) float Cs[2][CT_BK][CT_BC + 4];
    extern __shared__ __align__(16) uint8_t ct_smem[];
    const int P = a.P;
    const int dk = (a.d + CT_BK - 1) / CT_BK * CT_BK;                  // d padded to the chunk
    float* Qs = reinterpret_cast<float*>(ct_smem);                     // [dk][BQ + 4], resident
    uint64_t* lists = reinterpret_cast<uint64_t*>(Qs + (size_t)dk * (CT_BQ + 4));  // [BQ][2][P]
    uint64_t* buf = lists + (size_t)CT_BQ * 2 * P;                     // [BQ][BC]
    int* cnt = reinterpret_cast<int*>(buf + (size_t)CT_BQ * CT_BC);   // [BQ]
    int* cur = cnt + CT_BQ;                                            // [BQ]
    uint64_t* tau = reinterpret_cast<uint64_t*>(cur + CT_BQ);          // [BQ]
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nq = a.qcount ? *a.qcount : a.nq;
    const int cb = blockIdx.x * a.slice, ce = min(a.nc, cb + a.slice);
    // grid-stride over query blocks (one iteration unless the grid was sized
    // below the query count, as for the tensor-core path's exact re-do)
    for (int q0 = blockIdx.y * CT_BQ; q0 < nq; q0 += gridDim.y * CT_BQ) {
    for (int i = threadIdx.x; i < CT_BQ * 2 * P; i += 256) lists[i] = ~0ull;
    // queries, transposed: Qs[t][q]; zero-padded dims add fl(acc + 0) = acc
    for (int i = threadIdx.x; i < CT_BQ * dk; i += 256) {
        const int r = i / dk, t = i - r * dk;
        const int qi = q0 + r < nq ? (a.qlist ? a.qlist[q0 + r] : q0 + r) : -1;
        Qs[(size_t)t * (CT_BQ + 4) + r] = (qi >= 0 && t < a.d) ? a.Q[(size_t)qi * a.d + t] : 0.0f;
    }
    if (threadIdx.x < CT_BQ) {
        cnt[threadIdx.x] = 0;
        cur[threadIdx.x] = 0;
        tau[threadIdx.x] = ~0ull;
    }
    // centroid chunk loader: 64 centroids x 16 dims, 4 values per thread
    const int lr = threadIdx.x >> 2, lk = (threadIdx.x & 3) * 4;  // row, first dim of this thread's 4
    auto load_chunk = [&](int c0, int k0, float (&v)[4]) {
        const int cr = c0 + lr;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int kd = k0 + lk + u;
            v[u] = (cr < ce && kd < a.d) ? __ldg(a.C + (size_t)cr * a.d + kd) : 0.0f;
        }
    };
    const int nchunk = dk / CT_BK;
    float pre[4];
    load_chunk(cb, 0, pre);
    int buf_i = 0;
    __syncthreads();

    for (int c0 = cb; c0 < ce; c0 += CT_BC) {
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
        for (int kc = 0; kc < nchunk; ++kc) {
            // publish the prefetched chunk, prefetch the next one (next tile's first at the end)
#pragma unroll
            for (int u = 0; u < 4; ++u) Cs[buf_i][lk + u][lr] = pre[u];
            if (kc + 1 < nchunk) load_chunk(c0, (kc + 1) * CT_BK, pre);
            else if (c0 + CT_BC < ce) load_chunk(c0 + CT_BC, 0, pre);
            __syncthreads();
            const float* qb = Qs + (size_t)kc * CT_BK * (CT_BQ + 4);
#pragma unroll
            for (int kk = 0; kk < CT_BK; ++kk) {
                const float4 qv = *reinterpret_cast<const float4*>(qb + kk * (CT_BQ + 4) + ty * 4);
                const float4 cv = *reinterpret_cast<const float4*>(&Cs[buf_i][kk][tx * 4]);
                const float qa[4] = {qv.x, qv.y, qv.z, qv.w};
                const unsigned long long c01 = ct_pk2(cv.x, cv.y), c23 = ct_pk2(cv.z, cv.w);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const unsigned long long qq = ct_pk2(qa[i], qa[i]);
                    const unsigned long long d01 = ct_sub2(c01, qq), d23 = ct_sub2(c23, qq);
                    float s0, s1, s2, s3;
                    ct_upk2(ct_mul2(d01, d01), s0, s1);
                    ct_upk2(ct_mul2(d23, d23), s2, s3);
                    acc[i][0] = __fadd_rn(acc[i][0], s0);
                    acc[i][1] = __fadd_rn(acc[i][1], s1);
                    acc[i][2] = __fadd_rn(acc[i][2], s2);
                    acc[i][3] = __fadd_rn(acc[i][3], s3);
                }
            }
            buf_i ^= 1;  // the other buffer is written next chunk; its readers passed this barrier
        }
        // candidates under the query's running P-th key
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int ql = ty * 4 + i;
            const uint64_t t = tau[ql];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int c = c0 + tx * 4 + j;
                if (c < ce) {
                    const uint64_t key = ((uint64_t)__float_as_uint(acc[i][j]) << 32) | (uint32_t)a.l2g[c];
                    if (key < t) buf[(size_t)ql * CT_BC + atomicAdd(&cnt[ql], 1)] = key;
                }
            }
        }
        __syncthreads();
        // merge: one warp per query
        for (int ql = warp; ql < CT_BQ; ql += 8) {
            const int n = cnt[ql];
            if (n == 0) continue;
            uint64_t* b = buf + (size_t)ql * CT_BC;
            // rank-sort the candidates (keys unique: distinct centroid ids)
            uint64_t x0 = lane < n ? b[lane] : ~0ull, x1 = lane + 32 < n ? b[lane + 32] : ~0ull;
            int r0 = 0, r1 = 0;
            for (int j = 0; j < n; ++j) {
                const uint64_t y = b[j];
                r0 += y < x0;
                r1 += y < x1;
            }
            __syncwarp();
            if (lane < n) b[r0] = x0;
            if (lane + 32 < n) b[r1] = x1;
            __syncwarp();
            const uint64_t* A = lists + ((size_t)ql * 2 + cur[ql]) * P;
            uint64_t* O = lists + ((size_t)ql * 2 + (cur[ql] ^ 1)) * P;
            for (int i = lane; i < P; i += 32) {
                const uint64_t v = A[i];
                const int pos = i + lower_bound_u64(b, n, v);
                if (pos < P) O[pos] = v;
            }
            for (int i = lane; i < n; i += 32) {
                const uint64_t v = b[i];
                const int pos = i + lower_bound_u64(A, P, v);
                if (pos < P) O[pos] = v;
            }
            __syncwarp();
            if (lane == 0) {
                cur[ql] ^= 1;
                tau[ql] = O[P - 1];
                cnt[ql] = 0;
            }
            __syncwarp();
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < CT_BQ * P; i += 256) {
        const int ql = i / P, k = i - ql * P;
        if (q0 + ql < nq)
            a.out[((size_t)blockIdx.x * a.nq + q0 + ql) * P + k] = lists[((size_t)ql * 2 + cur[ql]) * P + k];
    }
    __syncthreads();
    }
}

}  // namespace ivfpq
