// Ingest kernels: PQ code assignment and coarse
// assignment on the GPU, so 10M / 100M-row indexes can be populated at all.
//
// pq_encode (pq.py:92-110) is BIT-EXACT with the reference for sub_d <= 4.
// The reference calls assign_to_centroids (kmeans.py:49-69) per subspace:
//     dot  = block @ centers[j].T          numpy -> OpenBLAS sgemm
//     dist = -2 * dot; dist += ||c||^2; dist += ||x||^2; max(dist, 0); argmin
// with the norms from np.einsum("ij,ij->i").  Probed in this container
// (numpy 2.3.5, OpenBLAS 0.3.30 SkylakeX; tests/golden/make_golden.py pins it
// with reference outputs):
//   * sgemm dot = sequential FMA chain over t: acc = fma(x_t, c_t, acc), acc0 = 0
//   * einsum ||v||^2 = sequential fl(acc + fl(v_t^2)) for n <= 3 and
//     fl(fl(v0^2 + v1^2) + fl(v2^2 + v3^2)) for n = 4
//   * fl(fl(-2 dot) + cn) == fma(-2, dot, cn) because -2*dot is exact
//   * argmin = first index of the minimum (ties -> lower code)
// These FMAs are the reference's own (BLAS) arithmetic; the search kernels
// stay FMA-free (tests/test_capi_host.py checks that per kernel).
//
// assign_to_centroids at full dimension (d = 96..960) uses the same
// expanded form; einsum's norm order for n >= 16 is a SIMD reduction with no
// simple model, so coarse assignment has decision-level
// parity (argmin agrees except on near-ties).
#pragma once
#include <stdint.h>

namespace ivfpq {

template <int SUB_D>
__device__ __forceinline__ float einsum_sq(const float (&v)[SUB_D]) {
    if constexpr (SUB_D == 4) {
        const float a = __fadd_rn(__fmul_rn(v[0], v[0]), __fmul_rn(v[1], v[1]));
        const float b = __fadd_rn(__fmul_rn(v[2], v[2]), __fmul_rn(v[3], v[3]));
        return __fadd_rn(a, b);
    } else {
        float acc = __fmul_rn(v[0], v[0]);
#pragma unroll
        for (int t = 1; t < SUB_D; ++t) acc = __fadd_rn(acc, __fmul_rn(v[t], v[t]));
        return acc;
    }
}

constexpr int ENC_THREADS = 128;  // vectors per CTA
constexpr int ENC_JG = 8;         // subspaces per CTA

// grid (ceil(n / ENC_THREADS), ceil(s / ENC_JG)); one thread per vector, the
// CTA's ENC_JG codebook rows staged in smem as records {c_0..c_{SUB_D-1}, cn}
// padded to CS floats (all threads read the same record: broadcast).
// Residual rows are fl(x - coarse[assign[i]]) when coarse != nullptr
// (compute_residuals, pq.py:54-63), else x itself.
template <int SUB_D>
__global__ void __launch_bounds__(ENC_THREADS) pq_encode_kernel(const float* __restrict__ X, int64_t n, int d,
                                                                const float* __restrict__ coarse,
                                                                const int64_t* __restrict__ assign,
                                                                const float* __restrict__ centers, int s, int N,
                                                                uint8_t* __restrict__ codes) {
    constexpr int CS = SUB_D <= 3 ? 4 : 8;
    extern __shared__ __align__(16) float enc_smem[];
    const int j0 = blockIdx.y * ENC_JG;
    const int jn = min(ENC_JG, s - j0);
    for (int e = threadIdx.x; e < jn * N; e += blockDim.x) {
        const float* c = centers + ((size_t)j0 * N + e) * SUB_D;
        float v[SUB_D];
#pragma unroll
        for (int t = 0; t < SUB_D; ++t) v[t] = c[t];
        float* r = enc_smem + (size_t)e * CS;
#pragma unroll
        for (int t = 0; t < SUB_D; ++t) r[t] = v[t];
        r[SUB_D] = einsum_sq<SUB_D>(v);
    }
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * ENC_THREADS + threadIdx.x;
    if (i >= n) return;
    const float* x = X + (size_t)i * d;
    const float* cv = coarse ? coarse + (size_t)assign[i] * d : nullptr;
#pragma unroll 1
    for (int jj = 0; jj < jn; ++jj) {
        const int j = j0 + jj;
        float r[SUB_D];
#pragma unroll
        for (int t = 0; t < SUB_D; ++t) {
            const float xv = __ldg(x + j * SUB_D + t);
            r[t] = cv ? __fsub_rn(xv, __ldg(cv + j * SUB_D + t)) : xv;
        }
        const float xn = einsum_sq<SUB_D>(r);
        const float* rec = enc_smem + (size_t)jj * N * CS;
        float best = __int_as_float(0x7f800000);
        int bi = 0;
#pragma unroll 4
        for (int m = 0; m < N; ++m) {
            const float4 c0 = *reinterpret_cast<const float4*>(rec + m * CS);
            float cc[CS == 4 ? 4 : 8];
            cc[0] = c0.x, cc[1] = c0.y, cc[2] = c0.z, cc[3] = c0.w;
            if constexpr (CS == 8) {
                const float4 c1 = *reinterpret_cast<const float4*>(rec + m * CS + 4);
                cc[4] = c1.x, cc[5] = c1.y, cc[6] = c1.z, cc[7] = c1.w;
            }
            float dot = __fmul_rn(r[0], cc[0]);  // fma(x0, c0, +0) = fl(x0 c0)
#pragma unroll
            for (int t = 1; t < SUB_D; ++t) dot = __fmaf_rn(r[t], cc[t], dot);
            float dist = __fadd_rn(__fmaf_rn(-2.0f, dot, cc[SUB_D]), xn);
            dist = dist < 0.0f ? 0.0f : dist;
            if (dist < best) {
                best = dist;
                bi = m;
            }
        }
        codes[(size_t)i * s + j] = (uint8_t)bi;
    }
}

// assign_to_centroids (kmeans.py:49-69) at full dimension: CTA = 64 rows x
// all centroids in 64-column tiles, 16x16 threads with 4x4 micro-tiles; each
// dot is a sequential FMA chain over t (the sgemm order probed for k <= 128).
// cn / xn: sequential fl(acc + fl(v_t^2)).  Each thread keeps the first
// minimum over its columns; the 16 column threads of a row reduce by
// (dist, index).
constexpr int AS_TM = 64, AS_TN = 64, AS_TK = 32;
__global__ void __launch_bounds__(256) assign_kernel(const float* __restrict__ X, int64_t n, int d,
                                                     const float* __restrict__ C, int nc,
                                                     const float* __restrict__ cn, int64_t* __restrict__ out_a,
                                                     float* __restrict__ out_d2) {
    __shared__ float xs[AS_TK][AS_TM + 4];
    __shared__ float cs[AS_TK][AS_TN + 4];
    __shared__ float xn_s[AS_TM];
    __shared__ float red_d[AS_TM][17];
    __shared__ int red_i[AS_TM][17];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t r0 = (int64_t)blockIdx.x * AS_TM;
    // row norms: 4 threads per row, then a sequential combine is NOT the
    // reference order -- so one thread per row, sequential over t.
    if (threadIdx.x < AS_TM) {
        const int64_t r = r0 + threadIdx.x;
        float acc = 0.0f;
        if (r < n) {
            const float* x = X + (size_t)r * d;
            acc = __fmul_rn(x[0], x[0]);
            for (int t = 1; t < d; ++t) acc = __fadd_rn(acc, __fmul_rn(x[t], x[t]));
        }
        xn_s[threadIdx.x] = acc;
    }
    float best[4];
    int bidx[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        best[a] = __int_as_float(0x7f800000);
        bidx[a] = 0x7fffffff;
    }
    for (int c0 = 0; c0 < nc; c0 += AS_TN) {
        float acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = 0.0f;
        for (int k0 = 0; k0 < d; k0 += AS_TK) {
            __syncthreads();
            for (int e = threadIdx.x; e < AS_TM * AS_TK; e += 256) {
                const int rr = e / AS_TK, kk = e % AS_TK;
                const int64_t r = r0 + rr;
                const int c = c0 + rr;
                xs[kk][rr] = (r < n && k0 + kk < d) ? X[(size_t)r * d + k0 + kk] : 0.0f;
                cs[kk][rr] = (c < nc && k0 + kk < d) ? C[(size_t)c * d + k0 + kk] : 0.0f;
            }
            __syncthreads();
            const int kmax = min(AS_TK, d - k0);
            for (int kk = 0; kk < kmax; ++kk) {
                const float4 xv = *reinterpret_cast<const float4*>(&xs[kk][ty * 4]);
                const float4 cvv = *reinterpret_cast<const float4*>(&cs[kk][tx * 4]);
                const float xa[4] = {xv.x, xv.y, xv.z, xv.w};
                const float ca[4] = {cvv.x, cvv.y, cvv.z, cvv.w};
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) acc[a][b] = __fmaf_rn(xa[a], ca[b], acc[a][b]);
            }
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int c = c0 + tx * 4 + b;
            if (c >= nc) continue;
            const float cnv = cn[c];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                float dist = __fadd_rn(__fmaf_rn(-2.0f, acc[a][b], cnv), xn_s[ty * 4 + a]);
                dist = dist < 0.0f ? 0.0f : dist;
                if (dist < best[a] || (dist == best[a] && c < bidx[a])) {
                    best[a] = dist;
                    bidx[a] = c;
                }
            }
        }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        red_d[ty * 4 + a][tx] = best[a];
        red_i[ty * 4 + a][tx] = bidx[a];
    }
    __syncthreads();
    if (threadIdx.x < AS_TM) {
        const int rr = threadIdx.x;
        float bd = red_d[rr][0];
        int bi = red_i[rr][0];
        for (int t = 1; t < 16; ++t) {
            const float dv = red_d[rr][t];
            const int iv = red_i[rr][t];
            if (dv < bd || (dv == bd && iv < bi)) {
                bd = dv;
                bi = iv;
            }
        }
        const int64_t r = r0 + rr;
        if (r < n) {
            out_a[r] = bi;
            if (out_d2) out_d2[r] = bd;
        }
    }
}

// ||c||^2 per centroid (sequential), for assign_kernel.
__global__ void row_sqnorm_kernel(const float* __restrict__ C, int64_t nc, int d, float* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nc) return;
    const float* c = C + (size_t)i * d;
    float acc = __fmul_rn(c[0], c[0]);
    for (int t = 1; t < d; ++t) acc = __fadd_rn(acc, __fmul_rn(c[t], c[t]));
    out[i] = acc;
}

// squared_l2_to_all (datasets.py:166-176): d2[i] = sequential fp32 sum over
// t of fl(fl(base[i][t] - q[t])^2), one thread per base row (no FMA).
__global__ void sq_l2_all_kernel(const float* __restrict__ base, int64_t n, int d, const float* __restrict__ q,
                                 float* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* b = base + i * d;
    float acc = 0.0f;
    for (int t = 0; t < d; ++t) {
        const float df = __fsub_rn(b[t], q[t]);
        acc = __fadd_rn(acc, __fmul_rn(df, df));
    }
    out[i] = acc;
}

// compute_residuals (pq.py:54-63): fl(x[i][t] - c[a[i]][t]).
__global__ void residuals_kernel(const float* __restrict__ x, int64_t n, int d, const float* __restrict__ c,
                                 const int64_t* __restrict__ a, float* __restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * d) return;
    const int64_t i = e / d;
    const int t = (int)(e - i * d);
    out[e] = __fsub_rn(x[e], c[a[i] * d + t]);
}

// reconstruct (pq.py:113-127): out[i][j*sub_d + t] = centers[j][codes[i][j]][t].
__global__ void reconstruct_kernel(const uint8_t* __restrict__ codes, int64_t n, int s, int N, int sub_d,
                                   const float* __restrict__ centers, float* __restrict__ out) {
    const int d = s * sub_d;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * d) return;
    const int64_t i = e / d;
    const int r = (int)(e - i * d), j = r / sub_d, t = r - j * sub_d;
    out[e] = centers[((int64_t)j * N + codes[i * s + j]) * sub_d + t];
}

}  // namespace ivfpq
