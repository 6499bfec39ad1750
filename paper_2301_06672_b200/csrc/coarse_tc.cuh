// K1 on the 5th-generation tensor cores: queries x centroids on tcgen05 (TF32,
// accumulators in TMEM), threshold shortlist in the epilogue, exact re-rank.
//
// Reference semantics (search.py:91-97, datasets.py:166-176): probes are the
// nprobe smallest (d2, cluster id) with d2 the *sequential fp32* squared L2.
// Tensor-core dot products are not that number, so they only nominate:
//   1. S = Q . C^T on tcgen05.mma.kind::tf32 (M=128 queries, N=128 centroids,
//      K=8 per instruction).  A (the query block) lives in TMEM, written once
//      by the epilogue warps (tcgen05.st), so the tensor core reads only B
//      from shared memory -- SS mode at N=128 would need 128 B/clk of smem for
//      the operands alone.  B = 128B-swizzled K-major centroid tiles
//      (pre-swizzled once per index) streamed by cp.async.bulk through a
//      6-stage mbarrier ring; D double-buffered in TMEM so the epilogue of
//      tile t overlaps the MMAs of tile t+1.
//   2. Two passes over the slice's tiles (the centroid images stay in L2).
//      The GEMM yields the score s = |c|^2 - 2 q.c directly (K is augmented
//      with |c|^2, see coarse_tc_prep_kernel).  Two epilogue threads own one
//      query (= one TMEM lane; one per column half).  Pass 1 keeps, in
//      registers, the minimum score of each of 64 column groups -- branch-free --
//      and takes thr = the TC_GJ-th smallest group minimum (at least TC_GJ
//      scores are <= thr; ~90 expected for TC_GJ = 48).  Pass 2 appends every
//      centroid with s <= thr to the query's buffer (predicated store).
//   3. coarse_rerank_kernel re-ranks the nominated centroids with the
//      reference formula (bit-exact keys) and keeps the P smallest.
//   4. Guard: every centroid not nominated has s > thr.  TF32 keeps 10
//      mantissa bits, so |q.c - S| <= 2^-9 |q| |c| (+ fp32 accumulation, far
//      smaller); with E = 2^-8 |q| Cmax + 2^-12 (|q|^2 + Cmax^2) (the second
//      term covers |c|^2's split, TF32 accumulation, |q|^2's rounding) and the
//      reference sum's own rounding (relative <= d 2^-24 < 2^-16):
//          ref_d2(c) > (|q|^2 + thr - E) (1 - 2^-16)  =: lower.
//      If lower <= the P-th exact distance (or the buffer overflowed) the
//      query is flagged and re-done by the exact SIMT kernel.  The result is
//      therefore always the reference's; the statistics above only decide how
//      often the re-do runs (never, on the BASELINE configs).
#pragma once
#include <stdint.h>

#include "topk.cuh"

namespace ivfpq {

constexpr int TC_M = 128;        // queries per CTA (TMEM lanes)
constexpr int TC_N = 128;        // centroids per tile (TMEM columns per accumulator)
constexpr int TC_KC = 32;        // fp32 per 128-byte swizzled row (one K chunk)
constexpr int TC_GROUPS = 64;    // column groups of pass 1
constexpr int TC_GJ = 48;        // thr = TC_GJ-th smallest group minimum
constexpr int TC_CAP = 128;      // nominated centroids per (query, slice)
constexpr int TC_STAGES = 6;
constexpr int TC_ACOL = 256;     // TMEM columns [0, 256): two accumulators; [256, 512): the query block (A)
constexpr int TC_MAXD = TC_ACOL - 2;  // A = [-2q, 1, 1] must fit 256 TMEM columns
constexpr int TC_MAXP = 96;      // nprobe served by this path (P > 32 uses >= ceil(P/32) slices)
constexpr int TC_P_PER_SLICE = 32;  // nprobe covered per slice by its ~TC_GJ..90 nominations
constexpr int TC_MAXSL = 4;      // centroid slices per query block
constexpr int TC_EPI = 8;        // epilogue warps: 2 per TMEM lane quarter (column halves)
constexpr int TC_THREADS = 128 + 32 * TC_EPI;  // warp 0 producer, 1 MMA, 2 TMEM alloc, 4.. epilogue

struct CoarseTcArgs {
    const float* Q;          // [nq, d]
    const float* cimg;       // [ntiles][nkc][TC_N rows x 32 fp32], swizzled images of [c, hi(|c|^2), lo(|c|^2)]
    int32_t* cand;           // [nslices][nq][TC_CAP] nominated local centroid ids
    int32_t* ncand;          // [nslices][nq] count (TC_CAP + 1 = overflow)
    float* thr;              // [nslices][nq]
    int nq, nc, d, tiles_per_slice, nkc;
};

struct CoarseRerankArgs {
    const float* Q;          // [nq, d]
    const float* C;          // [nc, d]
    const int32_t* l2g;      // [nc]
    const int32_t* cand;     // from coarse_tc_kernel
    const int32_t* ncand;
    const float* thr;
    uint64_t* out;           // [nq][P] exact keys (d2 bits << 32 | global id)
    int* flag_count;         // queries whose guard failed (re-done exactly)
    int* flag_list;
    float cmax;              // max |c| over the centroids
    int nq, nc, d, P, nsl, force_flag;
};

// K of the GEMM: d coordinates + the two halves of |c|^2 (see coarse_tc_prep_kernel)
__host__ __device__ inline int coarse_tc_nkc(int d) { return (d + 2 + TC_KC - 1) / TC_KC; }

__host__ __device__ inline size_t coarse_tc_smem(int d) {
    const int nkc = coarse_tc_nkc(d);
    (void)nkc;
    return 1024 /* align */ + (size_t)TC_STAGES * TC_N * 128 /* B */ + (size_t)TC_M * TC_CAP * 4 /* nominations */ +
           1024 /* counts, barriers, tmem addr */;
}

// max over rows of |c|, rounded up (guard constant)
inline float coarse_tc_cmax(const float* C, long long nc, long long d) {
    double m = 0.0;
    for (long long c = 0; c < nc; ++c) {
        double s = 0.0;
        for (long long t = 0; t < d; ++t) s += (double)C[c * d + t] * C[c * d + t];
        if (s > m) m = s;
    }
    return (float)(__builtin_sqrt(m) * (1.0 + 1e-6));
}

// byte offset of element (row r, k) inside a [rows x 32 fp32] 128B-swizzled K-major image
__host__ __device__ __forceinline__ uint32_t sw128_off(int r, int k) {
    return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 2) ^ (r & 7)) & 7) << 4) + (k & 3) * 4);
}

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    // start >> 4 | LBO (16 B) | SBO (1024 B) | version 1 | SWIZZLE_128B
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ uint32_t tc_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tc_mbar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem(b)), "r"(n));
}
__device__ __forceinline__ void tc_mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n\t}" ::"r"(tc_smem(b)),
        "r"(ph)
        : "memory");
}
__device__ __forceinline__ void tc_mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc_smem(b)) : "memory");
}
__device__ __forceinline__ void tc_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc_smem(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tc_bulk(uint32_t dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(tc_smem(b))
                 : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]^T  (A from tensor memory: only B is read from shared memory)
__device__ __forceinline__ void tc_mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tc_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
        "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(tc_smem(b))
                 : "memory");
}
__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

// Centroid tiles -> swizzled K-major images [tile][kc][TC_N x 32 fp32] of the
// augmented rows [c_0 .. c_{d-1}, hi, lo, 0 ...] with hi + lo = |c|^2 (hi has
// 10 mantissa bits, exact in TF32; lo's TF32 error <= 2^-20 |c|^2).  The
// query rows are [-2 q, 1, 1, 0 ...], so the GEMM yields s = |c|^2 - 2 q.c.
// Padding rows (c >= nc) score 1e30.
__global__ void coarse_tc_prep_kernel(const float* __restrict__ C, int nc, int d, int nkc, float* __restrict__ img) {
    __shared__ float cn_s[TC_N];
    const int tile = blockIdx.x;
    for (int r = threadIdx.x; r < TC_N; r += blockDim.x) {
        const int c = tile * TC_N + r;
        float s = 1e30f;
        if (c < nc) {
            s = 0.0f;
            for (int k = 0; k < d; ++k) s = __fadd_rn(s, __fmul_rn(C[(size_t)c * d + k], C[(size_t)c * d + k]));
        }
        cn_s[r] = s;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < TC_N * nkc * TC_KC; i += blockDim.x) {
        const int r = i / (nkc * TC_KC), k = i - r * (nkc * TC_KC);
        const int c = tile * TC_N + r, kc = k / TC_KC;
        const float hi = __uint_as_float(__float_as_uint(cn_s[r]) & 0xffffe000u);
        float v = 0.0f;
        if (k < d) v = c < nc ? C[(size_t)c * d + k] : 0.0f;
        else if (k == d) v = hi;
        else if (k == d + 1) v = c < nc ? __fsub_rn(cn_s[r], hi) : 0.0f;
        uint8_t* base = reinterpret_cast<uint8_t*>(img) + ((size_t)tile * nkc + kc) * (TC_N * 128);
        *reinterpret_cast<float*>(base + sw128_off(r, k - kc * TC_KC)) = v;
    }
}

// k-th smallest (0-based, compile-time) of 64 register values: bitonic sort.
template <int KTH>
__device__ __forceinline__ float tc_kth_of_64(float (&g)[TC_GROUPS]) {
#pragma unroll
    for (int k = 2; k <= TC_GROUPS; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < TC_GROUPS; ++i) {
                const int l = i ^ j;
                if (l > i) {
                    const float a = g[i], b = g[l];
                    const bool up = (i & k) == 0;
                    g[i] = up ? fminf(a, b) : fmaxf(a, b);
                    g[l] = up ? fmaxf(a, b) : fminf(a, b);
                }
            }
    return g[KTH];
}

__global__ void __launch_bounds__(TC_THREADS, 1) coarse_tc_kernel(const CoarseTcArgs a) {
    extern __shared__ uint8_t tc_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)tc_raw + 1023) & ~(uintptr_t)1023);
    const int nkc = a.nkc;
    uint8_t* sB = smem;                                   // [STAGES][128 x 128 B]
    int32_t* nom = reinterpret_cast<int32_t*>(sB + (size_t)TC_STAGES * TC_N * 128);  // [TC_CAP][128]
    int* cnt = nom + (size_t)TC_M * TC_CAP;                                            // [128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(cnt + TC_M);
    uint64_t* full = bars;                 // [STAGES]
    uint64_t* empty = full + TC_STAGES;    // [STAGES]
    uint64_t* accf = empty + TC_STAGES;    // [2]
    uint64_t* acce = accf + 2;             // [2]
    uint64_t* aready = acce + 2;           // A written to TMEM
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aready + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q0 = blockIdx.y * TC_M;
    const int t_begin = blockIdx.x * a.tiles_per_slice;
    const int ntiles_total = (a.nc + TC_N - 1) / TC_N;
    const int t_end = min(ntiles_total, t_begin + a.tiles_per_slice);
    const int ntl = max(0, t_end - t_begin);
    const int nsteps = 2 * ntl;  // pass 1 then pass 2 over the same tiles

    // ---- setup: barriers, TMEM (2 accumulators x 128 columns + A)
    if (threadIdx.x < TC_M) cnt[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            tc_mbar_init(full + s, 1);
            tc_mbar_init(empty + s, 1);
        }
        for (int s = 0; s < 2; ++s) {
            tc_mbar_init(accf + s, 1);
            tc_mbar_init(acce + s, TC_EPI);  // one arrival per epilogue warp
        }
        tc_mbar_init(aready, 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tc_smem(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---- producer: centroid tile images through the stage ring (both passes)
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            int it = 0;
            for (int st = 0; st < nsteps; ++st) {
                const int t = st < ntl ? st : st - ntl;
                for (int kc = 0; kc < nkc; ++kc, ++it) {
                    if (it >= TC_STAGES) tc_mbar_wait(empty + s, ph ^ 1);
                    tc_expect_tx(full + s, TC_N * 128);
                    tc_bulk(tc_smem(sB + (size_t)s * TC_N * 128),
                            a.cimg + ((size_t)(t_begin + t) * nkc + kc) * (TC_N * 32), TC_N * 128, full + s);
                    if (++s == TC_STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---- MMA issuer (one thread)
        if (lane == 0) {
            constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_N >> 3) << 17) |
                                       ((uint32_t)(TC_M >> 4) << 24);
            int s = 0;
            uint32_t ph = 0;
            tc_mbar_wait(aready, 0);
            for (int st = 0; st < nsteps; ++st) {
                const int ab = st & 1;
                if (st >= 2) tc_mbar_wait(acce + ab, ((st >> 1) - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t dcol = tmem + (uint32_t)(ab * TC_N);
                for (int kc = 0; kc < nkc; ++kc) {
                    tc_mbar_wait(full + s, ph);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t b0 = tc_smem(sB + (size_t)s * TC_N * 128);
#pragma unroll
                    for (int ks = 0; ks < TC_KC / 8; ++ks)
                        tc_mma_tf32_ts(dcol, tmem + (uint32_t)(TC_ACOL + kc * TC_KC + ks * 8),
                                       umma_desc_sw128(b0 + ks * 32), idesc, (kc | ks) != 0);
                    tc_commit(empty + s);  // frees the stage when these MMAs have read it
                    if (++s == TC_STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                tc_commit(accf + ab);  // accumulator ready
            }
        }
    } else if (warp >= 4) {
        // ---- epilogue: thread r = TMEM lane r = query q0 + r; warp half h owns
        // tile columns [64h, 64h + 64) and column groups 32h + (c mod 32)
        const int r = ((warp & 3) << 5) | lane;
        const int h = (warp - 4) >> 2;
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        if (h == 0) {
            // A row of query q0 + r -> TMEM lane r, columns TC_ACOL + k: [-2 q, 1, 1, 0 ...]
            const bool valid = q0 + r < a.nq;
            const float* qrow = a.Q + (size_t)(q0 + r) * a.d;
            for (int kc = 0; kc < nkc; ++kc) {
                uint32_t x[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int k = kc * TC_KC + j;
                    float v = 0.0f;
                    if (valid) v = k < a.d ? __fmul_rn(-2.0f, __ldg(qrow + k)) : (k < a.d + 2 ? 1.0f : 0.0f);
                    x[j] = __float_as_uint(v);
                }
                tc_st32(tmem + lane_base + (uint32_t)(TC_ACOL + kc * TC_KC), x);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) tc_mbar_arrive(aready);
        }
        float gmin[32];
#pragma unroll
        for (int g = 0; g < 32; ++g) gmin[g] = __int_as_float(0x7f800000);
        float thr = __int_as_float(0x7f800000);
        for (int st = 0; st < nsteps; ++st) {
            const int ab = st & 1;
            const bool pass2 = st >= ntl;
            if (st == ntl) {
                // thr = TC_GJ-th smallest of the query's 64 group minima (both halves)
                float* gm = reinterpret_cast<float*>(nom);  // [64][128], free until pass 2 appends
#pragma unroll
                for (int g = 0; g < 32; ++g) gm[(h * 32 + g) * TC_M + r] = gmin[g];
                asm volatile("bar.sync 1, %0;" ::"n"(32 * TC_EPI) : "memory");
                float all[TC_GROUPS];
#pragma unroll
                for (int g = 0; g < TC_GROUPS; ++g) all[g] = gm[g * TC_M + r];
                thr = tc_kth_of_64<TC_GJ - 1>(all);
                if (q0 + r >= a.nq) thr = -__int_as_float(0x7f800000);  // padding row: nominate nothing
                asm volatile("bar.sync 1, %0;" ::"n"(32 * TC_EPI) : "memory");
            }
            tc_mbar_wait(accf + ab, (st >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            uint32_t v0[32], v1[32];
            const uint32_t col = tmem + lane_base + (uint32_t)(ab * TC_N + 64 * h);
            tc_ld32(col, v0);
            tc_ld32(col + 32, v1);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            // accumulator consumed: release it to the MMA warp before the bookkeeping
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) tc_mbar_arrive(acce + ab);
            if (!pass2) {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    gmin[j] = fminf(gmin[j], fminf(__uint_as_float(v0[j]), __uint_as_float(v1[j])));
            } else {
                uint32_t m0 = 0, m1 = 0;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    m0 |= (uint32_t)(__uint_as_float(v0[j]) <= thr) << j;
                    m1 |= (uint32_t)(__uint_as_float(v1[j]) <= thr) << j;
                }
                const int cb = (t_begin + st - ntl) * TC_N + 64 * h;
                uint64_t m = ((uint64_t)m1 << 32) | m0;
                while (m) {
                    const int j = __ffsll((long long)m) - 1;
                    m &= m - 1;
                    const int c = cb + j;
                    if (c < a.nc) {
                        const int n = atomicAdd(cnt + r, 1);
                        if (n < TC_CAP) nom[(size_t)n * TC_M + r] = c;
                    }
                }
            }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * TC_EPI) : "memory");
        if (h == 0 && q0 + r < a.nq) {
            const size_t row = (size_t)blockIdx.x * a.nq + q0 + r;
            const int n = cnt[r];
            const int nw = min(n, TC_CAP);
            int32_t* o = a.cand + row * TC_CAP;
            for (int i = 0; i < nw; ++i) o[i] = nom[(size_t)i * TC_M + r];
            a.ncand[row] = n > TC_CAP ? TC_CAP + 1 : n;
            a.thr[row] = thr;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// One warp per query: re-rank the slices' nominated centroids with the
// reference formula (fl(c - q), fl(x * x), fl(acc + .) sequential in t --
// datasets.py:166-176), keep the P smallest exact keys (rank selection; keys
// are unique: distinct ids) and apply the guard.
constexpr int TC_RR_WARPS = 4;
constexpr int TC_RR_STG = 32 * 33;  // per-warp staging: 32 dims x 32 candidate rows (+1 pad)
__host__ __device__ inline size_t coarse_rerank_smem(int nsl, int d) {
    return (size_t)TC_RR_WARPS * ((size_t)nsl * TC_CAP * 12 + (size_t)((d + 3) & ~3) * 4 + TC_RR_STG * 4);
}

__device__ __forceinline__ float tc_sq_acc(float acc, float x, float q) {
    const float e = __fsub_rn(x, q);
    return __fadd_rn(acc, __fmul_rn(e, e));
}

// Exact squared L2 (reference formula, sequential in t) of up to 32 centroid
// rows rowid(0..nb-1) against qs; lane i returns candidate i's distance.  Dims
// are walked in chunks of 32, each chunk's rows brought in with coalesced
// 128-byte loads and staged transposed ([t][33], conflict-free) in stg.
template <class RowId>
__device__ __forceinline__ float tc_exact_batch(const float* __restrict__ C, int d, const float* qs, float* stg,
                                                int nb, RowId rowid) {
    const int lane = threadIdx.x & 31;
    float acc = 0.0f;
    if ((d & 3) == 0) {
        const int seg = lane & 7;
        const float* rows[8];
#pragma unroll
        for (int it = 0; it < 8; ++it) {
            const int r = 4 * it + (lane >> 3);
            rows[it] = C + (size_t)rowid(r < nb ? r : 0) * d;
        }
        float4 pre[8];
        auto load = [&](int ch) {
            const int t = ch * 32 + seg * 4;
#pragma unroll
            for (int it = 0; it < 8; ++it)
                pre[it] = t < d ? __ldg(reinterpret_cast<const float4*>(rows[it] + t)) : make_float4(0, 0, 0, 0);
        };
        const int nchunk = (d + 31) >> 5;
        load(0);
        for (int ch = 0; ch < nchunk; ++ch) {
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const int r = 4 * it + (lane >> 3);
                stg[(seg * 4 + 0) * 33 + r] = pre[it].x;
                stg[(seg * 4 + 1) * 33 + r] = pre[it].y;
                stg[(seg * 4 + 2) * 33 + r] = pre[it].z;
                stg[(seg * 4 + 3) * 33 + r] = pre[it].w;
            }
            __syncwarp();
            if (ch + 1 < nchunk) load(ch + 1);
            const int tn = min(32, d - ch * 32);
            const float* qc = qs + ch * 32;
            for (int t = 0; t < tn; ++t) acc = tc_sq_acc(acc, stg[t * 33 + lane], qc[t]);
            __syncwarp();
        }
    } else {
        const float* row = C + (size_t)rowid(lane < nb ? lane : 0) * d;
        for (int t = 0; t < d; ++t) acc = tc_sq_acc(acc, __ldg(row + t), qs[t]);
    }
    return acc;
}

__global__ void __launch_bounds__(32 * TC_RR_WARPS) coarse_rerank_kernel(const CoarseRerankArgs a) {
    extern __shared__ __align__(16) uint8_t rr_smem[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = blockIdx.x * TC_RR_WARPS + w;
    if (q >= a.nq) return;
    const int maxn = a.nsl * TC_CAP;
    const int dq = (a.d + 3) & ~3;
    uint8_t* base = rr_smem + (size_t)w * ((size_t)maxn * 12 + (size_t)dq * 4 + TC_RR_STG * 4);
    uint64_t* K = reinterpret_cast<uint64_t*>(base);
    float* qs = reinterpret_cast<float*>(K + maxn);
    float* stg = qs + dq;                                     // [32 dims][33]
    int32_t* ids = reinterpret_cast<int32_t*>(stg + TC_RR_STG);
    // gather the nominations of every slice
    int n = 0;
    bool overflow = false;
    float thr = __int_as_float(0x7f800000);
    for (int s = 0; s < a.nsl; ++s) {
        const size_t row = (size_t)s * a.nq + q;
        const int ns = a.ncand[row];
        thr = fminf(thr, a.thr[row]);
        if (ns > TC_CAP) {
            overflow = true;
            continue;
        }
        for (int i = lane; i < ns; i += 32) ids[n + i] = a.cand[row * TC_CAP + i];
        n += ns;
    }
    const float* qg = a.Q + (size_t)q * a.d;
    float qn = 0.0f;
    for (int t = lane; t < a.d; t += 32) {
        const float v = qg[t];
        qs[t] = v;
        qn = __fadd_rn(qn, __fmul_rn(v, v));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) qn += __shfl_xor_sync(0xffffffffu, qn, o);
    __syncwarp();
    // exact distances: batches of 32 candidates (lane i <-> candidate i)
    for (int b0 = 0; b0 < n; b0 += 32) {
        const int nb = min(32, n - b0);
        const float acc = tc_exact_batch(a.C, a.d, qs, stg, nb, [&](int r) { return ids[b0 + r]; });
        if (lane < nb) K[b0 + lane] = ((uint64_t)__float_as_uint(acc) << 32) | (uint32_t)a.l2g[ids[b0 + lane]];
    }
    __syncwarp();
    // rank selection of the P smallest exact keys
    uint64_t* outq = a.out + (size_t)q * a.P;
    uint64_t kp = ~0ull;  // the P-th key
    for (int i = lane; i < n; i += 32) {
        const uint64_t x = K[i];
        int rank = 0;
        for (int j = 0; j < n; ++j) rank += K[j] < x;
        if (rank < a.P) outq[rank] = x;
        if (rank == a.P - 1) kp = x;
    }
    for (int i = n + lane; i < a.P; i += 32) outq[i] = ~0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const uint64_t y = __shfl_xor_sync(0xffffffffu, kp, o);
        kp = y < kp ? y : kp;
    }
    if (lane == 0) {
        bool ok = !overflow && n >= a.P;
        if (ok && thr != __int_as_float(0x7f800000)) {  // thr = inf: every centroid was nominated
            float qnorm;  // approximate sqrt (rel. error ~2^-22), padded by 2^-12
            asm("sqrt.approx.f32 %0, %1;" : "=f"(qnorm) : "f"(qn));
            qnorm = __fmul_rn(qnorm, 1.000244140625f);
            const float E = __fadd_rn(__fmul_rn(__fmul_rn(qnorm, a.cmax), 0.00390625f),                // 2^-8
                                      __fmul_rn(__fadd_rn(qn, __fmul_rn(a.cmax, a.cmax)), 2.44140625e-04f));  // 2^-12
            const float lower = __fmul_rn(__fsub_rn(__fadd_rn(qn, thr), E), 0.9999847412109375f);          // 1 - 2^-16
            const float dP = __uint_as_float((uint32_t)(kp >> 32));
            ok = lower > dP;  // false for NaN as well
        }
        if (!ok || a.force_flag) a.flag_list[atomicAdd(a.flag_count, 1)] = q;
    }
}

// Exact re-do of the queries whose guard failed: one CTA per flagged query
// (grid-stride), every owned centroid through tc_exact_batch, block top-P.
inline size_t coarse_redo_smem(int P, int d) {
    return BlockTopK::smem_bytes(P) + (size_t)(TK_BLOCK / 32) * TC_RR_STG * 4 + (size_t)((d + 3) & ~3) * 4;
}

__global__ void __launch_bounds__(TK_BLOCK) coarse_redo_kernel(const float* __restrict__ Q, const float* __restrict__ C,
                                                              const int32_t* __restrict__ l2g, int nc, int d, int P,
                                                              const int* flag_count, const int* flag_list,
                                                              uint64_t* __restrict__ out) {
    extern __shared__ __align__(16) uint8_t rd_smem[];
    BlockTopK tk;
    tk.bind(rd_smem, P);
    float* stg = reinterpret_cast<float*>(rd_smem + BlockTopK::smem_bytes(P)) + (threadIdx.x >> 5) * TC_RR_STG;
    float* qs = reinterpret_cast<float*>(rd_smem + BlockTopK::smem_bytes(P)) + (TK_BLOCK / 32) * TC_RR_STG;
    const int nf = *flag_count;
    for (int f = blockIdx.x; f < nf; f += gridDim.x) {
        const int q = flag_list[f];
        for (int t = threadIdx.x; t < d; t += TK_BLOCK) qs[t] = Q[(size_t)q * d + t];
        tk.init();  // includes a barrier
        for (int base = 0; base < nc; base += TK_BLOCK) {
            const int c0 = base + (threadIdx.x & ~31);
            const int nb = max(0, min(32, nc - c0));
            uint64_t key = ~0ull;
            if (nb > 0) {
                const float acc = tc_exact_batch(C, d, qs, stg, nb, [&](int r) { return c0 + r; });
                const int c = c0 + (threadIdx.x & 31);
                if (c < nc) key = ((uint64_t)__float_as_uint(acc) << 32) | (uint32_t)l2g[c];
            }
            tk.offer(key, key < tk.tau());
            if (base + TK_BLOCK < nc) tk.maybe_merge();
        }
        tk.merge();
        for (int i = threadIdx.x; i < P; i += TK_BLOCK) out[(size_t)q * P + i] = tk.result()[i];
        __syncthreads();
    }
}

}  // namespace ivfpq
