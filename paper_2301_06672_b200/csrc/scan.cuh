// K2 + K3 + K4 -- per-(query, probed list) LUT build, PQ-code scan and top-k.
//
// Reference: search.py:158-184 (`search`): for every probed cluster c,
// rq = q - coarse[c] (search.py:173), build_lut (search.py:114-127 ->
// _raw_table :100-111), scan_list (:130-142), then top_k over the union
// (:145-155).
//
// One block per query walks its probe list in groups of G probes:
//   1. rq_g = fl(q - coarse[c_g])                                  (smem)
//   2. G LUTs built together: each thread owns table entries e and reads the
//      codebook row centers[e] ONCE for all G residuals, then stores the
//      entry in the storage dtype straight into shared memory (K2).
//        T[j][m] = sum_t fl(acc + fl(fl(centers[j][m][t] - rq[j*sub_d+t])^2))
//   3. The G inverted lists are scanned as one concatenated range; each
//      thread owns one vector and accumulates R = sum_j widen(T[j][code_j])
//      sequentially in j in fp32 (K3) -- bit-identical to scan_list.  Codes
//      are streamed with 16-byte non-allocating loads from the interleaved
//      layout, so a warp's load is 512
//      contiguous bytes.
//   4. (R bits << 32 | id) keys below the running K-th key go through the
//      block top-K (K4).  Ids are only read for keys that can still enter.
#pragma once
#include <stdint.h>

#include "codec.cuh"
#include "topk.cuh"

namespace ivfpq {

constexpr int SCAN_MAX_G = 8;

struct ScanArgs {
    const float* queries;     // [nq, d]
    const uint64_t* probes;   // [nq, P] keys, global cluster id in the low 32 bits
    const float* coarse;      // [nlist_local, d]
    const int32_t* g2l;       // [nlist_global] -> local list or -1
    const int64_t* glen;      // [nlist_global] global list lengths
    const int64_t* off;       // [nlist_local + 1] vector offsets
    const uint32_t* ids;      // [n_local]
    const uint8_t* codes;     // interleaved, s_pad bytes per vector
    const float* centers;     // [s, 2^p, sub_d]
    int nq, d, P, s, sub_d, s_pad, K, G;
    // outputs: keys mode (multi-GPU) or final mode (single GPU)
    uint64_t* out_keys;       // [nq, K] or null
    int64_t* out_ncand;       // [nq] or null
    int64_t* out_ids;         // [nq, K]
    float* out_dists;         // [nq, K]
    int32_t* out_short;       // [nq]
};

// L2 policy for the code stream: evict_last.  The code store (64 MB at cfg2)
// is re-read by every query that probes a list and fits the 126 MB L2; a
// default/no-allocate load stream measured 7x the DRAM traffic (4.9 GB vs
// 0.67 GB per cfg2 launch).  Not volatile: the compiler hoists it.
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint4 ld_stream16(const uint8_t* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(l2_evict_last_policy()));
    return r;
}

// Accumulate up to 16 table lookups from one 16-byte code chunk, j ascending.
template <int DT, int LOGN, bool FULL>
__device__ __forceinline__ float lookup16(float acc, uint4 w, const typename LutTraits<DT>::T* L, int nvalid) {
    const uint32_t words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int b = 0; b < 16; ++b) {
        if (FULL || b < nvalid) {
            uint32_t code = __byte_perm(words[b >> 2], 0u, 0x4440u | (b & 3));
            acc = __fadd_rn(acc, lut_widen<DT>(L[(b << LOGN) + code]));
        }
    }
    return acc;
}

// R for one vector: `vb` points at the vector's 16-byte slot of chunk 0 of its
// 32-vector block; chunks of the block are nb*16 bytes apart.
template <int DT, int LOGN>
__device__ __forceinline__ float scan_vector(const uint8_t* vb, int nb, const typename LutTraits<DT>::T* lut,
                                             int s) {
    const size_t cstride = (size_t)nb * 16;
    const int full = s >> 4;
    float acc = 0.0f;
    int cq = 0;
    for (; cq + 4 <= full; cq += 4) {
        uint4 w0 = ld_stream16(vb + (cq + 0) * cstride);
        uint4 w1 = ld_stream16(vb + (cq + 1) * cstride);
        uint4 w2 = ld_stream16(vb + (cq + 2) * cstride);
        uint4 w3 = ld_stream16(vb + (cq + 3) * cstride);
        acc = lookup16<DT, LOGN, true>(acc, w0, lut + ((cq + 0) << (4 + LOGN)), 16);
        acc = lookup16<DT, LOGN, true>(acc, w1, lut + ((cq + 1) << (4 + LOGN)), 16);
        acc = lookup16<DT, LOGN, true>(acc, w2, lut + ((cq + 2) << (4 + LOGN)), 16);
        acc = lookup16<DT, LOGN, true>(acc, w3, lut + ((cq + 3) << (4 + LOGN)), 16);
    }
    for (; cq < full; ++cq) {
        uint4 w = ld_stream16(vb + cq * cstride);
        acc = lookup16<DT, LOGN, true>(acc, w, lut + (cq << (4 + LOGN)), 16);
    }
    if (s & 15) {
        uint4 w = ld_stream16(vb + full * cstride);
        acc = lookup16<DT, LOGN, false>(acc, w, lut + (full << (4 + LOGN)), s & 15);
    }
    return lut_finish<DT>(acc);
}

// K2: build ng LUTs (one per residual) for the entries this thread owns.
template <int DT, int LOGN>
__device__ __forceinline__ void build_luts(typename LutTraits<DT>::T* lut, int lut_elems, const float* centers,
                                           const float* rq, int d, int sub_d, int ng) {
    for (int e = threadIdx.x; e < lut_elems; e += blockDim.x) {
        const int j = e >> LOGN;
        const float* cw = centers + (size_t)e * sub_d;
        const float* r0 = rq + j * sub_d;
        float acc[SCAN_MAX_G];
#pragma unroll
        for (int g = 0; g < SCAN_MAX_G; ++g) acc[g] = 0.0f;
        for (int t = 0; t < sub_d; ++t) {
            const float c = __ldg(cw + t);
#pragma unroll
            for (int g = 0; g < SCAN_MAX_G; ++g) {
                if (g < ng) {
                    float df = __fsub_rn(c, r0[g * d + t]);
                    acc[g] = __fadd_rn(acc[g], __fmul_rn(df, df));
                }
            }
        }
#pragma unroll
        for (int g = 0; g < SCAN_MAX_G; ++g)
            if (g < ng) lut[(size_t)g * lut_elems + e] = lut_store<DT>(acc[g]);
    }
}

struct ScanSmemLayout {
    size_t q, rq, grp, lut, tk, total;
    __host__ __device__ ScanSmemLayout(int d, int G, size_t lut_bytes_each, int K) {
        q = 0;
        rq = q + (size_t)d * 4;
        grp = rq + (size_t)G * d * 4;
        grp = (grp + 15) & ~(size_t)15;
        lut = grp + 256;
        tk = lut + (((size_t)G * lut_bytes_each + 15) & ~(size_t)15);
        total = tk + BlockTopK::smem_bytes(K);
    }
};

template <int DT, int LOGN>
// glut: null = LUTs in shared memory; else a per-block global LUT scratch
// [gridDim.x][G][s << p] for tables larger than shared memory.
__global__ void __launch_bounds__(TK_BLOCK) scan_kernel(const ScanArgs a, void* glut) {
    using T = typename LutTraits<DT>::T;
    extern __shared__ __align__(16) uint8_t smem[];
    const int lut_elems = a.s << LOGN;
    const ScanSmemLayout lay(a.d, a.G, glut ? 0 : (size_t)lut_elems * sizeof(T), a.K);
    float* qv = reinterpret_cast<float*>(smem + lay.q);
    float* rq = reinterpret_cast<float*>(smem + lay.rq);
    int* g_pref = reinterpret_cast<int*>(smem + lay.grp);       // [G+1]
    int* g_len = g_pref + (SCAN_MAX_G + 1);                      // [G]
    int* g_lc = g_len + SCAN_MAX_G;                              // [G]
    int* g_n = g_lc + SCAN_MAX_G;                                // [1]
    long long* g_off = reinterpret_cast<long long*>(smem + lay.grp + 128);  // [G]
    // Tables beyond shared memory (f32 LUT at s=240, p=8: 240 KiB) live in
    // this block's slice of a global scratch (L1/L2-resident; generic loads),
    // and the grid strides over the queries so the scratch stays bounded.
    T* lut = glut ? reinterpret_cast<T*>(glut) + (size_t)blockIdx.x * a.G * lut_elems
                    : reinterpret_cast<T*>(smem + lay.lut);
    BlockTopK tk;
    tk.bind(smem + lay.tk, a.K);

    for (int qi = blockIdx.x; qi < a.nq; qi += gridDim.x) {
    __syncthreads();  // the previous query's results were read from tk
    for (int t = threadIdx.x; t < a.d; t += blockDim.x) qv[t] = a.queries[(size_t)qi * a.d + t];
    tk.init();

    const uint64_t* probes = a.probes + (size_t)qi * a.P;
    int cursor = 0;          // thread 0 only
    long long ncand = 0;     // thread 0 only
    while (true) {
        if (threadIdx.x == 0) {
            int ng = 0, pref = 0;
            while (cursor < a.P && ng < a.G) {
                const uint64_t key = probes[cursor++];
                if (key == ~0ull) continue;
                const uint32_t gid = (uint32_t)key;
                ncand += a.glen[gid];
                const int lc = a.g2l[gid];
                if (lc < 0) continue;
                const long long o = a.off[lc], L = a.off[lc + 1] - o;
                if (L == 0) continue;
                g_lc[ng] = lc;
                g_len[ng] = (int)L;
                g_off[ng] = o;
                g_pref[ng] = pref;
                pref += (int)((L + 31) & ~31LL);
                ++ng;
            }
            g_pref[ng] = pref;
            *g_n = ng;
        }
        __syncthreads();
        const int ng = *g_n;
        if (ng == 0) break;

        // 1. residuals
        for (int i = threadIdx.x; i < ng * a.d; i += blockDim.x) {
            const int g = i / a.d, t = i - g * a.d;
            rq[i] = __fsub_rn(qv[t], a.coarse[(size_t)g_lc[g] * a.d + t]);
        }
        __syncthreads();
        // 2. LUTs
        build_luts<DT, LOGN>(lut, lut_elems, a.centers, rq, a.d, a.sub_d, ng);
        __syncthreads();
        // 3+4. scan the concatenated lists
        const int total = g_pref[ng];
        for (int base = 0; base < total; base += blockDim.x) {
            const int idx = base + threadIdx.x;
            int g = 0;
            while (g + 1 < ng && idx >= g_pref[g + 1]) ++g;
            const int v = idx - g_pref[g];
            uint64_t key = ~0ull;
            bool pass = false;
            if (idx < total && v < g_len[g]) {
                const int vblk = v & ~31;
                const int nb = min(32, g_len[g] - vblk);
                const uint8_t* vb = a.codes + (size_t)(g_off[g] + vblk) * a.s_pad + (size_t)(v & 31) * 16;
                const float R = scan_vector<DT, LOGN>(vb, nb, lut + (size_t)g * lut_elems, a.s);
                const uint32_t rb = __float_as_uint(R);
                const uint64_t tau = tk.tau();
                if (rb <= (uint32_t)(tau >> 32)) {
                    key = ((uint64_t)rb << 32) | a.ids[g_off[g] + v];
                    pass = key < tau;
                }
            }
            tk.offer(key, pass);
            if (base + (int)blockDim.x < total) tk.maybe_merge();
        }
        tk.merge();
    }

    // the candidate count must include probes after the last non-empty group
    if (threadIdx.x == 0) {
        while (cursor < a.P) {
            const uint64_t key = probes[cursor++];
            if (key != ~0ull) ncand += a.glen[(uint32_t)key];
        }
    }
    const uint64_t* r = tk.result();
    if (a.out_keys) {
        for (int i = threadIdx.x; i < a.K; i += blockDim.x) a.out_keys[(size_t)qi * a.K + i] = r[i];
        if (threadIdx.x == 0) a.out_ncand[qi] = ncand;
    } else {
        for (int i = threadIdx.x; i < a.K; i += blockDim.x) {
            const uint64_t key = r[i];
            const bool empty = key == ~0ull;
            a.out_ids[(size_t)qi * a.K + i] = empty ? -1LL : (long long)(uint32_t)key;
            a.out_dists[(size_t)qi * a.K + i] = empty ? __int_as_float(0x7f800000) : __uint_as_float((uint32_t)(key >> 32));
        }
        if (threadIdx.x == 0) a.out_short[qi] = ncand < a.K ? 1 : 0;
    }
    }  // queries
}

}  // namespace ivfpq
