// ivfpq_b200 -- device index, kernel launches and the C ABI (include/ivfpq_b200.h).
//
// Everything here runs on the GPU; there is no CPU compute path.  Host code
// only validates arguments, moves buffers and launches kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ivfpq_b200.h"
#define IVFPQ_DEFINE_PLAN_KERNEL
#include "codec.cuh"
#include "coarse.cuh"
#include "coarse_tc.cuh"
#include "ingest.cuh"
#include "scan.cuh"
#include "topk.cuh"
#include "ws_launch.cuh"

using namespace ivfpq;

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return set_err(IVFPQ_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),    \
                           __FILE__, __LINE__);                                                    \
    } while (0)

std::atomic<long long> g_launches{0};

// After every kernel launch: count it (ivfpq_launch_count) and check it.
#define KCHECK()                                              \
    do {                                                      \
        g_launches.fetch_add(1, std::memory_order_relaxed);   \
        CK(cudaGetLastError());                               \
    } while (0)

#define CKR(expr)                    \
    do {                             \
        int r_ = (expr);             \
        if (r_ != IVFPQ_OK) return r_; \
    } while (0)

constexpr int MAX_K = 4096;
constexpr size_t SMEM_LIMIT = 227 * 1024;
constexpr size_t COARSE_CHUNK_BYTES = 256ull << 20;

size_t lut_budget_bytes() {
    static size_t v = [] {
        const char* e = getenv("IVFPQ_LUT_BUDGET_KB");
        return (size_t)(e ? atoi(e) : 64) * 1024;
    }();
    return v;
}

// Device buffer that only grows.
struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    int ensure(size_t bytes) {
        if (bytes <= n) return IVFPQ_OK;
        if (p) {
            CK(cudaDeviceSynchronize());
            CK(cudaFree(p));
            p = nullptr;
            n = 0;
        }
        CK(cudaMalloc(&p, bytes));
        n = bytes;
        return IVFPQ_OK;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

}  // namespace

struct ivfpq_index {
    int device = 0;
    int64_t nlist = 0, nlist_local = 0, d = 0, s = 0, p = 0, sub_d = 0, s_pad = 0, n_local = 0;
    float* coarse = nullptr;     // [nlist_local, d]
    int32_t* l2g = nullptr;      // [nlist_local]
    int32_t* g2l = nullptr;      // [nlist]
    int64_t* glen = nullptr;     // [nlist]
    int64_t* off = nullptr;      // [nlist_local + 1]
    uint32_t* ids = nullptr;     // [n_local]
    uint8_t* codes = nullptr;    // [n_local * s_pad] interleaved
    float* centers = nullptr;    // [s, 2^p, sub_d]
    float* tc_img = nullptr;     // K1 tensor-core operand: swizzled centroid tiles (coarse_tc.cuh)
    float tc_cmax = 0.0f;        // max |c|
    bool tc_used = false;        // last select took the tensor-core path
    int64_t bytes = 0;
    cudaStream_t stream = nullptr;
    std::mutex mu;
    // stream ordering of calls that share the scratch below (StreamOrder)
    cudaEvent_t last_ev = nullptr;
    cudaStream_t last_stream = nullptr;
    bool last_used = false;
    // scratch
    DevBuf q, dist, pkeys, oids, odist, oshort, keys, ncand, work, plan_jobs, plan_rq, plan_nj, plan_nc, tc_sl, flags, glut,
        part;
    int64_t max_len = 0;  // longest owned list (chunked scan: partial-sum scratch per warp)
    int32_t* h_short = nullptr;  // pinned host copy of the short flags (ivfpq_search)
    int64_t h_short_cap = 0;
    int num_sms = 0;
    int64_t l2_bytes = 0;  // device L2 size (scan: bulk L2 prefetch when the code store exceeds it)
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Row-major [L, s] per list -> interleaved 32-vector blocks of 16-byte chunks:
// vector v of list c (block b = v/32, nb = min(32, L-32b)), chunk q lives at
//   (off_c + 32b) * s_pad + q * nb * 16 + (v % 32) * 16.
__global__ void interleave_codes_kernel(const uint8_t* __restrict__ src, const int64_t* __restrict__ off, int s,
                                        int s_pad, uint8_t* __restrict__ dst) {
    const int c = blockIdx.x;
    const int64_t o = off[c], L = off[c + 1] - o;
    const int nch = s_pad / 16;
    for (int64_t i = threadIdx.x; i < L * nch; i += blockDim.x) {
        const int64_t v = i / nch;
        const int q = (int)(i - v * nch);
        const int64_t vb = v & ~31LL;
        const int nb = (int)(L - vb < 32 ? L - vb : 32);
        uint8_t* out = dst + (o + vb) * s_pad + (int64_t)q * nb * 16 + (v & 31) * 16;
        const uint8_t* in = src + (o + v) * s;
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            const int j = q * 16 + b;
            out[b] = j < s ? in[j] : 0;
        }
    }
}

// qlist/qcount (optional): block b merges row b and writes it to row qlist[b], b < *qcount.
__global__ void merge_keys_kernel(const uint64_t* __restrict__ in, int W, int nq, int n_in, int n_out,
                                  uint64_t* __restrict__ out, const int* qlist = nullptr,
                                  const int* qcount = nullptr) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int nrows = qcount ? *qcount : nq;
    for (int row = blockIdx.x; row < nrows; row += gridDim.x) {
        const int orow = qlist ? qlist[row] : row;
        BlockTopK tk;
        tk.bind(smem, n_out);
        tk.init();
        const int total = W * n_in;
        for (int base = 0; base < total; base += TK_BLOCK) {
            const int i = base + threadIdx.x;
            uint64_t key = ~0ull;
            if (i < total) {
                const int w = i / n_in, j = i - w * n_in;
                key = in[((size_t)w * nq + row) * n_in + j];
            }
            tk.offer(key, key != ~0ull && key < tk.tau());
            if (base + TK_BLOCK < total) tk.maybe_merge();
        }
        tk.merge();
        for (int i = threadIdx.x; i < n_out; i += TK_BLOCK) out[(size_t)orow * n_out + i] = tk.result()[i];
        __syncthreads();
    }
}

// Merge of W ascending key runs per row ([W][nq][n_in] -> [nq][n_out]) by a
// tree of pairwise merge-paths in shared memory, one warp per row: the
// multi-GPU protocol's two merges (probe keys, top-k keys) get rows that are
// already sorted by the ranks, so no selection is needed.  Equal keys (only
// the UINT64_MAX padding) are placed by lower / upper bounds: every output
// slot is written exactly once.
constexpr int MS_WARPS = 4;
__global__ void __launch_bounds__(32 * MS_WARPS) merge_sorted_kernel(const uint64_t* __restrict__ in, int W, int nq,
                                                                     int n_in, int n_out, uint64_t* __restrict__ out) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * MS_WARPS + warp;
    if (row >= nq) return;
    const int cap = W * n_in;
    uint64_t* buf = reinterpret_cast<uint64_t*>(smem) + (size_t)warp * 2 * cap;
    uint64_t* cur = buf;
    uint64_t* nxt = buf + cap;
    for (int i = lane; i < cap; i += 32) {
        const int w = i / n_in, j = i - w * n_in;
        cur[i] = in[((size_t)w * nq + row) * n_in + j];
    }
    // runs r = 0..nr-1 of length len (the last run may be shorter after truncation)
    int nr = W, len = n_in;
    __syncwarp();
    while (nr > 1) {
        const int olen = min(2 * len, max(n_out, len));   // merged run length kept
        const int np = (nr + 1) / 2;
        for (int r = 0; r < np; ++r) {
            const uint64_t* A = cur + (size_t)(2 * r) * len;
            uint64_t* O = nxt + (size_t)r * olen;
            if (2 * r + 1 < nr) {
                const uint64_t* B = A + len;
                for (int i = lane; i < len; i += 32) {
                    const int pa = i + lower_bound_u64(B, len, A[i]);
                    if (pa < olen) O[pa] = A[i];
                    const int pb = i + upper_bound_u64(A, len, B[i]);
                    if (pb < olen) O[pb] = B[i];
                }
                for (int i = 2 * len + lane; i < olen; i += 32) O[i] = ~0ull;  // (olen <= 2 len)
            } else {
                for (int i = lane; i < olen; i += 32) O[i] = i < len ? A[i] : ~0ull;
            }
        }
        __syncwarp();
        uint64_t* t = cur;
        cur = nxt;
        nxt = t;
        nr = np;
        len = olen;
    }
    for (int i = lane; i < n_out; i += 32) out[(size_t)row * n_out + i] = i < len ? cur[i] : ~0ull;
}

__global__ void finalize_kernel(const uint64_t* __restrict__ keys, const int64_t* __restrict__ ncand, int nq, int K,
                                int64_t* __restrict__ ids, float* __restrict__ dists, int32_t* __restrict__ shrt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < (int64_t)nq * K) {
        const uint64_t key = keys[i];
        const bool empty = key == ~0ull;
        ids[i] = empty ? -1LL : (long long)(uint32_t)key;
        dists[i] = empty ? __int_as_float(0x7f800000) : __uint_as_float((uint32_t)(key >> 32));
    }
    if (i < nq) shrt[i] = ncand[i] < K ? 1 : 0;
}

__global__ void keys_to_gid_kernel(const uint64_t* __restrict__ keys, int64_t n, int64_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (long long)(uint32_t)keys[i];
}

// ---- conformance-hook kernels ------------------------------------------------
template <int DT>
__global__ void encode_kernel(const float* __restrict__ x, int64_t n, typename LutTraits<DT>::T* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = lut_store<DT>(x[i]);
}

template <int DT>
__global__ void decode_kernel(const typename LutTraits<DT>::T* __restrict__ in, int64_t n, float* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        if constexpr (DT == LUT_F16) out[i] = __half2float(__ushort_as_half(in[i]));
        else out[i] = fp8_decode_exact<LutTraits<DT>::m, LutTraits<DT>::bias>(in[i]);
    }
}

// build_lut hook: the same device routine the search kernel uses (ng = 1).
template <int DT, int LOGN>
__global__ void __launch_bounds__(TK_BLOCK) build_lut_kernel(const float* centers, int s, int sub_d, const float* rq_g,
                                                             typename LutTraits<DT>::T* out, int direct) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int d = s * sub_d;
    float* rq = reinterpret_cast<float*>(smem);
    // direct: a table larger than shared memory is written straight to `out`
    auto* lut = direct ? out : reinterpret_cast<typename LutTraits<DT>::T*>(smem + (((size_t)d * 4 + 15) & ~(size_t)15));
    for (int t = threadIdx.x; t < d; t += blockDim.x) rq[t] = rq_g[t];
    __syncthreads();
    build_luts<DT, LOGN>(lut, s << LOGN, centers, rq, d, sub_d, 1);
    if (direct) return;
    __syncthreads();
    for (int e = threadIdx.x; e < (s << LOGN); e += blockDim.x) out[e] = lut[e];
}

// scan_list hook: LUT staged in smem, one thread per vector, row-major codes
// -- the same lookup16 / lut_widen / lut_finish arithmetic as the search kernel.
template <int DT, int LOGN>
__global__ void __launch_bounds__(TK_BLOCK) scan_list_kernel(const uint8_t* codes, int64_t L, int s, const void* entries,
                                                             float* out, int direct) {
    using T = typename LutTraits<DT>::T;
    extern __shared__ __align__(16) uint8_t smem[];
    const T* g = reinterpret_cast<const T*>(entries);
    // direct: a table larger than shared memory is gathered from global memory
    T* st = reinterpret_cast<T*>(smem);
    if (!direct) {
        for (int e = threadIdx.x; e < (s << LOGN); e += blockDim.x) st[e] = g[e];
        __syncthreads();
    }
    const T* lut = direct ? g : st;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < L; v += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t* row = codes + v * s;
        float acc = 0.0f;
        for (int j0 = 0; j0 < s; j0 += 16) {
            uint32_t w[4] = {0, 0, 0, 0};
            for (int b = 0; b < 16 && j0 + b < s; ++b) w[b >> 2] |= (uint32_t)row[j0 + b] << (8 * (b & 3));
            acc = lookup16<DT, LOGN, false>(acc, make_uint4(w[0], w[1], w[2], w[3]), lut + (j0 << LOGN), s - j0);
        }
        out[v] = lut_finish<DT>(acc);
    }
}

// top_k hook: arbitrary fp32 distances -> order-preserving uint32.
__device__ __forceinline__ uint32_t f32_order(float f) {
    uint32_t b = __float_as_uint(f == 0.0f ? 0.0f : f);  // -0 == +0 as in numpy
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float f32_unorder(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}
__global__ void topk_hook_kernel(const int64_t* ids, const float* dists, int n, int K, int64_t* out_ids,
                                 float* out_d) {
    extern __shared__ __align__(16) uint8_t smem[];
    BlockTopK tk;
    tk.bind(smem, K);
    tk.init();
    for (int base = 0; base < n; base += TK_BLOCK) {
        const int i = base + threadIdx.x;
        uint64_t key = ~0ull;
        if (i < n) key = ((uint64_t)f32_order(dists[i]) << 32) | (uint32_t)ids[i];
        tk.offer(key, i < n && key < tk.tau());
        if (base + TK_BLOCK < n) tk.maybe_merge();
    }
    tk.merge();
    for (int i = threadIdx.x; i < K && i < n; i += TK_BLOCK) {
        const uint64_t key = tk.result()[i];
        out_ids[i] = (long long)(uint32_t)key;
        out_d[i] = f32_unorder((uint32_t)(key >> 32));
    }
}

// ---- dispatch -------------------------------------------------------------------
template <int DT, int LOGN>
int launch_scan_t(const ScanArgs& a, size_t smem, void* glut, int grid, cudaStream_t st) {
    CK(cudaFuncSetAttribute(scan_kernel<DT, LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_LIMIT));  // per-device: set every launch
    scan_kernel<DT, LOGN><<<grid, TK_BLOCK, smem, st>>>(a, glut);
    KCHECK();
    return IVFPQ_OK;
}

template <int DT>
int launch_scan_dt(int logn, const ScanArgs& a, size_t smem, void* glut, int grid, cudaStream_t st) {
    switch (logn) {
        case 1: return launch_scan_t<DT, 1>(a, smem, glut, grid, st);
        case 2: return launch_scan_t<DT, 2>(a, smem, glut, grid, st);
        case 3: return launch_scan_t<DT, 3>(a, smem, glut, grid, st);
        case 4: return launch_scan_t<DT, 4>(a, smem, glut, grid, st);
        case 5: return launch_scan_t<DT, 5>(a, smem, glut, grid, st);
        case 6: return launch_scan_t<DT, 6>(a, smem, glut, grid, st);
        case 7: return launch_scan_t<DT, 7>(a, smem, glut, grid, st);
        case 8: return launch_scan_t<DT, 8>(a, smem, glut, grid, st);
    }
    return set_err(IVFPQ_EINVAL, "pq_bits %d out of range 1..8", logn);
}

#define DISPATCH_DT_LOGN(dt, logn, FN, ...)                                           \
    [&]() -> int {                                                                    \
        switch (dt) {                                                                 \
            case LUT_F32: return FN<LUT_F32>(logn, __VA_ARGS__);                     \
            case LUT_F16: return FN<LUT_F16>(logn, __VA_ARGS__);                     \
            case LUT_E5M3: return FN<LUT_E5M3>(logn, __VA_ARGS__);                   \
            case LUT_E4M4: return FN<LUT_E4M4>(logn, __VA_ARGS__);                   \
        }                                                                             \
        return set_err(IVFPQ_EINVAL, "unknown LUT dtype %d", dt);                    \
    }()

int check_dtype(int dt) {
    if (dt < 0 || dt > 3) return set_err(IVFPQ_EINVAL, "unknown LUT precision code %d", dt);
    return IVFPQ_OK;
}

size_t topk_smem(int K) { return BlockTopK::smem_bytes(K); }

int set_smem_attr(const void* fn, size_t bytes) {
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    return IVFPQ_OK;
}

// `stream` is used as given: NULL is the legacy default stream, exactly as in
// the CUDA runtime (torch's default stream has handle 0).
cudaStream_t pick_stream(ivfpq_index*, void* stream) { return reinterpret_cast<cudaStream_t>(stream); }

// Every call on an index writes the index's scratch buffers (probe keys, job
// plans, LUT scratch, staging).  Calls are serialised on the host by idx->mu;
// on the device, a call issued on a different stream than the previous one
// first waits for the previous call's work (event), so scratch is never
// overwritten while an earlier call's kernels still read it.
struct StreamOrder {
    ivfpq_index* idx;
    cudaStream_t st;
    StreamOrder(ivfpq_index* i, cudaStream_t s) : idx(i), st(s) {
        if (idx->last_used && idx->last_stream != st) cudaStreamWaitEvent(st, idx->last_ev, 0);
    }
    ~StreamOrder() {
        cudaEventRecord(idx->last_ev, st);
        idx->last_stream = st;
        idx->last_used = true;
    }
};

// 0 = auto (tensor-core K1 when the shape fits), 1 = SIMT only, 2 = tensor
// core with every query re-done by the exact fallback (tests the fallback);
// set by ivfpq_set_select_kernel or IVFPQ_SELECT_SIMT=1.
std::atomic<int> g_select_mode{-1};

int select_mode() {
    int m = g_select_mode.load();
    if (m < 0) {
        const char* e = getenv("IVFPQ_SELECT_SIMT");
        m = (e && atoi(e) != 0) ? 1 : 0;
        g_select_mode.store(m);
    }
    return m;
}

int launch_coarse_topk(ivfpq_index* idx, const float* d_q, int64_t nq, int64_t P, int64_t nsl, int64_t slice,
                       uint64_t* out, const int* qlist, const int* qcount, cudaStream_t st, int64_t max_qblocks = 0) {
    CKR(set_smem_attr((const void*)coarse_topk_kernel, SMEM_LIMIT - 10 * 1024));  // per-device: set every launch
    CoarseTopkArgs ca{d_q, idx->coarse, idx->l2g, out, (int)nq, (int)idx->nlist_local, (int)idx->d, (int)P, (int)slice};
    ca.qlist = qlist;
    ca.qcount = qcount;
    int64_t qblocks = (nq + CT_BQ - 1) / CT_BQ;
    if (max_qblocks > 0) qblocks = std::min(qblocks, max_qblocks);
    coarse_topk_kernel<<<dim3((unsigned)nsl, (unsigned)qblocks), 256, coarse_topk_smem((int)P, (int)idx->d), st>>>(ca);
    KCHECK();
    return IVFPQ_OK;
}

int launch_merge(const uint64_t* in, int64_t W, int64_t nq, int64_t P, uint64_t* out, const int* qlist,
                 const int* qcount, cudaStream_t st, int64_t max_blocks = 0) {
    CKR(set_smem_attr((const void*)merge_keys_kernel, SMEM_LIMIT));  // per-device: set every launch
    const int64_t blocks = max_blocks > 0 ? std::min(nq, max_blocks) : nq;
    merge_keys_kernel<<<(unsigned)blocks, TK_BLOCK, topk_smem((int)P), st>>>(in, (int)W, (int)nq, (int)P, (int)P, out,
                                                                           qlist, qcount);
    KCHECK();
    return IVFPQ_OK;
}

// Tensor-core K1 (coarse_tc.cuh): TF32 GEMM + shortlist, exact re-rank + guard,
// exact SIMT re-do of the (rare) queries whose guard failed.
int run_select_tc(ivfpq_index* idx, const float* d_q, int64_t nq, int64_t P, uint64_t* d_keys, cudaStream_t st) {
    const int64_t nc = idx->nlist_local, d = idx->d;
    const int64_t ntiles = (nc + TC_N - 1) / TC_N, nkc = coarse_tc_nkc((int)d);
    const int64_t qblocks = (nq + TC_M - 1) / TC_M;
    // slices: fill the SMs; large nprobe needs ceil(P / 32) slices so each
    // slice's ~48..90 nominations cover its share of the top-P with margin
    // (else the guard would send the query to the exact re-do)
    const int64_t nsl_p = std::min<int64_t>(TC_MAXSL, (P + TC_P_PER_SLICE - 1) / TC_P_PER_SLICE);
    const int64_t nsl = std::max<int64_t>(
        1, std::min<int64_t>(ntiles, std::max<int64_t>(nsl_p, std::min<int64_t>(TC_MAXSL, idx->num_sms / qblocks))));
    const int64_t tps = (ntiles + nsl - 1) / nsl;
    const size_t rows = (size_t)nsl * nq;
    CKR(idx->tc_sl.ensure(rows * TC_CAP * 4 + rows * 8));
    int32_t* cand = idx->tc_sl.as<int32_t>();
    int32_t* ncand = cand + rows * TC_CAP;
    float* thr = reinterpret_cast<float*>(ncand + rows);
    CKR(idx->flags.ensure((size_t)(nq + 1) * 4));
    int* fcount = idx->flags.as<int>();
    int* flist = fcount + 1;
    CK(cudaMemsetAsync(fcount, 0, sizeof(int), st));
    idx->tc_used = true;
    // dynamic-smem attributes are per device context: set before every launch
    CKR(set_smem_attr((const void*)coarse_tc_kernel, coarse_tc_smem(TC_MAXD)));
    CoarseTcArgs ta{d_q, idx->tc_img, cand, ncand, thr, (int)nq, (int)nc, (int)d, (int)tps, (int)nkc};
    coarse_tc_kernel<<<dim3((unsigned)nsl, (unsigned)qblocks), TC_THREADS, coarse_tc_smem((int)d), st>>>(ta);
    KCHECK();
    CoarseRerankArgs ra{d_q, idx->coarse, idx->l2g, cand, ncand, thr, d_keys, fcount, flist, idx->tc_cmax,
                        (int)nq, (int)nc, (int)d, (int)P, (int)nsl, select_mode() == 2};
    coarse_rerank_kernel<<<(unsigned)((nq + TC_RR_WARPS - 1) / TC_RR_WARPS), 32 * TC_RR_WARPS,
                           coarse_rerank_smem((int)nsl, (int)d), st>>>(ra);
    KCHECK();
    // exact re-do of flagged queries: grid-stride over the device-side list
    // (blocks past *fcount exit at once; no host round trip)
    CKR(set_smem_attr((const void*)coarse_redo_kernel, SMEM_LIMIT));
    coarse_redo_kernel<<<(unsigned)std::min<int64_t>(nq, 2 * idx->num_sms), TK_BLOCK,
                         coarse_redo_smem((int)P, (int)d), st>>>(d_q, idx->coarse, idx->l2g, (int)nc, (int)d, (int)P,
                                                                fcount, flist, d_keys);
    KCHECK();
    return IVFPQ_OK;
}

// K1 over the owned centroids: keys [nq, P] (ascending d2, then global id).
// P <= CT_MAXP: fused exact distance + top-P kernel over centroid slices,
// slices merged by merge_keys_kernel.  Larger P: distance tiles + block select.
int run_select(ivfpq_index* idx, const float* d_q, int64_t nq, int64_t P, uint64_t* d_keys, cudaStream_t st) {
    const int64_t nc = idx->nlist_local;
    if (P > MAX_K) return set_err(IVFPQ_EUNSUPPORTED, "nprobe=%lld exceeds the device limit %d", (long long)P, MAX_K);
    if (nq <= 0) return IVFPQ_OK;
    if (nc == 0) {
        CK(cudaMemsetAsync(d_keys, 0xff, (size_t)nq * P * 8, st));
        return IVFPQ_OK;
    }
    const int smode = select_mode();
    idx->tc_used = false;
    if (idx->tc_img && smode != 1 && P <= TC_MAXP && nc >= 2 * TC_N &&
        coarse_topk_smem((int)P, (int)idx->d) <= SMEM_LIMIT - 24 * 1024)
        return run_select_tc(idx, d_q, nq, P, d_keys, st);
    if (P <= CT_MAXP && coarse_topk_smem((int)P, (int)idx->d) <= SMEM_LIMIT - 24 * 1024) {
        // slices: ~CT_WAVES CTAs per SM in flight, each slice >= 256 centroids
        const int64_t qblocks = (nq + CT_BQ - 1) / CT_BQ;
        static const int waves = [] {
            const char* e = getenv("IVFPQ_CT_WAVES");
            return e ? atoi(e) : 6;
        }();
        int64_t nsl = std::max<int64_t>(1, std::min<int64_t>((waves * idx->num_sms + qblocks - 1) / qblocks, nc / 256));
        int64_t slice = ((nc + nsl - 1) / nsl + CT_BC - 1) / CT_BC * CT_BC;
        nsl = (nc + slice - 1) / slice;
        uint64_t* out = d_keys;
        if (nsl > 1) {
            CKR(idx->dist.ensure((size_t)nsl * nq * P * 8));
            out = reinterpret_cast<uint64_t*>(idx->dist.p);
        }
        CKR(launch_coarse_topk(idx, d_q, nq, P, nsl, slice, out, nullptr, nullptr, st));
        if (nsl > 1) CKR(launch_merge(out, nsl, nq, P, d_keys, nullptr, nullptr, st));
        return IVFPQ_OK;
    }
    int64_t rows = std::max<int64_t>(1, std::min<int64_t>(nq, (int64_t)(COARSE_CHUNK_BYTES / (nc * 4))));
    CKR(idx->dist.ensure((size_t)rows * nc * 4));
    const size_t sm = topk_smem((int)P);
    CKR(set_smem_attr((const void*)select_probes_kernel, SMEM_LIMIT));  // per-device: set every launch
    for (int64_t r0 = 0; r0 < nq; r0 += rows) {
        const int64_t nr = std::min(rows, nq - r0);
        dim3 grid((unsigned)((nc + CL_BC - 1) / CL_BC), (unsigned)((nr + CL_BQ - 1) / CL_BQ));
        coarse_l2_kernel<<<grid, 256, 0, st>>>(d_q + r0 * idx->d, (int)nr, idx->coarse, (int)nc, (int)idx->d,
                                                idx->dist.as<float>());
        KCHECK();
        select_probes_kernel<<<(unsigned)nr, TK_BLOCK, sm, st>>>(idx->dist.as<float>(), (int)nc, idx->l2g, (int)P,
                                                                 d_keys + r0 * P);
        KCHECK();
    }
    return IVFPQ_OK;
}

struct WsPlan {
    int G, NBUF;
    size_t smem;
    int gmem;
    int nh = 1, rc = 0;  // row-chunked LUT jobs: nh chunks of rc rows (nh = 1: unchunked)
};

// 0 = auto (v2 when the shape fits), 1 = force v1; set by ivfpq_set_scan_kernel
// or the IVFPQ_SCAN_V1 environment variable.
std::atomic<int> g_scan_mode{-1};

bool ws_disabled() {
    int m = g_scan_mode.load();
    if (m < 0) {
        const char* e = getenv("IVFPQ_SCAN_V1");
        m = (e && atoi(e) != 0) ? 1 : 0;
        g_scan_mode.store(m);
    }
    return m == 1;
}

// Can the v2 kernel run this shape?  Builder registers: ceil(s / R) subspaces
// of a 4-code quad, R = 1024 / 2^p row groups, at most 32 / sub_d of them.
template <class C>
bool ws_plan(const ivfpq_index* idx, int64_t P, int64_t K, int dt, WsPlan* plan) {
    if (ws_disabled() || idx->num_sms <= 0) return false;
    const int64_t N = 1LL << idx->p;
    if (idx->p < 2 || idx->sub_d < 1 || idx->sub_d > 4 || K > WS_MAX_K) return false;
    const int64_t R = C::R((int)N);
    const int64_t jpt = C::JPT((int)idx->sub_d);
    // rows per builder thread beyond the TMEM budget: codebook read from global
    const bool gmem = (idx->s_pad + R - 1) / R > jpt;
    const size_t lut_each = WsLayout<C>((int)idx->d, (int)idx->s, (int)idx->sub_d, (int)idx->p, lut_bytes_of((int)dt), 1,
                                     2, (int)K, (int)idx->s_pad).lut_each;
    int G = (int)std::max<size_t>(1, std::min<size_t>(WS_MAX_G, lut_budget_bytes() / lut_each));
    G = (int)std::min<int64_t>(G, std::max<int64_t>(1, P));
    static const int env_nb = [] {
        const char* e = getenv("IVFPQ_WS_NBUF");
        return e ? atoi(e) : 0;
    }();
    const int G0 = G;
    const int esz = lut_bytes_of((int)dt);
    auto fits = [&](int g, int nb, int rc) {
        return WsLayout<C>((int)idx->d, (int)idx->s, (int)idx->sub_d, (int)idx->p, esz, g, nb, (int)K, (int)idx->s_pad, rc)
            .total;
    };
    // unchunked: the largest G with >= min_nb LUT slots
    auto unchunked = [&](int min_nb, int min_g) -> bool {
        for (int g = G0; g >= min_g; --g)
            for (int nb = env_nb ? env_nb : WS_MAX_NBUF; nb >= min_nb; --nb)
                if (fits(g, nb, 0) <= SMEM_LIMIT) {
                    *plan = WsPlan{g, nb, fits(g, nb, 0), gmem ? 1 : 0};
                    return true;
                }
        return false;
    };
    // row-chunked: rc rows per job (a multiple of 16 -- whole code chunks --
    // and of R -- whole builder rows -- dividing s_pad), the largest rc and
    // then G with >= min_nb slots; the lists' partial sums are carried in a
    // per-warp scratch between the nh = s_pad / rc jobs of a group
    auto chunked = [&](int min_nb, int min_g) -> bool {
        if (idx->p < 5) return false;  // (row-chunked kernels are built for 2^p >= 32)
        const int64_t step = std::max<int64_t>(16, R) % 16 == 0 ? std::max<int64_t>(16, R) : 16 * R;
        for (int64_t rc = idx->s_pad - step; rc >= step; rc -= step) {
            if (idx->s_pad % rc) continue;
            const size_t le = WsLayout<C>((int)idx->d, (int)idx->s, (int)idx->sub_d, (int)idx->p, esz, 1, 1, (int)K,
                                       (int)idx->s_pad, (int)rc).lut_each;
            const int g0 = (int)std::min<int64_t>(std::min<size_t>(WS_MAX_G, std::max<size_t>(1, lut_budget_bytes() / le)),
                                                  std::max<int64_t>(1, P));
            for (int g = g0; g >= min_g; --g)
                for (int nb = WS_MAX_NBUF; nb >= min_nb; --nb)
                    if (fits(g, nb, (int)rc) <= SMEM_LIMIT) {
                        *plan = WsPlan{g, nb, fits(g, nb, (int)rc), gmem ? 1 : 0, (int)(idx->s_pad / rc), (int)rc};
                        return true;
                    }
        }
        return false;
    };
    // Preference (measured): >= 3 LUT slots (builders and scanners decoupled by
    // a job of slack) with G >= 2 (cfg2), then fewer slots down to one (cfg3 p8
    // f16, 120 KiB: one slot 107 ms vs row chunks 127 ms); a table larger than
    // shared memory is row-chunked, the largest chunk first (cfg3 p8 f32:
    // 48-row chunks 145 ms, 16-row chunks x 4 lists 178 ms, the per-query
    // kernel with a global-memory table ~275 ms).  Scan mode 2 prefers chunks.
    if (g_scan_mode.load() == 2 && chunked(3, 1)) return true;
    return unchunked(3, 2) || unchunked(3, 1) || unchunked(2, 1) || unchunked(1, 1) || chunked(3, 1) || chunked(2, 1) ||
           chunked(1, 1);
}

// Shapes the layout-B kernels are built for (ws_launch.cuh): cfg4 (p 8, sub_d 2,
// s 48), cfg5 (p 8, sub_d 3, s 32), cfg3 p5 (p 5, sub_d 4, s 240), codebook in
// TMEM.  (cfg3 p8 on layout B, codebook in global memory: 81.2 ms vs 78.8 on
// A -- its 4 builder warps become the bottleneck; profiles/r02_scan_experiments.txt.)
bool ws_layout_b_supported(const ivfpq_index* idx) {
    const int64_t nch = idx->s_pad / 16;
    if (idx->s_pad > WsCfgB::R((int)(1 << idx->p)) * WsCfgB::JPT((int)idx->sub_d)) return false;  // not TMEM
    return (idx->p == 8 && idx->sub_d == 2 && nch == 3) || (idx->p == 8 && idx->sub_d == 3 && nch == 2) ||
           (idx->p == 5 && idx->sub_d == 4 && nch == 15);
}

// Plan + launch of the persistent scan kernel with warp layout C; *done =
// false when the shape cannot be planned or the build has no kernel for it.
template <class C>
int run_scan_ws(ivfpq_index* idx, ScanArgs a, int64_t nq, int64_t P, int64_t K, int dt, cudaStream_t st, int layout,
                bool* done) {
    *done = false;
    WsPlan plan;
    if (!ws_plan<C>(idx, P, K, dt, &plan)) return IVFPQ_OK;
    if (layout == 1 && plan.nh > 1) return IVFPQ_OK;
    a.G = plan.G;
    WsArgs w;
    w.a = a;
    w.NBUF = plan.NBUF;
    w.gmem = plan.gmem;
    // code store larger than L2: builders prefetch each job's start; the
    // scanners prefetch ahead of their grabs in layout B (IVFPQ_WS_SPF=0
    // turns the scanner part off, for measurements; the layout-A kernels are
    // built without it: measured no gain at cfg3 p8 / cfg4)
    static const int env_spf = [] {
        const char* e = getenv("IVFPQ_WS_SPF");
        return e ? atoi(e) : -1;
    }();
    const bool spf = env_spf >= 0 ? env_spf != 0 : C::SCAN_PF;
    w.l2pf = (int64_t)idx->n_local * idx->s_pad > idx->l2_bytes ? (1 | (spf ? 2 : 0)) : 0;
    w.n_codes_bytes = (long long)idx->n_local * idx->s_pad;
    w.nqs = ws_nqs((int)K);
    w.wsz = ws_wsz((int)K);
    w.nh = plan.nh;
    w.rc = plan.nh > 1 ? plan.rc : 0;
    w.rcc = (int)(plan.nh > 1 ? plan.rc / 16 : idx->s_pad / 16);
    w.maxp = 0;
    w.part = nullptr;
    CKR(idx->work.ensure(16));
    w.work = idx->work.as<int>();
    CK(cudaMemsetAsync(w.work, 0, sizeof(int), st));
    // plan: job descriptors + residual rows per query
    const WsLayout<C> lay((int)idx->d, (int)idx->s, (int)idx->sub_d, (int)idx->p, lut_bytes_of(dt), plan.G, plan.NBUF,
                       (int)K, (int)idx->s_pad, w.rc);
    const int d_pad = (int)lay.d_pad;
    const int JMAX = (int)std::max<int64_t>(1, (P + plan.G - 1) / plan.G) * plan.nh;
    const int grid = std::min<int64_t>(idx->num_sms, nq);
    if (plan.nh > 1) {
        // pairs one scanner warp owns in a job: ceil(ceil(blocks / 2) / SW),
        // blocks <= G * ceil(longest list / 32)
        const int64_t blocks = (int64_t)plan.G * ((idx->max_len + 31) / 32);
        w.maxp = (int)std::max<int64_t>(1, ((blocks + 1) / 2 + C::SW - 1) / C::SW);
        CKR(idx->part.ensure((size_t)grid * C::SW * w.maxp * 64 * 4));
        w.part = idx->part.as<float>();
    }
    CKR(idx->plan_jobs.ensure((size_t)nq * JMAX * sizeof(WsJob)));
    CKR(idx->plan_rq.ensure((size_t)nq * JMAX * plan.G * d_pad * 4));
    CKR(idx->plan_nj.ensure((size_t)nq * 4));
    CKR(idx->plan_nc.ensure((size_t)nq * 8));
    w.plan_jobs = idx->plan_jobs.as<WsJob>();
    w.plan_rq = idx->plan_rq.as<float>();
    w.plan_njobs = idx->plan_nj.as<int>();
    w.plan_ncand = idx->plan_nc.as<long long>();
    w.JMAX = JMAX;
    ws_plan_kernel<<<(unsigned)((nq + 7) / 8), 256, 0, st>>>(a, plan.G, d_pad, JMAX, plan.nh,
                                                               idx->plan_jobs.as<WsJob>(),
                                                               idx->plan_rq.as<float>(), idx->plan_nj.as<int>(),
                                                               idx->plan_nc.as<long long>());
    KCHECK();
    cudaError_t e = cudaErrorInvalidValue;
    switch (dt) {
        case LUT_F32: e = ws_launch_f32(layout, (int)idx->p, (int)idx->sub_d, w, plan.smem, grid, st); break;
        case LUT_F16: e = ws_launch_f16(layout, (int)idx->p, (int)idx->sub_d, w, plan.smem, grid, st); break;
        case LUT_E5M3: e = ws_launch_e5m3(layout, (int)idx->p, (int)idx->sub_d, w, plan.smem, grid, st); break;
        case LUT_E4M4: e = ws_launch_e4m4(layout, (int)idx->p, (int)idx->sub_d, w, plan.smem, grid, st); break;
    }
    if (e == cudaSuccess) {
        g_launches.fetch_add(1, std::memory_order_relaxed);
        *done = true;
        return IVFPQ_OK;
    }
    if (e != cudaErrorNotSupported)
        return set_err(IVFPQ_ECUDA, "scan_ws launch failed: %s", cudaGetErrorString(e));
    return IVFPQ_OK;  // no kernel for this shape in this build: the caller falls back
}

int run_scan(ivfpq_index* idx, const float* d_q, int64_t nq, const uint64_t* d_pk, int64_t P, int64_t K, int dt,
             uint64_t* out_keys, int64_t* out_ncand, int64_t* out_ids, float* out_d, int32_t* out_short,
             cudaStream_t st) {
    if (K > MAX_K) return set_err(IVFPQ_EUNSUPPORTED, "k=%lld exceeds the device limit %d", (long long)K, MAX_K);
    CKR(check_dtype(dt));
    const size_t lut_each = (size_t)(idx->s << idx->p) * lut_bytes_of(dt);
    const size_t fixed = ScanSmemLayout((int)idx->d, 1, 0, (int)K).total;
    if (fixed > SMEM_LIMIT)
        return set_err(IVFPQ_EUNSUPPORTED, "d=%lld, k=%lld: scan state does not fit shared memory", (long long)idx->d,
                       (long long)K);
    // A table larger than shared memory (f32 LUT at s=240, p=8) is built in a
    // per-block global scratch; the per-query kernel then strides over the
    // queries with a bounded grid.  (Only reachable when v2 cannot plan it.)
    const bool glut = fixed + lut_each > SMEM_LIMIT;
    int G = glut ? 1 : (int)std::max<size_t>(1, std::min<size_t>(SCAN_MAX_G, lut_budget_bytes() / lut_each));
    G = (int)std::min<int64_t>(G, std::max<int64_t>(1, P));
    while (G > 1 && ScanSmemLayout((int)idx->d, G, lut_each, (int)K).total > SMEM_LIMIT) --G;
    const size_t smem = ScanSmemLayout((int)idx->d, G, glut ? 0 : lut_each, (int)K).total;
    int grid = (int)std::max<int64_t>(nq, 1);
    void* glut_p = nullptr;
    if (glut) {
        grid = (int)std::min<int64_t>(grid, (int64_t)std::max(idx->num_sms, 1) * 4);
        CKR(idx->glut.ensure((size_t)grid * lut_each));
        glut_p = idx->glut.p;
    }
    ScanArgs a;
    a.queries = d_q;
    a.probes = d_pk;
    a.coarse = idx->coarse;
    a.g2l = idx->g2l;
    a.glen = idx->glen;
    a.off = idx->off;
    a.ids = idx->ids;
    a.codes = idx->codes;
    a.centers = idx->centers;
    a.nq = (int)nq;
    a.d = (int)idx->d;
    a.P = (int)P;
    a.s = (int)idx->s;
    a.sub_d = (int)idx->sub_d;
    a.s_pad = (int)idx->s_pad;
    a.K = (int)K;
    a.G = G;
    a.out_keys = out_keys;
    a.out_ncand = out_ncand;
    a.out_ids = out_ids;
    a.out_dists = out_d;
    a.out_short = out_short;
    if (nq == 0) return IVFPQ_OK;
    // v2 (persistent, warp-specialised, codebook in tensor memory) when the
    // shape fits its register/smem budget; v1 otherwise.  Layout B (4 builder +
    // 15 scanner warps) for scan-heavy shapes (>= 4 lookups per LUT entry on
    // average: cfg5 ~6, cfg3 p5 ~7.6), layout A (8 + 11) otherwise.  Measured
    // (scan ms, e5m3, A -> B): cfg5 48.4 -> 40.2, cfg3 p5 46.7 -> 38.6, but
    // cfg4 (2.4 per entry, k = 100) 11.7 -> 13.2.
    const int mode = g_scan_mode.load();
    const double per_entry = (double)idx->n_local / (double)std::max<int64_t>(1, idx->nlist_local) / (double)(1 << idx->p);
    const bool want_b = mode == 4 || (mode == 0 && per_entry >= 4.0);
    if (want_b && ws_layout_b_supported(idx)) {
        bool done = false;
        CKR(run_scan_ws<WsCfgB>(idx, a, nq, P, K, dt, st, 1, &done));
        if (done) return IVFPQ_OK;
    }
    {
        bool done = false;
        CKR(run_scan_ws<WsCfgA>(idx, a, nq, P, K, dt, st, 0, &done));
        if (done) return IVFPQ_OK;
    }
    return DISPATCH_DT_LOGN(dt, (int)idx->p, launch_scan_dt, a, smem, glut_p, grid, st);
}

int validate_search(ivfpq_index* idx, int64_t nq, int64_t k, int64_t nprobe, int dt) {
    if (!idx) return set_err(IVFPQ_EINVAL, "null index");
    if (nq < 0) return set_err(IVFPQ_EINVAL, "nq must be >= 0");
    if (k < 1) return set_err(IVFPQ_EINVAL, "k must be at least 1");
    if (nprobe < 1 || nprobe > idx->nlist)
        return set_err(IVFPQ_EINVAL, "nprobe=%lld out of range 1..%lld", (long long)nprobe, (long long)idx->nlist);
    if (k > MAX_K) return set_err(IVFPQ_EUNSUPPORTED, "k=%lld exceeds the device limit %d", (long long)k, MAX_K);
    if (nprobe > MAX_K)
        return set_err(IVFPQ_EUNSUPPORTED, "nprobe=%lld exceeds the device limit %d", (long long)nprobe, MAX_K);
    return check_dtype(dt);
}

int search_device_impl(ivfpq_index* idx, const float* d_q, int64_t nq, int64_t k, int64_t nprobe, int dt,
                       int64_t* d_ids, float* d_d, int32_t* d_short, cudaStream_t st) {
    CKR(idx->pkeys.ensure((size_t)std::max<int64_t>(nq, 1) * nprobe * 8));
    CKR(run_select(idx, d_q, nq, nprobe, idx->pkeys.as<uint64_t>(), st));
    return run_scan(idx, d_q, nq, idx->pkeys.as<uint64_t>(), nprobe, k, dt, nullptr, nullptr, d_ids, d_d, d_short, st);
}

unsigned blocks_for(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

}  // namespace

// =============================================================================
extern "C" {

const char* ivfpq_last_error(void) { return g_err.c_str(); }
int ivfpq_version(void) { return 1; }
int ivfpq_max_k(void) { return MAX_K; }

int ivfpq_set_select_kernel(int mode) {
    if (mode < 0 || mode > 2)
        return set_err(IVFPQ_EINVAL, "select kernel mode must be 0 (auto), 1 (SIMT) or 2 (tensor core, all re-done)");
    g_select_mode.store(mode);
    return IVFPQ_OK;
}

int ivfpq_set_scan_kernel(int mode) {
    if (mode < 0 || mode > 4)
        return set_err(IVFPQ_EINVAL,
                       "scan kernel mode must be 0 (auto), 1 (v1), 2 (prefer row-chunked LUT jobs), 3 (warp layout A "
                       "only) or 4 (warp layout B where built)");
    g_scan_mode.store(mode);
    return IVFPQ_OK;
}

// Debug: queries of the last tensor-core K1 on this index whose guard failed
// (re-done by the exact kernel); -1 if the last select did not use it.
int ivfpq_debug_select_flagged(ivfpq_index* idx, int64_t* out) {
    if (!idx || !out) return set_err(IVFPQ_EINVAL, "null argument");
    DeviceGuard guard(idx->device);
    int n = -1;
    if (idx->tc_used) {
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(&n, idx->flags.p, sizeof(int), cudaMemcpyDeviceToHost));
    }
    *out = n;
    return IVFPQ_OK;
}

// Debug: copy the per-warp cycle counters of the last profiled launch.

int ivfpq_launch_count(int64_t* out) {
    if (!out) return set_err(IVFPQ_EINVAL, "null argument");
    *out = g_launches.load();
    return IVFPQ_OK;
}

int ivfpq_device_count(int* n) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        cudaGetLastError();
        c = 0;
    }
    *n = c;
    return IVFPQ_OK;
}

int ivfpq_index_create(int device, const float* coarse, int64_t nlist, int64_t d, const float* centers, int64_t s,
                       int64_t p, const int64_t* list_off, const int64_t* ids, const uint8_t* codes,
                       const int32_t* owned, int64_t n_owned, ivfpq_index** out) {
    if (!out) return set_err(IVFPQ_EINVAL, "null output handle");
    *out = nullptr;
    if (nlist < 1 || d < 1 || s < 1 || p < 1 || p > 8 || d % s != 0)
        return set_err(IVFPQ_EINVAL, "invalid index shape nlist=%lld d=%lld s=%lld p=%lld", (long long)nlist,
                       (long long)d, (long long)s, (long long)p);
    if (nlist >= (1LL << 31) - 1) return set_err(IVFPQ_EUNSUPPORTED, "nlist too large");
    const int64_t N = list_off[nlist];
    if (list_off[0] != 0) return set_err(IVFPQ_EINVAL, "list_off[0] must be 0");
    for (int64_t c = 0; c < nlist; ++c)
        if (list_off[c + 1] < list_off[c]) return set_err(IVFPQ_EINVAL, "list_off must be non-decreasing");
    std::vector<int32_t> own;
    if (owned) {
        own.assign(owned, owned + n_owned);
        for (int32_t c : own)
            if (c < 0 || c >= nlist) return set_err(IVFPQ_EINVAL, "owned list %d out of range", c);
        std::sort(own.begin(), own.end());
        own.erase(std::unique(own.begin(), own.end()), own.end());
    } else {
        own.resize(nlist);
        for (int64_t c = 0; c < nlist; ++c) own[c] = (int32_t)c;
    }
    const int64_t sub_d = d / s, n_codes = 1LL << p, s_pad = (s + 15) & ~15LL;
    const int64_t nl = (int64_t)own.size();

    // gather the owned lists (host staging)
    std::vector<int64_t> off(nl + 1, 0);
    for (int64_t i = 0; i < nl; ++i) off[i + 1] = off[i] + (list_off[own[i] + 1] - list_off[own[i]]);
    const int64_t n_local = off[nl];
    std::vector<uint32_t> hid(n_local);
    std::vector<uint8_t> hcodes((size_t)n_local * s);
    std::vector<float> hco((size_t)nl * d);
    std::vector<int32_t> l2g(nl), g2l(nlist, -1);
    std::vector<int64_t> glen(nlist);
    for (int64_t c = 0; c < nlist; ++c) glen[c] = list_off[c + 1] - list_off[c];
    for (int64_t i = 0; i < nl; ++i) {
        const int64_t c = own[i], lo = list_off[c], L = list_off[c + 1] - lo;
        l2g[i] = (int32_t)c;
        g2l[c] = (int32_t)i;
        memcpy(&hco[(size_t)i * d], coarse + (size_t)c * d, sizeof(float) * d);
        for (int64_t v = 0; v < L; ++v) {
            const int64_t id = ids[lo + v];
            if (id < 0 || id >= 0xffffffffLL) return set_err(IVFPQ_EUNSUPPORTED, "id %lld outside [0, 2^32-1)", (long long)id);
            hid[off[i] + v] = (uint32_t)id;
        }
        const uint8_t* src = codes + (size_t)lo * s;
        for (int64_t b = 0; b < L * s; ++b)
            if (src[b] >= n_codes) return set_err(IVFPQ_EINVAL, "code byte out of range for p=%lld", (long long)p);
        memcpy(&hcodes[(size_t)off[i] * s], src, (size_t)L * s);
    }
    (void)N;

    DeviceGuard guard(device);
    CK(cudaSetDevice(device));
    ivfpq_index* idx = new ivfpq_index();
    idx->device = device;
    idx->nlist = nlist;
    idx->nlist_local = nl;
    idx->d = d;
    idx->s = s;
    idx->p = p;
    idx->sub_d = sub_d;
    idx->s_pad = s_pad;
    idx->n_local = n_local;
    for (int64_t i = 0; i < nl; ++i) idx->max_len = std::max<int64_t>(idx->max_len, off[i + 1] - off[i]);
    auto fail = [&](int rc) {
        ivfpq_index_destroy(idx);
        return rc;
    };
#define CKI(call)                                                                                       \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess)                                                                          \
            return fail(set_err(IVFPQ_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_)));          \
    } while (0)
    CKI(cudaStreamCreateWithFlags(&idx->stream, cudaStreamNonBlocking));
    CKI(cudaEventCreateWithFlags(&idx->last_ev, cudaEventDisableTiming));
    CKI(cudaDeviceGetAttribute(&idx->num_sms, cudaDevAttrMultiProcessorCount, device));
    {
        int l2 = 0;
        CKI(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device));
        idx->l2_bytes = l2;
    }
    auto up = [&](void** dst, const void* src, size_t bytes) -> cudaError_t {
        cudaError_t e = cudaMalloc(dst, std::max<size_t>(bytes, 16));
        if (e != cudaSuccess) return e;
        idx->bytes += (int64_t)bytes;
        return bytes ? cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) : cudaSuccess;
    };
    CKI(up((void**)&idx->coarse, hco.data(), hco.size() * 4));
    CKI(up((void**)&idx->l2g, l2g.data(), l2g.size() * 4));
    CKI(up((void**)&idx->g2l, g2l.data(), g2l.size() * 4));
    CKI(up((void**)&idx->glen, glen.data(), glen.size() * 8));
    CKI(up((void**)&idx->off, off.data(), off.size() * 8));
    CKI(up((void**)&idx->ids, hid.data(), hid.size() * 4));
    CKI(up((void**)&idx->centers, centers, (size_t)s * n_codes * sub_d * 4));
    uint8_t* rowmajor = nullptr;
    CKI(up((void**)&rowmajor, hcodes.data(), hcodes.size()));
    CKI(cudaMalloc((void**)&idx->codes, std::max<size_t>((size_t)n_local * s_pad, 16)));
    idx->bytes += n_local * s_pad - (int64_t)hcodes.size();
    if (nl > 0) {
        interleave_codes_kernel<<<(unsigned)nl, 256, 0, idx->stream>>>(rowmajor, idx->off, (int)s, (int)s_pad,
                                                                       idx->codes);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        CKI(cudaGetLastError());
    }
    if (nl > 0 && d <= TC_MAXD) {
        // operand images for the tensor-core K1 (built once per index)
        const int64_t ntiles = (nl + TC_N - 1) / TC_N, nkc = coarse_tc_nkc((int)d);
        const size_t ib = (size_t)ntiles * nkc * TC_N * 128;
        CKI(cudaMalloc((void**)&idx->tc_img, ib));
        idx->bytes += (int64_t)ib;
        coarse_tc_prep_kernel<<<(unsigned)ntiles, 256, 0, idx->stream>>>(idx->coarse, (int)nl, (int)d, (int)nkc,
                                                                         idx->tc_img);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        CKI(cudaGetLastError());
        idx->tc_cmax = coarse_tc_cmax(hco.data(), nl, d);
    }
    CKI(cudaStreamSynchronize(idx->stream));
    cudaFree(rowmajor);
#undef CKI
    *out = idx;
    return IVFPQ_OK;
}

int ivfpq_index_destroy(ivfpq_index* idx) {
    if (!idx) return IVFPQ_OK;
    DeviceGuard guard(idx->device);
    if (idx->stream) cudaStreamSynchronize(idx->stream);
    void* ptrs[] = {idx->coarse, idx->l2g, idx->g2l, idx->glen, idx->off, idx->ids, idx->codes, idx->centers,
                    idx->tc_img};
    for (void* ptr : ptrs)
        if (ptr) cudaFree(ptr);
    for (DevBuf* b : {&idx->glut, &idx->part, &idx->q, &idx->dist, &idx->pkeys, &idx->oids, &idx->odist, &idx->oshort, &idx->keys, &idx->ncand,
                      &idx->work, &idx->plan_jobs, &idx->plan_rq, &idx->plan_nj, &idx->plan_nc, &idx->tc_sl,
                      &idx->flags})
        b->release();
    if (idx->stream) cudaStreamDestroy(idx->stream);
    if (idx->last_ev) cudaEventDestroy(idx->last_ev);
    if (idx->h_short) cudaFreeHost(idx->h_short);
    delete idx;
    return IVFPQ_OK;
}

int ivfpq_index_bytes(const ivfpq_index* idx, int64_t* bytes) {
    if (!idx || !bytes) return set_err(IVFPQ_EINVAL, "null argument");
    *bytes = idx->bytes;
    return IVFPQ_OK;
}

int ivfpq_search(ivfpq_index* idx, const float* queries, int64_t nq, int64_t k, int64_t nprobe, int dt,
                 int64_t* out_ids, float* out_dists, int64_t* out_n_short) {
    CKR(validate_search(idx, nq, k, nprobe, dt));
    std::lock_guard<std::mutex> lock(idx->mu);
    DeviceGuard guard(idx->device);
    cudaStream_t st = idx->stream;
    StreamOrder order(idx, st);
    const int64_t nq1 = std::max<int64_t>(nq, 1);
    CKR(idx->q.ensure((size_t)nq1 * idx->d * 4));
    CKR(idx->oids.ensure((size_t)nq1 * k * 8));
    CKR(idx->odist.ensure((size_t)nq1 * k * 4));
    CKR(idx->oshort.ensure((size_t)nq1 * 4));
    if (nq > 0) {
        CK(cudaMemcpyAsync(idx->q.p, queries, (size_t)nq * idx->d * 4, cudaMemcpyHostToDevice, st));
        CKR(search_device_impl(idx, idx->q.as<float>(), nq, k, nprobe, dt, idx->oids.as<int64_t>(),
                               idx->odist.as<float>(), idx->oshort.as<int32_t>(), st));
        CK(cudaMemcpyAsync(out_ids, idx->oids.p, (size_t)nq * k * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(out_dists, idx->odist.p, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, st));
    }
    // short flags into a pinned per-handle buffer (an async copy; a pageable
    // destination would be staged synchronously)
    if (nq > idx->h_short_cap) {
        CK(cudaStreamSynchronize(st));
        if (idx->h_short) CK(cudaFreeHost(idx->h_short));
        idx->h_short = nullptr;
        idx->h_short_cap = 0;
        CK(cudaHostAlloc((void**)&idx->h_short, (size_t)nq * 4, cudaHostAllocDefault));
        idx->h_short_cap = nq;
    }
    if (nq > 0) CK(cudaMemcpyAsync(idx->h_short, idx->oshort.p, (size_t)nq * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    int64_t ns = 0;
    for (int64_t i = 0; i < nq; ++i) ns += idx->h_short[i];
    if (out_n_short) *out_n_short = ns;
    return IVFPQ_OK;
}

int ivfpq_search_device(ivfpq_index* idx, const float* d_q, int64_t nq, int64_t k, int64_t nprobe, int dt,
                        int64_t* d_ids, float* d_d, int32_t* d_short, void* stream) {
    CKR(validate_search(idx, nq, k, nprobe, dt));
    std::lock_guard<std::mutex> lock(idx->mu);
    DeviceGuard guard(idx->device);
    if (nq == 0) return IVFPQ_OK;
    StreamOrder order(idx, pick_stream(idx, stream));
    return search_device_impl(idx, d_q, nq, k, nprobe, dt, d_ids, d_d, d_short, order.st);
}

int ivfpq_select_device(ivfpq_index* idx, const float* d_q, int64_t nq, int64_t nprobe, uint64_t* d_keys,
                        void* stream) {
    if (!idx) return set_err(IVFPQ_EINVAL, "null index");
    if (nprobe < 1 || nprobe > idx->nlist)
        return set_err(IVFPQ_EINVAL, "nprobe=%lld out of range 1..%lld", (long long)nprobe, (long long)idx->nlist);
    std::lock_guard<std::mutex> lock(idx->mu);
    DeviceGuard guard(idx->device);
    if (nq == 0) return IVFPQ_OK;
    StreamOrder order(idx, pick_stream(idx, stream));
    return run_select(idx, d_q, nq, nprobe, d_keys, order.st);
}

int ivfpq_merge_keys_device(const uint64_t* d_in, int64_t W, int64_t nq, int64_t n_in, int64_t n_out,
                            uint64_t* d_out, void* stream) {
    if (W < 1 || n_in < 1 || n_out < 1 || n_out > MAX_K)
        return set_err(IVFPQ_EINVAL, "invalid merge shape W=%lld n_in=%lld n_out=%lld", (long long)W,
                       (long long)n_in, (long long)n_out);
    if (nq == 0) return IVFPQ_OK;
    // rows arrive sorted (the contract): pairwise merge-paths, one warp per row,
    // when the runs fit shared memory; else the block top-k selection
    const size_t ms_smem = (size_t)MS_WARPS * 2 * W * n_in * 8;
    if (ms_smem <= SMEM_LIMIT) {
        CKR(set_smem_attr((const void*)merge_sorted_kernel, ms_smem));
        merge_sorted_kernel<<<(unsigned)((nq + MS_WARPS - 1) / MS_WARPS), 32 * MS_WARPS, ms_smem,
                              reinterpret_cast<cudaStream_t>(stream)>>>(d_in, (int)W, (int)nq, (int)n_in, (int)n_out,
                                                                        d_out);
        KCHECK();
        return IVFPQ_OK;
    }
    CKR(set_smem_attr((const void*)merge_keys_kernel, SMEM_LIMIT));  // per-device: set every launch
    merge_keys_kernel<<<(unsigned)nq, TK_BLOCK, topk_smem((int)n_out), reinterpret_cast<cudaStream_t>(stream)>>>(
        d_in, (int)W, (int)nq, (int)n_in, (int)n_out, d_out);
    KCHECK();
    return IVFPQ_OK;
}

int ivfpq_scan_device(ivfpq_index* idx, const float* d_q, int64_t nq, const uint64_t* d_pk, int64_t nprobe,
                      int64_t k, int dt, uint64_t* d_keys, int64_t* d_ncand, void* stream) {
    CKR(validate_search(idx, nq, k, nprobe, dt));
    std::lock_guard<std::mutex> lock(idx->mu);
    DeviceGuard guard(idx->device);
    StreamOrder order(idx, pick_stream(idx, stream));
    return run_scan(idx, d_q, nq, d_pk, nprobe, k, dt, d_keys, d_ncand, nullptr, nullptr, nullptr, order.st);
}

int ivfpq_finalize_device(const uint64_t* d_keys, const int64_t* d_ncand, int64_t nq, int64_t k, int64_t* d_ids,
                          float* d_d, int32_t* d_short, void* stream) {
    if (nq == 0) return IVFPQ_OK;
    const int64_t n = std::max(nq * k, nq);
    finalize_kernel<<<blocks_for(n), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(d_keys, d_ncand, (int)nq,
                                                                                      (int)k, d_ids, d_d, d_short);
    KCHECK();
    return IVFPQ_OK;
}

}  // extern "C"

// ---- conformance hooks ---------------------------------------------------------
namespace {
template <class T>
struct Tmp {
    T* p = nullptr;
    ~Tmp() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t n) { return cudaMalloc((void**)&p, std::max<size_t>(n, 1) * sizeof(T)); }
};
}  // namespace

extern "C" {

int ivfpq_fp8_encode(const float* x, int64_t n, int dt, uint8_t* out) {
    if (dt != LUT_E5M3 && dt != LUT_E4M4) return set_err(IVFPQ_EINVAL, "fp8 dtype must be e5m3 or e4m4");
    if (n == 0) return IVFPQ_OK;
    Tmp<float> dx;
    Tmp<uint8_t> dy;
    CK(dx.alloc(n));
    CK(dy.alloc(n));
    CK(cudaMemcpy(dx.p, x, n * 4, cudaMemcpyHostToDevice));
    if (dt == LUT_E5M3) encode_kernel<LUT_E5M3><<<blocks_for(n), 256>>>(dx.p, n, dy.p);
    else encode_kernel<LUT_E4M4><<<blocks_for(n), 256>>>(dx.p, n, dy.p);
    KCHECK();
    CK(cudaMemcpy(out, dy.p, n, cudaMemcpyDeviceToHost));
    return IVFPQ_OK;
}

int ivfpq_fp8_decode(const uint8_t* codes, int64_t n, int dt, float* out) {
    if (dt != LUT_E5M3 && dt != LUT_E4M4) return set_err(IVFPQ_EINVAL, "fp8 dtype must be e5m3 or e4m4");
    if (n == 0) return IVFPQ_OK;
    Tmp<uint8_t> dx;
    Tmp<float> dy;
    CK(dx.alloc(n));
    CK(dy.alloc(n));
    CK(cudaMemcpy(dx.p, codes, n, cudaMemcpyHostToDevice));
    if (dt == LUT_E5M3) decode_kernel<LUT_E5M3><<<blocks_for(n), 256>>>(dx.p, n, dy.p);
    else decode_kernel<LUT_E4M4><<<blocks_for(n), 256>>>(dx.p, n, dy.p);
    KCHECK();
    CK(cudaMemcpy(out, dy.p, n * 4, cudaMemcpyDeviceToHost));
    return IVFPQ_OK;
}

int ivfpq_f16_encode(const float* x, int64_t n, uint16_t* out) {
    if (n == 0) return IVFPQ_OK;
    Tmp<float> dx;
    Tmp<uint16_t> dy;
    CK(dx.alloc(n));
    CK(dy.alloc(n));
    CK(cudaMemcpy(dx.p, x, n * 4, cudaMemcpyHostToDevice));
    encode_kernel<LUT_F16><<<blocks_for(n), 256>>>(dx.p, n, dy.p);
    KCHECK();
    CK(cudaMemcpy(out, dy.p, n * 2, cudaMemcpyDeviceToHost));
    return IVFPQ_OK;
}

int ivfpq_f16_decode(const uint16_t* bits, int64_t n, float* out) {
    if (n == 0) return IVFPQ_OK;
    Tmp<uint16_t> dx;
    Tmp<float> dy;
    CK(dx.alloc(n));
    CK(dy.alloc(n));
    CK(cudaMemcpy(dx.p, bits, n * 2, cudaMemcpyHostToDevice));
    decode_kernel<LUT_F16><<<blocks_for(n), 256>>>(dx.p, n, dy.p);
    KCHECK();
    CK(cudaMemcpy(out, dy.p, n * 4, cudaMemcpyDeviceToHost));
    return IVFPQ_OK;
}

}  // extern "C"

namespace {
template <int DT>
int build_lut_dt(int logn, const float* dc, int s, int sub_d, const float* drq, void* dout, size_t smem) {
    using T = typename LutTraits<DT>::T;
    switch (logn) {
#define BL(L)                                                                                          \
    case L:                                                                                            \
        CKR(set_smem_attr((const void*)build_lut_kernel<DT, L>, SMEM_LIMIT));                           \
        build_lut_kernel<DT, L><<<1, TK_BLOCK, smem > SMEM_LIMIT ? ((size_t)s * sub_d * 4 + 15) & ~(size_t)15 : smem>>>( \
            dc, s, sub_d, drq, reinterpret_cast<T*>(dout), smem > SMEM_LIMIT); \
        break;
        BL(1) BL(2) BL(3) BL(4) BL(5) BL(6) BL(7) BL(8)
#undef BL
        default: return set_err(IVFPQ_EINVAL, "pq_bits out of range");
    }
    KCHECK();
    return IVFPQ_OK;
}
template <int DT>
int scan_list_dt(int logn, const uint8_t* dcodes, int64_t L, int s, const void* dent, float* dout, size_t smem) {
    const unsigned grid = (unsigned)std::min<int64_t>(1024, std::max<int64_t>(1, (L + TK_BLOCK - 1) / TK_BLOCK));
    switch (logn) {
#define SL(LG)                                                                                  \
    case LG:                                                                                    \
        CKR(set_smem_attr((const void*)scan_list_kernel<DT, LG>, SMEM_LIMIT));                   \
        scan_list_kernel<DT, LG><<<grid, TK_BLOCK, smem > SMEM_LIMIT ? 0 : smem>>>(dcodes, L, s, dent, dout, \
                                                                                smem > SMEM_LIMIT);     \
        break;
        SL(1) SL(2) SL(3) SL(4) SL(5) SL(6) SL(7) SL(8)
#undef SL
        default: return set_err(IVFPQ_EINVAL, "pq_bits out of range");
    }
    KCHECK();
    return IVFPQ_OK;
}
}  // namespace

extern "C" {

int ivfpq_build_lut(const float* centers, int64_t s, int64_t p, int64_t sub_d, const float* rq, int dt,
                    void* out_entries) {
    CKR(check_dtype(dt));
    if (s < 1 || p < 1 || p > 8 || sub_d < 1) return set_err(IVFPQ_EINVAL, "invalid codebook shape");
    const int64_t d = s * sub_d, ne = s << p;
    const size_t eb = lut_bytes_of(dt);
    const size_t smem = (((size_t)d * 4 + 15) & ~(size_t)15) + ne * eb;
    Tmp<float> dc, drq;
    Tmp<uint8_t> dout;
    CK(dc.alloc(ne * sub_d));
    CK(drq.alloc(d));
    CK(dout.alloc(ne * eb));
    CK(cudaMemcpy(dc.p, centers, ne * sub_d * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(drq.p, rq, d * 4, cudaMemcpyHostToDevice));
    CKR(DISPATCH_DT_LOGN(dt, (int)p, build_lut_dt, dc.p, (int)s, (int)sub_d, drq.p, dout.p, smem));
    CK(cudaMemcpy(out_entries, dout.p, ne * eb, cudaMemcpyDeviceToHost));
    return IVFPQ_OK;
}

int ivfpq_scan_list(const uint8_t* codes, int64_t L, int64_t s, int64_t p, const void* entries, int dt, float* out_r) {
    CKR(check_dtype(dt));
    if (s < 1 || p < 1 || p > 8 || L < 0) return set_err(IVFPQ_EINVAL, "invalid scan shape");
    const int64_t ne = s << p;
    const size_t eb = lut_bytes_of(dt);
    if (L == 0) return IVFPQ_OK;
    for (int64_t i = 0; i < L * s; ++i)
        if (codes[i] >= (1 << p)) return set_err(IVFPQ_EINVAL, "code byte out of range for the table");
    Tmp<uint8_t> dcodes, dent;
    Tmp<float> dout;
    CK(dcodes.alloc(L * s));
    CK(dent.alloc(ne * eb));
    CK(dout.alloc(L));
    CK(cudaMemcpy(dcodes.p, codes, L * s, cudaMemcpyHostToDevice));
    if (dt == LUT_E5M3 || dt == LUT_E4M4) {
        // The scan widens an fp8 entry with one shift (its value is scaled back
        // once per vector), which is the exact decode for every code the
        // encoder emits.  A caller-built table may also hold codes 1..2^m-1
        // (zero exponent field), which the reference decodes to 0.0
        // (minifloat.py:119-133): store those as 0 so the scan matches.
        const int m = dt == LUT_E5M3 ? LutTraits<LUT_E5M3>::m : LutTraits<LUT_E4M4>::m;
        std::vector<uint8_t> ent(static_cast<const uint8_t*>(entries), static_cast<const uint8_t*>(entries) + ne);
        for (auto& e : ent)
            if (e < (1u << m)) e = 0;
        CK(cudaMemcpy(dent.p, ent.data(), ne, cudaMemcpyHostToDevice));
    } else {
        CK(cudaMemcpy(dent.p, entries, ne * eb, cudaMemcpyHostToDevice));
    }
    CKR(DISPATCH_DT_LOGN(dt, (int)p, scan_list_dt, dcodes.p, L, (int)s, (const void*)dent.p, dout.p, ne * eb));
    CK(cudaMemcpy(out_r, dout.p, L * 4, cudaMemcpyDeviceToHost));
    return IVFPQ_OK;
}

int ivfpq_select_clusters(ivfpq_index* idx, const float* q, int64_t nq, int64_t nprobe, int64_t* out) {
    if (!idx) return set_err(IVFPQ_EINVAL, "null index");
    if (nprobe < 1 || nprobe > idx->nlist)
        return set_err(IVFPQ_EINVAL, "nprobe=%lld out of range 1..%lld", (long long)nprobe, (long long)idx->nlist);
    if (nprobe > MAX_K) return set_err(IVFPQ_EUNSUPPORTED, "nprobe exceeds the device limit %d", MAX_K);
    std::lock_guard<std::mutex> lock(idx->mu);
    DeviceGuard guard(idx->device);
    if (nq == 0) return IVFPQ_OK;
    cudaStream_t st = idx->stream;
    StreamOrder order(idx, st);
    CKR(idx->q.ensure((size_t)nq * idx->d * 4));
    CKR(idx->pkeys.ensure((size_t)nq * nprobe * 8));
    CKR(idx->oids.ensure((size_t)nq * nprobe * 8));
    CK(cudaMemcpyAsync(idx->q.p, q, (size_t)nq * idx->d * 4, cudaMemcpyHostToDevice, st));
    CKR(run_select(idx, idx->q.as<float>(), nq, nprobe, idx->pkeys.as<uint64_t>(), st));
    keys_to_gid_kernel<<<blocks_for(nq * nprobe), 256, 0, st>>>(idx->pkeys.as<uint64_t>(), nq * nprobe,
                                                                 idx->oids.as<int64_t>());
    KCHECK();
    CK(cudaMemcpyAsync(out, idx->oids.p, (size_t)nq * nprobe * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return IVFPQ_OK;
}

int ivfpq_top_k(const int64_t* ids, const float* dists, int64_t n, int64_t k, int64_t* out_ids, float* out_dists) {
    if (n < 1) return set_err(IVFPQ_EINVAL, "top_k requires at least one candidate");
    if (k < 1) return set_err(IVFPQ_EINVAL, "k must be at least 1");
    if (k > MAX_K) return set_err(IVFPQ_EUNSUPPORTED, "k exceeds the device limit %d", MAX_K);
    if (n >= (1LL << 31)) return set_err(IVFPQ_EUNSUPPORTED, "too many candidates");
    for (int64_t i = 0; i < n; ++i)
        if (ids[i] < 0 || ids[i] >= 0xffffffffLL) return set_err(IVFPQ_EUNSUPPORTED, "ids must be in [0, 2^32-1)");
    Tmp<int64_t> di, doi;
    Tmp<float> dd, dod;
    CK(di.alloc(n));
    CK(dd.alloc(n));
    CK(doi.alloc(k));
    CK(dod.alloc(k));
    CK(cudaMemcpy(di.p, ids, n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dd.p, dists, n * 4, cudaMemcpyHostToDevice));
    CKR(set_smem_attr((const void*)topk_hook_kernel, SMEM_LIMIT));
    topk_hook_kernel<<<1, TK_BLOCK, topk_smem((int)k)>>>(di.p, dd.p, (int)n, (int)k, doi.p, dod.p);
    KCHECK();
    const int64_t m = std::min(n, k);
    CK(cudaMemcpy(out_ids, doi.p, m * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out_dists, dod.p, m * 4, cudaMemcpyDeviceToHost));
    return IVFPQ_OK;
}

}  // extern "C"

// ---- ingest: pq_encode / assign_to_centroids (ingest.cuh) ---------------------
namespace {
template <int SUB_D>
int launch_pq_encode(const float* x, int64_t n, int d, const float* coarse, const int64_t* assign,
                     const float* centers, int s, int N, uint8_t* codes, cudaStream_t st) {
    constexpr int CS = SUB_D <= 3 ? 4 : 8;
    const size_t smem = (size_t)ENC_JG * N * CS * 4;
    CKR(set_smem_attr((const void*)pq_encode_kernel<SUB_D>, smem));
    const dim3 grid((unsigned)((n + ENC_THREADS - 1) / ENC_THREADS), (unsigned)((s + ENC_JG - 1) / ENC_JG));
    pq_encode_kernel<SUB_D><<<grid, ENC_THREADS, smem, st>>>(x, n, d, coarse, assign, centers, s, N, codes);
    KCHECK();
    return IVFPQ_OK;
}

int check_encode_shape(int64_t n, int64_t d, int64_t s, int64_t p) {
    if (n < 0) return set_err(IVFPQ_EINVAL, "n must be non-negative");
    if (p < 1 || p > 8) return set_err(IVFPQ_EINVAL, "p must be in 1..8 (one byte per sub-code)");
    if (s < 1 || d % s != 0) return set_err(IVFPQ_EINVAL, "d=%lld not divisible by s=%lld", (long long)d, (long long)s);
    if (d / s > 4)
        return set_err(IVFPQ_EUNSUPPORTED, "bit-exact pq_encode is implemented for sub_d <= 4 (got %lld)",
                       (long long)(d / s));
    if (n >= (1LL << 31) * ENC_THREADS) return set_err(IVFPQ_EUNSUPPORTED, "too many rows");
    return IVFPQ_OK;
}
}  // namespace

extern "C" {

int ivfpq_pq_encode_device(const float* d_x, int64_t n, int64_t d, const float* d_coarse, const int64_t* d_assign,
                           const float* d_centers, int64_t s, int64_t p, uint8_t* d_codes, void* stream) {
    CKR(check_encode_shape(n, d, s, p));
    if ((d_coarse == nullptr) != (d_assign == nullptr))
        return set_err(IVFPQ_EINVAL, "coarse and assign must be given together");
    if (n == 0) return IVFPQ_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int N = 1 << p;
    switch (d / s) {
        case 1: return launch_pq_encode<1>(d_x, n, (int)d, d_coarse, d_assign, d_centers, (int)s, N, d_codes, st);
        case 2: return launch_pq_encode<2>(d_x, n, (int)d, d_coarse, d_assign, d_centers, (int)s, N, d_codes, st);
        case 3: return launch_pq_encode<3>(d_x, n, (int)d, d_coarse, d_assign, d_centers, (int)s, N, d_codes, st);
        default: return launch_pq_encode<4>(d_x, n, (int)d, d_coarse, d_assign, d_centers, (int)s, N, d_codes, st);
    }
}

int ivfpq_pq_encode(const float* x, int64_t n, int64_t d, const float* centers, int64_t s, int64_t p,
                    uint8_t* codes) {
    CKR(check_encode_shape(n, d, s, p));
    if (n == 0) return IVFPQ_OK;
    Tmp<float> dx, dc;
    Tmp<uint8_t> dk;
    CK(dx.alloc(n * d));
    CK(dc.alloc((s << p) * (d / s)));
    CK(dk.alloc(n * s));
    CK(cudaMemcpy(dx.p, x, n * d * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dc.p, centers, (size_t)(s << p) * (d / s) * 4, cudaMemcpyHostToDevice));
    CKR(ivfpq_pq_encode_device(dx.p, n, d, nullptr, nullptr, dc.p, s, p, dk.p, nullptr));
    CK(cudaMemcpy(codes, dk.p, n * s, cudaMemcpyDeviceToHost));
    return IVFPQ_OK;
}

int ivfpq_squared_l2_to_all(const float* base, int64_t n, int64_t d, const float* q, float* out) {
    if (n < 0 || d < 1) return set_err(IVFPQ_EINVAL, "invalid shape n=%lld d=%lld", (long long)n, (long long)d);
    if (n == 0) return IVFPQ_OK;
    Tmp<float> db, dq, dout;
    CK(db.alloc(n * d));
    CK(dq.alloc(d));
    CK(dout.alloc(n));
    CK(cudaMemcpy(db.p, base, n * d * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dq.p, q, d * 4, cudaMemcpyHostToDevice));
    sq_l2_all_kernel<<<blocks_for(n), 256>>>(db.p, n, (int)d, dq.p, dout.p);
    KCHECK();
    CK(cudaMemcpy(out, dout.p, n * 4, cudaMemcpyDeviceToHost));
    return IVFPQ_OK;
}

int ivfpq_compute_residuals(const float* x, int64_t n, int64_t d, const float* c, int64_t nc, const int64_t* assign,
                            float* out) {
    if (n < 0 || d < 1 || nc < 1) return set_err(IVFPQ_EINVAL, "invalid shape");
    for (int64_t i = 0; i < n; ++i)
        if (assign[i] < 0 || assign[i] >= nc) return set_err(IVFPQ_EINVAL, "assignment index out of range");
    if (n == 0) return IVFPQ_OK;
    Tmp<float> dx, dc, dout;
    Tmp<int64_t> da;
    CK(dx.alloc(n * d));
    CK(dc.alloc(nc * d));
    CK(da.alloc(n));
    CK(dout.alloc(n * d));
    CK(cudaMemcpy(dx.p, x, n * d * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dc.p, c, nc * d * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(da.p, assign, n * 8, cudaMemcpyHostToDevice));
    residuals_kernel<<<blocks_for(n * d), 256>>>(dx.p, n, (int)d, dc.p, da.p, dout.p);
    KCHECK();
    CK(cudaMemcpy(out, dout.p, n * d * 4, cudaMemcpyDeviceToHost));
    return IVFPQ_OK;
}

int ivfpq_reconstruct(const uint8_t* codes, int64_t n, const float* centers, int64_t s, int64_t p, int64_t sub_d,
                      float* out) {
    if (n < 0 || s < 1 || p < 1 || p > 8 || sub_d < 1) return set_err(IVFPQ_EINVAL, "invalid shape");
    for (int64_t i = 0; i < n * s; ++i)
        if (codes[i] >= (1 << p)) return set_err(IVFPQ_EINVAL, "code byte out of range for p=%lld", (long long)p);
    if (n == 0) return IVFPQ_OK;
    Tmp<uint8_t> dk;
    Tmp<float> dc, dout;
    CK(dk.alloc(n * s));
    CK(dc.alloc((s << p) * sub_d));
    CK(dout.alloc(n * s * sub_d));
    CK(cudaMemcpy(dk.p, codes, n * s, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dc.p, centers, (size_t)(s << p) * sub_d * 4, cudaMemcpyHostToDevice));
    reconstruct_kernel<<<blocks_for(n * s * sub_d), 256>>>(dk.p, n, (int)s, 1 << (int)p, (int)sub_d, dc.p, dout.p);
    KCHECK();
    CK(cudaMemcpy(out, dout.p, n * s * sub_d * 4, cudaMemcpyDeviceToHost));
    return IVFPQ_OK;
}

int ivfpq_assign_device(const float* d_x, int64_t n, int64_t d, const float* d_c, int64_t nc, int64_t* d_assign,
                        float* d_d2, void* stream) {
    if (n < 0 || d < 1) return set_err(IVFPQ_EINVAL, "invalid data shape");
    if (nc < 1) return set_err(IVFPQ_EINVAL, "need at least one centroid");
    if (nc >= (1LL << 31) || n >= (1LL << 31) * AS_TM) return set_err(IVFPQ_EUNSUPPORTED, "too many rows");
    if (n == 0) return IVFPQ_OK;
    cudaStream_t st = (cudaStream_t)stream;
    Tmp<float> cn;
    CK(cn.alloc(nc));
    row_sqnorm_kernel<<<blocks_for(nc), 256, 0, st>>>(d_c, nc, (int)d, cn.p);
    KCHECK();
    assign_kernel<<<(unsigned)((n + AS_TM - 1) / AS_TM), 256, 0, st>>>(d_x, n, (int)d, d_c, (int)nc, cn.p, d_assign,
                                                                        d_d2);
    KCHECK();
    CK(cudaStreamSynchronize(st));  // cn is freed on return
    return IVFPQ_OK;
}

int ivfpq_assign(const float* x, int64_t n, int64_t d, const float* c, int64_t nc, int64_t* assign, float* d2) {
    if (n < 0 || d < 1) return set_err(IVFPQ_EINVAL, "invalid data shape");
    if (n == 0) return IVFPQ_OK;
    Tmp<float> dx, dc, dd;
    Tmp<int64_t> da;
    CK(dx.alloc(n * d));
    CK(dc.alloc(nc * d));
    CK(da.alloc(n));
    CK(dd.alloc(n));
    CK(cudaMemcpy(dx.p, x, n * d * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dc.p, c, nc * d * 4, cudaMemcpyHostToDevice));
    CKR(ivfpq_assign_device(dx.p, n, d, dc.p, nc, da.p, dd.p, nullptr));
    CK(cudaMemcpy(assign, da.p, n * 8, cudaMemcpyDeviceToHost));
    if (d2) CK(cudaMemcpy(d2, dd.p, n * 4, cudaMemcpyDeviceToHost));
    return IVFPQ_OK;
}

}  // extern "C"

// ---- K7: exact k-NN (brute_force_knn, datasets.py:179-201) ---------------------
// The reference's ground truth is K1's arithmetic over the base rows instead of
// the centroids: d2 = sequential fl(acc + fl(diff^2)) (squared_l2_to_all,
// datasets.py:166-176), stable argsort -> (d2, id) keys.  A k-NN handle is an
// index whose "centroids" are the base rows (no lists), searched with the
// same select path (tensor-core nomination + exact re-rank + guard).
extern "C" {

int ivfpq_knn_create(int device, const float* base, int64_t n, int64_t d, ivfpq_index** out) {
    if (!out) return set_err(IVFPQ_EINVAL, "null output handle");
    *out = nullptr;
    if (n < 1 || d < 1) return set_err(IVFPQ_EINVAL, "invalid base shape n=%lld d=%lld", (long long)n, (long long)d);
    if (n >= (1LL << 31) - 1) return set_err(IVFPQ_EUNSUPPORTED, "base too large for one k-NN handle");
    DeviceGuard guard(device);
    CK(cudaSetDevice(device));
    ivfpq_index* idx = new ivfpq_index();
    idx->device = device;
    idx->nlist = idx->nlist_local = n;
    idx->d = d;
    idx->s = 1;
    idx->p = 1;
    idx->sub_d = d;
    auto fail = [&](int rc) {
        ivfpq_index_destroy(idx);
        return rc;
    };
#define CKI(call)                                                                              \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            return fail(set_err(IVFPQ_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_))); \
    } while (0)
    CKI(cudaStreamCreateWithFlags(&idx->stream, cudaStreamNonBlocking));
    CKI(cudaEventCreateWithFlags(&idx->last_ev, cudaEventDisableTiming));
    CKI(cudaDeviceGetAttribute(&idx->num_sms, cudaDevAttrMultiProcessorCount, device));
    {
        int l2 = 0;
        CKI(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device));
        idx->l2_bytes = l2;
    }
    CKI(cudaMalloc((void**)&idx->coarse, (size_t)n * d * 4));
    CKI(cudaMemcpy(idx->coarse, base, (size_t)n * d * 4, cudaMemcpyHostToDevice));
    std::vector<int32_t> ident(n);
    for (int64_t i = 0; i < n; ++i) ident[i] = (int32_t)i;
    CKI(cudaMalloc((void**)&idx->l2g, (size_t)n * 4));
    CKI(cudaMemcpy(idx->l2g, ident.data(), (size_t)n * 4, cudaMemcpyHostToDevice));
    idx->bytes = n * d * 4 + n * 4;
    if (d <= TC_MAXD) {
        const int64_t ntiles = (n + TC_N - 1) / TC_N, nkc = coarse_tc_nkc((int)d);
        const size_t ib = (size_t)ntiles * nkc * TC_N * 128;
        CKI(cudaMalloc((void**)&idx->tc_img, ib));
        idx->bytes += (int64_t)ib;
        coarse_tc_prep_kernel<<<(unsigned)ntiles, 256, 0, idx->stream>>>(idx->coarse, (int)n, (int)d, (int)nkc,
                                                                         idx->tc_img);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        CKI(cudaGetLastError());
        idx->tc_cmax = coarse_tc_cmax(base, n, d);
    }
    CKI(cudaStreamSynchronize(idx->stream));
#undef CKI
    *out = idx;
    return IVFPQ_OK;
}

int ivfpq_brute_force_knn(const float* base, int64_t n, int64_t d, const float* queries, int64_t nq, int64_t k,
                          int64_t* out_ids, float* out_dists) {
    if (k < 1) return set_err(IVFPQ_EINVAL, "k must be at least 1");
    if (k > n) return set_err(IVFPQ_EINVAL, "k=%lld exceeds base size %lld", (long long)k, (long long)n);
    if (k > MAX_K) return set_err(IVFPQ_EUNSUPPORTED, "k exceeds the device limit %d", MAX_K);
    ivfpq_index* h = nullptr;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CKR(ivfpq_knn_create(dev, base, n, d, &h));
    struct Closer {
        ivfpq_index* h;
        ~Closer() { ivfpq_index_destroy(h); }
    } closer{h};
    if (nq == 0) return IVFPQ_OK;
    cudaStream_t st = h->stream;
    const int64_t chunk = std::min<int64_t>(nq, 16384);
    CKR(h->q.ensure((size_t)chunk * d * 4));
    CKR(h->pkeys.ensure((size_t)chunk * k * 8));
    CKR(h->oids.ensure((size_t)chunk * k * 8));
    CKR(h->odist.ensure((size_t)chunk * k * 4));
    CKR(h->ncand.ensure((size_t)chunk * 8));
    CKR(h->oshort.ensure((size_t)chunk * 4));
    for (int64_t q0 = 0; q0 < nq; q0 += chunk) {
        const int64_t m = std::min(chunk, nq - q0);
        CK(cudaMemcpyAsync(h->q.p, queries + q0 * d, (size_t)m * d * 4, cudaMemcpyHostToDevice, st));
        CKR(run_select(h, h->q.as<float>(), m, k, h->pkeys.as<uint64_t>(), st));
        CK(cudaMemsetAsync(h->ncand.p, 0x7f, (size_t)m * 8, st));  // never short: k <= n
        finalize_kernel<<<blocks_for(m * k), 256, 0, st>>>(h->pkeys.as<uint64_t>(), h->ncand.as<int64_t>(), (int)m,
                                                          (int)k, h->oids.as<int64_t>(), h->odist.as<float>(),
                                                          h->oshort.as<int32_t>());
        KCHECK();
        CK(cudaMemcpyAsync(out_ids + q0 * k, h->oids.p, (size_t)m * k * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(out_dists + q0 * k, h->odist.p, (size_t)m * k * 4, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    return IVFPQ_OK;
}

}  // extern "C"
