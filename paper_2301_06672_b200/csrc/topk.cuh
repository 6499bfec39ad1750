// Block-level top-K over 64-bit keys, smallest first.
//
// Key = (fp32 bits of the distance) << 32 | id.  Distances are >= +0, so the
// raw bits order like the floats, and the key order is exactly the
// reference's lexicographic (distance, id) order: `np.lexsort((ids, R))`
// (search.py:150) and `argsort(kind="stable")` over cluster ids
// (search.py:97).  Ids are unique within one selection, so keys are unique.
// Empty slots hold ~0ull (sorts after every real key).
//
// Protocol (all threads of the block, control flow uniform):
//   tk.init();                        // K slots of ~0
//   loop rounds { tk.offer(key, pred) (<= 1 key per thread per round);
//                 tk.maybe_merge(); } // merges when the buffer may overflow
//   tk.merge();                       // flush
// Candidates are filtered against tau = current K-th key, so after the first
// merges only a trickle of keys reaches the buffer.
#pragma once
#include <stdint.h>

namespace ivfpq {

constexpr int TK_BLOCK = 256;           // threads per block using the top-K
constexpr int TK_CAP = 2 * TK_BLOCK;    // candidate buffer capacity

__device__ __forceinline__ int lower_bound_u64(const uint64_t* a, int n, uint64_t x) {
    int lo = 0, hi = n;  // count of a[i] < x, a sorted ascending
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ int upper_bound_u64(const uint64_t* a, int n, uint64_t x) {
    int lo = 0, hi = n;  // count of a[i] <= x, a sorted ascending
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1; else hi = mid;
    }
    return lo;
}
// Merge-path with equal keys: an element of the running list A goes before
// the equal elements of the new sorted run (lower bound), a new element after
// the equal elements of A (upper bound), so every output position is written
// exactly once even when keys repeat (caller-supplied duplicate (id, dist)
// pairs of the public top_k hook; reference np.lexsort keeps all copies).

struct BlockTopK {
    uint64_t* slots[2];  // K keys each, ascending; slots[cur] is live
    uint64_t* buf;       // TK_CAP unsorted candidates
    uint64_t* sorted;    // TK_CAP scratch
    int* count;          // candidates in buf
    int K;
    int cur;

    // smem bytes needed for K slots
    __host__ __device__ static size_t smem_bytes(int K) {
        return (size_t)2 * K * 8 + (size_t)2 * TK_CAP * 8 + 16;
    }
    __device__ void bind(uint8_t* p, int K_) {
        K = K_;
        cur = 0;
        slots[0] = reinterpret_cast<uint64_t*>(p);
        slots[1] = slots[0] + K;
        buf = slots[1] + K;
        sorted = buf + TK_CAP;
        count = reinterpret_cast<int*>(sorted + TK_CAP);
    }
    __device__ void init() {  // (re)start: empty slot 0 live, no candidates
        cur = 0;
        for (int i = threadIdx.x; i < K; i += blockDim.x) slots[0][i] = ~0ull;
        if (threadIdx.x == 0) *count = 0;
        __syncthreads();
    }
    __device__ __forceinline__ uint64_t tau() const { return slots[cur][K - 1]; }
    __device__ __forceinline__ const uint64_t* result() const { return slots[cur]; }

    // Warp-aggregated append; every lane of the warp must call it.
    __device__ __forceinline__ void offer(uint64_t key, bool pred) {
        unsigned mask = __ballot_sync(0xffffffffu, pred);
        if (mask == 0) return;
        int lane = threadIdx.x & 31;
        int leader = __ffs(mask) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(count, __popc(mask));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (pred) buf[base + __popc(mask & ((1u << lane) - 1))] = key;
    }

    // Merge buf into slots.  Block-wide; includes the barriers it needs.
    // Barrier, read the shared count, barrier: every thread sees the same
    // value and nobody can append before all have read it.
    __device__ __forceinline__ int synced_count() {
        __syncthreads();
        int n = *count;
        __syncthreads();
        return n;
    }

    __device__ void merge() { merge_n(synced_count()); }

    __device__ void merge_n(const int n) {
        if (n == 0) return;  // uniform
        // 1. rank-sort the candidates (stable: equal keys ranked by buffer index)
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            uint64_t x = buf[i];
            int r = 0;
            for (int j = 0; j < n; ++j) r += buf[j] < x || (buf[j] == x && j < i);
            sorted[r] = x;
        }
        __syncthreads();
        // 2. merge-path: position = own index + rank in the other sequence
        const uint64_t* A = slots[cur];
        uint64_t* O = slots[cur ^ 1];
        for (int i = threadIdx.x; i < K; i += blockDim.x) {
            uint64_t a = A[i];
            int pos = i + lower_bound_u64(sorted, n, a);
            if (pos < K) O[pos] = a;
        }
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            uint64_t b = sorted[i];
            int pos = i + upper_bound_u64(A, K, b);
            if (pos < K) O[pos] = b;
        }
        __syncthreads();
        cur ^= 1;
        if (threadIdx.x == 0) *count = 0;
        __syncthreads();
    }

    // Called between rounds: merge if another round could overflow buf.
    __device__ void maybe_merge() {
        int n = synced_count();
        if (n > TK_CAP - (int)blockDim.x) merge_n(n);
    }
};

}  // namespace ivfpq
