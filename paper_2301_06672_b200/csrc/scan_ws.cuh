// K2 + K3 + K4, v2: persistent, warp-specialised search kernel for sm_100a.
//
// Same arithmetic as the reference (search.py:158-184 -> build_lut :114-127,
// scan_list :130-142, top_k :145-155) and as scan.cuh, restructured for B200:
//
//  * one CTA per SM (persistent), queries handed out by a global atomic;
//  * the PQ codebook lives in TENSOR MEMORY (tcgen05.alloc/st/ld; up to 256 of
//    the SM's 512 columns): each of the BW BUILDER warps (8 in layout A, 4 in B) reads only its
//    own lane's columns.  Builder thread t owns a quad of codes m = 4u..4u+3
//    and the subspaces j = jr, jr+R, ... (u = t % (N/4), jr = t / (N/4),
//    R = 4 * WS_NB / N); one tcgen05.ld of a row's centers serves all G lists
//    of a job.  Per (j, quad) one broadcast read of rq[j] feeds 4 table
//    entries computed with packed f32x2 sub/mul/add (every op one IEEE
//    rounding, in the reference order), stored with one 4-, 8- or 16-byte STS:
//      fp8: mul.rz.ftz.f32x2 by 2^-(127-bias) (exact scaling; values below
//           min_normal become subnormal and flush to +0), then the code is
//           min(bits >> (23-m), 255), done two-at-a-time with u16x2 min.
//      f16: cvt.rn.satfinite.f16x2.f32 (= RNE of min(x, 65504)).
//  * SW SCANNER warps (11 in layout A, 15 in B) take pairs of 32-vector code blocks (16-byte
//    loads from L2 into registers, interleaved layout) and look the codes up
//    in the slot's LUTs; R accumulates sequentially in j (fp32).
//  * one PREP warp hands out queries and streams their planned jobs
//    (ws_plan_kernel: descriptor + residual rows) into an 8-deep ring by TMA.
//  * hand-offs: prep -> builders on mbarriers completed by the TMA (pfull);
//    builders -> scanners on mbarriers (full, one arrival per builder warp);
//    the two "slot free" hand-offs run on hardware NAMED barriers (bar.sync /
//    bar.arrive): a role that waits for a free slot is descheduled instead of
//    polling an mbarrier (measured: the polling loops of the builders and the
//    prep warp issued ~20% of all instructions of the kernel).
//  * top-k: each scanner warp filters against the query's shared threshold and
//    appends survivors to a private smem buffer; a full buffer is rank-sorted
//    and merged into the warp's PRIVATE sorted list (k <= 128), whose k-th key
//    lowers the query's threshold with a shared atomicMin.  The last warp to
//    finish a query merges the SW private lists and writes the results.
//    k > 128: one shared list per query, merged under a per-query lock.
#pragma once
#include <stdint.h>

#include "codec.cuh"
#include "scan.cuh"

namespace ivfpq {

// Checked build (-DIVFPQ_CHECKED, harness/checked_run.sh): device-side bounds
// and protocol assertions that trap on violation.  compute-sanitizer is closed
// on this GPU pool, so this build plus the CPU-oracle parity tests stand in for
// memcheck / racecheck.  Compiled out of the product library.
#ifdef IVFPQ_CHECKED
#define WS_CHECK(cond)          \
    do {                        \
        if (!(cond)) __trap();  \
    } while (0)
#else
#define WS_CHECK(cond) \
    do {               \
    } while (0)
#endif

// Warp layout of the CTA: BW builder warps (a multiple of 4: TMEM lane
// quarters), SW scanner warps, one prep warp.  Two layouts are built:
//  * WsCfgA = 8 + 11: LUT-build-heavy shapes (cfg2: ~1.7 lookups per entry);
//  * WsCfgB = 4 + 15: scan-heavy shapes (cfg5: 8 KiB LUTs and ~10-20 lookups
//    per entry; the 8 builder warps of layout A idle ~40% of the time there
//    while the scanners wait on the code stream).
template <int BW_, int SW_, bool SCAN_PF_>
struct WsCfg {
    static constexpr int BW = BW_;                     // builder warps
    static constexpr int SW = SW_;                     // scanner warps
    static constexpr bool SCAN_PF = SCAN_PF_;          // scanners bulk-prefetch codes ahead (code store > L2)
    static constexpr int NB = BW * 32;                 // builder threads
    static constexpr int PREP = BW + SW;               // the prep warp
    static constexpr int THREADS = (BW + SW + 1) * 32;
    static constexpr int BAR_EMPTY_N = NB + SW * 32;   // participants of a slot-free barrier
    static constexpr int BAR_PEMPTY_N = NB + 32;       // participants of a ring-entry barrier
    // Builder row geometry (shared by host plan and device): a builder thread
    // owns a quad of codes and ceil(s / R(N)) subspace rows, at most JPT(sub_d).
    __host__ __device__ static constexpr int R(int N) { return NB * 4 / N; }
    __host__ __device__ static constexpr int JPT(int sub_d) { return 64 / (sub_d * BW / 4); }
    static_assert(BW % 4 == 0, "builder warps fill TMEM lane quarters");
};
using WsCfgA = WsCfg<8, 11, false>;
using WsCfgB = WsCfg<4, 15, true>;

constexpr int WS_MAX_G = 8;
constexpr int WS_MAX_NBUF = 6;
#ifndef WS_NQS_CFG
#define WS_NQS_CFG 4
#endif
constexpr int WS_NQS = WS_NQS_CFG;           // per-query states (query top-k lists) in flight, at most
// query states in flight for k: 4, or 2 when the private per-warp lists are long (k > 32)
__host__ __device__ constexpr int ws_nqs(int K) { return K <= 32 ? WS_NQS : 2; }
constexpr int WS_PD = 8;                     // prep ring depth (jobs prepared ahead)
#ifndef WS_WBUF_CFG
#define WS_WBUF_CFG 64
#endif
constexpr int WS_WBUF = WS_WBUF_CFG;         // per-warp candidate buffer
constexpr int WS_MAX_K = 512;
constexpr int WS_PRIV_K = 128;               // K up to which every scanner warp keeps private top-k lists
#ifndef WS_PLAN_BALANCE
#define WS_PLAN_BALANCE 0                    // 1: ws_plan_kernel groups a query's lists into length-balanced jobs (P <= 32); measured slower, see below
#endif
#ifndef WS_GMEM_PF
#define WS_GMEM_PF 0                         // builders load global-memory codebook rows one iteration ahead (measured: no gain on layout A)
#endif
constexpr int WS_PF_PAIRS = 2;               // L2 prefetch distance, in rounds of pairs (x SW pairs)
// per-warp candidate buffer + sort scratch, each: WBUF keys, or K in the
// private mode (a merged list is written there)
__host__ __device__ constexpr int ws_wsz(int K) { return K <= WS_PRIV_K && K > WS_WBUF ? K : WS_WBUF; }

// Named barriers (16 per CTA; id 0 = __syncthreads):
constexpr int WS_BAR_BUILD = 1;              // builders only (teardown)
constexpr int WS_BAR_EMPTY0 = 2;             // + slot: LUT slot free   (builders sync, scanners arrive)
constexpr int WS_BAR_PEMPTY0 = WS_BAR_EMPTY0 + WS_MAX_NBUF;  // + ring entry: prep entry consumed
static_assert(WS_BAR_PEMPTY0 + WS_PD <= 16, "named barrier ids");


struct WsJob;
struct WsArgs {
    ScanArgs a;            // inputs/outputs shared with the v1 kernel
    const WsJob* plan_jobs;      // [nq][JMAX] job descriptors (ws_plan_kernel)
    const float* plan_rq;        // [nq][JMAX][G][d_pad] residuals
    const int* plan_njobs;       // [nq]
    const long long* plan_ncand; // [nq]
    int JMAX;
    int NBUF;
    int gmem;              // 1: builders read the codebook from global memory (does not fit TMEM)
    int l2pf;              // code store > L2: bit 0 builders bulk-prefetch each job's start into L2,
                           // bit 1 scanners prefetch WS_PF_PAIRS rounds of pairs ahead of their grabs
    long long n_codes_bytes;  // size of the code store (prefetch bound)
    int nqs;               // query states in flight (ws_nqs(K)), from the host
    int wsz;               // per-warp candidate buffer / sort scratch keys (ws_wsz(K)), from the host
    // Row-chunked LUTs (tables larger than the shared-memory budget, e.g. the
    // f32 LUT at s = 240, p = 8: 240 KiB): a group of G lists is processed as
    // nh consecutive jobs, job h holding LUT rows [h*rc, (h+1)*rc) = code
    // chunks [h*rcc, (h+1)*rcc); nh = 1 is the unchunked kernel.
    int nh, rc, rcc;
    int maxp;              // chunked: max pairs one scanner warp owns in a job
    float* part;           // chunked: partial sums [grid][SW][maxp][64] carried between the chunks
    int* work;             // global query counter (zeroed before launch)
};

struct WsJob {
    int qs, q, ng, last, nblk, h;  // h: LUT row chunk of the job (0 unless chunked)
    int pref[WS_MAX_G + 1];
    int len[WS_MAX_G];
    int lc[WS_MAX_G];
    long long off[WS_MAX_G];
};

struct WsPrepQ {  // prep warp's queue of resolved probes (<= 32 + G pending)
    int lc[32 + WS_MAX_G];
    int len[32 + WS_MAX_G];
    long long off[32 + WS_MAX_G];
};

struct WsQuery {
    uint64_t tau;
    long long ncand;
    int lock, done, cur, q;
};

// ---------------------------------------------------------------- PTX helpers
typedef uint64_t u64;
__device__ __forceinline__ u64 pk2(float a, float b) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk2(u64 v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
    u64 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
    u64 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
// Two scalar add.rn.f32 on the halves.  NOT add.rn.f32x2: ptxas (12.9)
// contracts mul.rn.f32x2 -> add.rn.f32x2 into FFMA2 even with --fmad=false,
// which would change the reference's rounding; scalar .rn adds are kept.
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
    u64 r;
    asm("{\n\t.reg .f32 a0, a1, b0, b1;\n\t"
        "mov.b64 {a0, a1}, %1;\n\tmov.b64 {b0, b1}, %2;\n\t"
        "add.rn.f32 a0, a0, b0;\n\tadd.rn.f32 a1, a1, b1;\n\t"
        "mov.b64 %0, {a0, a1};\n\t}"
        : "=l"(r)
        : "l"(a), "l"(b));
    return r;
}
// Packed add with flush-to-zero, for the LUT builders of the 8- and 16-bit
// storage dtypes only.  ptxas does not fuse a mul.rn.f32x2 into an
// add.rn.ftz.f32x2 (the FTZ modes differ; SASS-checked: FMUL2 + FADD2.FTZ),
// and the result is identical after the storage encode: FTZ changes a sum
// only when an operand or the result is below 2^-126, and then either the
// other addend is >= 2^-102 (the flushed part is under half an ulp: same RNE
// result) or the entry is < 2^-101, which f16 and e5m3/e4m4 store as +0
// whether or not it was flushed.  The f32 LUT keeps the exact scalar adds.
__device__ __forceinline__ u64 add2ftz(u64 a, u64 b) {
    u64 r;
    asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
// Packed add of two independent sums: (acc.x + x.x, acc.y + x.y), each one
// fl(acc + x).  Only for addends that are not multiply results (LUT values),
// so there is nothing for ptxas to contract.
__device__ __forceinline__ u64 addx2(u64 a, u64 b) {
    u64 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 mulrzftz2(u64 a, u64 b) {
    u64 r;
    asm("mul.rz.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint32_t min_u16x2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t cvt_f16x2_sat(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

__device__ __forceinline__ uint32_t smem_addr_(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(u64* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar))
                 : "memory");
}
// Wait on an mbarrier phase: try_wait with a suspend-time hint (the warp parks
// in NANOSLEEP.SYNCS and is woken by barrier traffic).
#ifndef WS_WAIT_HINT_NS
#define WS_WAIT_HINT_NS 1000000
#endif
__device__ __forceinline__ void mbar_wait(u64* bar, uint32_t parity) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(a),
        "r"(parity), "n"(WS_WAIT_HINT_NS)
        : "memory");
}
__device__ __forceinline__ bool mbar_try(u64* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr_(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_test(u64* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr_(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// TMA bulk copy global -> this CTA's shared memory, completing on `bar`.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, u64* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_addr_(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// Bulk L2 prefetch of a contiguous global range (16-byte aligned, multiple of 16 bytes).
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
    return r;
}
template <int NB>
__device__ __forceinline__ void bar_builders() { asm volatile("bar.sync %0, %1;" ::"n"(WS_BAR_BUILD), "n"(NB) : "memory"); }
// Named-barrier hand-off: the consumer of a free slot waits with bar.sync (the
// warp is descheduled, no polling), the releasing role signals with bar.arrive.
__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void lds_f32x2(uint32_t a, float& x, float& y) {
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
}
__device__ __forceinline__ void lds_f32x4(uint32_t a, float& x, float& y, float& z, float& w) {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
}
__device__ __forceinline__ void sts_b32(uint32_t a, uint32_t v) { asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v)); }
__device__ __forceinline__ void sts_v2(uint32_t a, uint32_t x, uint32_t y) {
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y));
}
__device__ __forceinline__ void sts_v4f(uint32_t a, float x, float y, float z, float w) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w));
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---- tensor memory (TMEM): the codebook lives here, one 32-bit column per
// float, builder thread (w, i) in lane 32*(w%4)+i, column half w/4.
template <int NCOL>
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "n"(NCOL));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <int NCOL>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOL));
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <int X>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&r)[X]) {
    if constexpr (X == 4) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                     : "r"(taddr));
    } else if constexpr (X == 8) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(taddr));
    } else {
        static_assert(X == 16, "x4 / x8 / x16 only");
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
    }
}
template <int X>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t (&r)[X]) {
    if constexpr (X == 4) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(r[0]),
                     "r"(r[1]), "r"(r[2]), "r"(r[3]));
    } else if constexpr (X == 8) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                     "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    } else {
        static_assert(X == 16, "x4 / x8 / x16 only");
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15, %16};" ::"r"(taddr),
            "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
            "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
    }
}

// --------------------------------------------------------------- smem layout
template <class C>
struct WsLayout {
    // lut rows are padded to R * jpt (jpt = ceil(s_pad / R)) so every builder
    // thread runs the same number of rows; rq vectors likewise to R*jpt*sub_d
    // (row-chunked jobs: rc rows, a multiple of R and of 16, dividing s_pad).
    // Rows j >= s hold +0 entries (zero centers, zero residual), so the scan
    // reads whole 16-code chunks: the zero-code lookups past s add +0, which
    // leaves every sum bit-identical.
    size_t bars, qfree, tmem, cnt, jobs, pjobs, prepq, qst, lists, wbuf, prq, lut, total, lut_each, d_pad;
    // rc: LUT rows held per job (row-chunked jobs), 0 = all R * jpt rows.
    __host__ __device__ WsLayout(int d, int s, int sub_d, int logn, int esize, int G, int NBUF, int K, int s_pad,
                                 int rc = 0) {
        const int N = 1 << logn, R = C::R(N), jpt = (s_pad + R - 1) / R;
        (void)d;
        (void)s;
        const int rows = rc > 0 ? rc : R * jpt;
        lut_each = (((size_t)rows * N * esize) + 255) & ~(size_t)255;  // 256-aligned (PRMT addressing)
        d_pad = (size_t)rows * sub_d;
        bars = 0;                                                         // pfull[PD], full[MAX_NBUF]
        qfree = (WS_PD + WS_MAX_NBUF) * 8;                                // query-state free barriers [NQS]
        tmem = qfree + WS_NQS * 8;                                        // u32: TMEM base address
        cnt = tmem + 16;                                                  // int[MAX_NBUF]: next pair of each slot
        jobs = cnt + 32;                                                  // WsJob[MAX_NBUF] (LUT slots)
        pjobs = jobs + WS_MAX_NBUF * sizeof(WsJob);                       // WsJob[PD] (prep ring, TMA-filled)
        pjobs = (pjobs + 127) & ~(size_t)127;
        prepq = pjobs + WS_PD * sizeof(WsJob);                            // int[PD]: query state of each prep entry
        qst = prepq + WS_PD * 4;                                          // WsQuery[NQS]
        qst = (qst + 15) & ~(size_t)15;
        lists = qst + WS_NQS * sizeof(WsQuery);                           // top-k lists (WarpTopK):
        lists = (lists + 15) & ~(size_t)15;                               //  u64[SW][nqs][K] (K <= WS_PRIV_K)
        wbuf = lists + (size_t)(K <= WS_PRIV_K ? C::SW * ws_nqs(K) * K : WS_NQS * 2 * K) * 8;  // or [NQS][2][K]
        //                                                                   u64[SW][2][wsz]
        prq = wbuf + (size_t)C::SW * 2 * ws_wsz(K) * 8;                   // f32[PD][G][d_pad] (TMA-filled)
        prq = (prq + 127) & ~(size_t)127;
        lut = prq + (size_t)WS_PD * G * d_pad * 4;                        // [NBUF][G][lut_each]
        lut = (lut + 255) & ~(size_t)255;
        total = lut + (size_t)NBUF * G * lut_each;
    }
};

// ------------------------------------------------------------- the builders
// Builder thread t owns codes m = 4u..4u+3 (u = t % (N/4)) of subspaces
// j = jr + R*i (jr = t / (N/4), R = 1024/N), i < jpt.  Its centers live in
// TMEM: for owned row i, CPI columns hold c[m0..m0+3][0..SUB_D) (pairs packed
// as (c[m0][x], c[m0+1][x]), (c[m0+2][x], c[m0+3][x])).
template <class C, int DT, int LOGN, int SUB_D, bool GMEM>
struct WsBuild {
    static constexpr int N = 1 << LOGN;
    static constexpr int NQ4 = N / 4;                                   // quads per subspace row
    static constexpr int R = C::R(N);                                   // row groups
    static constexpr int JPT = C::JPT(SUB_D);                           // max owned rows (host-checked)
    static constexpr int CPI = SUB_D == 1 ? 4 : SUB_D == 2 ? 8 : 16;    // TMEM columns per owned row
    static constexpr int HALF = JPT * CPI;                              // columns per builder column group
    static constexpr int NGRP = C::BW / 4;                              // warps sharing a TMEM lane quarter
    static constexpr int NCOL = NGRP * HALF <= 256 ? 256 : 512;         // TMEM allocation
    static_assert(NGRP * HALF <= 512, "codebook does not fit TMEM");
    using T = typename LutTraits<DT>::T;

    int u, jr;
    uint32_t tbase;  // this thread's TMEM address (lane quarter | column half)
    // Codebooks too large for TMEM (rows per thread > JPT, e.g. cfg3 p8: 960
    // KiB) are read per job from global memory (L2-resident) instead: gc !=
    // nullptr.  Same packing as the TMEM columns.
    const float* gc;
    int s_;

    __device__ void init(const float* __restrict__ centers, int s, int t, uint32_t tmem, bool gmem) {
        const int w = t >> 5;
        u = t % NQ4;
        jr = t / NQ4;
        tbase = tmem + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)((w >> 2) * HALF);
        (void)gmem;
        gc = GMEM ? centers : nullptr;
        s_ = s;
        if (GMEM) return;
#pragma unroll 1
        for (int i = 0; i < JPT; ++i) {
            const int j = jr + R * i;
            uint32_t r[CPI];
#pragma unroll
            for (int k = 0; k < CPI; ++k) r[k] = 0u;
            if (j < s) {
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int x = 0; x < SUB_D; ++x) {
                        const size_t e = (size_t)j * N + 4 * u + 2 * h;
                        r[(h * SUB_D + x) * 2 + 0] = __float_as_uint(__ldg(centers + e * SUB_D + x));
                        r[(h * SUB_D + x) * 2 + 1] = __float_as_uint(__ldg(centers + (e + 1) * SUB_D + x));
                    }
            }
            tmem_st<CPI>(tbase + i * CPI, r);
        }
        tmem_wait_st();
    }

    // One owned row's centers in the TMEM column packing: r[(h*SUB_D + x)*2 + e]
    // = c[4u + 2h + e][x] (zeros past the last subspace).
    __device__ __forceinline__ void row(int i, uint32_t (&r)[CPI]) const {
        if constexpr (!GMEM) {
            tmem_ld<CPI>(tbase + i * CPI, r);
            return;
        }
        const int j = jr + R * i;
#pragma unroll
        for (int k = 0; k < CPI; ++k) r[k] = 0u;
        if (j < s_) {
            // the quad's 4 x SUB_D floats are contiguous and 16-byte aligned:
            // SUB_D vector loads (a warp reads 32 x 16 B per instruction)
            const float4* src = reinterpret_cast<const float4*>(gc + ((size_t)j * N + 4 * u) * SUB_D);
            float f[4 * SUB_D];
#pragma unroll
            for (int q = 0; q < SUB_D; ++q) {
                const float4 v = __ldg(src + q);
                f[4 * q + 0] = v.x;
                f[4 * q + 1] = v.y;
                f[4 * q + 2] = v.z;
                f[4 * q + 3] = v.w;
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int x = 0; x < SUB_D; ++x) {
                    r[(h * SUB_D + x) * 2 + 0] = __float_as_uint(f[(2 * h) * SUB_D + x]);
                    r[(h * SUB_D + x) * 2 + 1] = __float_as_uint(f[(2 * h + 1) * SUB_D + x]);
                }
        }
    }

    // The LUTs of ng lists: rq[g] (smem, d_pad floats) -> lut[g] (smem, R*jpt
    // rows of N).  Centers of row i are read from TMEM once and reused for
    // every list of the job.  The residual loads and table stores are plain
    // C++ shared-memory accesses (not volatile asm), so ptxas can interleave
    // the independent entry chains of the two rows and of consecutive lists.
    // Rows i0 .. i0+jpt-1 of the thread's owned rows (a row chunk); rq and lut
    // hold the chunk only (local row il = i - i0).
    __device__ __forceinline__ void build(const uint8_t* rq, uint32_t rq_stride, uint8_t* lut, uint32_t lut_stride,
                                          int ng, int jpt, int i0) const {
        constexpr int E = sizeof(T);
        const uint8_t* rqb = rq + (size_t)jr * SUB_D * 4;
        uint8_t* lb = lut + ((size_t)jr * N + 4 * u) * E;
        // two owned rows per iteration: 2 x ng independent entry chains in flight
        int i = 0;
        // Codebook in global memory (L2-resident), WS_GMEM_PF: the next
        // iteration's two rows are loaded while this one computes (4 rows in
        // flight per thread).  cfg3 p8: 53% of the builders' stall samples are
        // long-scoreboard waits on these loads, but the builders also wait 30%
        // of the time for free slots on layout A, and the prefetch's spills
        // cost more than it saves there (78.8 -> 80.5 ms); off by default.
        uint32_t pf0[CPI], pf1[CPI];
        if constexpr (GMEM && WS_GMEM_PF) {
            row(i0, pf0);
            row(i0 + 1, pf1);
        }
#pragma unroll 1
        for (; i + 2 <= jpt; i += 2) {
            uint32_t c0[CPI], c1[CPI];
            if constexpr (GMEM && WS_GMEM_PF) {
#pragma unroll
                for (int k = 0; k < CPI; ++k) {
                    c0[k] = pf0[k];
                    c1[k] = pf1[k];
                }
                // rows past the chunk / the thread's share read valid rows or zeros
                row(i0 + i + 2, pf0);
                row(i0 + i + 3, pf1);
            } else {
                row(i0 + i, c0);
                row(i0 + i + 1, c1);
            }
            if constexpr (!GMEM) tmem_wait_ld();
            u64 cenA[2][SUB_D], cenB[2][SUB_D];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int x = 0; x < SUB_D; ++x) {
                    cenA[h][x] = pk2(__uint_as_float(c0[(h * SUB_D + x) * 2]), __uint_as_float(c0[(h * SUB_D + x) * 2 + 1]));
                    cenB[h][x] = pk2(__uint_as_float(c1[(h * SUB_D + x) * 2]), __uint_as_float(c1[(h * SUB_D + x) * 2 + 1]));
                }
            const uint8_t* raA = rqb + i * R * SUB_D * 4;
            const uint8_t* raB = raA + R * SUB_D * 4;
            uint8_t* laA = lb + (size_t)i * R * N * E;
            uint8_t* laB = laA + (size_t)R * N * E;
            // software-pipelined: the residuals of list g+1 are loaded before the
            // stores of list g (the stores may alias them as far as ptxas knows);
            // reading one list past the last is inside shared memory
            float rA[SUB_D], rB[SUB_D];
            load_rq(raA, rA);
            load_rq(raB, rB);
#ifndef WS_GUNROLL
#define WS_GUNROLL 2
#endif
            constexpr int kGU = WS_GUNROLL;  // lists per unrolled step (experiment knob)
#pragma unroll kGU
            for (int g = 0; g < ng; ++g) {
                float nA[SUB_D], nB[SUB_D];
                load_rq(raA + (g + 1) * rq_stride, nA);
                load_rq(raB + (g + 1) * rq_stride, nB);
                entry_quad(cenA, rA, laA + g * lut_stride);
                entry_quad(cenB, rB, laB + g * lut_stride);
#pragma unroll
                for (int x = 0; x < SUB_D; ++x) {
                    rA[x] = nA[x];
                    rB[x] = nB[x];
                }
            }
        }
        if (i < jpt) {
            uint32_t c[CPI];
            row(i0 + i, c);
            if constexpr (!GMEM) tmem_wait_ld();
            u64 cen[2][SUB_D];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int x = 0; x < SUB_D; ++x)
                    cen[h][x] = pk2(__uint_as_float(c[(h * SUB_D + x) * 2]), __uint_as_float(c[(h * SUB_D + x) * 2 + 1]));
            const uint8_t* ra0 = rqb + i * R * SUB_D * 4;
            uint8_t* la0 = lb + (size_t)i * R * N * E;
            float r0[SUB_D];
            load_rq(ra0, r0);
#pragma unroll 4
            for (int g = 0; g < ng; ++g) {
                float n0[SUB_D];
                load_rq(ra0 + (g + 1) * rq_stride, n0);
                entry_quad(cen, r0, la0 + g * lut_stride);
#pragma unroll
                for (int x = 0; x < SUB_D; ++x) r0[x] = n0[x];
            }
        }
    }

    // Four LUT entries (codes 4u..4u+3 of one subspace row) for one list:
    // T = seq_x fl(acc + fl(fl(c - rq)^2)), then the storage encode.
    __device__ __forceinline__ static void load_rq(const uint8_t* ra, float (&r)[SUB_D]) {
        if constexpr (SUB_D == 2) {
            const float2 v = *reinterpret_cast<const float2*>(ra);
            r[0] = v.x;
            r[1] = v.y;
        } else if constexpr (SUB_D == 4) {
            const float4 v = *reinterpret_cast<const float4*>(ra);
            r[0] = v.x;
            r[1] = v.y;
            r[2] = v.z;
            r[3] = v.w;
        } else {
#pragma unroll
            for (int x = 0; x < SUB_D; ++x) r[x] = reinterpret_cast<const float*>(ra)[x];
        }
    }

    __device__ __forceinline__ static void entry_quad(const u64 (&cen)[2][SUB_D], const float (&r)[SUB_D], uint8_t* dst) {
        u64 acc0 = 0, acc1 = 0;
#pragma unroll
        for (int x = 0; x < SUB_D; ++x) {
            const u64 rr = pk2(r[x], r[x]);
            const u64 d0 = sub2(cen[0][x], rr), d1 = sub2(cen[1][x], rr);
            const u64 q0 = mul2(d0, d0), q1 = mul2(d1, d1);
            // acc starts at +0: fl(0 + q) = q exactly (q >= +0)
            if constexpr (DT == LUT_F32) {
                acc0 = x == 0 ? q0 : add2(acc0, q0);
                acc1 = x == 0 ? q1 : add2(acc1, q1);
            } else {
                acc0 = x == 0 ? q0 : add2ftz(acc0, q0);
                acc1 = x == 0 ? q1 : add2ftz(acc1, q1);
            }
        }
        store(dst, acc0, acc1);
    }

    __device__ __forceinline__ static void store(uint8_t* dst, u64 a01, u64 a23) {
        if constexpr (DT == LUT_F32) {
            float a0, a1, a2, a3;
            upk2(a01, a0, a1);
            upk2(a23, a2, a3);
            *reinterpret_cast<float4*>(dst) = make_float4(a0, a1, a2, a3);
        } else if constexpr (DT == LUT_F16) {
            float a0, a1, a2, a3;
            upk2(a01, a0, a1);
            upk2(a23, a2, a3);
            *reinterpret_cast<uint2*>(dst) = make_uint2(cvt_f16x2_sat(a0, a1), cvt_f16x2_sat(a2, a3));
        } else {
            constexpr int M = LutTraits<DT>::m, BIAS = LutTraits<DT>::bias;
            // y = x * 2^-(127-bias), round-toward-zero + flush-to-zero: exact
            // for x >= min_normal, +0 below it (never rounds up into range).
            const float sc = __uint_as_float((uint32_t)(127 - (127 - BIAS)) << 23);
            const u64 s2 = pk2(sc, sc);
            const u64 y01 = mulrzftz2(a01, s2), y23 = mulrzftz2(a23, s2);
            float f0, f1, f2, f3;
            upk2(y01, f0, f1);
            upk2(y23, f2, f3);
            // code = min(bits >> (23-M), 255) = min(bits >> 16, lim) >> (7-M), two per u16x2
            constexpr uint32_t lim = (256u << (7 - M)) - 1u;  // 0x0FFF (m=3) / 0x07FF (m=4)
            uint32_t h01 = __byte_perm(__float_as_uint(f0), __float_as_uint(f1), 0x7632);
            uint32_t h23 = __byte_perm(__float_as_uint(f2), __float_as_uint(f3), 0x7632);
            h01 = min_u16x2(h01, lim | (lim << 16)) >> (7 - M);
            h23 = min_u16x2(h23, lim | (lim << 16)) >> (7 - M);
            *reinterpret_cast<uint32_t*>(dst) = __byte_perm(h01, h23, 0x6420);
        }
    }
};

// ------------------------------------------------------------- warp top-k
// Top-k state per query.  Two layouts, chosen by K at launch:
//  * K <= WS_PRIV_K ("private"): every scanner warp keeps its OWN sorted top-K
//    per query state (lists[warp][qs][K]; 2 query states in flight for K > 32); a flush merges the warp's buffer
//    into it and publishes its K-th key with a shared atomicMin into the
//    query's threshold tau.  tau = min over warps of their K-th key is a valid
//    filter: a key >= some warp's K-th key has K (unique) keys below it.  No
//    lock; at the query's end the last warp merges the SW private lists.
//  * larger K (up to WS_MAX_K): one shared double-buffered list per query
//    (lists[qs][2][K]) merged under a per-query lock (smem budget: SW x K keys
//    per query state would not fit next to the LUT slots).
struct WarpTopK {
    u64* buf;      // WS_WBUF
    u64* srt;      // WS_WBUF
    int n;         // warp-uniform count
    u64* priv;     // private mode: this warp's lists[sw][0..NQS)[K], else null

    __device__ __forceinline__ void offer(u64 key, bool pred) {
        const unsigned m = __ballot_sync(0xffffffffu, pred);
        WS_CHECK(n + __popc(m) <= WS_WBUF);
        if (pred) buf[n + __popc(m & ((1u << (threadIdx.x & 31)) - 1))] = key;
        n += __popc(m);
    }

    // Merge the buffer into the query's list (private or shared).  Candidates
    // are first re-filtered against the current threshold (it has usually
    // tightened since they were offered), so most flushes end early.
    // Inlined: out of line it costs ~25% (call-site register spills, measured).
    __device__ __forceinline__ void flush(WsQuery* S, u64* lists, int qs, int K) {
        const int lane = threadIdx.x & 31;
        __syncwarp();
        const u64 tau = *(volatile u64*)&S->tau;
        int m = 0;
        for (int i0 = 0; i0 < n; i0 += 32) {
            const u64 x = i0 + lane < n ? buf[i0 + lane] : ~0ull;
            const bool keep = x < tau;
            const unsigned bm = __ballot_sync(0xffffffffu, keep);
            if (keep) srt[m + __popc(bm & ((1u << lane) - 1))] = x;
            m += __popc(bm);
        }
        n = 0;
        if (m == 0) return;
        __syncwarp();
        // rank sort (keys are unique here: distinct vector ids)
        for (int i = lane; i < m; i += 32) {
            const u64 x = srt[i];
            int r = 0;
            for (int j = 0; j < m; ++j) r += srt[j] < x;
            buf[r] = x;
        }
        __syncwarp();
        if (priv) {
            // merge-path of the warp's list P (K) and the sorted run buf (m) into srt
            u64* P = priv + (size_t)qs * K;
            for (int i = lane; i < K; i += 32) {
                const u64 a = P[i];
                const int pos = i + lower_bound_u64(buf, m, a);
                if (pos < K) srt[pos] = a;
            }
            for (int i = lane; i < m; i += 32) {
                const u64 b = buf[i];
                const int pos = i + lower_bound_u64(P, K, b);
                if (pos < K) srt[pos] = b;
            }
            __syncwarp();
            for (int i = lane; i < K; i += 32) P[i] = srt[i];
            __syncwarp();
            if (lane == 0 && srt[K - 1] != ~0ull) atomicMin(reinterpret_cast<unsigned long long*>(&S->tau), srt[K - 1]);
            __syncwarp();
            return;
        }
        for (int i = lane; i < m; i += 32) srt[i] = buf[i];
        if (lane == 0) {
            // contended: back off so the spinning warp does not take issue slots
            while (atomicCAS(&S->lock, 0, 1) != 0) __nanosleep(64);
            __threadfence_block();
        }
        __syncwarp();
        u64* qlist = lists + (size_t)qs * 2 * K;
        const int cur = *(volatile int*)&S->cur;
        const u64* A = qlist + (size_t)cur * K;
        u64* O = qlist + (size_t)(cur ^ 1) * K;
        for (int i = lane; i < K; i += 32) {
            const u64 a = A[i];
            const int pos = i + lower_bound_u64(srt, m, a);
            if (pos < K) O[pos] = a;
        }
        for (int i = lane; i < m; i += 32) {
            const u64 b = srt[i];
            const int pos = i + lower_bound_u64(A, K, b);
            if (pos < K) O[pos] = b;
        }
        __syncwarp();
        if (lane == 0) {
            *(volatile int*)&S->cur = cur ^ 1;
            *(volatile u64*)&S->tau = O[K - 1];
            __threadfence_block();
            atomicExch(&S->lock, 0);
        }
        __syncwarp();
    }
};

// ---------------------------------------------------------------- scanners
// One LUT gather + widen.  fp8 with N >= 16: the LUT base is 256-byte aligned,
// so PRMT builds the address (base | code) in one instruction and the row
// offset b*N rides in the LDS immediate.
template <int DT, int LOGN, int B>
__device__ __forceinline__ float ws_gather(uint32_t word, uint32_t base) {
    constexpr int N = 1 << LOGN;
    constexpr int OFF = (B << LOGN) * (int)sizeof(typename LutTraits<DT>::T);
    if constexpr (DT == LUT_E5M3 || DT == LUT_E4M4) {
        uint32_t v;
        if constexpr (N >= 16) {
            const uint32_t addr = __byte_perm(word, base, 0x7650u | (B & 3));
            asm volatile("ld.shared.u8 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(OFF));
        } else {
            const uint32_t addr = base + __byte_perm(word, 0u, 0x4440u | (B & 3));
            asm volatile("ld.shared.u8 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(OFF));
        }
        return __uint_as_float(v << (23 - LutTraits<DT>::m));
    } else if constexpr (DT == LUT_F16) {
        const uint32_t addr = base + (__byte_perm(word, 0u, 0x4440u | (B & 3)) << 1);
        unsigned short h;
        asm volatile("ld.shared.u16 %0, [%1+%2];" : "=h"(h) : "r"(addr), "n"(OFF));
        return __half2float(__ushort_as_half(h));
    } else {
        const uint32_t addr = base + (__byte_perm(word, 0u, 0x4440u | (B & 3)) << 2);
        float v;
        asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(OFF));
        return v;
    }
}

// Two vectors per lane (consecutive blocks of the warp, possibly of two lists
// with LUT bases ba / bb): the two sequential sums advance together in one
// packed add per code -- 3.5 instructions per lookup instead of 4, and two
// independent dependency chains.
template <int DT, int LOGN, int B>
__device__ __forceinline__ u64 ws_acc1x2(u64 acc, uint4 wa, uint4 wb, uint32_t ba, uint32_t bb) {
    const uint32_t xa = B < 4 ? wa.x : B < 8 ? wa.y : B < 12 ? wa.z : wa.w;
    const uint32_t xb = B < 4 ? wb.x : B < 8 ? wb.y : B < 12 ? wb.z : wb.w;
    return addx2(acc, pk2(ws_gather<DT, LOGN, B>(xa, ba), ws_gather<DT, LOGN, B>(xb, bb)));
}

template <int DT, int LOGN>
__device__ __forceinline__ u64 ws_acc16x2(u64 acc, uint4 wa, uint4 wb, uint32_t ba, uint32_t bb) {
    acc = ws_acc1x2<DT, LOGN, 0>(acc, wa, wb, ba, bb);
    acc = ws_acc1x2<DT, LOGN, 1>(acc, wa, wb, ba, bb);
    acc = ws_acc1x2<DT, LOGN, 2>(acc, wa, wb, ba, bb);
    acc = ws_acc1x2<DT, LOGN, 3>(acc, wa, wb, ba, bb);
    acc = ws_acc1x2<DT, LOGN, 4>(acc, wa, wb, ba, bb);
    acc = ws_acc1x2<DT, LOGN, 5>(acc, wa, wb, ba, bb);
    acc = ws_acc1x2<DT, LOGN, 6>(acc, wa, wb, ba, bb);
    acc = ws_acc1x2<DT, LOGN, 7>(acc, wa, wb, ba, bb);
    acc = ws_acc1x2<DT, LOGN, 8>(acc, wa, wb, ba, bb);
    acc = ws_acc1x2<DT, LOGN, 9>(acc, wa, wb, ba, bb);
    acc = ws_acc1x2<DT, LOGN, 10>(acc, wa, wb, ba, bb);
    acc = ws_acc1x2<DT, LOGN, 11>(acc, wa, wb, ba, bb);
    acc = ws_acc1x2<DT, LOGN, 12>(acc, wa, wb, ba, bb);
    acc = ws_acc1x2<DT, LOGN, 13>(acc, wa, wb, ba, bb);
    acc = ws_acc1x2<DT, LOGN, 14>(acc, wa, wb, ba, bb);
    acc = ws_acc1x2<DT, LOGN, 15>(acc, wa, wb, ba, bb);
    return acc;
}

// A pair of consecutive 32-vector blocks of one job (possibly of two lists
// of the job), as handed to a scanner warp, with this lane's code source:
// chunk c of the lane's vector in block b is at p[b] + c * st[b] (interleaved
// layout).  Lanes past a block's vector count (and the whole
// second block when the job has an odd block count) read a valid vector of
// the pair instead -- their sums are never offered -- so the loads need no
// branches.
struct WsPair {
    uint32_t base0, base1;  // smem address of each block's LUT
    int nb0, nb1;           // vector count of each block (nb1 = 0: no second block)
    int vo0, vo1;           // first vector of each block (a device holds < 2^31 vectors)
    int qs;                 // query state of the job
    const uint8_t* p0;
    const uint8_t* p1;
    uint32_t st0, st1;
    int k, h;               // pair index in the job, the job's row chunk (chunked mode)
};

// A job's list table held lane-parallel (lane g < ng describes list g), read
// once per job: decoding a block is a ballot + 3 shuffles, no smem round trips.
struct WsJobTab {
    int pref;       // first block of list `lane` (INT_MAX for lanes >= ng)
    int len;        // its vector count
    int off;        // its first vector
    int nblk, qs;
    int h;          // the job's LUT row chunk (chunked mode), else 0
    int next;       // chunked mode: this warp's next pair index (static ownership)
    __device__ __forceinline__ void load(const WsJob* J, int lane, int sw) {
        const int ng = J->ng;
        nblk = J->nblk;
        qs = J->qs;
        h = J->h;
        next = sw;
        pref = lane < ng ? J->pref[lane] : 0x7fffffff;
        len = lane < ng ? J->len[lane] : 0;
        off = lane < ng ? (int)J->off[lane] : 0;
    }
    __device__ __forceinline__ void block(int b, int& g, int& nb, int& vo) const {
        const unsigned m = __ballot_sync(0xffffffffu, pref <= b);  // prefs ascend; pref[0] = 0
        WS_CHECK(m != 0u && b >= 0 && b < nblk);
        g = 31 - __clz(m);
        const int pg = __shfl_sync(0xffffffffu, pref, g);
        const int lg = __shfl_sync(0xffffffffu, len, g);
        const int og = __shfl_sync(0xffffffffu, off, g);
        const int vstart = (b - pg) * 32;
        nb = min(32, lg - vstart);
        vo = og + vstart;
    }
};

// Work distribution inside a job.  Unchunked: lane 0 takes the next pair
// index from the slot's counter (reset by the builders when they fill the
// slot), so scanner warps finish a job within one pair of each other.
// Chunked (CH): pair k is always scanned by warp k % SW, in every chunk job of
// its group, so the partial sums it carries between chunks stay with the warp
// (in its own scratch) and chunk h+1 of a pair never starts before chunk h.
template <class C, bool CH>
__device__ __forceinline__ bool ws_grab(WsJobTab& T, int* cnt, int slot, uint32_t slot_base, uint32_t lut_each,
                                        const uint8_t* codes, int s_pad, int rcc, int lane, WsPair& p,
                                        const uint8_t* pf_end) {
    int k = 0;
    if constexpr (CH) {
        k = T.next;
        T.next += C::SW;
    } else {
        if (lane == 0) k = atomicAdd(cnt + slot, 1);
        k = __shfl_sync(0xffffffffu, k, 0);
    }
    if (2 * k >= T.nblk) return false;
    if (C::SCAN_PF && !CH && pf_end != nullptr) {
        // bulk L2 prefetch of the two blocks WS_PF_PAIRS rounds of pairs ahead
        const int bf = 2 * (k + WS_PF_PAIRS * C::SW);
        if (bf < T.nblk) {
            int gf, nbf, vof;
            T.block(bf, gf, nbf, vof);
            const uint8_t* src = codes + (long long)vof * s_pad;
            if (lane == 0) prefetch_l2(src, (uint32_t)min((long long)(64 * s_pad), (long long)(pf_end - src)));
        }
    }
    p.qs = T.qs;
    p.k = k;
    p.h = T.h;
    int g;
    T.block(2 * k, g, p.nb0, p.vo0);
    p.base0 = slot_base + (uint32_t)g * lut_each;
    if (2 * k + 1 < T.nblk) {
        T.block(2 * k + 1, g, p.nb1, p.vo1);
        p.base1 = slot_base + (uint32_t)g * lut_each;
    } else {
        p.base1 = p.base0;
        p.nb1 = 0;
        p.vo1 = p.vo0;
    }
    WS_CHECK(p.nb0 >= 1 && p.nb0 <= 32 && p.nb1 >= 0 && p.nb1 <= 32 && p.vo0 >= 0 && p.vo1 >= 0);
    const int l0 = min(lane, p.nb0 - 1), l1 = min(lane, max(p.nb1 - 1, 0));
    p.st0 = (uint32_t)p.nb0 * 16u;
    p.st1 = (uint32_t)p.nb1 * 16u;
    // chunk 0 of the job's code range is chunk h*rcc of the vector (CH), else 0
    const int c0 = CH ? T.h * rcc : 0;
    p.p0 = codes + (long long)p.vo0 * s_pad + l0 * 16 + c0 * p.st0;
    p.p1 = codes + (long long)p.vo1 * s_pad + l1 * 16 + c0 * p.st1;
    return true;
}

__device__ __forceinline__ uint4 ws_ld(const uint8_t* p, u64 pol) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}

// End of this warp's part of the job in `slot`: at the query's last job, merge
// the warp's candidates and let the last warp write the results and free the
// query state; then release the LUT slot (named barrier, see the header).
template <class C, bool SMALLK>
__device__ __forceinline__ void ws_job_end(const ScanArgs& a, const WsJob* J, WsQuery* qst, u64* lists, int K,
                                           WarpTopK& tk, u64* qfree, int slot, int lane) {
    if (J->last) {
        const int qs = J->qs;
        WsQuery* S = qst + qs;
        if (tk.n > 0) tk.flush(S, lists, qs, K);
        __syncwarp();
        int d = 0;
        if (lane == 0) {
            __threadfence_block();  // this warp's list before its arrival
            d = atomicAdd(&S->done, 1);
        }
        d = __shfl_sync(0xffffffffu, d, 0);
        WS_CHECK(d >= 0 && d < C::SW);
        if (d == C::SW - 1) {
            __threadfence_block();
            const u64* r;
            if (tk.priv) {
                // merge the SW private lists of this query: running result in buf
                const size_t wstride = (size_t)(SMALLK ? WS_NQS : ws_nqs(K)) * K;
                const u64* L0 = lists + (size_t)qs * K;
                for (int i = lane; i < K; i += 32) tk.buf[i] = L0[i];
                for (int w = 1; w < C::SW; ++w) {
                    const u64* Lw = L0 + w * wstride;
                    __syncwarp();
                    for (int i = lane; i < K; i += 32) {
                        const u64 x = tk.buf[i];
                        const int pos = i + lower_bound_u64(Lw, K, x);
                        if (pos < K) tk.srt[pos] = x;
                    }
                    for (int i = lane; i < K; i += 32) {
                        const u64 y = Lw[i];
                        const int pos = i + upper_bound_u64(tk.buf, K, y);
                        if (pos < K) tk.srt[pos] = y;
                    }
                    __syncwarp();
                    for (int i = lane; i < K; i += 32) tk.buf[i] = tk.srt[i];
                }
                __syncwarp();
                r = tk.buf;
            } else {
                r = lists + (size_t)qs * 2 * K + (size_t)(*(volatile int*)&S->cur) * K;
            }
            const int q = S->q;
            const long long nc = S->ncand;
            for (int i = lane; i < K; i += 32) {
                const u64 key = r[i];
                if (a.out_keys) {
                    a.out_keys[(size_t)q * K + i] = key;
                } else {
                    const bool e = key == ~0ull;
                    a.out_ids[(size_t)q * K + i] = e ? -1LL : (long long)(uint32_t)key;
                    a.out_dists[(size_t)q * K + i] = e ? __int_as_float(0x7f800000) : __uint_as_float((uint32_t)(key >> 32));
                }
            }
            if (lane == 0) {
                if (a.out_keys) a.out_ncand[q] = nc;
                else a.out_short[q] = nc < K ? 1 : 0;
            }
            __syncwarp();
            if (tk.priv) {
                for (int i = lane; i < C::SW * K; i += 32)
                    lists[(size_t)(i / K) * (SMALLK ? WS_NQS : ws_nqs(K)) * K + (size_t)qs * K + (i % K)] = ~0ull;
            } else {
                u64* qlist = lists + (size_t)qs * 2 * K;
                for (int i = lane; i < 2 * K; i += 32) qlist[i] = ~0ull;
            }
            __syncwarp();
            if (lane == 0) {
                S->tau = ~0ull;
                S->cur = 0;
                S->done = 0;
                __threadfence_block();
                mbar_arrive(qfree + qs);  // release: state free
            }
        }
    }
    __syncwarp();
    nbar_arrive(WS_BAR_EMPTY0 + slot, C::BAR_EMPTY_N);
}

// Scanner warp main loop.  Per pair: the 2 x min(nch, 4) chunk registers of
// the current pair are consumed one chunk at a time and each freed register
// is immediately refilled with chunk c+4 of the same pair, or (for the last
// four chunks) with the same chunk of the NEXT pair, so the L2 latency of a
// pair's codes hides behind the scan of the previous pair.  The next pair
// comes from the same job, else from the next job if its LUTs are already
// built.  NCH > 0: the chunk count s_pad/16 as a compile-time constant (the
// BASELINE shapes; straight-line code), 0: read from the arguments.
template <class C, int DT, int LOGN, int NCH, bool CH, bool SMALLK>
__device__ void ws_scanner(const ScanArgs& a, const WsArgs& w, WsJob* jobs, int* cnt, u64* full, int NBUF,
                           WsQuery* qst, u64* lists, int K, uint32_t lut_s0, uint32_t slot_bytes, uint32_t lut_each,
                           WarpTopK& tk, u64* qfree, int sw, int lane) {
    constexpr int N = 1 << LOGN;
    constexpr int E = (int)sizeof(typename LutTraits<DT>::T);
    constexpr int NS = NCH == 0 || NCH >= 4 ? 4 : NCH;  // chunk registers per block
    // code chunks (16 codes) per job: all of them (LUT rows >= s are +0, so
    // whole chunks are exact), or a row chunk's rcc
    const int nch = NCH > 0 ? NCH : w.rcc;
    const int rcc = w.rcc, nh = w.nh;
    // chunked: this warp's partial sums, 64 floats (32 lanes x 2 vectors) per owned pair
    u64* part = CH ? reinterpret_cast<u64*>(w.part) + ((size_t)blockIdx.x * C::SW + sw) * w.maxp * 32 + lane : nullptr;
    const int s_pad = a.s_pad;
    u64 pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    const uint8_t* codes = a.codes;
    // end of the code store when the scanners bulk-prefetch into L2 (else null)
    // (compiled in for the layouts that use it only: its pointer costs
    // registers, and the layout-A kernels spill without it otherwise)
    const uint8_t* pf_end = C::SCAN_PF && (w.l2pf & 2) ? codes + (size_t)w.n_codes_bytes : nullptr;
    uint4 A[NS], B[NS];
    uint32_t idA = 0, idB = 0;
    int slot = 0, ph = 0;
    WsPair cur, nxt;
    WsJobTab ct, nt;
    mbar_wait(full, 0);
    if (jobs[0].qs < 0) return;
    ct.load(jobs, lane, sw);
    bool have = ws_grab<C, CH>(ct, cnt, 0, lut_s0, lut_each, codes, s_pad, rcc, lane, cur, pf_end);
    auto load_first = [&](const WsPair& p) {
#pragma unroll
        for (int u = 0; u < NS; ++u)
            if (u < nch) {
                A[u] = ws_ld(p.p0 + u * p.st0, pol);
                B[u] = ws_ld(p.p1 + u * p.st1, pol);
            }
        idA = lane < p.nb0 ? __ldg(a.ids + p.vo0 + lane) : 0u;
        idB = lane < p.nb1 ? __ldg(a.ids + p.vo1 + lane) : 0u;
    };
    if (have) load_first(cur);
    while (true) {
        if (!have) {
            ws_job_end<C, SMALLK>(a, jobs + slot, qst, lists, K, tk, qfree, slot, lane);
            if (++slot == NBUF) {
                slot = 0;
                ph ^= 1;
            }
            mbar_wait(full + slot, ph);
            if (jobs[slot].qs < 0) break;
            ct.load(jobs + slot, lane, sw);
            have = ws_grab<C, CH>(ct, cnt, slot, lut_s0 + (uint32_t)slot * slot_bytes, lut_each, codes, s_pad, rcc, lane,
                               cur, pf_end);
            if (have) load_first(cur);
            continue;
        }
        // ---- the next pair: same job, else the next job if its LUTs are ready
        bool hn = ws_grab<C, CH>(ct, cnt, slot, lut_s0 + (uint32_t)slot * slot_bytes, lut_each, codes, s_pad, rcc, lane,
                              nxt, pf_end);
        bool cross = false;
        if (!hn) {
            const int ns = slot + 1 == NBUF ? 0 : slot + 1;
            const int nph = slot + 1 == NBUF ? ph ^ 1 : ph;
            // (NBUF = 1: the "next" slot is this one; its previous phase would
            // test as complete, so there is no cross-job prefetch)
            if (NBUF > 1 && mbar_test(full + ns, (uint32_t)nph) && jobs[ns].qs >= 0) {
                nt.load(jobs + ns, lane, sw);
                hn = ws_grab<C, CH>(nt, cnt, ns, lut_s0 + (uint32_t)ns * slot_bytes, lut_each, codes, s_pad, rcc, lane,
                                 nxt, pf_end);
                cross = true;  // (an empty next job is left to the blocking path)
            }
        }
        // without a next pair the refills re-read the current pair (L2 hits, discarded)
        const uint8_t* n0 = hn ? nxt.p0 : cur.p0;
        const uint8_t* n1 = hn ? nxt.p1 : cur.p1;
        const uint32_t ns0 = hn ? nxt.st0 : cur.st0, ns1 = hn ? nxt.st1 : cur.st1;
        const uint32_t nidA = hn && lane < nxt.nb0 ? __ldg(a.ids + nxt.vo0 + lane) : 0u;
        const uint32_t nidB = hn && lane < nxt.nb1 ? __ldg(a.ids + nxt.vo1 + lane) : 0u;
        // ---- scan the current pair
        const uint32_t base0 = cur.base0, base1 = cur.base1;
        u64 acc = pk2(0.f, 0.f);
        // chunked: continue the sums of this pair's earlier row chunks (sequential in j)
        if (CH && cur.h > 0) acc = part[(size_t)((cur.k - sw) / C::SW) * 32];
#pragma unroll(NCH > 0 ? 1 : 1)
        for (int cg = 0; cg < nch; cg += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = cg + u;
                if (u < NS && c < nch) {
                    const uint32_t o = (uint32_t)(c * 16 * N * E);
                    acc = ws_acc16x2<DT, LOGN>(acc, A[u], B[u], base0 + o, base1 + o);
                    const bool same = c + 4 < nch;
                    A[u] = ws_ld(same ? cur.p0 + (c + 4) * cur.st0 : n0 + u * ns0, pol);
                    B[u] = ws_ld(same ? cur.p1 + (c + 4) * cur.st1 : n1 + u * ns1, pol);
                }
            }
        }
        // ---- offers against the query's shared threshold (chunked: after the last chunk)
        if (CH && cur.h < nh - 1) {
            part[(size_t)((cur.k - sw) / C::SW) * 32] = acc;
        } else {
            float r0, r1;
            upk2(acc, r0, r1);
            const int qs = cur.qs;
            WsQuery* S = qst + qs;
            const u64 tau = *(volatile u64*)&S->tau;
            const u64 k0 = ((u64)__float_as_uint(lut_finish<DT>(r0)) << 32) | idA;
            const u64 k1 = ((u64)__float_as_uint(lut_finish<DT>(r1)) << 32) | idB;
            tk.offer(k0, lane < cur.nb0 && k0 < tau);
            if (tk.n > WS_WBUF - 32) tk.flush(S, lists, qs, K);
            tk.offer(k1, lane < cur.nb1 && k1 < tau);
            if (tk.n > WS_WBUF - 32) tk.flush(S, lists, qs, K);
        }
        if (!hn) {
            have = false;
            continue;
        }
        if (cross) {  // this warp's part of the current job is done
            ws_job_end<C, SMALLK>(a, jobs + slot, qst, lists, K, tk, qfree, slot, lane);
            if (++slot == NBUF) {
                slot = 0;
                ph ^= 1;
            }
            ct = nt;
        }
        cur = nxt;
        idA = nidA;
        idB = nidB;
    }
}

// ---------------------------------------------------------------- planning
// One warp per query: resolve the probe keys (32 at a time) to owned,
// non-empty lists, group them G per job, and write each job's descriptor and
// its G padded residual rows rq = fl(q - coarse[c]) to global memory, where
// the search kernel's prep warp fetches them with two TMA bulk copies.
// Also the query's job count and candidate count (all probes, owned or not).
__global__ void __launch_bounds__(256) ws_plan_kernel(const ScanArgs a, int G, int d_pad, int JMAX, int nh, WsJob* jobs,
                                                      float* rq, int* njobs, long long* ncand)
#ifndef IVFPQ_DEFINE_PLAN_KERNEL
    ;  // defined in ivfpq_b200.cu
#else
{
    __shared__ int s_lc[8][32 + WS_MAX_G];
    __shared__ int s_len[8][32 + WS_MAX_G];
    __shared__ long long s_off[8][32 + WS_MAX_G];
    const int wq = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = blockIdx.x * 8 + wq;
    if (q >= a.nq) return;
    int* lcq = s_lc[wq];
    int* lenq = s_len[wq];
    long long* offq = s_off[wq];
    const u64* probes = a.probes + (size_t)q * a.P;
    const float* qv = a.queries + (size_t)q * a.d;
    int pend = 0, nj = 0;
    long long nc = 0;
    // One group of ng lists = nh jobs (row chunks h = 0..nh-1; nh = 1 unless
    // the LUT is row-chunked).  Job h's residual block holds the chunk's slice
    // of every list's rq (d_pad floats each), so the prep's TMA copy stays one
    // contiguous range.
    auto emit = [&](int from, int ng, bool last) {
        WS_CHECK(nj + nh <= JMAX && ng <= G);
        for (int h = 0; h < nh; ++h) {
            WsJob* J = jobs + (size_t)q * JMAX + nj + h;
            if (lane == 0) {
                int pref = 0;
                for (int g = 0; g < ng; ++g) {
                    J->lc[g] = lcq[from + g];
                    J->len[g] = lenq[from + g];
                    J->off[g] = offq[from + g];
                    J->pref[g] = pref;
                    pref += (lenq[from + g] + 31) >> 5;
                }
                J->pref[ng] = pref;
                J->nblk = pref;
                J->ng = ng;
                J->q = q;
                J->qs = 0;
                J->h = h;
                J->last = last && h == nh - 1 ? 1 : 0;
            }
            float* r = rq + ((size_t)q * JMAX + nj + h) * G * d_pad;
            for (int g = 0; g < ng; ++g) {
                const float* cv = a.coarse + (size_t)lcq[from + g] * a.d;
                for (int x = lane; x < d_pad; x += 32) {
                    const int t = h * d_pad + x;
                    r[g * d_pad + x] = t < a.d ? __fsub_rn(qv[t], cv[t]) : 0.0f;
                }
            }
        }
        nj += nh;
    };
    for (int base = 0; base < a.P; base += 32) {
        const int pi = base + lane;
        const u64 key = pi < a.P ? probes[pi] : ~0ull;
        const uint32_t gid = (uint32_t)key;
        const int lc = key == ~0ull ? -1 : a.g2l[gid];
        long long o = 0, len = 0, gl = key == ~0ull ? 0 : a.glen[gid];
        if (lc >= 0) {
            o = a.off[lc];
            len = a.off[lc + 1] - o;
        }
        for (int sh = 16; sh; sh >>= 1) gl += __shfl_xor_sync(0xffffffffu, gl, sh);
        nc += gl;
        const unsigned m = __ballot_sync(0xffffffffu, len > 0);
        if (len > 0) {
            const int at = pend + __popc(m & ((1u << lane) - 1));
            lcq[at] = lc;
            lenq[at] = (int)len;
            offq[at] = o;
        }
        pend += __popc(m);
        __syncwarp();
        const bool more = base + 32 < a.P;
        if (!more && base == 0 && WS_PLAN_BALANCE) {
            // All of the query's lists are known (P <= 32): group them into
            // nJ = ceil(n / G) jobs of balanced total length instead of probe
            // order -- rank by length, deal the ranks out in snake order
            // (round r: jobs 0..nJ-1, then nJ-1..0).  A job's scan time is
            // proportional to its vectors while its LUT build time is fixed,
            // so uneven jobs leave the builders waiting for free slots on long
            // jobs and the scanners waiting for LUTs on short ones (cfg2:
            // coefficient of variation of a job's length 0.33 -> 0.09).  The
            // result does not depend on the grouping: the top-k keys
            // (R, id) are a total order.  Measured slower at cfg2 / cfg4 e5m3
            // (3.74 -> 3.80 ms, 8.56 -> 8.88 ms): probe order scans the nearest
            // lists first, which tightens the top-k threshold early (fewer
            // offers); so it is off by default (WS_PLAN_BALANCE).
            const int n = pend;  // <= 32, one entry per lane
            int my_len = lane < n ? lenq[lane] : -1;
            int my_lc = lane < n ? lcq[lane] : 0;
            long long my_off = lane < n ? offq[lane] : 0;
            int rank = 0;
            for (int i = 0; i < n; ++i) {
                const int li = __shfl_sync(0xffffffffu, my_len, i);
                rank += (li > my_len || (li == my_len && i < lane)) ? 1 : 0;
            }
            const int nJ = (n + G - 1) / G;
            const int full = n / nJ, rem = n % nJ;  // full rounds, entries of the partial round
            const int rd = rank / nJ, pos = rank % nJ;
            const int job = (rd & 1) ? nJ - 1 - pos : pos;
            // job j holds `full` entries, one more if the partial round reached it
            auto partial_before = [&](int j) {  // jobs < j that the partial round reached
                return (full & 1) ? max(0, j - (nJ - rem)) : min(j, rem);
            };
            const int dst = job * full + partial_before(job) + rd;
            __syncwarp();
            if (lane < n) {
                lcq[dst] = my_lc;
                lenq[dst] = my_len;
                offq[dst] = my_off;
            }
            __syncwarp();
            for (int j = 0; j < nJ; ++j) {
                const int from = j * full + partial_before(j);
                const int cnt = full + (partial_before(j + 1) - partial_before(j));
                emit(from, cnt, j == nJ - 1);
            }
            pend = 0;
            break;
        }
        int taken = 0;
        // emit full jobs; keep >= 1 pending until the end so the final job is marked last
        while (pend - taken > G || (!more && pend - taken > 0)) {
            const int ng = min(G, pend - taken);
            emit(taken, ng, !more && pend - taken == ng);
            taken += ng;
        }
        const int rest = pend - taken;
        int lc2 = 0, len2 = 0;
        long long o2 = 0;
        if (lane < rest) {
            lc2 = lcq[taken + lane];
            len2 = lenq[taken + lane];
            o2 = offq[taken + lane];
        }
        __syncwarp();
        if (lane < rest) {
            lcq[lane] = lc2;
            lenq[lane] = len2;
            offq[lane] = o2;
        }
        __syncwarp();
        pend = rest;
    }
    if (nj == 0) {
        // no owned non-empty list: the result is the empty list, written here;
        // the search kernel skips the query (no query state, no jobs)
        for (int i = lane; i < a.K; i += 32) {
            if (a.out_keys) {
                a.out_keys[(size_t)q * a.K + i] = ~0ull;
            } else {
                a.out_ids[(size_t)q * a.K + i] = -1LL;
                a.out_dists[(size_t)q * a.K + i] = __int_as_float(0x7f800000);
            }
        }
        if (lane == 0) {
            if (a.out_keys) a.out_ncand[q] = nc;
            else a.out_short[q] = nc < a.K ? 1 : 0;
        }
    }
    if (lane == 0) {
        njobs[q] = nj;
        ncand[q] = nc;
    }
}
#endif

// SMALLK: k <= 32 (the common case): query-state count and warp scratch are
// compile-time constants (the runtime forms cost the cfg2 kernel ~4%: spills).
template <class C, int DT, int LOGN, int SUB_D, bool GMEM, int NCH, bool CH, bool SMALLK>
__global__ void __launch_bounds__(C::THREADS, 1) scan_ws_kernel(const WsArgs w) {
    using T = typename LutTraits<DT>::T;
    extern __shared__ __align__(1024) uint8_t ws_smem[];
    uint8_t* smem = ws_smem;
    const ScanArgs& a = w.a;
    const int G = a.G, NBUF = w.NBUF, K = a.K, NQS = SMALLK ? WS_NQS : w.nqs;
    const WsLayout<C> L(a.d, a.s, SUB_D, LOGN, (int)sizeof(T), G, NBUF, K, a.s_pad, CH ? w.rc : 0);
    const size_t lut_each = L.lut_each;
    const int d_pad = (int)L.d_pad;  // residual floats per list in a job (chunked: the chunk's rows)
    constexpr int RB = WsBuild<C, DT, LOGN, SUB_D, GMEM>::R;
    const int jpt = CH ? w.rc / RB : (a.s_pad + RB - 1) / RB;  // owned rows per builder thread per job
    u64* pfull = reinterpret_cast<u64*>(smem + L.bars);  // pfull[PD]: job + residuals prepared (TMA tx)
    u64* full = pfull + WS_PD;                            // full[NBUF]: LUTs ready
    WsJob* jobs = reinterpret_cast<WsJob*>(smem + L.jobs);
    WsJob* pjobs = reinterpret_cast<WsJob*>(smem + L.pjobs);
    WsQuery* qst = reinterpret_cast<WsQuery*>(smem + L.qst);
    u64* lists = reinterpret_cast<u64*>(smem + L.lists);
    float* prq = reinterpret_cast<float*>(smem + L.prq);
    uint8_t* lut_all = smem + L.lut;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if ((smem_addr(lut_all) & 255u) != 0u) __trap();  // PRMT LUT addressing needs 256-byte alignment

    // ---- setup
    for (int i = threadIdx.x; i < (SMALLK || K <= WS_PRIV_K ? C::SW * NQS * K : NQS * 2 * K); i += blockDim.x)
        lists[i] = ~0ull;
    if (threadIdx.x < NQS) {
        WsQuery* S = qst + threadIdx.x;
        S->tau = ~0ull;
        S->ncand = 0;
        S->lock = 0;
        S->done = 0;
        S->cur = 0;
        S->q = -1;
    }
    using Builder = WsBuild<C, DT, LOGN, SUB_D, GMEM>;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem);
    if (warp == 0) tmem_alloc<Builder::NCOL>(smem_addr(tmem_slot));
    if (threadIdx.x == 0) {
        for (int b = 0; b < WS_PD; ++b) mbar_init(pfull + b, 1);
        for (int b = 0; b < NBUF; ++b) mbar_init(full + b, C::BW);
        u64* qf = reinterpret_cast<u64*>(smem + L.qfree);
        for (int b = 0; b < NQS; ++b) mbar_init(qf + b, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == C::PREP) {
        // ============================ prep warp ============================

        // Hands out queries and streams their planned jobs (descriptor +
        // residual rows, from ws_plan_kernel) into the prep ring with TMA bulk
        // copies, up to WS_PD jobs ahead of the builders.  A ring entry is
        // reused once the builders have released it (named barrier).
        int* pqs = reinterpret_cast<int*>(smem + L.prepq);
        const uint32_t pjob_bytes = (uint32_t)sizeof(WsJob), prq_bytes = (uint32_t)(G * d_pad * 4);
        int job = 0, qseq = -1, ps = 0;
        while (true) {
            int q = 0;
            if (lane == 0) q = atomicAdd(w.work, 1);
            q = __shfl_sync(0xffffffffu, q, 0);
            if (q >= a.nq) {
                if (job >= WS_PD) nbar_sync(WS_BAR_PEMPTY0 + ps, C::BAR_PEMPTY_N);
                if (lane == 0) {
                    pqs[ps] = -1;
                    mbar_arrive(pfull + ps);
                }
                break;
            }
            const int nj = w.plan_njobs[q];
            if (nj == 0) continue;  // no owned non-empty list: ws_plan_kernel wrote its result
            ++qseq;
            const int qs = qseq % NQS;
            WsQuery* S = qst + qs;
            // the state is reused only after the query that last held it was finalised
            if (qseq >= NQS) mbar_wait(reinterpret_cast<u64*>(smem + L.qfree) + qs, ((qseq / NQS) - 1) & 1);
            if (lane == 0) {
                S->q = q;
                S->ncand = w.plan_ncand[q];
            }
            for (int j = 0; j < nj; ++j, ++job) {
                if (job >= WS_PD) nbar_sync(WS_BAR_PEMPTY0 + ps, C::BAR_PEMPTY_N);
                if (lane == 0) {
                    pqs[ps] = qs;
                    const size_t gj = (size_t)q * w.JMAX + j;
                    fence_proxy_async();  // builders' reads of this entry before the async overwrite
                    mbar_expect_tx(pfull + ps, pjob_bytes + prq_bytes);
                    bulk_g2s(smem_addr(pjobs + ps), w.plan_jobs + gj, pjob_bytes, pfull + ps);
                    bulk_g2s(smem_addr(prq + (size_t)ps * G * d_pad), w.plan_rq + gj * G * d_pad, prq_bytes, pfull + ps);
                }
                if (++ps == WS_PD) ps = 0;
            }
        }
    } else if (warp < C::BW) {
        // =========================== builders ===========================

        const int t = threadIdx.x;
        Builder B;
        B.init(a.centers, a.s, t, tmem, w.gmem != 0);
        int slot = 0, ps = 0, pph = 0;  // LUT slot, prep ring entry and its phase
        bool wrapped = false;
        for (;;) {
            mbar_wait(pfull + ps, pph);
            // the slot's previous job has been scanned by every scanner warp
            if (wrapped) nbar_sync(WS_BAR_EMPTY0 + slot, C::BAR_EMPTY_N);
            const WsJob* PJ = pjobs + ps;
            const int pq_s = reinterpret_cast<const int*>(smem + L.prepq)[ps];
            WS_CHECK(pq_s >= -1 && pq_s < NQS && (pq_s < 0 || (PJ->ng >= 1 && PJ->ng <= G && PJ->nblk >= PJ->ng)));
            if (t < 32) {  // the descriptor travels with the LUT slot (warp 0 copies it)
                const int* src = reinterpret_cast<const int*>(PJ);
                int* dst = reinterpret_cast<int*>(jobs + slot);
                for (int i = t; i < (int)(sizeof(WsJob) / 4); i += 32) dst[i] = src[i];
                __syncwarp();
                if (t == 0) {
                    jobs[slot].qs = pq_s;
                    reinterpret_cast<int*>(smem + L.cnt)[slot] = 0;  // scanners' pair counter
                }
            }
            if (pq_s < 0) {
                __syncwarp();
                if (lane == 0) mbar_arrive(full + slot);
                break;
            }
            // When the code store is larger than L2 (cfg5: 3.2 GB) the scanners'
            // register prefetch of one pair ahead does not cover the DRAM
            // latency, so codes are also pulled into L2 with bulk prefetches: the
            // start of the job here (a list's codes are one contiguous range in
            // the interleaved layout), the rest by the scanners, WS_PF_PAIRS
            // rounds of pairs ahead of their grabs.  (Whole jobs prefetched NBUF
            // jobs ahead overflowed L2 at cfg5: 225 GB of DRAM reads for 113 GB
            // of codes.)  With an L2-resident store it only adds requests (cfg2
            // +1.7%), so it is off there.
            if ((w.l2pf & 1) && PJ->h == 0 && t < PJ->ng) {
                // only the job's first 2 * WS_PF_PAIRS(SW) blocks: the scanners
                // prefetch the rest a fixed distance ahead of their grabs
                const int win = 2 * WS_PF_PAIRS * C::SW;
                const int b0 = PJ->pref[t], b1 = min(PJ->pref[t + 1], win);
                if (b0 < b1) {
                    const int nv = min(PJ->len[t], (b1 - b0) * 32);
                    prefetch_l2(a.codes + PJ->off[t] * a.s_pad, (uint32_t)nv * (uint32_t)a.s_pad);
                }
            }
            B.build(reinterpret_cast<const uint8_t*>(prq) + (size_t)ps * G * d_pad * 4, (uint32_t)(d_pad * 4),
                    lut_all + (size_t)slot * G * lut_each, (uint32_t)lut_each, PJ->ng, jpt, CH ? PJ->h * jpt : 0);
            __syncwarp();  // the warp's LUT stores / prep reads are ordered before its arrivals
            if (lane == 0) mbar_arrive(full + slot);
            nbar_arrive(WS_BAR_PEMPTY0 + ps, C::BAR_PEMPTY_N);
            if (++ps == WS_PD) {
                ps = 0;
                pph ^= 1;
            }
            if (++slot == NBUF) {
                slot = 0;
                wrapped = true;
            }
        }
        bar_builders<C::NB>();  // every builder is done with TMEM
        if (warp == 0) tmem_dealloc<Builder::NCOL>(tmem);
    } else {
        // =========================== scanners ===========================

        const int sw = warp - C::BW;
        const int wsz = SMALLK ? WS_WBUF : w.wsz;
        u64* wb = reinterpret_cast<u64*>(smem + L.wbuf) + (size_t)sw * 2 * wsz;
        WarpTopK tk{wb, wb + wsz, 0, SMALLK || K <= WS_PRIV_K ? lists + (size_t)sw * NQS * K : nullptr};
        ws_scanner<C, DT, LOGN, NCH, CH, SMALLK>(a, w, jobs, reinterpret_cast<int*>(smem + L.cnt), full, NBUF, qst, lists, K,
                                      smem_addr(lut_all), (uint32_t)(G * lut_each), (uint32_t)lut_each, tk,
                                      reinterpret_cast<u64*>(smem + L.qfree), sw, lane);
    }
}

}  // namespace ivfpq
