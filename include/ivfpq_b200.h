/*
 * ivfpq_b200 -- C ABI of the B200-native IVFPQ search path.
 *
 * Drop-in boundary for the reference package `ivfpq8`
 * (/root/reference/pkg/src/ivfpq8).  The reference is pure Python; every
 * entry point below names the Python function it replaces (file:line), and
 * INTEGRATION.md shows the ctypes stub a maintainer adds to bind it.
 *
 * Conventions
 *   - plain pointers and sizes only; no torch / CUDA types in signatures
 *     (`stream` is a cudaStream_t passed as void*; NULL = the legacy default
 *     stream, as in the CUDA runtime)
 *   - every function returns IVFPQ_OK (0) or an error code; the message is in
 *     ivfpq_last_error() (thread-local).  The Python shim validates arguments
 *     first and raises ValueError with the reference's wording.
 *   - "host" entry points take host buffers and are synchronous; "_device"
 *     entry points take device pointers and are asynchronous on `stream`.
 *   - an index handle is immutable after creation and may be shared by host
 *     threads; calls on one handle are serialised on the host, and a call on
 *     a different stream than the previous call first waits (stream-ordered,
 *     via an event) for the previous call's device work, because the calls
 *     share the handle's scratch buffers.
 *   - LUT dtypes: the reference's `LUT_PRECISIONS` (search.py:38).
 *   - Keys: uint64 (fp32 bits of the distance << 32 | id), ascending = the
 *     reference's lexicographic (distance, id) order (search.py:150); empty
 *     slot = UINT64_MAX.
 */
#ifndef IVFPQ_B200_H
#define IVFPQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum ivfpq_lut_dtype { IVFPQ_LUT_F32 = 0, IVFPQ_LUT_F16 = 1, IVFPQ_LUT_E5M3 = 2, IVFPQ_LUT_E4M4 = 3 };
enum ivfpq_status { IVFPQ_OK = 0, IVFPQ_EINVAL = 1, IVFPQ_ECUDA = 2, IVFPQ_EUNSUPPORTED = 3 };

typedef struct ivfpq_index ivfpq_index; /* opaque device-resident index */

const char *ivfpq_last_error(void);
int ivfpq_version(void);
/* Number of visible CUDA devices (0 when no GPU). */
int ivfpq_device_count(int *n);
/* Upper bound on k and nprobe supported by the device top-k. */
int ivfpq_max_k(void);
/* Scan kernel selection (testing; every mode is exact): 0 = auto (persistent
 * warp-specialised kernel when the shape fits -- warp layout B, 4 builder + 15
 * scanner warps, for scan-heavy shapes, else layout A, 8 + 11 -- otherwise the
 * per-query kernel), 1 = force the per-query kernel, 2 = prefer row-chunked
 * LUT jobs, 3 = layout A only, 4 = layout B wherever it is built. */
int ivfpq_set_scan_kernel(int mode);
/* Coarse-select (K1) kernel selection (testing): 0 = auto (tensor-core TF32
 * nomination + exact re-rank when the shape fits), 1 = exact SIMT kernel only,
 * 2 = tensor-core path with every query re-done by the exact fallback. */
int ivfpq_set_select_kernel(int mode);
/* Debug: number of queries in the last tensor-core coarse select on `idx`
 * whose error-bound guard failed (and were re-done exactly); -1 if the last
 * select did not take the tensor-core path.  Synchronises the device. */
int ivfpq_debug_select_flagged(ivfpq_index *idx, int64_t *out);
/* Number of CUDA kernels this library has launched since it was loaded. */
int ivfpq_launch_count(int64_t *out);

/* Upload an index.  Replaces the host-resident `IvfPqIndex`
 * (index.py:27-70): coarse f32[nlist,d] (index.py:35), codebook centers
 * f32[s, 2^p, d/s] (pq.py:22-23), and the inverted lists in CSR form:
 * list c = ids[list_off[c] .. list_off[c+1]) with codes row-major
 * uint8[L_c, s] (index.py:37-38).  `owned` (may be NULL = all lists) selects
 * the lists this device holds in a list-sharded multi-GPU search; lengths of
 * all lists are kept for the candidate count.  Ids must be < 2^32-1. */
int ivfpq_index_create(int device, const float *coarse, int64_t nlist, int64_t d, const float *centers,
                       int64_t s, int64_t p, const int64_t *list_off, const int64_t *ids,
                       const uint8_t *codes, const int32_t *owned, int64_t n_owned, ivfpq_index **out);
int ivfpq_index_destroy(ivfpq_index *idx);
/* Device bytes held by the index (codes, ids, centroids, codebook). */
int ivfpq_index_bytes(const ivfpq_index *idx, int64_t *bytes);

/* Replaces search_batch (search.py:187-203): queries f32[nq,d] host;
 * out_ids int64[nq,k] (-1 padded), out_dists f32[nq,k] (+inf padded),
 * *out_n_short = rows with fewer than k candidates (search.py:194-202). */
int ivfpq_search(ivfpq_index *idx, const float *queries, int64_t nq, int64_t k, int64_t nprobe, int lut_dtype,
                 int64_t *out_ids, float *out_dists, int64_t *out_n_short);

/* Same as ivfpq_search on device buffers; out_short int32[nq] (1 = short). */
int ivfpq_search_device(ivfpq_index *idx, const float *d_queries, int64_t nq, int64_t k, int64_t nprobe,
                        int lut_dtype, int64_t *d_out_ids, float *d_out_dists, int32_t *d_out_short,
                        void *stream);

/* --- staged pieces of the list-sharded multi-GPU search ------------------ */
/* K1 over the lists this device owns: per query the nprobe smallest
 * (d2, global cluster id) keys, ascending (select_clusters, search.py:91-97). */
int ivfpq_select_device(ivfpq_index *idx, const float *d_queries, int64_t nq, int64_t nprobe, uint64_t *d_keys,
                        void *stream);
/* Merge W key blocks [W][nq][n_in] (each row ascending) -> [nq][n_out]. */
int ivfpq_merge_keys_device(const uint64_t *d_in, int64_t W, int64_t nq, int64_t n_in, int64_t n_out,
                            uint64_t *d_out, void *stream);
/* K2-K4 over the owned lists among each query's probes (keys from
 * select/merge): local top-k keys [nq][k] and the global candidate count. */
int ivfpq_scan_device(ivfpq_index *idx, const float *d_queries, int64_t nq, const uint64_t *d_probe_keys,
                      int64_t nprobe, int64_t k, int lut_dtype, uint64_t *d_out_keys, int64_t *d_out_ncand,
                      void *stream);
/* keys + candidate counts -> ids / dists / short flags (search.py:194-202). */
int ivfpq_finalize_device(const uint64_t *d_keys, const int64_t *d_ncand, int64_t nq, int64_t k,
                          int64_t *d_out_ids, float *d_out_dists, int32_t *d_out_short, void *stream);

/* --- conformance hooks (host buffers, run on device 0) -------------------- */
/* minifloat.py:91-116 encode_array / :119-133 decode_array (dtype e5m3|e4m4) */
int ivfpq_fp8_encode(const float *x, int64_t n, int lut_dtype, uint8_t *out);
int ivfpq_fp8_decode(const uint8_t *codes, int64_t n, int lut_dtype, float *out);
/* minifloat.py:151-164 encode_f16_array / :167-169 decode_f16_array */
int ivfpq_f16_encode(const float *x, int64_t n, uint16_t *out);
int ivfpq_f16_decode(const uint16_t *bits, int64_t n, float *out);
/* search.py:114-127 build_lut: entries [s][2^p] as f32 / u16 / u8 */
int ivfpq_build_lut(const float *centers, int64_t s, int64_t p, int64_t sub_d, const float *rq, int lut_dtype,
                    void *out_entries);
/* search.py:130-142 scan_list: codes row-major uint8[L, s] */
int ivfpq_scan_list(const uint8_t *codes, int64_t L, int64_t s, int64_t p, const void *entries, int lut_dtype,
                    float *out_r);
/* search.py:91-97 select_clusters for host queries q f32[nq,d] -> int64[nq,nprobe] */
int ivfpq_select_clusters(ivfpq_index *idx, const float *q, int64_t nq, int64_t nprobe, int64_t *out);
/* search.py:145-155 top_k: out arrays hold min(n, k) entries */
int ivfpq_top_k(const int64_t *ids, const float *dists, int64_t n, int64_t k, int64_t *out_ids, float *out_dists);

/* --- ingest: populate an index on the GPU ----------- */
/* pq_encode (pq.py:92-110): nearest sub-centroid per subspace, ties -> lower
 * code, BIT-EXACT with the reference (its sgemm FMA chain + einsum norms,
 * ingest.cuh) for sub_d = d/s <= 4.  x f32[n,d] row-major; codes u8[n,s].
 * With d_coarse and d_assign (i64[n]) the residual rows fl(x - coarse[a])
 * of compute_residuals (pq.py:54-63) are formed on the fly. */
int ivfpq_pq_encode_device(const float *d_x, int64_t n, int64_t d, const float *d_coarse, const int64_t *d_assign,
                           const float *d_centers, int64_t s, int64_t p, uint8_t *d_codes, void *stream);
int ivfpq_pq_encode(const float *x, int64_t n, int64_t d, const float *centers, int64_t s, int64_t p,
                    uint8_t *codes);
/* compute_residuals (pq.py:54-63): out f32[n,d] = fl(x - c[assign]); assign
 * i64[n] in [0, nc). */
int ivfpq_compute_residuals(const float *x, int64_t n, int64_t d, const float *c, int64_t nc,
                            const int64_t *assign, float *out);
/* reconstruct (pq.py:113-127): out f32[n, s*sub_d] = the sub-centroids named
 * by codes u8[n,s]. */
int ivfpq_reconstruct(const uint8_t *codes, int64_t n, const float *centers, int64_t s, int64_t p, int64_t sub_d,
                      float *out);
/* assign_to_centroids (kmeans.py:49-69): nearest centroid under the expanded
 * squared L2 form clipped at 0, ties -> lower id; d2 may be NULL.  Parity is
 * decision-level (einsum's norm order at d >= 16 is not modelled). */
int ivfpq_assign_device(const float *d_x, int64_t n, int64_t d, const float *d_c, int64_t nc, int64_t *d_assign,
                        float *d_d2, void *stream);
int ivfpq_assign(const float *x, int64_t n, int64_t d, const float *c, int64_t nc, int64_t *assign, float *d2);

/* --- K7: exact k-NN ground truth --------------------- */
/* brute_force_knn (datasets.py:179-201): per query the k smallest
 * squared_l2_to_all distances (datasets.py:166-176: sequential fp32 sum of
 * fl(diff^2)), ties -> lower id; ids AND distances bit-exact with the
 * reference.  Reuses the K1 select path over the base rows.  A handle from
 * ivfpq_knn_create is searched with ivfpq_select_device (keys = d2 bits << 32
 * | row id) and freed with ivfpq_index_destroy. */
/* squared_l2_to_all (datasets.py:166-176): out f32[n] = sequential fp32
 * sum over t of fl(fl(base[i][t] - q[t])^2), bit-exact. */
int ivfpq_squared_l2_to_all(const float *base, int64_t n, int64_t d, const float *q, float *out);
int ivfpq_knn_create(int device, const float *base, int64_t n, int64_t d, ivfpq_index **out);
int ivfpq_brute_force_knn(const float *base, int64_t n, int64_t d, const float *queries, int64_t nq, int64_t k,
                          int64_t *out_ids, float *out_dists);

#ifdef __cplusplus
}
#endif
#endif /* IVFPQ_B200_H */
