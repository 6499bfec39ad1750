// LUT storage codecs, bit-exact with the reference `ivfpq8.minifloat`.
//
//  * e5m3 / e4m4 encode: minifloat.py:91-116 (`encode_array`): exponent rebase
//    by (bias-127), mantissa truncated to m bits, flush below min_normal,
//    clamp to 0xFF.  Closed form (verified exhaustively):
//        c = (bits >> (23-m)) - ((127-bias) << m);  c < 2^m -> 0;  c > 255 -> 255
//  * decode: minifloat.py:119-133 (`decode_array`), exact.
//  * f16: minifloat.py:151-164 = RNE binary16 of min(x, 65504).
//
// Scan-side fp8 decode uses the deferred power-of-two scale: the unscaled
// value  as_float(code << (23-m))  is a *normal* fp32 for every code the
// encoder emits (>= 2^m) and +0 for code 0, so accumulating unscaled values
// and multiplying by 2^(127-bias) once per vector is bit-identical to
// accumulating decode(code) (all partial sums are >= 2^-126, hence scaling by
// a power of two commutes with round-to-nearest-even).
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>
#include <string.h>

namespace ivfpq {

enum LutDtype : int { LUT_F32 = 0, LUT_F16 = 1, LUT_E5M3 = 2, LUT_E4M4 = 3 };

template <int DT> struct LutTraits;
template <> struct LutTraits<LUT_F32> { using T = float; static constexpr int bytes = 4; };
template <> struct LutTraits<LUT_F16> { using T = uint16_t; static constexpr int bytes = 2; };
template <> struct LutTraits<LUT_E5M3> {
    using T = uint8_t; static constexpr int bytes = 1, m = 3, bias = 15;
};
template <> struct LutTraits<LUT_E4M4> {
    using T = uint8_t; static constexpr int bytes = 1, m = 4, bias = 7;
};

__host__ __device__ inline int lut_bytes_of(int dt) { return dt == LUT_F32 ? 4 : dt == LUT_F16 ? 2 : 1; }

// minifloat.py:91-116, closed form.  Works on raw fp32 bits, so the -0.0
// quirk of the reference (sign bit read as exponent -> 0xFF) is reproduced.
template <int M, int BIAS>
__host__ __device__ __forceinline__ uint32_t fp8_encode_bits(uint32_t b) {
    int c = (int)(b >> (23 - M)) - ((127 - BIAS) << M);
    c = c < (1 << M) ? 0 : c;
    return (uint32_t)(c > 255 ? 255 : c);
}

template <int M, int BIAS>
__host__ __device__ __forceinline__ float fp8_decode_exact(uint32_t c) {
    uint32_t bits = c >= (1u << M) ? (c << (23 - M)) + ((uint32_t)(127 - BIAS) << 23) : 0u;
#ifdef __CUDA_ARCH__
    return __uint_as_float(bits);
#else
    float f; memcpy(&f, &bits, 4); return f;
#endif
}

// Storage encode of one fp32 table entry into the LUT element type.
template <int DT>
__device__ __forceinline__ typename LutTraits<DT>::T lut_store(float x) {
    if constexpr (DT == LUT_F32) {
        return x;
    } else if constexpr (DT == LUT_F16) {
        return __half_as_ushort(__float2half_rn(fminf(x, 65504.0f)));
    } else {
        return (uint8_t)fp8_encode_bits<LutTraits<DT>::m, LutTraits<DT>::bias>(__float_as_uint(x));
    }
}

// Scan-side widening of one stored entry (unscaled for fp8, see header).
template <int DT>
__device__ __forceinline__ float lut_widen(typename LutTraits<DT>::T v) {
    if constexpr (DT == LUT_F32) {
        return v;
    } else if constexpr (DT == LUT_F16) {
        return __half2float(__ushort_as_half(v));
    } else {
        return __uint_as_float((uint32_t)v << (23 - LutTraits<DT>::m));
    }
}

// Final per-vector scale: 2^(127-bias) for fp8 (exact), identity otherwise.
template <int DT>
__device__ __forceinline__ float lut_finish(float acc) {
    if constexpr (DT == LUT_E5M3 || DT == LUT_E4M4) {
        constexpr int e = 127 - LutTraits<DT>::bias;  // 112 or 120
        return __fmul_rn(acc, __uint_as_float((uint32_t)(127 + e) << 23));
    } else {
        return acc;
    }
}

}  // namespace ivfpq
