// gather.cuh -- the branch-free bitmap -> dense gather shared by the expand
// and fused decompress->GEMV kernels (selector tables + PRMT byte permutes),
// and the f16 dot product used by the GEMV consumers.
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

#include "common.cuh"

#ifndef ENDOR_STORE_CS
#define ENDOR_STORE_CS 0
#endif

namespace endor_b200 {

// ---- selector tables ---------------------------------------------------------
// A 4-element nibble q of the bitmap consumes popc(q) packed values.  The
// next four packed values are fetched as an unaligned 8-byte window {x, y}
// and PRMT drops each into its slot.  Zero bytes come from RZ (byte 4 of a
// zero second operand), so no compare/select is needed:
//   f16:  word0 (slots 0,1) = PRMT(x, 0, sel0)             -- needs v0..v1 at most
//         ym               = PRMT(y, 0, selm)              -- y, or y with v3 zeroed
//         word1 (slots 2,3) = PRMT(x, ym, sel1)            -- unset slots read ym bytes 6,7
//   i8:   word  (slots 0-3) = PRMT(x, 0, sel)
// selm keeps y whole only when q == 0xF (then no slot is unset).  The f16
// table packs sel0 | sel1 << 16 into one word: 16 words in 16 distinct banks,
// so a warp's lookups never conflict (one wavefront per LDS).
__shared__ uint32_t g_lut16[16];
__shared__ uint32_t g_lut8[16];

__device__ __forceinline__ void init_luts(int tid) {
    if (tid < 16) {
        const uint32_t q = tid;
        uint32_t s0 = 0, s1 = 0, j = 0, s8 = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool set = q & (1u << k);
            const uint32_t b0 = set ? 2 * j : (k < 2 ? 4u : 6u);
            const uint32_t b1 = set ? 2 * j + 1 : (k < 2 ? 4u : 7u);
            const uint32_t pos = (k & 1) * 8;
            if (k < 2) s0 |= (b0 << pos) | (b1 << (pos + 4));
            else s1 |= (b0 << pos) | (b1 << (pos + 4));
            s8 |= (set ? j : 4u) << (4 * k);
            j += set;
        }
        g_lut16[q] = s0 | (s1 << 16);
        g_lut8[q] = s8;
    }
}

// Expand one 16-byte output chunk.  m: the chunk's bitmap bits; a: shared
// address of its first packed value (any byte alignment).
template <int EB>
__device__ __forceinline__ uint4 gather_chunk(uint32_t m, uint32_t a) {
    uint32_t o[4];
    if constexpr (EB == 2) {
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const uint32_t q = (m >> (4 * g)) & 15u;
            const uint32_t sel = g_lut16[q];
            const uint32_t al = a & ~3u, sh = a << 3;  // funnel shifts wrap mod 32
            const uint32_t w0 = lds32(al), w1 = lds32(al + 4), w2 = lds32(al + 8);
            const uint32_t x = __funnelshift_r(w0, w1, sh);
            const uint32_t y = __funnelshift_r(w1, w2, sh);
            const uint32_t ym = __byte_perm(y, 0u, q == 15u ? 0x3210u : 0x4410u);
            o[2 * g] = __byte_perm(x, 0u, sel);
            o[2 * g + 1] = __byte_perm(x, ym, sel >> 16);
            a += 2 * __popc(q);
        }
    } else {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const uint32_t qa = (m >> (4 * g)) & 15u;
            const uint32_t sel = g_lut8[qa];
            const uint32_t al = a & ~3u, sh = a << 3;
            const uint32_t x = __funnelshift_r(lds32(al), lds32(al + 4), sh);
            o[g] = __byte_perm(x, 0u, sel);
            a += __popc(qa);
        }
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

// Fused INT8 dequant + decompress (decompress(dequantize_values(t)),
// codec.hpp:334-349 then :157): 8 output f16 slots per 16-byte chunk, each
// set slot = f32_to_f16(float(q) * scale) (float16.hpp:35-73, RNE), unset = +0.
// FAST (scale finite, sign bit clear): unset slots hold q = 0 -> +0 exactly,
// and a finite product is converted with the hardware RNE (identical to the
// reference's routine for every non-NaN input).  Otherwise the reference's
// own bit routine runs per slot and unset slots are masked to +0.
template <bool FAST>
__device__ __forceinline__ uint4 gather_chunk_dequant(uint32_t m, uint32_t a, float scale) {
    uint32_t o[4];
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        const uint32_t q = (m >> (4 * g)) & 15u;
        const uint32_t al = a & ~3u, sh = a << 3;
        const uint32_t x = __byte_perm(__funnelshift_r(lds32(al), lds32(al + 4), sh), 0u, g_lut8[q]);
        float f[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) f[k] = __fmul_rn(float(int8_t(x >> (8 * k))), scale);
        if constexpr (FAST) {
            const __half2 h0 = __floats2half2_rn(f[0], f[1]), h1 = __floats2half2_rn(f[2], f[3]);
            o[2 * g] = *reinterpret_cast<const uint32_t*>(&h0);
            o[2 * g + 1] = *reinterpret_cast<const uint32_t*>(&h1);
        } else {
            // NaN products follow the x86 SSE rules the reference runs under: a NaN
            // operand propagates quieted, 0 * inf gives the default NaN 0xFFC00000
            // (the GPU would produce a canonical 0x7FFFFFFF instead)
            const uint32_t sb = __float_as_uint(scale);
            const bool snan = (sb & 0x7FFFFFFFu) > 0x7F800000u;
            uint32_t h[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float v = f[k];
                if (v != v) v = __uint_as_float(snan ? (sb | 0x00400000u) : 0xFFC00000u);
                h[k] = (q >> k) & 1u ? f32_to_f16_bits(v) : 0u;
            }
            o[2 * g] = h[0] | (h[1] << 16);
            o[2 * g + 1] = h[2] | (h[3] << 16);
        }
        a += __popc(q);
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

// Element modes of the expand kernels: bytes per packed value (IN) and per
// dense output element (OUT).
constexpr int kModeI8 = 1, kModeF16 = 2, kModeDequant = 3;
__host__ __device__ constexpr int mode_in(int m) { return m == kModeF16 ? 2 : 1; }
__host__ __device__ constexpr int mode_out(int m) { return m == kModeI8 ? 1 : 2; }

template <int MODE>
__device__ __forceinline__ uint4 gather_mode(uint32_t m, uint32_t a, float scale, bool fast) {
    if constexpr (MODE == kModeDequant) {
        return fast ? gather_chunk_dequant<true>(m, a, scale) : gather_chunk_dequant<false>(m, a, scale);
    } else {
        return gather_chunk<MODE>(m, a);
    }
}

// bytes [lo_bytes, hi_bytes) of a 16-byte chunk (range ends)
__device__ __forceinline__ void store_partial(uint8_t* p, uint4 q, uint32_t hi_bytes, uint32_t lo_bytes = 0) {
    const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (uint32_t b = 0; b < 16; ++b)
        if (b >= lo_bytes && b < hi_bytes) p[b] = uint8_t(qw[b >> 2] >> ((b & 3) * 8));
}

// Expand one warp's 1024-element sub-tile.  word/excl: this lane's bitmap word
// (bits past the range already cleared) and its exclusive popcount within the
// warp; vbase: shared address of the sub-tile's first packed value.  Lane l
// writes chunks l, l+32, .. so every store instruction covers 512 contiguous
// bytes.  FULL: all 1024 elements valid (no bounds checks).  head_elems:
// leading elements that belong to another range (a chunk starting inside a
// bitmap word, decompress_chunk_into at an arbitrary chunk size): not written.
template <int MODE, bool FULL, int WE = 1024>
__device__ __forceinline__ void expand_subtile(uint32_t word, uint32_t excl, uint32_t vbase,
                                               uint8_t* out, int32_t valid_elems, int lane,
                                               float scale = 1.f, bool fast = true, int32_t head_elems = 0) {
    constexpr int IN = mode_in(MODE), OUT = mode_out(MODE);
    constexpr int EPC = 16 / OUT;             // output elements per 16-byte chunk
    constexpr int CPW = 32 / EPC;             // chunks per bitmap word (4 or 2)
    constexpr int ITERS = WE / EPC / 32;      // chunks per lane
    const uint32_t sh = (lane % CPW) * EPC;   // chunk position inside its word: lane-constant
    const uint32_t low = (1u << sh) - 1u;
    uint8_t* o = out + size_t(lane) * 16;
#pragma unroll
    for (int j = 0; j < ITERS; ++j) {
        const int src = (32 * j + lane) / CPW;
        const uint32_t wd = __shfl_sync(0xffffffffu, word, src);
        const uint32_t pre = __shfl_sync(0xffffffffu, excl, src);
        const uint32_t m = (wd >> sh) & ((1u << EPC) - 1u);
        const uint32_t r = pre + __popc(wd & low);
        const int e = (32 * j + lane) * EPC;
        if (!FULL && (e >= valid_elems || e + EPC <= head_elems)) continue;
        const uint4 q = gather_mode<MODE>(m, vbase + r * IN, scale, fast);
#if ENDOR_STORE_CS
        if (FULL || (e + EPC <= valid_elems && e >= head_elems)) __stcs(reinterpret_cast<uint4*>(o + j * 512), q);
#else
        if (FULL || (e + EPC <= valid_elems && e >= head_elems)) *reinterpret_cast<uint4*>(o + j * 512) = q;
#endif
        else store_partial(o + j * 512, q, uint32_t(min(valid_elems - e, EPC)) * OUT,
                           uint32_t(max(head_elems - e, 0)) * OUT);
    }
}

// acc += dot(w[0..7], x[0..7]) over f16 pairs with fp32 accumulation: the
// sm_100 mixed-precision FMA (PTX fma.rn.f32.f16, SASS FHFMA with .H0/.H1
// operand selects) -- one instruction per element, no f16->f32 conversions;
// bit-identical to fmaf(float(w), float(x), acc).
__device__ __forceinline__ float fma_f16x2(uint32_t w, uint32_t x, float acc) {
    asm("{\n\t.reg .b16 wl, wh, xl, xh;\n\t"
        "mov.b32 {wl, wh}, %1;\n\t"
        "mov.b32 {xl, xh}, %2;\n\t"
        "fma.rn.f32.f16 %0, wl, xl, %0;\n\t"
        "fma.rn.f32.f16 %0, wh, xh, %0;\n\t}"
        : "+f"(acc) : "r"(w), "r"(x));
    return acc;
}
__device__ __forceinline__ float dot8_f16(const uint4& w, const uint4& x, float acc) {
    acc = fma_f16x2(w.x, x.x, acc);
    acc = fma_f16x2(w.y, x.y, acc);
    acc = fma_f16x2(w.z, x.z, acc);
    acc = fma_f16x2(w.w, x.w, acc);
    return acc;
}

}  // namespace endor_b200
