/*
 * endor_oracle.c -- CPU restatement of the reference codec (TEST ORACLE ONLY).
 *
 * Not product code: see endor_oracle.h.  Plain C99 + pthreads; every function
 * cites the reference file:line (under /root/reference/proj/include/endor/)
 * whose behaviour it restates.  Pinned against the reference's golden vectors
 * by tests/test_oracle.py.
 */
#include "endor_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ---- bit helpers -------------------------------------------------------- */

/* Bit i lives in byte i>>3 at position i&7 (LSB-first), bitmap.hpp:14-17. */
static inline int bit_test(const uint8_t* bm, uint64_t i) { return (bm[i >> 3] >> (i & 7)) & 1; }

/* 64-bit little-endian word w of a ceil(n/8)-byte bitmap; bytes past the
 * buffer read as zero (the reference keeps padding bits zero,
 * bitmap.hpp:78-84). */
static inline uint64_t word_at(const uint8_t* bm, uint64_t nbytes, uint64_t w) {
    uint64_t v = 0;
    uint64_t b0 = w * 8;
    for (int j = 0; j < 8; ++j) {
        if (b0 + (uint64_t)j < nbytes) v |= (uint64_t)bm[b0 + j] << (8 * j);
    }
    return v;
}

uint64_t or_popcount(const uint8_t* bitmap, uint64_t n) {  /* bitmap.hpp:34-38 */
    uint64_t c = 0, nbytes = (n + 7) / 8;
    for (uint64_t b = 0; b < nbytes; ++b) {
        uint8_t v = bitmap[b];
        if (b == nbytes - 1 && (n & 7)) v &= (uint8_t)((1u << (n & 7)) - 1); /* bits < n only */
        c += (uint64_t)__builtin_popcount(v);
    }
    return c;
}

uint64_t or_rank_range(const uint8_t* bitmap, uint64_t begin, uint64_t end) {  /* bitmap.hpp:44-61 */
    if (begin >= end) return 0;
    uint64_t c = 0, i = begin;
    while (i < end && (i & 7)) c += bit_test(bitmap, i++);
    while (i + 8 <= end) { c += (uint64_t)__builtin_popcount(bitmap[i >> 3]); i += 8; }
    while (i < end) c += bit_test(bitmap, i++);
    return c;
}

int or_rank_index(const uint8_t* bitmap, uint64_t n, uint64_t cs, uint64_t* prefix_out) {
    /* bitmap.hpp:117-132: chunk_size must be a power of two >= 64 */
    if (cs < 64 || (cs & (cs - 1)) != 0) return OR_INVALID;
    uint64_t chunks = n == 0 ? 0 : (n + cs - 1) / cs, running = 0;
    for (uint64_t k = 0; k < chunks; ++k) {
        prefix_out[k] = running;
        uint64_t b = k * cs, e = b + cs < n ? b + cs : n;
        running += or_rank_range(bitmap, b, e);
    }
    return OR_OK;
}

/* ---- decompress ---------------------------------------------------------- */

void or_scatter_range(int eb, const uint8_t* bitmap, const uint8_t* values, uint64_t begin,
                      uint64_t end, uint64_t value_offset, uint8_t* dst) {
    /* codec.hpp:132-152: zero the range, then copy one value per set bit in
     * row-major order.  Word-at-a-time like the reference's loop :140-151. */
    memset(dst + begin * (uint64_t)eb, 0, (end - begin) * (uint64_t)eb);
    uint64_t nbytes = (end + 7) / 8; /* only bytes < ceil(end/8) are touched */
    uint64_t v = value_offset, i = begin;
    while (i < end) {
        uint64_t word = word_at(bitmap, nbytes, i >> 6) >> (i & 63);
        uint64_t span = 64 - (i & 63);
        if (span > end - i) span = end - i;
        if (span < 64) word &= (((uint64_t)1) << span) - 1;
        while (word) {
            uint64_t bit = (uint64_t)__builtin_ctzll(word);
            memcpy(dst + (i + bit) * (uint64_t)eb, values + v * (uint64_t)eb, (size_t)eb);
            ++v;
            word &= word - 1;
        }
        i += span;
    }
}

static int dims_ok(uint64_t rows, uint64_t cols) {  /* checked_element_count, dense_matrix.hpp:28-33 */
    return !(rows != 0 && cols > UINT64_MAX / rows);
}

int or_decompress(uint64_t rows, uint64_t cols, int eb, const uint8_t* bitmap,
                  const uint8_t* values, uint64_t nnz, uint8_t* dst) {
    if (!dims_ok(rows, cols)) return OR_SIZE;
    uint64_t n = rows * cols;
    if (or_popcount(bitmap, n) != nnz) return OR_CORRUPTION; /* codec.hpp:158-160 */
    if (n > 0) or_scatter_range(eb, bitmap, values, 0, n, 0, dst); /* codec.hpp:162-164 */
    return OR_OK;
}

int or_check_index(uint64_t n, const uint8_t* bitmap, uint64_t nnz, uint64_t cs,
                   const uint64_t* prefix, uint64_t chunk_count) {
    /* codec.hpp:170-184 */
    uint64_t chunks = (n == 0 || cs == 0) ? 0 : (n + cs - 1) / cs;
    if (cs == 0 || chunk_count != chunks) return OR_CORRUPTION;
    if (chunks > 0) {
        uint64_t last_begin = (chunks - 1) * cs;
        uint64_t tail = or_rank_range(bitmap, last_begin, n);
        if (prefix[chunks - 1] + tail != nnz) return OR_CORRUPTION;
    }
    return OR_OK;
}

int or_decompress_chunk_into(uint64_t rows, uint64_t cols, int eb, const uint8_t* bitmap,
                             const uint8_t* values, uint64_t nnz, uint64_t cs,
                             const uint64_t* prefix, uint64_t chunk_count, uint64_t k,
                             uint8_t* dst, uint64_t dst_bytes) {
    /* codec.hpp:191-201 */
    if (!dims_ok(rows, cols)) return OR_SIZE;
    uint64_t n = rows * cols;
    int st = or_check_index(n, bitmap, nnz, cs, prefix, chunk_count);
    if (st) return st;
    if (k >= chunk_count) return OR_BOUNDS;
    if (dst_bytes != n * (uint64_t)eb) return OR_INVALID;
    uint64_t b = k * cs, e = b + cs < n ? b + cs : n;
    or_scatter_range(eb, bitmap, values, b, e, prefix[k], dst);
    return OR_OK;
}

int or_decompress_chunked(uint64_t rows, uint64_t cols, int eb, const uint8_t* bitmap,
                          const uint8_t* values, uint64_t nnz, uint64_t cs,
                          const uint64_t* prefix, uint64_t chunk_count, uint8_t* dst) {
    /* codec.hpp:205-216 */
    if (!dims_ok(rows, cols)) return OR_SIZE;
    uint64_t n = rows * cols;
    int st = or_check_index(n, bitmap, nnz, cs, prefix, chunk_count);
    if (st) return st;
    for (uint64_t k = 0; k < chunk_count; ++k) {
        uint64_t b = k * cs, e = b + cs < n ? b + cs : n;
        or_scatter_range(eb, bitmap, values, b, e, prefix[k], dst);
    }
    return OR_OK;
}

/* ---- compress ------------------------------------------------------------ */

int or_compress(uint64_t rows, uint64_t cols, int eb, const uint8_t* dense, uint8_t* bitmap_out,
                uint8_t* values_out, uint64_t* nnz_out, int* negzero_out) {
    /* codec.hpp:97-126: f16 zero iff (h & 0x7FFF) == 0 (float16.hpp:75), -0
     * is dropped and flagged (codec.hpp:109-111); i8 zero iff byte == 0. */
    if (!dims_ok(rows, cols)) return OR_SIZE;
    uint64_t n = rows * cols, nnz = 0;
    int negzero = 0;
    memset(bitmap_out, 0, (size_t)((n + 7) / 8));
    for (uint64_t i = 0; i < n; ++i) {
        int nz;
        if (eb == 2) {
            uint16_t h = (uint16_t)(dense[2 * i] | (dense[2 * i + 1] << 8));
            nz = (h & 0x7FFFu) != 0;
            if (!nz && h == 0x8000u) negzero = 1;
        } else {
            nz = dense[i] != 0;
        }
        if (nz) {
            bitmap_out[i >> 3] |= (uint8_t)(1u << (i & 7));
            memcpy(values_out + nnz * (uint64_t)eb, dense + i * (uint64_t)eb, (size_t)eb);
            ++nnz;
        }
    }
    *nnz_out = nnz;
    *negzero_out = negzero;
    return OR_OK;
}

/* ---- f16 bit math (float16.hpp:12-73) ------------------------------------ */

static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

float or_f16_to_f32(uint16_t h) {  /* float16.hpp:12-33 */
    uint32_t sign = (uint32_t)(h & 0x8000u) << 16, exp = (h >> 10) & 0x1Fu, mant = h & 0x3FFu, out;
    if (exp == 0) {
        if (mant == 0) {
            out = sign;
        } else {
            int top = 31 - __builtin_clz(mant);
            out = sign | ((uint32_t)(top + 103) << 23) | ((mant << (23 - top)) & 0x7FFFFFu);
        }
    } else if (exp == 0x1F) {
        out = sign | 0x7F800000u | (mant << 13);
    } else {
        out = sign | ((exp + 112u) << 23) | (mant << 13);
    }
    return u2f(out);
}

uint16_t or_f32_to_f16(float f) {  /* float16.hpp:35-73, round to nearest even */
    uint32_t x = f2u(f);
    uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
    uint32_t mag = x & 0x7FFFFFFFu;
    if (mag >= 0x7F800000u) {
        if (mag == 0x7F800000u) return (uint16_t)(sign | 0x7C00u);
        uint16_t payload = (uint16_t)((mag >> 13) & 0x3FFu);
        if (payload == 0) payload = 0x200u;
        return (uint16_t)(sign | 0x7C00u | payload);
    }
    if (mag >= 0x477FF000u) return (uint16_t)(sign | 0x7C00u);
    uint32_t exp = mag >> 23;
    if (exp >= 0x71u) {
        uint32_t mant = mag & 0x7FFFFFu, half = ((exp - 0x70u) << 10) | (mant >> 13);
        uint32_t rem = mant & 0x1FFFu;
        half += (rem > 0x1000u) || (rem == 0x1000u && (half & 1u));
        return (uint16_t)(sign | half);
    }
    uint32_t m24 = (mag & 0x7FFFFFu) | 0x800000u, shift = 126u - exp;
    if (shift > 24u) return sign;
    uint32_t m = m24 >> shift, rem = m24 & ((1u << shift) - 1u), halfway = 1u << (shift - 1);
    m += (rem > halfway) || (rem == halfway && (m & 1u));
    return (uint16_t)(sign | m);
}

/* ---- synthetic weights (weight_gen.hpp) ---------------------------------- */

/* SplitMix64::next (weight_gen.hpp:21-26).  The k-th draw (1-based) of a
 * generator seeded with s is mix(s + k*golden): counter-based. */
static inline uint64_t splitmix_at(uint64_t seed, uint64_t k) {
    uint64_t z = seed + k * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void or_synth_weight(uint64_t n, int eb, uint64_t seed, uint8_t* out) {
    /* weight_gen.hpp:40-55; next_signed_unit :29-32 */
    for (uint64_t i = 0; i < n; ++i) {
        double u = (double)(splitmix_at(seed, i + 1) >> 11) * 0x1.0p-53;
        double s = 2.0 * u - 1.0;
        if (eb == 2) {
            uint16_t h = or_f32_to_f16((float)s);
            out[2 * i] = (uint8_t)(h & 0xFF);
            out[2 * i + 1] = (uint8_t)(h >> 8);
        } else {
            long v = lround(s * 127.0);
            if (v < -127) v = -127;
            if (v > 127) v = 127;
            out[i] = (uint8_t)(int8_t)v;
        }
    }
}

static inline uint32_t mag_key(const uint8_t* w, int eb, uint64_t i) {  /* weight_gen.hpp:61-64 */
    if (eb == 2) return (uint32_t)(w[2 * i] | (w[2 * i + 1] << 8)) & 0x7FFFu;
    int v = (int8_t)w[i];
    return (uint32_t)(v < 0 ? -v : v);
}

int or_magnitude_prune(uint64_t n, int eb, double sparsity, const uint8_t* in, uint8_t* out) {
    /* weight_gen.hpp:96-113 */
    if (!(sparsity >= 0.0 && sparsity < 1.0)) return OR_INVALID;
    memcpy(out, in, (size_t)(n * (uint64_t)eb));
    uint64_t target = (uint64_t)(sparsity * (double)n);
    if (target == 0) return OR_OK;
    uint64_t* hist = (uint64_t*)calloc(32768, sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) hist[mag_key(in, eb, i)]++;
    uint64_t below = 0;
    uint32_t K = 0;
    for (K = 0; K < 32768; ++K) {
        if (below + hist[K] >= target) break;
        below += hist[K];
    }
    free(hist);
    uint64_t ties = target - below; /* how many key==K elements to prune, lowest index first */
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t k = mag_key(in, eb, i);
        int prune = k < K || (k == K && ties > 0);
        if (k == K && ties > 0) --ties;
        if (prune) memset(out + i * (uint64_t)eb, 0, (size_t)eb);
    }
    return OR_OK;
}

int or_nm_prune(uint64_t rows, uint64_t cols, int eb, uint64_t nkeep, uint64_t m,
                const uint8_t* in, uint8_t* out) {
    /* weight_gen.hpp:118-141: in each aligned group of m in a row keep the
     * nkeep largest |v|; ties keep the higher index (prune the lower). */
    if (nkeep == 0 || nkeep > m) return OR_INVALID;
    memcpy(out, in, (size_t)(rows * cols * (uint64_t)eb));
    if (nkeep == m) return OR_OK;
    for (uint64_t r = 0; r < rows; ++r) {
        for (uint64_t g0 = 0; g0 < cols; g0 += m) {
            uint64_t g1 = g0 + m < cols ? g0 + m : cols, gs = g1 - g0;
            if (gs <= nkeep) continue;
            for (uint64_t a = g0; a < g1; ++a) {
                /* element a survives iff fewer than nkeep group members beat it
                 * under (key desc, index desc) */
                uint64_t ia = r * cols + a, better = 0;
                uint32_t ka = mag_key(in, eb, ia);
                for (uint64_t b = g0; b < g1; ++b) {
                    uint64_t ib = r * cols + b;
                    uint32_t kb = mag_key(in, eb, ib);
                    if (kb > ka || (kb == ka && ib > ia)) ++better;
                }
                if (better >= nkeep) memset(out + ia * (uint64_t)eb, 0, (size_t)eb);
            }
        }
    }
    return OR_OK;
}

/* ---- std::mt19937_64 / generate_canonical -------------------------------- */

void or_mt64_seed(or_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

uint64_t or_mt64_next(or_mt64* g) {
    const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull, A = 0xB5026F5AA96619E9ull;
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            g->mt[i] = g->mt[(i + 156) % 312] ^ (x >> 1) ^ ((x & 1) ? A : 0);
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

double or_mt64_coin(or_mt64* g) {
    /* uniform_real_distribution<double>(0,1) over mt19937_64 in libstdc++:
     * generate_canonical<double,53> takes one draw: u / 2^64, clamped below 1. */
    double r = (double)or_mt64_next(g) / 18446744073709551616.0;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r * (1.0 - 0.0) + 0.0;
}

void or_random_dense(uint64_t rows, uint64_t cols, int eb, uint64_t seed, double zf,
                     uint8_t* out) {
    /* test_helpers.hpp:15-38 */
    or_mt64 g;
    or_mt64_seed(&g, seed);
    uint64_t n = rows * cols;
    memset(out, 0, (size_t)(n * (uint64_t)eb));
    for (uint64_t i = 0; i < n; ++i) {
        if (or_mt64_coin(&g) < zf) continue;
        if (eb == 2) {
            uint16_t v;
            do { v = (uint16_t)or_mt64_next(&g); } while ((v & 0x7FFFu) == 0 || ((v >> 10) & 0x1Fu) == 0x1Fu);
            out[2 * i] = (uint8_t)(v & 0xFF);
            out[2 * i + 1] = (uint8_t)(v >> 8);
        } else {
            int8_t v;
            do { v = (int8_t)or_mt64_next(&g); } while (v == 0);
            out[i] = (uint8_t)v;
        }
    }
}

void or_acceptance_matrix(or_mt64* g, uint64_t rows, uint64_t cols, int eb, double zf,
                          uint8_t* out) {
    /* acceptance.cpp:53-74: like random_dense but keeps inf/NaN patterns */
    uint64_t n = rows * cols;
    memset(out, 0, (size_t)(n * (uint64_t)eb));
    for (uint64_t i = 0; i < n; ++i) {
        if (or_mt64_coin(g) < zf) continue;
        if (eb == 2) {
            uint16_t v;
            do { v = (uint16_t)or_mt64_next(g); } while ((v & 0x7FFFu) == 0);
            out[2 * i] = (uint8_t)(v & 0xFF);
            out[2 * i + 1] = (uint8_t)(v >> 8);
        } else {
            int8_t v;
            do { v = (int8_t)or_mt64_next(g); } while (v == 0);
            out[i] = (uint8_t)v;
        }
    }
}

void or_dequantize_values(const uint8_t* q, uint64_t nnz, float scale, uint16_t* out) {
    /* codec.hpp:334-349 */
    for (uint64_t i = 0; i < nnz; ++i) out[i] = or_f32_to_f16((float)(int8_t)q[i] * scale);
}

float or_quantize_values(const uint16_t* vals, uint64_t nnz, uint8_t* q_out) {
    /* codec.hpp:306-331: scale = absmax/127 (1.0 if nnz == 0 or absmax == 0),
     * q = clamp(lround(v / scale), -127, 127) */
    float absmax = 0.0f;
    for (uint64_t i = 0; i < nnz; ++i) {
        float a = fabsf(or_f16_to_f32(vals[i]));
        absmax = (absmax < a) ? a : absmax;  /* std::max(absmax, a) */
    }
    const float scale = (nnz == 0 || absmax == 0.0f) ? 1.0f : absmax / 127.0f;
    for (uint64_t i = 0; i < nnz; ++i) {
        long r = lroundf(or_f16_to_f32(vals[i]) / scale);
        if (r < -127) r = -127;
        if (r > 127) r = 127;
        q_out[i] = (uint8_t)(int8_t)r;
    }
    return scale;
}

/* ---- parallel chunk fan-out (port CPU baseline) -------------------------- */

typedef struct {
    uint64_t n, cs, k0, k1;
    int eb;
    const uint8_t *bitmap, *values;
    const uint64_t* prefix;
    uint8_t* dst;
} par_job;

static void* par_worker(void* p) {
    par_job* j = (par_job*)p;
    for (uint64_t k = j->k0; k < j->k1; ++k) {
        uint64_t b = k * j->cs, e = b + j->cs < j->n ? b + j->cs : j->n;
        or_scatter_range(j->eb, j->bitmap, j->values, b, e, j->prefix[k], j->dst);
    }
    return NULL;
}

double or_decompress_parallel(uint64_t n, int eb, const uint8_t* bitmap, const uint8_t* values,
                              uint64_t cs, const uint64_t* prefix, uint8_t* dst, int threads) {
    uint64_t chunks = n == 0 ? 0 : (n + cs - 1) / cs;
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    par_job* jobs = (par_job*)malloc(sizeof(par_job) * (size_t)threads);
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (int t = 0; t < threads; ++t) {
        par_job j = {n, cs, chunks * (uint64_t)t / (uint64_t)threads,
                     chunks * (uint64_t)(t + 1) / (uint64_t)threads, eb, bitmap, values, prefix, dst};
        jobs[t] = j;
        pthread_create(&th[t], NULL, par_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    free(th);
    free(jobs);
    return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}

void or_gemv_f16(uint64_t rows, uint64_t cols, const uint16_t* w, const uint16_t* x, float* y) {
    float* xf = (float*)malloc(sizeof(float) * (size_t)(cols ? cols : 1));
    for (uint64_t c = 0; c < cols; ++c) xf[c] = or_f16_to_f32(x[c]);
    for (uint64_t r = 0; r < rows; ++r) {
        double acc = 0.0;
        const uint16_t* row = w + r * cols;
        for (uint64_t c = 0; c < cols; ++c) acc += (double)or_f16_to_f32(row[c]) * (double)xf[c];
        y[r] = (float)acc;
    }
    free(xf);
}

/* ---- multi-threaded op generator (reference-arm inputs) ------------------ */

typedef struct {
    uint64_t i0, i1, seed, target_ties, K, tie_base, cnt;
    int phase;
    uint8_t* w;
    uint64_t* hist;  /* 32768 per worker */
    uint8_t *bitmap, *values;
    uint64_t voff;
} mk_job;

static void* mk_worker(void* p) {
    mk_job* j = (mk_job*)p;
    if (j->phase == 0) {  /* synth + key histogram (weight_gen.hpp:40-55, 61-64) */
        for (uint64_t i = j->i0; i < j->i1; ++i) {
            double u = (double)(splitmix_at(j->seed, i + 1) >> 11) * 0x1.0p-53;
            uint16_t h = or_f32_to_f16((float)(2.0 * u - 1.0));
            j->w[2 * i] = (uint8_t)(h & 0xFF);
            j->w[2 * i + 1] = (uint8_t)(h >> 8);
            j->hist[h & 0x7FFFu]++;
        }
    } else if (j->phase == 1) {  /* count key == K in range */
        uint64_t c = 0;
        for (uint64_t i = j->i0; i < j->i1; ++i) c += ((j->w[2 * i] | (j->w[2 * i + 1] << 8)) & 0x7FFF) == j->K;
        j->cnt = c;
    } else if (j->phase == 2) {  /* prune (ties cut in index order) + count survivors */
        uint64_t rank = j->tie_base, c = 0;
        for (uint64_t i = j->i0; i < j->i1; ++i) {
            uint32_t k = (uint32_t)(j->w[2 * i] | (j->w[2 * i + 1] << 8)) & 0x7FFFu;
            int prune = k < j->K;
            if (k == j->K) prune = rank++ < j->target_ties;
            if (prune) { j->w[2 * i] = 0; j->w[2 * i + 1] = 0; }
            else c += (k != 0);
        }
        j->cnt = c;
    } else {  /* compress (codec.hpp:97-126); ranges are multiples of 8 elements */
        uint64_t v = j->voff;
        for (uint64_t i = j->i0; i < j->i1; ++i) {
            uint16_t h = (uint16_t)(j->w[2 * i] | (j->w[2 * i + 1] << 8));
            if (h & 0x7FFFu) {
                j->bitmap[i >> 3] |= (uint8_t)(1u << (i & 7));
                j->values[2 * v] = (uint8_t)(h & 0xFF);
                j->values[2 * v + 1] = (uint8_t)(h >> 8);
                ++v;
            }
        }
    }
    return NULL;
}

uint64_t or_make_op_mt(uint64_t rows, uint64_t cols, uint64_t seed, double sparsity, int threads,
                       uint8_t* bitmap_out, uint8_t* values_out) {
    uint64_t n = rows * cols;
    if (threads < 1) threads = 1;
    uint8_t* w = (uint8_t*)malloc((size_t)(n * 2 + 16));
    mk_job* jobs = (mk_job*)calloc((size_t)threads, sizeof(mk_job));
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    uint64_t* hist = (uint64_t*)calloc((size_t)threads * 32768, sizeof(uint64_t));
    for (int t = 0; t < threads; ++t) {  /* ranges aligned to 8 elements for the bitmap */
        jobs[t].i0 = (n * (uint64_t)t / (uint64_t)threads) & ~7ull;
        jobs[t].i1 = t == threads - 1 ? n : ((n * (uint64_t)(t + 1) / (uint64_t)threads) & ~7ull);
        jobs[t].seed = seed;
        jobs[t].w = w;
        jobs[t].hist = hist + (size_t)t * 32768;
        jobs[t].bitmap = bitmap_out;
        jobs[t].values = values_out;
    }
#define RUN_PHASE(ph)                                                            \
    do {                                                                         \
        for (int t = 0; t < threads; ++t) { jobs[t].phase = ph; pthread_create(&th[t], NULL, mk_worker, &jobs[t]); } \
        for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);           \
    } while (0)
    RUN_PHASE(0);
    uint64_t target = (uint64_t)(sparsity * (double)n), below = 0, K = 0;
    if (target > 0) {
        for (K = 0; K < 32768; ++K) {
            uint64_t hk = 0;
            for (int t = 0; t < threads; ++t) hk += hist[(size_t)t * 32768 + K];
            if (below + hk >= target) break;
            below += hk;
        }
    } else {
        K = 0; /* prune nothing: no key < 0; ties = 0 */
    }
    for (int t = 0; t < threads; ++t) jobs[t].K = K;
    RUN_PHASE(1);
    uint64_t tb = 0;
    for (int t = 0; t < threads; ++t) {
        jobs[t].tie_base = tb;
        tb += jobs[t].cnt;
        jobs[t].target_ties = target > 0 ? target - below : 0;
    }
    RUN_PHASE(2);
    uint64_t vo = 0;
    for (int t = 0; t < threads; ++t) { jobs[t].voff = vo; vo += jobs[t].cnt; }
    memset(bitmap_out, 0, (size_t)((n + 7) / 8));
    RUN_PHASE(3);
#undef RUN_PHASE
    free(hist); free(th); free(jobs); free(w);
    return vo;
}
