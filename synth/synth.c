/*
 * synth.c — seeded synthetic-input generator (SURVEY.md §8(d) "Value generator").
 *
 * This module is shared test/bench infrastructure: it is the ONLY code that
 * both the CPU oracle (oracle/) and the CUDA path's harness (bench.py, tests)
 * use, and it holds none of the method's arithmetic (no planning, no merge,
 * no forward pass). It turns (seed, tensor name, element index) into a value:
 *
 *   u  = splitmix64((seed XOR fnv1a64(name)) + i)          (mod 2^64)
 *   U  = (u >> 40) / 2^24                                  in [0, 1)
 *   x  = center + (2U - 1) * a                             (computed in double)
 *   out = RNE_bf16((float)x)    or (float)x for fp32 output
 *
 * Token ids use the same stream:  tok_t = floor(U_t * V)  (integer arithmetic:
 * ((u >> 40) * V) >> 24).
 *
 * Build: gcc -O3 -fopenmp -shared -fPIC synth.c -o libpbsynth.so
 */
#include <stdint.h>
#include <string.h>
#include <math.h>

static inline uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t pbs_fnv1a64(const char* s) {
    uint64_t h = 0xCBF29CE484222325ULL;
    for (; *s; ++s) { h ^= (uint8_t)*s; h *= 0x100000001B3ULL; }
    return h;
}

static inline uint16_t f32_to_bf16_rne(float f) {
    uint32_t u; memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u) return (uint16_t)((u >> 16) | ((u & 0xFFFF) ? 0x40 : 0));
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;
    return (uint16_t)(u >> 16);
}

static inline float value_at(uint64_t base, int64_t i, double center, double a) {
    uint64_t u = splitmix64(base + (uint64_t)i);
    double U = (double)(u >> 40) * (1.0 / 16777216.0);
    return (float)(center + (2.0 * U - 1.0) * a);
}

/* Fill n bf16 values (row-major element index i = start + k). */
void pbs_fill_bf16(uint16_t* dst, int64_t n, int64_t start, uint64_t seed,
                   const char* name, double center, double a) {
    uint64_t base = seed ^ pbs_fnv1a64(name);
    #pragma omp parallel for schedule(static) if (n > (1 << 20))
    for (int64_t k = 0; k < n; ++k) dst[k] = f32_to_bf16_rne(value_at(base, start + k, center, a));
}

/* Fill n fp32 values. */
void pbs_fill_f32(float* dst, int64_t n, int64_t start, uint64_t seed,
                  const char* name, double center, double a) {
    uint64_t base = seed ^ pbs_fnv1a64(name);
    #pragma omp parallel for schedule(static) if (n > (1 << 20))
    for (int64_t k = 0; k < n; ++k) dst[k] = value_at(base, start + k, center, a);
}

/* Token ids in [0, vocab). */
void pbs_fill_tokens(int32_t* dst, int64_t n, uint64_t seed, const char* name, int64_t vocab) {
    uint64_t base = seed ^ pbs_fnv1a64(name);
    for (int64_t k = 0; k < n; ++k) {
        uint64_t u = splitmix64(base + (uint64_t)k);
        dst[k] = (int32_t)(((u >> 40) * (uint64_t)vocab) >> 24);
    }
}

/* Fill n bytes with a constant (used by the harness to put device-mirror host
 * buffers in a known state); kept here so the harness needs no numpy loops. */
void pbs_memset(void* dst, int value, int64_t n) {
    #pragma omp parallel for schedule(static) if (n > (1 << 24))
    for (int64_t k = 0; k < n; k += (1 << 22)) {
        int64_t len = n - k < (1 << 22) ? n - k : (1 << 22);
        memset((char*)dst + k, value, (size_t)len);
    }
}
