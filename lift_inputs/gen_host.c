/* Host twin of the seeded input recipe in lift_inputs/__init__.py (see its
 * docstring).  Holds none of the method's arithmetic.  Built with
 * -O2 -ffp-contract=off so `lo + (hi-lo)*u` is two RN fp64 ops, exactly like
 * the numpy spec and the CUDA twin (__dmul_rn/__dadd_rn). */
#include <stdint.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL
#define ID_MUL 0xD1B54A32D192ED03ULL

static inline uint64_t mix(uint64_t z) {
    z += GOLDEN;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* dist 0: uniform [lo,hi) ; dist 1: integers {-8..8}.  Returns 0 on success. */
int lift_inputs_fill_host(float *out, int64_t n, uint64_t seed, uint64_t tid,
                          int64_t i0, int dist, double lo, double hi) {
    if (n < 0 || (n > 0 && !out) || (dist != 0 && dist != 1)) return 1;
    const uint64_t base = seed * GOLDEN + tid * ID_MUL + (uint64_t)i0;
    const double span = hi - lo;
    if (dist == 0) {
        for (int64_t i = 0; i < n; ++i) {
            double u = (double)(mix(base + (uint64_t)i) >> 40) * 0x1p-24;
            out[i] = (float)(lo + span * u);   /* -ffp-contract=off: two RN ops */
        }
    } else {
        for (int64_t i = 0; i < n; ++i)
            out[i] = (float)((int64_t)((mix(base + (uint64_t)i) >> 32) % 17u) - 8);
    }
    return 0;
}
