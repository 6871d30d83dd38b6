/*
 * Strict-order CPU evaluator of one statement plan — TEST INFRASTRUCTURE ONLY
 * (the oracle's second route and the timed CPU baseline; never linked into the
 * product library).
 *
 * Restates pkg/src/elastencil/executor.py:86-176 (evaluate_statement): the
 * postorder plan of analysis.py:137-174 is interpreted one instruction at a
 * time over a block of output elements — here one output row (the innermost
 * axis) instead of a whole tile, which keeps the scratch stack in L1. Every
 * binary/unary instruction is one correctly rounded IEEE operation in the
 * plan's order; the file MUST be compiled with -ffp-contract=off (no FMA
 * contraction) and without -ffast-math, which makes the results bit-identical
 * to numpy's ufuncs (numpy >= 1.24, the reference's only dependency,
 * pkg/pyproject.toml:10-12).
 *
 * Arrays are whole C-order grids padded to rank 3 as (1,1,n) / (1,ny,nx).
 * Op codes: 0 const, 1 load, 2 neg, 3 abs, 4 sqrt, 5 add, 6 sub, 7 mul, 8 div.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAX_STACK 64

#define DEFINE_EVAL(NAME, T, SQRT, ABS)                                                   \
static int NAME(const int64_t *shape, T *out, const int64_t *lo, const int64_t *ext,     \
                const T *const *in, const int32_t *ops, const double *consts,            \
                const int32_t *slots, const int64_t *offs, int n_instr, int threads) {   \
    const int64_t ny = shape[1], nx = shape[2];                                          \
    const int64_t rows = ext[0] * ext[1], w = ext[2];                                    \
    int depth = 0, maxd = 0;                                                             \
    for (int k = 0; k < n_instr; ++k) {                                                  \
        depth += (ops[k] <= 1) ? 1 : (ops[k] <= 4 ? 0 : -1);                             \
        if (depth > maxd) maxd = depth;                                                  \
        if (depth < 0) return 2;                                                         \
    }                                                                                    \
    if (depth != 1 || maxd > MAX_STACK) return 2;                                        \
    int status = 0;                                                                      \
    _Pragma("omp parallel num_threads(threads > 0 ? threads : omp_get_max_threads())")   \
    {                                                                                    \
        T *scratch = (T *)malloc(sizeof(T) * (size_t)w * (size_t)(maxd + 1));            \
        if (!scratch) status = 3;                                                        \
        _Pragma("omp for schedule(static)")                                              \
        for (int64_t r = 0; r < rows; ++r) {                                             \
            if (!scratch) continue;                                                      \
            const int64_t z = lo[0] + r / ext[1], y = lo[1] + r % ext[1];                \
            int sp = 0;                                                                  \
            for (int k = 0; k < n_instr; ++k) {                                          \
                const int op = ops[k];                                                   \
                if (op == 0) {                                                           \
                    T *d = scratch + (size_t)sp * w; const T c = (T)consts[k];           \
                    for (int64_t i = 0; i < w; ++i) d[i] = c;                            \
                    ++sp;                                                                \
                } else if (op == 1) {                                                    \
                    T *d = scratch + (size_t)sp * w;                                     \
                    const int64_t *o = offs + 3 * k;                                     \
                    const T *s = in[slots[k]] + ((z + o[0]) * ny + (y + o[1])) * nx      \
                                 + lo[2] + o[2];                                         \
                    memcpy(d, s, sizeof(T) * (size_t)w);                                 \
                    ++sp;                                                                \
                } else if (op <= 4) {                                                    \
                    T *a = scratch + (size_t)(sp - 1) * w;                               \
                    if (op == 2)      for (int64_t i = 0; i < w; ++i) a[i] = -a[i];      \
                    else if (op == 3) for (int64_t i = 0; i < w; ++i) a[i] = ABS(a[i]);  \
                    else              for (int64_t i = 0; i < w; ++i) a[i] = SQRT(a[i]); \
                } else {                                                                 \
                    T *a = scratch + (size_t)(sp - 2) * w, *b = a + w;                   \
                    if (op == 5)      for (int64_t i = 0; i < w; ++i) a[i] = a[i] + b[i];\
                    else if (op == 6) for (int64_t i = 0; i < w; ++i) a[i] = a[i] - b[i];\
                    else if (op == 7) for (int64_t i = 0; i < w; ++i) a[i] = a[i] * b[i];\
                    else              for (int64_t i = 0; i < w; ++i) a[i] = a[i] / b[i];\
                    --sp;                                                                \
                }                                                                        \
            }                                                                            \
            memcpy(out + (z * ny + y) * nx + lo[2], scratch, sizeof(T) * (size_t)w);     \
        }                                                                                \
        free(scratch);                                                                   \
    }                                                                                    \
    return status;                                                                       \
}

DEFINE_EVAL(eval_f64, double, sqrt, fabs)
DEFINE_EVAL(eval_f32, float, sqrtf, fabsf)

/* dtype 0 = float64, 1 = float32.  Returns 0 on success. */
int oracle_eval_statement(int dtype, const int64_t *shape, void *out, const int64_t *lo,
                          const int64_t *ext, const void *const *inputs, int n_inputs,
                          const int32_t *ops, const double *consts, const int32_t *slots,
                          const int64_t *offs, int n_instr, int threads) {
    (void)n_inputs;
    if (ext[0] <= 0 || ext[1] <= 0 || ext[2] <= 0) return 0;
    if (dtype == 0)
        return eval_f64(shape, (double *)out, lo, ext, (const double *const *)inputs, ops,
                        consts, slots, offs, n_instr, threads);
    return eval_f32(shape, (float *)out, lo, ext, (const float *const *)inputs, ops, consts,
                    slots, offs, n_instr, threads);
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Position-keyed content hash (restates include/est.h est_hash_box for the
 * checker): sum over i of mix64(bits_i + 0x9e3779b97f4a7c15 * (i + 1)) mod 2^64,
 * bits = the float64 bit pattern (elem 8) or the zero-extended float32 one. */
static inline uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

uint64_t oracle_content_hash(const void *data, int64_t n, int elem, int threads) {
    uint64_t total = 0;
    _Pragma("omp parallel for reduction(+:total) schedule(static) num_threads(threads > 0 ? threads : omp_get_max_threads())")
    for (int64_t i = 0; i < n; ++i) {
        uint64_t bits = elem == 8 ? ((const uint64_t *)data)[i] : (uint64_t)((const uint32_t *)data)[i];
        total += mix64(bits + 0x9e3779b97f4a7c15ULL * (uint64_t)(i + 1));
    }
    return total;
}
