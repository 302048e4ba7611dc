/*
 * qv_oracle.c — TEST INFRASTRUCTURE ONLY. CPU restatement of the QVecOpt
 * reference's gate-application path, used as the parity checker for the CUDA
 * engine. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load this library; the product path never does.
 *
 * Parity is pinned (tests/test_oracle.py) against
 *   - the frozen amplitudes of random_circuit(3,20,42) in the reference's
 *     own test (reference proj/tests/test_dense.cpp:189-209), and
 *   - fixtures produced by the reference engine itself compiled here
 *     (oracle/_ref, recipe oracle/Makefile; generator tests/golden/make_golden.py).
 *
 * Build: gcc -O2 -ffp-contract=off (no FMA contraction), like the reference's
 * -O2 build without -march (reference proj/src/CMakeLists.txt:17).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Same layout as qvg_gate in include/qvg.h (80 bytes). */
typedef struct qvo_gate {
    uint32_t kind; /* 0 single, 1 controlled */
    uint32_t target;
    int32_t control; /* -1: none */
    uint32_t flags;
    double u[8]; /* re00 im00 re01 im01 re10 im10 re11 im11 */
} qvo_gate;

_Static_assert(sizeof(qvo_gate) == 80, "qvo_gate must match qvg_gate");

/* ------------------------------------------------------------------------
 * mt19937_64 (Matsumoto-Nishimura 64-bit Mersenne Twister, the generator the
 * reference seeds with std::mt19937_64, engine.cpp:234-238). Published
 * parameters: w=64 n=312 m=156 r=31.
 */
#define MT_N 312
#define MT_M 156
typedef struct qvo_mt {
    uint64_t mt[MT_N];
    int idx;
} qvo_mt;

void qvo_mt_seed(qvo_mt *g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i) {
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) +
                   (uint64_t)i;
    }
    g->idx = MT_N;
}

uint64_t qvo_mt_next(qvo_mt *g) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    if (g->idx >= MT_N) {
        for (int i = 0; i < MT_N; ++i) {
            uint64_t x = (g->mt[i] & upper) | (g->mt[(i + 1) % MT_N] & lower);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* reference engine.cpp:159-171 — rejection below 2^64 mod bound. */
uint64_t qvo_uniform_below(qvo_mt *g, uint64_t bound) {
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
        const uint64_t r = qvo_mt_next(g);
        if (r >= threshold) return r % bound;
    }
}

/* reference engine.cpp:173-175 */
double qvo_uniform_unit(qvo_mt *g) { return (double)(qvo_mt_next(g) >> 11) * 0x1.0p-53; }

/* ------------------------------------------------------------------------
 * Gate library (reference gates.cpp:29-93). Index order follows
 * builtin_gate_names() (gates.cpp:23-27) then cx, cz (engine.cpp:182-186).
 */
enum { G_H, G_X, G_Y, G_Z, G_S, G_SDG, G_T, G_TDG, G_RX, G_RY, G_RZ, G_U, G_CX, G_CZ };

static void set_u(double *u, double complex a, double complex b, double complex c,
                  double complex d) {
    u[0] = creal(a); u[1] = cimag(a);
    u[2] = creal(b); u[3] = cimag(b);
    u[4] = creal(c); u[5] = cimag(c);
    u[6] = creal(d); u[7] = cimag(d);
}

/* std::exp(i1 * x) as libstdc++ evaluates it: i1 * x = (0*x, 1*x), then cexp. */
static double complex exp_i(double x) { return cexp(CMPLX(0.0 * x, x)); }

static void fixed_gate(int id, const double *p, double *u) {
    const double rt2 = 1.0 / sqrt(2.0);
    const double pi = 3.14159265358979323846;
    switch (id) {
    case G_H: set_u(u, rt2, rt2, rt2, -rt2); break;
    case G_X: set_u(u, 0, 1, 1, 0); break;
    case G_Y: set_u(u, 0, CMPLX(0, -1), CMPLX(0, 1), 0); break;
    case G_Z: set_u(u, 1, 0, 0, -1); break;
    case G_S: set_u(u, 1, 0, 0, CMPLX(0, 1)); break;
    case G_SDG: set_u(u, 1, 0, 0, CMPLX(0, -1)); break;
    case G_T: set_u(u, 1, 0, 0, exp_i(pi / 4)); break;
    case G_TDG: set_u(u, 1, 0, 0, exp_i(-pi / 4)); break;
    case G_RX: {
        const double c = cos(p[0] / 2), s = sin(p[0] / 2);
        set_u(u, c, CMPLX(0, -s), CMPLX(0, -s), c);
        break;
    }
    case G_RY: {
        const double c = cos(p[0] / 2), s = sin(p[0] / 2);
        set_u(u, c, -s, s, c);
        break;
    }
    case G_RZ: {
        const double h = p[0] / 2;
        set_u(u, exp_i(-h), 0, 0, exp_i(h));
        break;
    }
    default: memcpy(u, p, 8 * sizeof(double)); break;
    }
}

/* complex * real, as libstdc++'s operator*(complex, T): (re*y, im*y). */
static double complex cmul_r(double complex a, double y) { return CMPLX(creal(a) * y, cimag(a) * y); }

/* reference engine.cpp:177-232. Fills ops[0..depth) and returns depth; also
 * writes the gate-library index of every op to names (may be NULL). */
uint32_t qvo_random_circuit(uint32_t n, uint32_t depth, uint64_t seed, qvo_gate *ops,
                            int32_t *names) {
    qvo_mt g;
    qvo_mt_seed(&g, seed);
    const uint64_t pool = n >= 2 ? 14 : 12;
    const double two_pi = 2.0 * 3.14159265358979323846;
    for (uint32_t k = 0; k < depth; ++k) {
        const int id = (int)qvo_uniform_below(&g, pool);
        const uint32_t target = (uint32_t)qvo_uniform_below(&g, n);
        qvo_gate *op = &ops[k];
        memset(op, 0, sizeof(*op));
        op->target = target;
        op->control = -1;
        if (names) names[k] = id;
        if (id == G_CX || id == G_CZ) {
            uint32_t control = (uint32_t)qvo_uniform_below(&g, n - 1);
            if (control >= target) ++control;
            op->kind = 1;
            op->control = (int32_t)control;
            fixed_gate(id == G_CX ? G_X : G_Z, NULL, op->u);
            continue;
        }
        if (id <= G_TDG) {
            fixed_gate(id, NULL, op->u);
        } else if (id <= G_RZ) {
            const double p = two_pi * qvo_uniform_unit(&g);
            fixed_gate(id, &p, op->u);
        } else {
            const double phi = two_pi * qvo_uniform_unit(&g);
            const double beta = two_pi * qvo_uniform_unit(&g);
            const double gamma = two_pi * qvo_uniform_unit(&g);
            const double delta = two_pi * qvo_uniform_unit(&g);
            const double c = cos(gamma / 2);
            const double s = sin(gamma / 2);
            const double complex u00 = cmul_r(exp_i(phi - beta / 2 - delta / 2), c);
            const double complex u01 = cmul_r(-exp_i(phi - beta / 2 + delta / 2), s);
            const double complex u10 = cmul_r(exp_i(phi + beta / 2 - delta / 2), s);
            const double complex u11 = cmul_r(exp_i(phi + beta / 2 + delta / 2), c);
            set_u(op->u, u00, u01, u10, u11);
        }
    }
    return depth;
}

/* ------------------------------------------------------------------------
 * The paired update. reference kernel.cpp:14-19 (apply_pair) with the
 * arithmetic std::complex<double> compiles to at -O2 without -march:
 * (a+bi)(c+di) = (ac - bd) + (ad + bc)i, then a complex add. No FMA.
 */
static inline void pair_update(double *lo, double *hi, const double *u) {
    const double ar = lo[0], ai = lo[1], br = hi[0], bi = hi[1];
    const double l_re = (u[0] * ar - u[1] * ai) + (u[2] * br - u[3] * bi);
    const double l_im = (u[0] * ai + u[1] * ar) + (u[2] * bi + u[3] * br);
    const double h_re = (u[4] * ar - u[5] * ai) + (u[6] * br - u[7] * bi);
    const double h_im = (u[4] * ai + u[5] * ar) + (u[6] * bi + u[7] * br);
    lo[0] = l_re; lo[1] = l_im;
    hi[0] = h_re; hi[1] = h_im;
}

/* One op over the whole state: every base index i (bit target == 0) whose
 * control bit is set (evaluated on the base index, kernel.cpp:21-24,72-77)
 * updates the pair (i, i ^ 2^target) (types.hpp:19-26). Traversal order is
 * irrelevant: pairs are disjoint. */
int qvo_apply_gate(uint32_t n, double *amps, const qvo_gate *op) {
    if (op->target >= n) return 1;
    if (op->kind == 1 && (op->control < 0 || (uint32_t)op->control >= n ||
                          (uint32_t)op->control == op->target))
        return 1;
    const uint64_t dim = 1ULL << n;
    const uint64_t stride = 1ULL << op->target;
    const int has_ctrl = op->kind == 1;
    const uint64_t cmask = has_ctrl ? (1ULL << op->control) : 0;
    /* The reference's (group, j) double loop (kernel.cpp:72-73) visits the
     * bases j = insert-0-at-target(p), p in [0, dim/2); pairs are disjoint,
     * so splitting p over OpenMP threads gives the same bits. */
    const int64_t npairs = (int64_t)(dim >> 1);
    const unsigned t = op->target;
#pragma omp parallel for schedule(static) if (npairs >= (1 << 16))
    for (int64_t p = 0; p < npairs; ++p) {
        const uint64_t j = (((uint64_t)p >> t) << (t + 1)) | ((uint64_t)p & (stride - 1));
        if (has_ctrl && !(j & cmask)) continue;
        pair_update(&amps[2 * j], &amps[2 * (j + stride)], op->u);
    }
    return 0;
}

int qvo_apply(uint32_t n, double *amps, const qvo_gate *ops, uint64_t count) {
    for (uint64_t k = 0; k < count; ++k) {
        if (qvo_apply_gate(n, amps, &ops[k])) return (int)(k + 1);
    }
    return 0;
}

/* |index> (BlockStore::create gives |0...0>, store.cpp:181-214). */
void qvo_basis_state(uint32_t n, double *amps, uint64_t index) {
    memset(amps, 0, (size_t)(2ULL << n) * sizeof(double));
    amps[2 * index] = 1.0;
}

/* std::norm = re*re + im*im (engine.cpp:518). */
void qvo_probabilities(uint64_t count, const double *amps, double *out) {
    for (uint64_t i = 0; i < count; ++i) out[i] = amps[2 * i] * amps[2 * i] + amps[2 * i + 1] * amps[2 * i + 1];
}

/* Kahan-compensated norm (store.cpp:301-316). */
double qvo_norm(uint64_t count, const double *amps) {
    double sum = 0.0, carry = 0.0;
    for (uint64_t i = 0; i < count; ++i) {
        const double term = (amps[2 * i] * amps[2 * i] + amps[2 * i + 1] * amps[2 * i + 1]) - carry;
        const double next = sum + term;
        carry = (next - sum) - term;
        sum = next;
    }
    return sqrt(sum);
}

/* max_i |a_i - b_i| (dense.cpp:174-183, std::abs = hypot). */
double qvo_max_deviation(uint64_t count, const double *a, const double *b) {
    double dev = 0.0;
    for (uint64_t i = 0; i < count; ++i) {
        const double d = hypot(a[2 * i] - b[2 * i], a[2 * i + 1] - b[2 * i + 1]);
        if (!(d <= dev)) dev = d;
    }
    return dev;
}
