/*
 * qsim_oracle.c — TEST INFRASTRUCTURE ONLY (see qsim_oracle.h).
 *
 * Plain-C restatement of the reference CPU path. Every function cites the
 * reference file:line (paths relative to /root/reference/proj) it restates.
 * Compiled with -ffp-contract=off so every product and sum rounds separately,
 * as the reference does on x86-64 without -march (no FMA contraction).
 */
#include "qsim_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];
static int g_threads = 1;

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* orc_last_error(void) { return g_err; }

void orc_set_threads(int threads) { g_threads = threads < 1 ? 1 : threads; }

/* ------------------------------------------------------------------ gates */

/* gates.cpp:27-36 (phase_matrix) and gates.cpp:40-77 (gate_matrix). */
int orc_gate_matrix(int32_t gate, double phi, double re[4], double im[4]) {
    for (int i = 0; i < 4; ++i) re[i] = im[i] = 0.0;
    const double pi = 3.14159265358979323846; /* std::numbers::pi */
    double p;
    switch (gate) {
    case QSB_GATE_H: {
        const double s = sqrt(0.5);
        re[0] = s; re[1] = s; re[2] = s; re[3] = -s;
        return ORC_OK;
    }
    case QSB_GATE_X: re[1] = 1.0; re[2] = 1.0; return ORC_OK;
    case QSB_GATE_Y: im[1] = -1.0; im[2] = 1.0; return ORC_OK;
    case QSB_GATE_Z: re[0] = 1.0; re[3] = -1.0; return ORC_OK;
    case QSB_GATE_S: p = pi / 2.0; break;
    case QSB_GATE_T: p = pi / 4.0; break;
    case QSB_GATE_R: p = phi; break;
    default: return fail(ORC_ERR_ARGUMENT, "unknown gate tag");
    }
    if (!isfinite(p)) return fail(ORC_ERR_ARGUMENT, "phase gate: phi must be finite");
    re[0] = 1.0;
    re[3] = cos(p);
    im[3] = sin(p);
    return ORC_OK;
}

/* gates.cpp:79-110 */
int orc_controlled_unitary(const double u_re[4], const double u_im[4], int64_t control_pos,
                           int64_t target_pos, int64_t span, double* re, double* im) {
    if (span < 2 || span > 30) return fail(ORC_ERR_ARGUMENT, "controlled_unitary: span must be in [2, 30]");
    if (control_pos == target_pos || control_pos >= span || target_pos >= span || control_pos < 0 ||
        target_pos < 0)
        return fail(ORC_ERR_ARGUMENT, "controlled_unitary: invalid control/target positions");
    const int64_t dim = (int64_t)1 << span;
    const int64_t cmask = (int64_t)1 << (span - 1 - control_pos);
    const int64_t tmask = (int64_t)1 << (span - 1 - target_pos);
    memset(re, 0, sizeof(double) * dim * dim);
    memset(im, 0, sizeof(double) * dim * dim);
    for (int64_t col = 0; col < dim; ++col) {
        if ((col & cmask) == 0) {
            re[col * dim + col] = 1.0;
            continue;
        }
        const int64_t tbit = (col & tmask) ? 1 : 0;
        const int64_t row0 = col & ~tmask;
        const int64_t row1 = col | tmask;
        re[row0 * dim + col] = u_re[0 * 2 + tbit];
        im[row0 * dim + col] = u_im[0 * 2 + tbit];
        re[row1 * dim + col] = u_re[1 * 2 + tbit];
        im[row1 * dim + col] = u_im[1 * 2 + tbit];
    }
    return ORC_OK;
}

/* ----------------------------------------------------------------- linalg */

/* linalg.cpp:109-129: block (ia, ja) of c is a(ia, ja) * b; zero a-entries skipped. */
int orc_kronecker(const double* a_re, const double* a_im, int64_t ar, int64_t ac,
                  const double* b_re, const double* b_im, int64_t br, int64_t bc,
                  double* c_re, double* c_im) {
    const int64_t cc = ac * bc;
    memset(c_re, 0, sizeof(double) * ar * br * cc);
    memset(c_im, 0, sizeof(double) * ar * br * cc);
    for (int64_t ia = 0; ia < ar; ++ia) {
        for (int64_t ja = 0; ja < ac; ++ja) {
            const double xr = a_re[ia * ac + ja];
            const double xi = a_im[ia * ac + ja];
            if (xr == 0.0 && xi == 0.0) continue;
            for (int64_t ib = 0; ib < br; ++ib) {
                const int64_t row = ia * br + ib;
                for (int64_t jb = 0; jb < bc; ++jb) {
                    const int64_t col = ja * bc + jb;
                    c_re[row * cc + col] = xr * b_re[ib * bc + jb] - xi * b_im[ib * bc + jb];
                    c_im[row * cc + col] = xr * b_im[ib * bc + jb] + xi * b_re[ib * bc + jb];
                }
            }
        }
    }
    return ORC_OK;
}

typedef struct {
    const double *a_re, *a_im, *b_re, *b_im;
    double *c_re, *c_im;
    int64_t k, n, row_begin, row_end;
} mm_job;

/* linalg.cpp:46-68 (matmul_rows): i-k-j order, k ascending per output entry. */
static void* matmul_rows(void* arg) {
    const mm_job* j = (const mm_job*)arg;
    for (int64_t i = j->row_begin; i < j->row_end; ++i) {
        double* cre = j->c_re + i * j->n;
        double* cim = j->c_im + i * j->n;
        for (int64_t x = 0; x < j->n; ++x) cre[x] = cim[x] = 0.0;
        for (int64_t kk = 0; kk < j->k; ++kk) {
            const double ar = j->a_re[i * j->k + kk];
            const double ai = j->a_im[i * j->k + kk];
            const double* bre = j->b_re + kk * j->n;
            const double* bim = j->b_im + kk * j->n;
            for (int64_t x = 0; x < j->n; ++x) {
                cre[x] += ar * bre[x] - ai * bim[x];
                cim[x] += ar * bim[x] + ai * bre[x];
            }
        }
    }
    return NULL;
}

/* linalg.cpp:72-87, with the row-chunk split of parallel.cpp:58-90. */
int orc_matmul(const double* a_re, const double* a_im, const double* b_re, const double* b_im,
               int64_t m, int64_t k, int64_t n, double* c_re, double* c_im) {
    int64_t workers = g_threads < m ? g_threads : m;
    if (workers < 1) workers = 1;
    mm_job jobs[256];
    pthread_t tids[256];
    if (workers > 256) workers = 256;
    for (int64_t w = 0; w < workers; ++w) {
        jobs[w] = (mm_job){a_re, a_im, b_re, b_im, c_re, c_im, k, n, m * w / workers, m * (w + 1) / workers};
    }
    if (workers == 1) {
        matmul_rows(&jobs[0]);
        return ORC_OK;
    }
    for (int64_t w = 0; w < workers; ++w) pthread_create(&tids[w], NULL, matmul_rows, &jobs[w]);
    for (int64_t w = 0; w < workers; ++w) pthread_join(tids[w], NULL);
    return ORC_OK;
}

/* linalg.cpp:89-107 */
int orc_matvec(const double* a_re, const double* a_im, int64_t m, int64_t k, const double* v_re,
               const double* v_im, double* out_re, double* out_im) {
    for (int64_t i = 0; i < m; ++i) {
        double sr = 0.0, si = 0.0;
        for (int64_t x = 0; x < k; ++x) {
            sr += a_re[i * k + x] * v_re[x] - a_im[i * k + x] * v_im[x];
            si += a_re[i * k + x] * v_im[x] + a_im[i * k + x] * v_re[x];
        }
        out_re[i] = sr;
        out_im[i] = si;
    }
    return ORC_OK;
}

/* linalg.cpp:131-155 */
int orc_is_unitary(const double* re, const double* im, int64_t n, double tol) {
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = 0; j < n; ++j) {
            double sr = 0.0, si = 0.0;
            for (int64_t k = 0; k < n; ++k) {
                sr += re[k * n + i] * re[k * n + j] + im[k * n + i] * im[k * n + j];
                si += re[k * n + i] * im[k * n + j] - im[k * n + i] * re[k * n + j];
            }
            if (i == j) sr -= 1.0;
            if (fabs(sr) > tol || fabs(si) > tol) return 0;
        }
    }
    return 1;
}

/* linalg.cpp:157-180 */
double orc_max_entry_diff(const double* a_re, const double* a_im, const double* b_re,
                          const double* b_im, int64_t count) {
    double worst = 0.0;
    for (int64_t i = 0; i < count; ++i) {
        const double d = hypot(a_re[i] - b_re[i], a_im[i] - b_im[i]);
        if (d > worst) worst = d;
    }
    return worst;
}

/* ------------------------------------------------------ unitary backend */

/* SpanOperand (unitary_backend.cpp:31-35): an op's contiguous qubit interval
 * and its dense block matrix. */
typedef struct {
    int64_t first, span;
    double *re, *im; /* (2^span)^2 */
} operand;

static void free_operand(operand* o) {
    free(o->re);
    free(o->im);
    o->re = o->im = NULL;
}

static int identity2(operand* o, int64_t first) {
    o->first = first;
    o->span = 1;
    o->re = calloc(4, sizeof(double));
    o->im = calloc(4, sizeof(double));
    if (!o->re || !o->im) return fail(ORC_ERR_NOMEM, "out of memory");
    o->re[0] = o->re[3] = 1.0;
    return ORC_OK;
}

/* unitary_backend.cpp:37-58 (make_operand) */
static int make_operand(const qsb_circuit* c, const qsb_op* op, operand* o) {
    o->re = o->im = NULL;
    if (op->kind == QSB_OP_GATE) {
        o->first = op->target;
        o->span = 1;
        o->re = malloc(4 * sizeof(double));
        o->im = malloc(4 * sizeof(double));
        if (!o->re || !o->im) return fail(ORC_ERR_NOMEM, "out of memory");
        return orc_gate_matrix(op->gate, op->phi, o->re, o->im);
    }
    if (op->kind == QSB_OP_CONTROL) {
        const int64_t lo = op->control < op->target ? op->control : op->target;
        const int64_t hi = op->control < op->target ? op->target : op->control;
        o->first = lo;
        o->span = hi - lo + 1;
        double ur[4], ui[4];
        int rc = orc_gate_matrix(op->gate, op->phi, ur, ui);
        if (rc) return rc;
        const int64_t dim = (int64_t)1 << o->span;
        o->re = malloc(sizeof(double) * dim * dim);
        o->im = malloc(sizeof(double) * dim * dim);
        if (!o->re || !o->im) return fail(ORC_ERR_NOMEM, "out of memory");
        return orc_controlled_unitary(ur, ui, op->control - lo, op->target - lo, o->span, o->re, o->im);
    }
    if (op->kind == QSB_OP_FUNCTION) {
        if (op->function < 0 || op->function >= c->n_functions)
            return fail(ORC_ERR_LOOKUP, "registry: no function with index %d", op->function);
        const qsb_function* f = &c->functions[op->function];
        if (f->dim != ((int64_t)1 << op->count))
            return fail(ORC_ERR_VALIDATION, "function %d no longer matches its registered dimension",
                        op->function);
        o->first = op->first;
        o->span = op->count;
        o->re = malloc(sizeof(double) * f->dim * f->dim);
        o->im = malloc(sizeof(double) * f->dim * f->dim);
        if (!o->re || !o->im) return fail(ORC_ERR_NOMEM, "out of memory");
        memcpy(o->re, f->re, sizeof(double) * f->dim * f->dim);
        memcpy(o->im, f->im, sizeof(double) * f->dim * f->dim);
        return ORC_OK;
    }
    if (op->kind == QSB_OP_INSTRUCTION) return identity2(o, op->target);
    return fail(ORC_ERR_ARGUMENT, "unknown operation kind %d", op->kind);
}

/* unitary_backend.cpp:31-58 interval of an op without building its matrix. */
static void op_interval(const qsb_op* op, int64_t* first, int64_t* span) {
    if (op->kind == QSB_OP_CONTROL) {
        const int64_t lo = op->control < op->target ? op->control : op->target;
        const int64_t hi = op->control < op->target ? op->target : op->control;
        *first = lo;
        *span = hi - lo + 1;
    } else if (op->kind == QSB_OP_FUNCTION) {
        *first = op->first;
        *span = op->count;
    } else {
        *first = op->target;
        *span = 1;
    }
}

/* unitary_backend.cpp:63-91 (layered_operands): greedy first-fit of the step's
 * ops, in insertion order, into layers of pairwise-disjoint intervals. */
int orc_step_layers(const qsb_circuit* c, int32_t step, int32_t* n_layers, int32_t* layer_of_op) {
    if (step < 0 || step >= c->n_steps) return fail(ORC_ERR_ARGUMENT, "step out of range");
    const int32_t b = c->step_offsets[step], e = c->step_offsets[step + 1];
    int32_t layers = 0;
    for (int32_t i = b; i < e; ++i) {
        int64_t f, s;
        op_interval(&c->ops[i], &f, &s);
        int32_t placed = -1;
        for (int32_t l = 0; l < layers && placed < 0; ++l) {
            int fits = 1;
            for (int32_t j = b; j < i && fits; ++j) {
                if (layer_of_op[j - b] != l) continue;
                int64_t of, os;
                op_interval(&c->ops[j], &of, &os);
                const int disjoint = f + s <= of || of + os <= f;
                if (!disjoint) fits = 0;
            }
            if (fits) placed = l;
        }
        if (placed < 0) placed = layers++;
        layer_of_op[i - b] = placed;
    }
    *n_layers = layers;
    return ORC_OK;
}

/* unitary_backend.cpp:95-125: fill_layer (sort by first, I2 gaps, qubit 0
 * first) followed by the left Kronecker fold. */
static int fold_layer(const qsb_circuit* c, int32_t step, int32_t layer, const int32_t* layer_of_op,
                      double** out_re, double** out_im) {
    const int64_t n = c->n_qubits;
    const int32_t b = c->step_offsets[step], e = c->step_offsets[step + 1];
    operand list[64];
    int nlist = 0, rc = ORC_OK;
    /* operands of this layer sorted by first (intervals are disjoint, so firsts are distinct) */
    int32_t idx[64];
    int nidx = 0;
    for (int32_t i = b; i < e; ++i)
        if (layer_of_op[i - b] == layer) idx[nidx++] = i;
    for (int x = 1; x < nidx; ++x) {
        int32_t v = idx[x];
        int64_t fv, sv;
        op_interval(&c->ops[v], &fv, &sv);
        int y = x - 1;
        while (y >= 0) {
            int64_t fy, sy;
            op_interval(&c->ops[idx[y]], &fy, &sy);
            if (fy <= fv) break;
            idx[y + 1] = idx[y];
            --y;
        }
        idx[y + 1] = v;
    }
    int64_t cursor = 0;
    for (int x = 0; x < nidx && rc == ORC_OK; ++x) {
        operand o;
        rc = make_operand(c, &c->ops[idx[x]], &o);
        if (rc) { free_operand(&o); break; }
        if (o.first < cursor) {
            free_operand(&o);
            rc = fail(ORC_ERR_VALIDATION, "step operands overlap on qubit %lld", (long long)o.first);
            break;
        }
        for (; cursor < o.first; ++cursor) {
            rc = identity2(&list[nlist++], cursor);
            if (rc) break;
        }
        cursor += o.span;
        list[nlist++] = o;
    }
    for (; rc == ORC_OK && cursor < n; ++cursor) rc = identity2(&list[nlist++], cursor);
    if (rc) {
        for (int x = 0; x < nlist; ++x) free_operand(&list[x]);
        return rc;
    }
    /* left fold: result = list[0]; result = kron(result, list[i]) */
    int64_t dim = (int64_t)1 << list[0].span;
    double* acc_re = list[0].re;
    double* acc_im = list[0].im;
    list[0].re = list[0].im = NULL;
    for (int x = 1; x < nlist; ++x) {
        const int64_t bd = (int64_t)1 << list[x].span;
        const int64_t nd = dim * bd;
        double* nr = malloc(sizeof(double) * nd * nd);
        double* ni = malloc(sizeof(double) * nd * nd);
        if (!nr || !ni) {
            free(nr); free(ni); free(acc_re); free(acc_im);
            for (int y = x; y < nlist; ++y) free_operand(&list[y]);
            return fail(ORC_ERR_NOMEM, "out of memory");
        }
        orc_kronecker(acc_re, acc_im, dim, dim, list[x].re, list[x].im, bd, bd, nr, ni);
        free(acc_re);
        free(acc_im);
        free_operand(&list[x]);
        acc_re = nr;
        acc_im = ni;
        dim = nd;
    }
    *out_re = acc_re;
    *out_im = acc_im;
    return ORC_OK;
}

static int check_step(const qsb_circuit* c, int32_t step) {
    if (!c || c->n_qubits < 1 || c->n_qubits > 30) return fail(ORC_ERR_ARGUMENT, "bad circuit");
    if (step < 0 || step >= c->n_steps) return fail(ORC_ERR_ARGUMENT, "step out of range");
    if (c->step_offsets[step + 1] - c->step_offsets[step] > 64)
        return fail(ORC_ERR_ARGUMENT, "oracle supports at most 64 ops per step");
    return ORC_OK;
}

int orc_layer_operator(const qsb_circuit* c, int32_t step, int32_t layer, double* re, double* im) {
    int rc = check_step(c, step);
    if (rc) return rc;
    int32_t nl, lo[64];
    rc = orc_step_layers(c, step, &nl, lo);
    if (rc) return rc;
    if (layer < 0 || layer >= nl) return fail(ORC_ERR_ARGUMENT, "layer out of range");
    double *r, *i;
    rc = fold_layer(c, step, layer, lo, &r, &i);
    if (rc) return rc;
    const int64_t N = (int64_t)1 << c->n_qubits;
    memcpy(re, r, sizeof(double) * N * N);
    memcpy(im, i, sizeof(double) * N * N);
    free(r);
    free(i);
    return ORC_OK;
}

/* unitary_backend.cpp:141-154: S = L_m * ... * L_1 (serial matmul per extra layer). */
int orc_step_unitary(const qsb_circuit* c, int32_t step, double* re, double* im) {
    int rc = check_step(c, step);
    if (rc) return rc;
    const int64_t N = (int64_t)1 << c->n_qubits;
    int32_t nl, lo[64];
    rc = orc_step_layers(c, step, &nl, lo);
    if (rc) return rc;
    if (nl == 0) { /* empty step -> identity (:144-146) */
        memset(re, 0, sizeof(double) * N * N);
        memset(im, 0, sizeof(double) * N * N);
        for (int64_t d = 0; d < N; ++d) re[d * N + d] = 1.0;
        return ORC_OK;
    }
    double *r, *i;
    rc = fold_layer(c, step, 0, lo, &r, &i);
    if (rc) return rc;
    const int saved = g_threads;
    g_threads = 1; /* the reference multiplies layers with the default ExecMode::Serial (:151) */
    for (int32_t l = 1; l < nl; ++l) {
        double *lr, *li;
        rc = fold_layer(c, step, l, lo, &lr, &li);
        if (rc) break;
        double* nr = malloc(sizeof(double) * N * N);
        double* ni = malloc(sizeof(double) * N * N);
        orc_matmul(lr, li, r, i, N, N, N, nr, ni);
        free(lr); free(li); free(r); free(i);
        r = nr;
        i = ni;
    }
    g_threads = saved;
    if (rc == ORC_OK) {
        memcpy(re, r, sizeof(double) * N * N);
        memcpy(im, i, sizeof(double) * N * N);
    }
    free(r);
    free(i);
    return rc;
}

/* tests/support/test_util.hpp:135-142: U = I; for each step U = step_unitary * U. */
int orc_circuit_unitary(const qsb_circuit* c, double* re, double* im) {
    const int64_t N = (int64_t)1 << c->n_qubits;
    double* sr = malloc(sizeof(double) * N * N);
    double* si = malloc(sizeof(double) * N * N);
    double* tr = malloc(sizeof(double) * N * N);
    double* ti = malloc(sizeof(double) * N * N);
    if (!sr || !si || !tr || !ti) { free(sr); free(si); free(tr); free(ti); return fail(ORC_ERR_NOMEM, "out of memory"); }
    memset(re, 0, sizeof(double) * N * N);
    memset(im, 0, sizeof(double) * N * N);
    for (int64_t d = 0; d < N; ++d) re[d * N + d] = 1.0;
    int rc = ORC_OK;
    for (int32_t s = 0; s < c->n_steps && rc == ORC_OK; ++s) {
        rc = orc_step_unitary(c, s, sr, si);
        if (rc) break;
        orc_matmul(sr, si, re, im, N, N, N, tr, ti);
        memcpy(re, tr, sizeof(double) * N * N);
        memcpy(im, ti, sizeof(double) * N * N);
    }
    free(sr); free(si); free(tr); free(ti);
    return rc;
}

/* backend_util.cpp:21-32: reset is only allowed in the final step. */
int orc_validate_instruction_placement(const qsb_circuit* c) {
    for (int32_t s = 0; s + 1 < c->n_steps; ++s)
        for (int32_t i = c->step_offsets[s]; i < c->step_offsets[s + 1]; ++i)
            if (c->ops[i].kind == QSB_OP_INSTRUCTION && c->ops[i].instruction == QSB_INSTR_RESET)
                return fail(ORC_ERR_VALIDATION, "reset is only supported in the final step");
    return ORC_OK;
}

/* unitary_backend.cpp:156-166 */
uint64_t orc_memory_estimate(int32_t n_qubits, int32_t kind) {
    if (n_qubits < 1 || n_qubits > 30) return 0;
    const uint64_t dim = (uint64_t)1 << n_qubits;
    return kind == 0 ? dim * dim * 8 + dim * 8 : dim * 8;
}

/* unitary_backend.cpp:168-179 */
uint64_t orc_engine_memory_estimate(int32_t n_qubits, int32_t kind) {
    if (n_qubits < 1 || n_qubits > 29) return 0;
    const uint64_t dim = (uint64_t)1 << n_qubits;
    return kind == 0 ? 3 * dim * dim * 16 + dim * 16 : dim * 16;
}

/* unitary_backend.cpp:181-192 */
void orc_format_bytes(uint64_t bytes, char* buf, size_t len) {
    static const char* units[] = {"B", "kB", "MB", "GB", "TB", "PB"};
    double v = (double)bytes;
    int u = 0;
    while (v >= 1000.0 && u + 1 < 6) { v /= 1000.0; ++u; }
    snprintf(buf, len, u == 0 ? "%.0f %s" : "%.2f %s", v, units[u]);
}

/* unitary_backend.cpp:194-215 */
int orc_unitary_simulate(const qsb_circuit* c, int32_t guard, double* psi_re, double* psi_im) {
    const int32_t g = guard > 0 ? guard : 14; /* kUnitaryQubitGuard, unitary_backend.hpp:52 */
    if (c->n_qubits > g) {
        char a[32], b[32];
        orc_format_bytes(orc_memory_estimate(c->n_qubits, 0), a, sizeof a);
        orc_format_bytes(orc_engine_memory_estimate(c->n_qubits, 0), b, sizeof b);
        return fail(ORC_ERR_RESOURCE,
                    "unitary backend refuses %d qubits (guard %d): estimated memory %llu bytes (%s at 8 "
                    "bytes per complex; engine-accurate %s)",
                    c->n_qubits, g, (unsigned long long)orc_memory_estimate(c->n_qubits, 0), a, b);
    }
    int rc = orc_validate_instruction_placement(c);
    if (rc) return rc;
    const int64_t N = (int64_t)1 << c->n_qubits;
    double* ur = malloc(sizeof(double) * N * N);
    double* ui = malloc(sizeof(double) * N * N);
    if (!ur || !ui) { free(ur); free(ui); return fail(ORC_ERR_NOMEM, "out of memory"); }
    rc = orc_circuit_unitary(c, ur, ui);
    if (rc == ORC_OK) {
        double* vr = calloc(N, sizeof(double));
        double* vi = calloc(N, sizeof(double));
        vr[0] = 1.0; /* zero_state, state.cpp:37-47 */
        orc_matvec(ur, ui, N, N, vr, vi, psi_re, psi_im);
        free(vr);
        free(vi);
    }
    free(ur);
    free(ui);
    return rc;
}

/* -------------------------------------------------------------- fsv path */

/* fsv_backend.cpp:40-59 (update_pairs) */
static void update_pairs(double* re, double* im, int64_t dim, const double ur[4], const double ui[4],
                         int64_t tmask, int64_t cmask) {
    for (int64_t i = 0; i < dim; ++i) {
        if ((i & tmask) != 0 || (i & cmask) != cmask) continue;
        const int64_t j = i | tmask;
        const double a0r = re[i], a0i = im[i], a1r = re[j], a1i = im[j];
        re[i] = ur[0] * a0r - ui[0] * a0i + ur[1] * a1r - ui[1] * a1i;
        im[i] = ur[0] * a0i + ui[0] * a0r + ur[1] * a1i + ui[1] * a1r;
        re[j] = ur[2] * a0r - ui[2] * a0i + ur[3] * a1r - ui[3] * a1i;
        im[j] = ur[2] * a0i + ui[2] * a0r + ur[3] * a1i + ui[3] * a1r;
    }
}

/* fsv_backend.cpp:85-131 (apply_function) */
static void apply_function(double* re, double* im, int64_t n, const qsb_function* f, int64_t first,
                           int64_t count) {
    const int64_t block = (int64_t)1 << count;
    const int64_t shift = n - first - count;
    const int64_t low = ((int64_t)1 << shift) - 1;
    const int64_t outer_count = (int64_t)1 << (n - count);
    double* in_r = malloc(sizeof(double) * block);
    double* in_i = malloc(sizeof(double) * block);
    double* out_r = malloc(sizeof(double) * block);
    double* out_i = malloc(sizeof(double) * block);
    for (int64_t outer = 0; outer < outer_count; ++outer) {
        const int64_t base = ((outer & ~low) << count) | (outer & low);
        for (int64_t j = 0; j < block; ++j) {
            in_r[j] = re[base | (j << shift)];
            in_i[j] = im[base | (j << shift)];
        }
        for (int64_t row = 0; row < block; ++row) {
            double sr = 0.0, si = 0.0;
            for (int64_t k = 0; k < block; ++k) {
                sr += f->re[row * block + k] * in_r[k] - f->im[row * block + k] * in_i[k];
                si += f->re[row * block + k] * in_i[k] + f->im[row * block + k] * in_r[k];
            }
            out_r[row] = sr;
            out_i[row] = si;
        }
        for (int64_t j = 0; j < block; ++j) {
            re[base | (j << shift)] = out_r[j];
            im[base | (j << shift)] = out_i[j];
        }
    }
    free(in_r); free(in_i); free(out_r); free(out_i);
}

/* fsv_backend.cpp:133-158 (FsvSimulator::simulate_full_state body, from any state) */
int orc_fsv_apply(const qsb_circuit* c, double* re, double* im) {
    const int64_t n = c->n_qubits;
    const int64_t dim = (int64_t)1 << n;
    int rc = orc_validate_instruction_placement(c);
    if (rc) return rc;
    for (int32_t s = 0; s < c->n_steps; ++s) {
        for (int32_t i = c->step_offsets[s]; i < c->step_offsets[s + 1]; ++i) {
            const qsb_op* op = &c->ops[i];
            double ur[4], ui[4];
            if (op->kind == QSB_OP_GATE) {
                if ((rc = orc_gate_matrix(op->gate, op->phi, ur, ui))) return rc;
                update_pairs(re, im, dim, ur, ui, (int64_t)1 << (n - 1 - op->target), 0);
            } else if (op->kind == QSB_OP_CONTROL) {
                if ((rc = orc_gate_matrix(op->gate, op->phi, ur, ui))) return rc;
                update_pairs(re, im, dim, ur, ui, (int64_t)1 << (n - 1 - op->target),
                             (int64_t)1 << (n - 1 - op->control));
            } else if (op->kind == QSB_OP_FUNCTION) {
                if (op->function < 0 || op->function >= c->n_functions)
                    return fail(ORC_ERR_LOOKUP, "registry: no function with index %d", op->function);
                const qsb_function* f = &c->functions[op->function];
                if (f->dim != ((int64_t)1 << op->count))
                    return fail(ORC_ERR_VALIDATION, "apply_function: matrix dimension mismatch");
                apply_function(re, im, n, f, op->first, op->count);
            }
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------ state.cpp */

/* state.cpp:26-31 */
uint64_t orc_splitmix64_next(uint64_t* state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* state.cpp:33-35 */
double orc_splitmix64_unit(uint64_t* state) {
    return (double)(orc_splitmix64_next(state) >> 11) * 0x1.0p-53;
}

/* state.cpp:49-56 */
double orc_norm_squared(const double* re, const double* im, int64_t dim) {
    double sum = 0.0;
    for (int64_t i = 0; i < dim; ++i) sum += re[i] * re[i] + im[i] * im[i];
    return sum;
}

/* state.cpp:58-65 */
void orc_probabilities(const double* re, const double* im, int64_t dim, double* p) {
    for (int64_t i = 0; i < dim; ++i) p[i] = re[i] * re[i] + im[i] * im[i];
}

/* state.cpp:81-98 */
uint64_t orc_collapse(const double* re, const double* im, int64_t dim, uint64_t seed) {
    uint64_t st = seed;
    const double u = orc_splitmix64_unit(&st);
    double cum = 0.0;
    uint64_t fallback = 0;
    for (int64_t i = 0; i < dim; ++i) {
        const double p = re[i] * re[i] + im[i] * im[i];
        if (p > 0.0) fallback = (uint64_t)i;
        cum += p;
        if (cum > u) return (uint64_t)i;
    }
    return fallback;
}
