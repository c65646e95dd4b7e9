/*
 * qsim_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's CPU unitary-simulation path
 * (/root/reference/proj, C++20 "qsim"), used as the parity checker for the
 * B200 kernels. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it; the product path never does.
 *
 * Parity is pinned: tests/test_oracle_golden.py checks every function here
 * against golden vectors produced by the reference library itself
 * (oracle/_ref, compiled from the reference sources by oracle/Makefile;
 * tests/golden/make_golden.py).
 *
 * Circuits use the same flat format as the product ABI (include/qsb.h), but
 * the oracle recomputes every gate matrix from (gate, phi) and ignores u_re/u_im.
 */
#ifndef QSIM_ORACLE_H_
#define QSIM_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "../include/qsb.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes mirror qsb_status / the qsim::Error hierarchy. */
enum { ORC_OK = 0, ORC_ERR_RESOURCE = 1, ORC_ERR_VALIDATION = 2, ORC_ERR_SHAPE = 3,
       ORC_ERR_ARGUMENT = 4, ORC_ERR_LOOKUP = 5, ORC_ERR_NOMEM = 9 };

const char* orc_last_error(void);

/* Worker threads for orc_matmul (row-chunk split, bit-identical to serial:
 * parallel.cpp:58-90). 0 or 1 = serial. */
void orc_set_threads(int threads);

/* gates.cpp:27-77 */
int orc_gate_matrix(int32_t gate, double phi, double re[4], double im[4]);
/* gates.cpp:79-110; out planes of (2^span)^2 */
int orc_controlled_unitary(const double u_re[4], const double u_im[4], int64_t control_pos,
                           int64_t target_pos, int64_t span, double* re, double* im);
/* linalg.cpp:109-129; c is (ar*br) x (ac*bc) */
int orc_kronecker(const double* a_re, const double* a_im, int64_t ar, int64_t ac,
                  const double* b_re, const double* b_im, int64_t br, int64_t bc,
                  double* c_re, double* c_im);
/* linalg.cpp:46-87; c = a * b, a is m x k, b is k x n */
int orc_matmul(const double* a_re, const double* a_im, const double* b_re, const double* b_im,
               int64_t m, int64_t k, int64_t n, double* c_re, double* c_im);
/* linalg.cpp:89-107 */
int orc_matvec(const double* a_re, const double* a_im, int64_t m, int64_t k, const double* v_re,
               const double* v_im, double* out_re, double* out_im);

/* unitary_backend.cpp:63-91: number of layers of one step, and for each op of
 * the step the layer it lands in (layer_of_op has step-op-count entries). */
int orc_step_layers(const qsb_circuit* c, int32_t step, int32_t* n_layers, int32_t* layer_of_op);
/* kronecker_fold(fill_layer(layer)) of one layer, unitary_backend.cpp:95-125 (N x N) */
int orc_layer_operator(const qsb_circuit* c, int32_t step, int32_t layer, double* re, double* im);
/* unitary_backend.cpp:141-154 (N x N) */
int orc_step_unitary(const qsb_circuit* c, int32_t step, double* re, double* im);
/* tests/support/test_util.hpp:135-142 (N x N) */
int orc_circuit_unitary(const qsb_circuit* c, double* re, double* im);
/* backend_util.cpp:21-32 */
int orc_validate_instruction_placement(const qsb_circuit* c);
/* unitary_backend.cpp:194-215 with an explicit guard (0 = kUnitaryQubitGuard = 14) */
int orc_unitary_simulate(const qsb_circuit* c, int32_t guard, double* psi_re, double* psi_im);
/* fsv_backend.cpp:40-158: apply every op of the circuit to a state in place */
int orc_fsv_apply(const qsb_circuit* c, double* psi_re, double* psi_im);

/* state.cpp:26-35 */
uint64_t orc_splitmix64_next(uint64_t* state);
double orc_splitmix64_unit(uint64_t* state);
/* state.cpp:49-65 */
double orc_norm_squared(const double* re, const double* im, int64_t dim);
void orc_probabilities(const double* re, const double* im, int64_t dim, double* p);
/* state.cpp:81-98 */
uint64_t orc_collapse(const double* re, const double* im, int64_t dim, uint64_t seed);

/* unitary_backend.cpp:156-192 */
uint64_t orc_memory_estimate(int32_t n_qubits, int32_t kind);
uint64_t orc_engine_memory_estimate(int32_t n_qubits, int32_t kind);
void orc_format_bytes(uint64_t bytes, char* buf, size_t len);

/* linalg.cpp:131-155, linalg.cpp:157-169 */
int orc_is_unitary(const double* re, const double* im, int64_t n, double tol);
double orc_max_entry_diff(const double* a_re, const double* a_im, const double* b_re,
                          const double* b_im, int64_t count);

#ifdef __cplusplus
}
#endif

#endif
