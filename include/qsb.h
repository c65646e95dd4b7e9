/*
 * qsb.h — C ABI of the B200-native unitary-simulation hot path
 * (TornadoQSim "UnitarySimulatorStandard", arXiv 2305.14398, Algorithms 1+2).
 *
 * This is the drop-in boundary. The reference keeps its C++ Circuit / Step /
 * Operation model, its gate library and its Simulator plugin interface; a thin
 * adapter (integration/b200_unitary_simulator.cpp, shown in INTEGRATION.md)
 * flattens a qsim::Circuit into a qsb_circuit and calls the entry points below.
 * Plain C types only: no C++ exceptions, no torch types, no STL cross the ABI.
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/proj):
 *   qsb_simulate_full_state  -> UnitarySimulator::simulate_full_state
 *                               core/src/unitary_backend.cpp:194-215
 *   qsb_build_unitary        -> test::circuit_unitary (the accumulated U)
 *                               tests/support/test_util.hpp:135-142
 *   qsb_simulate_and_collapse-> Simulator::simulate_and_collapse + collapse
 *                               core/src/simulator.cpp:26-30, core/src/state.cpp:81-98
 *   qsb_layer_operator       -> kronecker_fold(fill_layer(layer))  (one layer of step_unitary)
 *                               core/src/unitary_backend.cpp:95-125, 141-154
 *   qsb_probabilities        -> probabilities / norm_squared
 *                               core/src/state.cpp:49-65
 *   qsb_qubit_guard          -> Simulator::qubit_guard  core/include/qsim/simulator.hpp:40
 *   qsb_status + qsb_last_error -> the qsim::Error hierarchy
 *                               core/include/qsim/errors.hpp:23-56
 *
 * Orientation: the reference accumulates U = S_K ... S_2 S_1 by left
 * multiplication (unitary_backend.cpp:211). This library computes the same
 * product by row blocks, V <- V * L for every layer operator L from the last
 * to the first; a shard of rows is computed
 * with no communication.
 */
#ifndef QSB_H_
#define QSB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QSB_ABI_VERSION 1

/* Status codes; qsb_last_error() returns the message of the last failure on
 * the calling thread. The adapter maps them back onto qsim::Error subclasses. */
typedef enum qsb_status {
    QSB_OK = 0,
    QSB_ERR_RESOURCE = 1,   /* qsim::ResourceError  (qubit guard / HBM capacity) */
    QSB_ERR_VALIDATION = 2, /* qsim::ValidationError (reset placement, registry dims) */
    QSB_ERR_SHAPE = 3,      /* qsim::ShapeError */
    QSB_ERR_ARGUMENT = 4,   /* qsim::ArgumentError */
    QSB_ERR_LOOKUP = 5,     /* qsim::LookupError */
    QSB_ERR_CUDA = 6,       /* CUDA runtime / driver failure (incl. no device) */
    QSB_ERR_NCCL = 7,       /* NCCL failure */
    QSB_ERR_INTERNAL = 8
} qsb_status;

/* Operation kinds: the alternatives of qsim::Operation (circuit.hpp:79). */
enum {
    QSB_OP_GATE = 0,        /* Gate{gate, target}                 circuit.hpp:51-55 */
    QSB_OP_CONTROL = 1,     /* ControlGate{gate, control, target} circuit.hpp:57-62 */
    QSB_OP_FUNCTION = 2,    /* FunctionOp{name, first, count}     circuit.hpp:66-71 */
    QSB_OP_INSTRUCTION = 3  /* Instruction{kind, target}          circuit.hpp:73-77 */
};

/* GateTag (circuit.hpp:31); informational for the library, which consumes u. */
enum { QSB_GATE_H = 0, QSB_GATE_X, QSB_GATE_Y, QSB_GATE_Z, QSB_GATE_S, QSB_GATE_T, QSB_GATE_R };
/* InstructionKind (circuit.hpp:49). */
enum { QSB_INSTR_MEASURE = 0, QSB_INSTR_RESET = 1 };

/* One qsim::Operation. For QSB_OP_GATE / QSB_OP_CONTROL the caller fills u_re/u_im
 * with gate_matrix(gate) (gates.cpp:40-77), row-major 2x2; the library uses
 * exactly those values, so the caller's gate library stays authoritative. */
typedef struct qsb_op {
    int32_t kind;        /* QSB_OP_* */
    int32_t gate;        /* QSB_GATE_* (gate / control gate) */
    int32_t target;      /* gate, control gate, instruction: target qubit */
    int32_t control;     /* control gate: control qubit */
    int32_t first;       /* function: first_qubit */
    int32_t count;       /* function: qubit_count */
    int32_t function;    /* function: index into qsb_circuit.functions */
    int32_t instruction; /* instruction: QSB_INSTR_* */
    double phi;          /* R(phi) angle (informational) */
    double u_re[4];
    double u_im[4];
} qsb_op;

/* A GateRegistry entry resolved for this circuit: a dim x dim row-major matrix
 * in split re/im planes (the storage of qsim::ComplexMatrix, linalg.hpp:39-70). */
typedef struct qsb_function {
    int64_t dim;
    const double* re;
    const double* im;
} qsb_function;

/* A qsim::Circuit after Circuit::append's greedy last-step packing
 * (circuit.cpp:81-103): ops of step s are ops[step_offsets[s] .. step_offsets[s+1]),
 * in insertion order. */
typedef struct qsb_circuit {
    int32_t n_qubits;
    int32_t n_steps;
    const int32_t* step_offsets; /* n_steps + 1 entries */
    const qsb_op* ops;
    int32_t n_functions;
    const qsb_function* functions;
} qsb_circuit;

/* GEMM arithmetic. 4M = four real DMMA sub-GEMMs per complex product; 3M =
 * three (Gauss), fewer FLOPs, still credited 8 N^3 in reports. */
enum { QSB_GEMM_AUTO = 0, QSB_GEMM_4M = 1, QSB_GEMM_3M = 2 };

typedef struct qsb_options {
    int32_t device;       /* CUDA device ordinal (used when n_devices == 0) */
    int32_t qubit_guard;  /* 0 = derive from HBM capacity (simulator.hpp:53-56 override otherwise) */
    int32_t gemm_mode;    /* QSB_GEMM_* */
    int32_t flags;        /* QSB_FLAG_* */
    int32_t n_devices;    /* > 1: the host-API calls shard U by row blocks over these devices */
    int32_t reserved;
    const int32_t* devices; /* n_devices ordinals (repeats allowed: virtual shards on one GPU) */
} qsb_options;

enum {
    QSB_FLAG_NO_GRAPH = 1,        /* do not capture plan execution in a CUDA graph */
    QSB_FLAG_MATERIALIZE = 2,     /* materialise each layer operator with K1 and run the
                                     GEMM on it instead of generating tiles in shared memory */
    QSB_FLAG_COLUMN_BLOCKS = 4,   /* shard U by column blocks instead of row blocks:
                                     U[:, cols] <- S_k U[:, cols] in application order, the
                                     reference's association; a plan's "rows" are then the columns
                                     [row_begin, row_begin + row_count) of U, its unitary buffer
                                     holds U[:, cols]^T and its state buffer the full-length share
                                     U[:, cols] psi0[cols] (2^n entries per plane) */
    QSB_FLAG_NO_PLAN_CACHE = 16,  /* host-API calls compile and upload every call (no reuse of the last
                                     call's plans): the cold-call cost */
    QSB_FLAG_NCCL_GATHER = 8      /* host-API calls all-gather the shards' psi rows over NCCL into a
                                     device-resident psi on every device even when the handle has a
                                     single device (a one-rank communicator; tests). With several
                                     DISTINCT devices the NCCL all-gather is always used; repeated
                                     device ids (virtual shards) cannot form a communicator and copy
                                     each shard's rows to the host instead */
};

typedef struct qsb_handle qsb_handle;
typedef struct qsb_plan qsb_plan;

/* Statistics of one plan (one circuit on one row shard). */
typedef struct qsb_plan_info {
    int32_t n_qubits;
    int32_t n_steps;
    int32_t n_layers;          /* layer operators in the circuit (sum over steps) */
    int32_t n_gemms;           /* dense complex GEMMs executed per run */
    int32_t n_identity_layers; /* instruction-only layers (exact identities, not multiplied) */
    int32_t n_launches;        /* kernels launched per run */
    int64_t row_begin;
    int64_t row_count;
    double gemm_flops;         /* 8 * row_count * N^2 per GEMM, summed */
    double expand_bytes;       /* bytes written by the K1 expansion */
    int32_t gemm_tile;         /* K2 variant: QSB_TILE_* */
    int32_t v_planes;          /* planes per V buffer (2, or 3 with the 3M sum plane) */
    int32_t gemm_splits;       /* split-K cluster size of the K2 launches (1, 2, 4, 8), or -1:
                                  stream-K (persistent CTAs share the tile x k-tile iterations) */
    int32_t n_real_gemms;      /* GEMMs whose operator is real: two real products instead of 3M's three */
    double gemm_hw_flops;      /* FP64 FLOPs the DMMAs actually execute: 6 M N^2 (3M), 4 M N^2 (real
                                  layer), 8 M N^2 (4M) per GEMM, summed; gemm_flops credits 8 M N^2 */
} qsb_plan_info;

/* K2 variants reported in qsb_plan_info.gemm_tile. */
enum { QSB_TILE_128x64 = 0, QSB_TILE_64x64 = 1, QSB_TILE_32x32 = 2, QSB_TILE_WS4M = 3, QSB_TILE_WS3M = 4,
       QSB_TILE_WS3M_SUMPLANE = 5,
       QSB_TILE_WS_CHAIN = 6 /* K2c: every GEMM of the chain in one persistent launch (3M sum-plane
                                tiles, real layers as two real products), gemm_splits = its k-splits */ };

int qsb_abi_version(void);

/* Copies the last error message of the calling thread into buf (NUL-terminated). */
size_t qsb_last_error(char* buf, size_t len);

qsb_status qsb_create(const qsb_options* options, qsb_handle** out);
qsb_status qsb_destroy(qsb_handle* handle);

/* Largest qubit count accepted (guard, or HBM-derived default). */
qsb_status qsb_qubit_guard(const qsb_handle* handle, int32_t* guard);

/* Algorithm 1: psi = U |0...0>, written to host planes of length 2^n.
 * Host in, host out; thread-safe on one handle (internally serialised). With
 * n_devices > 1 every device computes its row block of U with no
 * communication and writes its psi rows straight into the host planes. */
qsb_status qsb_simulate_full_state(qsb_handle* handle, const qsb_circuit* circuit,
                                   double* psi_re, double* psi_im);

/* Same, from an arbitrary initial state psi0 (host planes, length 2^n). */
qsb_status qsb_simulate_from_state(qsb_handle* handle, const qsb_circuit* circuit,
                                   const double* psi0_re, const double* psi0_im,
                                   double* psi_re, double* psi_im);

/* The accumulated circuit unitary U (host planes, 2^n x 2^n row-major). */
qsb_status qsb_build_unitary(qsb_handle* handle, const qsb_circuit* circuit,
                             double* u_re, double* u_im);

/* simulate_full_state + inverse-CDF collapse with SplitMix64(seed). */
qsb_status qsb_simulate_and_collapse(qsb_handle* handle, const qsb_circuit* circuit,
                                     uint64_t seed, uint64_t* basis_index);

/* collapse (state.cpp:81-98) of a host state: K4 probabilities on the GPU, then the
 * reference's sequential inverse-CDF walk with one SplitMix64(seed) draw on the host. */
qsb_status qsb_collapse(qsb_handle* handle, const double* psi_re, const double* psi_im, int64_t dim,
                        uint64_t seed, uint64_t* basis_index);

/* Number of layers step `step` factors into (first-fit, unitary_backend.cpp:63-91). */
qsb_status qsb_step_layer_count(const qsb_circuit* circuit, int32_t step, int32_t* layers);

/* K1: the dense operator of layer `layer` of step `step`, expanded on the GPU
 * (host planes, 2^n x 2^n). Bit-exact with the reference's kronecker_fold. */
qsb_status qsb_layer_operator(qsb_handle* handle, const qsb_circuit* circuit, int32_t step,
                              int32_t layer, double* re, double* im);

/* K4: p_i = re_i^2 + im_i^2 and sum p_i of a host state, computed on the GPU. */
qsb_status qsb_probabilities(qsb_handle* handle, const double* psi_re, const double* psi_im,
                             int64_t dim, double* p, double* norm_squared);

/* is_unitary (linalg.cpp:131-155) as GateRegistry::register_function runs it
 * on every registered matrix (gates.cpp:112-125, tol = kRegistryUnitaryTol):
 * result = 1 iff every |(A^H A - I)_ij| <= tol. A^H A is formed on the FP64
 * tensor cores (dim >= 64) — the O(dim^3) check behind DJ circuit construction.
 * Host planes, dim x dim row-major. max_deviation (optional) receives the max. */
qsb_status qsb_is_unitary(qsb_handle* handle, const double* re, const double* im, int64_t dim, double tol,
                          int32_t* result, double* max_deviation);

/* ---- device-resident plans (bench, multi-GPU row shards) ---- */

/* Compile `circuit` for rows [row_begin, row_begin + row_count) of U and upload
 * every descriptor; buffers are allocated on the handle's device. */
qsb_status qsb_plan_create(qsb_handle* handle, const qsb_circuit* circuit, int64_t row_begin,
                           int64_t row_count, qsb_plan** out);
qsb_status qsb_plan_destroy(qsb_plan* plan);
qsb_status qsb_plan_get_info(const qsb_plan* plan, qsb_plan_info* info);

/* Run the whole chain on `stream` (a cudaStream_t; NULL = the handle's stream):
 * V = rows of U, then psi_rows = V * psi0 (psi0 = |0...0> unless set). Async.
 * Plans on ONE device must not execute concurrently on different streams: a
 * stream-K GEMM is a persistent grid sized to the SM count whose tile owners
 * wait on other CTAs of the same grid, so two of them sharing the SMs can both
 * be partly resident and wait forever (the host-API calls use one stream per
 * physical device for this reason). */
qsb_status qsb_plan_execute(qsb_plan* plan, void* stream);

/* Record CUDA events around the K1 / K2 / K3 phases of every execute (disables
 * the plan's CUDA graph); read them back with qsb_plan_last_timing. enable = 2
 * also brackets every K2 launch with its own event pair (qsb_plan_gemm_times);
 * those events sit between chained launches and serialise them, so mode 2 is
 * for a per-kind breakdown, not for timing the chain. */
qsb_status qsb_plan_set_timing(qsb_plan* plan, int32_t enable);

/* Per-K2-launch durations (ms) of the last mode-2 execute, in chain order, and
 * each launch's kind: bit 0 = real layer (two real products), bit 1 = operand
 * materialised by K1t, bit 2 = 4M arithmetic (else 3M). Fills min(cap, count)
 * entries; *count = GEMMs per execute. ms / kinds may be NULL. */
qsb_status qsb_plan_gemm_times(qsb_plan* plan, double* ms, int32_t* kinds, int32_t cap, int32_t* count);

/* Replace psi0 (default |0...0>) with re/im planes of length 2^n (host or device
 * pointers), async on `stream`. */
qsb_status qsb_plan_set_initial_state(qsb_plan* plan, const double* re, const double* im, void* stream);

/* Device pointers of the plan's results (valid until the next execute/destroy):
 * U rows (row_count x 2^n, leading dimension 2^n) and psi rows (row_count).
 * A plan split into row-block parts (QSB_PARTS) keeps its U rows per part: this
 * call then synchronises the device and assembles them into one block first
 * (call it after the execute, not concurrently with one). */
qsb_status qsb_plan_unitary_device(const qsb_plan* plan, const double** re, const double** im);
qsb_status qsb_plan_state_device(const qsb_plan* plan, const double** re, const double** im);

/* Copy psi rows into caller device buffers (e.g. a slice of an all-gather buffer), async. */
qsb_status qsb_plan_copy_state(const qsb_plan* plan, double* dst_re, double* dst_im, void* stream);

/* ---- NCCL: the all-gather of psi rows (north star "only the final state
 * vector is all-gathered with NCCL over NVLink") ----
 *
 * One process per GPU: rank 0 calls qsb_nccl_unique_id, the caller broadcasts the
 * QSB_NCCL_ID_BYTES bytes (MPI, torch.distributed, a file ...), every rank calls
 * qsb_comm_create on its handle (ncclCommInitRank on the handle's device). The
 * in-process multi-device handle (qsb_options.n_devices > 1) builds its own
 * communicator with ncclCommInitAll and needs none of this. */
#define QSB_NCCL_ID_BYTES 128
typedef struct qsb_comm qsb_comm;

qsb_status qsb_nccl_unique_id(void* id_out);
qsb_status qsb_comm_create(qsb_handle* handle, const void* id, int32_t n_ranks, int32_t rank, qsb_comm** out);
qsb_status qsb_comm_destroy(qsb_comm* comm);
/* NCCL version (e.g. 22809) of the library in use; loads libnccl. */
qsb_status qsb_nccl_version(int32_t* version);

/* qsb_simulate_full_state for one process per GPU (a rank of `comm`): this rank
 * computes rows [rank 2^n / n_ranks, +2^n / n_ranks) of U with no communication,
 * the ranks' psi rows are all-gathered over NCCL, and every rank receives the whole
 * psi in its host planes (length 2^n). Same plan cache as the single-process call. */
qsb_status qsb_simulate_full_state_sharded(qsb_handle* handle, qsb_comm* comm, const qsb_circuit* circuit,
                                           double* psi_re, double* psi_im);

/* All-gather the psi rows of every rank's plan into full-length device planes
 * (2^n doubles each) on every rank, async on `stream`. Rank r's plan must own
 * rows [r * 2^n / n_ranks, (r + 1) * 2^n / n_ranks) (row blocks, not column blocks). */
qsb_status qsb_plan_allgather_state(const qsb_plan* plan, qsb_comm* comm, double* psi_re, double* psi_im,
                                    void* stream);

/* The optional second exchange of SURVEY 8(e): all-gather every rank's rows of U into
 * full 2^n x 2^n device planes on every rank (16 N^2 / G bytes sent per rank), async. */
qsb_status qsb_plan_allgather_unitary(const qsb_plan* plan, qsb_comm* comm, double* u_re, double* u_im,
                                      void* stream);

/* Kernel timing of the last execute, from CUDA events on the launching stream:
 * total, the K2 GEMM chain, and the mean single-GEMM duration (ms). Synchronises. */
qsb_status qsb_plan_last_timing(qsb_plan* plan, double* total_ms, double* gemm_ms,
                                double* gemm_mean_ms);

/* ---- state-vector engine: the fsv backend and the structured unitary ----
 *
 * One engine evolves a [2][2^n][W] split-plane array by the reference's
 * full-state-vector operations (fsv_backend.cpp:40-158) in circuit order:
 * W = 1 is FsvSimulator (one state), W = 2^n columns is the structured unitary
 * U[:, c] = fsv(e_c) — the same U as the dense path, built with HBM-bound pair
 * updates instead of dense GEMMs (a different algorithm, reported separately
 * and never counted against the FP64 tensor roofline). Results are bit-exact
 * with the reference's fsv backend (up to the sign of zeros). */
enum { QSB_SV_STATE = 0, QSB_SV_UNITARY = 1 };

typedef struct qsb_sv_plan qsb_sv_plan;

typedef struct qsb_sv_plan_info {
    int32_t n_qubits;
    int32_t mode;              /* QSB_SV_* */
    int32_t n_ops;             /* operations applied (instructions excluded) */
    int32_t n_passes;          /* launches over the whole array (batches + large functions) */
    int32_t n_function_passes; /* apply_function blocks too large for a shared-memory slab */
    int32_t n_launches;        /* kernels per execute, including initialisation */
    int32_t slab_bits;         /* log2 elements staged per CTA */
    int32_t max_batch_targets; /* most target bits in one batch */
    int64_t col_begin;         /* QSB_SV_UNITARY: first column of U computed */
    int64_t col_count;         /* QSB_SV_UNITARY: columns (power of two); QSB_SV_STATE: 1 */
    double bytes_per_run;      /* HBM bytes read + written by the passes of one execute */
} qsb_sv_plan_info;

/* FsvSimulator::qubit_guard (fsv_backend.hpp:47-51): options.qubit_guard, else HBM-derived. */
qsb_status qsb_fsv_qubit_guard(const qsb_handle* handle, int32_t* guard);

/* FsvSimulator::simulate_full_state (fsv_backend.cpp:135-158): psi = ops |0...0>. */
qsb_status qsb_fsv_simulate_full_state(qsb_handle* handle, const qsb_circuit* circuit,
                                       double* psi_re, double* psi_im);

/* Same from an arbitrary state psi0 (host planes, length 2^n); the in-place
 * apply_gate / apply_control_gate / apply_function sequence of fsv_backend.cpp:59-132. */
qsb_status qsb_fsv_simulate_from_state(qsb_handle* handle, const qsb_circuit* circuit,
                                       const double* psi0_re, const double* psi0_im,
                                       double* psi_re, double* psi_im);

qsb_status qsb_structured_qubit_guard(const qsb_handle* handle, int32_t* guard);

/* U with U[:, c] = fsv(e_c) (host planes, 2^n x 2^n row-major). With
 * n_devices > 1 the columns are sharded over the devices, no communication. */
qsb_status qsb_structured_build_unitary(qsb_handle* handle, const qsb_circuit* circuit,
                                        double* u_re, double* u_im);

/* psi = U e_0 of the structured U (Algorithm 1's final matvec is a column read). */
qsb_status qsb_structured_simulate_full_state(qsb_handle* handle, const qsb_circuit* circuit,
                                              double* psi_re, double* psi_im);

/* Device-resident plans (bench, multi-GPU column shards). QSB_SV_UNITARY computes
 * columns [col_begin, col_begin + col_count) of U (col_count a power of two
 * dividing 2^n, col_begin a multiple of it); QSB_SV_STATE ignores them. */
qsb_status qsb_sv_plan_create(qsb_handle* handle, const qsb_circuit* circuit, int32_t mode,
                              int64_t col_begin, int64_t col_count, qsb_sv_plan** out);
qsb_status qsb_sv_plan_destroy(qsb_sv_plan* plan);
qsb_status qsb_sv_plan_get_info(const qsb_sv_plan* plan, qsb_sv_plan_info* info);
/* QSB_SV_STATE: initial state (host or device planes of length 2^n; default |0...0>), async. */
qsb_status qsb_sv_plan_set_state(qsb_sv_plan* plan, const double* re, const double* im, void* stream);
/* Initialise (psi0 or identity columns) and apply every pass on `stream` (NULL = handle stream). Async. */
qsb_status qsb_sv_plan_execute(qsb_sv_plan* plan, void* stream);
/* Device planes of the result, [2^n][col_count] row-major (valid until the next execute/destroy). */
qsb_status qsb_sv_plan_result_device(const qsb_sv_plan* plan, const double** re, const double** im);

/* Reference memory accounting (unitary_backend.cpp:156-179), BackendKind 0 = Unitary, 1 = Fsv:
 * memory_estimate (8 bytes per complex) and engine_memory_estimate (the reference
 * engine's 3 N^2 + N complex doubles); 0 outside the reference's qubit ranges. */
uint64_t qsb_memory_estimate(int32_t n_qubits, int32_t kind);
uint64_t qsb_engine_memory_estimate(int32_t n_qubits, int32_t kind);
/* This library's device footprint for a one-device dense run: two 2^n x 2^n complex
 * V buffers + psi0 + psi (the HBM-derived guard budgets it at 92 % of device memory). */
uint64_t qsb_hbm_footprint(int32_t n_qubits);

#ifdef __cplusplus
}
#endif

#endif /* QSB_H_ */
