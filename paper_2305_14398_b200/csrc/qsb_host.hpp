// qsb_host.hpp — host-side plumbing shared by the runtimes behind the C ABI
// (qsb_runtime.cpp: the dense unitary path; qsb_sv.cpp: the state-vector
// engine behind the fsv and structured-unitary backends): error transport
// across the ABI, device scoping, device buffers, the handle, and the circuit
// checks the reference performs on every operation.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/qsb.h"

namespace qsbh {

// Message of the last failure on the calling thread (qsb_last_error).
inline thread_local std::string g_error;

struct Failure {
    qsb_status code;
    std::string msg;
};

[[noreturn]] inline void raise(qsb_status code, const char* fmt, ...) {
    char buf[768];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw Failure{code, buf};
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) raise(QSB_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}
inline void cuda_check(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }

// Runs f, converting every C++ exception into a status code + message: no
// exception crosses the ABI.
template <typename F>
qsb_status guarded(F&& f) {
    try {
        f();
        return QSB_OK;
    } catch (const Failure& e) {
        g_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_error = "host allocation failed";
        return QSB_ERR_RESOURCE;
    } catch (const std::exception& e) {
        g_error = e.what();
        return QSB_ERR_INTERNAL;
    }
}

// Restores the caller's current device on scope exit.
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceScope() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void ensure(size_t bytes) {
        if (bytes <= cap) return;
        release();
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            raise(QSB_ERR_RESOURCE, "device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
        }
        cap = bytes;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), cap(o.cap) { o.p = nullptr; o.cap = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; cap = o.cap; o.p = nullptr; o.cap = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
};

struct Buffers {
    DevBuf v[2];     // dense path: [planes][M][N] doubles each (V and V'); sv engine: state ping-pong
    DevBuf psi;      // [2][M]
    DevBuf x;        // [2][N] initial state
    DevBuf layers;   // LayerDesc[] for the one-CTA path; SvLocalOp[] for the sv engine
    DevBuf tables;   // registered function matrices
    DevBuf p;        // probabilities
    DevBuf partial;  // reduction partials + norm
    DevBuf lmat;     // dense path: a materialised (transposed) layer operator for K2's TMA B operand
    DevBuf skws;     // dense path: stream-K partial accumulators
    DevBuf skflags;  // dense path: stream-K per-tile arrival counters
};

}  // namespace qsbh

// One CUDA device (or one virtual shard on it) driven by a handle.
struct DeviceCtx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool owns_stream = true;  // virtual shards on one device share that device's first stream
    double total_mem = 0.0;   // bytes of device memory (cudaGetDeviceProperties)
    // Free device memory, queried only for allocations that are a visible share of the
    // device (cudaMemGetInfo is a driver round trip on every plan of a cold host call).
    bool fits(double bytes, double fraction) const {
        if (bytes < 0.25 * total_mem) return true;
        size_t free_b = 0, total_b = 0;
        qsbh::cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
        return bytes <= fraction * static_cast<double>(free_b);
    }
    qsbh::Buffers cache;
    void* nccl_comm = nullptr;  // ncclComm_t of this device in the handle's communicator (distinct devices)
    qsbh::DevBuf gathered;      // [2][N] psi all-gathered over NCCL  // reused by the host-API calls
    // Pinned host staging for uploads on `stream` (descriptor arrays): reused by
    // the next call only after that call's stream synchronisation.
    struct Pinned {
        void* p = nullptr;
        size_t cap = 0;
        void* get(size_t bytes) {
            if (bytes > cap) {
                if (p) cudaFreeHost(p);
                p = nullptr;
                cap = 0;
                qsbh::cuda_check(cudaMallocHost(&p, bytes), "cudaMallocHost");
                cap = bytes;
            }
            return p;
        }
        ~Pinned() {
            if (p) cudaFreeHost(p);
        }
    };
    Pinned pinned_in, pinned_out;  // uploads / downloads of small results
    void* stage(size_t bytes) { return pinned_in.get(bytes); }
    void* stage_out(size_t bytes) { return pinned_out.get(bytes); }
};

struct qsb_handle {
    int guard = 0;             // unitary backends (dense and structured share the 2^n x 2^n budget)
    int fsv_guard = 0;         // state-vector backend
    int structured_guard = 0;  // structured unitary (one 2^n x 2^n buffer instead of two)
    int gemm_mode = QSB_GEMM_AUTO;
    int flags = 0;
    std::vector<std::unique_ptr<DeviceCtx>> devs;
    int nccl_ranks = 0;  // devices in the current NCCL communicator (devs[0 .. nccl_ranks)), 0 = none
    // Host-API plan cache (qsb_runtime.cpp run_full): the last call's plans, one per
    // row block, keyed by the circuit's structure; registry matrix contents are kept
    // and compared on reuse. Any path that needs the devices' memory drops it first.
    std::vector<qsb_plan*> cached;
    std::vector<char> cache_key;
    std::vector<std::vector<double>> cached_fn;  // [2 * function + plane] contents, used functions only
    void (*drop_cache)(qsb_handle*) = nullptr;
    void drop_plan_cache() {
        if (drop_cache) drop_cache(this);
    }
    std::mutex mu;
    DeviceCtx& dev0() { return *devs.front(); }
};

namespace qsbh {

inline void validate_circuit_shape(const qsb_circuit* c) {
    if (!c) raise(QSB_ERR_ARGUMENT, "circuit is null");
    if (c->n_qubits < 1 || c->n_qubits > 30)
        raise(QSB_ERR_ARGUMENT, "circuit qubit count must be in [1, 30], got %d", c->n_qubits);
    if (c->n_steps < 0) raise(QSB_ERR_ARGUMENT, "negative step count");
    if (c->n_steps > 0 && (!c->step_offsets || !c->ops)) raise(QSB_ERR_ARGUMENT, "circuit arrays are null");
}

// validate_instruction_placement (backend_util.cpp:21-32): reset only in the final step.
inline void check_reset_placement(const qsb_circuit* c) {
    for (int s = 0; s + 1 < c->n_steps; ++s)
        for (int i = c->step_offsets[s]; i < c->step_offsets[s + 1]; ++i)
            if (c->ops[i].kind == QSB_OP_INSTRUCTION && c->ops[i].instruction == QSB_INSTR_RESET)
                raise(QSB_ERR_VALIDATION, "reset is only supported in the final step");
}

// Per-operation checks (qubit ranges: fsv_backend.cpp:25-31, 74-79, 86-97;
// registry dimension: unitary_backend.cpp:50-53).
inline void check_op(const qsb_circuit* c, const qsb_op& op) {
    const int n = c->n_qubits;
    auto q = [&](int v) {
        if (v < 0 || v >= n) raise(QSB_ERR_ARGUMENT, "qubit index %d out of range for a %d-qubit circuit", v, n);
    };
    switch (op.kind) {
    case QSB_OP_GATE: q(op.target); break;
    case QSB_OP_CONTROL:
        q(op.control);
        q(op.target);
        if (op.control == op.target) raise(QSB_ERR_ARGUMENT, "control gate: control and target must differ");
        break;
    case QSB_OP_FUNCTION: {
        if (op.count < 1) raise(QSB_ERR_ARGUMENT, "function must span at least one qubit");
        q(op.first);
        if (op.first + op.count > n) raise(QSB_ERR_ARGUMENT, "function range exceeds circuit size");
        if (op.function < 0 || op.function >= c->n_functions || !c->functions)
            raise(QSB_ERR_LOOKUP, "registry: no function with index %d", op.function);
        const qsb_function& f = c->functions[op.function];
        if (f.dim != (int64_t{1} << op.count))  // unitary_backend.cpp:50-53
            raise(QSB_ERR_VALIDATION, "function %d no longer matches its registered dimension", op.function);
        if (!f.re || !f.im) raise(QSB_ERR_ARGUMENT, "function %d has null data", op.function);
        break;
    }
    case QSB_OP_INSTRUCTION: q(op.target); break;
    default: raise(QSB_ERR_ARGUMENT, "unknown operation kind %d", op.kind);
    }
}

// format_bytes (unitary_backend.cpp:181-192): decimal units, two decimals above bytes.
inline void format_bytes(uint64_t bytes, char* buf, size_t len) {
    static const char* units[] = {"B", "kB", "MB", "GB", "TB", "PB"};
    double v = static_cast<double>(bytes);
    int u = 0;
    while (v >= 1000.0 && u + 1 < 6) { v /= 1000.0; ++u; }
    std::snprintf(buf, len, u == 0 ? "%.0f %s" : "%.2f %s", v, units[u]);
}

}  // namespace qsbh
