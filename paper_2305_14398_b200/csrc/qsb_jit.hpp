// qsb_jit.hpp — run-time compilation of straight-line sm_100a kernels (NVRTC)
// for the state-vector engine's register batches.
//
// A register batch is a fixed sequence of pair updates on 2^K register-resident
// elements. Interpreting it (qsb_sv.cu: sv_reg_kernel) costs a dispatch branch
// per operation and register moves at every merge point — ncu shows ~70 % of
// its instructions are moves. Compiled straight-line, targets / controls /
// classes are constants, X and CNOT inside the batch become free renaming, and
// the 2x2 coefficients are read from the kernel's parameter space as
// constant-bank operands. The generated source depends only on the circuit's
// structure (not on angles), so it is cached per process and reused across
// calls and plans.
//
// NVRTC and the driver API are resolved at run time (dlopen /
// cudaGetDriverEntryPoint): without them the engine keeps the interpreted
// kernel (bit-identical results).
#pragma once

#include <string>
#include <vector>

namespace qsbjit {

// NVRTC present and QSB_SV_JIT != "0".
bool available();

// QSB_SV_JIT == "1": compile every register batch, whatever the array size
// (by default only arrays of >= 2^18 elements, where compilation pays off).
bool forced();

// CUfunction handles (as void*) for `names` in `source`, compiled for the
// current device (sm_100a) or taken from the process-wide cache.
std::vector<void*> kernels(const std::string& source, const std::vector<std::string>& names);

// cuLaunchKernel(fn, grid x 1 x 1, block x 1 x 1, smem bytes of dynamic shared memory).
int launch(void* fn, unsigned grid, unsigned block, void* stream, void** args, int smem = 0);

}  // namespace qsbjit
