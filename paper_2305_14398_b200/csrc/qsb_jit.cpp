// qsb_jit.cpp — NVRTC compilation + driver-API module cache (qsb_jit.hpp).
#include "qsb_jit.hpp"

#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "qsb_host.hpp"

namespace qsbjit {

namespace {

// The subset of nvrtc.h used here (resolved with dlsym).
using nvrtcProgram = void*;
using CreateFn = int (*)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*);
using CompileFn = int (*)(nvrtcProgram, int, const char* const*);
using SizeFn = int (*)(nvrtcProgram, size_t*);
using GetFn = int (*)(nvrtcProgram, char*);
using DestroyFn = int (*)(nvrtcProgram*);

struct Nvrtc {
    bool ok = false;
    CreateFn create = nullptr;
    CompileFn compile = nullptr;
    SizeFn log_size = nullptr;
    GetFn log = nullptr;
    SizeFn cubin_size = nullptr;
    GetFn cubin = nullptr;
    DestroyFn destroy = nullptr;
};

const Nvrtc& nvrtc() {
    static Nvrtc n = [] {
        Nvrtc r;
        void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnvrtc.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) return r;
        r.create = reinterpret_cast<CreateFn>(dlsym(h, "nvrtcCreateProgram"));
        r.compile = reinterpret_cast<CompileFn>(dlsym(h, "nvrtcCompileProgram"));
        r.log_size = reinterpret_cast<SizeFn>(dlsym(h, "nvrtcGetProgramLogSize"));
        r.log = reinterpret_cast<GetFn>(dlsym(h, "nvrtcGetProgramLog"));
        r.cubin_size = reinterpret_cast<SizeFn>(dlsym(h, "nvrtcGetCUBINSize"));
        r.cubin = reinterpret_cast<GetFn>(dlsym(h, "nvrtcGetCUBIN"));
        r.destroy = reinterpret_cast<DestroyFn>(dlsym(h, "nvrtcDestroyProgram"));
        r.ok = r.create && r.compile && r.log_size && r.log && r.cubin_size && r.cubin && r.destroy;
        return r;
    }();
    return n;
}

template <typename F>
F driver(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return nullptr;
    return reinterpret_cast<F>(p);
}

using ModuleLoadFn = CUresult (*)(CUmodule*, const void*);
using GetFunctionFn = CUresult (*)(CUfunction*, CUmodule, const char*);
using LaunchFn = CUresult (*)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                              CUstream, void**, void**);

std::mutex g_mu;
// (device, source) -> module; kernels looked up per name.
std::map<std::pair<int, std::string>, CUmodule> g_modules;

}  // namespace

bool available() {
    const char* e = std::getenv("QSB_SV_JIT");
    if (e && std::strcmp(e, "0") == 0) return false;
    return nvrtc().ok && driver<ModuleLoadFn>("cuModuleLoadData") && driver<LaunchFn>("cuLaunchKernel");
}

bool forced() {
    const char* e = std::getenv("QSB_SV_JIT");
    return e && std::strcmp(e, "1") == 0 && available();
}

std::vector<void*> kernels(const std::string& source, const std::vector<std::string>& names) {
    using qsbh::raise;
    int dev = 0;
    qsbh::cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    // make sure the runtime's primary context is current for the driver calls
    qsbh::cuda_check(cudaFree(nullptr), "cudaFree(0)");
    std::lock_guard<std::mutex> lk(g_mu);
    CUmodule mod = nullptr;
    auto key = std::make_pair(dev, source);
    auto it = g_modules.find(key);
    if (it != g_modules.end()) {
        mod = it->second;
    } else {
        const Nvrtc& n = nvrtc();
        if (!n.ok) raise(QSB_ERR_INTERNAL, "NVRTC is not available");
        nvrtcProgram prog = nullptr;
        if (n.create(&prog, source.c_str(), "qsb_sv_jit.cu", 0, nullptr, nullptr) != 0)
            raise(QSB_ERR_INTERNAL, "nvrtcCreateProgram failed");
        const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "--fmad=false", "-default-device",
                              "--extra-device-vectorization"};
        const int rc = n.compile(prog, 5, opts);
        if (rc != 0) {
            size_t ls = 0;
            n.log_size(prog, &ls);
            std::string log(ls, '\0');
            if (ls) n.log(prog, &log[0]);
            n.destroy(&prog);
            const size_t from = log.size() > 700 ? log.size() - 700 : 0;  // the errors come last
            raise(QSB_ERR_INTERNAL, "NVRTC compile failed: ...%s", log.c_str() + from);
        }
        size_t cs = 0;
        n.cubin_size(prog, &cs);
        std::vector<char> cubin(cs);
        n.cubin(prog, cubin.data());
        n.destroy(&prog);
        auto load = driver<ModuleLoadFn>("cuModuleLoadData");
        if (!load || load(&mod, cubin.data()) != CUDA_SUCCESS) raise(QSB_ERR_CUDA, "cuModuleLoadData failed");
        g_modules.emplace(key, mod);
    }
    auto getf = driver<GetFunctionFn>("cuModuleGetFunction");
    if (!getf) raise(QSB_ERR_CUDA, "cuModuleGetFunction unavailable");
    std::vector<void*> out;
    for (const std::string& name : names) {
        CUfunction f = nullptr;
        if (getf(&f, mod, name.c_str()) != CUDA_SUCCESS) raise(QSB_ERR_CUDA, "kernel %s not in module", name.c_str());
        out.push_back(reinterpret_cast<void*>(f));
    }
    return out;
}

int launch(void* fn, unsigned grid, unsigned block, void* stream, void** args, int smem) {
    static LaunchFn l = driver<LaunchFn>("cuLaunchKernel");
    using SetAttrFn = CUresult (*)(CUfunction, CUfunction_attribute, int);
    static SetAttrFn set_attr = driver<SetAttrFn>("cuFuncSetAttribute");
    if (!l) return static_cast<int>(cudaErrorNotSupported);
    if (smem > 48 * 1024) {
        if (!set_attr ||
            set_attr(reinterpret_cast<CUfunction>(fn), CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem) !=
                CUDA_SUCCESS)
            return static_cast<int>(cudaErrorLaunchFailure);
    }
    const CUresult r = l(reinterpret_cast<CUfunction>(fn), grid, 1, 1, block, 1, 1, static_cast<unsigned>(smem),
                         reinterpret_cast<CUstream>(stream), args, nullptr);
    return r == CUDA_SUCCESS ? 0 : static_cast<int>(cudaErrorLaunchFailure);
}

}  // namespace qsbjit
