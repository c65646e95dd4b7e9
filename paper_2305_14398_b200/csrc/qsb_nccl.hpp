// qsb_nccl.hpp — NCCL for the one exchange of the row-sharded path (SURVEY.md
// 8(e)): the all-gather of every shard's psi rows over NVLink / NVSwitch.
//
// libnccl is opened at first use, so libqsb.so keeps no link-time dependency and a
// missing NCCL surfaces as QSB_ERR_NCCL on the calls that need it — never as a
// silent fallback. Which copy: $QSB_NCCL_LIB when set (the Python binding points it
// at the NCCL torch ships, so a torch imported later finds a compatible
// libnccl.so.2 already loaded), else a libnccl.so.2 already in the process, else
// the system's.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <string>
#include <type_traits>

#include "qsb_host.hpp"

namespace qsbh {

struct NcclApi {
    bool ok = false;
    std::string why;
    int version = 0;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*get_version)(int*) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

inline const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* lib = nullptr;
        if (const char* path = std::getenv("QSB_NCCL_LIB"))
            if (*path) lib = dlopen(path, RTLD_NOW | RTLD_LOCAL);
        if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL | RTLD_NOLOAD);
        for (const char* name : {"libnccl.so.2", "libnccl.so", "/usr/lib/x86_64-linux-gnu/libnccl.so.2"})
            if (!lib && (lib = dlopen(name, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
        if (!lib) {
            const char* e = dlerror();
            a.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "unknown error");
            return a;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(lib, name));
            if (!fn && a.why.empty()) a.why = std::string("libnccl lacks ") + name;
        };
        sym(a.get_unique_id, "ncclGetUniqueId");
        sym(a.comm_init_rank, "ncclCommInitRank");
        sym(a.comm_init_all, "ncclCommInitAll");
        sym(a.comm_destroy, "ncclCommDestroy");
        sym(a.all_gather, "ncclAllGather");
        sym(a.group_start, "ncclGroupStart");
        sym(a.group_end, "ncclGroupEnd");
        sym(a.get_version, "ncclGetVersion");
        sym(a.error_string, "ncclGetErrorString");
        a.ok = a.why.empty();
        if (a.ok) a.get_version(&a.version);
        return a;
    }();
    return api;
}

inline const NcclApi& nccl_or_raise() {
    const NcclApi& a = nccl();
    if (!a.ok) raise(QSB_ERR_NCCL, "%s", a.why.c_str());
    return a;
}

inline void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) raise(QSB_ERR_NCCL, "%s: %s", what, nccl().error_string ? nccl().error_string(r) : "?");
}

}  // namespace qsbh
