// nccl_api.h -- NCCL entry points resolved at run time with dlopen/dlsym.
//
// libtgv.so has no load-time dependency on libnccl: a process that already
// loaded NCCL (e.g. torch's bundled libnccl.so.2) shares that copy, otherwise
// the system libnccl.so.2 is opened on first multi-rank use.  Single-GPU use
// never touches NCCL.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <mutex>

struct NcclApi {
    decltype(&::ncclGetUniqueId) GetUniqueId;
    decltype(&::ncclCommInitRank) CommInitRank;
    decltype(&::ncclCommDestroy) CommDestroy;
    decltype(&::ncclCommAbort) CommAbort;
    decltype(&::ncclCommGetAsyncError) CommGetAsyncError;
    decltype(&::ncclGetErrorString) GetErrorString;
    decltype(&::ncclGroupStart) GroupStart;
    decltype(&::ncclGroupEnd) GroupEnd;
    decltype(&::ncclSend) Send;
    decltype(&::ncclRecv) Recv;
    decltype(&::ncclAllReduce) AllReduce;
    decltype(&::ncclAllGather) AllGather;
};

// Returns nullptr (and fills err) if libnccl.so.2 or a symbol is missing.
inline const NcclApi* nccl_api(char* err, size_t errlen)
{
    static NcclApi api;
    static bool ok = false;
    static char msg[256] = "";
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            snprintf(msg, sizeof msg, "dlopen(libnccl.so.2) failed: %s", dlerror());
            return;
        }
#define TGV_SYM(name)                                                                   \
    api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, "nccl" #name));           \
    if (!api.name) {                                                                    \
        snprintf(msg, sizeof msg, "libnccl.so.2 lacks nccl" #name);                     \
        return;                                                                         \
    }
        TGV_SYM(GetUniqueId) TGV_SYM(CommInitRank) TGV_SYM(CommDestroy) TGV_SYM(CommAbort)
        TGV_SYM(CommGetAsyncError) TGV_SYM(GetErrorString) TGV_SYM(GroupStart) TGV_SYM(GroupEnd)
        TGV_SYM(Send) TGV_SYM(Recv) TGV_SYM(AllReduce) TGV_SYM(AllGather)
#undef TGV_SYM
        ok = true;
    });
    if (!ok) {
        snprintf(err, errlen, "%s", msg);
        return nullptr;
    }
    return &api;
}
