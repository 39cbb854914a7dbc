// ma_nccl.cpp — NCCL for the data-parallel entry points of the C ABI
// (ma_comm_*, ma_step_allgather, ma_allgather_params, ma_exchange_rows).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, RTLD_NOLOAD first) so
// the library binds to the NCCL the process already uses — torch's bundled
// copy inside a torch process, the system one for a plain C++ caller — and
// libmicroadam_cuda.so has no link-time NCCL dependency. A communicator made by
// one NCCL build must only ever be driven by that build; resolving through the
// already-loaded soname guarantees it. MA_NCCL_LIB overrides the path.
//
// The reference has no distributed path (SPEC.md:366 lists it as a non-goal);
// what the collectives must preserve is the block decomposition
// (compress.cpp:73-85) and the global step used for bias correction
// (window.cpp:43), both of which are replicated per rank by the shard handles.
#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "ma_internal.h"

namespace ma {
namespace nccl {

namespace {

Api g_api;
std::string g_err;
bool g_loaded = false;
std::once_flag g_once;

template <class F>
bool sym(void* lib, const char* name, F*& out) {
    out = reinterpret_cast<F*>(dlsym(lib, name));
    return out != nullptr;
}

void load() {
    const char* env = std::getenv("MA_NCCL_LIB");
    void* lib = nullptr;
    if (env && env[0]) {
        lib = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    } else {
        lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's own NCCL
        if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!lib) {
        const char* e = dlerror();
        g_err = std::string("cannot load NCCL (libnccl.so.2): ") + (e ? e : "?");
        return;
    }
    Api a{};
    bool ok = sym(lib, "ncclGetUniqueId", a.GetUniqueId) && sym(lib, "ncclCommInitRank", a.CommInitRank) &&
              sym(lib, "ncclCommDestroy", a.CommDestroy) && sym(lib, "ncclCommCount", a.CommCount) &&
              sym(lib, "ncclCommUserRank", a.CommUserRank) && sym(lib, "ncclAllGather", a.AllGather) &&
              sym(lib, "ncclAllReduce", a.AllReduce) && sym(lib, "ncclBroadcast", a.Broadcast) &&
              sym(lib, "ncclGroupStart", a.GroupStart) && sym(lib, "ncclGroupEnd", a.GroupEnd) &&
              sym(lib, "ncclGetErrorString", a.GetErrorString) && sym(lib, "ncclGetVersion", a.GetVersion);
    if (!ok) {
        g_err = "NCCL library lacks a required symbol";
        return;
    }
    g_api = a;
    g_loaded = true;
}

}  // namespace

const Api* api(std::string* err) {
    std::call_once(g_once, load);
    if (!g_loaded) {
        if (err) *err = g_err;
        return nullptr;
    }
    return &g_api;
}

std::string describe(const Api* a, int rc) {
    const char* s = a && a->GetErrorString ? a->GetErrorString(rc) : nullptr;
    return std::string("NCCL error ") + std::to_string(rc) + (s ? std::string(": ") + s : std::string());
}

}  // namespace nccl
}  // namespace ma
