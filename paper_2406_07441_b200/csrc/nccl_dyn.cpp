// Run-time binding of NCCL (nccl_dyn.hpp).
#include "nccl_dyn.hpp"

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "solver.hpp"

namespace kfb {

namespace {

void* open_nccl()
{
    // 1) an NCCL already mapped into the process (e.g. by torch)
    if (void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD)) return h;
    // 2) an explicit override, then the loader's search path
    if (const char* p = std::getenv("KF_NCCL_LIB"))
        if (void* h = dlopen(p, RTLD_NOW | RTLD_GLOBAL)) return h;
    return dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
}

template <class F>
void bind(void* h, F& f, const char* name)
{
    f = reinterpret_cast<F>(dlsym(h, name));
    if (!f) throw SolverError(5, std::string("libnccl lacks ") + name);
}

}  // namespace

const NcclApi& nccl()
{
    static NcclApi api{};
    static std::once_flag once;
    static std::string error;
    std::call_once(once, [] {
        void* h = open_nccl();
        if (!h) {
            error = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        try {
            bind(h, api.GetUniqueId, "ncclGetUniqueId");
            bind(h, api.CommInitRank, "ncclCommInitRank");
            bind(h, api.CommDestroy, "ncclCommDestroy");
            bind(h, api.GroupStart, "ncclGroupStart");
            bind(h, api.GroupEnd, "ncclGroupEnd");
            bind(h, api.Send, "ncclSend");
            bind(h, api.Recv, "ncclRecv");
            bind(h, api.AllReduce, "ncclAllReduce");
            bind(h, api.GetErrorString, "ncclGetErrorString");
        } catch (const SolverError& e) {
            error = e.what();
        }
    });
    if (!error.empty()) throw SolverError(5, error);
    return api;
}

void nccl_check(ncclResult_t r, const char* what)
{
    if (r != ncclSuccess)
        throw SolverError(5, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace kfb
