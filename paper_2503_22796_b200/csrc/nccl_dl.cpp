// nccl_dl.cpp — NCCL for the multi-GPU layer, bound at run
// time with dlopen("libnccl.so.2").
//
// The library does not link NCCL: a process that already loaded it (torch's
// bundled libnccl, or the caller's own) gets that copy back from dlopen by
// its soname, so a communicator created by the caller can be passed straight
// in; a plain C/C++ caller gets the system libnccl.so.2. Only the types of
// nccl.h are used (ABI-stable since NCCL 2.x); the entry points are looked up
// by name.
#include "nccl_dl.h"

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

namespace dfa2nccl {
namespace {

struct Api {
    void* handle = nullptr;
    std::string why;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    decltype(&ncclCommCount) comm_count = nullptr;
    decltype(&ncclCommUserRank) comm_user_rank = nullptr;
};

Api& api() {
    static Api a;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            a.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (a.handle)
                break;
        }
        if (!a.handle) {
            const char* e = dlerror();
            a.why = std::string("dlopen(libnccl.so.2) failed: ") + (e ? e : "?");
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(a.handle, name));
            if (!fn && a.why.empty())
                a.why = std::string("libnccl.so.2 lacks ") + name;
        };
        sym(a.get_unique_id, "ncclGetUniqueId");
        sym(a.comm_init_rank, "ncclCommInitRank");
        sym(a.comm_destroy, "ncclCommDestroy");
        sym(a.group_start, "ncclGroupStart");
        sym(a.group_end, "ncclGroupEnd");
        sym(a.broadcast, "ncclBroadcast");
        sym(a.error_string, "ncclGetErrorString");
        sym(a.comm_count, "ncclCommCount");
        sym(a.comm_user_rank, "ncclCommUserRank");
    });
    return a;
}

std::string err(int r) {
    Api& a = api();
    return a.error_string ? a.error_string(static_cast<ncclResult_t>(r)) : ("nccl error " + std::to_string(r));
}

}  // namespace

bool available(std::string* why) {
    Api& a = api();
    if (why)
        *why = a.why;
    return a.why.empty();
}

std::string unique_id(char* out) {
    std::string why;
    if (!available(&why))
        return why;
    ncclUniqueId id;
    const ncclResult_t r = api().get_unique_id(&id);
    if (r != ncclSuccess)
        return "ncclGetUniqueId: " + err(r);
    static_assert(sizeof(id.internal) == kUniqueIdBytes, "NCCL unique id size");
    for (int i = 0; i < kUniqueIdBytes; ++i)
        out[i] = id.internal[i];
    return {};
}

std::string comm_init(void** comm, int nranks, const char* id_bytes, int rank) {
    std::string why;
    if (!available(&why))
        return why;
    ncclUniqueId id;
    for (int i = 0; i < kUniqueIdBytes; ++i)
        id.internal[i] = id_bytes[i];
    ncclComm_t c = nullptr;
    const ncclResult_t r = api().comm_init_rank(&c, nranks, id, rank);
    if (r != ncclSuccess)
        return "ncclCommInitRank: " + err(r);
    *comm = c;
    return {};
}

std::string comm_destroy(void* comm) {
    std::string why;
    if (!available(&why))
        return why;
    const ncclResult_t r = api().comm_destroy(static_cast<ncclComm_t>(comm));
    return r == ncclSuccess ? std::string() : "ncclCommDestroy: " + err(r);
}

std::string comm_shape(void* comm, int* nranks, int* rank) {
    std::string why;
    if (!available(&why))
        return why;
    ncclResult_t r = api().comm_count(static_cast<ncclComm_t>(comm), nranks);
    if (r == ncclSuccess)
        r = api().comm_user_rank(static_cast<ncclComm_t>(comm), rank);
    return r == ncclSuccess ? std::string() : "ncclCommCount/UserRank: " + err(r);
}

// All-gather with unequal parts, in place: part r (bytes [off[r], off[r+1])
// of buf) is broadcast from rank r; one NCCL group, so the W broadcasts run
// concurrently over NVLink / NVSwitch.
std::string allgather_v(void* comm, void* buf, const int64_t* off, int world, cudaStream_t stream) {
    std::string why;
    if (!available(&why))
        return why;
    Api& a = api();
    ncclResult_t r = a.group_start();
    if (r != ncclSuccess)
        return "ncclGroupStart: " + err(r);
    for (int p = 0; p < world && r == ncclSuccess; ++p) {
        const size_t bytes = static_cast<size_t>(off[p + 1] - off[p]);
        if (!bytes)
            continue;
        char* base = static_cast<char*>(buf) + off[p];
        r = a.broadcast(base, base, bytes, ncclUint8, p, static_cast<ncclComm_t>(comm), stream);
    }
    const ncclResult_t e = a.group_end();
    if (r != ncclSuccess)
        return "ncclBroadcast: " + err(r);
    if (e != ncclSuccess)
        return "ncclGroupEnd: " + err(e);
    return {};
}

}  // namespace dfa2nccl
