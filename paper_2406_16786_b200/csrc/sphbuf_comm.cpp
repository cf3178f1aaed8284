// sphbuf_comm.cpp — the library's own communicator for the x-slab decomposition
// (§5 "the library owns its ncclComm_t so a step can be CUDA-graph
// captured").  Two exchanges per update, both enqueued on the caller's stream:
//   * the count allgather: every rank's per-port create/delete counts
//     (int32 [2 max_ports]) -> the count matrix the compaction turns into
//     GPU-count-independent IDs (reading R14);
//   * the neighbour exchange: the migration buffer of particles that left the
//     slab through its lower face goes to rank r-1, the upper one to r+1 (the
//     candidates are spatially local, and particles move less than a
//     cell per step, so only neighbours exchange).
// NCCL is loaded with dlopen("libnccl.so.2") at the first sph_comm_* call, so
// libsphbuf.so itself has no link-time NCCL dependency; inside a process that
// already imported torch this resolves to torch's NCCL (one instance, shared
// with torch.distributed).  A loopback transport (ranks = contexts of one
// process on one device, device copies instead of NCCL) exercises the same host
// logic and buffers on a single GPU.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "sphbuf_internal.h"

namespace sphbuf {

namespace {

struct NcclApi {
    bool tried = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
};

NcclApi &api()
{
    static NcclApi a;
    static std::mutex m;
    std::lock_guard<std::mutex> g(m);
    if (a.tried) return a;
    a.tried = true;
    const char *env = getenv("SPHBUF_NCCL_LIB");
    void *h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        a.err = std::string("cannot load NCCL: ") + dlerror();
        return a;
    }
    auto sym = [&](const char *n) {
        void *p = dlsym(h, n);
        if (!p && a.err.empty()) a.err = std::string("NCCL symbol missing: ") + n;
        return p;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.CommGetAsyncError = reinterpret_cast<decltype(a.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    return a;
}

bool nccl_ok(ncclResult_t r, const char *what, std::string *err)
{
    if (r == ncclSuccess) return true;
    NcclApi &a = api();
    if (err) *err = std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "NCCL error");
    return false;
}

}  // namespace

int comm_unique_id(void *out, std::string *err)
{
    NcclApi &a = api();
    if (!a.err.empty()) {
        *err = a.err;
        return -1;
    }
    ncclUniqueId id;
    if (!nccl_ok(a.GetUniqueId(&id), "ncclGetUniqueId", err)) return -1;
    static_assert(sizeof(ncclUniqueId) == SPH_COMM_ID_BYTES, "ncclUniqueId size");
    memcpy(out, &id, sizeof(id));
    return 0;
}

Comm *comm_nccl(const void *id, int nranks, int rank, std::string *err)
{
    NcclApi &a = api();
    if (!a.err.empty()) {
        *err = a.err;
        return nullptr;
    }
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclComm_t comm = nullptr;
    if (!nccl_ok(a.CommInitRank(&comm, nranks, uid, rank), "ncclCommInitRank", err)) return nullptr;
    Comm *c = new Comm();
    c->kind = Comm::NCCL;
    c->nccl = comm;
    c->nranks = nranks;
    c->rank = rank;
    return c;
}

void comm_destroy(Comm *c)
{
    if (!c) return;
    if (c->kind == Comm::NCCL && c->nccl) {
        NcclApi &a = api();
        if (a.CommDestroy) a.CommDestroy(static_cast<ncclComm_t>(c->nccl));
    }
    delete c;
}

int comm_allgather_i32(Comm *c, const int32_t *send, int32_t *recv, size_t count, cudaStream_t s,
                       const std::vector<const int32_t *> &loop_send, std::string *err)
{
    if (c->kind == Comm::NCCL) {
        NcclApi &a = api();
        return nccl_ok(a.AllGather(send, recv, count, ncclInt32, static_cast<ncclComm_t>(c->nccl), s),
                       "ncclAllGather", err) ? 0 : -1;
    }
    // loopback: every member's counts (all enqueued earlier on this stream)
    for (int r = 0; r < c->nranks; ++r) {
        const int32_t *src = r == c->rank ? send : loop_send[r];
        if (!src) {
            *err = "loopback allgather: a member has not run sph_buffer_update";
            return -1;
        }
        cudaError_t e = cudaMemcpyAsync(recv + (size_t)r * count, src, count * sizeof(int32_t),
                                        cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) {
            *err = std::string("loopback allgather: ") + cudaGetErrorString(e);
            return -1;
        }
    }
    return 0;
}

int comm_neighbour_exchange(Comm *c, const float *send_lo, const float *send_hi, float *recv_lo, float *recv_hi,
                            size_t count, cudaStream_t s, const float *loop_lo_peer, const float *loop_hi_peer,
                            std::string *err)
{
    const int r = c->rank, P = c->nranks;
    if (P <= 1) return 0;
    if (c->kind == Comm::NCCL) {
        NcclApi &a = api();
        ncclComm_t comm = static_cast<ncclComm_t>(c->nccl);
        if (!nccl_ok(a.GroupStart(), "ncclGroupStart", err)) return -1;
        bool ok = true;
        if (r > 0) {
            ok = ok && nccl_ok(a.Send(send_lo, count, ncclFloat32, r - 1, comm, s), "ncclSend", err);
            ok = ok && nccl_ok(a.Recv(recv_lo, count, ncclFloat32, r - 1, comm, s), "ncclRecv", err);
        }
        if (r < P - 1) {
            ok = ok && nccl_ok(a.Send(send_hi, count, ncclFloat32, r + 1, comm, s), "ncclSend", err);
            ok = ok && nccl_ok(a.Recv(recv_hi, count, ncclFloat32, r + 1, comm, s), "ncclRecv", err);
        }
        const bool ended = nccl_ok(a.GroupEnd(), "ncclGroupEnd", ok ? err : nullptr);
        return ok && ended ? 0 : -1;
    }
    // loopback: rank r-1's upper buffer is our lower receive, rank r+1's lower buffer our upper one
    cudaError_t e = cudaSuccess;
    if (r > 0) e = cudaMemcpyAsync(recv_lo, loop_lo_peer, count * sizeof(float), cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && r < P - 1)
        e = cudaMemcpyAsync(recv_hi, loop_hi_peer, count * sizeof(float), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) {
        *err = std::string("loopback exchange: ") + cudaGetErrorString(e);
        return -1;
    }
    return 0;
}

int comm_async_error(Comm *c, std::string *err)
{
    if (!c || c->kind != Comm::NCCL) return 0;
    NcclApi &a = api();
    ncclResult_t r = ncclSuccess;
    if (!nccl_ok(a.CommGetAsyncError(static_cast<ncclComm_t>(c->nccl), &r), "ncclCommGetAsyncError", err))
        return -1;
    return nccl_ok(r, "NCCL (asynchronous)", err) ? 0 : -1;
}

}  // namespace sphbuf
