// pr_comm.cu -- the communicator of the interval-sharded path (include/pr.h
// "distribution"): what crosses GPUs in the sharded rSVD build and Parareal
// (DESIGN.md section 9).  Three operations, all stream-ordered on the
// caller's stream:
//   shift_right  rank r sends a buffer to rank r+1 (the interval-boundary
//                state of the coarse sweep; and U_{q0-1} once)
//   all_gather_v concatenation of per-rank blocks of different sizes, in rank
//                order (the k-dimensional sweep data; coarse sweep matrices)
//   all_reduce_max of a few doubles (delta, eps of eq. bounds_delta_eps)
// Two backends:
//   NCCL   one process per GPU; libnccl.so.2 is loaded at run time (the one
//          the process already has, e.g. PyTorch's, else the system's), so
//          libpr itself has no link-time NCCL dependency.
//   local  `world` virtual ranks in one process on one GPU, each driven by its
//          own host thread and stream: buffers move with device-to-device
//          copies ordered by CUDA events, ranks meet at a host barrier.  No
//          kernel ever waits for another rank.  It runs the sharded schedule
//          with more ranks than GPUs.
#include <dlfcn.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include <condition_variable>
#include <memory>
#include <mutex>
#include <vector>

#include "pr_internal.cuh"

namespace pr {

// --------------------------------------------------------------- NCCL loader
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

static const NcclApi *nccl_api()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // already in the process
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        auto sym = [&](const char *n) { return dlsym(h, n); };
        api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
        api.Send = (decltype(api.Send))sym("ncclSend");
        api.Recv = (decltype(api.Recv))sym("ncclRecv");
        api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
        api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
        api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
        api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv &&
                 api.AllGather && api.AllReduce && api.GroupStart && api.GroupEnd && api.GetErrorString;
    });
    return api.ok ? &api : nullptr;
}

static pr_status nccl_fail(ncclResult_t r, const char *where)
{
    const NcclApi *a = nccl_api();
    char buf[256];
    snprintf(buf, sizeof buf, "NCCL error %d (%s) at %s", (int)r, a ? a->GetErrorString(r) : "?", where);
    set_error(buf);
    return PR_ENCCL;
}

#define PR_NCCL(call)                                         \
    do {                                                      \
        ncclResult_t _r = (call);                             \
        if (_r != ncclSuccess) return nccl_fail(_r, #call);   \
    } while (0)

// ------------------------------------------------------------------ backends
pr_status Comm::all_gather_v(const void *send, void *recv, const long *counts, size_t elem,
                             cudaStream_t s)
{
    // padded all-gather of max(counts) elements per rank, then compaction in
    // rank order (NCCL has no all-gather-v)
    long mx = 0, tot = 0;
    for (int r = 0; r < world; ++r) { mx = counts[r] > mx ? counts[r] : mx; tot += counts[r]; }
    if (mx == 0) return PR_OK;
    const size_t blk = (size_t)mx * elem;
    char *tmp = (char *)ws_alloc(blk * (world + 1), s);
    if (!tmp) { set_error("out of device memory"); return PR_EOOM; }
    char *mine = tmp + blk * world;
    if (counts[rank] > 0) PR_CUDA(cudaMemcpyAsync(mine, send, counts[rank] * elem, cudaMemcpyDeviceToDevice, s));
    pr_status st = all_gather(mine, tmp, blk, s);
    if (st == PR_OK) {
        size_t off = 0;
        for (int r = 0; r < world && st == PR_OK; ++r) {
            if (counts[r] > 0) {
                cudaError_t e = cudaMemcpyAsync((char *)recv + off, tmp + blk * r, counts[r] * elem,
                                                cudaMemcpyDeviceToDevice, s);
                if (e != cudaSuccess) st = cuda_fail(e, "all_gather_v compaction");
            }
            off += counts[r] * elem;
        }
    }
    ws_free(tmp, s);
    return st;
}

__global__ void k_max_rows(const double *in, int world, int count, double *out)
{
    const int i = threadIdx.x;
    if (i >= count) return;
    double m = in[i];
    for (int r = 1; r < world; ++r) m = fmax(m, in[(long)r * count + i]);
    out[i] = m;
}

struct NcclComm : Comm {
    ncclComm_t c = nullptr;
    pr_status shift_right(const void *send, void *recv, size_t bytes, cudaStream_t s) override
    {
        if (world == 1 || bytes == 0) return PR_OK;
        const NcclApi *a = nccl_api();
        PR_NCCL(a->GroupStart());
        if (rank < world - 1) PR_NCCL(a->Send(send, bytes, ncclChar, rank + 1, c, s));
        if (rank > 0) PR_NCCL(a->Recv(recv, bytes, ncclChar, rank - 1, c, s));
        PR_NCCL(a->GroupEnd());
        return PR_OK;
    }
    pr_status all_gather(const void *send, void *recv, size_t bytes, cudaStream_t s) override
    {
        if (world == 1) {
            if (bytes && send != recv) PR_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s));
            return PR_OK;
        }
        PR_NCCL(nccl_api()->AllGather(send, recv, bytes, ncclChar, c, s));
        return PR_OK;
    }
    pr_status all_reduce_max(double *buf, int count, cudaStream_t s) override
    {
        if (world == 1) return PR_OK;
        PR_NCCL(nccl_api()->AllReduce(buf, buf, (size_t)count, ncclFloat64, ncclMax, c, s));
        return PR_OK;
    }
    ~NcclComm() override
    {
        if (c && nccl_api()) nccl_api()->CommDestroy(c);
    }
};

// In-process group of virtual ranks.
struct LocalGroup {
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    std::vector<const void *> send;
    std::vector<cudaEvent_t> ready, done;
    int alive;
    explicit LocalGroup(int w) : world(w), send(w, nullptr), ready(w, nullptr), done(w, nullptr), alive(w)
    {
        for (int r = 0; r < w; ++r) {
            cudaEventCreateWithFlags(&ready[r], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming);
        }
    }
    ~LocalGroup()
    {
        for (int r = 0; r < world; ++r) { cudaEventDestroy(ready[r]); cudaEventDestroy(done[r]); }
    }
    void barrier()
    {
        std::unique_lock<std::mutex> lk(mu);
        const long g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

struct LocalComm : Comm {
    std::shared_ptr<LocalGroup> g;
    pr_status shift_right(const void *send, void *recv, size_t bytes, cudaStream_t s) override
    {
        if (world == 1 || bytes == 0) return PR_OK;
        g->send[rank] = send;
        PR_CUDA(cudaEventRecord(g->ready[rank], s));
        g->barrier();                                      // every rank's buffer is published
        if (rank > 0) {
            PR_CUDA(cudaStreamWaitEvent(s, g->ready[rank - 1], 0));
            PR_CUDA(cudaMemcpyAsync(recv, g->send[rank - 1], bytes, cudaMemcpyDeviceToDevice, s));
            PR_CUDA(cudaEventRecord(g->done[rank], s));
        }
        g->barrier();                                      // every copy is enqueued
        if (rank < world - 1) PR_CUDA(cudaStreamWaitEvent(s, g->done[rank + 1], 0));   // my send was read
        g->barrier();                                      // slots may be reused
        return PR_OK;
    }
    pr_status all_gather(const void *send, void *recv, size_t bytes, cudaStream_t s) override
    {
        if (world == 1) {
            if (bytes && send != recv) PR_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s));
            return PR_OK;
        }
        g->send[rank] = send;
        PR_CUDA(cudaEventRecord(g->ready[rank], s));
        g->barrier();
        for (int r = 0; r < world; ++r) {
            if (r != rank) PR_CUDA(cudaStreamWaitEvent(s, g->ready[r], 0));
            PR_CUDA(cudaMemcpyAsync((char *)recv + bytes * r, g->send[r], bytes, cudaMemcpyDeviceToDevice, s));
        }
        PR_CUDA(cudaEventRecord(g->done[rank], s));
        g->barrier();
        for (int r = 0; r < world; ++r)
            if (r != rank) PR_CUDA(cudaStreamWaitEvent(s, g->done[r], 0));
        g->barrier();
        return PR_OK;
    }
    pr_status all_reduce_max(double *buf, int count, cudaStream_t s) override
    {
        if (world == 1 || count == 0) return PR_OK;
        double *tmp = (double *)ws_alloc((size_t)count * world * sizeof(double), s);
        if (!tmp) { set_error("out of device memory"); return PR_EOOM; }
        pr_status st = all_gather(buf, tmp, (size_t)count * sizeof(double), s);
        if (st == PR_OK) {
            note_launch();
            k_max_rows<<<1, 32 * ((count + 31) / 32), 0, s>>>(tmp, world, count, buf);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) st = cuda_fail(e, "k_max_rows");
        }
        ws_free(tmp, s);
        return st;
    }
};

}  // namespace pr

using namespace pr;

struct pr_comm_s {
    std::unique_ptr<Comm> c;
};

Comm *pr::comm_of(pr_comm h) { return h ? h->c.get() : nullptr; }

extern "C" {

pr_status pr_comm_nccl_unique_id(void *id)
{
    PR_REQUIRE(id, PR_EINVAL, "id is NULL");
    const NcclApi *a = nccl_api();
    PR_REQUIRE(a, PR_ENCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId u;
    PR_NCCL(a->GetUniqueId(&u));
    memcpy(id, &u, sizeof u);
    return PR_OK;
}

pr_status pr_comm_create_nccl(int rank, int world, const void *id, pr_comm *out)
{
    PR_REQUIRE(out && id, PR_EINVAL, "NULL argument");
    PR_REQUIRE(world >= 1 && rank >= 0 && rank < world, PR_EINVAL, "bad rank / world");
    *out = nullptr;
    const NcclApi *a = nccl_api();
    PR_REQUIRE(a, PR_ENCCL, "libnccl.so.2 could not be loaded");
    auto c = std::make_unique<NcclComm>();
    c->rank = rank;
    c->world = world;
    ncclUniqueId u;
    memcpy(&u, id, sizeof u);
    PR_NCCL(a->CommInitRank(&c->c, world, u, rank));
    *out = new pr_comm_s{std::move(c)};
    return PR_OK;
}

pr_status pr_comm_create_local(int world, pr_comm *out)
{
    PR_REQUIRE(out && world >= 1 && world <= 64, PR_EINVAL, "world must be 1..64");
    auto grp = std::make_shared<LocalGroup>(world);
    for (int r = 0; r < world; ++r) {
        auto c = std::make_unique<LocalComm>();
        c->rank = r;
        c->world = world;
        c->g = grp;
        out[r] = new pr_comm_s{std::move(c)};
    }
    return PR_OK;
}

pr_status pr_comm_info(pr_comm h, int *rank, int *world)
{
    PR_REQUIRE(h, PR_EINVAL, "NULL communicator");
    if (rank) *rank = h->c->rank;
    if (world) *world = h->c->world;
    return PR_OK;
}

pr_status pr_comm_destroy(pr_comm h)
{
    delete h;
    return PR_OK;
}

}  // extern "C"
