// xport.cpp -- NCCL and loopback transports of the z-slab plan (xport.h).
#include "xport.h"

#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <vector>

#include "../../include/nufft.h"

namespace nufft {

namespace {

// ------------------------------------------------------------------------ NCCL
struct NcclXport final : Xport {
    ncclComm_t comm = nullptr;
    ~NcclXport() override {
        if (comm) ncclCommDestroy(comm);
    }
    static int st(ncclResult_t e) { return e == ncclSuccess ? NUFFT_OK : NUFFT_ERR_NCCL; }
    int group_start() override { return st(ncclGroupStart()); }
    int send(const void* buf, size_t bytes, int peer, cudaStream_t s) override {
        return st(ncclSend(buf, bytes, ncclChar, peer, comm, s));
    }
    int recv(void* buf, size_t bytes, int peer, cudaStream_t s) override {
        return st(ncclRecv(buf, bytes, ncclChar, peer, comm, s));
    }
    int group_end(cudaStream_t) override { return st(ncclGroupEnd()); }
    int alltoall(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        return st(ncclAlltoAll(send, recv, bytes, ncclChar, comm, s));
    }
    int allreduce_max_u64(unsigned long long* v, cudaStream_t s) override {
        return st(ncclAllReduce(v, v, 1, ncclUint64, ncclMax, comm, s));
    }
};

// -------------------------------------------------------------------- loopback
struct Msg {
    const void* src;
    void* dst;
    size_t bytes;
    int peer;
};

struct LoopShared {
    int P = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long gen = 0;
    struct Post {
        std::vector<Msg> sends;
        cudaEvent_t ready = nullptr, done = nullptr;
    };
    std::vector<Post> posts;
    std::vector<unsigned long long> red;
    int refs = 0;

    // every rank's host thread meets here
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const unsigned long long g = gen;
        if (++arrived == P) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

struct LoopXport final : Xport {
    std::shared_ptr<LoopShared> sh;
    std::vector<Msg> sends, recvs;
    ~LoopXport() override {
        LoopShared::Post& me = sh->posts[r];
        if (me.ready) cudaEventDestroy(me.ready);
        if (me.done) cudaEventDestroy(me.done);
    }
    int group_start() override {
        sends.clear();
        recvs.clear();
        return NUFFT_OK;
    }
    int send(const void* buf, size_t bytes, int peer, cudaStream_t) override {
        if (peer < 0 || peer >= P) return NUFFT_ERR_ARG;
        sends.push_back(Msg{buf, nullptr, bytes, peer});
        return NUFFT_OK;
    }
    int recv(void* buf, size_t bytes, int peer, cudaStream_t) override {
        if (peer < 0 || peer >= P) return NUFFT_ERR_ARG;
        recvs.push_back(Msg{nullptr, buf, bytes, peer});
        return NUFFT_OK;
    }
    // publish the sends, copy every receive from the matching send (k-th receive from
    // q <- k-th send of q to this rank) once q's data is ready, and keep the sender's
    // stream from overwriting a send buffer before its receivers have copied it.  All
    // ranks pass every barrier even after a local error (no rank is left waiting).
    int group_end(cudaStream_t s) override {
        int status = NUFFT_OK;
        LoopShared::Post& me = sh->posts[r];
        me.sends = sends;
        if (cudaEventRecord(me.ready, s) != cudaSuccess) status = NUFFT_ERR_CUDA;
        sh->barrier();
        std::vector<int> taken(P, 0);
        for (const Msg& rv : recvs) {
            const LoopShared::Post& q = sh->posts[rv.peer];
            int k = taken[rv.peer]++, seen = 0;
            const Msg* match = nullptr;
            for (const Msg& sd : q.sends)
                if (sd.peer == r && seen++ == k) {
                    match = &sd;
                    break;
                }
            if (!match) {
                status = NUFFT_ERR_ARG;
                continue;
            }
            const size_t n = match->bytes < rv.bytes ? match->bytes : rv.bytes;
            if (!n) continue;
            if (cudaStreamWaitEvent(s, q.ready, 0) != cudaSuccess ||
                cudaMemcpyAsync(rv.dst, match->src, n, cudaMemcpyDeviceToDevice, s) !=
                    cudaSuccess)
                status = NUFFT_ERR_CUDA;
        }
        if (cudaEventRecord(me.done, s) != cudaSuccess) status = NUFFT_ERR_CUDA;
        sh->barrier();
        for (const Msg& sd : sends)
            if (cudaStreamWaitEvent(s, sh->posts[sd.peer].done, 0) != cudaSuccess)
                status = NUFFT_ERR_CUDA;
        sh->barrier();  // every wait is enqueued before any event is recorded again
        sends.clear();
        recvs.clear();
        return status;
    }
    int alltoall(const void* send_buf, void* recv_buf, size_t bytes, cudaStream_t s) override {
        group_start();
        for (int q = 0; q < P; ++q) {
            send(static_cast<const char*>(send_buf) + (size_t)q * bytes, bytes, q, s);
            recv(static_cast<char*>(recv_buf) + (size_t)q * bytes, bytes, q, s);
        }
        return group_end(s);
    }
    int allreduce_max_u64(unsigned long long* v, cudaStream_t s) override {
        int status = NUFFT_OK;
        unsigned long long h = 0;
        if (cudaMemcpyAsync(&h, v, sizeof(h), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            status = NUFFT_ERR_CUDA;
        sh->red[r] = h;
        sh->barrier();
        unsigned long long mx = 0;
        for (int q = 0; q < P; ++q) mx = sh->red[q] > mx ? sh->red[q] : mx;
        sh->barrier();
        if (cudaMemcpyAsync(v, &mx, sizeof(mx), cudaMemcpyHostToDevice, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            status = NUFFT_ERR_CUDA;
        return status;
    }
};

}  // namespace

Xport* xport_nccl(const char id[128], int nranks, int rank) {
    NcclXport* x = new (std::nothrow) NcclXport();
    if (!x) return nullptr;
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    if (ncclCommInitRank(&x->comm, nranks, u, rank) != ncclSuccess) {
        x->comm = nullptr;
        delete x;
        return nullptr;
    }
    x->P = nranks;
    x->r = rank;
    return x;
}

void xport_nccl_unique_id(char id[128], int* status) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId u;
    if (ncclGetUniqueId(&u) != ncclSuccess) {
        *status = NUFFT_ERR_NCCL;
        return;
    }
    std::memcpy(id, &u, 128);
    *status = NUFFT_OK;
}

int xport_loopback(int nranks, Xport** out) {
    if (nranks < 1 || !out) return NUFFT_ERR_ARG;
    auto sh = std::make_shared<LoopShared>();
    sh->P = nranks;
    sh->posts.resize(nranks);
    sh->red.assign(nranks, 0);
    for (int q = 0; q < nranks; ++q) {
        if (cudaEventCreateWithFlags(&sh->posts[q].ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&sh->posts[q].done, cudaEventDisableTiming) != cudaSuccess) {
            for (auto& pq : sh->posts) {
                if (pq.ready) cudaEventDestroy(pq.ready);
                if (pq.done) cudaEventDestroy(pq.done);
                pq.ready = pq.done = nullptr;
            }
            return NUFFT_ERR_CUDA;
        }
    }
    for (int q = 0; q < nranks; ++q) {
        LoopXport* x = new (std::nothrow) LoopXport();
        if (!x) {
            for (int k = 0; k < q; ++k) delete out[k];  // each destroys its rank's events
            for (int k = q; k < nranks; ++k) {
                cudaEventDestroy(sh->posts[k].ready);
                cudaEventDestroy(sh->posts[k].done);
            }
            return NUFFT_ERR_ALLOC;
        }
        x->P = nranks;
        x->r = q;
        x->sh = sh;
        out[q] = x;
    }
    return NUFFT_OK;
}

}  // namespace nufft
