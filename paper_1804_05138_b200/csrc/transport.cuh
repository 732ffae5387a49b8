// transport.cuh -- the exchanges of the multi-GPU schedule,
// behind one interface with two implementations:
//
//  * NcclTransport: NCCL (dlopen'd, dist.cuh) over NVLink/NVSwitch; one rank
//    per process and GPU.  Production path.
//  * LoopTransport: P contexts of ONE process on ONE device, each driven by
//    its own host thread (testing API rqrcp_create_loopback_group).  Every
//    collective is a host rendezvous plus cudaMemcpyAsync / a small summing
//    kernel ordered by CUDA events: no kernel ever waits on another rank's
//    kernel (kernels of different ranks never spin on each other), so the
//    P-rank driver logic runs on a single GPU.  Used by the GPU P-invariance
//    tests; never on the bench path.
//
// The driver only needs four fixed-size, stream-ordered collectives (no host
// knowledge of the pivots, so no host synchronisation inside the panel loop):
//   allgather(send, recv, bytes)      recv = [rank 0 | rank 1 | ...]
//   bcast(buf, bytes, root)
//   reduce_u64(send, recv, n, root)   recv (root) = elementwise sum of the
//                                     ranks' uint64 words; the driver packs
//                                     fp64 columns so that every element has
//                                     ONE non-zero contributor (the owner):
//                                     the integer sum is then the exact bit
//                                     pattern (no rounding, -0.0 preserved)
//   poll(err)                         asynchronous communicator errors
#pragma once
#include <chrono>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "dist.cuh"

namespace rq {

struct Transport {
    int nranks = 1, rank = 0;
    virtual ~Transport() {}
    virtual int allgather(const void *send, void *recv, size_t bytes, cudaStream_t st, std::string &err) = 0;
    virtual int bcast(void *buf, size_t bytes, int root, cudaStream_t st, std::string &err) = 0;
    virtual int reduce_u64(const uint64_t *send, uint64_t *recv, size_t n, int root, cudaStream_t st,
                           std::string &err) = 0;
    // 0: fine; non-zero: the communicator reported an asynchronous error (err set)
    virtual int poll(std::string &err) { (void)err; return 0; }
    virtual void abort() {}
    virtual const char *kind() const = 0;
};

// ---------------------------------------------------------------------------
// NCCL
// ---------------------------------------------------------------------------
struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    ~NcclTransport() override {
        if (comm && nccl().ok) nccl().CommDestroy(comm);
    }
    static int check(ncclResult_t r, const char *what, std::string &err) {
        if (r == 0) return 0;
        err = std::string(what) + ": " + nccl().GetErrorString(r);
        return 2;  // RQRCP_E_NCCL
    }
    int allgather(const void *send, void *recv, size_t bytes, cudaStream_t st, std::string &err) override {
        return check(nccl().AllGather(send, recv, bytes, ncclUint8, comm, st), "ncclAllGather", err);
    }
    int bcast(void *buf, size_t bytes, int root, cudaStream_t st, std::string &err) override {
        return check(nccl().Broadcast(buf, buf, bytes, ncclUint8, root, comm, st), "ncclBroadcast", err);
    }
    int reduce_u64(const uint64_t *send, uint64_t *recv, size_t n, int root, cudaStream_t st,
                   std::string &err) override {
        return check(nccl().Reduce(send, recv, n, ncclUint64, ncclSum, root, comm, st), "ncclReduce", err);
    }
    int poll(std::string &err) override {
        if (!comm || !nccl().CommGetAsyncError) return 0;
        ncclResult_t a = 0;
        if (nccl().CommGetAsyncError(comm, &a) != 0) return 0;
        if (a == 0 || a == 7 /* ncclInProgress */) return 0;
        err = std::string("NCCL asynchronous error: ") + nccl().GetErrorString(a);
        return 2;
    }
    void abort() override {
        if (comm && nccl().CommAbort) {
            nccl().CommAbort(comm);
            comm = nullptr;
        }
    }
    const char *kind() const override { return "nccl"; }
};

// ---------------------------------------------------------------------------
// In-process loopback (testing): shared state of a group of P contexts
// ---------------------------------------------------------------------------
constexpr int LOOP_MAXP = 16;

struct U64Srcs {
    const uint64_t *p[LOOP_MAXP];
};
__global__ void loop_u64_sum_kernel(U64Srcs s, int P, uint64_t *dst, size_t n) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        uint64_t acc = 0;
        for (int r = 0; r < P; ++r) acc += s.p[r][e];
        dst[e] = acc;
    }
}

struct LoopGroup {
    int P = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    bool broken = false;
    std::vector<const void *> ptr;
    std::vector<cudaEvent_t> ev_ready, ev_done;
    double timeout_s = 300.0;
    explicit LoopGroup(int p) : P(p), ptr(p, nullptr), ev_ready(p, nullptr), ev_done(p, nullptr) {
        for (int r = 0; r < P; ++r) {
            cudaEventCreateWithFlags(&ev_ready[r], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&ev_done[r], cudaEventDisableTiming);
        }
    }
    ~LoopGroup() {
        for (int r = 0; r < P; ++r) {
            if (ev_ready[r]) cudaEventDestroy(ev_ready[r]);
            if (ev_done[r]) cudaEventDestroy(ev_done[r]);
        }
    }
    // host rendezvous of the P driver threads; false on timeout / a broken group
    bool barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (broken) return false;
        const uint64_t g = gen;
        if (++arrived == P) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return true;
        }
        const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return gen != g || broken; });
        if (!ok || broken) {
            broken = true;
            cv.notify_all();
            return false;
        }
        return true;
    }
    void mark_broken() {
        std::lock_guard<std::mutex> lk(mu);
        broken = true;
        cv.notify_all();
    }
};

struct LoopTransport : Transport {
    std::shared_ptr<LoopGroup> grp;
    int fail(std::string &err, const char *what) {
        err = std::string("loopback ") + what + ": rendezvous failed (another rank stopped or timed out)";
        return 2;
    }
    int cu(cudaError_t e, std::string &err) {
        if (e == cudaSuccess) return 0;
        err = std::string("loopback: ") + cudaGetErrorString(e);
        grp->mark_broken();
        return 1;
    }
    // publish this rank's pointer with a ready event, meet the others
    int publish(const void *p, cudaStream_t st, std::string &err, const char *what) {
        grp->ptr[rank] = p;
        if (int rc = cu(cudaEventRecord(grp->ev_ready[rank], st), err)) return rc;
        return grp->barrier() ? 0 : fail(err, what);
    }
    // after this rank's copies: record done, meet, and order this stream after
    // every rank's copies (no rank may overwrite a source another still reads)
    int finish(cudaStream_t st, std::string &err, const char *what) {
        if (int rc = cu(cudaEventRecord(grp->ev_done[rank], st), err)) return rc;
        if (!grp->barrier()) return fail(err, what);
        for (int r = 0; r < nranks; ++r)
            if (r != rank)
                if (int rc = cu(cudaStreamWaitEvent(st, grp->ev_done[r], 0), err)) return rc;
        return 0;
    }
    int allgather(const void *send, void *recv, size_t bytes, cudaStream_t st, std::string &err) override {
        if (int rc = publish(send, st, err, "allgather")) return rc;
        for (int r = 0; r < nranks; ++r) {
            if (int rc = cu(cudaStreamWaitEvent(st, grp->ev_ready[r], 0), err)) return rc;
            if (bytes)
                if (int rc = cu(cudaMemcpyAsync((char *)recv + (size_t)r * bytes, grp->ptr[r], bytes,
                                                cudaMemcpyDeviceToDevice, st), err))
                    return rc;
        }
        return finish(st, err, "allgather");
    }
    int bcast(void *buf, size_t bytes, int root, cudaStream_t st, std::string &err) override {
        if (int rc = publish(buf, st, err, "bcast")) return rc;
        if (rank != root) {
            if (int rc = cu(cudaStreamWaitEvent(st, grp->ev_ready[root], 0), err)) return rc;
            if (bytes)
                if (int rc = cu(cudaMemcpyAsync(buf, grp->ptr[root], bytes, cudaMemcpyDeviceToDevice, st), err)) return rc;
        }
        return finish(st, err, "bcast");
    }
    int reduce_u64(const uint64_t *send, uint64_t *recv, size_t n, int root, cudaStream_t st,
                   std::string &err) override {
        if (int rc = publish(send, st, err, "reduce")) return rc;
        if (rank == root && n) {
            U64Srcs s{};
            for (int r = 0; r < nranks; ++r) {
                if (int rc = cu(cudaStreamWaitEvent(st, grp->ev_ready[r], 0), err)) return rc;
                s.p[r] = (const uint64_t *)grp->ptr[r];
            }
            const int blocks = (int)std::min<size_t>(1024, (n + 255) / 256);
            loop_u64_sum_kernel<<<blocks, 256, 0, st>>>(s, nranks, recv, n);
            if (int rc = cu(cudaGetLastError(), err)) return rc;
        }
        return finish(st, err, "reduce");
    }
    void abort() override { grp->mark_broken(); }
    const char *kind() const override { return "loopback"; }
};

}  // namespace rq
