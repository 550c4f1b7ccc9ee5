// Data-parallel weight-gradient all-reduce (north_star: the batch is sharded
// over the GPUs of one node, backward-weights gradients are summed over NVLink
// with NCCL, the only collective). SURVEY.md §8(e); the reference is a
// single-process CPU library with no multi-device analog.
//
// Design (one process per GPU):
// * gradients are registered in the order the backward pass produces them
//   (reverse layer order) and grouped into fp32 buckets of ~bucket_bytes;
// * primkit_dp_grad_ready(i) is called right after the backward-weights
//   kernel of gradient i was enqueued on the handle's stream; when a bucket's
//   last gradient is ready, an event on the compute stream gates the comm
//   stream, which packs the bucket (bf16 -> fp32), runs ncclAllReduce(sum) and
//   unpacks (x scale, back to the gradient's type) — overlapping the dgrad /
//   wgrad kernels of the layers still to come;
// * primkit_dp_finish() joins the comm stream back into the compute stream.
// Everything is stream-ordered, so a whole step (convolutions + all-reduces)
// can be captured into one CUDA graph. fp32 reduction: every rank's bf16
// gradient is exact in fp32, the sum is rounded once.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": the copy torch already
// loaded, else the system one), so libprimkit.so has no link-time NCCL
// dependency and never mixes two NCCL versions in one process.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../cuda/kernels.h"
#include "dp.hpp"
#include "handle.hpp"

namespace primkit {
namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_get_async_error)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*comm_abort)(ncclComm_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*get_error_string)(ncclResult_t) = nullptr;
    std::string error;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.error = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
        api.comm_get_async_error =
            reinterpret_cast<decltype(api.comm_get_async_error)>(sym("ncclCommGetAsyncError"));
        api.comm_abort = reinterpret_cast<decltype(api.comm_abort)>(sym("ncclCommAbort"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
        api.get_error_string = reinterpret_cast<decltype(api.get_error_string)>(sym("ncclGetErrorString"));
        if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.comm_destroy ||
            !api.comm_abort || !api.comm_get_async_error || !api.get_error_string)
            api.error = "libnccl.so.2 lacks a required entry point";
    });
    if (!api.error.empty()) throw std::runtime_error("primkit dp: " + api.error);
    return api;
}

void check_nccl(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw std::runtime_error(std::string("primkit dp: ") + what + ": " + nccl().get_error_string(r));
}

}  // namespace

struct DpBucket {
    std::vector<int> members;       // gradient indices
    std::size_t elems = 0;          // fp32 elements
    long long max_elems = 0;        // largest member
    float* buf = nullptr;           // fp32 bucket (device)
    pk_dp_seg* segs = nullptr;      // member table (device)
    cudaEvent_t ready = nullptr;    // compute stream: last member produced
    cudaEvent_t done = nullptr;     // comm stream: all-reduce + unpack finished
    int pending = 0;                // members not yet marked ready this step
    bool issued = false;
};

class DataParallel {
public:
    DataParallel(Handle& h, const ncclUniqueId& id, int nranks, int rank, bool average)
        : h_(h), nranks_(nranks), rank_(rank), scale_(average ? 1.0f / nranks : 1.0f) {
        if (nranks < 1 || rank < 0 || rank >= nranks)
            throw_error(ErrorCode::InvalidValue, "primkit dp: bad rank / world size");
        h_.activate();
        check_nccl(nccl().comm_init_rank(&comm_, nranks, id, rank), "ncclCommInitRank");
        check_cuda(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
        // the in-kernel split-K grid barrier assumes every SM is free
        pk_cuda_allow_grid_barriers(0);
    }
    ~DataParallel() {
        h_.activate();
        if (comm_stream_) cudaStreamSynchronize(comm_stream_);
        for (DpBucket& b : buckets_) {
            if (b.buf) cudaFree(b.buf);
            if (b.segs) cudaFree(b.segs);
            if (b.ready) cudaEventDestroy(b.ready);
            if (b.done) cudaEventDestroy(b.done);
        }
        if (comm_) aborted_ ? (void)0 : (void)nccl().comm_destroy(comm_);
        if (comm_stream_) cudaStreamDestroy(comm_stream_);
        pk_cuda_allow_grid_barriers(1);
    }

    void set_bucket_bytes(std::size_t b) {
        if (sealed_) throw_error(ErrorCode::InvalidValue, "primkit dp: buckets already built");
        bucket_bytes_ = b ? b : 1;
    }

    int add(void* grad, std::uint64_t elems, ElementType et) {
        if (sealed_) throw_error(ErrorCode::InvalidValue, "primkit dp: buckets already built");
        if (!grad || elems == 0) throw_error(ErrorCode::InvalidValue, "primkit dp: empty gradient");
        grads_.push_back({grad, (long long)elems, 0, et == ElementType::BF16 ? PK_BF16 : PK_F32, 0});
        return (int)grads_.size() - 1;
    }

    // Greedy consecutive grouping in registration (= production) order.
    void seal() {
        if (sealed_) return;
        h_.activate();
        bucket_of_.assign(grads_.size(), -1);
        DpBucket cur;
        auto flush = [&] {
            if (cur.members.empty()) return;
            buckets_.push_back(std::move(cur));
            cur = DpBucket{};
        };
        for (int i = 0; i < (int)grads_.size(); ++i) {
            if (!cur.members.empty() && (cur.elems + grads_[i].elems) * 4 > bucket_bytes_) flush();
            grads_[i].offset = (long long)cur.elems;
            // 16-byte aligned members inside the bucket (vector pack / unpack)
            cur.elems += (std::size_t)(grads_[i].elems + 3) / 4 * 4;
            cur.max_elems = std::max(cur.max_elems, grads_[i].elems);
            cur.members.push_back(i);
            bucket_of_[i] = (int)buckets_.size();
        }
        flush();
        for (DpBucket& b : buckets_) {
            check_cuda(cudaMalloc(&b.buf, b.elems * 4), "cudaMalloc");
            std::vector<pk_dp_seg> segs;
            for (int m : b.members) segs.push_back(grads_[m]);
            check_cuda(cudaMalloc(&b.segs, segs.size() * sizeof(pk_dp_seg)), "cudaMalloc");
            check_cuda(cudaMemcpy(b.segs, segs.data(), segs.size() * sizeof(pk_dp_seg),
                                  cudaMemcpyHostToDevice),
                       "cudaMemcpy");
            check_cuda(cudaEventCreateWithFlags(&b.ready, cudaEventDisableTiming), "cudaEventCreate");
            check_cuda(cudaEventCreateWithFlags(&b.done, cudaEventDisableTiming), "cudaEventCreate");
            b.pending = (int)b.members.size();
        }
        sealed_ = true;
    }

    void ready(int i) {
        seal();
        if (i < 0 || i >= (int)grads_.size()) throw_error(ErrorCode::InvalidValue, "primkit dp: bad gradient index");
        DpBucket& b = buckets_[(size_t)bucket_of_[(size_t)i]];
        if (--b.pending == 0) issue(b);
        if (b.pending < 0) throw_error(ErrorCode::InvalidValue, "primkit dp: gradient marked ready twice");
    }

    void finish() {
        seal();
        h_.activate();
        for (DpBucket& b : buckets_) {
            if (!b.issued) issue(b);  // gradients never marked: reduce them now
            check_cuda(cudaStreamWaitEvent(h_.stream(), b.done, 0), "cudaStreamWaitEvent");
            b.issued = false;
            b.pending = (int)b.members.size();
        }
    }

    void check() {
        ncclResult_t async = ncclSuccess;
        check_nccl(nccl().comm_get_async_error(comm_, &async), "ncclCommGetAsyncError");
        if (async != ncclSuccess && async != ncclInProgress) {
            nccl().comm_abort(comm_);
            aborted_ = true;
            throw std::runtime_error(std::string("primkit dp: NCCL asynchronous error, communicator "
                                                 "aborted: ") +
                                     nccl().get_error_string(async));
        }
    }

    int bucket_count() {
        seal();
        return (int)buckets_.size();
    }
    int bucket_of(int i) {
        seal();
        if (i < 0 || i >= (int)grads_.size()) throw_error(ErrorCode::InvalidValue, "primkit dp: bad gradient index");
        return bucket_of_[(size_t)i];
    }

private:
    void issue(DpBucket& b) {
        h_.activate();
        check_cuda(cudaEventRecord(b.ready, h_.stream()), "cudaEventRecord");
        check_cuda(cudaStreamWaitEvent(comm_stream_, b.ready, 0), "cudaStreamWaitEvent");
        check_cuda(pk_cuda_dp_pack(b.segs, (int)b.members.size(), b.max_elems, b.buf, comm_stream_),
                   "dp_pack");
        check_nccl(nccl().all_reduce(b.buf, b.buf, b.elems, ncclFloat32, ncclSum, comm_, comm_stream_),
                   "ncclAllReduce");
        check_cuda(pk_cuda_dp_unpack(b.segs, (int)b.members.size(), b.max_elems, b.buf, scale_,
                                     comm_stream_),
                   "dp_unpack");
        check_cuda(cudaEventRecord(b.done, comm_stream_), "cudaEventRecord");
        b.issued = true;
    }

    Handle& h_;
    int nranks_, rank_;
    float scale_;
    ncclComm_t comm_ = nullptr;
    cudaStream_t comm_stream_ = nullptr;
    bool aborted_ = false;
    bool sealed_ = false;
    std::size_t bucket_bytes_ = 25u << 20;
    std::vector<pk_dp_seg> grads_;
    std::vector<int> bucket_of_;
    std::vector<DpBucket> buckets_;
};

void dp_unique_id(unsigned char out[128]) {
    ncclUniqueId id;
    check_nccl(nccl().get_unique_id(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId");
    std::memcpy(out, &id, 128);
}

DataParallel* dp_create(Handle& h, const unsigned char id[128], int nranks, int rank, bool average) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    return new DataParallel(h, uid, nranks, rank, average);
}
void dp_destroy(DataParallel* dp) { delete dp; }
void dp_set_bucket_bytes(DataParallel& dp, std::size_t b) { dp.set_bucket_bytes(b); }
int dp_add(DataParallel& dp, void* g, std::uint64_t n, ElementType et) { return dp.add(g, n, et); }
void dp_ready(DataParallel& dp, int i) { dp.ready(i); }
void dp_finish(DataParallel& dp) { dp.finish(); }
void dp_check(DataParallel& dp) { dp.check(); }
int dp_bucket_count(DataParallel& dp) { return dp.bucket_count(); }
int dp_bucket_of(DataParallel& dp, int i) { return dp.bucket_of(i); }

}  // namespace primkit
