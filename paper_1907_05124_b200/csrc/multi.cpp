// multi.cpp -- run_batch over several GPUs inside one C-ABI call (SURVEY.md 8(b) "device
// mask", 8(e) multi-GPU).
//
// The reference's only parallelism is its worker pool over run indices (runner.cpp:90-124);
// runs are independent and each result depends only on its index.  Here every device replica
// of the problem gets a contiguous shard of the run indices, one host thread and its own
// stream; the shards run concurrently, then the ranks exchange once:
//   (i)   AllReduce(min) of the shard best energies          -> the batch best energy
//   (ii)  AllReduce(min) of each shard's first index reaching it -> the best index (the
//         reference's first strict minimum, runner.cpp:147-150)
//   (iii) Broadcast of that run's spins from the rank owning it
//   (iv)  AllGather of every shard's records (status, energy, cut, iterations, elapsed)
// and rank 0 aggregates in index order exactly like runner.cpp:126-167.
//
// The exchange is written against a Transport: NcclTransport (device buffers, NCCL loaded at
// run time, ncclCommInitAll over the replicas' devices) for real batches, and HostTransport
// (host memory, the rank threads meeting at a barrier) so the same shard / exchange code is
// testable on a machine without GPUs (mars_debug_exchange).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mars_b200.h"
#include "host_internal.hpp"

namespace marsb200 {
namespace {

// ------------------------------------------------------------------ shard plan

// contiguous shard of run indices for `rank` of `ranks` (same split as mars.py shard_range)
void shard_of(std::int64_t runs, int rank, int ranks, std::int64_t* first, std::int64_t* count) {
    const std::int64_t base = runs / ranks, extra = runs % ranks;
    *first = rank * base + std::min<std::int64_t>(rank, extra);
    *count = base + (rank < extra ? 1 : 0);
}

// packed per-rank record block for the AllGather: [status u8 x m][pad to 8][energy f64 x m]
// [cut f64 x m][iters i64 x m][elapsed f64 x m], m = the largest shard
struct Packing {
    std::int64_t m;
    std::size_t off_energy, off_cut, off_iters, off_elapsed, bytes;
    explicit Packing(std::int64_t maxc) : m(maxc) {
        off_energy = (static_cast<std::size_t>(m) + 7) / 8 * 8;
        off_cut = off_energy + 8 * m;
        off_iters = off_cut + 8 * m;
        off_elapsed = off_iters + 8 * m;
        bytes = off_elapsed + 8 * m;
    }
};

// ------------------------------------------------------------------ transports

struct Transport {
    virtual ~Transport() = default;
    virtual int allreduce_min_f64(int rank, double* buf) = 0;       // buf: 1 element, rank memory
    virtual int allreduce_min_i64(int rank, std::int64_t* buf) = 0;
    virtual int broadcast(int rank, void* buf, std::size_t bytes, int root) = 0;
    virtual int allgather(int rank, const void* send, void* recv, std::size_t bytes_each) = 0;
    virtual void* alloc(int rank, std::size_t bytes) = 0;
    virtual void release(int rank, void* p) = 0;
    virtual int to_host(int rank, void* dst, const void* src, std::size_t bytes) = 0;
    virtual int from_host(int rank, void* dst, const void* src, std::size_t bytes) = 0;
    virtual int copy_local(int rank, void* dst, const void* src, std::size_t bytes) = 0;
};

// In-memory transport: the rank threads meet at a generation barrier; rank 0 combines.
class HostTransport final : public Transport {
  public:
    explicit HostTransport(int ranks) : ranks_(ranks), slots_(ranks, nullptr), sends_(ranks, nullptr) {}
    int allreduce_min_f64(int rank, double* buf) override {
        return combine(rank, buf, [&](int) {
            double v = std::numeric_limits<double>::infinity();
            for (void* s : slots_) v = std::min(v, *static_cast<double*>(s));
            for (void* s : slots_) *static_cast<double*>(s) = v;
        });
    }
    int allreduce_min_i64(int rank, std::int64_t* buf) override {
        return combine(rank, buf, [&](int) {
            std::int64_t v = std::numeric_limits<std::int64_t>::max();
            for (void* s : slots_) v = std::min(v, *static_cast<std::int64_t*>(s));
            for (void* s : slots_) *static_cast<std::int64_t*>(s) = v;
        });
    }
    int broadcast(int rank, void* buf, std::size_t bytes, int root) override {
        return combine(rank, buf, [&](int) {
            for (int r = 0; r < ranks_; ++r)
                if (r != root) std::memcpy(slots_[r], slots_[root], bytes);
        });
    }
    int allgather(int rank, const void* send, void* recv, std::size_t bytes_each) override {
        return combine(rank, recv, [&](int) {
            for (int r = 0; r < ranks_; ++r)
                for (int s = 0; s < ranks_; ++s)
                    std::memcpy(static_cast<char*>(slots_[r]) + s * bytes_each, sends_[s], bytes_each);
        }, send);
    }
    void* alloc(int, std::size_t bytes) override { return std::calloc(std::max<std::size_t>(bytes, 8), 1); }
    void release(int, void* p) override { std::free(p); }
    int to_host(int, void* dst, const void* src, std::size_t b) override { std::memcpy(dst, src, b); return MARS_OK; }
    int from_host(int, void* dst, const void* src, std::size_t b) override { std::memcpy(dst, src, b); return MARS_OK; }
    int copy_local(int, void* dst, const void* src, std::size_t b) override { std::memcpy(dst, src, b); return MARS_OK; }

  private:
    template <class F>
    int combine(int rank, void* buf, F&& op, const void* send = nullptr) {
        std::unique_lock<std::mutex> lk(mu_);
        // wait for the previous collective to drain (its arrived counter back at zero)
        cv_.wait(lk, [&] { return !draining_; });
        slots_[rank] = buf;
        sends_[rank] = send;
        if (++arrived_ == ranks_) {
            op(rank);
            draining_ = true;
            ++gen_;
            cv_.notify_all();
        } else {
            const std::uint64_t g = gen_;
            cv_.wait(lk, [&] { return gen_ != g; });
        }
        if (--arrived_ == 0) {
            draining_ = false;
            cv_.notify_all();
        }
        return MARS_OK;
    }
    int ranks_;
    std::vector<void*> slots_;
    std::vector<const void*> sends_;
    std::mutex mu_;
    std::condition_variable cv_;
    int arrived_ = 0;
    bool draining_ = false;
    std::uint64_t gen_ = 0;
};

// NCCL over the replicas' devices (NVLink / NVSwitch); libnccl.so.2 is loaded at run time so
// the library has no link-time NCCL dependency (the process's already-loaded copy is reused).
struct NcclApi {
    void* h = nullptr;
    decltype(&ncclCommInitAll) init_all = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclAllReduce) allreduce = nullptr;
    decltype(&ncclBroadcast) bcast = nullptr;
    decltype(&ncclAllGather) allgather = nullptr;
    decltype(&ncclGetErrorString) err = nullptr;
    bool load(std::string* why) {
        if (h) return true;
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            *why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return false;
        }
        init_all = reinterpret_cast<decltype(init_all)>(dlsym(h, "ncclCommInitAll"));
        destroy = reinterpret_cast<decltype(destroy)>(dlsym(h, "ncclCommDestroy"));
        allreduce = reinterpret_cast<decltype(allreduce)>(dlsym(h, "ncclAllReduce"));
        bcast = reinterpret_cast<decltype(bcast)>(dlsym(h, "ncclBroadcast"));
        allgather = reinterpret_cast<decltype(allgather)>(dlsym(h, "ncclAllGather"));
        err = reinterpret_cast<decltype(err)>(dlsym(h, "ncclGetErrorString"));
        if (!init_all || !destroy || !allreduce || !bcast || !allgather || !err) {
            *why = "libnccl.so.2 lacks a required entry point";
            return false;
        }
        return true;
    }
};

class NcclTransport final : public Transport {
  public:
    NcclTransport(NcclApi& api, std::vector<int> devs, std::vector<cudaStream_t> streams)
        : api_(api), devs_(std::move(devs)), streams_(std::move(streams)), comms_(devs_.size(), nullptr) {}
    ~NcclTransport() override {
        for (ncclComm_t c : comms_)
            if (c) api_.destroy(c);
    }
    int init() {
        const ncclResult_t r = api_.init_all(comms_.data(), static_cast<int>(devs_.size()), devs_.data());
        return r == ncclSuccess ? MARS_OK : host_fail(MARS_ERR_NCCL, std::string("ncclCommInitAll: ") + api_.err(r));
    }
    int allreduce_min_f64(int rank, double* buf) override {
        return check(api_.allreduce(buf, buf, 1, ncclFloat64, ncclMin, comms_[rank], streams_[rank]), rank, "ncclAllReduce");
    }
    int allreduce_min_i64(int rank, std::int64_t* buf) override {
        return check(api_.allreduce(buf, buf, 1, ncclInt64, ncclMin, comms_[rank], streams_[rank]), rank, "ncclAllReduce");
    }
    int broadcast(int rank, void* buf, std::size_t bytes, int root) override {
        return check(api_.bcast(buf, buf, bytes, ncclUint8, root, comms_[rank], streams_[rank]), rank, "ncclBroadcast");
    }
    int allgather(int rank, const void* send, void* recv, std::size_t bytes_each) override {
        return check(api_.allgather(send, recv, bytes_each, ncclUint8, comms_[rank], streams_[rank]), rank, "ncclAllGather");
    }
    void* alloc(int rank, std::size_t bytes) override {
        void* p = nullptr;
        cudaSetDevice(devs_[rank]);
        if (cudaMalloc(&p, std::max<std::size_t>(bytes, 8)) != cudaSuccess) return nullptr;
        cudaMemsetAsync(p, 0, std::max<std::size_t>(bytes, 8), streams_[rank]);
        return p;
    }
    void release(int rank, void* p) override {
        cudaSetDevice(devs_[rank]);
        cudaStreamSynchronize(streams_[rank]);
        cudaFree(p);
    }
    int to_host(int rank, void* dst, const void* src, std::size_t b) override {
        return cuda(cudaMemcpyAsync(dst, src, b, cudaMemcpyDeviceToHost, streams_[rank]), rank, true);
    }
    int from_host(int rank, void* dst, const void* src, std::size_t b) override {
        return cuda(cudaMemcpyAsync(dst, src, b, cudaMemcpyHostToDevice, streams_[rank]), rank, true);
    }
    int copy_local(int rank, void* dst, const void* src, std::size_t b) override {
        return cuda(cudaMemcpyAsync(dst, src, b, cudaMemcpyDeviceToDevice, streams_[rank]), rank, false);
    }

  private:
    int check(ncclResult_t r, int rank, const char* what) {
        if (r != ncclSuccess) return host_fail(MARS_ERR_NCCL, std::string(what) + ": " + api_.err(r));
        return cuda(cudaSuccess, rank, true);
    }
    int cuda(cudaError_t e, int rank, bool sync) {
        if (e == cudaSuccess && sync) e = cudaStreamSynchronize(streams_[rank]);
        return e == cudaSuccess ? MARS_OK : host_fail(MARS_ERR_CUDA, cudaGetErrorString(e));
    }
    NcclApi& api_;
    std::vector<int> devs_;
    std::vector<cudaStream_t> streams_;
    std::vector<ncclComm_t> comms_;
};

// ------------------------------------------------------------------ the exchange

// One rank's shard records, in the transport's memory (shard-local indexing).
struct Shard {
    std::int64_t first = 0, count = 0;
    const std::uint8_t* status = nullptr;
    const double* energy = nullptr;
    const double* cut = nullptr;
    const std::int64_t* iters = nullptr;
    const double* elapsed = nullptr;
    const std::int8_t* spins = nullptr;   // [count][n]
};

struct Merged {                 // rank 0's host result
    std::vector<std::uint8_t> status;
    std::vector<double> energy, cut, elapsed;
    std::vector<std::int64_t> iters;
    std::vector<std::int8_t> best_spins;
    std::int64_t best_index = -1;
    double best_energy = 0.0;
};

// Every rank thread calls this with its shard; rank 0 fills `out`.  Returns a MARS_* code.
int exchange(Transport& T, int rank, int ranks, std::int64_t total, int n, const Shard& sh, Merged* out) {
    std::int64_t maxc = 0;
    for (int r = 0; r < ranks; ++r) {
        std::int64_t f, c;
        shard_of(total, r, ranks, &f, &c);
        maxc = std::max(maxc, c);
    }
    const Packing pk(maxc);
    // host copies of this shard's status / energy (the candidate scan is a host loop)
    std::vector<std::uint8_t> st(sh.count);
    std::vector<double> en(sh.count);
    int rc = MARS_OK;
    if (sh.count) {
        if ((rc = T.to_host(rank, st.data(), sh.status, sh.count))) return rc;
        if ((rc = T.to_host(rank, en.data(), sh.energy, sh.count * sizeof(double)))) return rc;
    }
    double* d_e = static_cast<double*>(T.alloc(rank, sizeof(double)));
    std::int64_t* d_i = static_cast<std::int64_t*>(T.alloc(rank, sizeof(std::int64_t)));
    std::int8_t* d_sp = static_cast<std::int8_t*>(T.alloc(rank, static_cast<std::size_t>(n)));
    unsigned char* d_send = static_cast<unsigned char*>(T.alloc(rank, pk.bytes));
    unsigned char* d_recv = static_cast<unsigned char*>(T.alloc(rank, pk.bytes * ranks));
    struct Free {
        Transport& T;
        int rank;
        std::vector<void*> ps;
        ~Free() {
            for (void* p : ps) if (p) T.release(rank, p);
        }
    } guard{T, rank, {d_e, d_i, d_sp, d_send, d_recv}};
    if (!d_e || !d_i || !d_sp || !d_send || !d_recv) return host_fail(MARS_ERR_CUDA, "exchange buffer allocation failed");
    // (i) the batch best energy
    double local_best = std::numeric_limits<double>::infinity();
    for (std::int64_t k = 0; k < sh.count; ++k)
        if (st[k] == MARS_RUN_OK) local_best = std::min(local_best, en[k]);
    if ((rc = T.from_host(rank, d_e, &local_best, sizeof(double)))) return rc;
    if ((rc = T.allreduce_min_f64(rank, d_e))) return rc;
    double best = 0.0;
    if ((rc = T.to_host(rank, &best, d_e, sizeof(double)))) return rc;
    // (ii) the first run index attaining it (index order = rank order for contiguous shards)
    std::int64_t cand = std::numeric_limits<std::int64_t>::max();
    for (std::int64_t k = 0; k < sh.count; ++k)
        if (st[k] == MARS_RUN_OK && en[k] == best) {
            cand = sh.first + k;
            break;
        }
    if ((rc = T.from_host(rank, d_i, &cand, sizeof(cand)))) return rc;
    if ((rc = T.allreduce_min_i64(rank, d_i))) return rc;
    std::int64_t best_idx = 0;
    if ((rc = T.to_host(rank, &best_idx, d_i, sizeof(best_idx)))) return rc;
    // (iii) the winning spins from the rank that owns the index
    int owner = 0;
    for (int r = 0; r < ranks; ++r) {
        std::int64_t f, c;
        shard_of(total, r, ranks, &f, &c);
        if (best_idx >= f && best_idx < f + c) owner = r;
    }
    const bool have_best = best_idx != std::numeric_limits<std::int64_t>::max();
    if (have_best && rank == owner && sh.spins)
        if ((rc = T.copy_local(rank, d_sp, sh.spins + static_cast<std::size_t>(best_idx - sh.first) * n, n))) return rc;
    if ((rc = T.broadcast(rank, d_sp, static_cast<std::size_t>(n), owner))) return rc;
    // (iv) every shard's records, packed, to every rank
    if (sh.count) {
        if ((rc = T.copy_local(rank, d_send, sh.status, sh.count))) return rc;
        if ((rc = T.copy_local(rank, d_send + pk.off_energy, sh.energy, sh.count * 8))) return rc;
        if ((rc = T.copy_local(rank, d_send + pk.off_cut, sh.cut, sh.count * 8))) return rc;
        if ((rc = T.copy_local(rank, d_send + pk.off_iters, sh.iters, sh.count * 8))) return rc;
        if ((rc = T.copy_local(rank, d_send + pk.off_elapsed, sh.elapsed, sh.count * 8))) return rc;
    }
    if ((rc = T.allgather(rank, d_send, d_recv, pk.bytes))) return rc;
    if (rank != 0) return MARS_OK;
    std::vector<unsigned char> all(pk.bytes * ranks);
    if ((rc = T.to_host(rank, all.data(), d_recv, all.size()))) return rc;
    out->status.assign(total, 0);
    out->energy.assign(total, 0.0);
    out->cut.assign(total, 0.0);
    out->iters.assign(total, 0);
    out->elapsed.assign(total, 0.0);
    for (int r = 0; r < ranks; ++r) {
        std::int64_t f, c;
        shard_of(total, r, ranks, &f, &c);
        const unsigned char* blk = all.data() + pk.bytes * r;
        std::memcpy(out->status.data() + f, blk, c);
        std::memcpy(out->energy.data() + f, blk + pk.off_energy, c * 8);
        std::memcpy(out->cut.data() + f, blk + pk.off_cut, c * 8);
        std::memcpy(out->iters.data() + f, blk + pk.off_iters, c * 8);
        std::memcpy(out->elapsed.data() + f, blk + pk.off_elapsed, c * 8);
    }
    out->best_spins.assign(n, 0);
    if ((rc = T.to_host(rank, out->best_spins.data(), d_sp, n))) return rc;
    out->best_index = have_best ? best_idx : -1;
    out->best_energy = best;
    return MARS_OK;
}

// Runs `body(rank)` on one thread per rank; the first failure's code and message are re-raised
// on the calling thread (mars_last_error is thread-local).
template <class F>
int on_rank_threads(int ranks, F&& body) {
    std::vector<int> rc(ranks, MARS_OK);
    std::vector<std::string> msg(ranks);
    std::vector<std::thread> th;
    for (int r = 0; r < ranks; ++r)
        th.emplace_back([&, r] {
            rc[r] = body(r);
            if (rc[r]) msg[r] = mars_last_error();
        });
    for (auto& t : th) t.join();
    for (int r = 0; r < ranks; ++r)
        if (rc[r]) return host_fail(rc[r], "rank " + std::to_string(r) + ": " + msg[r]);
    return MARS_OK;
}

int finish(const Merged& m, std::int64_t total, double tol, double secs, mars_records_t* records, mars_stats_t* stats,
           std::int8_t* best_spins, int n) {
    if (records) {
        if (records->status) std::copy(m.status.begin(), m.status.end(), records->status);
        if (records->energy) std::copy(m.energy.begin(), m.energy.end(), records->energy);
        if (records->cut) std::copy(m.cut.begin(), m.cut.end(), records->cut);
        if (records->descent_iters) std::copy(m.iters.begin(), m.iters.end(), records->descent_iters);
        if (records->elapsed_seconds) std::copy(m.elapsed.begin(), m.elapsed.end(), records->elapsed_seconds);
    }
    if (int rc = mars_aggregate(total, m.status.data(), m.energy.data(), m.cut.data(), m.elapsed.data(), tol, secs,
                                stats))
        return rc;
    if (stats->best_index != m.best_index)
        return host_fail(MARS_ERR_RUNTIME, "exchanged best index " + std::to_string(m.best_index) +
                                               " disagrees with the index-order aggregation " +
                                               std::to_string(stats->best_index));
    if (best_spins && m.best_index >= 0) std::copy(m.best_spins.begin(), m.best_spins.begin() + n, best_spins);
    return MARS_OK;
}

NcclApi g_nccl;
std::mutex g_nccl_mu;

}  // namespace
}  // namespace marsb200

using namespace marsb200;

extern "C" {

int mars_run_batch_multi(mars_problem_t* const* replicas, int32_t count, const mars_params_t* prm, int64_t runs,
                         uint64_t base_seed, mars_records_t* records, mars_stats_t* stats, int8_t* best_spins) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!replicas || count < 1 || !stats) return host_fail(MARS_ERR_INPUT, "null argument");
    std::int64_t total = 0;
    if (int rc = mars_run_count(prm, runs, &total)) return rc;      // InputError before any run
    // one replica is mars_run_batch; MARS_MULTI_FORCE=1 keeps the NCCL exchange (a single-rank
    // communicator) so the exchange path can be exercised on a one-GPU machine
    const char* force = std::getenv("MARS_MULTI_FORCE");
    if (count == 1 && !(force && std::atoi(force) == 1))
        return mars_run_batch(replicas[0], prm, runs, base_seed, records, stats, best_spins);
    std::vector<mars_problem_info_t> info(count);
    for (int r = 0; r < count; ++r) {
        if (!replicas[r]) return host_fail(MARS_ERR_INPUT, "null replica");
        if (int rc = mars_problem_info(replicas[r], &info[r])) return rc;
        if (info[r].n != info[0].n) return host_fail(MARS_ERR_INPUT, "replicas of different problems");
        for (int s = 0; s < r; ++s)
            if (info[s].device == info[r].device) return host_fail(MARS_ERR_INPUT, "two replicas on one device");
    }
    const int n = info[0].n;
    std::string why;
    {
        std::lock_guard<std::mutex> lk(g_nccl_mu);
        if (!g_nccl.load(&why)) return host_fail(MARS_ERR_NCCL, why);
    }
    // shards run concurrently, one host thread each
    std::vector<mars_batch_t*> batches(count, nullptr);
    std::vector<BatchDevView> views(count);
    struct Destroy {
        std::vector<mars_batch_t*>& b;
        ~Destroy() {
            for (auto* x : b) mars_batch_destroy(x);
        }
    } destroy{batches};
    int rc = on_rank_threads(count, [&](int r) {
        std::int64_t first, cnt;
        shard_of(total, r, count, &first, &cnt);
        if (int e = mars_batch_create(replicas[r], prm, runs, base_seed, first, cnt, &batches[r])) return e;
        if (int e = mars_batch_upload(batches[r])) return e;
        if (int e = mars_batch_execute(batches[r], nullptr)) return e;
        return batch_device_view(batches[r], &views[r]);
    });
    if (rc) return rc;
    std::vector<int> devs(count);
    std::vector<cudaStream_t> streams(count);
    for (int r = 0; r < count; ++r) {
        devs[r] = views[r].device;
        streams[r] = views[r].stream;
    }
    NcclTransport T(g_nccl, devs, streams);
    if ((rc = T.init())) return rc;
    Merged m;
    rc = on_rank_threads(count, [&](int r) {
        cudaSetDevice(devs[r]);
        const BatchDevView& v = views[r];
        Shard sh{v.first, v.count, v.status, v.energy, v.cut, reinterpret_cast<const std::int64_t*>(v.iters),
                 v.elapsed, v.spins};
        return exchange(T, r, count, total, n, sh, &m);
    });
    if (rc) return rc;
    if (records && records->spins)
        for (int r = 0; r < count; ++r) {
            cudaSetDevice(devs[r]);
            const BatchDevView& v = views[r];
            if (v.count && cudaMemcpy(records->spins + static_cast<std::size_t>(v.first) * n, v.spins,
                                      static_cast<std::size_t>(v.count) * n, cudaMemcpyDeviceToHost) != cudaSuccess)
                return host_fail(MARS_ERR_CUDA, "spins D2H failed");
        }
    if (records && records->fail_temp)
        for (int r = 0; r < count; ++r) {
            mars_records_t part{};
            part.fail_temp = records->fail_temp + views[r].first;
            if (int e = mars_batch_fetch(batches[r], &part, nullptr, nullptr)) return e;
        }
    if (records && records->start_temp) plan_start_temps(prm, base_seed, total, records->start_temp);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return finish(m, total, info[0].integral ? 0.0 : 1e-9, secs, records, stats, best_spins, n);
}

// TEST-ONLY: the shard / exchange logic above on host memory (HostTransport, one thread per
// rank) over caller-given full-batch records: each rank takes its contiguous shard, the four
// collectives run, rank 0 aggregates.  Lets the CPU test suite check the multi-device path.
int mars_debug_exchange(int32_t ranks, int64_t total, int32_t n, const uint8_t* status, const double* energy,
                        const double* cut, const int64_t* iters, const double* elapsed, const int8_t* spins,
                        double tol, mars_records_t* records, mars_stats_t* stats, int8_t* best_spins) {
    if (ranks < 1 || total < 1 || n < 1 || !status || !energy || !cut || !iters || !elapsed || !spins || !stats)
        return host_fail(MARS_ERR_INPUT, "bad argument");
    HostTransport T(ranks);
    Merged m;
    int rc = on_rank_threads(ranks, [&](int r) {
        std::int64_t first, cnt;
        shard_of(total, r, ranks, &first, &cnt);
        Shard sh{first, cnt, status + first, energy + first, cut + first, iters + first, elapsed + first,
                 spins + static_cast<std::size_t>(first) * n};
        return exchange(T, r, ranks, total, n, sh, &m);
    });
    if (rc) return rc;
    return finish(m, total, tol, 0.0, records, stats, best_spins, n);
}

}  // extern "C"
