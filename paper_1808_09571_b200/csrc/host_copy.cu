// Host <-> device copies of caller (pageable) buffers at pinned-memory speed.
//
// The caller's arrays (numpy, std::vector, a TriangleMesh) are pageable; a
// plain cudaMemcpyAsync from them runs at the driver's single-threaded
// staging rate (~10 GB/s on the B200 boxes, scripts/wkt_probe.py). Large
// copies here go through a per-thread ring of two pinned 64 MiB buffers:
// host threads copy chunk k+1 into one buffer while the DMA engine moves
// chunk k out of the other (~35 GB/s of parallel memcpy, 55 GB/s of DMA).
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "runtime.h"

namespace tdb {

namespace {

constexpr size_t kStageBytes = 64ull << 20;
constexpr size_t kDirectBelow = 8ull << 20;  // small copies: plain cudaMemcpyAsync
constexpr size_t kPiece = 4ull << 20;        // memcpy work unit

// A fixed pool of host threads for the memcpy pieces; run() is serialised.
class Pool {
  public:
    Pool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const unsigned n = std::min(8u, hw > 1 ? hw - 1 : 1u);
        for (unsigned i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void run(size_t tasks, const std::function<void(size_t)>& f) {
        std::lock_guard<std::mutex> serial(run_mu_);
        {
            std::lock_guard<std::mutex> g(m_);
            job_ = &f;
            next_ = 0;
            total_ = tasks;
            left_ = tasks;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> g(m_);
        done_.wait(g, [this] { return left_ == 0; });
        job_ = nullptr;
    }

  private:
    void work() {
        for (;;) {
            size_t k;
            const std::function<void(size_t)>* f;
            {
                std::lock_guard<std::mutex> g(m_);
                if (!job_ || next_ >= total_) return;
                k = next_++;
                f = job_;
            }
            (*f)(k);
            std::lock_guard<std::mutex> g(m_);
            if (--left_ == 0) done_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return stop_ || (gen_ != seen && job_ && next_ < total_); });
                if (stop_) return;
                seen = gen_;
            }
            work();
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_, run_mu_;
    std::condition_variable cv_, done_;
    const std::function<void(size_t)>* job_ = nullptr;
    size_t next_ = 0, total_ = 0, left_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

Pool& pool() {
    static Pool p;
    return p;
}

void par_memcpy(char* dst, const char* src, size_t n) {
    const size_t tasks = (n + kPiece - 1) / kPiece;
    pool().run(tasks, [&](size_t k) {
        const size_t o = k * kPiece;
        std::memcpy(dst + o, src + o, std::min(kPiece, n - o));
    });
}

struct Stage {
    int device = -1;
    char* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    ~Stage() { release(); }
    void release() {
        for (int b = 0; b < 2; ++b) {
            if (ev[b]) cudaEventSynchronize(ev[b]), cudaEventDestroy(ev[b]);
            if (buf[b]) cudaFreeHost(buf[b]);
            buf[b] = nullptr;
            ev[b] = nullptr;
        }
    }
    void ensure() {
        int dev = 0;
        CK(cudaGetDevice(&dev));
        if (dev == device && buf[0]) return;
        release();
        device = dev;
        for (int b = 0; b < 2; ++b) {
            CK(cudaHostAlloc(reinterpret_cast<void**>(&buf[b]), kStageBytes, cudaHostAllocPortable));
            CK(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
            CK(cudaEventRecord(ev[b], 0));
        }
    }
};

thread_local Stage t_stage;

// Page-locked (cudaHostAlloc / cudaHostRegister) host memory: the copy
// engine reads it directly.
bool pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

}  // namespace

void h2d(void* dst, const void* src, size_t n, cudaStream_t st) {
    if (n < kDirectBelow || pinned(src)) {
        if (n) CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st));
        return;
    }
    Stage& s = t_stage;
    s.ensure();
    for (size_t off = 0, c = 0; off < n; off += kStageBytes, ++c) {
        const int b = (int)(c & 1);
        const size_t len = std::min(kStageBytes, n - off);
        CK(cudaEventSynchronize(s.ev[b]));  // the buffer's previous DMA is done
        par_memcpy(s.buf[b], static_cast<const char*>(src) + off, len);
        CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, s.buf[b], len, cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(s.ev[b], st));
    }
}

void d2h(void* dst, const void* src, size_t n, cudaStream_t st) {
    if (n < kDirectBelow || pinned(dst)) {
        if (n) CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return;
    }
    Stage& s = t_stage;
    s.ensure();
    // DMA chunk k+1 into one buffer while the host drains chunk k
    const size_t chunks = (n + kStageBytes - 1) / kStageBytes;
    auto issue = [&](size_t c) {
        const int b = (int)(c & 1);
        const size_t off = c * kStageBytes, len = std::min(kStageBytes, n - off);
        CK(cudaMemcpyAsync(s.buf[b], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(s.ev[b], st));
    };
    CK(cudaEventSynchronize(s.ev[0]));
    CK(cudaEventSynchronize(s.ev[1]));
    issue(0);
    for (size_t c = 0; c < chunks; ++c) {
        const int b = (int)(c & 1);
        if (c + 1 < chunks) issue(c + 1);
        CK(cudaEventSynchronize(s.ev[b]));
        const size_t off = c * kStageBytes, len = std::min(kStageBytes, n - off);
        par_memcpy(static_cast<char*>(dst) + off, s.buf[b], len);
    }
}

}  // namespace tdb
