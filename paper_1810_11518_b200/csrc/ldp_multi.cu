// ldp_multi.cu -- several GPUs in one process (include/aldp_cuda.h).
//
// Images are independent (no cross-image state; the 3x3 halo never leaves an
// image), so a batch splits into contiguous image ranges with no collective on
// the data path. The host-buffer entry point gives each range its own
// persistent worker thread: the thread binds its device and runs the chunked
// H2D / kernel / D2H pipeline of aldp_ldp_batch_host (ldp_host.cu), whose
// pinned staging and streams live in thread-local storage and so are reused
// call after call. Each device copies its codes and histograms straight into
// its slice of the caller's buffers. The reference's only concurrency is the
// same fan-out over image ranges on CPU threads (proj/src/verify.cpp:85-98).
#include <cuda_runtime.h>

#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "aldp_cuda.h"

namespace aldp_b200 {

aldp_status set_error(aldp_status s, const std::string& msg);  // ldp_kernels.cu

namespace {

// One persistent host thread running one task at a time.
class Worker {
  public:
    Worker() : th_([this] { loop(); }) {}
    ~Worker() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        th_.join();
    }
    void run(std::function<void()> f) {
        {
            std::lock_guard<std::mutex> g(m_);
            task_ = std::move(f);
            done_ = false;
        }
        cv_.notify_all();
    }
    void wait() {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [this] { return done_; });
    }

  private:
    void loop() {
        std::unique_lock<std::mutex> l(m_);
        for (;;) {
            cv_.wait(l, [this] { return stop_ || task_; });
            if (stop_) return;
            auto f = std::move(task_);
            task_ = nullptr;
            l.unlock();
            f();
            l.lock();
            done_ = true;
            cv_.notify_all();
        }
    }
    std::mutex m_;
    std::condition_variable cv_;
    std::function<void()> task_;
    bool done_ = true, stop_ = false;
    std::thread th_;
};

// Workers by range index; one multi-device call at a time uses them.
std::mutex g_multi_m;
std::vector<std::unique_ptr<Worker>> g_workers;

aldp_status host_multi(const uint8_t* px, int n, int rows, int cols, int k, int cell_rows, int cell_cols,
                       uint8_t* codes, uint32_t* hist, const int* devices, int n_devices, bool lbp) {
    if (n < 0) return set_error(ALDP_EINVAL, "negative image count");
    if (rows < 3 || cols < 3)
        return set_error(ALDP_EINVAL, "descriptor extraction needs at least a 3x3 image, got " +
                                          std::to_string(rows) + "x" + std::to_string(cols));
    const int nbins = lbp ? 256 : aldp_n_bins(k);
    if (nbins == 0) return set_error(ALDP_EINVAL, "k must be in [1, 7]");
    const int64_t cells = aldp_grid_cells(rows, cols, cell_rows, cell_cols);
    if (cells < 0) return set_error(ALDP_EINVAL, "invalid window/cell size for this image");
    std::vector<int> devs;
    if (devices) {
        if (n_devices < 1) return set_error(ALDP_EINVAL, "n_devices must be >= 1");
        devs.assign(devices, devices + n_devices);
    } else {
        int count = 0;
        cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess) return set_error(ALDP_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
        for (int d = 0; d < count; ++d) devs.push_back(d);
    }
    if (devs.empty()) return set_error(ALDP_ECUDA, "no CUDA device");
    const int nd = int(devs.size());
    const size_t plane = size_t(rows) * cols, hist_per_img = size_t(cells) * nbins;

    std::lock_guard<std::mutex> g(g_multi_m);
    while (int(g_workers.size()) < nd) g_workers.emplace_back(new Worker());
    std::vector<aldp_status> st(nd, ALDP_OK);
    std::vector<std::string> msg(nd);
    for (int i = 0; i < nd; ++i) {
        const int lo = int(int64_t(n) * i / nd), hi = int(int64_t(n) * (i + 1) / nd);
        const int dev = devs[i];
        g_workers[i]->run([=, &st, &msg] {
            cudaError_t e = cudaSetDevice(dev);
            if (e != cudaSuccess) {
                st[i] = ALDP_ECUDA;
                msg[i] = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
                return;
            }
            const uint8_t* p = px + plane * lo;
            uint8_t* c = codes ? codes + plane * lo : nullptr;
            uint32_t* h = hist ? hist + hist_per_img * lo : nullptr;
            st[i] = lbp ? aldp_lbp_batch_host(p, hi - lo, rows, cols, cell_rows, cell_cols, c, h, nullptr)
                        : aldp_ldp_batch_host(p, hi - lo, rows, cols, k, cell_rows, cell_cols, c, h, nullptr);
            if (st[i] != ALDP_OK) msg[i] = aldp_last_error();
        });
    }
    for (int i = 0; i < nd; ++i) g_workers[i]->wait();
    for (int i = 0; i < nd; ++i)
        if (st[i] != ALDP_OK) return set_error(st[i], "device " + std::to_string(devs[i]) + ": " + msg[i]);
    return ALDP_OK;
}

}  // namespace
}  // namespace aldp_b200

using namespace aldp_b200;

extern "C" {

aldp_status aldp_ldp_batch_host_multi(const uint8_t* pixels, int n_images, int rows, int cols, int k,
                                      int cell_rows, int cell_cols, uint8_t* codes, uint32_t* hist,
                                      const int* devices, int n_devices) {
    return host_multi(pixels, n_images, rows, cols, k, cell_rows, cell_cols, codes, hist, devices, n_devices,
                      false);
}

aldp_status aldp_lbp_batch_host_multi(const uint8_t* pixels, int n_images, int rows, int cols, int cell_rows,
                                      int cell_cols, uint8_t* codes, uint32_t* hist, const int* devices,
                                      int n_devices) {
    return host_multi(pixels, n_images, rows, cols, 3, cell_rows, cell_cols, codes, hist, devices, n_devices,
                      true);
}

aldp_status aldp_ldp_batch_multi(const aldp_ldp_args* args, const int* devices, void* const* streams, int n) {
    if (n < 1 || !args || !devices) return set_error(ALDP_EINVAL, "aldp_ldp_batch_multi: need n >= 1 args and devices");
    int cur = 0;
    cudaError_t e = cudaGetDevice(&cur);
    if (e != cudaSuccess) return set_error(ALDP_ECUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
    aldp_status s = ALDP_OK;
    for (int i = 0; i < n && s == ALDP_OK; ++i) {
        e = cudaSetDevice(devices[i]);
        if (e != cudaSuccess) {
            s = set_error(ALDP_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
            break;
        }
        s = aldp_ldp_batch(&args[i], streams ? streams[i] : nullptr);
    }
    cudaSetDevice(cur);
    return s;
}

aldp_status aldp_gather_peer(void* dst, int dst_device, const void* const* srcs, const int* src_devices,
                             const size_t* bytes, int n, void* stream) {
    if (n < 0 || (n > 0 && (!dst || !srcs || !src_devices || !bytes)))
        return set_error(ALDP_EINVAL, "aldp_gather_peer: bad arguments");
    size_t off = 0;
    for (int i = 0; i < n; ++i) {
        cudaError_t e = cudaMemcpyPeerAsync(static_cast<uint8_t*>(dst) + off, dst_device, srcs[i], src_devices[i],
                                            bytes[i], static_cast<cudaStream_t>(stream));
        if (e != cudaSuccess)
            return set_error(ALDP_ECUDA, std::string("cudaMemcpyPeerAsync: ") + cudaGetErrorString(e));
        off += bytes[i];
    }
    return ALDP_OK;
}

}  // extern "C"
