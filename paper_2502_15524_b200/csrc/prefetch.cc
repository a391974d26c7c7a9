// prefetch.cc — the model prefetcher (§5.1 "Model Prefetching", lines 528-549) and
// the stream-side gate the loader uses to consume its output ("The worker
// performs model prefetching and loading in a pipelined fashion ... the first eight bytes ...
// store the address that represents the end of currently fetched model weights").
//
// B200 mapping: the prefetcher is a library thread that reads the model file (the host image's
// byte layout, include/hs.h: header first, like SafeTensors) into the caller's pinned region
// and publishes the fetched end in an 8-byte watermark in mapped pinned memory.  The loader does
// not poll it from a host thread: before every H2D chunk it enqueues cuStreamWaitValue64
// (watermark >= chunk end) on the copy stream, so the copy engine itself starts each chunk the
// moment its bytes are in host memory, and the compute stream gates a prefill's embedding-row
// reads from the host image the same way.
#include <fcntl.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <mutex>
#include <thread>

#include "common.h"

struct hs_prefetch {
  std::thread th;
  std::atomic<bool> stop{false};
  hs_status status = HS_OK;
  uint64_t fetched = 0;
  double seconds = 0;
  int fd = -1;
};

namespace hs {

using PFN_waitValue64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

static PFN_waitValue64 get_wait64() {
  static PFN_waitValue64 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_waitValue64>(p);
  });
  return fn;
}

// Enqueues "wait until *watermark >= value" on st (the watermark lives in mapped pinned memory).
hs_status stream_wait_watermark(cudaStream_t st, const uint64_t* watermark, uint64_t value) {
  if (!watermark) return HS_OK;
  auto fn = get_wait64();
  if (!fn) HS_FAIL(HS_E_CUDA, "cuStreamWaitValue64 unavailable");
  void* dp = nullptr;
  HS_CUDA(cudaHostGetDevicePointer(&dp, const_cast<uint64_t*>(watermark), 0));
  const CUresult r = fn(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(dp), (cuuint64_t)value,
                        CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) HS_FAIL(HS_E_CUDA, "cuStreamWaitValue64 failed (%d)", (int)r);
  return HS_OK;
}

}  // namespace hs

extern "C" hs_status hs_prefetch_start(const char* path, uint64_t file_offset, void* dst, uint64_t bytes,
                                       uint64_t chunk_bytes, double max_gbps, uint64_t* watermark, hs_prefetch** out) {
  if (!path || !dst || !watermark || !out) HS_FAIL(HS_E_INVAL, "null argument");
  const int fd = open(path, O_RDONLY);
  if (fd < 0) HS_FAIL(HS_E_INVAL, "cannot open %s", path);
  if (chunk_bytes == 0) chunk_bytes = 8ull << 20;
  hs_prefetch* p = new hs_prefetch();
  p->fd = fd;
  __atomic_store_n(watermark, file_offset, __ATOMIC_RELEASE);
  p->th = std::thread([=] {
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    uint8_t* d = static_cast<uint8_t*>(dst);
    uint64_t done = 0;
    while (done < bytes && !p->stop.load(std::memory_order_relaxed)) {
      const uint64_t n = std::min(chunk_bytes, bytes - done);
      uint64_t got = 0;
      while (got < n) {
        const ssize_t r = pread(fd, d + done + got, n - got, (off_t)(file_offset + done + got));
        if (r <= 0) {
          p->status = HS_E_INVAL;  // short file / read error: the watermark stops here
          p->fetched = done + got;
          p->seconds = std::chrono::duration<double>(clk::now() - t0).count();
          return;
        }
        got += (uint64_t)r;
      }
      done += n;
      if (max_gbps > 0) {  // emulate the remote-storage bandwidth (Eq. 1's b)
        const auto due = t0 + std::chrono::duration<double>((double)done / (max_gbps * 1e9));
        std::this_thread::sleep_until(due);
      }
      // release: the bytes above are visible before the watermark that covers them
      __atomic_store_n(watermark, file_offset + done, __ATOMIC_RELEASE);
    }
    p->fetched = done;
    p->seconds = std::chrono::duration<double>(clk::now() - t0).count();
  });
  *out = p;
  return HS_OK;
}

extern "C" hs_status hs_prefetch_wait(hs_prefetch* p, uint64_t* fetched, double* seconds) {
  if (!p) HS_FAIL(HS_E_INVAL, "null prefetcher");
  if (p->th.joinable()) p->th.join();
  if (fetched) *fetched = p->fetched;
  if (seconds) *seconds = p->seconds;
  if (p->status != HS_OK) HS_FAIL(p->status, "prefetch stopped at byte %llu (read error or short file)",
                                  (unsigned long long)p->fetched);
  return HS_OK;
}

extern "C" hs_status hs_prefetch_destroy(hs_prefetch* p) {
  if (!p) return HS_OK;
  p->stop = true;
  if (p->th.joinable()) p->th.join();
  if (p->fd >= 0) close(p->fd);
  delete p;
  return HS_OK;
}
