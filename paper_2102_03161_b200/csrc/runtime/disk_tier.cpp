// AutoCache disk tier: the third level of the hierarchical store
// (reference: CacheTierSim, proj/src/autocache.cpp:69-150, parameters
// CacheTierParams autocache.hpp:11-20).  The reference *models* a disk tier
// holding every cached boundary activation and a host tier holding a sliding
// window of `window_batches` batches, refilled block by block
// (`block_batches` batches per prefetch) from disk while batches are consumed
// in order; a batch whose block has not arrived stalls the step.  This is the
// real thing for datasets whose boundary activations exceed host memory:
//
//   * a backing file of `rows` fixed-size rows (one cached sample each),
//     addressed by sample id; rows are padded to 4 KiB so reads and writes
//     can bypass the page cache (O_DIRECT, when the filesystem allows it);
//   * a page-locked host window of `window_blocks` block slots; block k of
//     the epoch holds batches [k*block_batches, (k+1)*block_batches) of the
//     epoch's consumption order, rows contiguous, so the device side copies
//     a batch with one 2D memcpy;
//   * a pool of I/O threads that fill slots in block order (pread per row:
//     the epoch order is a per-epoch shuffle, autodp.cpp:113-151, so rows
//     are scattered in the file), evicting a block once all its batches are
//     released and refilling the slot with the next block, like
//     CacheTierSim::advance / issue_prefetches;
//   * acquire(batch) blocks until the batch's block is resident and reports
//     the stall (the measured counterpart of WindowStep::stall_seconds).
//
// Host-side only: no kernels.  The buffer is registered with CUDA when a
// device is present (async H2D copies); the CPU tests drive it without one.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "eps_capi.h"

namespace {

constexpr int64_t kAlign = 4096;

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

struct DiskTier {
  int fd = -1;
  bool direct = false;
  bool registered = false;
  int64_t rows = 0, row_bytes = 0, stride = 0;  // stride: row_bytes padded to 4 KiB
  int64_t batch_rows = 0;
  int block_batches = 0, window_blocks = 0;
  uint8_t* window = nullptr;  // window_blocks slots of block_batches * batch_rows rows
  int64_t slot_bytes = 0;
  std::vector<std::thread> workers;

  std::mutex mu;
  std::condition_variable cv_work, cv_done;
  bool stop = false;
  // epoch state
  std::vector<int64_t> order;  // consumption order (sample ids)
  std::vector<int64_t> offs;   // batch b = order rows [offs[b], offs[b+1])
  int64_t n_batches = 0, n_blocks = 0;
  int64_t next_fetch = 0;      // next block to issue
  int64_t lowest = 0;          // lowest resident block
  std::deque<int64_t> queue;   // blocks waiting for a worker
  std::vector<char> ready;     // per block
  std::vector<char> released;  // per batch
  int error = 0;
  // stats
  double bytes_read = 0, bytes_written = 0, read_busy_s = 0, stall_s = 0;
  double max_resident = 0;
  int64_t prefetches = 0, evictions = 0;

  uint8_t* slot_ptr(int64_t block) { return window + (block % window_blocks) * slot_bytes; }
  int64_t block_of(int64_t batch) const { return batch / block_batches; }
  int64_t first_row(int64_t block) const { return offs[size_t(block * block_batches)]; }
  int64_t block_rows(int64_t block) const {
    const int64_t b1 = std::min<int64_t>((block + 1) * block_batches, n_batches);
    return offs[size_t(b1)] - first_row(block);
  }

  // called with mu held
  void issue() {
    while (next_fetch < n_blocks && next_fetch - lowest < window_blocks) {
      queue.push_back(next_fetch++);
      ++prefetches;
      max_resident = std::max(max_resident,
                              double(std::min<int64_t>(next_fetch - lowest, window_blocks)) *
                                  double(slot_bytes));
    }
    cv_work.notify_all();
  }

  int read_row(int64_t id, uint8_t* dst) {
    int64_t off = id * stride, done = 0;
    const int64_t want = direct ? stride : row_bytes;
    while (done < want) {
      const ssize_t r = pread(fd, dst + done, size_t(want - done), off + done);
      if (r < 0 && errno == EINTR) continue;
      if (r <= 0) return EPS_EIO;
      done += r;
    }
    return EPS_OK;
  }

  void worker() {
    for (;;) {
      int64_t block;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv_work.wait(lk, [&] { return stop || !queue.empty(); });
        if (stop) return;
        block = queue.front();
        queue.pop_front();
      }
      const double t0 = now_s();
      uint8_t* dst = slot_ptr(block);
      const int64_t r0 = first_row(block), nr = block_rows(block);
      int rc = EPS_OK;
      for (int64_t i = 0; i < nr && rc == EPS_OK; ++i)
        rc = read_row(order[size_t(r0 + i)], dst + i * stride);
      const double t1 = now_s();
      std::lock_guard<std::mutex> lk(mu);
      read_busy_s += t1 - t0;
      bytes_read += double(nr) * double(direct ? stride : row_bytes);
      if (rc != EPS_OK) error = rc;
      ready[size_t(block)] = 1;
      cv_done.notify_all();
    }
  }
};

}  // namespace

extern "C" {

int eps_disk_tier_open(const char* path, int64_t rows, int64_t row_bytes, int64_t batch_rows,
                       int block_batches, int window_batches, int threads, int create,
                       eps_disk_tier_t** out) {
  if (path == nullptr || out == nullptr || rows < 1 || row_bytes < 1 || batch_rows < 1 ||
      block_batches < 1 || window_batches < block_batches || threads < 1)
    return EPS_EINVAL;
  auto* t = new DiskTier();
  t->rows = rows;
  t->row_bytes = row_bytes;
  t->stride = (row_bytes + kAlign - 1) / kAlign * kAlign;
  t->batch_rows = batch_rows;
  t->block_batches = block_batches;
  t->window_blocks = window_batches / block_batches;  // CacheTierSim: window / block_batches
  t->slot_bytes = int64_t(block_batches) * batch_rows * t->stride;
  const int flags = O_RDWR | (create ? O_CREAT : 0);
  t->fd = open(path, flags | O_DIRECT, 0600);
  t->direct = t->fd >= 0;
  if (t->fd < 0) t->fd = open(path, flags, 0600);  // filesystem without O_DIRECT
  if (t->fd < 0) {
    delete t;
    return EPS_EIO;
  }
  if (create && ftruncate(t->fd, off_t(rows * t->stride)) != 0) {
    close(t->fd);
    delete t;
    return EPS_EIO;
  }
  const size_t wbytes = size_t(t->window_blocks) * size_t(t->slot_bytes);
  if (posix_memalign(reinterpret_cast<void**>(&t->window), kAlign, wbytes) != 0) {
    close(t->fd);
    delete t;
    return EPS_ECAPACITY;
  }
  int dev = 0;
  if (cudaGetDeviceCount(&dev) == cudaSuccess && dev > 0)
    t->registered = cudaHostRegister(t->window, wbytes, cudaHostRegisterPortable) == cudaSuccess;
  else
    cudaGetLastError();
  for (int i = 0; i < threads; ++i) t->workers.emplace_back([t] { t->worker(); });
  *out = reinterpret_cast<eps_disk_tier_t*>(t);
  return EPS_OK;
}

int eps_disk_tier_close(eps_disk_tier_t* h) {
  auto* t = reinterpret_cast<DiskTier*>(h);
  if (t == nullptr) return EPS_EINVAL;
  {
    std::lock_guard<std::mutex> lk(t->mu);
    t->stop = true;
  }
  t->cv_work.notify_all();
  for (auto& w : t->workers) w.join();
  if (t->registered) cudaHostUnregister(t->window);
  free(t->window);
  close(t->fd);
  delete t;
  return EPS_OK;
}

int eps_disk_tier_info(eps_disk_tier_t* h, int64_t* stride, int* direct, int* window_blocks,
                       void** window) {
  auto* t = reinterpret_cast<DiskTier*>(h);
  if (t == nullptr) return EPS_EINVAL;
  if (stride) *stride = t->stride;
  if (direct) *direct = t->direct ? 1 : 0;
  if (window_blocks) *window_blocks = t->window_blocks;
  if (window) *window = t->window;
  return EPS_OK;
}

int eps_disk_tier_write(eps_disk_tier_t* h, const int64_t* ids, int64_t n, const void* src,
                        int64_t src_stride) {
  auto* t = reinterpret_cast<DiskTier*>(h);
  if (t == nullptr || (n > 0 && (ids == nullptr || src == nullptr)) || src_stride < t->row_bytes)
    return EPS_EINVAL;
  for (int64_t i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= t->rows) return EPS_EINVAL;
  // rows go through a 4 KiB-aligned bounce buffer (O_DIRECT needs aligned
  // source, offset and size), written by the I/O thread count in parallel
  const int nt = int(std::min<int64_t>(int64_t(t->workers.size()), std::max<int64_t>(n, 1)));
  std::atomic<int64_t> next{0};
  std::atomic<int> err{EPS_OK};
  std::vector<std::thread> pool;
  for (int w = 0; w < nt; ++w)
    pool.emplace_back([&] {
      uint8_t* bounce = nullptr;
      if (posix_memalign(reinterpret_cast<void**>(&bounce), kAlign, size_t(t->stride)) != 0) {
        err = EPS_ECAPACITY;
        return;
      }
      std::memset(bounce, 0, size_t(t->stride));
      for (int64_t i = next++; i < n; i = next++) {
        std::memcpy(bounce, static_cast<const uint8_t*>(src) + i * src_stride, size_t(t->row_bytes));
        const int64_t want = t->direct ? t->stride : t->row_bytes;
        int64_t done = 0;
        while (done < want) {
          const ssize_t r = pwrite(t->fd, bounce + done, size_t(want - done),
                                   off_t(ids[i] * t->stride + done));
          if (r < 0 && errno == EINTR) continue;
          if (r <= 0) {
            err = EPS_EIO;
            break;
          }
          done += r;
        }
      }
      free(bounce);
    });
  for (auto& p : pool) p.join();
  std::lock_guard<std::mutex> lk(t->mu);
  t->bytes_written += double(n) * double(t->direct ? t->stride : t->row_bytes);
  return err.load();
}

int eps_disk_tier_begin_epoch(eps_disk_tier_t* h, const int64_t* order, int64_t n,
                              const int64_t* batch_offsets, int64_t n_batches) {
  auto* t = reinterpret_cast<DiskTier*>(h);
  if (t == nullptr || n < 0 || (n > 0 && order == nullptr)) return EPS_EINVAL;
  for (int64_t i = 0; i < n; ++i)
    if (order[i] < 0 || order[i] >= t->rows) return EPS_EINVAL;
  std::vector<int64_t> offs;
  if (batch_offsets != nullptr) {  // explicit batches (uneven replica shards)
    if (n_batches < 0 || batch_offsets[0] != 0 || batch_offsets[n_batches] != n) return EPS_EINVAL;
    for (int64_t b = 0; b < n_batches; ++b)
      if (batch_offsets[b + 1] <= batch_offsets[b] ||
          batch_offsets[b + 1] - batch_offsets[b] > t->batch_rows)
        return EPS_EINVAL;
    offs.assign(batch_offsets, batch_offsets + n_batches + 1);
  } else {  // batch_rows-row batches, the last one ragged
    for (int64_t r = 0; r < n; r += t->batch_rows) offs.push_back(r);
    offs.push_back(n);
  }
  std::unique_lock<std::mutex> lk(t->mu);
  // the previous epoch's reads must be finished before its order is replaced
  t->cv_done.wait(lk, [&] {
    for (int64_t b = t->lowest; b < t->next_fetch; ++b)
      if (!t->ready[size_t(b)]) return false;
    return true;
  });
  t->queue.clear();
  t->order.assign(order, order + n);
  t->offs = std::move(offs);
  t->n_batches = int64_t(t->offs.size()) - 1;
  t->n_blocks = (t->n_batches + t->block_batches - 1) / t->block_batches;
  t->next_fetch = t->lowest = 0;
  t->ready.assign(size_t(t->n_blocks), 0);
  t->released.assign(size_t(t->n_batches), 0);
  t->error = EPS_OK;
  t->issue();  // the leading window is staged before the first batch
  return EPS_OK;
}

int eps_disk_tier_acquire(eps_disk_tier_t* h, int64_t batch, const void** rows,
                          int64_t* n_rows, double* stall_s) {
  auto* t = reinterpret_cast<DiskTier*>(h);
  if (t == nullptr || rows == nullptr) return EPS_EINVAL;
  std::unique_lock<std::mutex> lk(t->mu);
  if (batch < 0 || batch >= t->n_batches) return EPS_EDOMAIN;
  const int64_t block = t->block_of(batch);
  if (block < t->lowest) return EPS_ELOGIC;  // already evicted
  if (block >= t->next_fetch) return EPS_ELOGIC;  // outside the window: release earlier batches
  const double t0 = now_s();
  t->cv_done.wait(lk, [&] { return t->ready[size_t(block)] != 0 || t->error != EPS_OK; });
  const double st = now_s() - t0;
  t->stall_s += st;
  if (stall_s) *stall_s = st;
  if (t->error != EPS_OK) return t->error;
  const int64_t r0 = t->offs[size_t(batch)];
  *rows = t->slot_ptr(block) + (r0 - t->first_row(block)) * t->stride;
  if (n_rows) *n_rows = t->offs[size_t(batch + 1)] - r0;
  return EPS_OK;
}

int eps_disk_tier_release(eps_disk_tier_t* h, int64_t batch) {
  auto* t = reinterpret_cast<DiskTier*>(h);
  if (t == nullptr) return EPS_EINVAL;
  std::lock_guard<std::mutex> lk(t->mu);
  if (batch < 0 || batch >= t->n_batches) return EPS_EDOMAIN;
  t->released[size_t(batch)] = 1;
  // evict leading blocks whose batches are all consumed, then refill
  while (t->lowest < t->n_blocks) {
    const int64_t b0 = t->lowest * t->block_batches;
    const int64_t b1 = std::min<int64_t>(b0 + t->block_batches, t->n_batches);
    bool done = t->ready[size_t(t->lowest)] != 0;
    for (int64_t b = b0; b < b1 && done; ++b) done = t->released[size_t(b)] != 0;
    if (!done) break;
    ++t->lowest;
    ++t->evictions;
  }
  t->issue();
  return EPS_OK;
}

// out[0] bytes read, [1] seconds the I/O threads spent reading, [2] stall
// seconds in acquire, [3] max resident window bytes, [4] prefetches,
// [5] evictions, [6] bytes written, [7] O_DIRECT (1) or buffered (0).
int eps_disk_tier_stats(eps_disk_tier_t* h, double* out) {
  auto* t = reinterpret_cast<DiskTier*>(h);
  if (t == nullptr || out == nullptr) return EPS_EINVAL;
  std::lock_guard<std::mutex> lk(t->mu);
  out[0] = t->bytes_read;
  out[1] = t->read_busy_s;
  out[2] = t->stall_s;
  out[3] = t->max_resident;
  out[4] = double(t->prefetches);
  out[5] = double(t->evictions);
  out[6] = t->bytes_written;
  out[7] = t->direct ? 1.0 : 0.0;
  return EPS_OK;
}

}  // extern "C"
