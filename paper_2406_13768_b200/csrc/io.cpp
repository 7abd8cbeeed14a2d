// Asynchronous NVMe I/O engines.
//
// PAPER.md §4.1: FastPersist "relies on newer I/O libraries (e.g., libaio
// and io_uring in Linux) that are designed with asynchronous and parallelism
// optimizations"; §5.1 P:535 extends DeepSpeed's AIO module to "multiple
// segment writes to increasing offset positions". This is an io_uring engine
// written against the raw syscalls (no liburing in this image): one SQ/CQ pair
// per rank, fixed (registered) pinned buffers -> IORING_OP_WRITE_FIXED,
// queue depth = fp_config.io_depth. The pwrite thread pool is the fallback
// when io_uring_setup is refused (seccomp) and the buffered variant is the
// page-cache path for file systems without O_DIRECT (reading R13).
#include <fcntl.h>
#include <linux/io_uring.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <sys/uio.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>

#include "fp_internal.h"

namespace fp {

// ---------------------------------------------------------------------------
// io_uring (raw syscalls)
// ---------------------------------------------------------------------------
static int sys_setup(unsigned entries, io_uring_params* p) {
  return (int)syscall(__NR_io_uring_setup, entries, p);
}
static int sys_enter(int fd, unsigned to_submit, unsigned min_complete, unsigned flags) {
  return (int)syscall(__NR_io_uring_enter, fd, to_submit, min_complete, flags, nullptr, 0);
}
static int sys_register(int fd, unsigned op, const void* arg, unsigned nr) {
  return (int)syscall(__NR_io_uring_register, fd, op, arg, nr);
}

class Uring final : public IoEngine {
 public:
  int init(uint32_t depth) {
    io_uring_params p;
    memset(&p, 0, sizeof(p));
    unsigned entries = 1;
    while (entries < depth) entries <<= 1;
    fd_ = sys_setup(entries, &p);
    if (fd_ < 0) return -errno;
    sq_entries_ = p.sq_entries;
    depth_ = std::min<uint32_t>(depth, p.sq_entries);
    sq_sz_ = p.sq_off.array + p.sq_entries * sizeof(unsigned);
    cq_sz_ = p.cq_off.cqes + p.cq_entries * sizeof(io_uring_cqe);
    single_ = (p.features & IORING_FEAT_SINGLE_MMAP) != 0;
    if (single_) sq_sz_ = cq_sz_ = std::max(sq_sz_, cq_sz_);
    sq_ptr_ = mmap(nullptr, sq_sz_, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd_,
                   IORING_OFF_SQ_RING);
    if (sq_ptr_ == MAP_FAILED) return -errno;
    cq_ptr_ = single_ ? sq_ptr_
                      : mmap(nullptr, cq_sz_, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE,
                             fd_, IORING_OFF_CQ_RING);
    if (cq_ptr_ == MAP_FAILED) return -errno;
    sqes_sz_ = p.sq_entries * sizeof(io_uring_sqe);
    sqes_ = (io_uring_sqe*)mmap(nullptr, sqes_sz_, PROT_READ | PROT_WRITE,
                                MAP_SHARED | MAP_POPULATE, fd_, IORING_OFF_SQES);
    if (sqes_ == MAP_FAILED) return -errno;
    char* sq = (char*)sq_ptr_;
    sq_head_ = (unsigned*)(sq + p.sq_off.head);
    sq_tail_ = (unsigned*)(sq + p.sq_off.tail);
    sq_mask_ = *(unsigned*)(sq + p.sq_off.ring_mask);
    sq_array_ = (unsigned*)(sq + p.sq_off.array);
    char* cq = (char*)cq_ptr_;
    cq_head_ = (unsigned*)(cq + p.cq_off.head);
    cq_tail_ = (unsigned*)(cq + p.cq_off.tail);
    cq_mask_ = *(unsigned*)(cq + p.cq_off.ring_mask);
    cqes_ = (io_uring_cqe*)(cq + p.cq_off.cqes);
    return 0;
  }
  ~Uring() override {
    if (sqes_ && sqes_ != MAP_FAILED) munmap(sqes_, sqes_sz_);
    if (cq_ptr_ && cq_ptr_ != MAP_FAILED && !single_) munmap(cq_ptr_, cq_sz_);
    if (sq_ptr_ && sq_ptr_ != MAP_FAILED) munmap(sq_ptr_, sq_sz_);
    if (fd_ >= 0) close(fd_);
  }
  int kind() const override { return FP_IO_URING; }
  uint32_t capacity() const override { return depth_; }

  int register_buffers(void* base, uint64_t slot_bytes, uint32_t slots) override {
    std::vector<iovec> iov(slots);
    for (uint32_t i = 0; i < slots; ++i) {
      iov[i].iov_base = (char*)base + i * slot_bytes;
      iov[i].iov_len = slot_bytes;
    }
    int r = sys_register(fd_, IORING_REGISTER_BUFFERS, iov.data(), slots);
    if (r < 0) return -errno;
    fixed_ = true;
    return 0;
  }

  int queue(bool write, int fd, void* buf, uint32_t len, uint64_t off, int buf_index,
            uint64_t user) override {
    const unsigned tail = *sq_tail_;
    const unsigned head = __atomic_load_n(sq_head_, __ATOMIC_ACQUIRE);
    if (tail - head >= sq_entries_) return -EAGAIN;
    const unsigned idx = tail & sq_mask_;
    io_uring_sqe* s = &sqes_[idx];
    memset(s, 0, sizeof(*s));
    const bool fixed = fixed_ && buf_index >= 0;
    s->opcode = write ? (fixed ? IORING_OP_WRITE_FIXED : IORING_OP_WRITE)
                      : (fixed ? IORING_OP_READ_FIXED : IORING_OP_READ);
    s->fd = fd;
    s->off = off;
    s->addr = (uint64_t)(uintptr_t)buf;
    s->len = len;
    if (fixed) s->buf_index = (uint16_t)buf_index;
    s->user_data = user;
    sq_array_[idx] = idx;
    __atomic_store_n(sq_tail_, tail + 1, __ATOMIC_RELEASE);
    ++pending_;
    return 0;
  }

  int submit() override {
    while (pending_) {
      int r = sys_enter(fd_, pending_, 0, 0);
      if (r < 0) {
        if (errno == EINTR || errno == EAGAIN) continue;
        return -errno;
      }
      pending_ -= (unsigned)r;
    }
    return 0;
  }

  int reap(IoDone* out, int max, int min_wait) override {
    int got = 0;
    for (;;) {
      unsigned head = *cq_head_;
      const unsigned tail = __atomic_load_n(cq_tail_, __ATOMIC_ACQUIRE);
      while (head != tail && got < max) {
        io_uring_cqe* c = &cqes_[head & cq_mask_];
        out[got].user = c->user_data;
        out[got].res = c->res;
        ++got;
        ++head;
      }
      __atomic_store_n(cq_head_, head, __ATOMIC_RELEASE);
      if (got >= min_wait || got >= max) return got;
      int r = sys_enter(fd_, 0, (unsigned)(min_wait - got), IORING_ENTER_GETEVENTS);
      if (r < 0 && errno != EINTR && errno != EAGAIN) return -errno;
    }
  }

  int fdatasync(int fd) override {
    // IORING_OP_FSYNC(DATASYNC) through the ring; the caller has drained
    // every write first, so no IOSQE_IO_DRAIN is needed.
    const unsigned tail = *sq_tail_;
    const unsigned idx = tail & sq_mask_;
    io_uring_sqe* s = &sqes_[idx];
    memset(s, 0, sizeof(*s));
    s->opcode = IORING_OP_FSYNC;
    s->fd = fd;
    s->fsync_flags = IORING_FSYNC_DATASYNC;
    s->user_data = ~0ull;
    sq_array_[idx] = idx;
    __atomic_store_n(sq_tail_, tail + 1, __ATOMIC_RELEASE);
    ++pending_;
    int r = submit();
    if (r) return r;
    IoDone d;
    for (;;) {
      int n = reap(&d, 1, 1);
      if (n < 0) return n;
      if (n == 1 && d.user == ~0ull) return d.res < 0 ? d.res : 0;
    }
  }

 private:
  int fd_ = -1;
  unsigned sq_entries_ = 0, depth_ = 0, pending_ = 0;
  size_t sq_sz_ = 0, cq_sz_ = 0, sqes_sz_ = 0;
  bool single_ = false, fixed_ = false;
  void *sq_ptr_ = nullptr, *cq_ptr_ = nullptr;
  io_uring_sqe* sqes_ = nullptr;
  unsigned *sq_head_, *sq_tail_, *sq_array_, sq_mask_ = 0;
  unsigned *cq_head_, *cq_tail_, cq_mask_ = 0;
  io_uring_cqe* cqes_ = nullptr;
};

IoEngine* make_uring(uint32_t depth, int* err) {
  Uring* u = new Uring();
  int r = u->init(depth);
  if (r) {
    delete u;
    *err = r;
    return nullptr;
  }
  *err = 0;
  return u;
}

// ---------------------------------------------------------------------------
// pwrite/pread thread pool (fallback engine)
// ---------------------------------------------------------------------------
class PwritePool final : public IoEngine {
 public:
  PwritePool(uint32_t threads, bool direct) : direct_(direct) {
    if (threads < 1) threads = 1;
    for (uint32_t i = 0; i < threads; ++i) workers_.emplace_back([this] { run(); });
    depth_ = threads * 2;
  }
  ~PwritePool() override {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  int kind() const override { return direct_ ? FP_IO_PWRITE : FP_IO_BUFFERED; }
  uint32_t capacity() const override { return depth_; }
  int queue(bool write, int fd, void* buf, uint32_t len, uint64_t off, int, uint64_t user) override {
    std::lock_guard<std::mutex> g(mu_);
    q_.push_back({write, fd, buf, len, off, user});
    return 0;
  }
  int submit() override {
    cv_.notify_all();
    return 0;
  }
  int reap(IoDone* out, int max, int min_wait) override {
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return (int)done_.size() >= std::min(min_wait, max) || min_wait == 0; });
    int got = 0;
    while (!done_.empty() && got < max) {
      out[got++] = done_.front();
      done_.pop_front();
    }
    return got;
  }
  int fdatasync(int fd) override { return ::fdatasync(fd) ? -errno : 0; }

 private:
  struct Req {
    bool write;
    int fd;
    void* buf;
    uint32_t len;
    uint64_t off;
    uint64_t user;
  };
  void run() {
    for (;;) {
      Req r;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || !q_.empty(); });
        if (stop_ && q_.empty()) return;
        r = q_.front();
        q_.pop_front();
      }
      uint64_t done = 0;
      int32_t res = 0;
      while (done < r.len) {
        ssize_t n = r.write ? pwrite(r.fd, (char*)r.buf + done, r.len - done, r.off + done)
                            : pread(r.fd, (char*)r.buf + done, r.len - done, r.off + done);
        if (n < 0) {
          if (errno == EINTR) continue;
          res = -errno;
          break;
        }
        if (n == 0) break;
        done += (uint64_t)n;
      }
      if (res == 0) res = (int32_t)done;
      {
        std::lock_guard<std::mutex> g(mu_);
        done_.push_back({r.user, res});
      }
      done_cv_.notify_all();
    }
  }
  bool direct_;
  uint32_t depth_ = 2;
  bool stop_ = false;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::deque<Req> q_;
  std::deque<IoDone> done_;
  std::vector<std::thread> workers_;
};

IoEngine* make_pwrite(uint32_t threads, bool direct) { return new PwritePool(threads, direct); }

// ---------------------------------------------------------------------------
// null sink (ablation): every request completes immediately with its full
// length; nothing reaches storage. Used to measure the GPU side of the path.
// ---------------------------------------------------------------------------
class NullSink final : public IoEngine {
 public:
  explicit NullSink(uint32_t depth) : depth_(depth) {}
  int kind() const override { return FP_IO_NULL; }
  uint32_t capacity() const override { return depth_; }
  int queue(bool, int, void*, uint32_t len, uint64_t, int, uint64_t user) override {
    done_.push_back({user, (int32_t)len});
    return 0;
  }
  int submit() override { return 0; }
  int reap(IoDone* out, int max, int) override {
    int got = 0;
    while (!done_.empty() && got < max) {
      out[got++] = done_.front();
      done_.pop_front();
    }
    return got;
  }
  int fdatasync(int) override { return 0; }

 private:
  uint32_t depth_;
  std::deque<IoDone> done_;
};

IoEngine* make_null(uint32_t depth) { return new NullSink(depth); }

}  // namespace fp
