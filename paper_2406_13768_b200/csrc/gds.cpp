// GPUDirect Storage engine: pack kernel -> device slab ->
// cuFileWrite straight from HBM to the shard file, no pinned host ring.
//
// PAPER.md §4.1 P:473 stages through page-locked host memory because direct
// GPU<->NVMe DMA was "not yet broadly available"; cuFile (libcufile, shipped
// with CUDA) is that path today. With nvidia-fs and NVMe behind the GPU's PCIe
// switch the DMA is peer to peer; without them (the gpurun box: one virtio
// disk, no nvidia-fs) libcufile runs in its documented compatibility mode —
// its own pinned bounce buffers + POSIX I/O — and stats.fallback reports 2.
//
// Pipeline per rank: the device slab is doubled; pack group g+1 is enqueued
// into one half while the writer threads cuFileWrite group g from the other
// (cuFileWrite is synchronous, so a small pool of threads keeps several
// requests in flight). The GPU CRC-32 of each group is computed from the slab
// as in the ring path. libcufile is loaded with dlopen so the library builds
// and runs without it (FP_IO_GDS then fails with -ENOSYS at init).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cufile.h>
#include <dlfcn.h>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <condition_variable>
#include <memory>
#include <deque>
#include <mutex>
#include <thread>
#include <unistd.h>

#include "ctx.h"

namespace fp {

namespace {

struct CuFileApi {
  bool ok = false;
  bool p2p = false;  // the driver reports NVMe (P2P) support: not compat mode
  CUfileError_t (*DriverOpen)(void);
  CUfileError_t (*DriverGetProperties)(CUfileDrvProps_t*);
  CUfileError_t (*HandleRegister)(CUfileHandle_t*, CUfileDescr_t*);
  void (*HandleDeregister)(CUfileHandle_t);
  CUfileError_t (*BufRegister)(const void*, size_t, int);
  CUfileError_t (*BufDeregister)(const void*);
  ssize_t (*Write)(CUfileHandle_t, const void*, size_t, off_t, off_t);
  ssize_t (*Read)(CUfileHandle_t, void*, size_t, off_t, off_t);
};

CuFileApi g_api;
std::once_flag g_once;
bool g_dbg = getenv("FP_DEBUG_GDS") != nullptr;
#define GDS_DBG(...)                                  \
  do {                                                \
    if (g_dbg) {                                      \
      fprintf(stderr, "[fp gds %.6f] ", now_s());     \
      fprintf(stderr, __VA_ARGS__);                   \
      fputc('\n', stderr);                            \
    }                                                 \
  } while (0)

void load_api() {
  GDS_DBG("dlopen libcufile");
  void* h = dlopen("libcufile.so.0", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libcufile.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return;
  auto sym = [&](const char* n) { return dlsym(h, n); };
#define FP_SYM(field, name)                               \
  g_api.field = reinterpret_cast<decltype(g_api.field)>(sym(name)); \
  if (!g_api.field) return;
  FP_SYM(DriverOpen, "cuFileDriverOpen");
  FP_SYM(DriverGetProperties, "cuFileDriverGetProperties");
  FP_SYM(HandleRegister, "cuFileHandleRegister");
  FP_SYM(HandleDeregister, "cuFileHandleDeregister");
  FP_SYM(BufRegister, "cuFileBufRegister");
  FP_SYM(BufDeregister, "cuFileBufDeregister");
  FP_SYM(Write, "cuFileWrite");
  FP_SYM(Read, "cuFileRead");
#undef FP_SYM
  // Diagnosed on the gpurun B200 boxes (tools/diag/gds_hang_probe.sh,
  // rip_sample.c): libcufile's RDMA setup reads /proc/modules (looking for
  // nvidia_peermem) in a `while (!eof) getline` loop; a sandboxed procfs
  // without /proc/modules makes the open fail, the stream never reaches EOF
  // and cuFileDriverOpen spins forever. Fail fast there. (With the open
  // redirected to an empty file — an LD_PRELOAD shim, diagnosis only —
  // the driver opens in compatibility mode, and cuFileHandleRegister then
  // fails (5030) because those boxes have no udev database for the volume
  // holding the file.)
  if (access("/proc/modules", R_OK) != 0 && !getenv("FP_GDS_SKIP_PRECHECK")) {
    fprintf(stderr, "fastpersist: /proc/modules is not readable: libcufile's driver open "
                    "would spin forever; FP_IO_GDS unavailable\n");
    return;
  }
  // Any other hang: cuFileDriverOpen runs on a detached thread and is
  // abandoned after FP_GDS_OPEN_TIMEOUT seconds (default 20), which makes
  // FP_IO_GDS unavailable (-ENOSYS) instead of hanging the caller.
  GDS_DBG("cuFileDriverOpen");
  struct OpenState {
    std::mutex mu;
    std::condition_variable cv;
    bool done = false;
    CUfileError_t e;
  };
  auto os = std::make_shared<OpenState>();
  auto open_fn = g_api.DriverOpen;
  std::thread([os, open_fn] {
    CUfileError_t e = open_fn();
    std::lock_guard<std::mutex> g(os->mu);
    os->e = e;
    os->done = true;
    os->cv.notify_all();
  }).detach();
  const double tmo = (double)env_u64("FP_GDS_OPEN_TIMEOUT", 20);
  CUfileError_t e;
  {
    std::unique_lock<std::mutex> g(os->mu);
    if (!os->cv.wait_for(g, std::chrono::duration<double>(tmo), [&] { return os->done; })) {
      fprintf(stderr, "fastpersist: cuFileDriverOpen did not return within %.0f s "
                      "(no nvidia-fs / GDS on this host?); FP_IO_GDS unavailable\n", tmo);
      return;
    }
    e = os->e;
  }
  GDS_DBG("cuFileDriverOpen -> %d", (int)e.err);
  if (e.err != CU_FILE_SUCCESS) {
    fprintf(stderr, "fastpersist: cuFileDriverOpen failed (%d)\n", (int)e.err);
    return;
  }
  CUfileDrvProps_t props;
  memset(&props, 0, sizeof(props));
  if (g_api.DriverGetProperties(&props).err == CU_FILE_SUCCESS)
    g_api.p2p = (props.nvfs.dstatusflags & (1u << CU_FILE_NVME_SUPPORTED)) != 0;
  GDS_DBG("props: nvfs %u.%u dstatus 0x%x dcontrol 0x%x p2p %d", props.nvfs.major_version,
          props.nvfs.minor_version, props.nvfs.dstatusflags, props.nvfs.dcontrolflags, (int)g_api.p2p);
  g_api.ok = true;
}

}  // namespace

// A fixed pool of threads issuing synchronous cuFile calls (one outstanding
// request per thread).
class GdsPool {
 public:
  struct Job {
    bool write;
    CUfileHandle_t fh;
    void* base;
    uint64_t buf_off, file_off, len;
  };
  GdsPool(uint32_t n, int device) {
    for (uint32_t i = 0; i < std::max<uint32_t>(1, n); ++i)
      th_.emplace_back([this, device] {
        cudaSetDevice(device);  // libcufile stages through the calling thread's context
        run();
      });
  }
  ~GdsPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void post(const Job& j) {
    {
      std::lock_guard<std::mutex> g(mu_);
      q_.push_back(j);
      ++pending_;
    }
    cv_.notify_one();
  }
  // wait for every posted job; returns the first error (0, -errno or -EIO)
  int wait_all(double* stall) {
    const double t0 = now_s();
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return pending_ == 0; });
    if (stall) *stall += now_s() - t0;
    int e = err_;
    err_ = 0;
    return e;
  }

 private:
  void run() {
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || !q_.empty(); });
        if (q_.empty()) return;
        j = q_.front();
        q_.pop_front();
      }
      int e = 0;
      uint64_t done = 0;
      GDS_DBG("%s fo=%llu len=%llu", j.write ? "write" : "read", (unsigned long long)j.file_off,
              (unsigned long long)j.len);
      while (done < j.len && !e) {
        const ssize_t n = j.write ? g_api.Write(j.fh, j.base, j.len - done, (off_t)(j.file_off + done),
                                                (off_t)(j.buf_off + done))
                                  : g_api.Read(j.fh, j.base, j.len - done, (off_t)(j.file_off + done),
                                               (off_t)(j.buf_off + done));
        if (n < 0)
          e = n == -1 ? -errno : -EIO;  // -1: errno set; other negatives: CUfileOpError
        else if (n == 0)
          e = -EIO;
        else
          done += (uint64_t)n;
      }
      {
        std::lock_guard<std::mutex> g(mu_);
        if (e && !err_) err_ = e;
        --pending_;
      }
      done_cv_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::deque<Job> q_;
  uint64_t pending_ = 0;
  int err_ = 0;
  bool stop_ = false;
};

int gds_available(bool* p2p) {
  std::call_once(g_once, load_api);
  if (p2p) *p2p = g_api.p2p;
  return g_api.ok ? 0 : -ENOSYS;
}

GdsPool* gds_pool_new(uint32_t threads, int device) { return new GdsPool(threads, device); }
void gds_pool_delete(GdsPool* p) { delete p; }

int gds_buf_register(void* d, uint64_t bytes) {
  if (!g_api.ok) return -ENOSYS;
  GDS_DBG("cuFileBufRegister %p %llu", d, (unsigned long long)bytes);
  const int r = g_api.BufRegister(d, bytes, 0).err == CU_FILE_SUCCESS ? 0 : -EIO;
  GDS_DBG("cuFileBufRegister -> %d", r);
  return r;
}
void gds_buf_deregister(void* d) {
  if (g_api.ok) g_api.BufDeregister(d);
}

int gds_handle_open(int fd, void** fh_out) {
  if (!g_api.ok) return -ENOSYS;
  CUfileDescr_t d;
  memset(&d, 0, sizeof(d));
  d.type = CU_FILE_HANDLE_TYPE_OPAQUE_FD;
  d.handle.fd = fd;
  CUfileHandle_t fh = nullptr;
  GDS_DBG("cuFileHandleRegister fd=%d", fd);
  CUfileError_t e = g_api.HandleRegister(&fh, &d);
  GDS_DBG("cuFileHandleRegister -> %d", (int)e.err);
  if (e.err != CU_FILE_SUCCESS) {
    fprintf(stderr, "fastpersist: cuFileHandleRegister failed (%d)\n", (int)e.err);
    return -EIO;
  }
  *fh_out = fh;
  return 0;
}
void gds_handle_close(void* fh) {
  if (g_api.ok && fh) g_api.HandleDeregister((CUfileHandle_t)fh);
}

// Split [0, len) of base+buf_off into pieces of `piece` bytes for the pool.
void gds_post(GdsPool* pool, bool write, void* fh, void* base, uint64_t buf_off,
              uint64_t file_off, uint64_t len, uint64_t piece) {
  for (uint64_t o = 0; o < len; o += piece)
    pool->post({write, (CUfileHandle_t)fh, base, buf_off + o, file_off + o,
                std::min<uint64_t>(piece, len - o)});
}
int gds_wait(GdsPool* pool, double* stall) { return pool->wait_all(stall); }

}  // namespace fp

// ---------------------------------------------------------------------------
// save: pack groups double-buffered in the device slab, cuFileWrite each
// ---------------------------------------------------------------------------
int fp_ctx::save_shard_gds(int fd) {
  using namespace fp;
  void* fh = nullptr;
  int r = gds_handle_open(fd, &fh);
  if (r) return r;
  const uint64_t S = cfg.slot_bytes, P = cfg.pack_bytes;
  const uint64_t C = item_lo.size() - 1;       // chunks
  const uint64_t G = std::max<uint64_t>(1, P / S);  // chunks per group
  const uint64_t NG = (C + G - 1) / G;
  const bool want_crc = !(cfg.flags & FP_CFG_NO_CRC);
  const bool gpu_crc = want_crc && S % 4096 == 0 && d_crc_tabs;
  const uint64_t piece = std::max<uint64_t>(cfg.sqe_bytes, 4ull << 20);
  int status = 0;
  const uint64_t PPG = P / 4096 + 1;  // page CRC entries per slab half
  auto enqueue = [&](uint64_t g) -> int {
    const int h = (int)(g & 1);
    const uint64_t c0 = g * G, c1 = std::min<uint64_t>(c0 + G, C);
    const uint64_t gbytes = std::min<uint64_t>(c1 * S, plan.shard_bytes) - c0 * S;
    uint8_t* slab = d_slab + (size_t)h * P;
    if (g == 0) CK(cudaStreamWaitEvent(stream, ev_producer, 0));
    CK(cudaEventRecord(gds_ev[3 * h], stream));
    const bool bulk_crc = gpu_crc && cfg.pack_impl == FP_PACK_BULK && !group_tile_off.empty();
    const bool lsu_crc = gpu_crc && cfg.pack_impl == FP_PACK_LSU && !group_tile_off.empty();
    const bool fused = bulk_crc || lsu_crc;
    int rr = bulk_crc ? pack_bulk_crc_launch(d_items + item_lo[c0], d_tiles + group_tile_off[g],
                                             (uint32_t)((gbytes + kTile - 1) / kTile), gbytes,
                                             slab, d_crc_tabs, d_page_crc, pack_ctas, stream)
             : lsu_crc ? pack_lsu_crc_launch(d_items + item_lo[c0], d_tiles + group_tile_off[g],
                                             gbytes, slab, d_crc_tabs, d_page_crc, pack_ctas,
                                             stream)
             : pack_launch(cfg.pack_impl == FP_PACK_BULK ? FP_PACK_BULK : FP_PACK_V4,
                           d_items + item_lo[c0], item_lo[c1] - item_lo[c0], slab, pack_ctas,
                           stream);
    if (rr) return rr;
    CK(cudaEventRecord(gds_ev[3 * h + 1], stream));
    st.kernel_launches += 1;
    if (gpu_crc) {
      rr = fused ? 0 : crc_pages_launch(slab, round_up(gbytes, 4096), d_crc_tabs, d_page_crc, stream);
      if (rr) return rr;
      CK(cudaMemcpyAsync(h_gds_pcrc + (size_t)h * PPG, d_page_crc, round_up(gbytes, 4096) / 4096 * 4,
                         cudaMemcpyDeviceToHost, stream));
      st.kernel_launches += fused ? 0 : 1;
    }
    CK(cudaEventRecord(gds_ev[3 * h + 2], stream));
    ++st.pack_launches;
    st.pack_bytes += gbytes;
    return 0;
  };
  if (NG) status = enqueue(0);
  for (uint64_t g = 0; g < NG && !status; ++g) {
    const int h = (int)(g & 1);
    // the other half's previous group was written (wait_all below), so the
    // next pack may overwrite it while this group is on its way to storage
    if (g + 1 < NG) {
      status = enqueue(g + 1);
      if (status) break;
    }
    GDS_DBG("group %llu/%llu: wait pack", (unsigned long long)g, (unsigned long long)NG);
    if (cudaEventSynchronize(gds_ev[3 * h + 2]) != cudaSuccess) {
      status = FP_ECUDA;
      break;
    }
    float ms = 0;
    if (cudaEventElapsedTime(&ms, gds_ev[3 * h], gds_ev[3 * h + 1]) == cudaSuccess)
      st.pack_ms += ms;
    const uint64_t c0 = g * G, c1 = std::min<uint64_t>(c0 + G, C);
    const uint64_t gbytes = std::min<uint64_t>(c1 * S, plan.shard_bytes) - c0 * S;
    if (want_crc) {
      for (uint64_t c = c0; c < c1; ++c) {
        const uint64_t len = std::min<uint64_t>(S, plan.shard_bytes - c * S);
        if (gpu_crc && len % 4096 == 0 && xcrc.pages_ok(c * S, len)) {
          xcrc.add_pages(c * S, h_gds_pcrc + (size_t)h * PPG + (c - c0) * (S / 4096), len / 4096);
        } else {  // ragged last chunk (4 KiB-aligned shards never take this)
          std::vector<uint8_t> tmp(len);
          if (cudaMemcpy(tmp.data(), d_slab + (size_t)h * P + (c - c0) * S, len,
                         cudaMemcpyDeviceToHost) != cudaSuccess) {
            status = FP_ECUDA;
            break;
          }
          xcrc.add_bytes(c * S, tmp.data(), len);
        }
      }
      if (status) break;
    }
    gds_post(gds_pool, true, fh, d_slab, (uint64_t)h * P, c0 * S, gbytes, piece);
    st.io_requests += (gbytes + piece - 1) / piece;
    st.chunks += c1 - c0;
    status = gds_wait(gds_pool, &st.t_io_stall);
    GDS_DBG("group %llu written: %d", (unsigned long long)g, status);
  }
  cudaStreamSynchronize(stream);  // never leave a pack writing into the slab
  gds_handle_close(fh);
  return status;
}
