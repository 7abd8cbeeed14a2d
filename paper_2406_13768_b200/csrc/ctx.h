// Internal runtime context of libfastpersist (shared by runtime.cpp and
// load.cpp; not part of the C-ABI).
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdio>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "fp_internal.h"
#include "nvtx3/nvToolsExt.h"  // header-only NVTX v3 (no link; no-op without a tool)

namespace fp {


// NVTX range for nsys / ncu timelines (SURVEY §5 tracing)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

double now_s();
uint64_t env_u64(const char* k, uint64_t dflt);
std::string join_path(const std::string& a, const std::string& b);
int mkdirs(const std::string& path);
int fsync_dir(const std::string& dir);
std::string shard_file(int r, int k);

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "fastpersist: %s failed: %s\n", #x, cudaGetErrorString(e_));  \
      return FP_ECUDA;                                                               \
    }                                                                                \
  } while (0)

// GPUDirect Storage (gds.cpp): libcufile loaded at run time
class GdsPool;
int gds_available(bool* p2p);  // 0 or -ENOSYS; *p2p: NVMe P2P (not compat mode)
GdsPool* gds_pool_new(uint32_t threads, int device);
void gds_pool_delete(GdsPool* p);
int gds_buf_register(void* d, uint64_t bytes);
void gds_buf_deregister(void* d);
int gds_handle_open(int fd, void** fh);
void gds_handle_close(void* fh);
void gds_post(GdsPool* pool, bool write, void* fh, void* base, uint64_t buf_off,
              uint64_t file_off, uint64_t len, uint64_t piece);
int gds_wait(GdsPool* pool, double* stall);

}  // namespace fp

using fp::Extent;
using fp::IoEngine;
using fp::Item;
using fp::Plan;
using fp::TensorRef;

struct fp_ctx {
  fp_config cfg;
  std::string dirs_copy;
  std::vector<std::string> roots;
  int dev = -1;
  int numa_node = -1;  // NUMA node of the GPU (ring + helper placed there), -1 unknown
  fp_comm comm;
  bool has_comm = false;
  // resources
  uint8_t* ring = nullptr;
  uint8_t* d_ring = nullptr;  // device alias of the mapped ring (FP_PACK_HOST)
  size_t ring_bytes = 0;
  bool ring_cuda_registered = false;
  uint8_t* d_slab = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_producer = nullptr;
  std::vector<cudaEvent_t> ev_p0, ev_p1, ev_c1, ev_d0, ev_d2h;  // pack, CRC end, D2H
  std::vector<uint8_t> has_pack;  // per ring slot: its chunk led a pack launch
  // Host -> GPU signals live in one mapped pinned page, read on the GPU by
  // fp_wait_flag (a 1-warp kernel spinning with ld.acquire.sys; stream
  // memory operations, cuStreamWaitValue32, are disabled on some platforms —
  // the gpurun B200s report CAN_USE_STREAM_MEM_OPS = 0 and the wait never
  // releases).
  //  gate: the pack group's [event, kernel, event, crc] are queued behind a
  //  wait on `gate` that the host releases after the whole group is enqueued,
  //  so the events time the kernel, not the host API latency of an idle stream
  //  done: id of the checkpoint whose shard became durable (or failed), waited
  //  for on the caller's stream by fp_ckpt_fence
  // [0] gate, [16] done, [32] fence timeout
  volatile uint32_t* h_sig = nullptr;
  uint32_t* d_sig = nullptr;
  bool gate_on = false;
  uint32_t gate_seq = 0;
  uint32_t ckpt_seq = 0;
  // fault injection (tests): FP_FAULT_EIO_AT=<n>[@<rank>] turns the n-th write
  // completion of a checkpoint (of that rank, or any rank) into -EIO
  int64_t fault_eio_at = -1;
  int fault_rank = -1;
  // crash injection (tests): FP_FAULT_KILL_AT=<n>[@<rank>] SIGKILLs the
  // process at the n-th write completion of a checkpoint (a torn generation)
  int64_t fault_kill_at = -1;
  int fault_kill_rank = -1;
  // CRC-32 of the shard
  uint32_t* d_crc_tabs = nullptr;  // crc_device_tables() blob
  uint32_t* d_page_crc = nullptr;  // page CRCs of one pack group (device)
  uint32_t* h_pcrc = nullptr;      // pinned: page CRCs of each ring slot's chunk
  fp::ExtentCrc xcrc;              // this rank's shard, per extent, file order
  uint32_t ext_crc[2] = {0, 0};    // per-extent CRC-32 of the last checkpoint
  uint32_t n_ext_crc = 0;
  IoEngine* io = nullptr;
  int pack_ctas = 0;
  // GPUDirect Storage (FP_IO_GDS): writer pool, per-half events
  // [pack start, pack end, group done] x 2, pinned chunk CRCs of both halves
  bool gds = false, gds_p2p = false, gds_slab_registered = false;
  fp::GdsPool* gds_pool = nullptr;
  cudaEvent_t gds_ev[6] = {};
  uint32_t* h_gds_pcrc = nullptr;  // pinned page CRCs of both slab halves
  // plan cache
  bool planned = false;
  uint64_t sig_meta = 0, sig_ptr = 0;
  uint64_t items_key = 0;  // (sig_meta, sig_ptr) the uploaded work items belong to; 0 = stale
  Plan plan;
  std::vector<TensorRef> rep, loc;
  bool host = false;
  std::vector<Item> items;
  std::vector<uint32_t> item_lo;
  std::vector<Item> runs;          // FP_PACK_CE: items merged into contiguous runs
  std::vector<uint32_t> run_lo;
  Item* d_items = nullptr;
  size_t d_items_cap = 0;
  std::vector<uint32_t> tile_lo;          // fused pack + CRC: tiles of each pack group
  std::vector<uint64_t> group_tile_off;
  uint32_t* d_tiles = nullptr;
  size_t d_tiles_cap = 0;
  uint8_t* d_hdr = nullptr;
  size_t d_hdr_cap = 0;
  std::vector<uint8_t> h_hdr;
  std::vector<std::vector<Extent>> all_extents;
  // per rank, 3 words: whole shard, extent 0, extent 1 (bit 32 = valid,
  // low 32 = CRC-32)
  std::vector<uint64_t> shard_crcs;
  // request
  std::string shard_dir, manifest_dir;
  int rank = 0, k = 1;
  // helper thread
  std::thread th;
  std::mutex mu;
  std::condition_variable cv;
  enum State { IDLE, PENDING, RUNNING, DONE } state = IDLE;
  fp_load_stats ld{};  // of the last load on this context
  bool stop = false;
  int result = 0;
  fp_stats st;
  double t_begin = 0;

  int save_shard();
  int save_shard_gds(int fd);
  int finish_shard(int fd, int status, double t0);
  void helper();
  int write_manifest();
};

namespace fp {
// plan setup shared by save and load (runtime.cpp)
int ensure_plan(fp_ctx* c, const fp_tensor* t, size_t n, int rank, int k);
int build_items(fp_ctx* c, bool for_save);
void resolve_dirs(fp_ctx* c, const char* path, int rank);
}  // namespace fp
