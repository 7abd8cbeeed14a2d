// libfastpersist load paths: fp_ckpt_load (single box: every needed extent
// read from whichever shard holds it) and fp_ckpt_load_parallel (the paper's
// two-step load, §4.2: own partition + all-gather).
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>

#include <algorithm>
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <functional>

#include "ctx.h"

using namespace fp;

namespace {

// --------------------------------------------------------------------------
// minimal JSON reader for our own manifest (objects, arrays, ints, strings)
// --------------------------------------------------------------------------
struct JVal {
  enum T { NUL, NUM, STR, ARR, OBJ } t = NUL;
  unsigned long long num = 0;
  std::string str;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const char* k) const {
    for (auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct JParser {
  const char* p;
  const char* e;
  bool ok = true;
  void ws() {
    while (p < e && (*p == ' ' || *p == '\n' || *p == '\t' || *p == '\r')) ++p;
  }
  bool str(std::string* out) {
    if (p >= e || *p != '"') return ok = false;
    ++p;
    while (p < e && *p != '"') {
      if (*p == '\\' && p + 1 < e) ++p;
      out->push_back(*p++);
    }
    if (p >= e) return ok = false;
    ++p;
    return true;
  }
  JVal val() {
    JVal v;
    ws();
    if (p >= e) {
      ok = false;
      return v;
    }
    if (*p == '{') {
      v.t = JVal::OBJ;
      ++p;
      ws();
      if (p < e && *p == '}') {
        ++p;
        return v;
      }
      while (ok) {
        ws();
        std::string k;
        if (!str(&k)) break;
        ws();
        if (p >= e || *p != ':') {
          ok = false;
          break;
        }
        ++p;
        v.obj.push_back({k, val()});
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == '}') {
          ++p;
          break;
        }
        ok = false;
      }
    } else if (*p == '[') {
      v.t = JVal::ARR;
      ++p;
      ws();
      if (p < e && *p == ']') {
        ++p;
        return v;
      }
      while (ok) {
        v.arr.push_back(val());
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == ']') {
          ++p;
          break;
        }
        ok = false;
      }
    } else if (*p == '"') {
      v.t = JVal::STR;
      str(&v.str);
    } else {
      v.t = JVal::NUM;
      char* end = nullptr;
      v.num = strtoull(p, &end, 10);
      if (end == p) ok = false;
      p = end;
    }
    return v;
  }
};

// Loads plan with the writer's partition as the manifest records it: its
// writer subset (absent = 1) and its balance unit ("bytes" or pages).
struct PartitionScope {
  fp_ctx* c;
  uint32_t saved_ws, saved_flags;
  PartitionScope(fp_ctx* ctx, unsigned long long ws, bool bytes)
      : c(ctx), saved_ws(ctx->cfg.writer_stride), saved_flags(ctx->cfg.flags) {
    c->cfg.writer_stride = (ws == ~0ull || ws == 0) ? 1u : (uint32_t)ws;
    c->cfg.flags = bytes ? (c->cfg.flags | FP_CFG_BALANCE_BYTES)
                         : (c->cfg.flags & ~FP_CFG_BALANCE_BYTES);
  }
  ~PartitionScope() {
    c->cfg.writer_stride = saved_ws;
    c->cfg.flags = saved_flags;
  }
};
bool manifest_bytes_balance(const JVal& m) {
  const JVal* b = m.get("balance");
  return b && b->t == JVal::STR && b->str == "bytes";
}

// Read-ahead over the pinned ring (the load-side mirror of the save pipeline,
// §4.1 P:473 double buffering): chunk j's reads land in ring slot j % R and up
// to R chunks are in flight, so the NVMe queue does not drain while chunk j is
// copied to the GPU and scattered. A slot is refilled only after the consumer
// released the chunk that used it and, on the device path, after the H2D copy
// out of it (the event the consumer recorded) has completed.
struct ReadReq {
  int fd;
  uint64_t file_off;
  uint64_t buf_off;  // inside the slot
  uint32_t len;
};

class ReadAhead {
 public:
  using ReqFn = std::function<int(uint64_t chunk, std::vector<ReadReq>* out)>;
  ReadAhead(fp_ctx* c, uint64_t n_chunks, bool dev_events, ReqFn fn)
      : c_(c), n_(n_chunks), R_(c->cfg.ring_slots), dev_(dev_events), fn_(std::move(fn)),
        outstanding_(R_, 0) {}
  ~ReadAhead() { drain(); }

  uint8_t* slot_of(uint64_t j) const { return c_->ring + (size_t)(j % R_) * c_->cfg.slot_bytes; }

  // Block until every read of chunk j has completed; 0 or the first error.
  int wait(uint64_t j) {
    for (;;) {
      issue(false);
      if (status_) return status_;
      // slot j % R holds chunk j only (issue() stays below released_ + R)
      if (next_ > j && outstanding_[j % R_] == 0) return 0;
      if (inflight_ > 0) {
        int r = pump(1);
        if (r && !status_) status_ = r;
        continue;
      }
      // nothing in flight and chunk j not fully queued: its slot is still
      // being copied to the GPU; wait for that copy
      issue(true);
      if (!status_ && inflight_ == 0 && next_ <= j) status_ = -EIO;  // no progress possible
    }
  }
  // The consumer is done with chunk j (its slot may be refilled once the
  // device has finished reading it: ev_d2h[slot], recorded by the consumer).
  void release(uint64_t j) { released_ = j + 1; }
  void finish() { drain(); }
  int status() const { return status_; }

 private:
  // queue requests of chunks [next_, released_ + R) while the engine has room
  void issue(bool block_on_slot) {
    while (next_ < n_ && next_ < released_ + R_ && !status_) {
      const uint32_t s = (uint32_t)(next_ % R_);
      if (cur_.empty() && pos_ == 0) {
        if (outstanding_[s]) return;  // previous user of the slot still reading
        if (dev_ && next_ >= R_) {
          cudaEvent_t e = c_->ev_d2h[s];
          cudaError_t q = cudaEventQuery(e);
          if (q == cudaErrorNotReady) {
            if (!block_on_slot) return;
            q = cudaEventSynchronize(e);
          }
          if (q != cudaSuccess) {
            status_ = FP_ECUDA;
            return;
          }
        }
        int r = fn_(next_, &cur_);
        if (r) {
          status_ = r;
          return;
        }
        if (cur_.empty()) {  // nothing to read for this chunk
          ++next_;
          continue;
        }
      }
      while (pos_ < cur_.size()) {
        if (inflight_ >= c_->io->capacity()) {
          c_->io->submit();
          return;
        }
        const ReadReq& q = cur_[pos_];
        const uint64_t user = ((uint64_t)s << 56) | q.len;
        int r = c_->io->queue(false, q.fd, slot_of(next_) + q.buf_off, q.len, q.file_off, (int)s,
                              user);
        if (r == -EAGAIN) {
          c_->io->submit();
          return;
        }
        if (r) {
          status_ = r;
          return;
        }
        ++outstanding_[s];
        ++inflight_;
        ++pos_;
      }
      cur_.clear();
      pos_ = 0;
      ++next_;
      block_on_slot = false;
    }
    int r = c_->io->submit();
    if (r && !status_) status_ = r;
  }
  int pump(int min_wait) {
    int r = c_->io->submit();
    if (r) return r;
    IoDone done[64];
    int n = c_->io->reap(done, 64, min_wait);
    if (n < 0) return n;
    for (int i = 0; i < n; ++i) {
      const uint32_t s = (uint32_t)(done[i].user >> 56);
      const int64_t want = (int64_t)(done[i].user & 0xFFFFFFFFull);
      if (done[i].res != want && !status_) status_ = done[i].res < 0 ? done[i].res : -EIO;
      --outstanding_[s];
      --inflight_;
    }
    return 0;
  }
  void drain() {
    while (inflight_ > 0)
      if (pump(1)) break;
  }

  fp_ctx* c_;
  uint64_t n_;
  uint32_t R_;
  bool dev_;
  ReqFn fn_;
  std::vector<uint32_t> outstanding_;
  uint64_t next_ = 0, released_ = 0;
  std::vector<ReadReq> cur_;
  size_t pos_ = 0;
  uint32_t inflight_ = 0;
  int status_ = 0;
};

// Page CRCs of the chunks a load copies to the device (fp_crc_pages over the
// H2D'd bytes), folded on the host in chunk order: chunk j's page
// CRCs land in the pinned slot j % R of ctx->h_pcrc; that slot's previous
// chunk (j - R, the oldest one pending) is folded first. A chunk that cannot
// be folded as pages (ragged, or an extent boundary inside a page) is folded
// from the host bytes by the caller after flush().
class LoadCrc {
 public:
  using FoldFn = std::function<void(uint64_t chunk, const uint32_t* pages)>;
  LoadCrc(fp_ctx* c, FoldFn fn)
      : c_(c), R_(c->cfg.ring_slots), pps_(std::max<uint64_t>(1, c->cfg.slot_bytes / 4096)),
        fn_(std::move(fn)), pend_(R_, -1) {}
  // page CRCs of d_buf[0, len) (len % 4096 == 0) for chunk j, on stream st
  int enqueue(uint64_t j, const uint8_t* d_buf, uint64_t len, cudaStream_t st) {
    const uint32_t s = (uint32_t)(j % R_);
    int r = fold_slot(s);
    if (r) return r;
    if (crc_pages_launch(d_buf, len, c_->d_crc_tabs, c_->d_page_crc, st) ||
        cudaMemcpyAsync(c_->h_pcrc + s * pps_, c_->d_page_crc, len / 4096 * 4,
                        cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaEventRecord(c_->ev_c1[s], st) != cudaSuccess)
      return FP_ECUDA;
    pend_[s] = (int64_t)j;
    ++launches_;
    return 0;
  }
  // fold every pending chunk, oldest first
  int flush() {
    for (;;) {
      int64_t best = -1;
      uint32_t bs = 0;
      for (uint32_t s = 0; s < R_; ++s)
        if (pend_[s] >= 0 && (best < 0 || pend_[s] < best)) best = pend_[s], bs = s;
      if (best < 0) return 0;
      int r = fold_slot(bs);
      if (r) return r;
    }
  }
  uint64_t launches() const { return launches_; }

 private:
  int fold_slot(uint32_t s) {
    if (pend_[s] < 0) return 0;
    if (cudaEventSynchronize(c_->ev_c1[s]) != cudaSuccess) return FP_ECUDA;
    fn_((uint64_t)pend_[s], c_->h_pcrc + s * pps_);
    pend_[s] = -1;
    return 0;
  }
  fp_ctx* c_;
  uint32_t R_;
  uint64_t pps_;
  FoldFn fn_;
  std::vector<int64_t> pend_;
  uint64_t launches_ = 0;
};

// manifest CRC records of shard w: "crc32" (whole file) and "extent_crc32"
struct ShardCrcRec {
  bool has_file = false;
  uint32_t file = 0;
  std::vector<int64_t> ext;  // -1 = absent
};
ShardCrcRec crc_record(const JVal& m, int w, size_t n_ext) {
  ShardCrcRec r;
  r.ext.assign(n_ext, -1);
  const JVal* sh = m.get("shards");
  if (!sh || sh->t != JVal::ARR || (size_t)w >= sh->arr.size()) return r;
  const JVal& rec = sh->arr[w];
  if (const JVal* f = rec.get("crc32"))
    if (f->t == JVal::NUM) r.has_file = true, r.file = (uint32_t)f->num;
  if (const JVal* e = rec.get("extent_crc32"))
    if (e->t == JVal::ARR && e->arr.size() == n_ext)
      for (size_t i = 0; i < n_ext; ++i)
        if (e->arr[i].t == JVal::NUM) r.ext[i] = (int64_t)(uint32_t)e->arr[i].num;
  return r;
}

// Compare what was read of shard `name` with its manifest record: every
// extent read whole against its extent CRC, the whole file against "crc32".
// Returns 0 or FP_ECORRUPT (naming the shard and extent on stderr).
int verify_crc(const ExtentCrc& acc, const ShardCrcRec& rec, const std::string& name) {
  if (!acc.ok()) {
    fprintf(stderr, "fastpersist: %s: CRC runs out of order (internal error)\n", name.c_str());
    return FP_ECORRUPT;
  }
  for (size_t i = 0; i < acc.n(); ++i) {
    if (!acc.complete(i) || rec.ext[i] < 0) continue;
    const uint32_t got = acc.extent_crc(i);
    if (got != (uint32_t)rec.ext[i]) {
      fprintf(stderr, "fastpersist: %s extent %zu CRC-32 %08x != manifest %08x (corrupt data)\n",
              name.c_str(), i, got, (unsigned)rec.ext[i]);
      return FP_ECORRUPT;
    }
  }
  if (rec.has_file && acc.complete() && acc.file_crc() != rec.file) {
    fprintf(stderr, "fastpersist: %s CRC-32 %08x != manifest %08x (corrupt data)\n", name.c_str(),
            acc.file_crc(), rec.file);
    return FP_ECORRUPT;
  }
  return 0;
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------------------
// load: manifest -> header check -> O_DIRECT reads -> H2D -> unpack kernel
// ---------------------------------------------------------------------------
static int read_file(const std::string& path, std::string* out) {
  int fd = open(path.c_str(), O_RDONLY);
  if (fd < 0) return -errno;
  char buf[65536];
  for (;;) {
    ssize_t n = read(fd, buf, sizeof(buf));
    if (n < 0) {
      if (errno == EINTR) continue;
      int e = -errno;
      close(fd);
      return e;
    }
    if (n == 0) break;
    out->append(buf, (size_t)n);
  }
  close(fd);
  return 0;
}

static int pread_all(int fd, void* buf, uint64_t len, uint64_t off) {
  uint64_t done = 0;
  while (done < len) {
    ssize_t n = pread(fd, (char*)buf + done, len - done, (off_t)(off + done));
    if (n < 0) {
      if (errno == EINTR) continue;
      return -errno;
    }
    if (n == 0) return -EIO;
    done += (uint64_t)n;
  }
  return 0;
}

int fp_ckpt_load(fp_ctx* c, const fp_tensor* t, size_t n, const char* path, int dp_rank,
                 int dp_size, void* stream) {
  NvtxRange nv("fp.load");
  if (c) memset(&c->ld, 0, sizeof(c->ld));
  const double t_call = now_s();
  if (!c || (!t && n) || !path || dp_size < 1 || dp_rank < 0 || dp_rank >= dp_size)
    return -EINVAL;
  if (dp_size > 1 && !c->has_comm) return -EINVAL;
  if (c->cfg.io_engine == FP_IO_NULL) return -EINVAL;  // nothing was ever written
  {
    std::lock_guard<std::mutex> g(c->mu);
    if (c->state != fp_ctx::IDLE) return -EBUSY;
  }
  resolve_dirs(c, path, dp_rank);
  const std::string mpath = join_path(c->manifest_dir, "manifest.json");
  std::string mtxt;
  int r = read_file(mpath, &mtxt);
  if (r) {
    fprintf(stderr, "fastpersist: cannot read %s: %s\n", mpath.c_str(), strerror(-r));
    return r;
  }
  JParser jp{mtxt.data(), mtxt.data() + mtxt.size()};
  JVal m = jp.val();
  if (!jp.ok || m.t != JVal::OBJ) return FP_ECORRUPT;
  auto num = [&](const char* k) -> uint64_t {
    const JVal* v = m.get(k);
    return v && v->t == JVal::NUM ? v->num : ~0ull;
  };
  if (num("dp_size") != (uint64_t)dp_size || num("alignment") != c->cfg.alignment)
    return FP_EMISMATCH;
  // the partition is the writer's (its writer subset), not this context's
  PartitionScope wss(c, num("writer_stride"), manifest_bytes_balance(m));
  r = ensure_plan(c, t, n, dp_rank, dp_size);
  if (r) return r;
  Plan& p = c->plan;
  if (num("image_bytes") != p.image_bytes || num("layout_digest") != p.digest)
    return FP_EMISMATCH;
  const JVal* shards = m.get("shards");
  if (!shards || shards->t != JVal::ARR || (int)shards->arr.size() != dp_size) return FP_ECORRUPT;
  // open every shard we may read from (single box: all files visible; the
  // NCCL all-gather variant of P:503 reads only its own shard)
  const size_t nroots = c->roots.empty() ? 1 : c->roots.size();
  std::vector<int> fds(dp_size, -1), bfds(dp_size, -1);
  auto close_all = [&] {
    for (int fd : fds)
      if (fd >= 0) close(fd);
    for (int fd : bfds)
      if (fd >= 0) close(fd);
  };
  for (int w = 0; w < dp_size; ++w) {
    const std::string dir =
        c->roots.empty() ? std::string(path) : join_path(c->roots[w % nroots], path);
    const std::string f = join_path(dir, shard_file(w, dp_size));
    int fd = open(f.c_str(), O_RDONLY | O_DIRECT);
    if (fd < 0 && errno == EINVAL) fd = open(f.c_str(), O_RDONLY);
    if (fd < 0) {
      r = -errno;
      fprintf(stderr, "fastpersist: missing shard %s: %s\n", f.c_str(), strerror(errno));
      close_all();
      return r;
    }
    struct stat sb;
    uint64_t want = 0;
    for (auto& e : c->all_extents[w]) want += e.len;
    if (fstat(fd, &sb) || (uint64_t)sb.st_size != want) {
      fprintf(stderr, "fastpersist: shard %s has %lld bytes, expected %llu\n", f.c_str(),
              (long long)sb.st_size, (unsigned long long)want);
      fds[w] = fd;
      close_all();
      return FP_ECORRUPT;
    }
    fds[w] = fd;
    // requests that are not block-aligned (byte-granular partitions: shard
    // suffixes and unaligned local-region starts) take a buffered descriptor
    bfds[w] = open(f.c_str(), O_RDONLY);
    if (bfds[w] < 0) {
      r = -errno;
      close_all();
      return r;
    }
  }
  // image offset -> (shard, file offset) for the bytes this rank needs
  const uint32_t A = p.align;
  auto locate = [&](uint64_t io, int* w_out, uint64_t* fo, uint64_t* avail) -> bool {
    for (int w = 0; w < dp_size; ++w)
      for (auto& e : c->all_extents[w])
        if (io >= e.image_off && io < e.image_off + e.len) {
          *w_out = w;
          *fo = e.file_off + (io - e.image_off);
          *avail = e.image_off + e.len - io;
          return true;
        }
    return false;
  };
  // 1) header check: GHDR and our LREG header must match the target list
  {
    std::vector<std::pair<uint64_t, const std::vector<uint8_t>*>> hdrs = {{0, &p.ghdr.bytes}};
    if (!p.regions.empty()) hdrs.push_back({p.regions[dp_rank].first, &p.lhdr.bytes});
    for (auto& h : hdrs) {
      std::vector<uint8_t> tmp;
      uint64_t got = 0;
      while (got < h.second->size()) {
        int w;
        uint64_t fo, avail;
        if (!locate(h.first + got, &w, &fo, &avail)) {
          close_all();
          return FP_ECORRUPT;
        }
        const uint64_t nn = std::min<uint64_t>(avail, h.second->size() - got);
        // bounce through an aligned buffer for O_DIRECT
        const uint64_t span = round_up(nn, A);
        void* bb = nullptr;
        if (posix_memalign(&bb, A, span)) {
          close_all();
          return -ENOMEM;
        }
        int fd2 = open(join_path(c->roots.empty() ? std::string(path)
                                                  : join_path(c->roots[w % nroots], path),
                                 shard_file(w, dp_size))
                           .c_str(),
                       O_RDONLY);
        r = fd2 < 0 ? -errno : pread_all(fd2, bb, nn, fo);
        if (fd2 >= 0) close(fd2);
        if (r) {
          free(bb);
          close_all();
          return r;
        }
        tmp.insert(tmp.end(), (uint8_t*)bb, (uint8_t*)bb + nn);
        free(bb);
        got += nn;
      }
      if (memcmp(tmp.data(), h.second->data(), tmp.size())) {
        fprintf(stderr, "fastpersist: header at image offset %llu does not match the target "
                        "tensors (corrupt or different state)\n",
                (unsigned long long)h.first);
        close_all();
        return FP_ECORRUPT;
      }
    }
  }
  // 2) load stream = replicated region, then our local region
  Plan lp = p;
  lp.extents.clear();
  lp.extents.push_back({0, 0, p.rep_bytes});
  uint64_t total = p.rep_bytes;
  if (!p.regions.empty()) {
    lp.extents.push_back({p.regions[dp_rank].first, total, p.regions[dp_rank].second});
    total += p.regions[dp_rank].second;
  }
  lp.shard_bytes = total;
  plan_pieces(&lp, c->rep, c->loc, 0);  // header pieces -> skip items
  std::vector<Item> items;
  std::vector<uint32_t> lo;
  plan_items(lp, c->cfg.slot_bytes, c->cfg.slot_bytes, &items, &lo);
  Item* d_items = nullptr;
  if (!c->host && !items.empty()) {
    if (cudaMalloc(&d_items, items.size() * sizeof(Item)) != cudaSuccess ||
        cudaMemcpy(d_items, items.data(), items.size() * sizeof(Item), cudaMemcpyHostToDevice) !=
            cudaSuccess) {
      if (d_items) cudaFree(d_items);
      close_all();
      return FP_ECUDA;
    }
  }
  const uint64_t S = c->cfg.slot_bytes, SQ = c->cfg.sqe_bytes;
  const uint64_t C = lo.size() - 1;
  cudaStream_t st = (cudaStream_t)stream;
  int status = 0;
  // load-stream chunk ch -> runs {offset in chunk, shard, file offset, bytes},
  // cut wherever the source shard or extent changes
  struct Run {
    uint64_t pos;
    int w;
    uint64_t fo, n;
  };
  auto chunk_runs = [&](uint64_t ch, std::vector<Run>* out) -> int {
    out->clear();
    const uint64_t len = std::min<uint64_t>(S, total - ch * S);
    for (uint64_t pos = 0; pos < len;) {
      const uint64_t ls = ch * S + pos;  // load-stream offset -> image offset
      uint64_t io = 0, lavail = 0;
      for (auto& e : lp.extents)
        if (ls >= e.file_off && ls < e.file_off + e.len) {
          io = e.image_off + (ls - e.file_off);
          lavail = e.file_off + e.len - ls;
        }
      int w;
      uint64_t fo, avail;
      if (!lavail || !locate(io, &w, &fo, &avail)) return FP_ECORRUPT;
      const uint64_t nn = std::min<uint64_t>({len - pos, avail, lavail});
      out->push_back({pos, w, fo, nn});
      pos += nn;
    }
    return 0;
  };
  // integrity: every extent read whole is checked against the
  // manifest's per-extent CRC-32 (page CRCs of each H2D'd chunk on the GPU,
  // folded per shard extent on the host)
  const bool want_crc = !(c->cfg.flags & FP_CFG_NO_CRC);
  std::vector<ExtentCrc> acc(dp_size);
  std::vector<ShardCrcRec> recs(dp_size);
  for (int w = 0; w < dp_size; ++w) {
    acc[w].reset(c->all_extents[w]);
    recs[w] = crc_record(m, w, c->all_extents[w].size());
  }
  std::vector<Run> fold_runs;
  LoadCrc lcrc(c, [&](uint64_t ch, const uint32_t* pages) {
    if (chunk_runs(ch, &fold_runs)) return;
    for (const Run& u : fold_runs) acc[u.w].add_pages(u.fo, pages + u.pos / 4096, u.n / 4096);
  });
  {
    // chunk ch = [ch*S, ch*S+len) of the load stream, read from whichever
    // shard holds each piece, R chunks ahead of the GPU scatter
    std::vector<Run> rr;
    ReadAhead ra(c, C, !c->host, [&](uint64_t ch, std::vector<ReadReq>* out) -> int {
      int e = chunk_runs(ch, &rr);
      if (e) return e;
      for (const Run& u : rr)
        for (uint64_t o = 0; o < u.n; o += SQ) {
          const uint32_t len = (uint32_t)std::min<uint64_t>(SQ, u.n - o);
          const bool aligned = (u.fo + o) % A == 0 && len % A == 0 && (u.pos + o) % A == 0;
          out->push_back({aligned ? fds[u.w] : bfds[u.w], u.fo + o, u.pos + o, len});
        }
      return 0;
    });
    std::vector<Run> cr;
    for (uint64_t ch = 0; ch < C && !status; ++ch) {
      const uint32_t s = (uint32_t)(ch % c->cfg.ring_slots);
      const uint64_t len = std::min<uint64_t>(S, total - ch * S);
      status = ra.wait(ch);
      if (status) break;
      const uint8_t* slot = ra.slot_of(ch);
      bool pages = false;
      if (want_crc) {
        status = chunk_runs(ch, &cr);
        if (status) break;
        pages = !c->host && c->d_crc_tabs && len % 4096 == 0;
        for (const Run& u : cr)
          pages = pages && u.pos % 4096 == 0 && u.n % 4096 == 0 && acc[u.w].pages_ok(u.fo, u.n);
        if (!pages) {  // host bytes, in order behind every pending page fold
          status = lcrc.flush();
          for (const Run& u : cr) acc[u.w].add_bytes(u.fo, slot + u.pos, u.n);
        }
      }
      if (c->host) {
        for (uint32_t i = lo[ch]; i < lo[ch + 1]; ++i)
          if (items[i].src)
            memcpy((void*)(uintptr_t)items[i].src, slot + items[i].dst, items[i].len);
      } else if (cudaMemcpyAsync(c->d_slab, slot, len, cudaMemcpyHostToDevice, st) != cudaSuccess ||
                 cudaEventRecord(c->ev_d2h[s], st) != cudaSuccess ||
                 (pages && lcrc.enqueue(ch, c->d_slab, len, st)) ||
                 unpack_launch(d_items + lo[ch], lo[ch + 1] - lo[ch], c->d_slab, c->pack_ctas,
                               st)) {
        status = FP_ECUDA;
      }
      ra.release(ch);
    }
  }  // ~ReadAhead drains reads still in flight (error paths)
  if (!c->host && cudaStreamSynchronize(st) != cudaSuccess && !status) status = FP_ECUDA;
  if (!status) status = lcrc.flush();
  for (int w = 0; w < dp_size && !status && want_crc; ++w)
    status = verify_crc(acc[w], recs[w], shard_file(w, dp_size));
  c->ld.bytes_read = total;
  c->ld.kernel_launches = C * (c->host ? 0 : 1) + lcrc.launches();
  c->ld.status = status;
  c->ld.t_total = now_s() - t_call;
  if (d_items) cudaFree(d_items);
  close_all();
  return status;
}

// ---------------------------------------------------------------------------
// parallel load: own shard only + one all-gather per chunk + unpack
// ---------------------------------------------------------------------------

static int status_min(fp_ctx* c, int k, int s) {
  if (k <= 1) return s;
  int32_t v = s;
  if (c->comm.allreduce_min_i32(c->comm.ctx, &v)) return s ? s : FP_ECOMM;
  return v;
}

// Items scattering image range [io0, io0+len) (located at buffer offset
// `base`) into the tensors; header/padding pieces are skipped.
static void scatter_items(const std::vector<Piece>& pcs, uint64_t io0, uint64_t len, uint64_t base,
                          std::vector<Item>* items, uint32_t len_tag) {
  const uint64_t io1 = io0 + len;
  size_t lo = 0, hi = pcs.size();
  while (lo < hi) {  // first piece ending after io0
    const size_t mid = (lo + hi) / 2;
    if (pcs[mid].image_off + pcs[mid].len <= io0)
      lo = mid + 1;
    else
      hi = mid;
  }
  for (size_t i = lo; i < pcs.size() && pcs[i].image_off < io1; ++i) {
    if (!pcs[i].src) continue;
    uint64_t a = std::max(io0, pcs[i].image_off);
    const uint64_t b = std::min(io1, pcs[i].image_off + pcs[i].len);
    while (a < b) {
      const uint64_t nn = std::min<uint64_t>(b - a, kTile);
      items->push_back({pcs[i].src + (a - pcs[i].image_off), (uint32_t)(base + a - io0),
                        (uint32_t)nn | len_tag});
      a += nn;
    }
  }
}

int fp_ckpt_load_parallel(fp_ctx* c, const fp_tensor* t, size_t n, const char* path,
                          int dp_rank, int dp_size, void* stream) {
  NvtxRange nv("fp.load_parallel");
  if (!c || (!t && n) || !path || dp_size < 1 || dp_rank < 0 || dp_rank >= dp_size)
    return -EINVAL;
  if (dp_size > 1 && !c->has_comm) return -EINVAL;
  if (c->cfg.io_engine == FP_IO_NULL) return -EINVAL;
  const double t_call = now_s();
  memset(&c->ld, 0, sizeof(c->ld));
  {
    std::lock_guard<std::mutex> g(c->mu);
    if (c->state != fp_ctx::IDLE) return -EBUSY;
  }
  const int k = dp_size, rank = dp_rank;
  resolve_dirs(c, path, rank);
  // 1) manifest; every rank must succeed before the (collective) plan setup
  const std::string mpath = join_path(c->manifest_dir, "manifest.json");
  std::string mtxt;
  int r = read_file(mpath, &mtxt);
  if (r) fprintf(stderr, "fastpersist: cannot read %s: %s\n", mpath.c_str(), strerror(-r));
  JVal m;
  if (!r) {
    JParser jp{mtxt.data(), mtxt.data() + mtxt.size()};
    m = jp.val();
    if (!jp.ok || m.t != JVal::OBJ) r = FP_ECORRUPT;
  }
  auto num = [&](const char* key) -> uint64_t {
    const JVal* v = m.get(key);
    return v && v->t == JVal::NUM ? v->num : ~0ull;
  };
  if (!r && (num("dp_size") != (uint64_t)k || num("alignment") != c->cfg.alignment))
    r = FP_EMISMATCH;
  r = status_min(c, k, r);
  if (r) return r;
  PartitionScope wss(c, num("writer_stride"), manifest_bytes_balance(m));  // the writer's partition
  r = ensure_plan(c, t, n, rank, k);  // all-gather of sizes when the signature is new
  if (r) return r;
  const Plan& p = c->plan;
  if (num("image_bytes") != p.image_bytes || num("layout_digest") != p.digest) r = FP_EMISMATCH;
  // 2) this rank's own shard, nothing else
  const std::string sf = join_path(c->shard_dir, shard_file(rank, k));
  int fd = -1, bfd = -1;  // bfd: buffered, for requests that are not block-aligned
  if (!r) {
    bfd = open(sf.c_str(), O_RDONLY);
    fd = open(sf.c_str(), O_RDONLY | O_DIRECT);
    if (fd < 0 && errno == EINVAL) fd = open(sf.c_str(), O_RDONLY);
    if (fd < 0) {
      r = -errno;
      fprintf(stderr, "fastpersist: missing shard %s: %s\n", sf.c_str(), strerror(errno));
    } else {
      struct stat sb;
      uint64_t want = 0;
      for (auto& e : c->all_extents[rank]) want += e.len;
      if (fstat(fd, &sb) || (uint64_t)sb.st_size != want) {
        fprintf(stderr, "fastpersist: shard %s has %lld bytes, expected %llu\n", sf.c_str(),
                (long long)sb.st_size, (unsigned long long)want);
        r = FP_ECORRUPT;
      }
    }
  }
  r = status_min(c, k, r);
  if (r) {
    if (fd >= 0) close(fd);
    if (bfd >= 0) close(bfd);
    return r;
  }
  // 3) geometry: replicated partitions (the writer's page-balanced split)
  auto part_off = [&](int w) {  // image offset of writer w's partition
    uint64_t f, n;
    rep_share(p, w, &f, &n);
    return f;
  };
  auto part_bytes = [&](int w) {
    uint64_t f, n;
    rep_share(p, w, &f, &n);
    return n;
  };
  const uint64_t CH = c->cfg.slot_bytes, M = part_bytes(0);  // writer 0 has the largest part
  const uint64_t nrep = (M + CH - 1) / CH;
  const bool dev = !c->host;
  cudaStream_t st = (cudaStream_t)stream;
  Plan rp = p;  // whole replicated region (+ own local region) as one source map
  rp.extents.assign(1, {0, 0, p.rep_bytes});
  if (!p.regions.empty()) rp.extents.push_back({p.regions[rank].first, p.rep_bytes,
                                                p.regions[rank].second});
  plan_pieces(&rp, c->rep, c->loc, 0);  // header pieces -> src 0 (skipped)
  const uint64_t lreg_off = p.regions.empty() ? 0 : p.regions[rank].first;
  const uint64_t lreg_len = p.regions.empty() ? 0 : p.regions[rank].second;
  const uint64_t nloc = (lreg_len + CH - 1) / CH;
  const uint64_t total_chunks = nrep + nloc;
  // this rank's bytes of chunk j: (length, offset in the own shard file)
  auto my_span = [&](uint64_t j, uint64_t* foff) -> uint64_t {
    if (j < nrep) {
      const uint64_t pb = part_bytes(rank);
      *foff = j * CH;
      return j * CH < pb ? std::min(CH, pb - j * CH) : 0;
    }
    const uint64_t jj = j - nrep;
    *foff = part_bytes(rank) + jj * CH;
    return std::min(CH, lreg_len - jj * CH);
  };

  // 4) the exchange. Default (device state, k > 1): over peer memory — each
  // rank's whole replicated partition lands in its own device buffer, the
  // buffers are mapped into every rank (CUDA IPC; same address space for
  // thread ranks) and one unpack launch per chunk reads every writer's chunk
  // straight from its buffer (fp_unpack_peer). Fallback (host state, IPC
  // unavailable, FP_LOAD_EXCHANGE=nccl): one comm->allgather_bytes per chunk
  // into a gathered buffer, then fp_unpack_v4. Collective decision.
  const char* xm = getenv("FP_LOAD_EXCHANGE");
  const std::string xmode = xm ? xm : "auto";
  int status = 0;
  uint8_t* pbuf = nullptr;  // peer mode: [4 KiB: ready-flag source word | own partition]
  const uint64_t flag_bytes = 4096;
  PeerTab tab{};
  std::vector<void*> opened;
  bool peer = false;
  // Ready flags: one u32 per (writer, chunk) in a POSIX shared-memory segment
  // that rank 0 creates and every rank maps and registers with CUDA. Writer
  // w's copy engine sets flag (w, j) right behind the H2D of its chunk j (a
  // 4-byte D2H on the same stream); a consumer's HOST waits for the flags of
  // chunk j before it launches the unpack of chunk j. No kernel ever spins:
  // with streams of several ranks (or several streams of one rank) sharing a
  // hardware queue, a GPU-side wait could sit in front of the very copy it
  // waits for.
  volatile uint32_t* rflags = nullptr;
  size_t rflags_bytes = 0;
  bool rflags_reg = false;
  std::string shm_name;
  auto drop_flags = [&](bool unlink_it) {
    if (rflags_reg) cudaHostUnregister((void*)rflags);
    if (rflags) munmap((void*)rflags, rflags_bytes);
    rflags = nullptr;
    rflags_reg = false;
    if (unlink_it && rank == 0 && !shm_name.empty()) shm_unlink(shm_name.c_str());
  };
  if (dev && k > 1 && k <= kMaxPeers && xmode != "nccl") {
    int ok = 1;
    cudaIpcMemHandle_t h{};
    if (cudaMalloc(&pbuf, flag_bytes + std::max<uint64_t>(part_bytes(rank), 4096)) != cudaSuccess) {
      cudaGetLastError();
      pbuf = nullptr;
      ok = 0;
    }
    // the source word of this rank's flag copies (nonzero), ready before use
    if (ok && (cudaMemsetAsync(pbuf, 1, 4, c->stream) != cudaSuccess ||
               cudaStreamSynchronize(c->stream) != cudaSuccess))
      ok = 0;
    const bool ipc_ok = ok && cudaIpcGetMemHandle(&h, pbuf) == cudaSuccess;
    if (!ipc_ok) cudaGetLastError();
    static std::atomic<uint64_t> seq{0};
    const uint64_t my_seq = ++seq;
    rflags_bytes = round_up((uint64_t)k * std::max<uint64_t>(nrep, 1) * 4, 4096);
    if (ok && rank == 0) {  // created (zero-filled) before anyone learns its name
      const std::string nm = "/fpld." + std::to_string(getpid()) + "." + std::to_string(my_seq);
      shm_unlink(nm.c_str());  // a stale segment of a crashed process with our pid
      const int sfd = shm_open(nm.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
      if (sfd < 0 || ftruncate(sfd, (off_t)rflags_bytes)) ok = 0;
      if (sfd >= 0) close(sfd);
      if (ok) shm_name = nm;
    }
    std::vector<uint64_t> mine(13, 0), all(13 * (size_t)k, 0);
    mine[0] = (uint64_t)getpid();
    mine[1] = (uint64_t)(int64_t)c->dev;
    mine[2] = ipc_ok ? 1 : 0;
    mine[3] = (uint64_t)(uintptr_t)pbuf;
    memcpy(&mine[4], &h, sizeof(h));
    mine[12] = my_seq;
    int32_t v = ok;
    if (c->comm.allreduce_min_i32(c->comm.ctx, &v)) v = -1;
    if (v == 1 && c->comm.allgather_u64(c->comm.ctx, mine.data(), all.data(), 13)) v = -1;
    if (v == 1) {
      int mok = 1;
      shm_name = "/fpld." + std::to_string(all[0]) + "." + std::to_string(all[12]);
      const int sfd = shm_open(shm_name.c_str(), O_RDWR, 0600);
      void* mp = sfd < 0 ? MAP_FAILED
                         : mmap(nullptr, rflags_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, sfd, 0);
      if (sfd >= 0) close(sfd);
      if (mp == MAP_FAILED) {
        mok = 0;
      } else {
        rflags = (volatile uint32_t*)mp;
        rflags_reg = cudaHostRegister(mp, rflags_bytes, cudaHostRegisterPortable) == cudaSuccess;
        if (!rflags_reg) {
          cudaGetLastError();
          mok = 0;
        }
      }
      for (int w = 0; w < k && mok; ++w) {
        const uint64_t* q = &all[13 * (size_t)w];
        void* ptr = nullptr;
        if (q[0] == (uint64_t)getpid()) {  // same process (thread ranks): same address space
          ptr = (void*)(uintptr_t)q[3];
          const int pd = (int)(int64_t)q[1];
          if (pd != c->dev) {
            const cudaError_t e = cudaDeviceEnablePeerAccess(pd, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) mok = 0;
            cudaGetLastError();
          }
        } else if (q[2]) {
          cudaIpcMemHandle_t ph;
          memcpy(&ph, &q[4], sizeof(ph));
          if (cudaIpcOpenMemHandle(&ptr, ph, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) {
            opened.push_back(ptr);
          } else {
            cudaGetLastError();
            mok = 0;
          }
        } else {
          mok = 0;
        }
        tab.base[w] = (uint64_t)(uintptr_t)ptr + flag_bytes;
      }
      v = mok;
      if (c->comm.allreduce_min_i32(c->comm.ctx, &v)) v = -1;
    }
    peer = v == 1;
    if (!peer) {
      for (void* q : opened) cudaIpcCloseMemHandle(q);
      opened.clear();
      drop_flags(false);
      if (pbuf) cudaFree(pbuf);
      pbuf = nullptr;
      if (xmode == "peer") status = -ENOSYS;  // peer exchange was required
      if (v < 0) status = FP_ECOMM;
      // every rank has stopped using the segment (the all-reduce above)
      if (rank == 0 && !shm_name.empty()) shm_unlink(shm_name.c_str());
      shm_name.clear();
    }
  }
  if (!status && k > 1 && !peer && !c->comm.allgather_bytes) status = -ENOSYS;
  c->ld.exchange = k == 1 ? 0 : peer ? 2 : 1;

  // work items: chunk j = the j-th CH bytes of every writer's partition
  std::vector<Item> items;
  std::vector<uint32_t> lo(1, 0);
  std::vector<uint64_t> wmask(nrep, 0);
  for (uint64_t j = 0; j < nrep; ++j) {
    for (int w = 0; w < k; ++w) {
      const uint64_t pb = part_bytes(w);
      if (j * CH >= pb) continue;
      wmask[j] |= 1ull << (w & 63);
      // peer: offset inside writer w's chunk + writer tag in len bits 24..31;
      // gathered buffer: offset w*CH
      scatter_items(rp.pieces, part_off(w) + j * CH, std::min(CH, pb - j * CH),
                    peer ? 0 : (uint64_t)w * CH, &items, peer ? (uint32_t)w << 24 : 0);
    }
    lo.push_back((uint32_t)items.size());
  }
  for (uint64_t j = 0; j < nloc; ++j) {
    scatter_items(rp.pieces, lreg_off + j * CH, std::min(CH, lreg_len - j * CH), 0, &items, 0);
    lo.push_back((uint32_t)items.size());
  }
  // 5) buffers: send = one chunk (two with GDS), recv = k chunks (gathered
  // mode only); device, or host for host state
  uint8_t *send = nullptr, *recv = nullptr;
  Item* d_items = nullptr;
  PeerTab* d_tab = nullptr;
  // GPUDirect Storage: own-shard chunks are read with cuFileRead
  // straight into device memory (no ring, no H2D)
  const bool use_gds = dev && c->gds;
  void* gfh = nullptr;
  if (use_gds && !status && fd >= 0) status = gds_handle_open(fd, &gfh);
  uint32_t* h_allpc = nullptr;
  uint32_t* d_allpc = nullptr;
  const uint64_t shard_pages = (part_bytes(rank) + lreg_len) / 4096 + 1;
  cudaStream_t cs = c->stream;     // peer mode: H2D copies + ready flags (copy engine only)
  cudaStream_t crcs = nullptr;     // peer mode: page CRCs (never waited on before the end)
  cudaEvent_t ev_h2d = nullptr;
  if (dev && !status) {
    if (cudaMalloc(&send, CH * (use_gds ? 2 : 1)) != cudaSuccess ||
        (!peer && cudaMalloc(&recv, CH * k) != cudaSuccess) ||
        (peer && (cudaMalloc(&d_tab, sizeof(PeerTab)) != cudaSuccess ||
                  cudaMemcpy(d_tab, &tab, sizeof(PeerTab), cudaMemcpyHostToDevice) != cudaSuccess)) ||
        (!items.empty() && (cudaMalloc(&d_items, items.size() * sizeof(Item)) != cudaSuccess ||
                            cudaMemcpy(d_items, items.data(), items.size() * sizeof(Item),
                                       cudaMemcpyHostToDevice) != cudaSuccess)))
      status = -ENOMEM;
    if (peer && !status &&
        (cudaStreamCreateWithFlags(&crcs, cudaStreamNonBlocking) != cudaSuccess ||
         cudaEventCreateWithFlags(&ev_h2d, cudaEventDisableTiming) != cudaSuccess))
      status = FP_ECUDA;
    // peer mode keeps every page CRC of the own shard (4 B per 4 KiB) until
    // the end: no host wait on a CRC kernel while unpacks spin on peers'
    // flags. Allocated here, before the status all-reduce that releases the
    // ranks into the exchange loop: an allocation call may wait for the
    // device, and once any rank spins on flags this rank must not block on
    // anything but its own copies.
    if (peer && !status && !(c->cfg.flags & FP_CFG_NO_CRC) &&
        (cudaHostAlloc(&h_allpc, shard_pages * 4, cudaHostAllocPortable) != cudaSuccess ||
         cudaMalloc(&d_allpc, shard_pages * 4) != cudaSuccess))
      status = -ENOMEM;
  } else if (!dev) {
    send = (uint8_t*)aligned_alloc(4096, round_up(CH, 4096));
    recv = (uint8_t*)aligned_alloc(4096, round_up(CH * k, 4096));
    if (!send || !recv) status = -ENOMEM;
  }
  status = status_min(c, k, status);
  std::vector<uint8_t> ghdr_got(p.ghdr.bytes.size(), 0), lhdr_got(p.lhdr.bytes.size(), 0);
  const uint32_t R = c->cfg.ring_slots;
  auto fetch_hdr = [&](const uint8_t* buf, uint64_t io0, uint64_t len, uint64_t base,
                       uint64_t h0, std::vector<uint8_t>* out) {
    // copy the header bytes [h0, h0+out.size()) that fall in this buffer
    const uint64_t a = std::max(io0, h0), b = std::min(io0 + len, h0 + out->size());
    if (a >= b) return;
    if (dev)
      cudaMemcpyAsync(out->data() + (a - h0), buf + base + (a - io0), b - a,
                      cudaMemcpyDefault, st);
    else
      memcpy(out->data() + (a - h0), buf + base + (a - io0), b - a);
  };
  // CRC-32 of the own shard as it is read (page CRCs on the GPU, folded per
  // extent on the host), checked against the manifest
  const bool check_crc = !(c->cfg.flags & FP_CFG_NO_CRC);
  ExtentCrc acc;
  acc.reset(c->all_extents[rank]);
  const ShardCrcRec rec = crc_record(m, rank, c->all_extents[rank].size());
  const bool run = status == 0;  // agreed on every rank by the all-reduce above
  LoadCrc lcrc(c, [&](uint64_t j, const uint32_t* pages) {
    uint64_t fo = 0;
    const uint64_t n = my_span(j, &fo);
    acc.add_pages(fo, pages, n / 4096);
  });
  // peer mode, replicated chunks: (file offset, bytes, raw CRC or ~0 = pages
  // in d_allpc), folded in file order at the end
  struct Deferred {
    uint64_t fo, n;
    uint32_t raw;
    bool pages;
  };
  std::vector<Deferred> deferred;
  // own-shard reads run R chunks ahead of the exchange + scatter
  ReadAhead ra(c, run && !use_gds ? total_chunks : 0, dev,
               [&](uint64_t j, std::vector<ReadReq>* out) -> int {
    uint64_t foff = 0;
    const uint64_t len = my_span(j, &foff);
    const uint64_t al = p.align;
    for (uint64_t pos = 0; pos < len; pos += c->cfg.sqe_bytes) {
      const uint32_t n1 = (uint32_t)std::min<uint64_t>(c->cfg.sqe_bytes, len - pos);
      const bool aligned = (foff + pos) % al == 0 && n1 % al == 0;
      out->push_back({aligned ? fd : bfd, foff + pos, pos, n1});
    }
    return 0;
  });
  const double spin_s = (double)env_u64("FP_PEER_TIMEOUT_S", 600);
  bool peer_failed = false;
  c->ld.t_setup = now_s() - t_call;
  uint64_t launches = 0;
  for (uint64_t j = 0; run && j < total_chunks; ++j) {  // every rank runs every exchange
    const bool is_rep = j < nrep;
    const uint32_t s = (uint32_t)(j % R);
    uint8_t* slot = ra.slot_of(j);
    uint64_t foff = 0;
    const uint64_t mylen = my_span(j, &foff);
    const bool gpu_crc =
        check_crc && dev && mylen % 4096 == 0 && c->d_crc_tabs && acc.pages_ok(foff, mylen);
    auto host_crc = [&](const uint8_t* q) {  // in order behind the pending page folds
      if (peer && is_rep) {
        deferred.push_back({foff, mylen, crc_raw_update(0, q, mylen), false});
        return;
      }
      if (lcrc.flush() && !status) status = FP_ECUDA;
      acc.add_bytes(foff, q, mylen);
    };
    // where this rank's bytes of chunk j land on the device
    uint8_t* sbuf = peer && is_rep ? pbuf + flag_bytes + j * CH
                    : use_gds ? send + (j & 1) * CH : send;
    cudaStream_t xs = peer && is_rep ? cs : st;  // stream of the H2D
    if (use_gds) {
      // the unpack of chunk j-2 read this half: wait for it, then read into it
      if (!(peer && is_rep) && j >= 2 && cudaEventSynchronize(c->gds_ev[j & 1]) != cudaSuccess &&
          !status)
        status = FP_ECUDA;
      if (mylen && !status) {
        gds_post(c->gds_pool, false, gfh, sbuf, 0, foff, mylen,
                 std::max<uint64_t>(c->cfg.sqe_bytes, 4ull << 20));
        int rr = gds_wait(c->gds_pool, nullptr);
        if (rr && !status) status = rr;  // keep exchanging so the collectives stay matched
      }
      if (check_crc && mylen && !gpu_crc && !status) {  // ragged chunk: CRC on the host
        if (cudaMemcpy(slot, sbuf, mylen, cudaMemcpyDeviceToHost) != cudaSuccess)
          status = FP_ECUDA;
        else
          host_crc(slot);
      }
    } else {
      const double t_r = now_s();
      int rr = status ? 0 : ra.wait(j);
      c->ld.t_read_wait += now_s() - t_r;
      if (rr && !status) status = rr;  // keep exchanging so the peers are not left waiting
      if (check_crc && mylen && !gpu_crc && !status) host_crc(slot);
    }
    if (dev) {
      if (!use_gds) {
        if (mylen && !status &&
            cudaMemcpyAsync(sbuf, slot, mylen, cudaMemcpyHostToDevice, xs) != cudaSuccess)
          status = FP_ECUDA;
        cudaEventRecord(c->ev_d2h[s], xs);
      }
      if (peer && is_rep && mylen) {
        // ready flag (rank, j): a 4-byte copy behind the data on the copy
        // stream into the shared segment (no kernel: a flag never waits for
        // an SM)
        if (cudaMemcpyAsync((void*)&rflags[(size_t)rank * nrep + j], pbuf, 4,
                            cudaMemcpyDeviceToHost, cs) != cudaSuccess && !status)
          status = FP_ECUDA;
      }
      if (gpu_crc && mylen) {
        int e = 0;
        if (peer && is_rep) {  // deferred: CRC stream after the H2D, pages kept to the end
          e = cudaEventRecord(ev_h2d, xs) != cudaSuccess ||
              cudaStreamWaitEvent(crcs, ev_h2d, 0) != cudaSuccess ||
              crc_pages_launch(sbuf, mylen, c->d_crc_tabs, d_allpc + foff / 4096, crcs);
          deferred.push_back({foff, mylen, 0, true});
        } else {
          e = lcrc.enqueue(j, sbuf, mylen, st);
        }
        if (e && !status) status = FP_ECUDA;
        ++launches;
      }
    } else if (mylen) {
      memcpy(send, slot, mylen);
    }
    const uint8_t* src = sbuf;
    if (is_rep && !peer) {
      if (k > 1) {
        if (c->comm.allgather_bytes(c->comm.ctx, sbuf, recv, CH, dev ? 1 : 0, stream)) {
          status = status ? status : FP_ECOMM;
          break;
        }
        src = recv;
      }
      for (int w = 0; w < k; ++w) {
        const uint64_t pb = part_bytes(w);
        if (j * CH >= pb) continue;
        fetch_hdr(src, part_off(w) + j * CH, std::min(CH, pb - j * CH),
                  k > 1 ? (uint64_t)w * CH : 0, 0, &ghdr_got);
      }
    } else if (!is_rep) {
      const uint64_t jj = j - nrep;
      fetch_hdr(src, lreg_off + jj * CH, mylen, 0, lreg_off, &lhdr_got);
    }
    const uint32_t i0 = lo[j], i1 = lo[j + 1];
    if (peer && is_rep) {
      // every writer's chunk j has landed in its buffer (its flag): then the
      // unpack reads them all straight from the writers' buffers
      if (!peer_failed) {
        const double t_w = now_s();
        for (int w = 0; w < k && !peer_failed; ++w) {
          if (!((wmask[j] >> w) & 1)) continue;
          const volatile uint32_t* f = &rflags[(size_t)w * nrep + j];
          for (uint32_t spins = 0; !__atomic_load_n(f, __ATOMIC_ACQUIRE); ++spins) {
            if (now_s() - t_w > spin_s) {
              fprintf(stderr, "fastpersist: rank %d: chunk %llu of rank %d never arrived "
                              "(peer exchange timed out)\n", rank, (unsigned long long)j, w);
              peer_failed = true;
              break;
            }
            if (spins > 64) usleep(20);
          }
        }
        c->ld.t_exchange_wait += now_s() - t_w;
      }
      if (peer_failed) {
        if (!status) status = FP_ECOMM;  // keep publishing our flags: peers are not left waiting
      } else if (unpack_peer_launch(d_items + i0, i1 - i0, d_tab, (uint32_t)j, CH, c->pack_ctas,
                                    st) && !status) {
        status = FP_ECUDA;
      }
      ++launches;
    } else if (i1 > i0 && status == 0) {
      if (dev) {
        if (unpack_launch(d_items + i0, i1 - i0, src, c->pack_ctas, st)) status = FP_ECUDA;
        ++launches;
      } else {
        for (uint32_t i = i0; i < i1; ++i)
          memcpy((void*)(uintptr_t)items[i].src, src + items[i].dst, items[i].len);
      }
    }
    if (use_gds && !(peer && is_rep) && cudaEventRecord(c->gds_ev[j & 1], st) != cudaSuccess &&
        !status)
      status = FP_ECUDA;  // this half is free once the work above has run
    ra.release(j);
  }
  ra.finish();  // reads still in flight after an error land before the ring is reused
  if (dev && cudaStreamSynchronize(st) != cudaSuccess && !status) status = FP_ECUDA;
  if (peer) {
    if (cudaStreamSynchronize(cs) != cudaSuccess && !status) status = FP_ECUDA;
    // GHDR bytes straight from the writers' buffers
    for (int w = 0; w < k && run && !status; ++w) {
      const uint64_t a0 = part_off(w), pb = part_bytes(w);
      const uint64_t a1 = std::min<uint64_t>(a0 + pb, ghdr_got.size());
      if (a0 < a1 && cudaMemcpy(ghdr_got.data() + a0, (const void*)(uintptr_t)tab.base[w],
                                a1 - a0, cudaMemcpyDefault) != cudaSuccess)
        status = FP_ECUDA;
    }
    if (crcs && cudaStreamSynchronize(crcs) != cudaSuccess && !status) status = FP_ECUDA;
    if (!status && run && check_crc && !deferred.empty()) {
      if (h_allpc && cudaMemcpy(h_allpc, d_allpc, shard_pages * 4, cudaMemcpyDeviceToHost) !=
                         cudaSuccess)
        status = FP_ECUDA;
      // replicated chunks in file order (the local region's are already in acc)
      for (const Deferred& d : deferred) {
        if (d.pages)
          acc.add_pages(d.fo, h_allpc + d.fo / 4096, d.n / 4096);
        else
          acc.add_raw(d.fo, d.n, d.raw);
      }
    }
  }
  if (!status && run && check_crc) {
    status = lcrc.flush();
    if (!status) status = verify_crc(acc, rec, sf);
  }
  if (!status && (memcmp(ghdr_got.data(), p.ghdr.bytes.data(), ghdr_got.size()) ||
                  memcmp(lhdr_got.data(), p.lhdr.bytes.data(), lhdr_got.size()))) {
    fprintf(stderr, "fastpersist: header bytes gathered from the shards do not match the "
                    "target tensors (corrupt or different state)\n");
    status = FP_ECORRUPT;
  }
  for (void* q : opened) cudaIpcCloseMemHandle(q);  // before the owners free (barrier below)
  if (peer) drop_flags(false);
  status = status_min(c, k, status);
  if (peer && rank == 0 && !shm_name.empty()) shm_unlink(shm_name.c_str());  // all unmapped
  c->ld.kernel_launches = launches;
  c->ld.bytes_read = part_bytes(rank) + lreg_len;
  c->ld.status = status;
  c->ld.t_total = now_s() - t_call;
  if (gfh) gds_handle_close(gfh);
  if (crcs) cudaStreamDestroy(crcs);
  if (ev_h2d) cudaEventDestroy(ev_h2d);
  if (h_allpc) cudaFreeHost(h_allpc);
  if (d_allpc) cudaFree(d_allpc);
  if (dev) {
    if (send) cudaFree(send);
    if (recv) cudaFree(recv);
    if (d_items) cudaFree(d_items);
    if (d_tab) cudaFree(d_tab);
    if (pbuf) cudaFree(pbuf);
  } else {
    free(send);
    free(recv);
  }
  close(fd);
  if (bfd >= 0) close(bfd);
  return status;
}

}  // extern "C"
