// Internal declarations of libfastpersist (not part of the C-ABI).
#pragma once

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "fastpersist.h"

namespace fp {

// ---------------------------------------------------------------------------
// FPCK v2 layout constants
// ---------------------------------------------------------------------------
constexpr uint32_t kVersion = 2;
constexpr uint64_t kFixedHdr = 64;
constexpr uint64_t kEntry = 128;
constexpr uint64_t kRegion = 16;
constexpr uint32_t kFlagHasLocal = 1;
constexpr uint32_t kFlagLocal = 2;

inline uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
int dtype_size(uint8_t dtype);  // 0 if unknown
uint64_t fnv1a64(const uint8_t* p, size_t n, uint64_t h = 0xCBF29CE484222325ull);

struct TensorRef {
  uint64_t ptr;      // device or host address
  uint64_t nbytes;
  std::string name;
  int64_t shape[8];
  int32_t owner;
  uint8_t dtype, section, ndim, flags;
};

// Validate + copy the caller's tensor table. Returns 0 or -EINVAL.
int import_tensors(const fp_tensor* t, size_t n, int dp_rank, std::vector<TensorRef>* rep,
                   std::vector<TensorRef>* loc, bool* host);

// One header (GHDR or LREG): encoded bytes + payload offsets.
struct Header {
  std::vector<uint8_t> bytes;
  uint64_t digest = 0;
};
uint64_t header_len(uint64_t n_tensors, uint64_t n_regions, uint64_t names_bytes, uint64_t align);
void encode_header(const std::vector<TensorRef>& ts, const std::vector<uint64_t>& offs,
                   const std::vector<std::pair<uint64_t, uint64_t>>& regions, uint32_t align,
                   uint64_t total_bytes, int64_t owner, uint32_t flags, Header* out);

struct Extent {
  uint64_t image_off, file_off, len;
};

// A contiguous run of image bytes with a single source.
struct Piece {
  uint64_t image_off;
  uint64_t len;
  uint64_t src;  // address (device or host); 0 = zero fill
};

// Everything rank `rank` needs to write (or read) its shard.
struct Plan {
  uint32_t align = 4096, writer_stride = 1;
  // replicated-region partition unit: `align` (page-granular, reading R5) or
  // 1 (byte-granular, FP_CFG_BALANCE_BYTES: the paper's <= 1 byte imbalance)
  uint64_t unit = 4096;
  int rank = 0, k = 1;
  uint64_t header_bytes = 0, rep_bytes = 0, image_bytes = 0, digest = 0;
  std::vector<std::pair<uint64_t, uint64_t>> regions;  // (offset, bytes) per rank or empty
  Header ghdr, lhdr;
  std::vector<uint64_t> rep_off, loc_off;
  std::vector<Extent> extents;  // this rank, image order
  uint64_t shard_bytes = 0;
  // sources of this rank's image bytes, sorted by image_off (header sources
  // point at hdr_base + offset: device copy of ghdr||lhdr, or the host copy)
  std::vector<Piece> pieces;
};

// Layout pass 1 (local): replicated header + offsets, and what this rank
// contributes to the all-gather: {local_region_bytes, n_local, digest}.
struct LocalFacts {
  uint64_t region_bytes, n_local, digest, rep_bytes;
};
void plan_local_facts(const std::vector<TensorRef>& rep, const std::vector<TensorRef>& loc,
                      uint32_t align, LocalFacts* out);
// Replicated-region partition (writer subsets P:495-499): the Q
// pages go to the writers w = 0, s, 2s, ... (s = writer_stride, 0/1 = every
// rank) in contiguous page-balanced ranges in rank order, the lowest writers
// taking the extra pages; a non-writer gets no pages.
void rep_partition(uint64_t Q, int k, uint32_t writer_stride, int w, uint64_t* first_page,
                   uint64_t* n_pages);
// Layout pass 2: needs all ranks' facts (k entries). Returns 0 / FP_EMISMATCH.
int plan_build(const std::vector<TensorRef>& rep, const std::vector<TensorRef>& loc,
               uint32_t align, int rank, int k, uint32_t writer_stride, bool balance_bytes,
               const std::vector<LocalFacts>& all, Plan* out);
// (image offset, bytes) of writer w's share of the replicated region
void rep_share(const Plan& p, int w, uint64_t* off, uint64_t* bytes);
// Rebase header pieces onto hdr_base (ghdr at +0, lhdr at +ghdr.size());
// hdr_base == 0 turns header pieces into skip (zero) items, as load needs.
void plan_pieces(Plan* p, const std::vector<TensorRef>& rep, const std::vector<TensorRef>& loc,
                 uint64_t hdr_base);

// Work items of the pack/unpack kernels: one tile of <= kTile bytes.
constexpr uint32_t kTile = 32768;
struct Item {
  uint64_t src;  // gather source (0 = zero fill); for unpack: scatter destination
  uint32_t dst;  // byte offset inside the slab
  uint32_t len;  // <= kTile
};
static_assert(sizeof(Item) == 16, "Item must be 16 bytes");

// Items for every chunk of the shard file (chunk = slot_bytes of file bytes).
// item_lo has n_chunks+1 entries. Item.dst is relative to the start of the
// chunk's pack group (group = group_bytes/slot_bytes consecutive chunks that
// one pack launch gathers into one device slab). An item never spans two
// pieces (so never two allocations) and is at most max_item bytes.
void plan_items(const Plan& p, uint64_t slot_bytes, uint64_t group_bytes,
                std::vector<Item>* items, std::vector<uint32_t>* item_lo,
                uint64_t max_item = kTile);

// Per pack group: tile_lo[off_g + t] = first item (relative to the group's
// first item) of 32 KiB slab tile t, t = 0..n_tiles_g (n_tiles_g + 1 entries
// per group, groups concatenated; group_tile_off[g] = off_g).
void plan_tiles(const std::vector<Item>& items, const std::vector<uint32_t>& item_lo,
                uint64_t shard_bytes, uint64_t slot_bytes, uint64_t group_bytes,
                std::vector<uint32_t>* tile_lo, std::vector<uint64_t>* group_tile_off);

// ---------------------------------------------------------------------------
// I/O engines
// ---------------------------------------------------------------------------
struct IoDone {
  uint64_t user;
  int32_t res;
};

class IoEngine {
 public:
  virtual ~IoEngine() {}
  virtual int kind() const = 0;
  // Optional fixed-buffer registration (io_uring). 0 or -errno (non-fatal).
  virtual int register_buffers(void* base, uint64_t slot_bytes, uint32_t slots) { return -1; }
  // Queue one request (buf_index >= 0: registered slot). 0 or -errno.
  virtual int queue(bool write, int fd, void* buf, uint32_t len, uint64_t off, int buf_index,
                    uint64_t user) = 0;
  virtual int submit() = 0;                                 // push queued requests
  virtual int reap(IoDone* out, int max, int min_wait) = 0;  // >= 0 count or -errno
  virtual int fdatasync(int fd) = 0;
  virtual uint32_t capacity() const = 0;
};

IoEngine* make_uring(uint32_t depth, int* err);
IoEngine* make_pwrite(uint32_t threads, bool direct);
IoEngine* make_null(uint32_t depth);

// ---------------------------------------------------------------------------
// kernels (pack.cu)
// ---------------------------------------------------------------------------
int pack_launch(int impl, const Item* d_items, uint32_t n_items, uint8_t* d_slab, int ctas,
                void* stream);
int unpack_launch(const Item* d_items, uint32_t n_items, const uint8_t* d_slab, int ctas,
                  void* stream);
int pack_default_ctas(int impl, int device);
// peer-exchange load (fp_unpack_peer): writer w's replicated partition at base[w]
constexpr int kMaxPeers = 64;
struct PeerTab {
  uint64_t base[kMaxPeers];
};
// items of exchange chunk `chunk` (Item.len bits 24..31 = writer) scattered
// from base[w] + chunk * ch_bytes + Item.dst (launched once every writer's
// chunk has landed)
int unpack_peer_launch(const Item* d_items, uint32_t n_items, const PeerTab* d_tab, uint32_t chunk,
                       uint64_t ch_bytes, int ctas, void* stream);
// one-warp kernel on `stream` that waits until the mapped word *d_flag
// reaches `value` (or max_ns passes; then *d_timed_out = 1 if non-null)
int flag_wait_launch(const uint32_t* d_flag, uint32_t value, uint64_t max_ns,
                     uint32_t* d_timed_out, void* stream);
// raw CRC-32 (init 0, no xorout) of every 4 KiB page of d_buf[0, bytes)
// -> d_page_crc[bytes / 4096] (bytes: a multiple of 4096; d_tabs: the blob of
// crc_device_tables); the host folds them (ExtentCrc)
int crc_pages_launch(const uint8_t* d_buf, uint64_t bytes, const uint32_t* d_tabs,
                     uint32_t* d_page_crc, void* stream);
// fused TMA-engine pack + page CRCs (fp_pack_bulk_crc, the default with
// FP_PACK_BULK): tiles as below, gbytes = slab bytes of the group; the raw CRC
// of every page starting below gbytes -> d_page_crc (a ragged last page's CRC
// covers stale bytes: the host CRCs ragged chunks itself)
int pack_bulk_crc_launch(const Item* d_items, const uint32_t* d_tile_lo, uint32_t n_tiles,
                         uint64_t gbytes, uint8_t* d_slab, const uint32_t* d_tabs,
                         uint32_t* d_page_crc, int ctas, void* stream);
// LSU pack + page CRCs from the registers it copies through (fp_pack_lsu_crc,
// FP_PACK_LSU, ablation): tiles as below, gbytes = slab bytes of the group; the raw CRC
// of every whole page -> d_page_crc (a ragged last page gets 0: the host CRCs
// ragged chunks itself)
int pack_lsu_crc_launch(const Item* d_items, const uint32_t* d_tile_lo, uint64_t gbytes,
                        uint8_t* d_slab, const uint32_t* d_tabs, uint32_t* d_page_crc, int ctas,
                        void* stream);
// device CRC table blob layout (uint32 offsets)
constexpr uint32_t kTabS4 = 0;
constexpr uint32_t kTabLaneK = 4 * 256;  // 32 lane-combine constants x^(8*128*(31-l))
// fp_pack_lsu_crc: products by a constant as 8 nibble lookups, entry
// [j * 16 + n] = K * (n << 4j) (reflected): K = x^(8*512) (the stride between
// a lane's 16-B chunks), and per lane l K_l = x^(8*16*(31-l))
constexpr uint32_t kTabNibX = kTabLaneK + 32;
constexpr uint32_t kTabNibK = kTabNibX + 128;  // [l * 128 + j * 16 + n]
constexpr uint32_t kTabWords = kTabNibK + 32 * 128;

// ---------------------------------------------------------------------------
// CRC-32 helpers (crc32.cpp)
// ---------------------------------------------------------------------------
uint32_t gf_mul(uint32_t a, uint32_t b);          // a*b mod P, reflected
uint32_t gf_x8n(uint64_t n);                      // x^(8n) mod P
uint32_t crc_raw_update(uint32_t c, const uint8_t* p, uint64_t n);
uint32_t crc_zeros(uint64_t n);                   // standard CRC-32 of n zero bytes
const uint32_t* crc_tables8();                    // 8 x 256 slicing tables, contiguous
// the kTabWords-word blob fp_crc_pages reads (layout: pack.cu)
std::vector<uint32_t> crc_device_tables();

// Raw CRC-32 of a file accumulated per extent, in file order. The
// GPU delivers one raw CRC per 4 KiB page; the host folds them with one
// constant product per page (R <- R * x^(8*4096) ^ page), so the manifest can
// carry a CRC per extent (what a partial reader such as fp_ckpt_load verifies)
// and per file. Runs that are not page-foldable (ragged tails, extents not on
// 4 KiB boundaries) are added as bytes.
class ExtentCrc {
 public:
  void reset(const std::vector<Extent>& ext);  // extents in file order
  // [fo, fo + n) can be added as page CRCs: page-aligned, and every extent
  // boundary inside it is a page boundary
  bool pages_ok(uint64_t fo, uint64_t n) const;
  void add_pages(uint64_t fo, const uint32_t* page_crc, uint64_t n_pages);
  void add_bytes(uint64_t fo, const uint8_t* p, uint64_t n);
  // a run [fo, fo + n) inside one extent given as its raw CRC
  void add_raw(uint64_t fo, uint64_t n, uint32_t raw);
  size_t n() const { return beg_.size(); }
  uint64_t len(size_t i) const { return len_[i]; }
  bool complete(size_t i) const { return ok_ && done_[i] == len_[i]; }
  bool complete() const;
  uint32_t extent_crc(size_t i) const;  // standard CRC-32 (= zlib.crc32) of extent i
  uint32_t file_crc() const;            // standard CRC-32 of the whole file
  bool ok() const { return ok_; }       // false if a run arrived out of order
 private:
  size_t find(uint64_t fo);
  std::vector<uint64_t> beg_, len_, done_;
  std::vector<uint32_t> raw_;
  size_t cur_ = 0;
  bool ok_ = true;
};

}  // namespace fp
