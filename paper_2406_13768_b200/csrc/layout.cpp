// FPCK v2 layout, DP partition plan and pack work items (host side).
//
// Paper passages implemented here:
//  - serialized tensors + metadata, in caller order (§2.1.3 P:189;
//    §4.1 P:479 "the order in which tensors (and their bytes) are persisted
//    ... remains unchanged")
//  - aligned image for DMA/NVMe (§4.1; alignment 4096 = reading R4)
//  - partition fixed at setup, communication-free per checkpoint (§4.2),
//    balanced on bytes after serialization (§4.2; page granular,
//    reading R5)
#include <algorithm>
#include <cerrno>

#include "fp_internal.h"

namespace fp {

int dtype_size(uint8_t dtype) {
  switch (dtype) {
    case FP_F32: return 4;
    case FP_BF16: return 2;
    case FP_F16: return 2;
    case FP_F64: return 8;
    case FP_I64: return 8;
    case FP_I32: return 4;
    case FP_U8: return 1;
    default: return 0;
  }
}

uint64_t fnv1a64(const uint8_t* p, size_t n, uint64_t h) {
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ull;
  }
  return h;
}

int import_tensors(const fp_tensor* t, size_t n, int dp_rank, std::vector<TensorRef>* rep,
                   std::vector<TensorRef>* loc, bool* host) {
  rep->clear();
  loc->clear();
  int n_host = 0, n_dev = 0;
  for (size_t i = 0; i < n; ++i) {
    const fp_tensor& x = t[i];
    int isz = dtype_size(x.dtype);
    if (!isz || x.ndim > 8 || x.section > FP_SEC_OTHER || !x.name) return -EINVAL;
    size_t nl = strnlen(x.name, 65536);
    if (nl == 0 || nl > 65535) return -EINVAL;
    uint64_t numel = 1;
    for (int d = 0; d < x.ndim; ++d) {
      if (x.shape[d] < 0) return -EINVAL;
      numel *= (uint64_t)x.shape[d];
    }
    if (numel * (uint64_t)isz != x.nbytes) return -EINVAL;
    if (x.nbytes && !x.data) return -EINVAL;
    if (x.owner != -1 && x.owner != dp_rank) return -EINVAL;
    TensorRef r;
    r.ptr = (uint64_t)(uintptr_t)x.data;
    r.nbytes = x.nbytes;
    r.name.assign(x.name, nl);
    for (int d = 0; d < 8; ++d) r.shape[d] = d < x.ndim ? x.shape[d] : 0;
    r.owner = x.owner;
    r.dtype = x.dtype;
    r.section = x.section;
    r.ndim = x.ndim;
    r.flags = x.flags;
    if (x.nbytes) (x.flags & FP_TENSOR_HOST) ? ++n_host : ++n_dev;
    (x.owner < 0 ? rep : loc)->push_back(std::move(r));
  }
  if (n_host && n_dev) return -EINVAL;  // one checkpoint: all host or all device
  *host = n_host > 0;
  return 0;
}

uint64_t header_len(uint64_t n_tensors, uint64_t n_regions, uint64_t names_bytes,
                    uint64_t align) {
  return round_up(kFixedHdr + kEntry * n_tensors + kRegion * n_regions + names_bytes, align);
}

static void put32(uint8_t* p, uint32_t v) { memcpy(p, &v, 4); }
static void put64(uint8_t* p, uint64_t v) { memcpy(p, &v, 8); }

static uint64_t names_bytes(const std::vector<TensorRef>& ts) {
  uint64_t s = 0;
  for (auto& t : ts) s += t.name.size();
  return s;
}

void encode_header(const std::vector<TensorRef>& ts, const std::vector<uint64_t>& offs,
                   const std::vector<std::pair<uint64_t, uint64_t>>& regions, uint32_t align,
                   uint64_t total_bytes, int64_t owner, uint32_t flags, Header* out) {
  const uint64_t nb = names_bytes(ts);
  const uint64_t hl = header_len(ts.size(), regions.size(), nb, align);
  std::vector<uint8_t>& h = out->bytes;
  h.assign(hl, 0);
  uint8_t* tab = h.data() + kFixedHdr;
  uint8_t* reg = tab + kEntry * ts.size();
  uint8_t* pool = reg + kRegion * regions.size();
  uint32_t name_off = 0;
  for (size_t i = 0; i < ts.size(); ++i) {
    uint8_t* e = tab + kEntry * i;
    const TensorRef& t = ts[i];
    put64(e + 0, offs[i]);
    put64(e + 8, t.nbytes);
    put32(e + 16, name_off);
    put32(e + 20, (uint32_t)t.name.size());
    e[24] = t.dtype;
    e[25] = t.section;
    e[26] = t.ndim;
    e[27] = 0;
    put32(e + 28, (uint32_t)t.owner);
    for (int d = 0; d < 8; ++d) put64(e + 32 + 8 * d, (uint64_t)t.shape[d]);
    memcpy(pool + name_off, t.name.data(), t.name.size());
    name_off += (uint32_t)t.name.size();
  }
  for (size_t r = 0; r < regions.size(); ++r) {
    put64(reg + kRegion * r, regions[r].first);
    put64(reg + kRegion * r + 8, regions[r].second);
  }
  // layout digest: FNV-1a-64 over (entry table || names pool)
  uint64_t dg = fnv1a64(tab, kEntry * ts.size());
  dg = fnv1a64(pool, nb, dg);
  uint8_t* f = h.data();
  memcpy(f, "FPCK", 4);
  put32(f + 4, kVersion);
  put32(f + 8, align);
  put32(f + 12, flags);
  put64(f + 16, hl);
  put64(f + 24, total_bytes);
  put32(f + 32, (uint32_t)ts.size());
  put32(f + 36, (uint32_t)regions.size());
  put64(f + 40, nb);
  put64(f + 48, dg);
  put64(f + 56, (uint64_t)owner);
  out->digest = dg;
}

// Position-independent signature of the replicated list (what must agree
// across DP ranks before any offset is assigned).
static uint64_t signature_digest(const std::vector<TensorRef>& ts) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (auto& t : ts) {
    uint8_t meta[4 + 8 + 64];
    meta[0] = t.dtype;
    meta[1] = t.section;
    meta[2] = t.ndim;
    meta[3] = 0;
    memcpy(meta + 4, &t.nbytes, 8);
    memcpy(meta + 12, t.shape, 64);
    h = fnv1a64(meta, sizeof(meta), h);
    h = fnv1a64((const uint8_t*)t.name.data(), t.name.size(), h);
    uint8_t sep = 0;
    h = fnv1a64(&sep, 1, h);
  }
  return h;
}

void plan_local_facts(const std::vector<TensorRef>& rep, const std::vector<TensorRef>& loc,
                      uint32_t align, LocalFacts* out) {
  uint64_t lb = header_len(loc.size(), 0, names_bytes(loc), align);
  for (auto& t : loc) lb += round_up(t.nbytes, align);
  uint64_t rb = 0;
  for (auto& t : rep) rb += round_up(t.nbytes, align);
  out->region_bytes = lb;
  out->n_local = loc.size();
  out->digest = signature_digest(rep);
  out->rep_bytes = rb;
}

void rep_partition(uint64_t Q, int k, uint32_t writer_stride, int w, uint64_t* first_page,
                   uint64_t* n_pages) {
  const uint64_t s = writer_stride > 1 ? writer_stride : 1;
  const uint64_t nw = ((uint64_t)k + s - 1) / s;  // writers: ranks 0, s, 2s, ...
  const uint64_t q = Q / nw, rem = Q % nw;
  if ((uint64_t)w % s) {  // not a writer: empty range at the next writer's start
    const uint64_t i = (uint64_t)w / s + 1;
    *first_page = i >= nw ? Q : i * q + std::min<uint64_t>(i, rem);
    *n_pages = 0;
    return;
  }
  const uint64_t i = (uint64_t)w / s;
  *first_page = i * q + std::min<uint64_t>(i, rem);
  *n_pages = q + (i < rem ? 1 : 0);
}

void rep_share(const Plan& p, int w, uint64_t* off, uint64_t* bytes) {
  uint64_t f = 0, n = 0;
  rep_partition(p.rep_bytes / p.unit, p.k, p.writer_stride, w, &f, &n);
  *off = f * p.unit;
  *bytes = n * p.unit;
}

int plan_build(const std::vector<TensorRef>& rep, const std::vector<TensorRef>& loc,
               uint32_t align, int rank, int k, uint32_t writer_stride, bool balance_bytes,
               const std::vector<LocalFacts>& all, Plan* p) {
  for (int r = 1; r < k; ++r)
    if (all[r].digest != all[0].digest || all[r].rep_bytes != all[0].rep_bytes)
      return FP_EMISMATCH;
  bool has_local = false;
  for (int r = 0; r < k; ++r) has_local |= all[r].n_local > 0;
  const uint64_t n_reg = has_local ? (uint64_t)k : 0;
  p->align = align;
  p->unit = balance_bytes ? 1 : align;
  p->writer_stride = writer_stride > 1 ? writer_stride : 1;
  p->rank = rank;
  p->k = k;
  p->header_bytes = header_len(rep.size(), n_reg, names_bytes(rep), align);
  uint64_t cur = p->header_bytes;
  p->rep_off.clear();
  for (auto& t : rep) {
    p->rep_off.push_back(cur);
    cur += round_up(t.nbytes, align);
  }
  p->rep_bytes = cur;
  p->regions.clear();
  for (uint64_t r = 0; r < n_reg; ++r) {
    p->regions.push_back({cur, all[r].region_bytes});
    cur += all[r].region_bytes;
  }
  p->image_bytes = cur;
  encode_header(rep, p->rep_off, p->regions, align, p->image_bytes, -1,
                has_local ? kFlagHasLocal : 0, &p->ghdr);
  p->digest = p->ghdr.digest;
  p->loc_off.clear();
  p->lhdr.bytes.clear();
  if (has_local) {
    const uint64_t start = p->regions[rank].first;
    uint64_t c = start + header_len(loc.size(), 0, names_bytes(loc), align);
    for (auto& t : loc) {
      p->loc_off.push_back(c);
      c += round_up(t.nbytes, align);
    }
    if (c - start != p->regions[rank].second) return FP_EMISMATCH;
    encode_header(loc, p->loc_off, {}, align, c - start, rank, kFlagLocal, &p->lhdr);
  }
  // partition of the replicated region: Q units (pages, or bytes) over the
  // writers, contiguous in rank order, sizes differ by <= 1 unit, lowest
  // writers take the extras
  uint64_t first = 0, nb = 0;
  rep_share(*p, rank, &first, &nb);
  p->extents.clear();
  uint64_t fo = 0;
  if (nb) {
    p->extents.push_back({first, 0, nb});
    fo = nb;
  }
  if (has_local) {
    p->extents.push_back({p->regions[rank].first, fo, p->regions[rank].second});
    fo += p->regions[rank].second;
  }
  p->shard_bytes = fo;
  return 0;
}

void plan_pieces(Plan* p, const std::vector<TensorRef>& rep, const std::vector<TensorRef>& loc,
                 uint64_t hdr_base) {
  const uint64_t A = p->align;
  std::vector<Piece> all;
  all.push_back({0, p->header_bytes, hdr_base});
  for (size_t i = 0; i < rep.size(); ++i) {
    const uint64_t o = p->rep_off[i], n = rep[i].nbytes;
    if (n) all.push_back({o, n, rep[i].ptr});
    const uint64_t pad = round_up(n, A) - n;
    if (pad) all.push_back({o + n, pad, 0});
  }
  if (!p->regions.empty()) {
    const uint64_t start = p->regions[p->rank].first;
    all.push_back({start, (uint64_t)p->lhdr.bytes.size(),
                   hdr_base ? hdr_base + p->ghdr.bytes.size() : 0});
    for (size_t i = 0; i < loc.size(); ++i) {
      const uint64_t o = p->loc_off[i], n = loc[i].nbytes;
      if (n) all.push_back({o, n, loc[i].ptr});
      const uint64_t pad = round_up(n, A) - n;
      if (pad) all.push_back({o + n, pad, 0});
    }
  }
  // clip to this rank's extents (pieces and extents are both image-ordered)
  p->pieces.clear();
  size_t j = 0;
  for (const Extent& e : p->extents) {
    const uint64_t lo = e.image_off, hi = e.image_off + e.len;
    while (j < all.size() && all[j].image_off + all[j].len <= lo) ++j;
    for (size_t i = j; i < all.size() && all[i].image_off < hi; ++i) {
      const uint64_t a = std::max(lo, all[i].image_off);
      const uint64_t b = std::min(hi, all[i].image_off + all[i].len);
      if (a >= b) continue;
      const uint64_t src = all[i].src ? all[i].src + (a - all[i].image_off) : 0;
      p->pieces.push_back({a, b - a, src});
    }
  }
}

void plan_items(const Plan& p, uint64_t slot_bytes, uint64_t group_bytes,
                std::vector<Item>* items, std::vector<uint32_t>* item_lo, uint64_t max_item) {
  const uint64_t per_group = group_bytes / slot_bytes;
  items->clear();
  item_lo->clear();
  const uint64_t n_chunks = (p.shard_bytes + slot_bytes - 1) / slot_bytes;
  // map pieces to file space, then cut at chunk boundaries and kTile
  size_t e = 0;
  uint64_t chunk = 0;
  item_lo->push_back(0);
  for (const Piece& pc : p.pieces) {
    while (pc.image_off >= p.extents[e].image_off + p.extents[e].len) ++e;
    uint64_t fo = p.extents[e].file_off + (pc.image_off - p.extents[e].image_off);
    uint64_t left = pc.len, src = pc.src;
    while (left) {
      while (fo >= (chunk + 1) * slot_bytes) {
        item_lo->push_back((uint32_t)items->size());
        ++chunk;
      }
      const uint64_t cend = (chunk + 1) * slot_bytes;
      const uint64_t gbase = chunk / per_group * per_group * slot_bytes;
      uint64_t n = std::min<uint64_t>({left, max_item, cend - fo});
      // tile-sized items never cross a kTile boundary of their group (the
      // fused pack + CRC kernel works on whole tiles)
      if (max_item <= kTile) n = std::min<uint64_t>(n, kTile - (fo - gbase) % kTile);
      items->push_back({src, (uint32_t)(fo - gbase), (uint32_t)n});
      fo += n;
      left -= n;
      if (src) src += n;
    }
  }
  while (item_lo->size() < n_chunks + 1) item_lo->push_back((uint32_t)items->size());
}

void plan_tiles(const std::vector<Item>& items, const std::vector<uint32_t>& item_lo,
                uint64_t shard_bytes, uint64_t slot_bytes, uint64_t group_bytes,
                std::vector<uint32_t>* tile_lo, std::vector<uint64_t>* group_tile_off) {
  const uint64_t per_group = std::max<uint64_t>(1, group_bytes / slot_bytes);
  const uint64_t n_chunks = item_lo.size() - 1;
  tile_lo->clear();
  group_tile_off->clear();
  for (uint64_t c0 = 0; c0 < n_chunks; c0 += per_group) {
    const uint64_t c1 = std::min(c0 + per_group, n_chunks);
    const uint64_t gbytes = std::min(c1 * slot_bytes, shard_bytes) - c0 * slot_bytes;
    const uint64_t nt = (gbytes + kTile - 1) / kTile;
    group_tile_off->push_back(tile_lo->size());
    const uint32_t i0 = item_lo[c0], i1 = item_lo[c1];
    uint32_t i = i0;
    for (uint64_t t = 0; t <= nt; ++t) {  // first item whose dst >= t * kTile
      while (i < i1 && items[i].dst < t * kTile) ++i;
      tile_lo->push_back(i - i0);
    }
  }
}

}  // namespace fp
