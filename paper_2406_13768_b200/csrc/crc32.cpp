// CRC-32 (IEEE 802.3, reflected polynomial 0xEDB88320, init and xorout
// 0xFFFFFFFF — the checksum of zlib's crc32()) for per-shard integrity
// records in the manifest (SPEC.md S:157 checksums in the
// manifest). The GPU computes *raw* CRCs (init 0, no xorout), which are
// linear in the data: R(A||B) = R(A)*x^(8|B|) xor R(B) (mod P), zero bytes
// contribute nothing and leading zeros are invisible. A standard CRC is
// recovered as crc(M) = R(M) xor crc(0^|M|). Polynomial products are done in
// the reflected bit order (bit 31 = x^0). gf_mul and gf_x8n are the standard
// GF(2) routines zlib uses for crc32_combine (zlib's crc32.c multmodp and
// x2nmodp, permissive zlib license), restated here.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>

#include "fp_internal.h"

namespace fp {

static constexpr uint32_t kPoly = 0xEDB88320u;

uint32_t gf_mul(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
  }
  return p;
}

static uint32_t x2n[32];  // x^(2^k) mod P
static std::once_flag x2n_once;

static void init_x2n() {
  std::call_once(x2n_once, [] {
    uint32_t p = 1u << 30;  // x^1
    x2n[0] = p;
    for (int k = 1; k < 32; ++k) x2n[k] = p = gf_mul(p, p);
  });
}

uint32_t gf_x8n(uint64_t n) {  // x^(8n) mod P
  init_x2n();
  uint32_t p = 1u << 31;  // x^0
  int k = 3;
  while (n) {
    if (n & 1) p = gf_mul(x2n[k & 31], p);
    n >>= 1;
    ++k;
  }
  return p;
}

static uint32_t tab[8][256];
static std::once_flag tab_once;

static void init_tab() {
  std::call_once(tab_once, [] {
    for (uint32_t b = 0; b < 256; ++b) {
      uint32_t c = b;
      for (int i = 0; i < 8; ++i) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
      tab[0][b] = c;
    }
    for (int t = 1; t < 8; ++t)
      for (uint32_t b = 0; b < 256; ++b) tab[t][b] = (tab[t - 1][b] >> 8) ^ tab[0][tab[t - 1][b] & 0xFF];
  });
}

const uint32_t* crc_tables8() {
  init_tab();
  return &tab[0][0];
}

// raw CRC register update (no init / xorout applied here), slicing-by-8
uint32_t crc_raw_update(uint32_t c, const uint8_t* p, uint64_t n) {
  init_tab();
  while (n && ((uintptr_t)p & 7)) {
    c = (c >> 8) ^ tab[0][(c ^ *p++) & 0xFF];
    --n;
  }
  while (n >= 8) {
    uint64_t w;
    memcpy(&w, p, 8);
    const uint32_t lo = (uint32_t)w ^ c, hi = (uint32_t)(w >> 32);
    c = tab[7][lo & 0xFF] ^ tab[6][(lo >> 8) & 0xFF] ^ tab[5][(lo >> 16) & 0xFF] ^
        tab[4][lo >> 24] ^ tab[3][hi & 0xFF] ^ tab[2][(hi >> 8) & 0xFF] ^
        tab[1][(hi >> 16) & 0xFF] ^ tab[0][hi >> 24];
    p += 8;
    n -= 8;
  }
  while (n--) c = (c >> 8) ^ tab[0][(c ^ *p++) & 0xFF];
  return c;
}

// four 256-entry tables for the product by the constant k: M[i][b] = k*(b << 8i)
static void mul_tables(uint32_t k, uint32_t* m) {
  for (int i = 0; i < 4; ++i)
    for (uint32_t b = 0; b < 256; ++b) m[256 * i + b] = gf_mul(k, b << (8 * i));
}

std::vector<uint32_t> crc_device_tables() {
  init_tab();
  std::vector<uint32_t> t(kTabWords, 0);
  for (int k = 0; k < 4; ++k) memcpy(&t[kTabS4 + 256 * k], tab[k], 256 * 4);
  for (uint32_t l = 0; l < 32; ++l) t[kTabLaneK + l] = gf_x8n(128ull * (31 - l));
  const uint32_t x512 = gf_x8n(512);
  for (uint32_t j = 0; j < 8; ++j)
    for (uint32_t n = 0; n < 16; ++n) {
      t[kTabNibX + j * 16 + n] = gf_mul(x512, n << (4 * j));
      for (uint32_t l = 0; l < 32; ++l)
        t[kTabNibK + l * 128 + j * 16 + n] = gf_mul(gf_x8n(16ull * (31 - l)), n << (4 * j));
    }
  return t;
}

uint32_t crc_zeros(uint64_t n) {  // standard CRC-32 of n zero bytes
  return gf_mul(gf_x8n(n), 0xFFFFFFFFu) ^ 0xFFFFFFFFu;
}

// ---------------------------------------------------------------------------
// ExtentCrc
// ---------------------------------------------------------------------------
static uint32_t page_tab[1024];  // product by x^(8*4096), four 256-entry tables
static std::once_flag page_tab_once;

static inline uint32_t mul_page(uint32_t a) {
  return page_tab[a & 255] ^ page_tab[256 + ((a >> 8) & 255)] ^ page_tab[512 + ((a >> 16) & 255)] ^
         page_tab[768 + (a >> 24)];
}

void ExtentCrc::reset(const std::vector<Extent>& ext) {
  std::call_once(page_tab_once, [] { mul_tables(gf_x8n(4096), page_tab); });
  beg_.clear();
  len_.clear();
  for (const Extent& e : ext) {
    beg_.push_back(e.file_off);
    len_.push_back(e.len);
  }
  done_.assign(beg_.size(), 0);
  raw_.assign(beg_.size(), 0);
  cur_ = 0;
  ok_ = true;
}

size_t ExtentCrc::find(uint64_t fo) {
  if (cur_ >= beg_.size() || fo < beg_[cur_]) cur_ = 0;
  while (cur_ < beg_.size() && fo >= beg_[cur_] + len_[cur_]) ++cur_;
  return cur_;
}

bool ExtentCrc::pages_ok(uint64_t fo, uint64_t n) const {
  if (fo % 4096 || n % 4096) return false;
  for (size_t i = 0; i < beg_.size(); ++i) {
    const uint64_t b = beg_[i], e = beg_[i] + len_[i];
    if ((b > fo && b < fo + n && b % 4096) || (e > fo && e < fo + n && e % 4096)) return false;
  }
  return true;
}

void ExtentCrc::add_pages(uint64_t fo, const uint32_t* pc, uint64_t n_pages) {
  for (uint64_t p = 0; p < n_pages; ++p, fo += 4096) {
    const size_t i = find(fo);
    if (i >= beg_.size() || fo != beg_[i] + done_[i] || done_[i] + 4096 > len_[i]) {
      ok_ = false;
      return;
    }
    raw_[i] = mul_page(raw_[i]) ^ pc[p];
    done_[i] += 4096;
  }
}

void ExtentCrc::add_bytes(uint64_t fo, const uint8_t* p, uint64_t n) {
  while (n) {
    const size_t i = find(fo);
    if (i >= beg_.size() || fo != beg_[i] + done_[i]) {
      ok_ = false;
      return;
    }
    const uint64_t m = std::min<uint64_t>(n, len_[i] - done_[i]);
    raw_[i] = crc_raw_update(raw_[i], p, m);
    done_[i] += m;
    fo += m;
    p += m;
    n -= m;
  }
}

void ExtentCrc::add_raw(uint64_t fo, uint64_t n, uint32_t raw) {
  if (!n) return;
  const size_t i = find(fo);
  if (i >= beg_.size() || fo != beg_[i] + done_[i] || done_[i] + n > len_[i]) {
    ok_ = false;
    return;
  }
  raw_[i] = gf_mul(gf_x8n(n), raw_[i]) ^ raw;
  done_[i] += n;
}

bool ExtentCrc::complete() const {
  for (size_t i = 0; i < beg_.size(); ++i)
    if (done_[i] != len_[i]) return false;
  return ok_;
}

uint32_t ExtentCrc::extent_crc(size_t i) const { return raw_[i] ^ crc_zeros(len_[i]); }

uint32_t ExtentCrc::file_crc() const {
  uint32_t r = 0;
  uint64_t tot = 0;
  for (size_t i = 0; i < beg_.size(); ++i) {
    r = gf_mul(gf_x8n(len_[i]), r) ^ raw_[i];
    tot += len_[i];
  }
  return r ^ crc_zeros(tot);
}

}  // namespace fp
