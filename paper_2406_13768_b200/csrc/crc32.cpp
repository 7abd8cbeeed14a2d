// CRC-32 (IEEE 802.3, reflected polynomial 0xEDB88320, init and xorout
// 0xFFFFFFFF — the checksum of zlib's crc32()) for per-shard integrity
// records in the manifest (SPEC.md S:157 checksums in the
// manifest). The GPU computes *raw* CRCs (init 0, no xorout), which are
// linear in the data: R(A||B) = R(A)*x^(8|B|) xor R(B) (mod P), zero bytes
// contribute nothing and leading zeros are invisible. A standard CRC is
// recovered as crc(M) = R(M) xor crc(0^|M|). Polynomial products are done in
// the reflected bit order (bit 31 = x^0), as in zlib's crc32_combine.
#include <cstdint>
#include <cstring>

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
static bool x2n_ready = false;

static void init_x2n() {
  if (x2n_ready) return;
  uint32_t p = 1u << 30;  // x^1
  x2n[0] = p;
  for (int k = 1; k < 32; ++k) x2n[k] = p = gf_mul(p, p);
  x2n_ready = true;
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
static bool tab_ready = false;

static void init_tab() {
  if (tab_ready) return;
  for (uint32_t b = 0; b < 256; ++b) {
    uint32_t c = b;
    for (int i = 0; i < 8; ++i) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
    tab[0][b] = c;
  }
  for (int t = 1; t < 8; ++t)
    for (uint32_t b = 0; b < 256; ++b) tab[t][b] = (tab[t - 1][b] >> 8) ^ tab[0][tab[t - 1][b] & 0xFF];
  tab_ready = true;
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
  for (uint32_t v = 0; v < kLaneLevels; ++v) mul_tables(gf_x8n(32ull << v), &t[kTabLane + 1024 * v]);
  for (uint32_t j = 0; j < kCrcPageLevels; ++j) mul_tables(gf_x8n(4096ull << j), &t[kTabPage + 1024 * j]);
  return t;
}

uint32_t crc_zeros(uint64_t n) {  // standard CRC-32 of n zero bytes
  return gf_mul(gf_x8n(n), 0xFFFFFFFFu) ^ 0xFFFFFFFFu;
}

}  // namespace fp
