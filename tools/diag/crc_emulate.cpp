// Host emulation of the device CRC-32 scheme (pack.cu: page_crc_warp as used
// by fp_crc_pages / fp_crc_pages_tma / fp_pack_bulk_crc, and fp_pack_lsu_crc) and the host fold of page
// CRCs per extent (ExtentCrc): the same table blob (crc_device_tables), the
// same per-lane chain and register lane combine, compared with the plain slicing CRC
// (crc_raw_update) on random pages, for several page and extent counts. Built and run by
// tests/test_crc_scheme_cpu.py (no GPU needed).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "fp_internal.h"
using namespace fp;
int main() {
  auto T = crc_device_tables();
  const uint32_t* t0 = &T[kTabS4], *t1 = t0 + 256, *t2 = t0 + 512, *t3 = t0 + 768;
  for (uint32_t n_pages : {1u, 2u, 3u, 37u, 1024u, 1500u, 2049u}) for (uint32_t ppc : {1u, 3u, 16u, 1024u, 2048u}) {
    std::vector<uint8_t> buf((size_t)n_pages * 4096);
    for (auto& b : buf) b = rand() & 255;
    std::vector<uint32_t> pc(n_pages);
    for (uint32_t pg = 0; pg < n_pages; ++pg) {
      // pack.cu page_crc_warp / fp_crc_pages_tma: one slicing-by-4 chain per
      // lane over its 128 bytes, then R_l * K_l (K_l = x^(8*128*(31-l)), the
      // product through kv[i] = K_l * x^i as lane_k_init / gf_mul_k do), XOR
      uint32_t crc = 0;
      for (int lane = 0; lane < 32; ++lane) {
        const uint32_t* w = (const uint32_t*)(buf.data() + (size_t)pg * 4096 + lane * 128);
        // two chains (words 0..15, 16..31) joined by x^(8*64), as the kernels do
        uint32_t c0 = 0, c1 = 0;
        for (int q = 0; q < 16; ++q) {
          uint32_t x = c0 ^ w[q]; c0 = t3[x & 255] ^ t2[(x >> 8) & 255] ^ t1[(x >> 16) & 255] ^ t0[x >> 24];
          x = c1 ^ w[16 + q]; c1 = t3[x & 255] ^ t2[(x >> 8) & 255] ^ t1[(x >> 16) & 255] ^ t0[x >> 24];
        }
        const uint32_t c = gf_mul(c0, gf_x8n(64)) ^ c1;
        uint32_t kv[32];
        kv[0] = T[kTabLaneK + lane];
        for (int i = 1; i < 32; ++i) kv[i] = (kv[i - 1] >> 1) ^ ((kv[i - 1] & 1) ? 0xEDB88320u : 0u);
        uint32_t p = 0;
        for (int i = 0; i < 32; ++i) p ^= (0u - ((c >> (31 - i)) & 1u)) & kv[i];
        crc ^= p;
      }
      pc[pg] = crc;
      if (pc[pg] != crc_raw_update(0, buf.data() + (size_t)pg * 4096, 4096)) { printf("page mismatch\n"); return 1; }
      // pack.cu fp_pack_lsu_crc: lane l holds the 16-B chunks 32u + l
      // (u = 0..7, the coalesced load pattern); a chain per chunk from 0, the
      // chunks joined by Horner with x^(8*512) and the lane's term times
      // x^(8*16*(31-l)), both products as 8 nibble lookups (kTabNibX/kTabNibK)
      auto nib = [&](uint32_t a, const uint32_t* nt) {
        uint32_t r = 0;
        for (int j = 0; j < 8; ++j) r ^= nt[j * 16 + ((a >> (4 * j)) & 15)];
        return r;
      };
      uint32_t crc2 = 0;
      for (int lane = 0; lane < 32; ++lane) {
        uint32_t s = 0;
        for (int u = 0; u < 8; ++u) {
          const uint32_t* w = (const uint32_t*)(buf.data() + (size_t)pg * 4096 + (32 * u + lane) * 16);
          uint32_t c = 0;
          for (int q = 0; q < 4; ++q) {
            const uint32_t x = c ^ w[q];
            c = t3[x & 255] ^ t2[(x >> 8) & 255] ^ t1[(x >> 16) & 255] ^ t0[x >> 24];
          }
          s = (u ? nib(s, &T[kTabNibX]) : 0u) ^ c;
        }
        crc2 ^= nib(s, &T[kTabNibK + lane * 128]);
      }
      if (crc2 != crc) { printf("lsu page mismatch\n"); return 1; }
    }
    // host fold (ExtentCrc): the pages split into extents at page boundaries
    // (every ppc pages), some runs added as pages and some as bytes; each
    // extent's CRC and the file CRC == the standard CRC-32 of those bytes
    std::vector<Extent> ext;
    for (uint32_t p0 = 0; p0 < n_pages; p0 += ppc)
      ext.push_back({0, (uint64_t)p0 * 4096, (uint64_t)std::min(ppc, n_pages - p0) * 4096});
    ExtentCrc acc;
    acc.reset(ext);
    for (uint32_t p0 = 0; p0 < n_pages;) {
      const uint32_t n = std::min<uint32_t>(n_pages - p0, 1 + rand() % 700);
      if (rand() & 3) acc.add_pages((uint64_t)p0 * 4096, pc.data() + p0, n);
      else acc.add_bytes((uint64_t)p0 * 4096, buf.data() + (size_t)p0 * 4096, (size_t)n * 4096);
      p0 += n;
    }
    if (!acc.complete()) { printf("fold incomplete\n"); return 1; }
    auto std_crc = [](const uint8_t* p, size_t n) { return crc_raw_update(0xFFFFFFFFu, p, n) ^ 0xFFFFFFFFu; };
    for (size_t i = 0; i < ext.size(); ++i)
      if (acc.extent_crc(i) != std_crc(buf.data() + ext[i].file_off, ext[i].len)) { printf("extent mismatch n=%u ppc=%u i=%zu\n", n_pages, ppc, i); return 1; }
    if (acc.file_crc() != std_crc(buf.data(), buf.size())) { printf("file mismatch\n"); return 1; }
  }
  printf("emulation ok\n");
}
