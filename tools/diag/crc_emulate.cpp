// Host emulation of the device CRC-32 scheme (pack.cu: page_crc_warp as used
// by fp_crc_pages / fp_crc_pages_tma / fp_pack_crc) and the host fold of page
// CRCs per extent (ExtentCrc): the same table blob (crc_device_tables), the
// same chain split and lane tree, compared with the plain slicing CRC
// (crc_raw_update) on random pages, for several page and extent counts. Built and run by
// tests/test_crc_scheme_cpu.py (no GPU needed).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "fp_internal.h"
using namespace fp;
static uint32_t mul_tab(const uint32_t* m, uint32_t a) {
  return m[a & 255] ^ m[256 + ((a >> 8) & 255)] ^ m[512 + ((a >> 16) & 255)] ^ m[768 + (a >> 24)];
}
int main() {
  auto T = crc_device_tables();
  const uint32_t* t0 = &T[kTabS4], *t1 = t0 + 256, *t2 = t0 + 512, *t3 = t0 + 768;
  for (uint32_t n_pages : {1u, 2u, 3u, 37u, 1024u, 1500u, 2049u}) for (uint32_t ppc : {1u, 3u, 16u, 1024u, 2048u}) {
    std::vector<uint8_t> buf((size_t)n_pages * 4096);
    for (auto& b : buf) b = rand() & 255;
    std::vector<uint32_t> pc(n_pages);
    for (uint32_t pg = 0; pg < n_pages; ++pg) {
      uint32_t lc[32];
      const int chains = (pg & 1) ? 4 : 1;  // both variants of page_crc_warp
      for (int lane = 0; lane < 32; ++lane) {
        const uint32_t* w = (const uint32_t*)(buf.data() + (size_t)pg * 4096 + lane * 128);
        uint32_t c[4] = {0,0,0,0};
        const int kw = 32 / chains;
        for (int q = 0; q < kw; ++q) for (int j = 0; j < chains; ++j) { uint32_t x = c[j] ^ w[kw*j + q]; c[j] = t3[x & 255] ^ t2[(x >> 8) & 255] ^ t1[(x >> 16) & 255] ^ t0[x >> 24]; }
        if (chains == 4) {
          uint32_t ab = mul_tab(&T[kTabLane], c[0]) ^ c[1], cd = mul_tab(&T[kTabLane], c[2]) ^ c[3];
          lc[lane] = mul_tab(&T[kTabLane + 1024], ab) ^ cd;
        } else {
          lc[lane] = c[0];
        }
      }
      for (int v = 0; v < 5; ++v) {
        uint32_t nc[32];
        for (int l = 0; l < 32; ++l) { uint32_t o = l + (1 << v) < 32 ? lc[l + (1 << v)] : lc[l];
          nc[l] = ((l & ((2 << v) - 1)) == 0) ? mul_tab(&T[kTabLane + 1024 * (2 + v)], lc[l]) ^ o : lc[l]; }
        for (int l = 0; l < 32; ++l) lc[l] = nc[l];
      }
      pc[pg] = lc[0];
      if (pc[pg] != crc_raw_update(0, buf.data() + (size_t)pg * 4096, 4096)) { printf("page mismatch\n"); return 1; }
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
