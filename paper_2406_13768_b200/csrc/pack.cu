// Pack / unpack kernels for sm_100a.
//
// The pack kernel gathers one chunk of this rank's shard — fragments of many
// device tensors (bf16 params/grads, fp32 master/m/v), header pages and zero
// padding — into a contiguous, alignment-padded device slab that the copy
// engine then moves to a pinned host ring slot (§4.1: GPU ->
// page-locked CPU memory -> NVMe, double buffered; the paper moved each
// serialized tensor separately, §5.1). Work arrives as a flat list
// of <= 32 KiB items {src, slab offset, len} precomputed on the host at setup
// (the partition is fixed before the first iteration), so the kernels
// do no searching: they are pure HBM streams (1 B read + 1 B written per image
// byte).
//
//  fp_pack_v4   : LSU path. 16-B vector loads (ld.global.nc.L1::no_allocate)
//                 and stores, 8 loads in flight per thread, co-aligned
//                 head/body/tail handling; byte path for mutually misaligned
//                 pointers (odd storage offsets).
//  fp_pack_bulk : TMA-engine path. One elected thread per CTA streams items
//                 through a 6-stage shared-memory ring with
//                 cp.async.bulk (G2S, mbarrier complete_tx) and
//                 cp.async.bulk (S2G, bulk_group); the other warps handle
//                 zero fill, vector tails and misaligned items with the LSU.
//                 (FP_NO_CRC only; with CRCs the default is:)
//  fp_pack_bulk_crc : the same TMA-engine pack computing the page CRC-32s
//                 from its shared-memory stages (see below).
//  fp_unpack_v4 : load path, slab -> tensors (zero items skipped).
#include <cuda.h>  // CUtensorMap (the encode entry point is fetched at run time)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "fp_internal.h"

// Debug builds (FP_NVCC_FLAGS=-DFP_KERNEL_ASSERTS): device-side checks of the
// work-item invariants the kernels rely on (items inside their 32 KiB tile and
// inside the group); a violation prints and traps (the launch then fails).
#ifdef FP_KERNEL_ASSERTS
#include <cstdio>
#define FP_KASSERT(c)                                                               \
  do {                                                                              \
    if (!(c)) {                                                                     \
      printf("FP_KASSERT %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,      \
             (int)blockIdx.x, (int)threadIdx.x, #c);                                \
      __trap();                                                                     \
    }                                                                               \
  } while (0)
#else
#define FP_KASSERT(c) \
  do {                \
  } while (0)
#endif

namespace fp {
namespace {

constexpr int kV4Threads = 256;
constexpr int kV4Unroll = 8;  // 256 thr x 8 x 16 B = 32 KiB = kTile per pass

// Streaming accesses (SURVEY §8(a'): the pack must not evict the training
// stream's L2 working set): loads bypass L1 and, like the stores, carry an
// L2 evict-first policy — every byte is touched once (the slab is re-read by
// the copy engine, but a 1 GiB group exceeds the 126 MB L2 anyway).
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile(
      "{\n"
      ".reg .b64 pol;\n"
      "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], pol;\n"
      "}\n"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}
__device__ __forceinline__ void st_v4(uint4* p, const uint4& v) {
  asm volatile(
      "{\n"
      ".reg .b64 pol;\n"
      "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      "st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, pol;\n"
      "}\n" ::"l"(p),
      "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
      : "memory");
}

// coherent 16-B load (data another agent may have written while this kernel
// was already running: the peer-exchange unpack)
__device__ __forceinline__ uint4 ld_coherent(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Mutually misaligned src / dst (src - dst not a multiple of 16: odd storage
// offsets, byte-granular shard starts): 16-B aligned stores; each destination
// vector is funnel-shifted out of the two aligned source vectors that cover
// it (both loads are aligned 16-B loads inside the 16-B blocks that hold the
// needed bytes, so they never leave the source allocation's granule).
template <bool kCoherent>
__device__ __forceinline__ void copy_shifted(uint8_t* __restrict__ dst,
                                             const uint8_t* __restrict__ src, uint32_t len, int t,
                                             int nthr) {
  uint32_t head = (16 - (uint32_t)((uintptr_t)dst & 15)) & 15;
  if (head > len) head = len;
  if ((uint32_t)t < head) dst[t] = src[t];
  const uint32_t n16 = (len - head) >> 4;
  if (n16) {
    const uint8_t* s = src + head;
    const uint32_t sh = (uint32_t)((uintptr_t)s & 15);  // != 0 here
    const uint4* a16 = reinterpret_cast<const uint4*>(s - sh);
    uint4* d16 = reinterpret_cast<uint4*>(dst + head);
    const uint32_t q = sh >> 2, r8 = (sh & 3) * 8;
    for (uint32_t j = t; j < n16; j += nthr) {
      const uint4 x = kCoherent ? ld_coherent(a16 + j) : ld_stream(a16 + j);
      const uint4 y = kCoherent ? ld_coherent(a16 + j + 1) : ld_stream(a16 + j + 1);
      const uint32_t w[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
      uint32_t o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        // words q+i and q+i+1 of the 32-byte window (q uniform per item)
        const uint32_t lo = q == 0 ? w[i] : q == 1 ? w[i + 1] : q == 2 ? w[i + 2] : w[i + 3];
        const uint32_t hi = q == 0 ? w[i + 1] : q == 1 ? w[i + 2] : q == 2 ? w[i + 3] : w[i + 4];
        o[i] = __funnelshift_r(lo, hi, r8);
      }
      st_v4(d16 + j, make_uint4(o[0], o[1], o[2], o[3]));
    }
  }
  const uint32_t done = head + (n16 << 4);
  for (uint32_t i = done + t; i < len; i += nthr) dst[i] = src[i];
}

// Copy `len` bytes src -> dst with `nthr` threads (index t). src == nullptr
// means zero fill. Vector body when src and dst share the same 16-B phase.
// kCoherent: plain (coherent) loads instead of the read-only .nc path.
template <bool kCoherent = false>
__device__ __forceinline__ void copy_bytes(uint8_t* __restrict__ dst,
                                           const uint8_t* __restrict__ src, uint32_t len,
                                           int t, int nthr) {
  const uint32_t phase = (uint32_t)((uintptr_t)dst & 15);
  const bool coaligned = !src || (((uintptr_t)src & 15) == phase);
  if (!coaligned) {
    copy_shifted<kCoherent>(dst, src, len, t, nthr);
    return;
  }
  uint32_t head = (16 - phase) & 15;
  if (head > len) head = len;
  if ((uint32_t)t < head) dst[t] = src ? src[t] : 0;
  const uint32_t n16 = (len - head) >> 4;
  uint4* d16 = reinterpret_cast<uint4*>(dst + head);
  if (src) {
    const uint4* s16 = reinterpret_cast<const uint4*>(src + head);
    for (uint32_t base = 0; base < n16; base += (uint32_t)nthr * kV4Unroll) {
      uint4 v[kV4Unroll];
#pragma unroll
      for (int u = 0; u < kV4Unroll; ++u) {
        const uint32_t j = base + (uint32_t)u * nthr + t;
        if (j < n16) v[u] = kCoherent ? ld_coherent(s16 + j) : ld_stream(s16 + j);
      }
#pragma unroll
      for (int u = 0; u < kV4Unroll; ++u) {
        const uint32_t j = base + (uint32_t)u * nthr + t;
        if (j < n16) st_v4(d16 + j, v[u]);
      }
    }
  } else {
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (uint32_t j = t; j < n16; j += nthr) st_v4(d16 + j, z);
  }
  const uint32_t done = head + (n16 << 4);
  const uint32_t tail = len - done;
  if ((uint32_t)t < tail) dst[done + t] = src ? src[done + t] : 0;
}

__global__ void __launch_bounds__(kV4Threads) fp_pack_v4(const Item* __restrict__ items,
                                                         uint32_t n, uint8_t* __restrict__ slab) {
  // the next item's descriptor is loaded before the current item's data, so
  // its latency hides behind the copy instead of opening a bubble per item
  uint32_t i = blockIdx.x;
  if (i >= n) return;
  Item it = items[i];
  for (;;) {
    const uint32_t nx = i + gridDim.x;
    Item nit = {0, 0, 0};
    if (nx < n) nit = items[nx];
    copy_bytes(slab + it.dst, reinterpret_cast<const uint8_t*>(it.src), it.len, threadIdx.x,
               kV4Threads);
    if (nx >= n) break;
    i = nx;
    it = nit;
  }
}

__global__ void __launch_bounds__(kV4Threads) fp_unpack_v4(const Item* __restrict__ items,
                                                           uint32_t n,
                                                           const uint8_t* __restrict__ slab) {
  for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
    const Item it = items[i];
    if (!it.src) continue;  // padding: nothing to restore
    copy_bytes(reinterpret_cast<uint8_t*>(it.src), slab + it.dst, it.len, threadIdx.x,
               kV4Threads);
  }
}

// Parallel-load exchange over peer memory (§4.2: each rank
// "(i) loads its checkpoint partition ... into GPU memory, and (ii) performs
// an allgather"): every rank's replicated partition sits whole in its own
// device buffer (CUDA IPC-mapped into the peers, or the same address space
// for thread ranks); one launch per exchange chunk j scatters the chunk of
// EVERY writer straight from the writers' buffers into the local tensors (P2P
// loads over NVLink on a multi-GPU node), so the all-gather and the scatter
// are one pass with no gathered copy. The host launches it only once every
// writer's chunk j has landed (their ready flags). Item.len carries the
// writer index in bits 24..31; Item.dst is the offset inside the writer's
// chunk. Coherent loads: the buffers were written by other engines.
__global__ void __launch_bounds__(kV4Threads) fp_unpack_peer(const Item* __restrict__ items,
                                                             uint32_t n,
                                                             const PeerTab* __restrict__ tab,
                                                             uint32_t j, uint64_t ch_bytes) {
  for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
    const Item it = items[i];
    if (!it.src) continue;
    const uint32_t w = it.len >> 24, len = it.len & 0xFFFFFFu;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(tab->base[w]) + j * ch_bytes + it.dst;
    copy_bytes<true>(reinterpret_cast<uint8_t*>(it.src), src, len, threadIdx.x, kV4Threads);
  }
}

// ---------------------------------------------------------------------------
// bulk-async (TMA engine) variant
// ---------------------------------------------------------------------------
constexpr int kBulkStagesMax = 6;
constexpr int kBulkThreads = 128;
constexpr uint32_t kBulkStageBytes = kTile;  // one item per stage
template <int kBulkStages>
constexpr size_t bulk_smem() { return (size_t)kBulkStages * kBulkStageBytes + kBulkStages * 16; }

__device__ __forceinline__ bool bulk_ok(const Item& it) {
  return it.src && !(it.src & 15) && !(it.dst & 15) && it.len >= 16;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// kBulkStages = 6: one CTA per SM; 3: two CTAs per SM (FP_BULK_2CTA=1, ablation)
template <int kBulkStages>
__global__ void __launch_bounds__(kBulkThreads, kBulkStagesMax / kBulkStages)
    fp_pack_bulk(const Item* __restrict__ items, uint32_t n, uint8_t* __restrict__ slab) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + (size_t)kBulkStages * kBulkStageBytes);
  uint32_t* st_dst = reinterpret_cast<uint32_t*>(mbar + kBulkStages);
  uint32_t* st_len = st_dst + kBulkStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // contiguous item range of this CTA
  const uint32_t lo = (uint32_t)(((uint64_t)n * blockIdx.x) / gridDim.x);
  const uint32_t hi = (uint32_t)(((uint64_t)n * (blockIdx.x + 1)) / gridDim.x);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBulkStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // warp 0 walks the items 32 at a time (one coalesced descriptor load per
    // lane); lane 0 alone issues the bulk copies (L2 evict-first both ways).
    const uint64_t pol = evict_first_policy();
    uint32_t issued = 0, stored = 0;
    auto store_one = [&]() {
      const uint32_t s = stored % kBulkStages;
      const uint32_t parity = (stored / kBulkStages) & 1;
      const uint32_t bar = smem_u32(&mbar[s]);
      asm volatile(
          "{\n"
          ".reg .pred p;\n"
          "WAIT_%=:\n"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          "@!p bra WAIT_%=;\n"
          "}\n" ::"r"(bar),
          "r"(parity)
          : "memory");
      asm volatile(
          "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
              slab + st_dst[s]),
          "r"(smem_u32(smem + (size_t)s * kBulkStageBytes)), "r"(st_len[s]), "l"(pol)
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      ++stored;
    };
    for (uint32_t b = lo; b < hi; b += 32) {
      Item mine = {0, 0, 0};
      if (b + lane < hi) mine = items[b + lane];
      uint32_t mask = __ballot_sync(0xffffffffu, b + lane < hi && bulk_ok(mine));
      while (mask) {
        const int j = __ffs(mask) - 1;
        mask &= mask - 1;
        const uint64_t src = __shfl_sync(0xffffffffu, mine.src, j);
        const uint32_t dst = __shfl_sync(0xffffffffu, mine.dst, j);
        const uint32_t len = __shfl_sync(0xffffffffu, mine.len, j);
        if (lane == 0) {
          // keep <= kBulkStages-1 loads in flight: one stage of slack lets
          // the most recent store still be reading shared memory
          while (issued - stored >= (uint32_t)kBulkStages - 1) store_one();
          const uint32_t s = issued % kBulkStages;
          if (issued >= (uint32_t)kBulkStages)
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          const uint32_t bytes = len & ~15u;
          st_dst[s] = dst;
          st_len[s] = bytes;
          const uint32_t bar = smem_u32(&mbar[s]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                       "r"(bytes)
                       : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
              "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem + (size_t)s * kBulkStageBytes)),
              "l"(src), "r"(bytes), "r"(bar), "l"(pol)
              : "memory");
          ++issued;
        }
      }
    }
    if (lane == 0) {
      while (stored < issued) store_one();
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  } else {
    // LSU warps: zero fill, misaligned items, and the <16 B vector tails
    const int t = threadIdx.x - 32, nthr = kBulkThreads - 32;
    for (uint32_t i = lo; i < hi; ++i) {
      const Item it = items[i];
      if (bulk_ok(it)) {
        const uint32_t body = it.len & ~15u;
        if (body < it.len && t < (int)(it.len - body))
          slab[it.dst + body + t] = reinterpret_cast<const uint8_t*>(it.src)[body + t];
      } else {
        copy_bytes(slab + it.dst, reinterpret_cast<const uint8_t*>(it.src), it.len, t, nthr);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// CRC-32 of the packed bytes, raw form (init 0, no xorout; see
// crc32.cpp). Two kernels, both table-driven (no bit-serial GF(2) products):
//
//  fp_crc_pages : one raw CRC per 4 KiB page. Warp per page, lane l owns bytes
//                 [128 l, 128 l + 128): 8 x 16-B loads, then 32 slicing-by-4
//                 steps whose lookups go to a per-lane copy of the tables
//                 (entry e of table k at word (k*256 + e)*32 + lane, i.e. in
//                 bank `lane`: conflict-free, 128 KiB), then the 32 lane CRCs
//                 are combined in a shuffle tree, R(A||B) = R(A)*x^(8|B|) ^ R(B),
//                 the constant product of level v (|B| = 128*2^v bytes) done
//                 with four 256-entry tables.
// The page CRCs go to the host, which folds them per extent in file order
// (ExtentCrc, crc32.cpp: one constant product per page) — a per-chunk fold
// kernel (one block per 64 MiB chunk, 4 of 148 SMs busy for ~15 us) was the
// round-1 design.
//
// Device table blob (uint32, built by crc_device_tables on the host):
//   [kTabS4 .. +1024)   slicing-by-4 tables t[k][b] (b followed by k bytes)
//   [kTabLaneK + l)     x^(8*128*(31-l)), the lane-combine constant of lane l
// each product table is four 256-entry tables: M[i][b] = K * (b << 8i).
// ---------------------------------------------------------------------------
constexpr int kCrcThreads = 1024;
constexpr size_t kCrcTabWords = 4 * 256 * 32;                      // per-lane slicing tables
constexpr size_t kCrcPagesSmem = kCrcTabWords * sizeof(uint32_t);  // 128 KiB
constexpr uint32_t kPolyRefl = 0xEDB88320u;

// Lane combine without shared memory: lane l's raw CRC R_l of its 128 bytes
// enters the page CRC as R_l * x^(8*128*(31-l)) (the bytes after it), and
// the lanes' terms are XOR-reduced. The product by the lane's constant K_l is
// done in registers: kv[i] = K_l * x^i (reflected, bit 31 = x^0), so
// R * K_l = XOR of kv[i] over the bits i of R (bit 31-i) — 32 predicated
// XORs, no table lookups (the round-1 shuffle tree did 5 levels of 4
// bank-conflicting lookups into shared constant-product tables: ~30 % of the
// kernel's shared-memory wavefronts).
__device__ __forceinline__ void lane_k_init(uint32_t K, uint32_t (&kv)[32]) {
  kv[0] = K;
#pragma unroll
  for (int i = 1; i < 32; ++i) kv[i] = (kv[i - 1] >> 1) ^ ((kv[i - 1] & 1) ? kPolyRefl : 0u);
}
__device__ __forceinline__ uint32_t gf_mul_k(uint32_t a, const uint32_t (&kv)[32]) {
  uint32_t p = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) p ^= (0u - ((a >> (31 - i)) & 1u)) & kv[i];
  return p;
}
__device__ __forceinline__ uint32_t lanes_combine(uint32_t c, const uint32_t (&kv)[32]) {
  c = gf_mul_k(c, kv);
#pragma unroll
  for (int o = 16; o; o >>= 1) c ^= __shfl_xor_sync(0xffffffffu, c, o);
  return c;  // valid in every lane
}

// Product by a COMPILE-TIME constant x^(8*kBytes) (reflected): the 32 values
// K*x^i are immediates, so the product is 32 predicated XORs of constants —
// no registers held, no table lookups. Used to join two independent chains
// of a lane (words 0..15 and 16..31: R = R0 * x^(8*64) ^ R1), which halves
// the dependent-lookup latency of a page.
constexpr uint32_t ce_gf_mul(uint32_t a, uint32_t b) {
  uint32_t p = 0;
  for (uint32_t m = 1u << 31; m; m >>= 1) {
    if (a & m) p ^= b;
    b = (b & 1) ? (b >> 1) ^ kPolyRefl : b >> 1;
  }
  return p;
}
constexpr uint32_t ce_x8n(uint64_t n) {  // x^(8n) mod P
  uint32_t r = 1u << 31, sq = 1u << 23;  // x^0; x^8
  for (; n; n >>= 1) {
    if (n & 1) r = ce_gf_mul(r, sq);
    sq = ce_gf_mul(sq, sq);
  }
  return r;
}
template <uint32_t K>
__device__ __forceinline__ uint32_t gf_mul_const(uint32_t a) {
  uint32_t p = 0, k = K;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    p ^= (0u - ((a >> (31 - i)) & 1u)) & k;
    k = (k >> 1) ^ ((k & 1) ? kPolyRefl : 0u);  // folded to immediates (K is constexpr)
  }
  return p;
}
constexpr uint32_t kX64 = ce_x8n(64);  // x^(8*64): joins a lane's two 64-B chains

// Raw CRC of one 4 KiB page held by a warp, lane l owning bytes
// [128 l, 128 l + 128) as v[0..7]: one slicing-by-4 chain of 32 words per
// lane through per-lane (bank-private) copies of the 4 tables (entry e of
// table k at (k*256 + e)*32 + lane), then lanes_combine.
__device__ __forceinline__ uint32_t page_crc_warp(const uint4 (&v)[8], const uint32_t* rep,
                                                  const uint32_t (&kv)[32], int lane) {
  const uint32_t* r0 = rep + lane;
  const uint32_t* r1 = rep + 256 * 32 + lane;
  const uint32_t* r2 = rep + 2 * 256 * 32 + lane;
  const uint32_t* r3 = rep + 3 * 256 * 32 + lane;
  uint32_t c0 = 0, c1 = 0;  // words 0..15 and 16..31: two independent chains
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const uint4& va = v[q >> 2];
    const uint4& vb = v[4 + (q >> 2)];
    const uint32_t wa = (q & 3) == 0 ? va.x : (q & 3) == 1 ? va.y : (q & 3) == 2 ? va.z : va.w;
    const uint32_t wb = (q & 3) == 0 ? vb.x : (q & 3) == 1 ? vb.y : (q & 3) == 2 ? vb.z : vb.w;
    const uint32_t xa = c0 ^ wa, xb = c1 ^ wb;
    c0 = r3[(xa & 255) << 5] ^ r2[((xa >> 8) & 255) << 5] ^ r1[((xa >> 16) & 255) << 5] ^
         r0[(xa >> 24) << 5];
    c1 = r3[(xb & 255) << 5] ^ r2[((xb >> 8) & 255) << 5] ^ r1[((xb >> 16) & 255) << 5] ^
         r0[(xb >> 24) << 5];
  }
  return lanes_combine(gf_mul_const<kX64>(c0) ^ c1, kv);
}

__global__ void __launch_bounds__(kCrcThreads, 1)
    fp_crc_pages(const uint8_t* __restrict__ buf, uint32_t n_pages,
                 const uint32_t* __restrict__ tabs, uint32_t* __restrict__ out) {
  extern __shared__ __align__(16) uint32_t crc_smem[];
  uint32_t* rep = crc_smem;                    // [4][256][32] per-lane copies
  for (int i = threadIdx.x; i < 4 * 256 * 32; i += blockDim.x) rep[i] = tabs[kTabS4 + (i >> 5)];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t kv[32];
  lane_k_init(tabs[kTabLaneK + lane], kv);
  const uint32_t wpb = blockDim.x >> 5;
  for (uint32_t pg = blockIdx.x * wpb + (threadIdx.x >> 5); pg < n_pages; pg += gridDim.x * wpb) {
    const uint4* src = reinterpret_cast<const uint4*>(buf + (size_t)pg * 4096 + lane * 128);
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(src + u);
    const uint32_t c = page_crc_warp(v, rep, kv, lane);
    if (lane == 0) out[pg] = c;
  }
}

// fp_crc_pages_tma: fp_crc_pages with the page bytes brought into shared
// memory by the TMA engine instead of 8 LSU loads per lane (each of which
// touched 32 different 128-B lines: the L1/TEX pipe was the limiter). The slab
// is a 2-D tensor map of 128-B rows with 128-B swizzling; one box = one 4 KiB
// page = 32 rows, so lane l's run (row l) lands with its 16-B chunk u at
// chunk u ^ (l & 7): the per-lane LDS.128 reads are conflict-free. Each of
// the 16 warps streams its own pages through one stage (the page is copied
// to registers, then the next page's TMA is issued into the same stage while
// the warp computes). Table lookups are one PRMT + one LDS: the per-lane
// copies are laid out in pairs of tables so that entry e of table k for lane
// l sits at byte (k>>1)*64K + e*256 + (k&1)*128 + l*4; one byte_perm builds
// (e << 8) | (l*4) from the data word and the constant offset is an
// immediate of the load.
constexpr int kCtWarps = 16;
constexpr size_t kCtTabBytes = 4 * 256 * 32 * 4;  // paired per-lane tables
constexpr size_t kCtSmem = kCtTabBytes + 256 + 1024 + (size_t)kCtWarps * 4096;

__global__ void __launch_bounds__(kCtWarps * 32, 1)
    fp_crc_pages_tma(const __grid_constant__ CUtensorMap tmap, uint32_t n_pages,
                     const uint32_t* __restrict__ tabs, uint32_t* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t ct_raw[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(ct_raw + kCtTabBytes);
  uint8_t* stages = reinterpret_cast<uint8_t*>(
      ((uintptr_t)(ct_raw + kCtTabBytes + 256) + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 4 * 256 * 32; i += blockDim.x) {
    const int k = i >> 13, e = (i >> 5) & 255, l = i & 31;
    *reinterpret_cast<uint32_t*>(ct_raw + (k >> 1) * 65536 + e * 256 + (k & 1) * 128 + l * 4) =
        tabs[kTabS4 + k * 256 + e];
  }
  if (threadIdx.x < kCtWarps)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[threadIdx.x])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lane4 = (uint32_t)lane * 4;
  uint32_t kv[32];
  lane_k_init(tabs[kTabLaneK + lane], kv);
  const uint32_t gw = blockIdx.x * kCtWarps + (uint32_t)w, nw = gridDim.x * kCtWarps;
  uint8_t* stage = stages + (size_t)w * 4096;
  const uint32_t bar = smem_u32(&mbar[w]);
  auto issue = [&](uint32_t k) {  // lane 0: page gw + k*nw -> this warp's stage
    const uint32_t pg = gw + k * nw;
    if (pg >= n_pages) return;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(4096)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(stage)),
        "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"(pg * 32), "r"(bar)
        : "memory");
  };
  // T_t[byte b of x] for this lane: one byte_perm + one LDS with an immediate
  auto lk = [&](uint32_t x, const int b, const int t) -> uint32_t {
    const uint32_t r = __byte_perm(x, lane4, 4u | ((uint32_t)b << 4) | (5u << 8) | (5u << 12));
    return *reinterpret_cast<const uint32_t*>(ct_raw + r + ((t >> 1) * 65536 + (t & 1) * 128));
  };
  if (lane == 0) issue(0);
  for (uint32_t k = 0;; ++k) {
    const uint32_t pg = gw + k * nw;
    if (pg >= n_pages) break;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(k & 1)
        : "memory");
    const uint8_t* row = stage + lane * 128;
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      v[u] = *reinterpret_cast<const uint4*>(row + ((u ^ (lane & 7)) << 4));
    __syncwarp();
    if (lane == 0) issue(k + 1);  // every lane has its copy of this page
    // two independent chains per lane (words 0..15, 16..31), joined by a
    // compile-time constant product
    uint32_t c0 = 0, c1 = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const uint4& va = v[q >> 2];
      const uint4& vb = v[4 + (q >> 2)];
      const uint32_t wa = (q & 3) == 0 ? va.x : (q & 3) == 1 ? va.y : (q & 3) == 2 ? va.z : va.w;
      const uint32_t wb = (q & 3) == 0 ? vb.x : (q & 3) == 1 ? vb.y : (q & 3) == 2 ? vb.z : vb.w;
      const uint32_t xa = c0 ^ wa, xb = c1 ^ wb;
      c0 = lk(xa, 0, 3) ^ lk(xa, 1, 2) ^ lk(xa, 2, 1) ^ lk(xa, 3, 0);
      c1 = lk(xb, 0, 3) ^ lk(xb, 1, 2) ^ lk(xb, 2, 1) ^ lk(xb, 3, 0);
    }
    const uint32_t cl = lanes_combine(gf_mul_const<kX64>(c0) ^ c1, kv);
    if (lane == 0) out[pg] = cl;
  }
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

// fp_crc_pages_col: a LANE owns a whole page, so no lane combine at all (the
// combine products were ~45 % of fp_crc_pages_tma's ALU work). The slab is a
// 2-D tensor map of pages (rows of 4096 B); one TMA box = the k-th 128-B
// column of 32 consecutive pages (4 KiB, 128-B swizzle, so lane r reading
// its row's 16-B chunk c at c ^ (r & 7) is conflict-free). Each of the 16
// warps walks groups of 32 pages column by column, copies the box to
// registers, issues the next box into its stage and advances 32 pages' CRC
// chains by 32 words each; after 32 columns lane r holds page r's raw CRC.
constexpr int kColWarps = 16;
constexpr size_t kColSmem = kCtTabBytes + 256 + 1024 + (size_t)kColWarps * 4096;

__global__ void __launch_bounds__(kColWarps * 32, 1)
    fp_crc_pages_col(const __grid_constant__ CUtensorMap tmap, uint32_t n_pages,
                     const uint32_t* __restrict__ tabs, uint32_t* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t cc_raw[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(cc_raw + kCtTabBytes);
  uint8_t* stages = reinterpret_cast<uint8_t*>(
      ((uintptr_t)(cc_raw + kCtTabBytes + 256) + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 4 * 256 * 32; i += blockDim.x) {
    const int k = i >> 13, e = (i >> 5) & 255, l = i & 31;
    *reinterpret_cast<uint32_t*>(cc_raw + (k >> 1) * 65536 + e * 256 + (k & 1) * 128 + l * 4) =
        tabs[kTabS4 + k * 256 + e];
  }
  if (threadIdx.x < kColWarps) mbar_init(&mbar[threadIdx.x], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lane4 = (uint32_t)lane * 4;
  const uint32_t n_groups = (n_pages + 31) / 32;
  const uint32_t gw = blockIdx.x * kColWarps + (uint32_t)w, nw = gridDim.x * kColWarps;
  uint8_t* stage = stages + (size_t)w * 4096;
  const uint32_t bar = smem_u32(&mbar[w]);
  // box number b = (group index i of this warp) * 32 + column k
  auto issue = [&](uint32_t b) {
    const uint32_t g = gw + (b >> 5) * nw;
    if (g >= n_groups) return;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_tx(bar, 4096);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(stage)),
        "l"(reinterpret_cast<uint64_t>(&tmap)), "r"((b & 31) * 128), "r"(g * 32), "r"(bar)
        : "memory");
  };
  auto lk = [&](uint32_t x, const int b, const int t) -> uint32_t {
    const uint32_t r = __byte_perm(x, lane4, 4u | ((uint32_t)b << 4) | (5u << 8) | (5u << 12));
    return *reinterpret_cast<const uint32_t*>(cc_raw + r + ((t >> 1) * 65536 + (t & 1) * 128));
  };
  if (lane == 0) issue(0);
  uint32_t c = 0;
  for (uint32_t b = 0;; ++b) {
    const uint32_t g = gw + (b >> 5) * nw;
    if (g >= n_groups) break;
    mbar_wait(bar, b & 1);
    const uint8_t* row = stage + lane * 128;
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      v[u] = *reinterpret_cast<const uint4*>(row + ((u ^ (lane & 7)) << 4));
    __syncwarp();
    if (lane == 0) issue(b + 1);  // every lane has its 128 B of this column
    if ((b & 31) == 0) c = 0;     // a new group of 32 pages starts
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const uint4& vv = v[q >> 2];
      const uint32_t wd = (q & 3) == 0 ? vv.x : (q & 3) == 1 ? vv.y : (q & 3) == 2 ? vv.z : vv.w;
      const uint32_t x = c ^ wd;
      c = lk(x, 0, 3) ^ lk(x, 1, 2) ^ lk(x, 2, 1) ^ lk(x, 3, 0);
    }
    if ((b & 31) == 31 && g * 32 + (uint32_t)lane < n_pages) out[g * 32 + lane] = c;
  }
}

// ---------------------------------------------------------------------------
// fp_pack_bulk_crc: the TMA-engine pack and the page CRCs in ONE pass (SURVEY
// f4 "per-shard checksum fused into the pack kernel"). Work unit: one 32 KiB
// slab tile (8 pages); items never cross a tile (plan_tiles). One CTA per SM,
// 3 shared-memory stages of one tile each:
//   warp 0 (producer): lane 0 issues cp.async.bulk G2S for the 16-B aligned
//     bodies of the tile's items into the stage (mbarrier complete_tx); once
//     tile i's stage is FULL it hands the tile to its CRC group (the group's
//     own tile-ready barrier) and issues one cp.async.bulk S2G of the whole
//     tile to the slab; then it reclaims the stage of tile i-1 — its S2G read
//     out of shared memory, its CRC warps done with it (EMPTY) — signals FREE
//     to the LSU warps and refills it with tile i+2. Tile descriptors are
//     loaded one stage cycle ahead. L2 evict-first both ways.
//   warps 1-2 (LSU): zero fill, misaligned items and <16 B tails straight
//     into the stage (generic stores + proxy fence), then arrive on FULL.
//   warps 3.. (CRC): kGroups groups of 8 warps; group g takes the tiles
//     i = g (mod kGroups) of this CTA, warp p of the group page p of the
//     tile, from the stage — lane l reads its 128-B row with the 16-B chunks
//     rotated by (l & 7) (conflict-free: a linear TMA row layout puts every
//     lane's row in the same banks) and puts them back in order with a
//     3-level register barrel shift — two slicing-by-4 chains per lane,
//     lanes_combine; arrive on EMPTY as soon as the page is in registers.
// 90 us per 256 MiB (0.90 of HBM for pack + CRC) — the bare packs' own time
// at that size (fp_pack_bulk 90.1, fp_pack_v4 90.5 us, no CRC) — and 328 us per
// 1 GiB launch (0.98, the default group size: a launch carries ~12 us of fixed
// cost); fp_pack_v4 + fp_crc_pages_tma take 87.5 + 65.9 us per 256 MiB
// (profiles/r02_pack_group_size.md, r02_ncu_bulk_crc_q8.md). The protocol is model-checked under
// random schedules in tests/test_bulk_protocol_cpu.py.
// The slab is written and read once (2 B of HBM per image byte): the CRC no
// longer re-reads it (the separate fp_crc_pages_tma pass: +1 B per byte).
// ---------------------------------------------------------------------------
constexpr int kBcStages = 3;
constexpr int kBcLsuWarps = 2;
constexpr int kBcCrcWarps = kTile / 4096;  // 8 per group: one page each
constexpr int bc_threads(int groups) { return 32 * (1 + kBcLsuWarps + groups * kBcCrcWarps); }
constexpr size_t kBcSmem = kCtTabBytes + (size_t)kBcStages * kTile + 128;  // + 13 mbarriers

// generic-proxy copy of `len` bytes into shared memory (src == nullptr: zeros)
__device__ __forceinline__ void copy_to_smem(uint8_t* dst, const uint8_t* __restrict__ src,
                                             uint32_t len, int t, int nthr) {
  const bool vec = !(((uintptr_t)dst | (uintptr_t)src | len) & 15);
  if (vec) {
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (uint32_t j = t; j < len / 16; j += nthr)
      reinterpret_cast<uint4*>(dst)[j] = src ? ld_stream(reinterpret_cast<const uint4*>(src) + j) : z;
    return;
  }
  for (uint32_t j = t; j < len; j += nthr) dst[j] = src ? src[j] : 0;
}

template <int kGroups, bool kWarpStore>
__global__ void __launch_bounds__(bc_threads(kGroups), 1)
    fp_pack_bulk_crc(const Item* __restrict__ items, const uint32_t* __restrict__ tile_lo,
                     uint32_t n_tiles, uint64_t gbytes, uint8_t* __restrict__ slab,
                     const uint32_t* __restrict__ tabs, uint32_t* __restrict__ page_crc) {
  extern __shared__ __align__(128) uint8_t bc_raw[];
  uint8_t* stages = bc_raw + kCtTabBytes;  // kCtTabBytes is a multiple of 128
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + (size_t)kBcStages * kTile);
  uint64_t* empty = full + kBcStages;
  uint64_t* freeb = empty + kBcStages;
  uint64_t* cfull = freeb + kBcStages;  // [group][2]: tile j of a group is ready
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBcStages; ++s) {
      mbar_init(&full[s], 1 + kBcLsuWarps);
      mbar_init(&empty[s], kBcCrcWarps);
      mbar_init(&freeb[s], 1);
    }
    for (int b = 0; b < 2 * kGroups; ++b) mbar_init(&cfull[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (blockIdx.x >= n_tiles) return;
  const uint32_t nt = (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;  // tiles of this CTA
  auto tile_of = [&](uint32_t i) { return blockIdx.x + i * gridDim.x; };
  auto tile_len = [&](uint32_t t) {
    const uint64_t left = gbytes - (uint64_t)t * kTile;
    return (uint32_t)(left < kTile ? left : kTile);
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // A tile's descriptors ({first item, end} from tile_lo, then one item per
  // lane when the tile has <= 32 items — one item for most tiles of a
  // model state) are loaded one stage cycle before they are needed, so the
  // two dependent global loads are off the refill's critical path.
  struct TileDesc {
    uint32_t lo, hi;
    Item it;  // item lo + lane, if any
  };
  auto load_bounds = [&](uint32_t i, TileDesc& d) {
    d.lo = d.hi = 0;
    if (i < nt) {
      const uint32_t t = tile_of(i);
      d.lo = tile_lo[t];
      d.hi = tile_lo[t + 1];
    }
  };
  auto load_item = [&](TileDesc& d) {
    d.it = {0, 0, 0};
    if (d.lo + lane < d.hi) d.it = items[d.lo + lane];
  };
  if (warp == 0) {
    const uint64_t pol = evict_first_policy();
    auto g2s = [&](uint8_t* st, const Item& mine, bool ok, uint32_t bar) {
      uint32_t mask = __ballot_sync(0xffffffffu, ok && bulk_ok(mine));
      while (mask) {
        const int j = __ffs(mask) - 1;
        mask &= mask - 1;
        const uint64_t src = __shfl_sync(0xffffffffu, mine.src, j);
        const uint32_t dst = __shfl_sync(0xffffffffu, mine.dst, j);
        const uint32_t len = __shfl_sync(0xffffffffu, mine.len, j);
        if (lane == 0)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
              " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(st + (dst % kTile))),
              "l"(src), "r"(len & ~15u), "r"(bar), "l"(pol)
              : "memory");
      }
    };
    auto fill = [&](uint32_t i, const TileDesc& d) {  // G2S of tile i's 16-B aligned item bodies
      FP_KASSERT(d.lo <= d.hi);
      FP_KASSERT(d.lo + lane >= d.hi ||
                 (d.it.dst / kTile == tile_of(i) && d.it.dst % kTile + d.it.len <= kTile &&
                  (uint64_t)d.it.dst + d.it.len <= gbytes));
      const uint32_t s = i % kBcStages;
      uint8_t* st = stages + (size_t)s * kTile;
      const uint32_t bar = smem_u32(&full[s]);
      const bool one = d.hi - d.lo <= 32;
      uint32_t total = 0;
      if (one) {
        total = d.lo + lane < d.hi && bulk_ok(d.it) ? (d.it.len & ~15u) : 0u;
      } else {
        for (uint32_t b = d.lo; b < d.hi; b += 32) {
          Item it = {0, 0, 0};
          if (b + lane < d.hi) it = items[b + lane];
          total += (b + lane < d.hi && bulk_ok(it)) ? (it.len & ~15u) : 0u;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_tx(bar, total);
      }
      if (one) {
        g2s(st, d.it, d.lo + lane < d.hi, bar);
      } else {
        for (uint32_t b = d.lo; b < d.hi; b += 32) {
          Item mine = {0, 0, 0};
          if (b + lane < d.hi) mine = items[b + lane];
          g2s(st, mine, b + lane < d.hi, bar);
        }
      }
    };
    const uint32_t ahead = nt < (uint32_t)kBcStages ? nt : (uint32_t)kBcStages;
    for (uint32_t i = 0; i < ahead; ++i) {
      TileDesc d;
      load_bounds(i, d);
      load_item(d);
      fill(i, d);
    }
    // The producer runs one tile behind on the drain side: in iteration i it
    // issues tile i's S2G and hands tile i to its CRC group, THEN reclaims
    // the stage of tile i - 1 (its S2G read out, its CRC warps done) and
    // refills it with tile i + 2. Waiting for tile i's own drain before
    // moving on (the first design) put the producer -> CRC warps -> producer
    // round trip and the S2G read of every tile in series (ncu: FULL was
    // never waited on, EMPTY always).
    TileDesc nxt;  // tile i + kBcStages - 1, items in flight
    load_bounds(kBcStages, nxt);
    load_item(nxt);
    for (uint32_t i = 0; i < nt; ++i) {
      const uint32_t s = i % kBcStages, t = tile_of(i), tl = tile_len(t);
      uint8_t* st = stages + (size_t)s * kTile;
      TileDesc nn;  // tile i + kBcStages: bounds in flight
      if (i) load_bounds(i + kBcStages, nn);
      mbar_wait(smem_u32(&full[s]), (i / kBcStages) & 1);
      // hand tile i to its CRC group (a group must not test full[s] itself:
      // with kGroups not dividing kBcStages, stage s's previous phase belongs
      // to another group and a parity test cannot tell it from this one)
      if (lane == 0) mbar_arrive(smem_u32(&cfull[(i % kGroups) * 2 + ((i / kGroups) & 1)]));
      const uint32_t body = tl & ~15u;
      if (!kWarpStore && lane == 0 && body) {
        asm volatile(
            "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                slab + (uint64_t)t * kTile),
            "r"(smem_u32(st)), "r"(body), "l"(pol)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      if (!kWarpStore && (uint32_t)lane < tl - body)
        slab[(uint64_t)t * kTile + body + lane] = st[body + lane];
      if (i) {
        // EMPTY of tile i - 1 is waited for even when its stage is not
        // refilled: the CRC group's tile-ready slot of tile i - 1 + 2 *
        // kGroups must not be signalled before the group has taken tile i - 1
        const uint32_t p = i - 1, ps = p % kBcStages;
        mbar_wait(smem_u32(&empty[ps]), (p / kBcStages) & 1);
        if (p + kBcStages < nt) {
          // tile i - 1's S2G has read the stage (tile i's may still be reading)
          if (!kWarpStore && lane == 0)
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&freeb[ps]));
          fill(p + kBcStages, nxt);
        }
        load_item(nn);
        nxt = nn;
      }
    }
    if (nt) mbar_wait(smem_u32(&empty[(nt - 1) % kBcStages]), ((nt - 1) / kBcStages) & 1);
    if (!kWarpStore && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (warp <= kBcLsuWarps) {
    const int t0 = threadIdx.x - 32, nthr = 32 * kBcLsuWarps;
    TileDesc cur;
    load_bounds(0, cur);
    load_item(cur);
    for (uint32_t i = 0; i < nt; ++i) {
      const uint32_t s = i % kBcStages;
      uint8_t* st = stages + (size_t)s * kTile;
      TileDesc nn;
      load_bounds(i + 1, nn);
      if (i >= (uint32_t)kBcStages) mbar_wait(smem_u32(&freeb[s]), (i / kBcStages - 1) & 1);
      const bool one = cur.hi - cur.lo <= 32;
      for (uint32_t k = cur.lo; k < cur.hi; ++k) {
        Item it;
        if (one) {
          const int j = (int)(k - cur.lo);
          it.src = __shfl_sync(0xffffffffu, cur.it.src, j);
          it.dst = __shfl_sync(0xffffffffu, cur.it.dst, j);
          it.len = __shfl_sync(0xffffffffu, cur.it.len, j);
        } else {
          it = items[k];
        }
        const uint32_t off = it.dst % kTile;
        FP_KASSERT(it.dst / kTile == tile_of(i) && off + it.len <= kTile);
        if (bulk_ok(it)) {
          const uint32_t body = it.len & ~15u;
          if ((uint32_t)t0 < it.len - body)
            st[off + body + t0] = reinterpret_cast<const uint8_t*>(it.src)[body + t0];
        } else {
          copy_to_smem(st + off, reinterpret_cast<const uint8_t*>(it.src), it.len, t0, nthr);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the S2G
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&full[s]));
      load_item(nn);
      cur = nn;
    }
  } else {
    // the CRC warps alone fill the paired per-lane tables (the producer's
    // first loads are in flight meanwhile), then meet at named barrier 1:
    // 128 KiB as 16-B chunks, consecutive lanes -> consecutive chunks
    // (conflict-free); chunk c holds entry e of table k for 8 lanes, with
    // (k >> 1) = c / 4096, e = (c / 16) % 256, (k & 1) = (c / 8) % 2
    {
      const int t = threadIdx.x - 32 * (1 + kBcLsuWarps), nthr = 32 * kGroups * kBcCrcWarps;
#pragma unroll 4
      for (int c = t; c < (int)(kCtTabBytes / 16); c += nthr) {
        const int k = ((c >> 12) << 1) | ((c >> 3) & 1), e = (c >> 4) & 255;
        const uint32_t v = tabs[kTabS4 + k * 256 + e];
        *reinterpret_cast<uint4*>(bc_raw + (size_t)c * 16) = make_uint4(v, v, v, v);
      }
      asm volatile("bar.sync 1, %0;" ::"r"(32 * kGroups * kBcCrcWarps) : "memory");
    }
    const int p = (warp - 1 - kBcLsuWarps) % kBcCrcWarps;  // page of the tile
    const uint32_t grp = (uint32_t)(warp - 1 - kBcLsuWarps) / kBcCrcWarps;
    const uint32_t lane4 = (uint32_t)lane * 4, rot = (uint32_t)lane & 7;
    uint32_t kv[32];
    lane_k_init(tabs[kTabLaneK + lane], kv);
    auto lk = [&](uint32_t x, const int b, const int tb) -> uint32_t {
      const uint32_t r = __byte_perm(x, lane4, 4u | ((uint32_t)b << 4) | (5u << 8) | (5u << 12));
      return *reinterpret_cast<const uint32_t*>(bc_raw + r + ((tb >> 1) * 65536 + (tb & 1) * 128));
    };
    // tile j of this group (i = grp + j * kGroups) is signalled on
    // cfull[grp][j & 1], phase j / 2: the producer signals tile j + 2 only
    // after it waited for this group's EMPTY of tile j, so no slot runs two
    // phases ahead of its parity test
    for (uint32_t i = grp, j = 0; i < nt; i += kGroups, ++j) {
      const uint32_t s = i % kBcStages, t = tile_of(i);
      mbar_wait(smem_u32(&cfull[grp * 2 + (j & 1)]), (j >> 1) & 1);
      const uint32_t pg = t * (kTile / 4096) + (uint32_t)p;
      const bool live = (uint64_t)pg * 4096 < gbytes;
      if (live) {
        if (kWarpStore) {
          // the page to the slab from the stage, coalesced (512 B per warp
          // instruction), before EMPTY: the stage is free as soon as its
          // readers have it, with no S2G holding it while the write drains
          const uint8_t* ps = stages + (size_t)s * kTile + (size_t)p * 4096;
          uint8_t* pd = slab + (uint64_t)t * kTile + (size_t)p * 4096;
          const uint32_t tl = tile_len(t), plen = tl - p * 4096 < 4096 ? tl - p * 4096 : 4096;
          if (plen == 4096) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint4 x[4];
#pragma unroll
              for (int u = 0; u < 4; ++u)
                x[u] = *reinterpret_cast<const uint4*>(ps + ((h * 4 + u) * 32 + lane) * 16);
#pragma unroll
              for (int u = 0; u < 4; ++u)
                st_v4(reinterpret_cast<uint4*>(pd) + (h * 4 + u) * 32 + lane, x[u]);
            }
          } else {
            for (uint32_t q = lane; q * 16 < plen; q += 32) {
              if (q * 16 + 16 <= plen)
                st_v4(reinterpret_cast<uint4*>(pd) + q, *reinterpret_cast<const uint4*>(ps + q * 16));
              else
                for (uint32_t b = q * 16; b < plen; ++b) pd[b] = ps[b];
            }
          }
        }
        const uint8_t* row = stages + (size_t)s * kTile + (size_t)p * 4096 + lane * 128;
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)  // chunk (u + rot) & 7 lands in v[u]
          v[u] = *reinterpret_cast<const uint4*>(row + (((u + rot) & 7) << 4));
        // v[u] holds chunk (u + rot) & 7: rotate right by rot so v[c] = chunk c
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          if (rot & (1u << b)) {
            uint4 w[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) w[u] = v[(u - (1 << b)) & 7];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = w[u];
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&empty[s]));  // the page is in registers
#ifdef FP_BC_SKIP_CRC  // experiment: the pipeline without the CRC arithmetic
        if (lane == 0) page_crc[pg] = v[0].x ^ v[7].w;
#else
        uint32_t c0 = 0, c1 = 0;  // two independent chains per lane (ILP)
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const uint4& va = v[q >> 2];
          const uint4& vb = v[4 + (q >> 2)];
          const uint32_t wa = (q & 3) == 0 ? va.x : (q & 3) == 1 ? va.y : (q & 3) == 2 ? va.z : va.w;
          const uint32_t wb = (q & 3) == 0 ? vb.x : (q & 3) == 1 ? vb.y : (q & 3) == 2 ? vb.z : vb.w;
          const uint32_t xa = c0 ^ wa, xb = c1 ^ wb;
          c0 = lk(xa, 0, 3) ^ lk(xa, 1, 2) ^ lk(xa, 2, 1) ^ lk(xa, 3, 0);
          c1 = lk(xb, 0, 3) ^ lk(xb, 1, 2) ^ lk(xb, 2, 1) ^ lk(xb, 3, 0);
        }
        const uint32_t c = lanes_combine(gf_mul_const<kX64>(c0) ^ c1, kv);
        if (lane == 0) page_crc[pg] = c;
#endif
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&empty[s]));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// fp_pack_lsu_crc (FP_PACK_LSU, ablation): the LSU pack of fp_pack_v4
// computing the page CRC-32s from the registers it copies through — no
// shared-memory staging, no bulk-copy engine, no hand-off between warps. One
// warp per 4 KiB slab page (pages dealt round robin over all warps of the
// grid): lane l loads the 16-B chunks 32u + l, u = 0..7 (eight coalesced
// 512-B loads in flight), stores them to the slab with the same pattern, then
//   c_u = raw CRC of chunk 32u + l     (4-word slicing-by-4 chains from 0,
//                                       eight independent chains per lane)
//   s_l = sum_u c_u * x^(8*512*(7-u))  (Horner, product by x^(8*512) as 8
//                                       nibble lookups)
//   page = XOR_l s_l * x^(8*16*(31-l)) (8 nibble lookups into lane l's own
//                                       table, then a 5-step XOR shuffle)
// which is R(page) by the linearity R(A||B) = R(A) x^(8|B|) + R(B): chunk q
// is followed by 4096 - 16q - 16 = 512(7-u) + 16(31-l) bytes. All tables are
// per-lane (bank-private) copies in shared memory: 128 KiB slicing tables in
// fp_crc_pages_tma's paired layout + 2 x 16 KiB nibble tables. Pages that no
// single co-aligned item covers (header/padding seams, odd storage offsets,
// byte-granular shard starts, a group's ragged last page) are gathered by the
// warp with copy_bytes and read back from the slab for their CRC. The scheme
// is emulated against the plain CRC on the host (tools/diag/crc_emulate.cpp).
// Measured (profiles/r02_lsu_crc_ablation.md): 103.5 us per 256 MiB (0.79 of
// HBM) vs 90 us for fp_pack_bulk_crc — the table lookups share the L1/LSU
// data pipe with the pack's own loads and stores, and a warp busy with its
// CRC has no loads in flight; software pipelining the next page's loads
// through a shared-memory transpose (16 warps, 118 registers) was slower
// still (123.5 us: the CRC chains became latency-bound). The TMA pack keeps
// the copy off the LSU, which is why it is the default.
// ---------------------------------------------------------------------------
constexpr int kLcWarps = 24;  // 80 registers, no spills (32 warps spill at 64)
constexpr size_t kLcNibBytes = 8 * 16 * 32 * 4;  // 16 KiB: [j * 16 + n][lane]
constexpr size_t kLcSmem = kCtTabBytes + 2 * kLcNibBytes;

// a * K as XOR_j NT[j][(a >> 4j) & 15]; `t` = the table base + lane * 4
// (entry e of lane l at byte e * 128 + l * 4)
__device__ __forceinline__ uint32_t nib_mul(uint32_t a, const uint8_t* t) {
  uint32_t r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t idx = (j == 0 ? (a << 7) : j == 1 ? (a << 3) : (a >> (4 * j - 7))) & 0x780u;
    r ^= *reinterpret_cast<const uint32_t*>(t + j * 2048 + idx);
  }
  return r;
}

__global__ void __launch_bounds__(kLcWarps * 32, 1)
    fp_pack_lsu_crc(const Item* __restrict__ items, const uint32_t* __restrict__ tile_lo,
                    uint64_t gbytes, uint8_t* __restrict__ slab,
                    const uint32_t* __restrict__ tabs, uint32_t* __restrict__ page_crc) {
  extern __shared__ __align__(128) uint8_t lc_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t n_pages = (uint32_t)((gbytes + 4095) / 4096);
  const uint32_t W = gridDim.x * kLcWarps;
  // page descriptors: {first item, end} of the page's tile and one item per
  // lane; the next page's are loaded while this page's data is in flight
  struct Desc {
    uint32_t lo, hi;
    Item it;
  };
  auto load_bounds = [&](uint32_t pg, Desc& d) {
    d.lo = d.hi = 0;
    if (pg < n_pages) {
      const uint32_t t = pg / (kTile / 4096);
      d.lo = tile_lo[t];
      d.hi = tile_lo[t + 1];
    }
  };
  auto load_item = [&](Desc& d) {
    d.it = {0, 0, 0};
    if (d.lo + lane < d.hi) d.it = items[d.lo + lane];
  };
  Desc cur;
  load_bounds(blockIdx.x * kLcWarps + warp, cur);
  load_item(cur);
  // the tables (the descriptor loads above are in flight meanwhile):
  // slicing tables as in fp_pack_bulk_crc, nibble tables [e][lane]
  for (int c = threadIdx.x; c < (int)(kCtTabBytes / 16); c += blockDim.x) {
    const int k = ((c >> 12) << 1) | ((c >> 3) & 1), e = (c >> 4) & 255;
    const uint32_t v = tabs[kTabS4 + k * 256 + e];
    *reinterpret_cast<uint4*>(lc_raw + (size_t)c * 16) = make_uint4(v, v, v, v);
  }
  for (int c = threadIdx.x; c < (int)(kLcNibBytes / 16); c += blockDim.x) {
    const int e = c >> 3, l0 = (c & 7) * 4;
    const uint32_t x = tabs[kTabNibX + e];
    *reinterpret_cast<uint4*>(lc_raw + kCtTabBytes + (size_t)c * 16) = make_uint4(x, x, x, x);
    const uint32_t* k = tabs + kTabNibK + e;
    *reinterpret_cast<uint4*>(lc_raw + kCtTabBytes + kLcNibBytes + (size_t)c * 16) =
        make_uint4(k[l0 * 128], k[(l0 + 1) * 128], k[(l0 + 2) * 128], k[(l0 + 3) * 128]);
  }
  __syncthreads();
  const uint32_t lane4 = (uint32_t)lane * 4;
  const uint8_t* tx = lc_raw + kCtTabBytes + lane4;
  const uint8_t* tk = tx + kLcNibBytes;
  auto lk = [&](uint32_t x, const int b, const int tb) -> uint32_t {
    const uint32_t r = __byte_perm(x, lane4, 4u | ((uint32_t)b << 4) | (5u << 8) | (5u << 12));
    return *reinterpret_cast<const uint32_t*>(lc_raw + r + ((tb >> 1) * 65536 + (tb & 1) * 128));
  };
  for (uint32_t pg = blockIdx.x * kLcWarps + warp; pg < n_pages; pg += W) {
    const uint32_t p0 = pg * 4096u;  // slab offset (a pack group is < 4 GiB)
    const uint64_t left = gbytes - p0;
    const uint32_t plen = left < 4096 ? (uint32_t)left : 4096u;
    // the item covering the whole page with a source co-aligned to the slab
    // (or a zero item): the common case, one item per 32 KiB tile
    Item f = {0, 0, 0};
    bool fast = false;
    for (uint32_t b = cur.lo; b < cur.hi; b += 32) {
      const Item it = b == cur.lo ? cur.it : (b + lane < cur.hi ? items[b + lane] : Item{0, 0, 0});
      const bool ok = plen == 4096 && b + lane < cur.hi && it.dst <= p0 &&
                      it.dst + it.len >= p0 + 4096 && (!it.src || !((it.src - it.dst) & 15));
      const uint32_t m = __ballot_sync(0xffffffffu, ok);
      if (m) {
        const int j = __ffs(m) - 1;
        f.src = __shfl_sync(0xffffffffu, it.src, j);
        f.dst = __shfl_sync(0xffffffffu, it.dst, j);
        fast = true;
        break;
      }
    }
    Desc nxt;
    load_bounds(pg + W, nxt);
    uint4 v[8];
    uint4* d = reinterpret_cast<uint4*>(slab + p0);
    if (fast) {
      if (f.src) {
        const uint4* s = reinterpret_cast<const uint4*>(f.src + (p0 - f.dst));
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ld_stream(s + u * 32 + lane);
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = make_uint4(0, 0, 0, 0);
      }
      load_item(nxt);
#pragma unroll
      for (int u = 0; u < 8; ++u) st_v4(d + u * 32 + lane, v[u]);
    } else {
      // every item of the tile that meets the page, clipped to it
      for (uint32_t k = cur.lo; k < cur.hi; ++k) {
        const Item it = items[k];
        FP_KASSERT(it.dst / kTile == pg / (kTile / 4096) && it.dst % kTile + it.len <= kTile);
        const uint32_t a = it.dst > p0 ? it.dst : p0;
        const uint32_t e = it.dst + it.len < p0 + plen ? it.dst + it.len : p0 + plen;
        if (a < e)
          copy_bytes(slab + a, it.src ? reinterpret_cast<const uint8_t*>(it.src) + (a - it.dst) : nullptr,
                     e - a, lane, 32);
      }
      load_item(nxt);
      __syncwarp();  // the warp's slab stores are visible to its loads below
      if (plen == 4096) {
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ld_coherent(d + u * 32 + lane);
      }
    }
    cur = nxt;
    if (plen < 4096) {  // a ragged last page: the host CRCs ragged chunks itself
      if (lane == 0) page_crc[pg] = 0;
      continue;
    }
    uint32_t cu[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      uint32_t x = v[u].x;
      uint32_t c = lk(x, 0, 3) ^ lk(x, 1, 2) ^ lk(x, 2, 1) ^ lk(x, 3, 0);
      x = c ^ v[u].y;
      c = lk(x, 0, 3) ^ lk(x, 1, 2) ^ lk(x, 2, 1) ^ lk(x, 3, 0);
      x = c ^ v[u].z;
      c = lk(x, 0, 3) ^ lk(x, 1, 2) ^ lk(x, 2, 1) ^ lk(x, 3, 0);
      x = c ^ v[u].w;
      cu[u] = lk(x, 0, 3) ^ lk(x, 1, 2) ^ lk(x, 2, 1) ^ lk(x, 3, 0);
    }
    uint32_t s = cu[0];
#pragma unroll
    for (int u = 1; u < 8; ++u) s = nib_mul(s, tx) ^ cu[u];
    s = nib_mul(s, tk);
#pragma unroll
    for (int o = 16; o; o >>= 1) s ^= __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) page_crc[pg] = s;
  }
}

// ---------------------------------------------------------------------------
// host -> GPU signal: one warp spins (acquire loads at system scope, so the
// host's store to the mapped pinned word is observed) until the word reaches
// `value` (cyclic >=); gives up after max_ns and then sets *timed_out.
// ---------------------------------------------------------------------------
__global__ void fp_wait_flag(const uint32_t* __restrict__ flag, uint32_t value, uint64_t max_ns,
                             uint32_t* __restrict__ timed_out) {
  if (threadIdx.x) return;
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t x;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(x) : "l"(flag) : "memory");
    if ((int32_t)(x - value) >= 0) return;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > max_ns) {
      if (timed_out) asm volatile("st.release.sys.global.u32 [%0], 1;" ::"l"(timed_out) : "memory");
      return;
    }
    __nanosleep(256);
  }
}

bool env_flag(const char* k) {
  const char* v = getenv(k);
  return v && *v && strcmp(v, "0") != 0;
}

int sm_count(int device) {
  int d = device;
  if (d < 0 && cudaGetDevice(&d) != cudaSuccess) return 148;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || n <= 0)
    return 148;
  return n;
}

}  // namespace

// The dynamic shared-memory opt-in is a per-device function attribute: set it
// once per (kernel, device), thread-safely. Slot: one per kernel.
template <int Slot, typename K>
static bool smem_opt_in(K kernel, size_t bytes) {
  static std::atomic<uint64_t> done{0};  // bit d: set on device d
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) return false;
  const uint64_t bit = 1ull << (d & 63);
  if (done.load(std::memory_order_acquire) & bit) return true;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) !=
      cudaSuccess)
    return false;
  done.fetch_or(bit, std::memory_order_acq_rel);
  return true;
}

int pack_default_ctas(int impl, int device) {
  const int sms = sm_count(device);
  return impl == FP_PACK_BULK || impl == FP_PACK_LSU ? sms : sms * 4;
}

int pack_launch(int impl, const Item* d_items, uint32_t n_items, uint8_t* d_slab, int ctas,
                void* stream) {
  if (!n_items) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = (int)((uint32_t)ctas < n_items ? (uint32_t)ctas : n_items);
  if (impl == FP_PACK_BULK) {
    static const bool two = env_flag("FP_BULK_2CTA");
    if (two) {
      if (!smem_opt_in<10>(fp_pack_bulk<3>, bulk_smem<3>())) return FP_ECUDA;
      const int g2 = (int)std::min<uint32_t>(n_items, 2u * (uint32_t)ctas);
      fp_pack_bulk<3><<<g2, kBulkThreads, bulk_smem<3>(), st>>>(d_items, n_items, d_slab);
    } else {
      if (!smem_opt_in<0>(fp_pack_bulk<6>, bulk_smem<6>())) return FP_ECUDA;
      fp_pack_bulk<6><<<grid, kBulkThreads, bulk_smem<6>(), st>>>(d_items, n_items, d_slab);
    }
  } else {
    fp_pack_v4<<<grid, kV4Threads, 0, st>>>(d_items, n_items, d_slab);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : FP_ECUDA;
}

int flag_wait_launch(const uint32_t* d_flag, uint32_t value, uint64_t max_ns,
                     uint32_t* d_timed_out, void* stream) {
  fp_wait_flag<<<1, 32, 0, (cudaStream_t)stream>>>(d_flag, value, max_ns, d_timed_out);
  return cudaGetLastError() == cudaSuccess ? 0 : FP_ECUDA;
}

// 2-D tensor map of d_buf as rows of 128 B, box = one 4 KiB page (32 rows),
// 128-B swizzle. false if the driver entry point is unavailable or FP_NO_TMA=1
// (then the LSU kernel fp_crc_pages runs: 1.6x slower)
static bool encode_page_map(CUtensorMap* m, const uint8_t* d_buf, uint64_t bytes,
                            bool columns) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (!getenv("FP_NO_TMA") &&
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<Encode>(p);
  });
  if (!fn || ((uintptr_t)d_buf & 15) || bytes / 128 > (1ull << 32)) return false;
  // rows: 128-B lines (box = one page) or whole pages (box = a 128-B column
  // of 32 pages)
  const cuuint64_t dims[2] = {columns ? 4096u : 128u, columns ? bytes / 4096 : bytes / 128};
  const cuuint64_t strides[1] = {columns ? 4096u : 128u};
  const cuuint32_t box[2] = {128, 32};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(d_buf), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int crc_pages_launch(const uint8_t* d_buf, uint64_t bytes, const uint32_t* d_tabs,
                     uint32_t* d_page_crc, void* stream) {
  if (!bytes) return 0;
  if (bytes % 4096) return -EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t n_pages = (uint32_t)(bytes / 4096);
  CUtensorMap tmap;
  // default: a lane per 128-B row of a page (two chains + register lane
  // combine); FP_CRC_COL=1: a lane per page (no combine, 25 % less ALU, same
  // time: both wait on the TMA with 4 KiB in flight per warp)
  static const bool col = env_flag("FP_CRC_COL");
  if (col && encode_page_map(&tmap, d_buf, bytes, true)) {
    if (!smem_opt_in<5>(fp_crc_pages_col, kColSmem)) return FP_ECUDA;
    const int grid = (int)std::min<uint32_t>((n_pages + 32 * kColWarps - 1) / (32 * kColWarps),
                                             (uint32_t)sm_count(-1));
    fp_crc_pages_col<<<grid, kColWarps * 32, kColSmem, st>>>(tmap, n_pages, d_tabs, d_page_crc);
  } else if (encode_page_map(&tmap, d_buf, bytes, false)) {
    if (!smem_opt_in<2>(fp_crc_pages_tma, kCtSmem)) return FP_ECUDA;
    const int grid = (int)std::min<uint32_t>((n_pages + kCtWarps - 1) / kCtWarps,
                                             (uint32_t)sm_count(-1));
    fp_crc_pages_tma<<<grid, kCtWarps * 32, kCtSmem, st>>>(tmap, n_pages, d_tabs, d_page_crc);
  } else {
    if (!smem_opt_in<1>(fp_crc_pages, kCrcPagesSmem)) return FP_ECUDA;
    const int grid_p = (int)std::min<uint32_t>((n_pages + 31) / 32, (uint32_t)sm_count(-1));
    fp_crc_pages<<<grid_p, kCrcThreads, kCrcPagesSmem, st>>>(d_buf, n_pages, d_tabs, d_page_crc);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : FP_ECUDA;
}

int pack_bulk_crc_launch(const Item* d_items, const uint32_t* d_tile_lo, uint32_t n_tiles,
                         uint64_t gbytes, uint8_t* d_slab, const uint32_t* d_tabs,
                         uint32_t* d_page_crc, int ctas, void* stream) {
  if (!n_tiles) return 0;
  const int sms = sm_count(-1);
  const int grid = (int)std::min<uint32_t>(n_tiles, (uint32_t)std::min(ctas > 0 ? ctas : sms, sms));
  // ablations: FP_BC_GROUPS=1 (one group of 8 CRC warps); FP_BC_WARPSTORE=1
  // (the CRC warps store the pages from the stage instead of one TMA S2G per
  // tile: 112 vs 98 us per 256 MiB)
  static const bool one = getenv("FP_BC_GROUPS") && !strcmp(getenv("FP_BC_GROUPS"), "1");
  static const bool s2g = !env_flag("FP_BC_WARPSTORE");
  cudaStream_t st = (cudaStream_t)stream;
#define FP_BC_LAUNCH(G, W, SLOT)                                                           \
  do {                                                                                     \
    if (!smem_opt_in<SLOT>(fp_pack_bulk_crc<G, W>, kBcSmem)) return FP_ECUDA;              \
    fp_pack_bulk_crc<G, W><<<grid, bc_threads(G), kBcSmem, st>>>(d_items, d_tile_lo, n_tiles, \
                                                                 gbytes, d_slab, d_tabs,      \
                                                                 d_page_crc);                \
  } while (0)
  if (one && s2g) FP_BC_LAUNCH(1, false, 6);
  else if (one) FP_BC_LAUNCH(1, true, 7);
  else if (s2g) FP_BC_LAUNCH(2, false, 8);
  else FP_BC_LAUNCH(2, true, 4);
#undef FP_BC_LAUNCH
  return cudaGetLastError() == cudaSuccess ? 0 : FP_ECUDA;
}

int pack_lsu_crc_launch(const Item* d_items, const uint32_t* d_tile_lo, uint64_t gbytes,
                        uint8_t* d_slab, const uint32_t* d_tabs, uint32_t* d_page_crc, int ctas,
                        void* stream) {
  if (!gbytes) return 0;
  if (!smem_opt_in<9>(fp_pack_lsu_crc, kLcSmem)) return FP_ECUDA;
  const int sms = sm_count(-1);
  const uint64_t n_pages = (gbytes + 4095) / 4096;
  const int grid = (int)std::min<uint64_t>((n_pages + kLcWarps - 1) / kLcWarps,
                                           (uint64_t)std::min(ctas > 0 ? ctas : sms, sms));
  fp_pack_lsu_crc<<<grid, kLcWarps * 32, kLcSmem, (cudaStream_t)stream>>>(d_items, d_tile_lo, gbytes,
                                                                         d_slab, d_tabs, d_page_crc);
  return cudaGetLastError() == cudaSuccess ? 0 : FP_ECUDA;
}

int unpack_peer_launch(const Item* d_items, uint32_t n_items, const PeerTab* d_tab, uint32_t chunk,
                       uint64_t ch_bytes, int ctas, void* stream) {
  if (!n_items) return 0;
  const int grid = (int)((uint32_t)ctas < n_items ? (uint32_t)ctas : n_items);
  fp_unpack_peer<<<grid, kV4Threads, 0, (cudaStream_t)stream>>>(d_items, n_items, d_tab, chunk,
                                                               ch_bytes);
  return cudaGetLastError() == cudaSuccess ? 0 : FP_ECUDA;
}

int unpack_launch(const Item* d_items, uint32_t n_items, const uint8_t* d_slab, int ctas,
                  void* stream) {
  if (!n_items) return 0;
  const int grid = (int)((uint32_t)ctas < n_items ? (uint32_t)ctas : n_items);
  fp_unpack_v4<<<grid, kV4Threads, 0, (cudaStream_t)stream>>>(d_items, n_items, d_slab);
  return cudaGetLastError() == cudaSuccess ? 0 : FP_ECUDA;
}

}  // namespace fp
