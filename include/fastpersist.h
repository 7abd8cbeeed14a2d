/*
 * fastpersist.h — C-ABI of the B200-native FastPersist checkpoint-write path.
 *
 * The calls follow the paper's problem statement (PAPER.md, arXiv 2406.13768):
 *   - the checkpoint is written after the optimizer and overlapped with the
 *     next iteration's forward/backward, "blocks before optimizer to receive
 *     confirmation of the completion of the previous checkpoint" (§4.3,
 *     P:511-515)                                       -> fp_ckpt_begin / fp_ckpt_wait
 *   - each DP rank writes only its portion of the (replicated) checkpoint,
 *     partitioned at setup, byte-balanced after serialization (§4.2,
 *     P:483-503)                                        -> dp_rank / dp_size
 *   - "Loading parallel checkpoints ... loads its checkpoint partition"
 *     (§4.2)                                     -> fp_ckpt_load
 *   - NVMe-optimised async I/O, DMA-able page-locked double buffering, aligned
 *     writes (§4.1)                          -> fp_config
 * The on-disk image is FPCK v2.
 *
 * Conventions
 *   - Every int-returning call returns 0 on success or a NEGATIVE error:
 *     -errno (EINVAL, ENOMEM, EBUSY, EIO, ENOSPC, ENOENT, ...) or an FP_E* code.
 *   - No call throws; no call aborts the process on bad input.
 *   - Pointers passed in are borrowed; nothing is freed by the library
 *     except what it allocated itself (ctx, pinned ring, device slab).
 *   - No torch types: plain pointers, sizes and an opaque cudaStream_t.
 */
#ifndef FASTPERSIST_H
#define FASTPERSIST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FP_ABI_VERSION 2

/* ---- error codes beyond -errno ----------------------------------------- */
#define FP_EMISMATCH (-1001) /* layout differs across ranks, or load target != file */
#define FP_ECORRUPT  (-1002) /* manifest / header / extent inconsistent on load     */
#define FP_ECUDA     (-1003) /* a CUDA runtime call failed                           */
#define FP_ENODEV    (-1004) /* device tensors given but no CUDA device in this ctx  */
#define FP_ECOMM     (-1005) /* a comm callback returned an error                    */

/* ---- tensor metadata ("data type, data size, originating device") - */
enum fp_dtype { FP_F32 = 1, FP_BF16 = 2, FP_F16 = 3, FP_F64 = 4, FP_I64 = 5,
                FP_I32 = 6, FP_U8 = 7 };
enum fp_section { FP_SEC_PARAM = 0, FP_SEC_GRAD = 1, FP_SEC_MASTER = 2,
                  FP_SEC_EXP_AVG = 3, FP_SEC_EXP_AVG_SQ = 4, FP_SEC_OTHER = 5 };

#define FP_TENSOR_HOST 1u   /* data is a host pointer (host-resident state).     */

typedef struct fp_tensor {
  const void *data;   /* device pointer (or host pointer with FP_TENSOR_HOST);
                         contiguous bytes [data, data+nbytes). Borrowed: must stay
                         alive and UNMODIFIED from fp_ckpt_begin until
                         fp_ckpt_wait returns (the optimizer fence).
                         Any alignment is accepted; 16-B alignment takes the
                         vector/TMA fast path.                                  */
  uint64_t nbytes;    /* = numel * itemsize(dtype), else -EINVAL                 */
  const char *name;   /* UTF-8, NUL-terminated, 1..65535 bytes                    */
  int64_t shape[8];   /* first ndim entries used                                 */
  int32_t owner;      /* -1: replicated on all DP ranks (byte-range sharded,
                         P:485); r >= 0: rank r's own partition (ZeRO shard /
                         local experts), written whole by rank r; must equal
                         the caller's dp_rank                                    */
  uint8_t dtype;      /* enum fp_dtype   */
  uint8_t section;    /* enum fp_section */
  uint8_t ndim;       /* 0..8            */
  uint8_t flags;      /* FP_TENSOR_*     */
} fp_tensor;

/* ---- collectives supplied by the caller (torch.distributed NCCL group) -----
 * Called ONLY on the caller's thread, inside fp_ckpt_begin (first call for a
 * new tensor signature: all-gather of per-rank sizes + layout digest)
 * and fp_ckpt_wait (status all-reduce = completion barrier). Return 0 or <0. */
typedef struct fp_comm {
  void *ctx;
  /* send: n_per_rank values; recv: dp_size * n_per_rank values, rank-major   */
  int (*allgather_u64)(void *ctx, const uint64_t *send, uint64_t *recv,
                       uint64_t n_per_rank);
  /* in-place MIN over ranks                                                  */
  int (*allreduce_min_i32)(void *ctx, int32_t *inout);
  /* optional (NULL if unsupported; needed only by fp_ckpt_load_parallel with
   * dp_size > 1): all-gather of `bytes` bytes per rank, rank-major:
   * recv[r*bytes, (r+1)*bytes) = rank r's send. on_device = 1: send/recv are
   * device pointers and the exchange must be ordered on `stream`
   * (cudaStream_t) — after work already enqueued there, before work enqueued
   * after the call returns (NCCL all-gather over NVLink on the B200 box);
   * on_device = 0: host pointers, complete on return.                         */
  int (*allgather_bytes)(void *ctx, const void *send, void *recv, uint64_t bytes,
                         int on_device, void *stream);
} fp_comm;

/* ---- configuration ------------------------------------------------------ */
enum fp_io_engine { FP_IO_URING = 0,    /* io_uring, O_DIRECT, registered bufs */
                    FP_IO_PWRITE = 1,   /* pwrite thread pool, O_DIRECT         */
                    FP_IO_BUFFERED = 2, /* pwrite through the page cache        */
                    FP_IO_NULL = 3,     /* ablation: requests complete at once,
                                           nothing is written (measures the
                                           pack + D2H + ring ceiling)           */
                    FP_IO_GDS = 4       /* GPUDirect Storage: device
                                           state is packed into a doubled device
                                           slab and written with cuFileWrite from
                                           HBM (no pinned ring); libcufile is
                                           loaded at run time (fp_ckpt_init ->
                                           -ENOSYS without it). Without nvidia-fs
                                           libcufile runs in compatibility mode:
                                           stats.fallback = 2. Needs a device and
                                           a slab pack (v4/bulk); loads and host
                                           state use io_uring.                   */ };
enum fp_pack_impl { FP_PACK_V4 = 0,     /* LSU 16-B vector gather -> device slab,
                                           then copy engine -> pinned ring; the
                                           page CRCs by a second kernel over
                                           the slab                              */
                    FP_PACK_BULK = 1,   /* default: cp.async.bulk (TMA engine)
                                           via smem -> device slab, the page
                                           CRCs computed from the smem stages in
                                           the same kernel; then copy engine     */
                    FP_PACK_HOST = 2,   /* fused: the v4 kernel stores straight
                                           into the mapped pinned ring slot
                                           (zero-copy D2H over PCIe, no slab)    */
                    FP_PACK_CE = 3,     /* ablation, no kernel: one copy-engine
                                           cudaMemcpyAsync per contiguous run of
                                           a chunk, tensors -> pinned ring       */
                    FP_PACK_LSU = 4     /* LSU 16-B vector gather -> device slab,
                                           the page CRCs computed from the
                                           registers the data passes through (one
                                           kernel, no smem staging); then copy
                                           engine                                */ };

#define FP_CFG_NO_FSYNC 1u     /* skip fdatasync (benchmark ablation only)       */
#define FP_CFG_NO_CRC   4u     /* skip the per-shard CRC-32          */
#define FP_CFG_PRIO_LOW 2u     /* pack/D2H stream at the least priority (default:
                                  greatest)                    */
#define FP_CFG_BALANCE_BYTES 8u /* partition the replicated region on BYTE
                                  granularity (imbalance <= 1 byte;
                                  env FP_BALANCE_BYTES=1) instead of `alignment`
                                  pages: shard starts are then unaligned in the
                                  image (the pack gathers byte-shifted) and each
                                  shard's unaligned suffix (< alignment bytes)
                                  is written with buffered I/O into the same
                                  file (P:477 prefix/suffix); the manifest
                                  records it ("balance": "bytes") and loads
                                  follow the manifest                            */

typedef struct fp_config {
  uint32_t ring_slots;   /* pinned host slots; 2 = the paper's double buffer
                            (P:473); default 4                                   */
  uint32_t io_depth;     /* max in-flight I/O requests per rank; default 64      */
  uint64_t slot_bytes;   /* bytes per slot = one chunk; multiple of alignment;
                            default 64 MiB                                       */
  uint32_t sqe_bytes;    /* bytes per write request; default 1 MiB               */
  uint32_t alignment;    /* power of two >= 512; default 4096           */
  uint32_t io_engine;    /* enum fp_io_engine; default FP_IO_URING              */
  uint32_t pack_impl;    /* enum fp_pack_impl; default FP_PACK_BULK             */
  uint32_t pack_ctas;    /* 0 = whole GPU (burst); else CTA cap (background)    */
  uint32_t flags;        /* FP_CFG_*                                             */
  const char *dirs;      /* nullable: comma-separated roots; rank r's shard goes
                            under dirs[r % n]; the manifest under dirs[0].
                            NULL: `path` is used as given.                       */
  uint32_t writer_stride;/* writer subset: only ranks r with
                            r % writer_stride == 0 write replicated bytes
                            (e.g. one writer per CPU socket, the paper's
                            "Socket" strategy); 0/1 = every rank ("Replica").
                            Rank-local regions are always written by their
                            owner. Default 1 (env FP_WRITER_STRIDE).          */
  uint64_t pack_bytes;   /* bytes gathered per pack-kernel launch (device slab
                            size); rounded up to a multiple of slot_bytes, so one
                            launch feeds pack_bytes/slot_bytes ring slots; 0 =
                            slot_bytes; default 1 GiB (a launch carries ~12 us
                            of fixed cost: 256 MiB groups reach 0.90 of HBM,
                            1 GiB 0.98 — profiles/r02_pack_group_size.md),
                            max 2 GiB                                          */
} fp_config;

/* ---- per-checkpoint statistics ------------------------------------------ */
typedef struct fp_stats {
  uint64_t image_bytes;    /* whole FPCK image (all ranks)                       */
  uint64_t header_bytes;   /* GHDR bytes                                          */
  uint64_t shard_bytes;    /* bytes this rank wrote                               */
  uint64_t chunks;         /* ring chunks this rank staged                        */
  uint64_t io_requests;    /* write requests submitted                            */
  uint64_t pack_launches;  /* pack kernel launches                                */
  uint64_t pack_bytes;     /* slab bytes produced by those launches               */
  double   pack_ms;        /* sum of CUDA-event durations of the pack launches    */
  double   d2h_ms;         /* sum of CUDA-event durations of the D2H copies       */
  double   t_total;        /* s, begin -> wait return (incl. barrier + commit)    */
  double   t_helper;       /* s, helper start -> local durability                 */
  double   t_fsync;        /* s, fdatasync                                        */
  double   t_barrier;      /* s, status all-reduce in wait                        */
  double   t_commit;       /* s, manifest write + rename + dir fsync (rank 0)     */
  double   t_io_stall;     /* s, helper time blocked waiting for I/O completions  */
  uint32_t max_inflight;   /* peak in-flight I/O requests                         */
  uint32_t fallback;       /* 1 if O_DIRECT was unavailable -> buffered I/O;
                              2 if FP_IO_GDS ran in cuFile compatibility mode  */
  int32_t  engine;         /* enum fp_io_engine actually used                     */
  int32_t  status;         /* final status of this checkpoint                     */
  int64_t  err_offset;     /* file offset of the first failed request, or -1      */
  uint32_t shard_crc32;    /* CRC-32 (IEEE, = zlib.crc32) of this rank's shard
                              file; computed on the GPU from the packed slab
                              (host tensors: on the CPU); also in the manifest  */
  uint32_t crc_valid;      /* 1 if shard_crc32 was computed                       */
  uint64_t kernel_launches;/* all library kernels launched (pack, CRC, gate)      */
  double   crc_ms;         /* sum of CUDA-event durations of the page-CRC kernel
                              after each pack (folded per extent on the host)  */
  int32_t  numa_node;      /* NUMA node the pinned ring and helper thread were
                              placed on (the GPU's; -1: unknown / not placed)  */
} fp_stats;

/* ---- statistics of the last load (fp_ckpt_load / fp_ckpt_load_parallel) -- */
typedef struct fp_load_stats {
  uint64_t bytes_read;      /* bytes this rank read from storage                  */
  uint64_t kernel_launches; /* library kernels launched (unpack, page CRCs)       */
  double   t_total;         /* s, call -> return                                  */
  int32_t  exchange;        /* 0: none (dp_size 1, or fp_ckpt_load); 1: one
                               comm->allgather_bytes per chunk + fp_unpack_v4;
                               2: peer memory (fp_unpack_peer reads every
                               writer's partition from its device buffer)      */
  int32_t  status;          /* return code of that load                           */
  double   t_exchange_wait; /* s the host waited for peers' chunks (exchange 2)    */
  double   t_setup;         /* s from the call to the first chunk (manifest,
                               plan, buffers, exchange setup)                    */
  double   t_read_wait;     /* s the host waited for its own-shard reads          */
} fp_load_stats;

typedef struct fp_ctx fp_ctx;

/* Fill *cfg with the defaults above (env overrides: FP_RING_SLOTS,
 * FP_SLOT_BYTES, FP_SQE_BYTES, FP_QD, FP_IO_ENGINE=uring|pwrite|buffered|null|gds,
 * FP_PACK=bulk|lsu|v4|host|ce, FP_PACK_PRIO=low, FP_PACK_CTAS, FP_ALIGN, FP_PACK_BYTES,
 * FP_WRITER_STRIDE, FP_CKPT_DIRS, FP_NO_CRC). Returns 0.
 * Read at run time (not part of fp_config): FP_NO_TMA=1 (LSU page-CRC kernel
 * instead of the TMA-staged one), FP_LAUNCH_GATE=1 (measurement: queue each pack group
 * behind a one-warp gate the helper opens after enqueueing, so CUDA events
 * time the kernel alone; off by default and under a profiler), FP_NUMA=0 (do
 * not place the ring / helper on the GPU's NUMA node), FP_GDS_OPEN_TIMEOUT
 * (s, default 20), FP_DEBUG_GDS=1, FP_FAULT_EIO_AT=<n>[@rank] and
 * FP_FAULT_KILL_AT=<n>[@rank] (tests).                                         */
int fp_config_default(fp_config *cfg);

/* Create a context bound to CUDA device `cuda_device` (-1: host tensors only).
 * Allocates the pinned ring (slots*slot_bytes, page-locked and registered with
 * the I/O engine; its pages and the helper thread are placed on the GPU's
 * NUMA node), one device slab of pack_bytes, a CUDA stream and
 * the helper thread. `comm` may be NULL only if every call uses dp_size == 1.
 * *out receives the context. Errors: -EINVAL (bad config), -ENOMEM, FP_ECUDA. */
int fp_ckpt_init(const fp_config *cfg, int cuda_device, const fp_comm *comm,
                 fp_ctx **out);

/* Start checkpoint `path` (a directory; created if missing) of the tensor list
 * t[0..n) — caller order is image order (P:479 order preserved). Returns after
 * enqueueing (microseconds when the tensor signature is unchanged); the first
 * pack kernel waits on an event recorded on `producer_stream` (cudaStream_t;
 * NULL = legacy default stream), so it sees the optimizer's writes.
 * On a new signature this call runs the layout + partition setup, including
 * one comm->allgather_u64 (collective: all ranks must call begin together).
 * Rank r writes `<path>/shard-<r>-of-<dp_size>.fpck`.
 * Errors: -EINVAL (bad tensor, owner != dp_rank, dp_rank >= dp_size, mixed
 * host/device tensors), -EBUSY (a checkpoint is outstanding: at most one,
 * S:361), FP_EMISMATCH (replicated layouts differ across ranks), FP_ENODEV,
 * FP_ECOMM, -ENOMEM.                                                          */
int fp_ckpt_begin(fp_ctx *ctx, const fp_tensor *t, size_t n, const char *path,
                  int dp_rank, int dp_size, void *producer_stream);

/* Stream-ordered fence: enqueue on `stream` (cudaStream_t)
 * a wait (a one-warp kernel polling a mapped pinned word) that holds every
 * later operation of that stream until this rank's shard of the outstanding
 * checkpoint is durable (fdatasync'd) — or has failed. Returns at once: the
 * host thread keeps enqueueing the optimizer while the GPU, not the host,
 * waits (the paper's main thread blocks). fp_ckpt_wait is still
 * required afterwards for the cross-rank barrier, error status and manifest
 * commit; it returns -ETIMEDOUT if a fence gave up after one hour. 0 if
 * nothing is outstanding; -ENOSYS for a host-only context; FP_ECUDA.          */
int fp_ckpt_fence(fp_ctx *ctx, void *stream);

/* Block until the outstanding checkpoint is durable everywhere: this rank's
 * shard is fdatasync'd, the status all-reduce (barrier) has completed, and
 * rank 0 has committed manifest.json (tmp + rename + dir fsync). Collective
 * when dp_size > 1. Returns 0 if nothing is outstanding. On any rank's failure
 * every rank returns that (most negative) error and no manifest is committed.
 * `out` (nullable) receives the statistics.                                    */
int fp_ckpt_wait(fp_ctx *ctx, fp_stats *out);

/* Restore tensors t[0..n) (same names/dtypes/shapes/order as saved, each
 * rank passing its own local tensors) from checkpoint `path` written with
 * the same dp_size. Reads the manifest, validates every header against the
 * target list, O_DIRECT-reads the needed extents through the pinned ring and
 * scatters them into t[i].data with the unpack kernel on `stream`. Synchronous.
 * Errors: -ENOENT (missing manifest or shard, named on stderr), FP_ECORRUPT,
 * FP_EMISMATCH, -EIO, -EBUSY (a save is outstanding).                         */
int fp_ckpt_load(fp_ctx *ctx, const fp_tensor *t, size_t n, const char *path,
                 int dp_rank, int dp_size, void *stream);

/* Parallel restore, the paper's two-step load (§4.2: each rank "(i)
 * loads its checkpoint partition, if any, into GPU memory, and (ii) performs
 * an allgather"): rank r reads ONLY its own shard file, in slot_bytes chunks
 * (O_DIRECT through the pinned ring, ring_slots chunks ahead, then H2D; with
 * FP_IO_GDS, cuFileRead into device memory instead).
 * Exchange of the replicated partitions (fp_load_stats.exchange):
 *   2 = peer memory (default for device state, dp_size > 1): the whole own
 *       replicated partition is copied into a device buffer of this ctx
 *       (part bytes + 4 B per chunk of ready flags), the buffers are mapped
 *       into every rank (CUDA IPC handles exchanged with comm->allgather_u64;
 *       the same pointers for ranks that are threads of one process) and one
 *       fp_unpack_peer launch per chunk on `stream` scatters the chunk of
 *       every writer straight from its buffer into t[i] (P2P loads over
 *       NVLink). Each writer's copy engine sets a ready flag per chunk (a
 *       4-byte copy behind the chunk's H2D into a POSIX shared-memory
 *       segment registered with CUDA); the host launches the unpack of chunk
 *       j once every writer's flag j is set (no GPU-side spinning).
 *       FP_LOAD_EXCHANGE=peer requires it (-ENOSYS if a buffer cannot be
 *       mapped), =nccl disables it. FP_PEER_TIMEOUT_S (600) bounds the wait
 *       for a peer (then FP_ECOMM).
 *   1 = gathered (host state, or no IPC): one comm->allgather_bytes per chunk
 *       (bytes = slot_bytes per rank; shorter partitions send padding), then
 *       fp_unpack_v4 from the gathered buffer.
 * The rank's own local region comes from its own shard. GHDR / LHDR bytes
 * are checked against the target list after the exchange and the own shard's
 * CRC-32 (per extent) against the manifest. Collective: every rank of the DP
 * group calls it together; a failure on any rank is returned on all ranks
 * (status all-reduce before the first exchange and at the end). The targets
 * are written as chunks arrive: on an error return they hold unspecified
 * bytes. Synchronous.
 * Errors: those of fp_ckpt_load, plus -ENOSYS when dp_size > 1, peer mode is
 * unavailable and comm->allgather_bytes is NULL; FP_ECOMM.                    */
int fp_ckpt_load_parallel(fp_ctx *ctx, const fp_tensor *t, size_t n, const char *path,
                          int dp_rank, int dp_size, void *stream);

/* Statistics of the last fp_ckpt_load / fp_ckpt_load_parallel on this ctx.
 * 0, or -EINVAL for a NULL argument.                                          */
int fp_ckpt_load_stats(fp_ctx *ctx, fp_load_stats *out);

/* Image facts of the last planned checkpoint of this ctx: image/header bytes and
 * this rank's extents as (image_offset, file_offset, length) triples.
 * *n_ext receives the extent count; at most max_ext are written. -ENOENT if
 * nothing was planned yet.                                                    */
int fp_ckpt_plan_info(fp_ctx *ctx, uint64_t *image_bytes, uint64_t *header_bytes,
                      uint64_t *extents, uint32_t max_ext, uint32_t *n_ext);

/* Release everything (waits for an outstanding checkpoint first).            */
void fp_ckpt_destroy(fp_ctx *ctx);

/* Human-readable text for a return code (static storage).                    */
const char *fp_strerror(int err);

/* Storage roofline tool (the built-in substitute for fio): with the
 * configured engine (O_DIRECT, io_depth x sqe_bytes from a registered pinned
 * ring) write `bytes` of non-compressible host data to `<dir>/fp_iobench.<tag>`
 * and fdatasync (untimed pass: allocates every block), then overwrite the same
 * file sequentially and fdatasync again, twice (timed passes), unlink.
 * *gbps = bytes / (faster timed pass seconds) / 1e9 — a roofline is the best
 * the device did, not its average.                                            */
int fp_io_bench(const char *dir, uint64_t bytes, const fp_config *cfg, int tag,
                double *gbps);

/* Read roofline for the restore path: write `bytes` to
 * `<dir>/fp_iobench.<tag>` as fp_io_bench does (untimed, fdatasync'd), then
 * read the file back sequentially with the configured engine (O_DIRECT,
 * io_depth x sqe_bytes into the registered pinned ring), twice (timed), unlink.
 * *gbps = bytes / (faster timed read pass seconds) / 1e9. Same errors as
 * fp_io_bench.                                                                */
int fp_io_bench_read(const char *dir, uint64_t bytes, const fp_config *cfg, int tag,
                     double *gbps);

/* ---------------------------------------------------------------------------
 * Byte-stream writer: the paper's torch.save integration (§5.1 P:532-533:
 * "implementing FastPersist in a compatible object that we pass to
 * torch.save() ... with no change to other operations (e.g., tensor
 * serialization)") on the NVMe path of §4.1: the stream's bytes go through
 * an IO buffer of ring_slots x slot_bytes page-aligned host memory (P:467-473:
 * ring_slots = 1 is the paper's single-buffer mode, >= 2 double buffering —
 * slot i+1 fills while slot i is being written) and every full slot is
 * written with O_DIRECT at its file offset (cfg->io_engine, sqe_bytes per
 * request, io_depth in flight). At close the last slot's aligned prefix goes
 * the same way and the < alignment suffix through a buffered descriptor of
 * the same file ("the suffix using traditional I/O libraries, into
 * the same checkpoint file"), then both are fdatasync'd. The file is
 * byte-for-byte what a plain write() of the same stream gives.
 * ------------------------------------------------------------------------- */
typedef struct fp_stream fp_stream;
typedef struct {
  uint64_t bytes;         /* stream length = file size                         */
  uint64_t direct_bytes;  /* written by the engine (O_DIRECT unless fallback)  */
  uint64_t suffix_bytes;  /* written by the buffered descriptor (< alignment)  */
  double t_total;         /* open -> close return, s                           */
  double t_fill;          /* copying into the IO buffer (memcpy or D2H), s     */
  double t_io_wait;       /* waiting for a slot's writes to complete, s        */
  double t_fsync;         /* final fdatasync, s                                */
  uint32_t fallback;      /* 1: the file system refused O_DIRECT (buffered)    */
  uint32_t requests;      /* engine write requests                             */
} fp_stream_stats;

/* Create or overwrite `path` (an existing file is overwritten in place and
 * cut to the stream's length at close) and allocate the IO buffer (ring_slots x
 * slot_bytes; cfg NULL = defaults). cuda_device >= 0 also registers the
 * buffer with CUDA for fp_stream_write_device (page-locked); -1 = host
 * bytes only. The buffer of a closed stream is kept (two at most) and reused
 * by the next stream of the same ring shape, as the paper's helper allocates
 * its page-locked buffer once. Errors: -EINVAL (bad cfg), -ENOMEM,
 * -errno of open, FP_ECUDA.                                                  */
int fp_stream_open(const fp_config *cfg, int cuda_device, const char *path, fp_stream **out);
/* Append n host bytes (copied into the IO buffer; returns once they are
 * copied — full slots are written asynchronously). -EIO / -errno of a failed
 * earlier write (the stream is then failed; close still frees it).          */
int fp_stream_write(fp_stream *s, const void *buf, uint64_t n);
/* Append n bytes of device memory: copy-engine D2H straight into the
 * page-locked IO buffer on `stream` (cudaStream_t), slot by slot (GPU
 * -> page-locked CPU memory -> NVMe). Needs cuda_device >= 0 at open.
 * Synchronous with respect to the copies. -EINVAL without a device.        */
int fp_stream_write_device(fp_stream *s, const void *dev_ptr, uint64_t n, void *stream);
/* Flush (aligned prefix O_DIRECT, suffix buffered), fdatasync, close, free.
 * Always frees s. Returns 0 or the first error; *st (nullable) filled.      */
int fp_stream_close(fp_stream *s, fp_stream_stats *st);

#ifdef __cplusplus
}
#endif
#endif /* FASTPERSIST_H */
