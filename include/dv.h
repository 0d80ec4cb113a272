/*
 * dv.h -- C ABI of dvstream, a B200-native implementation of DejaVuLib's KV-cache streaming
 * hot path (Strati et al., "DejaVu: KV-cache Streaming for Fast, Fault-tolerant Generative LLM
 * Serving", arXiv 2403.01876).
 *
 * The three levels follow the paper's primitives (Table 1):
 *   dv_stream_out / dv_stream_in   "Given a source (or destination) worker, the KV cache, and the
 *                                   inference setup ... find the proper destinations (or sources)
 *                                   for the different chunks of KV cache. This might involve
 *                                   splitting the cache at the source or merging cache chunks at
 *                                   the destination."
 *   dv_scatter / dv_gather         "Given a non-contiguous region of KV cache, and a local or
 *                                   remote destination (or source), chunk the region to
 *                                   contiguous transfers and orchestrate movement."
 *   dv_flush / dv_fetch            "Copy a contiguous chunk of KV cache, on the same or remote
 *                                   host."
 * Note the naming: the paper's `scatter` is the SEND side (non-contiguous region -> contiguous
 * chunk); its kernel is called "pack" inside the library, `gather`'s kernel "unpack".
 *
 * Conventions (all calls):
 *   - Every function returns a dv_status; on failure dv_last_error() holds a message (thread-local).
 *   - Validation happens before anything is enqueued: an error has no partial effect.
 *   - Data calls are asynchronous and stream-ordered on `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream). No call synchronises the device except dv_destroy and the
 *     explicitly blocking dv_query on device-resident flags.
 *   - The caller owns KV caches, inboxes it allocated, and streams. The library owns its staging
 *     pool, ticket counters and anything returned by dv_host_alloc/dv_device_alloc until freed.
 *   - There is no CPU fallback: without a usable CUDA device every data call fails (DV_ECUDA).
 *
 * Data layout (reading Q1 of DESIGN.md; PAPER.md:131 fn 5, PAPER.md:119 preallocation):
 *   DV_LAYOUT_KV5D: K and V are each [n_layers][n_reqs][n_heads][max_seq][head_dim] arrays of
 *   elem_bytes-wide words, dense, row-major; element (l, r, h, s, d) (cache-local l, r) sits at
 *   byte ((((l*n_reqs + r)*n_heads + h)*max_seq + s)*head_dim + d)*elem_bytes.
 *   Words are opaque (fp16/bf16 bit patterns are moved, never converted; NaN payloads survive).
 *
 * Wire format (reading Q3): a region [l0,l1)x[r0,r1)x[s0,s1)x[h0,h1) packs to the dense array
 *   [l-l0][kv][r-r0][h-h0][s-s0][d]  (kv: 0 = K, 1 = V), 2*nL*nR*nH*n*D*e bytes, d fastest,
 *   whatever the cache layout (KV5D or FT6D) on either side.
 *
 * Alignment: cache bases, endpoint bases/offsets and head_dim*elem_bytes must be multiples of
 * 16 bytes (else DV_EALIGN).
 */
#ifndef DV_H_
#define DV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DV_ABI_VERSION 4   /* 4: device plans (dv_dplan_*), SM partitions (dv_partition_*) */

#if defined(__GNUC__)
#define DV_API __attribute__((visibility("default")))
#else
#define DV_API
#endif

typedef enum dv_status {
  DV_OK = 0,
  DV_EINVAL = 1,  /* malformed argument (NULL pointer, negative extent, bad enum, capacity)   */
  DV_EMAP = 2,    /* setups / caches do not hold the region's layers or requests */
  DV_ERANGE = 3,  /* pos_end exceeds max_seq on a side; message names the limit  */
  DV_EALIGN = 4,  /* a base/offset or head_dim*elem_bytes is not a multiple of 16 bytes        */
  DV_ENOMEM = 5,  /* staging pool or an allocation could not be satisfied                     */
  DV_EPEER = 6,   /* IPC export/open failed or a blob is malformed                            */
  DV_EBUSY = 7,   /* DV_NOWAIT: the inbox ring slot has no credit yet (receiver not done)     */
  DV_ECUDA = 8,   /* a CUDA runtime/driver call failed; its text is in dv_last_error()        */
  DV_ENOTSUP = 9  /* valid request this build does not implement                              */
} dv_status;

/* Cache layouts (reading Q1; PAPER.md:131 fn 5 "the key cache is a 6D tensor, and the value cache
 * is a 5D tensor"):
 *   DV_LAYOUT_KV5D  K and V both [n_layers][n_reqs][n_heads][max_seq][head_dim].
 *   DV_LAYOUT_FT6D  K [n_layers][n_reqs][n_heads][head_dim/x][max_seq][x] with x = 16/elem_bytes
 *                   (FasterTransformer's key layout: 16-byte packets of d, position-major inside
 *                   each packet column), V as in KV5D. */
enum { DV_LAYOUT_KV5D = 0, DV_LAYOUT_FT6D = 1 };

/* A worker's K and V cache, preallocated to max_seq. Descriptor only: the library
 * never allocates or frees caches. */
typedef struct dv_cache {
  void* k;             /* K base (device, mapped pinned host, or IPC-mapped peer memory)        */
  void* v;             /* V base                                                                 */
  int32_t device;      /* owning CUDA device ordinal, or -1 for pinned host memory              */
  int32_t layout;      /* DV_LAYOUT_*                                                           */
  int32_t elem_bytes;  /* bytes per word (2 for fp16/bf16); head_dim*elem_bytes % 16 == 0       */
  int32_t layer_begin; /* global id of the first layer held (a pipeline stage's layers)         */
  int32_t n_layers;
  int32_t req_begin;   /* global id of the first request held (a microbatch's requests)         */
  int32_t n_reqs;
  int32_t n_heads;     /* heads held (a tensor-parallel shard holds a head range)                */
  int32_t max_seq;     /* preallocated positions S                                              */
  int32_t head_dim;
  int32_t head_begin;  /* global id of the first head held (0 without tensor parallelism)        */
} dv_cache;

/* Half-open box of GLOBAL layer ids x GLOBAL request ids x absolute positions (reading Q5) x
 * GLOBAL head ids. head_begin == head_end == 0 means "all heads": the heads of the cache in the
 * level-2 calls (the source cache's for dv_remap), the heads covered by the setups in the route. */
typedef struct dv_region {
  int32_t layer_begin, layer_end;
  int32_t req_begin, req_end;
  int32_t pos_begin, pos_end;
  int32_t head_begin, head_end;
} dv_region;

/* A pipeline configuration: layers partitioned over n_stages stages (PP),
 * requests split into n_micro microbatches, and -- optionally -- heads split over n_tp tensor-
 * parallel ranks inside a stage. Bounds are global ids, strictly
 * increasing. n_tp = 0 (head_bounds NULL): no head split, every block holds all heads.
 * A block is (stage, micro, tp); its flat index is (stage*n_micro + micro)*max(n_tp,1) + tp. */
typedef struct dv_setup {
  int32_t n_stages;
  const int32_t* layer_bounds; /* n_stages + 1 entries */
  int32_t n_micro;
  const int32_t* req_bounds;   /* n_micro + 1 entries  */
  int32_t max_seq;
  int32_t n_tp;                /* 0 = no head split                    */
  const int32_t* head_bounds;  /* n_tp + 1 entries, or NULL            */
} dv_setup;

/* One route piece = region x source block x destination block (all non-empty).
 * Pieces come in lexicographic order of (src block flat index, dst block flat index).
 * src_wire_off / dst_wire_off: byte offset of this piece's wire chunk among the pieces leaving
 * the source block / entering the destination block, cumulative in piece order. head range
 * [0,0) means all heads (neither setup splits heads). */
typedef struct dv_piece {
  int32_t src_stage, src_micro, dst_stage, dst_micro;
  int32_t layer_begin, layer_end, req_begin, req_end, pos_begin, pos_end;
  uint64_t bytes;
  uint64_t src_wire_off;
  uint64_t dst_wire_off;
  int32_t src_tp, dst_tp;
  int32_t head_begin, head_end;
} dv_piece;

/* Where contiguous chunks go / come from (the paper's flush/fetch targets). */
enum {
  DV_EP_DEVICE = 0, /* local device memory (e.g. a staging buffer or local inbox)                */
  DV_EP_HOST = 1,   /* pinned, device-mapped host memory (swap arena / host log)  */
  DV_EP_PEER = 2    /* another GPU's memory mapped into this process (CUDA IPC) over NVLink     */
};

/* An inbox may be a RING of n_slots chunk slots with per-source CREDITS (SURVEY §8(a) A5 "inbox
 * credits per slot"; the paper's token machines consume a mailbox). Then, for flag
 * slot f (one per source block) and sequence number s >= 1:
 *   - the chunk of seq s lives in ring slot s % n_slots: at base + (s % n_slots)*slot_bytes + off,
 *     and off + chunk bytes must fit slot_bytes;
 *   - the SENDER (dv_scatter / dv_flush / dv_stream_out with flag slot f and seq s) may overwrite
 *     that slot only once the receiver has consumed seq s - n_slots: its copy is stream-ordered
 *     after credits[f] >= s - n_slots (a stream memory-op wait on host or own-GPU memory, a
 *     one-thread acquire-spin kernel on peer memory), or -- with DV_NOWAIT -- the call returns
 *     DV_EBUSY without enqueueing anything when the credit is not there yet;
 *   - the RECEIVER (dv_gather / dv_fetch / dv_stream_in with flag slot f and wait_seq s) reads ring
 *     slot s % n_slots after flags[f] >= s and, once its copy has read the chunk, releases
 *     credits[f] = s (the copy kernel's own release store, at the scope the memory needs).
 * Sequence numbers of one source are consecutive (1, 2, 3, ...). credits == NULL: ring addressing
 * without flow control. n_slots == 0: a plain buffer (no ring, no credits). */
typedef struct dv_endpoint {
  int32_t kind;     /* DV_EP_*                                                                  */
  int32_t device;   /* device owning the memory (-1 for host)                                  */
  void* base;       /* address usable from the calling device (device/host-mapped/IPC-mapped)  */
  uint64_t bytes;   /* capacity                                                                */
  uint64_t* flags;  /* n_flags monotone 64-bit sequence words (same accessibility as base), or NULL */
  int32_t n_flags;
  int32_t n_slots;      /* ring depth; 0 = no ring                                             */
  uint64_t slot_bytes;  /* bytes per ring slot (multiple of 16; n_slots * slot_bytes <= bytes)  */
  uint64_t* credits;    /* n_flags credit words (consumed seq per source), or NULL               */
} dv_endpoint;

/* Transfer-method flags for the data calls. DV_XFER_AUTO lets the library pick (DESIGN.md §6
 * "Transfer choice"): kernel stores for host writes < 32 MB, staged pipelined DMA above; kernel
 * loads for host reads < 4 MiB, staged DMA above; kernel copies for device / peer memory. When AUTO
 * picks staging but the pool cannot hold one staging unit (a run, a layer slab, or -- for K and V
 * of different layouts -- a (layer, K or V) half-slab), AUTO uses the kernel's own copies; an
 * explicit DV_XFER_STAGED / DV_XFER_DECOUPLED then fails with DV_ENOMEM before enqueueing anything.
 * Flags are released by the copy kernel itself at the scope the memory needs: system scope when
 * the payload or the flag is in pinned host or peer memory, GPU scope when both are this GPU's
 * HBM (every reader of that memory is served by this GPU's L2). */
enum {
  DV_XFER_AUTO = 0,
  DV_XFER_FUSED = 1u << 0,  /* SM kernel reads/writes the endpoint memory directly (zero-copy / P2P) */
  DV_XFER_STAGED = 1u << 1, /* kernel <-> local staging, copy engine DMA for the contiguous chunk */
  DV_PUBLISH_STREAMOP = 1u << 2, /* publish flags with a stream memory operation after the kernel
                                    instead of the kernel's own fenced release store            */
  DV_XFER_DECOUPLED = 1u << 3, /* scatter / stream_out to a pinned-HOST endpoint only: the caller's
                                  stream is ordered after the pack (the source may be rewritten),
                                  the copy-engine DMA and the flag store run on the context's DMA
                                  stream -- the FLAG is the only completion signal (PAPER.md:171,
                                  stream_out is non-blocking; the receiver's stream_in / dv_wait
                                  waits on the flag). Successive steps then overlap step t's DMA
                                  with step t+1's pack. Requires a flag (flag_slot >= 0, no
                                  DV_NO_FLAG); with AUTO it selects STAGED. Ignored for device and
                                  peer endpoints (the caller's stream already covers them). A
                                  slot may mix modes: once a context has published decoupled
                                  flags, its other publishes to pinned-host flags are ordered
                                  after them (an empty decoupled region publishes on the flag
                                  stream too), so a slot's seq never runs ahead of a DMA in
                                  flight -- except for launches captured into a CUDA graph, which
                                  the caller orders after earlier decoupled transfers.          */
  DV_NOWAIT = 1u << 4,      /* senders into a credited ring: DV_EBUSY instead of a stream-ordered
                               wait when a slot has no credit (checked from the host when called;
                               reading a device-memory credit is a small synchronous copy)     */
  DV_NO_FLAG = 1u << 8      /* do not publish / wait on sequence flags                           */
};

typedef struct dv_ctx dv_ctx;

typedef struct dv_config {
  uint64_t staging_bytes; /* device staging pool for DV_XFER_STAGED (0 = 256 MiB)                */
  int32_t max_ctas;       /* cap on CTAs per copy kernel (0 = 148 * 8)                           */
  int32_t host_ctas;      /* cap when the copy reads or writes pinned host memory (0 = 16): PCIe is
                             saturated by 8 SMs, the rest stay free for compute (DESIGN.md NEXT-2) */
} dv_config;

/* ---- errors ------------------------------------------------------------------------------ */
DV_API const char* dv_last_error(void);                 /* thread-local message of the last failure     */
DV_API const char* dv_status_str(dv_status s);
DV_API int32_t dv_abi_version(void);
/* Counters since the library was loaded (benchmark evidence): kernels launched by the library and
 * copy-engine DMA calls (cudaMemcpy*Async) it issued. Either pointer may be NULL. */
DV_API dv_status dv_stats(uint64_t* kernel_launches, uint64_t* dma_calls);

/* ---- pure host functions (no GPU needed) ------------------------------------------------- */
/* Bytes of K and V in a region: 2*nL*nR*(pos_end-pos_begin)*nH*head_dim*elem_bytes, nH = the
 * region's head count, or n_heads when its head range is [0,0) (SPEC.md:38
 * "2*L*hidden*element_bytes*batch*seq"). */
DV_API dv_status dv_region_bytes(const dv_region* region, int32_t n_heads, int32_t head_dim,
                          int32_t elem_bytes, uint64_t* out_bytes);

/* Route a region from src setup to dst setup (Table 1 stream_out/stream_in).
 * Writes up to `cap` pieces to `out` and the total count to *n (call with cap=0 to size).
 * n_heads is the model's head count used for byte sizes when neither setup splits heads.
 * Errors in order: DV_EINVAL (malformed setup/region; one setup splits heads and the other does
 * not), DV_EMAP (a setup does not hold the region's layers/requests/heads), DV_ERANGE (pos_end >
 * max_seq on either side). An empty region (any zero extent) yields 0 pieces. */
DV_API dv_status dv_route(const dv_setup* src, const dv_setup* dst, const dv_region* region,
                   int32_t n_heads, int32_t head_dim, int32_t elem_bytes, dv_piece* out,
                   uint64_t cap, uint64_t* n);

/* ---- context ----------------------------------------------------------------------------- */
/* One context per (process, device). Owns the staging pool, the release tickets and the CUDA
 * driver entry points it needs. `cfg` may be NULL. Loads every library kernel on `device` up front:
 * under CUDA lazy loading a first launch would otherwise wait for the device, and a consumer
 * kernel already spinning on one of our flags would block the very stream-out it waits for.
 * DV_ECUDA without a usable GPU (no CPU fallback); DV_ENOTSUP on a GPU other than sm_100 (B200):
 * the kernels are built for sm_100a only. */
DV_API dv_status dv_create(int32_t device, const dv_config* cfg, dv_ctx** out);
DV_API dv_status dv_destroy(dv_ctx* ctx); /* synchronises the device, frees library-owned memory */

/* ---- memory and peers -------------------------------------------------------------------- */
DV_API dv_status dv_host_alloc(uint64_t bytes, void** out);  /* pinned, portable, device-mapped */
/* Pinned host arena NUMA-local to `device` (SURVEY §8(b) "host memory"): on a multi-socket host
 * the pages are bound (mbind MPOL_BIND) to the host NUMA node closest to the GPU
 * (cudaDevAttrHostNumaId), populated, then page-locked and mapped (cudaHostRegister portable |
 * mapped), so PCIe transfers of that GPU never cross the socket interconnect. *node_out (may be
 * NULL) receives the node used, or -1 when the system has no NUMA information, in which case
 * this is dv_host_alloc. Free with dv_host_free. */
DV_API dv_status dv_host_alloc_near(int32_t device, uint64_t bytes, void** out, int32_t* node_out);
DV_API dv_status dv_host_free(void* p);
DV_API dv_status dv_device_alloc(int32_t device, uint64_t bytes, void** out); /* IPC-exportable */
DV_API dv_status dv_device_free(void* p);

/* One process driving several GPUs: let `device` access `peer`'s memory directly (NVLink P2P);
 * idempotent. Pointers of `peer` allocations can then be used as DV_EP_PEER endpoints or caches
 * in calls on `device`'s context. DV_EPEER if the pair cannot access each other. */
DV_API dv_status dv_peer_enable(int32_t device, int32_t peer);

typedef struct dv_ipc_blob { uint8_t bytes[128]; } dv_ipc_blob; /* opaque, copyable between processes */
/* Export device memory at `ptr` (any address inside a cudaMalloc allocation -- legacy CUDA IPC;
 * memory from the virtual-memory API, e.g. PyTorch with expandable_segments, or from
 * cudaMallocAsync pools cannot be exported this way: use dv_device_alloc or plain cudaMalloc for
 * inboxes, replica stores and flags that other processes map). DV_EPEER on failure. */
DV_API dv_status dv_ipc_export(const void* ptr, dv_ipc_blob* out);
/* Map a blob exported by another process (same or other GPU) into this process; returns the
 * address corresponding to the exported `ptr`. Same-process blobs map to the original pointer:
 * a blob carries a random 64-bit token of its exporting process (not the pid, which another PID
 * namespace may reuse). The blob records the exported extent (allocation end - ptr); every data
 * call checks that a cache or endpoint inside an IPC mapping fits the mapped extent (DV_EPEER). */
DV_API dv_status dv_ipc_open(const dv_ipc_blob* blob, void** out);
/* The exported extent of a blob in bytes (ptr .. end of its allocation), for sizing descriptors. */
DV_API dv_status dv_ipc_blob_bytes(const dv_ipc_blob* blob, uint64_t* out);
DV_API dv_status dv_ipc_close(void* mapped);

/* ---- level 3: flush / fetch ----------------------------------------------- */
/* Copy `bytes` contiguous bytes from local device memory `src` to `dst` at `dst_off`; then, if
 * flag_slot >= 0 and dst->flags, publish dst->flags[flag_slot] = seq (release, after the data). */
DV_API dv_status dv_flush(dv_ctx* ctx, const void* src, uint64_t bytes, const dv_endpoint* dst,
                   uint64_t dst_off, int32_t flag_slot, uint64_t seq, uint32_t xfer, void* stream);
/* Wait (stream-ordered) until src->flags[flag_slot] >= wait_seq when flag_slot >= 0, then copy
 * `bytes` from `src` at `src_off` to local device memory `dst`. */
DV_API dv_status dv_fetch(dv_ctx* ctx, const dv_endpoint* src, uint64_t src_off, int32_t flag_slot,
                   uint64_t wait_seq, void* dst, uint64_t bytes, uint32_t xfer, void* stream);

/* ---- level 2: scatter / gather (Opt (1) "buffered copies") --- */
/* Pack `region` of `src` into the wire format at dst->base + dst_off, then publish
 * dst->flags[flag_slot] = seq if flag_slot >= 0. DV_XFER_FUSED: one kernel stores straight into
 * the endpoint memory (device, pinned host over PCIe, or peer over NVLink) and publishes the flag
 * itself; DV_XFER_STAGED: kernel packs into library staging, the copy engine moves the chunk. */
DV_API dv_status dv_scatter(dv_ctx* ctx, const dv_cache* src, const dv_region* region,
                     const dv_endpoint* dst, uint64_t dst_off, int32_t flag_slot, uint64_t seq,
                     uint32_t xfer, void* stream);
/* Wait until src->flags[flag_slot] >= wait_seq (if flag_slot >= 0), then unpack the wire chunk
 * at src->base + src_off into `region` of `dst`. Words of `dst` outside the region are untouched. */
DV_API dv_status dv_gather(dv_ctx* ctx, const dv_endpoint* src, uint64_t src_off, int32_t flag_slot,
                    uint64_t wait_seq, const dv_cache* dst, const dv_region* region,
                    uint32_t xfer, void* stream);
/* Batched gather of a LOG of chunks: n_chunks canonical wire chunks stored back to back at
 * src->base + src_off; chunk k is the wire of `first` shifted by k*pos_step positions
 * (pos_step >= first's position count). Typical use: swap-in of a microbatch from its host log,
 * where every token step appended one chunk of one position (swap-out moves only the
 * step's delta; swap-in moves the whole prefix). One copy-engine stream of the whole
 * log (STAGED, the AUTO choice for host sources) or one kernel (FUSED) for all chunks. Waits for
 * src->flags[flag_slot] >= wait_seq first when flag_slot >= 0. */
DV_API dv_status dv_gather_chunks(dv_ctx* ctx, const dv_endpoint* src, uint64_t src_off,
                                  int32_t flag_slot, uint64_t wait_seq, const dv_cache* dst,
                                  const dv_region* first, int32_t n_chunks, int32_t pos_step,
                                  uint32_t xfer, void* stream);
/* Direct layout-to-layout copy of `region` (pack and unpack fused, no wire buffer). Either cache
 * may live in local device memory, pinned host memory (mirror-form arena) or mapped peer memory.
 * If `signal` is non-NULL and flag_slot >= 0, publishes signal->flags[flag_slot] = seq after. */
DV_API dv_status dv_remap(dv_ctx* ctx, const dv_cache* src, const dv_cache* dst, const dv_region* region,
                   const dv_endpoint* signal, int32_t flag_slot, uint64_t seq, uint32_t xfer,
                   void* stream);

/* ---- CUDA-graph forms (capture the per-token path once, replay per token) ----
 * The kernel reads a step k from device memory `d_step` when it runs, shifts the region's
 * positions by k (the token step t writes position p+t-1, reading Q4), the destination by k
 * positions (remap) or k*dst_step_bytes (scatter into a log), and publishes seq + k. Everything
 * is validated for every k in [0, max_step] at enqueue; at run time a k outside that range makes
 * the launch a no-op (nothing moves, nothing is published). Always the FUSED transfer. */
DV_API dv_status dv_scatter_dyn(dv_ctx* ctx, const dv_cache* src, const dv_region* region,
                                const dv_endpoint* dst, uint64_t dst_off, uint64_t dst_step_bytes,
                                int32_t flag_slot, uint64_t seq, const int32_t* d_step,
                                int32_t max_step, void* stream);
DV_API dv_status dv_remap_dyn(dv_ctx* ctx, const dv_cache* src, const dv_cache* dst,
                              const dv_region* region, const dv_endpoint* signal,
                              int32_t flag_slot, uint64_t seq, const int32_t* d_step,
                              int32_t max_step, void* stream);

/* ---- level 1: stream_out / stream_in ------------------------------ */
/* Sender side. `src` is the cache of source block (my_stage, my_micro) of `src_setup`. Routes
 * `region`; for every piece leaving this block, scatters it into inboxes[dst block flat index] at
 * the piece's dst_wire_off and publishes flag slot (this block's flat index) = seq in that inbox.
 * `inboxes` has one entry per destination block (entries never addressed may be zeroed). With
 * tensor parallelism (setups with n_tp > 0) my_tp selects this block's head group. */
DV_API dv_status dv_stream_out(dv_ctx* ctx, const dv_cache* src, const dv_region* region,
                        const dv_setup* src_setup, int32_t my_stage, int32_t my_micro,
                        int32_t my_tp, const dv_setup* dst_setup, const dv_endpoint* inboxes,
                        int32_t n_inboxes, uint64_t seq, uint32_t xfer, void* stream);
/* Receiver side. For every piece entering block (my_stage, my_micro, my_tp) of `dst_setup`: wait
 * for inbox->flags[source block flat index] >= wait_seq, then gather the piece from inbox at its
 * dst_wire_off into `dst`. */
DV_API dv_status dv_stream_in(dv_ctx* ctx, const dv_cache* dst, const dv_region* region,
                       const dv_setup* src_setup, const dv_setup* dst_setup, int32_t my_stage,
                       int32_t my_micro, int32_t my_tp, const dv_endpoint* inbox,
                       uint64_t wait_seq, uint32_t xfer, void* stream);
/* Sender side, direct form: every piece leaving (my_stage, my_micro, my_tp) is remapped straight
 * into dst_caches[dst block flat index] (mapped peer, host or local memory), then flag slot
 * (this block's flat index) of signals[dst block] (if non-NULL) is set to seq. */
DV_API dv_status dv_stream_out_direct(dv_ctx* ctx, const dv_cache* src, const dv_region* region,
                               const dv_setup* src_setup, int32_t my_stage, int32_t my_micro,
                               int32_t my_tp, const dv_setup* dst_setup, const dv_cache* dst_caches,
                               const dv_endpoint* signals, int32_t n_dst, uint64_t seq,
                               uint32_t xfer, void* stream);

/* ---- completion / ordering ---------------------------------------------- */
/* Stream-ordered wait until ep->flags[flag_slot] >= seq (64-bit unsigned compare). */
DV_API dv_status dv_wait(dv_ctx* ctx, const dv_endpoint* ep, int32_t flag_slot, uint64_t seq, void* stream);
/* Stream-ordered publish ep->flags[flag_slot] = seq after all prior work on `stream`. */
DV_API dv_status dv_signal(dv_ctx* ctx, const dv_endpoint* ep, int32_t flag_slot, uint64_t seq, void* stream);
/* Non-blocking poll from the host: *done = (flags[flag_slot] >= seq). Host-memory flags are read
 * directly; device-memory flags with a small synchronous copy. */
DV_API dv_status dv_query(dv_ctx* ctx, const dv_endpoint* ep, int32_t flag_slot, uint64_t seq, int32_t* done);

/* ---- persistent stream engine: the per-layer latency path (DESIGN.md §6 "Persistent engine") -
 * A few CTAs stay resident (a cooperative grid on the engine's own highest-priority stream) and
 * run REGISTERED plans when their doorbell rings, so a per-layer stream-out (PAPER.md:123-135,
 * Opt 2/3) pays no kernel launch, no wait for free SM slots (e.g. behind a GEMM) and no dependency
 * wait between "the producer wrote layer l's K/V" and the copy. A plan is a dv_scatter_dyn /
 * dv_remap_dyn shape: at step k its positions move by k (token step t writes p + t - 1, reading
 * Q4), the destination by k positions (remap) or k*dst_step_bytes (scatter), and it releases
 * flag seq + k at the scope the memory needs (system for host / peer memory). Ringing the doorbell
 * of a plan with step k asks for every step of that plan not yet executed up to k, in order.
 * While an engine runs, cudaDeviceSynchronize() (e.g. torch.cuda.synchronize()) cannot return:
 * park the engine first (dv_engine_park; the next kick relaunches it) or synchronise streams. */
typedef struct dv_engine dv_engine;
/* n_ctas resident CTAs of 256 threads forming ONE thread-block cluster (1 .. 16; 8 saturate PCIe
 * Gen5 x16): cluster rank 0 polls the doorbells, every CTA copies its static share (1,024-vector
 * units rank, rank + n_ctas, ...) of each requested (plan, step), cluster barriers order the
 * shares before rank 0's release of the flag. Jobs run one at a time in the order they are found,
 * so flags are released in order. While it runs, a kernel that is not yet loaded (CUDA lazy
 * loading, e.g. a torch op used for the first time) or a new stream cannot start: create streams
 * and warm every kernel before dv_engine_create / dv_engine_resume, or set CUDA_MODULE_LOADING=EAGER. */
DV_API dv_status dv_engine_create(dv_ctx* ctx, int32_t n_ctas, dv_engine** out);
DV_API dv_status dv_engine_destroy(dv_engine* e);   /* parks, then frees */
/* Stop the resident grid once the jobs already rung are done; blocks until it has exited. */
DV_API dv_status dv_engine_park(dv_engine* e);
/* Relaunch a parked engine (no-op if it runs): needed before producer kernels ring doorbells
 * themselves; dv_engine_kick does it implicitly. */
DV_API dv_status dv_engine_resume(dv_engine* e);
/* Register a plan (validated for every step k in [0, max_step], as dv_scatter_dyn / dv_remap_dyn;
 * K and V must share one copy plan, i.e. no FT6D key transpose) -> *plan. Up to 256 plans. */
DV_API dv_status dv_engine_plan_scatter(dv_engine* e, const dv_cache* src, const dv_region* region,
                                        const dv_endpoint* dst, uint64_t dst_off,
                                        uint64_t dst_step_bytes, int32_t flag_slot, uint64_t seq,
                                        int32_t max_step, int32_t* plan);
DV_API dv_status dv_engine_plan_remap(dv_engine* e, const dv_cache* src, const dv_cache* dst,
                                      const dv_region* region, const dv_endpoint* signal,
                                      int32_t flag_slot, uint64_t seq, int32_t max_step,
                                      int32_t* plan);
/* Ring plan's doorbell with step k after all prior work on `stream` (a stream memory write; the
 * engine is relaunched first if it was parked). */
DV_API dv_status dv_engine_kick(dv_engine* e, int32_t plan, int32_t step, void* stream);
/* The plan's doorbell word in device memory, for a PRODUCER KERNEL to ring itself (lowest
 * latency; include/dv_device.cuh dv_engine_ring): store step + 1 with a gpu-scope release once all
 * of the producer's stores are ordered before it. The engine must be running (not parked). Steps
 * beyond the plan's max_step are never run (the engine stops the plan there). */
DV_API dv_status dv_engine_doorbell(dv_engine* e, int32_t plan, uint64_t** word);
/* Steps of `plan` the engine has completed (flag released), read now (small synchronous copy). */
DV_API dv_status dv_engine_done(dv_engine* e, int32_t plan, uint64_t* steps);

/* ---- device plans: the stream-out fused into the PRODUCER kernel (Opt 2/3) --
 * The per-layer stream-out as a separate kernel waits for the producer (the kernel that writes the
 * layer's new K/V) to finish, then reads the K/V back. A device plan lets the producer itself store
 * each K/V row it computes both into its cache and straight to the destination -- pinned host
 * memory over PCIe, a peer GPU's memory over NVLink (IPC-mapped), or this GPU's HBM -- and release
 * the flag from its own last CTA (include/dv_device.cuh: dv_dplan_row, dv_dplan_release). There is
 * no second kernel, no dependency wait and no re-read. A plan covers a region at step 0; at step k
 * (the producer's argument) the positions move by k (token step t writes p + t - 1, reading Q4)
 * and, for a wire destination, the destination by k * dst_step_bytes; the flag becomes seq + k.
 * Validation (as dv_scatter_dyn / dv_remap_dyn for every k in [0, max_step]) happens here; the
 * plan is a plain struct the caller passes to its kernel by value. The release takes a ticket
 * owned by the plan: one producer launch per plan at a time (stream-ordered launches are fine).
 * Destination caches may be KV5D or FasterTransformer 6-D (the key's 16-byte packets lie S*16
 * bytes apart there: producers store packets through dv_dplan_packet, or whole rows through
 * dv_dplan_row where dv_dplan_row_contiguous holds). */
typedef struct dv_dplan {
  uint8_t* dst[2];          /* K and V destination of (layer o_l, request o_r, head o_h, pos o_s) */
  int64_t st_l, st_r, st_h;  /* destination byte strides per layer / request / head              */
  int64_t st_s[2], st_u[2];  /* K / V: byte stride per position and per 16-byte packet of a row
                                (KV5D: row bytes and 16; FasterTransformer's 6-D key: 16 and S*16) */
  int64_t step_bytes;       /* destination shift per step (wire destinations; 0 for caches) */
  int32_t o_l, o_r, o_h, o_s; /* global ids at the destination origin (step 0)                   */
  int32_t pos_shift;        /* 1: o_s moves with the step (wire); 0: absolute positions (caches) */
  int32_t l0, l1, r0, r1, h0, h1, s0, s1; /* the region at step 0 (global ids, half-open)        */
  int32_t row_bytes;        /* head_dim * elem_bytes                                           */
  int32_t sys_scope;        /* 1: release at system scope (host / peer memory), 0: gpu scope    */
  uint64_t* flag;           /* NULL: no release                                                 */
  uint64_t seq;
  uint32_t* ticket;         /* the plan's own CTA counter (zero between launches)               */
  uint64_t* trace;          /* optional (dvt): %globaltimer right after the release             */
} dv_dplan;
/* Plan rows of `region` of cache `src` (its geometry and head range) into the canonical wire at
 * dst + dst_off (+ k * dst_step_bytes at step k), releasing flag slot `flag_slot` (-1: none). */
DV_API dv_status dv_dplan_scatter(dv_ctx* ctx, const dv_cache* src, const dv_region* region,
                                  const dv_endpoint* dst, uint64_t dst_off, uint64_t dst_step_bytes,
                                  int32_t flag_slot, uint64_t seq, int32_t max_step, dv_dplan* out);
/* Plan rows of `region` into cache `dst` (KV5D or FT6D, e.g. the successor's replica mapped with
 * dv_ipc_open: PAPER.md:286), same positions, releasing signal's flag slot (signal may be NULL). */
DV_API dv_status dv_dplan_remap(dv_ctx* ctx, const dv_cache* src, const dv_cache* dst,
                                const dv_region* region, const dv_endpoint* signal,
                                int32_t flag_slot, uint64_t seq, int32_t max_step, dv_dplan* out);

/* Hand a plan's ticket back to the context (the plan then releases nothing): after the last
 * producer launch using it has completed. Plans never freed keep their tickets until dv_destroy;
 * a context has 65,536 plan / captured-launch tickets (DV_ENOMEM beyond). */
DV_API dv_status dv_dplan_free(dv_ctx* ctx, dv_dplan* plan);

/* Level 1 as device plans (dv_stream_out_direct fused into the producer; §4.2.1 the
 * prompt -> token hand-off, :286 ring replication): route `region` out of block (my_stage,
 * my_micro, my_tp) of src_setup into dst_setup's caches, one remap plan per route piece leaving
 * this block, each releasing signals[destination block] slot = this block's flat index with seq
 * (+ k at step k). The producer stores every packet through dv_dplan_set_packet (the pieces are
 * disjoint: at most one plan takes a packet) and ends with dv_dplan_set_release. At most
 * DV_DPLAN_SET_MAX pieces (DV_ENOTSUP beyond); n == 0 when no piece leaves this block. */
#define DV_DPLAN_SET_MAX 8
/* (dv_dplan_stream_out: the inbox form of the same -- each piece's rows go to inboxes[destination
 * block] at the piece's wire offset, releasing slot = this block's flat index, as dv_stream_out;
 * the receiver runs dv_stream_in. Ring inboxes are refused (DV_EINVAL): a producer cannot wait for
 * a credit.) */
typedef struct dv_dplan_set {
  int32_t n;
  int32_t reserved;
  dv_dplan plan[DV_DPLAN_SET_MAX];
} dv_dplan_set;
DV_API dv_status dv_dplan_stream_out_direct(dv_ctx* ctx, const dv_cache* src, const dv_region* region,
                                            const dv_setup* src_setup, int32_t my_stage, int32_t my_micro,
                                            int32_t my_tp, const dv_setup* dst_setup,
                                            const dv_cache* dst_caches, const dv_endpoint* signals,
                                            int32_t n_dst, uint64_t seq, int32_t max_step, dv_dplan_set* out);
DV_API dv_status dv_dplan_set_free(dv_ctx* ctx, dv_dplan_set* set);   /* dv_dplan_free of every plan */
DV_API dv_status dv_dplan_stream_out(dv_ctx* ctx, const dv_cache* src, const dv_region* region,
                                     const dv_setup* src_setup, int32_t my_stage, int32_t my_micro,
                                     int32_t my_tp, const dv_setup* dst_setup, const dv_endpoint* inboxes,
                                     int32_t n_inboxes, uint64_t seq, dv_dplan_set* out);

/* ---- SM partitions: an SM budget for streaming (NEXT-2; DESIGN.md §6
 * "SM partitions") ----------------------------------------------------------------------------
 * Splits device `device`'s SMs into two green contexts (disjoint SM sets): a STREAMING partition
 * of at least `streaming_sms` SMs (rounded up by the driver to its granularity: 8 on sm_100) and a
 * COMPUTE partition of the rest, and creates one non-blocking stream in each (`priority` for the
 * streaming one, 0 for the compute one; stream priorities as cudaStreamCreateWithPriority). Work
 * launched on *streaming_stream runs only on the streaming SMs and work on *compute_stream only on
 * the others, so a per-layer stream-out never waits for a GEMM's CTAs to retire (measured under a
 * saturating bf16 GEMM loop: DESIGN.md §6). Work on any OTHER stream of the device (e.g. a
 * framework's default stream) is not confined and may still occupy the streaming SMs: run the
 * model's compute on *compute_stream for the isolation to hold. The price is the compute
 * partition's smaller SM count (compute-bound kernels slow down; HBM-bound ones barely).
 * Streams are returned as cudaStream_t values (void*); the caller must not destroy them -- they
 * live until dv_partition_destroy, which must come after all work on them has completed.
 * *sms_streaming / *sms_compute (optional, may be NULL) receive the SM counts actually assigned.
 * Errors: DV_EINVAL (NULL outputs, streaming_sms < 1, or no SMs left for the compute partition),
 * DV_ENOTSUP (the driver has no green contexts), DV_ECUDA (driver failure; nothing is left
 * allocated). */
typedef struct dv_partition dv_partition;
DV_API dv_status dv_partition_create(int32_t device, int32_t streaming_sms, int32_t priority,
                                     dv_partition** out, void** streaming_stream,
                                     void** compute_stream, int32_t* sms_streaming,
                                     int32_t* sms_compute);
DV_API dv_status dv_partition_destroy(dv_partition* p);

#ifdef __cplusplus
}
#endif
#endif /* DV_H_ */
