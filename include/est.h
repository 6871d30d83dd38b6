/*
 * est.h — C ABI of libest.so, the B200 execution backend for the elastencil
 * stencil abstraction (arXiv 2512.19851).
 *
 * Every entry point is plain C (pointers, sizes, integers), returns 0 on
 * success or a stable error code — the reference's wire error space
 * (pkg/src/elastencil/errors.py:10-164; 1 = generic CUDA/NVRTC failure,
 * 14 InvalidShape, 15 UnsupportedOp, 16 MalformedDag, ...) — and leaves a
 * human-readable message for est_last_error() (thread local).
 *
 * Each group notes the reference interface it replaces. The reference is pure
 * Python/numpy; these calls sit under the worker seam, bound
 * through ctypes by paper_2512_19851_b200/_lib.py exactly as INTEGRATION.md shows
 * for a maintainer wiring it into pkg/src/elastencil/worker.py.
 */
#ifndef EST_H
#define EST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EST_ABI_VERSION 7

typedef struct est_ctx est_ctx;       /* one device + compute/copy streams      */
typedef struct est_module est_module; /* an NVRTC-compiled, loaded cubin        */
typedef struct est_event est_event;   /* CUDA event (optionally IPC-shareable)  */

/* ---- errors / versioning ------------------------------------------------ */
const char *est_last_error(void);
int est_abi_version(void);
int est_device_count(int *count);

/* ---- context: replaces the per-worker numpy state of executor.py:179-191 --
 * (Executor owns a ScratchPool and runs numpy inline); here: one context per
 * worker process, bound to its GPU, with stream 0 = compute lane and
 * stream 1 = copy lane (the paper's two-stream scheme). */
int est_ctx_create(int device, est_ctx **out);
int est_ctx_destroy(est_ctx *ctx);
int est_ctx_sync(est_ctx *ctx);                    /* both streams */
int est_stream_sync(est_ctx *ctx, int stream);
int est_device_info(est_ctx *ctx, int *sm_count, uint64_t *total_mem, uint64_t *free_mem,
                    int *cc_major, int *cc_minor);

/* ---- device memory: replaces np.zeros tile buffers (grid.py:146, 179-181) */
int est_alloc(est_ctx *ctx, uint64_t bytes, uint64_t *dptr);       /* zero-filled */
int est_free(est_ctx *ctx, uint64_t dptr);
int est_memset_zero(est_ctx *ctx, uint64_t dptr, uint64_t bytes, int stream);
int est_host_alloc(uint64_t bytes, uint64_t *hptr);                /* pinned      */
int est_host_free(uint64_t hptr);

/* 3-D pitched box copy (any direction; host side must be pinned or pageable).
 * Replaces interior_view copies / gather_slice_pieces (grid.py:186-230),
 * ensure_ghost_capacity's interior copy (grid.py:178-182), checkpoint_blob /
 * adopt_blob payload copies (grid.py:239-277) and tile migration
 * (worker.py:341-388). Pitches are in ELEMENTS; extents in elements. */
typedef struct est_box {
    uint64_t src, dst;                   /* addresses of the box origin        */
    int64_t src_py, src_pz, dst_py, dst_pz;
    int64_t nx, ny, nz;
} est_box;
int est_copy_box(est_ctx *ctx, const est_box *box, int elem_size, int stream);

/* Many small boxes in ONE kernel launch (device<->device, incl. IPC-mapped peer
 * memory). Replaces ExchangeManager.pack/_unpack + co-located strip copies
 * (exchange.py:147-165, 192-197). */
int est_copy_boxes(est_ctx *ctx, const est_box *boxes, int n, int elem_size, int stream);

/* Position-keyed content hash of one box (src side of `box`; dst unused):
 * sum over its elements of mix64(bits + 0x9e3779b97f4a7c15 * (g + 1)) mod 2^64,
 * g = the element's global C-order index in an array of dims `gdims`, the box
 * starting at global `origin` (z, y, x). Partial hashes of any decomposition
 * sum to the whole array's hash. Synchronous on the compute stream. Extension
 * (no reference counterpart): whole-array bit-equality checks across rescales
 * (the reference compares fetched arrays, pkg/tests/test_acceptance.py:266-315). */
int est_hash_box(est_ctx *ctx, const est_box *box, const int64_t origin[3], const int64_t gdims[3],
                 int elem_size, uint64_t *out);

/* ---- kernels: replaces evaluate_statement (executor.py:86-176) ------------
 * src is a generated sm_100a stencil skeleton instance (paper_2512_19851_b200/
 * codegen.py); it is compiled by NVRTC with FMA contraction off and IEEE div /
 * sqrt (bit-exact with numpy), cached on disk by content hash (cache_dir may be
 * NULL), and loaded into the context. */
int est_module_compile(est_ctx *ctx, const char *src, const char *const *opts, int n_opts,
                       const char *cache_dir, est_module **out, int *from_cache);
/* Compile into cache_dir without loading (offline prebuild, no GPU needed). */
int est_module_precompile(const char *src, const char *const *opts, int n_opts,
                          const char *cache_dir, int *was_cached);
int est_module_load_cubin(est_ctx *ctx, const void *image, est_module **out);
int est_module_kernel(est_module *mod, const char *name, uint64_t *fn);
int est_module_destroy(est_module *mod);
int est_kernel_set_smem(uint64_t fn, int bytes);
/* est_launch with flags: EST_LAUNCH_PDL = programmatic dependent launch (the
 * kernel may be scheduled while the previous kernel on the stream drains; it
 * must execute griddepcontrol.wait before touching memory that kernel wrote
 * or reads - every generated skeleton does; replaces the per-node launch gap
 * of executor.py:320-324's statement-at-a-time loop) */
#define EST_LAUNCH_PDL 1
/* EST_LAUNCH_COOPERATIVE: the driver guarantees every CTA of the grid is
 * co-resident (or the launch fails with an error instead of the grid-barrier
 * kernels spinning into their bounded trap); the kernel must take ONE
 * parameter (the params block). */
#define EST_LAUNCH_COOPERATIVE 2
int est_launch_ex(est_ctx *ctx, uint64_t fn, const uint32_t grid[3], const uint32_t block[3],
                  uint32_t smem, const void *params, uint32_t params_size, int stream, int flags);
/* resident CTAs per SM for a launch shape (persistent grids with grid-wide
 * barriers size themselves with it: every CTA must be co-resident) */
int est_kernel_occupancy(uint64_t fn, int block, int smem, int *blocks_per_sm);
/* Launch fn with ONE by-value parameter struct of params_size bytes. */
int est_launch(est_ctx *ctx, uint64_t fn, const uint32_t grid[3], const uint32_t block[3],
               uint32_t smem, const void *params, uint32_t params_size, int stream);
/* CUDA graphs: capture every launch of a batch once on a stream, replay it as
 * one graph launch (host batch path). */
typedef struct est_graph est_graph;
int est_graph_begin(est_ctx *ctx, int stream);
int est_graph_end(est_ctx *ctx, int stream, est_graph **out);
int est_graph_launch(est_ctx *ctx, est_graph *graph, int stream);
int est_graph_destroy(est_graph *graph);
/* TMA descriptor (CUtensorMap, 128 bytes written to out128) for a rank-3
 * padded tile buffer: dims/strides innermost first; l2_promotion 0 none,
 * 1 64B, 2 128B, 3 256B. Used by the streaming skeleton's
 * cp.async.bulk.tensor plane loads. */
int est_tmap_encode_3d(uint64_t base, int elem, const uint64_t dims[3],
                       const uint64_t strides_bytes[2], const uint32_t box[3], int l2_promotion,
                       void *out128);
/* Compile to a cubin image without loading (offline prebuild in build()). */
int est_nvrtc_compile(const char *src, const char *const *opts, int n_opts, const char *arch,
                      void **image, uint64_t *size);
void est_buffer_free(void *p);

/* ---- events / timing / cross-process ordering -------------------------------
 * Replaces the BatchStats wall clocks (executor.py:52-62) with device time,
 * and the PeerHub/TCP round signalling (worker.py:61-139) with IPC events. */
int est_event_create(est_ctx *ctx, int interprocess, est_event **out);
int est_event_destroy(est_event *ev);
int est_event_record(est_ctx *ctx, est_event *ev, int stream);
int est_event_wait(est_ctx *ctx, est_event *ev, int stream);  /* stream waits on ev */
int est_event_sync(est_event *ev);
int est_event_query(est_event *ev);                            /* 0 done, 600 pending */
int est_event_elapsed_ms(est_event *start, est_event *end, float *ms);
int est_stream_join(est_ctx *ctx, int waiter, int signaller);  /* intra-ctx ordering */

/* ---- device-side round flags (replace the per-round READY / PULLED signalling
 * of exchange.py:169-234 / worker.py:61-139 between worker processes) -------
 * est_flag_write: after all prior work on `stream`, store `value` to the 32-bit
 *   word at device address `addr` (implicit system-scope release barrier).
 * est_flag_wait: `stream` waits (front-end semaphore acquire, no SM spin) until
 *   the word at `addr` - possibly a peer's, IPC-mapped - satisfies
 *   (int32_t)(*addr - value) >= 0. */
int est_flag_write(est_ctx *ctx, uint64_t addr, uint32_t value, int stream);
int est_flag_wait(est_ctx *ctx, uint64_t addr, uint32_t value, int stream);

/* ---- CUDA IPC: replaces the TCP peer transport and the memory daemon's
 * host-side blob store (worker.py:211-224, daemon.py:29-143) --------------- */
int est_ipc_mem_handle(uint64_t dptr, uint8_t handle[64]);
int est_ipc_mem_open(est_ctx *ctx, const uint8_t handle[64], uint64_t *dptr);
int est_ipc_mem_close(uint64_t dptr);
int est_ipc_event_handle(est_event *ev, uint8_t handle[64]);
int est_ipc_event_open(const uint8_t handle[64], est_event **out);

#ifdef __cplusplus
}
#endif
#endif /* EST_H */
