/*
 * bplb.h -- C ABI of the B200 lower-bound-collection engine
 * (paper_2402_14821_b200/libbplb.so).
 *
 * This is the drop-in boundary for the reference's bound-engine plug-in
 *   BoundEngine = Callable[[ReducedInstance, int], BoundResult]
 *   (/root/reference/pkg/src/binpack/propagator.py:40, called at
 *    propagator.py:274-276 and search.py:352)
 * and for the functions behind it (bounds.py:463-527, parallel.py:122-174).
 * Plain pointers and sizes only; no CUDA or torch types cross the boundary
 * (streams are passed as void*).  INTEGRATION.md shows the ctypes binding a
 * reference maintainer would add.
 *
 * Conventions
 *  - Kinds: 0=MT 1=RAD2 2=FS1 3=CCM1 4=VB2 5=BJ1 (bounds.py:48-67 order).
 *  - Weights are int32 in [1, c]; 1 <= c <= BPLB_MAX_C.  Per-node r may be 0.
 *  - Every call returns 0 on success or a negative BPLB_E* code; the message
 *    of the last failure on the calling thread is bplb_last_error().
 *  - Calls on one engine are serialised by an internal mutex and are
 *    synchronous (they return after results are back in host memory), the
 *    "internally concurrent, externally synchronous" model of SPEC.md:223.
 *  - Caller owns every host array; outputs are caller-allocated.
 */
#ifndef BPLB_H
#define BPLB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define BPLB_API __attribute__((visibility("default")))
#else
#define BPLB_API
#endif

#define BPLB_OK 0
#define BPLB_EINVAL (-1)    /* bad argument (maps to ValueError)              */
#define BPLB_ERANGE (-2)    /* input outside the GPU integer envelope         */
#define BPLB_ECUDA (-3)     /* CUDA runtime / launch failure (RuntimeError)   */
#define BPLB_ENOMEM (-4)    /* device or pinned allocation failed             */
#define BPLB_ENODEV (-5)    /* no CUDA device / unsupported architecture      */

#define BPLB_NKINDS 6
#define BPLB_MAX_C ((int64_t)1 << 30)   /* capacity envelope */
#define BPLB_MAX_R ((int64_t)1 << 24)   /* items per reduced instance         */

/* flags */
#define BPLB_F_PHASED 0x1   /* kinds in order; stop after the first kind whose
                               best exceeds k (Alg. 2 early exit, bounds.py:523-525) */
#define BPLB_F_CANCEL 0x2   /* Alg. 4 guard "if lb <= k" per work unit
                               (parallel.py:76-77): units observing lb > k skip */
#define BPLB_F_TIMING 0x4   /* record device time of the last call (bplb_last_device_ms) */
#define BPLB_F_NOPRUNE 0x10 /* dense sweep: evaluate every lambda of the grid (the paper's
                               Alg. 2-4 work) instead of skipping the lambdas whose integer
                               upper bound cannot change the result (bplb_prune.cuh) */
#define BPLB_F_NOTC   0x20  /* batched calls: the table path on the FP32 pipe, not tcgen05 (parity testing) */
#define BPLB_F_NOTAB  0x8   /* batched calls: do not use the histogram x table kernel
                               (selects the warp-per-node kernel; parity testing) */

typedef struct bplb_engine bplb_engine;

/* Result of one feasibility check (BoundResult, bounds.py:101-108). */
typedef struct {
    int64_t best[BPLB_NKINDS];      /* per-kind best bound, indexed by kind id        */
    int64_t arg_lambda[BPLB_NKINDS];/* lowest lambda attaining best                   */
    int64_t n_lambda[BPLB_NKINDS];  /* |Lambda_k| (VB2 capped per instance)            */
    int64_t evals[BPLB_NKINDS];     /* lambda points actually evaluated per kind       */
    int32_t evaluated[BPLB_NKINDS]; /* 1 if any lambda of the kind was evaluated       */
    int32_t n_done;                 /* PHASED: number of kinds (in order) processed    */
    int32_t exceeded;               /* lb > k                                          */
    int64_t lb;                     /* max over evaluated kinds                        */
    int64_t evals_total;            /* sum of evals                                    */
} bplb_result;

/* Engine lifetime.  One engine owns a CUDA stream, grow-only device buffers
 * and pinned staging buffers on `device`. */
BPLB_API int bplb_engine_create(int device, bplb_engine **out);
BPLB_API int bplb_engine_destroy(bplb_engine *eng);

/* One feasibility check of one reduced instance (w[0..r)).
 * kinds[0..nkinds) gives the evaluation order (PHASED) / the subset.
 * Replaces: lower_bound_seq (bounds.py:504-527) when flags = PHASED,
 *           lower_bound_par (parallel.py:122-137) when flags = CANCEL or 0,
 *           ParallelBoundEngine.__call__ (parallel.py:160-163). */
BPLB_API int bplb_check(bplb_engine *eng, const int32_t *w, int64_t r, int64_t c, int64_t k,
               const int32_t *kinds, int32_t nkinds, int32_t flags, bplb_result *out);

/* Per-lambda bounds of one kind over [lo, hi] (inclusive), out[hi-lo+1].
 * Replaces: dff_bound_batch (bounds.py:463-501) and, with lo == hi,
 *           dff_bound (bounds.py:276-290).
 * [lo, hi] must lie inside the kind's (uncapped) parameter domain. */
BPLB_API int bplb_dff_bound_batch(bplb_engine *eng, int32_t kind, const int32_t *w, int64_t r,
                         int64_t c, int64_t lo, int64_t hi, int64_t *out);

/* Batched feasibility check over n_nodes reduced instances in CSR layout
 * (w_concat[offsets[i] .. offsets[i+1])), all with capacity c and budget k.
 * Outputs (host, caller-allocated; best/arg may be NULL):
 *   lb_out[n], exceeded_out[n], best_out[n*6], arg_out[n*6] (by kind id;
 *   kinds not evaluated report 0).  No reference counterpart: the reference
 *   evaluates one node per engine call (propagator.py:274-276). */
BPLB_API int bplb_check_batch(bplb_engine *eng, const int32_t *w_concat, const int64_t *offsets,
                     int64_t n_nodes, int64_t c, int64_t k, const int32_t *kinds,
                     int32_t nkinds, int32_t flags, int64_t *lb_out, uint8_t *exceeded_out,
                     int64_t *best_out, int64_t *arg_out);

/* bplb_check_batch with a compact weight dtype: wbytes = 4 (int32),
 * 2 (uint16, c <= 65535) or 1 (uint8, c <= 255).  Halves / quarters the
 * host->device bytes of a batch; values are validated on the device. */
BPLB_API int bplb_check_batch_ex(bplb_engine *eng, const void *w_concat, int32_t wbytes,
                        const int64_t *offsets, int64_t n_nodes, int64_t c, int64_t k,
                        const int32_t *kinds, int32_t nkinds, int32_t flags, int64_t *lb_out,
                        uint8_t *exceeded_out, int64_t *best_out, int64_t *arg_out);

/* Same as bplb_check_batch with every array already resident in device
 * memory (`stream` is a cudaStream_t, or NULL for the engine's stream; pass
 * cudaStreamLegacy, i.e. (void*)1, for the legacy default stream).
 * Asynchronous: returns after enqueueing; the caller synchronises.
 * d_best/d_arg may be NULL.  Work buffers are owned by the engine, so
 * concurrent device calls on one engine must be ordered on one stream. */
BPLB_API int bplb_check_batch_device(bplb_engine *eng, const int32_t *d_w_concat,
                            const int64_t *d_offsets, int64_t n_nodes, int64_t max_r,
                            int64_t c, int64_t k, const int32_t *kinds, int32_t nkinds,
                            int32_t flags, int64_t *d_lb, uint8_t *d_exceeded,
                            int64_t *d_best, int64_t *d_arg, void *stream);

/* Device-resident variant with a compact weight dtype (see _ex above). */
BPLB_API int bplb_check_batch_device_ex(bplb_engine *eng, const void *d_w_concat, int32_t wbytes,
                               const int64_t *d_offsets, int64_t n_nodes, int64_t max_r,
                               int64_t c, int64_t k, const int32_t *kinds, int32_t nkinds,
                               int32_t flags, int64_t *d_lb, uint8_t *d_exceeded,
                               int64_t *d_best, int64_t *d_arg, void *stream);

/* Device-side reduction of search-node states + batched check.
 * Node states are bin assignments: assign[node * n_items + i] is the bin
 * (0 <= b < n_bins) item i is committed to, or the all-ones value of the
 * element type (0xFF for abytes = 1, 0xFFFF for abytes = 2) while item i is
 * still open.  Each node is reduced on the GPU exactly as reduce_packing
 * (instances.py:262-282): open items' weights in item order, then the
 * positive committed bin loads in bin order; a load above c fails with
 * BPLB_EINVAL ("committed load exceeds capacity", ValueError in Python), as
 * does a bin id >= n_bins.  inst_w[n_items] are the instance weights.
 * Replaces, for a batch of nodes: reduce_packing + engine(red, k) in the
 * feasibility check (propagator.py:266-276).  Outputs as bplb_check_batch. */
BPLB_API int bplb_check_batch_assign(bplb_engine *eng, const int32_t *inst_w, int64_t n_items,
                            int64_t n_bins, const void *assign, int32_t abytes, int64_t n_nodes,
                            int64_t c, int64_t k, const int32_t *kinds, int32_t nkinds,
                            int32_t flags, int64_t *lb_out, uint8_t *exceeded_out,
                            int64_t *best_out, int64_t *arg_out);

/* The reduction alone (parity surface): writes the reduced CSR to host
 * arrays offsets_out[n_nodes + 1] and weights_out[total] (int32, capacity
 * n_nodes * n_items).  Same errors as bplb_check_batch_assign. */
BPLB_API int bplb_reduce_batch(bplb_engine *eng, const int32_t *inst_w, int64_t n_items,
                      int64_t n_bins, const void *assign, int32_t abytes, int64_t n_nodes,
                      int64_t c, int64_t *offsets_out, int32_t *weights_out);

/* Multi-GPU batched checks in one call.
 * bplb_multi_create makes one engine per entry of devices[ndev] (an id may
 * repeat: several engines on one GPU).  bplb_check_batch_multi shards the
 * nodes of a host CSR batch into contiguous ranges balanced by item count,
 * checks each range on its own engine / device from its own host thread
 * (upload, kernel and verdicts per shard, concurrently), and writes every
 * shard's outputs into the caller's arrays at the shard's node offset (the
 * gather).  Arguments, outputs and errors as bplb_check_batch_ex; the first
 * failing shard's error is returned.  bplb_multi_last_bounds writes the last
 * call's node boundaries (ndev + 1 values); bplb_multi_engine exposes an
 * engine (measurement hooks).  No reference counterpart: the reference runs
 * one node per call on one host (propagator.py:274-276, parallel.py:84-119). */
typedef struct bplb_multi bplb_multi;
BPLB_API int bplb_multi_create(const int32_t *devices, int32_t ndev, bplb_multi **out);
BPLB_API int bplb_multi_destroy(bplb_multi *m);
BPLB_API int bplb_multi_engine(bplb_multi *m, int32_t i, bplb_engine **out);
BPLB_API int bplb_multi_last_bounds(bplb_multi *m, int64_t *bounds_out);
BPLB_API int bplb_check_batch_multi(bplb_multi *m, const void *w_concat, int32_t wbytes,
                           const int64_t *offsets, int64_t n_nodes, int64_t c, int64_t k,
                           const int32_t *kinds, int32_t nkinds, int32_t flags, int64_t *lb_out,
                           uint8_t *exceeded_out, int64_t *best_out, int64_t *arg_out);

/* One reduced instance over every engine of m (the
 * cfg4-size single check sharded over GPUs): each kind's lambda range is cut
 * into contiguous slices, one per engine, each slice checked with bound
 * pruning on its own device from its own host thread, and the per-kind
 * (best, lowest arg lambda) merged as an allreduce(MAX) of packed keys would.
 * flags: 0 / NOPRUNE (full collection), PHASED (replayed on the merged
 * per-kind results: n_done, per-kind fields of unreached kinds zeroed), CANCEL
 * (runs the full collection).  Result as bplb_check's.  Replaces the
 * reference's lambda-chunk dispatch of one check over worker processes
 * (parallel.py:84-119) with one call over devices. */
BPLB_API int bplb_check_multi(bplb_multi *m, const int32_t *w, int64_t r, int64_t c, int64_t k,
                     const int32_t *kinds, int32_t nkinds, int32_t flags, bplb_result *out);

/* bplb_check restricted to per-kind lambda ranges [rng_lo[kd], rng_hi[kd]]
 * (empty when hi < lo; inside the kind's domain): one slice of a
 * lambda-split check (the per-rank primitive of the torch.distributed form).
 * Full collection only (PHASED / CANCEL -> BPLB_EINVAL); per-kind best / arg /
 * evals refer to the slice. */
BPLB_API int bplb_check_ranges(bplb_engine *eng, const int32_t *w, int64_t r, int64_t c, int64_t k,
                      const int32_t *kinds, int32_t nkinds, int32_t flags, const int64_t *rng_lo,
                      const int64_t *rng_hi, bplb_result *out);

/* Batched exact knapsack reasoning per bin, the bitset
 * subset-sum DP of propagator.py:98-224 for n_bins independent bins in one
 * launch.  Bin b: committed load committed[b] (>= 0), load interval
 * [lo[b], hi[b]] (0 <= lo <= hi <= c), open candidate items with weights
 * w_concat[offsets[b] .. offsets[b+1]) in [1, c], in the reference's
 * open_items_of_bin order.  Outputs:
 *   status_out[b]  0 ok; 1 Wipeout "no reachable load in its interval"
 *                  (_knapsack_bin :203-204 / knapsack_load_tightening :139-140)
 *   lo_out/hi_out  lowest / highest reachable load inside [lo, hi] (the
 *                  tightened interval, set_lo / set_hi :205-206); the input
 *                  interval when status is 1
 *   action_out[t]  per open item: 0 keep, 1 remove bin b from the item (no
 *                  load in the interval uses it), 2 commit it to b (none avoids
 *                  it), 3 Wipeout "unpackable with or without item" -- on the
 *                  tightened interval, all 0 when the tightened lo <= committed
 *                  (_knapsack_bin :208-227).  The reference stops at the first
 *                  3 in item order; the caller applies actions in that order.
 *   reach_out      optional (NULL to skip): n_bins * ((c + 32) / 32) u32 words,
 *                  bit v of bin b = load v reachable (reachable_sums :105-110)
 * BPLB_KN_REACH_ONLY: reach + tightening only (action_out may be NULL).
 * BPLB_KN_NO_TIGHTEN: filter on the INPUT interval with no committed-load
 *   skip (knapsack_item_filter :153-168 semantics).
 * Capacity <= 1023: one warp per bin (register bitsets); larger c: one CTA
 * per bin with shared-memory bitsets, BPLB_ERANGE when
 * (depth(max items) + 2) * words * 4 bytes exceed shared memory. */
#define BPLB_KN_REACH_ONLY 0x100
#define BPLB_KN_NO_TIGHTEN 0x200
BPLB_API int bplb_knapsack_bins(bplb_engine *eng, int64_t c, int64_t n_bins, const int32_t *committed,
                       const int32_t *lo, const int32_t *hi, const int32_t *w_concat,
                       const int64_t *offsets, int32_t flags, int32_t *status_out, int32_t *lo_out,
                       int32_t *hi_out, uint8_t *action_out, uint32_t *reach_out);
/* Device-resident form (device pointers; max_items bounds every bin's item
 * count; stream NULL = the engine's stream).  Returns after the launch
 * completed (error word checked). */
BPLB_API int bplb_knapsack_bins_device(bplb_engine *eng, int64_t c, int64_t n_bins,
                       const int32_t *d_committed, const int32_t *d_lo, const int32_t *d_hi,
                       const int32_t *d_w_concat, const int64_t *d_offsets, int64_t max_items,
                       int32_t flags, int32_t *d_status, int32_t *d_lo_out, int32_t *d_hi_out,
                       uint8_t *d_action, uint32_t *d_reach, void *stream);

/* Number of kernel launches issued by the engine since creation (for the
 * bench's gpu_launches claim), and device time of the last TIMING call. */
BPLB_API int64_t bplb_launch_count(bplb_engine *eng);
BPLB_API double bplb_last_device_ms(bplb_engine *eng);

/* Measurement hook: with on != 0 the engine brackets every launch of its
 * dominant batched kernel (the histogram x table contraction) with CUDA
 * events on the launching stream; bplb_last_kernel_ms waits for the last
 * one and returns its duration (0 if none was recorded). */
BPLB_API int bplb_profile_kernel(bplb_engine *eng, int on);
BPLB_API double bplb_last_kernel_ms(bplb_engine *eng);

/* Which kernel family served the engine's last check / batch launch (test
 * and measurement hook); *detail (optional) = table path: warps per
 * contraction CTA; prune path: 1 in lb mode, 0 in per-kind key mode;
 * node kernels: grid of a multi-CTA single check. */
#define BPLB_PATH_NONE 0
#define BPLB_PATH_TAB 1          /* histogram x table contraction (c <= 288 batches)   */
#define BPLB_PATH_TAB_SINGLE 2   /* table path, one check (cluster / counter kernel)   */
#define BPLB_PATH_WARP 3         /* warp-per-node kernel (dense sweep)                 */
#define BPLB_PATH_NODE_TABLE 4   /* CTA-per-node kernel, cumulative tables             */
#define BPLB_PATH_NODE_SORT 5    /* CTA-per-node kernel, sorted weights                */
#define BPLB_PATH_WIDE 6         /* grid-wide kernels (one large instance)             */
#define BPLB_PATH_PRUNE 7        /* CTA-per-node bound-pruned sweep (bplb_prune.cuh)   */
#define BPLB_PATH_KNAP 9         /* knapsack bins (bplb_knap.cuh); detail = threads per bin */
#define BPLB_PATH_TC 8           /* histogram x table contraction on tcgen05 (bplb_tc.cuh) */
BPLB_API int bplb_last_path(bplb_engine *eng, int32_t *detail);

/* Thread-local message describing the last error on this thread. */
BPLB_API const char *bplb_last_error(void);

/* Library / device description ("bplb <ver> sm_100a ..."). */
BPLB_API const char *bplb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BPLB_H */
