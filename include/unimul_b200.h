/*
 * unimul_b200.h — C-ABI of the B200-native one-sided distributed GEMM.
 *
 * This is the drop-in boundary for the reference's hot path (arXiv 2510.08874,
 * package `unimul`, mounted at /root/reference/pkg).  Every entry point below
 * replaces one reference interface; the citation names the file:line it
 * stands in for.  Plain pointers and sizes only: no torch, no CUDA types
 * (streams are passed as `void*` = cudaStream_t).
 *
 * Status convention: every function returns UM_OK (0) or an error code; the
 * message is available from um_last_error() (thread-local).  The Python shim
 * maps codes to the reference exception classes (errors.py:4-13).
 */
#ifndef UNIMUL_B200_H
#define UNIMUL_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define UM_API __attribute__((visibility("default")))
#else
#define UM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py:4-13 + builtin exceptions the reference raises) */
#define UM_OK          0
#define UM_ECONFIG     1  /* ConfigError(ValueError)        errors.py:4   */
#define UM_EOWNERSHIP  2  /* OwnershipError(RuntimeError)   errors.py:8   */
#define UM_ECONTRACT   3  /* ContractError(ValueError)      errors.py:12  */
#define UM_EINDEX      4  /* IndexError  (tiling.py:170,217, fabric.py:166) */
#define UM_EVALUE      5  /* ValueError  (tiling.py:24,38, opgen.py:64)   */
#define UM_ECUDA       6  /* RuntimeError: CUDA / driver failure           */
#define UM_ECAPACITY   7  /* caller buffer too small; *n_out holds the need */

/* ---- element types --------------------------------------------------------- */
#define UM_BF16 0
#define UM_F32  1

/* Mapping (tiling.py:97-99) */
#define UM_BLOCK        0
#define UM_BLOCK_CYCLIC 1

/* Stationarity (opgen.py:21-24) */
#define UM_STATIONARY_A 0
#define UM_STATIONARY_B 1
#define UM_STATIONARY_C 2

/*
 * Matrix descriptor: global shape + PartitionSpec + replication factor.
 * Replaces DistributedMatrix's placement state (distmatrix.py:65-114) and
 * PartitionSpec (tiling.py:102-122).
 */
typedef struct {
  int64_t rows, cols;            /* global shape                         */
  int64_t tile_rows, tile_cols;  /* PartitionSpec.tile_shape             */
  int64_t grid_pr, grid_pc;      /* PartitionSpec.proc_grid (per replica) */
  int32_t mapping;               /* UM_BLOCK | UM_BLOCK_CYCLIC           */
  int32_t c;                     /* replication factor                   */
} um_mat_desc;

/*
 * A 2D strided view of one tile slice: the tile base pointer plus the slice
 * [row_lo,row_hi) x [col_lo,col_hi) in tile-local coordinates.  This is the
 * form the TMA tensor maps consume directly (base = tile base, dims =
 * (col_hi,row_hi), start = (col_lo,row_lo)), so unaligned slices need no copy.
 * Replaces the numpy slice views of runtime.py:143-150 / kernels.py:13-17.
 */
typedef struct {
  void*   base;                  /* tile base (local, peer-mapped or IPC-mapped) */
  int64_t row_lo, row_hi;
  int64_t col_lo, col_hi;
  int64_t pitch;                 /* row pitch in elements; pitch*esize % 16 == 0 */
  int32_t dtype;                 /* UM_BF16 | UM_F32                      */
  int32_t device;                /* CUDA device that physically holds base */
} um_view;

/* ======================================================================== */
/* Planner (opgen.py:106-200, tiling.py:125-221)                             */
/* ======================================================================== */

/* Number of int64 fields per emitted op row. */
#define UM_OP_FIELDS 24
/* Field order of an op row:
 *   0  a_i   1  a_j   2  b_i   3  b_j   4  c_i   5  c_j
 *   6  m_lo  7  m_hi  8  k_lo  9  k_hi 10  n_lo 11  n_hi
 *  12..15  a_local rows.lo, rows.hi, cols.lo, cols.hi
 *  16..19  b_local rows.lo, rows.hi, cols.lo, cols.hi
 *  20..23  c_local rows.lo, rows.hi, cols.lo, cols.hi
 * i.e. exactly the fields of opgen.LocalMatMulOp (opgen.py:27-54), in the
 * order opgen.generate emits them (owned stationary tiles row-major, then the
 * overlap loops, zero-area ops skipped: opgen.py:117-131,145-159,169-183).
 */

/* opgen.generate(stationarity, A, B, C, caller)  (opgen.py:193-200).
 * Writes at most `cap` rows to ops_out; *n_out = number of ops.  Returns
 * UM_ECAPACITY (with *n_out set) when cap is too small.                    */
UM_API int um_plan(const um_mat_desc* A, const um_mat_desc* B, const um_mat_desc* C,
            int32_t nprocs, int32_t stationarity, int32_t caller,
            int64_t* ops_out, int64_t cap, int64_t* n_out);

/* iteration_offset(stationary_tile, nops)  (runtime.py:89-93).  */
UM_API int um_iteration_offset(int64_t ti, int64_t tj, int64_t nops, int64_t* out);

/* tiling.owner_of + DistributedMatrix.owner_rank (tiling.py:206-221,
 * distmatrix.py:109-114): global rank owning tile (i,j) of `replica`.      */
UM_API int um_owner_rank(const um_mat_desc* M, int32_t nprocs, int64_t i, int64_t j,
                  int32_t replica, int32_t* rank_out);

/* tiling.most_square_grid(p)  (tiling.py:125-135).                        */
UM_API int um_most_square_grid(int64_t p, int64_t* gr, int64_t* gc);

/* ======================================================================== */
/* K1: local tile GEMM on sm_100a (kernels.py:13-28, _gemmcore.pyx:10-25,     */
/*     runtime.local_gemm runtime.py:96-107)                                 */
/* ======================================================================== */

/* One component multiply C[c] += A[a] @ B[b] (bf16 in, fp32 accumulate).
 * c_remote = 0: epilogue TMA reduce-add into c (c on the launching device).
 * c_remote = 1: epilogue red.global.add straight into c (peer or IPC
 *               pointer) — the fused remote accumulate of fabric.py:203-234.
 * wait_flag != NULL: the op's operands are being delivered by a get (K2)
 *               that signals *wait_flag = wait_value on arrival (um_signal);
 *               the kernel's producer waits for it before loading this op's
 *               tiles, so gets overlap the GEMMs of earlier ops inside ONE
 *               launch — the ordering rule "a compute depends on its input
 *               fetches" (runtime.py:233-236 PendingTileCopy.wait). */
typedef struct {
  um_view a, b, c;
  int32_t c_remote;
  uint32_t wait_value;
  const uint32_t* wait_flag;
  int32_t a_get, b_get;    /* um_gemm_acc_fused: 1-based index of the get whose band holds
                              this op's a / b operand, waited for chunk by chunk (a: the
                              rows of each tile, all k; b: the rows of each k-block) —
                              the view must lie inside the band's columns and be
                              TMA-aligned; 0 = resident or covered by get_mask          */
  uint64_t get_mask;       /* bit i: the op starts loading only after gets[i] has landed  */
  uint32_t* done_flag;     /* non-NULL: when every op of the launch sharing this flag has
                              written all of its C tiles, the kernel adds the number of
                              those ops to *done_flag (release, system scope; may be a
                              peer / IPC-mapped word), so a consumer expecting n ops
                              waits for *done_flag >= n whatever the launch split  */
  int32_t done_piece;      /* nonzero: this entry is a piece of an op that another entry
                              sharing done_flag counts (not added); give the count to the
                              piece issued last, so launches in stream order cover all  */
  int32_t reserved;        /* zero */
} um_gemm_op;

/* A pull executed INSIDE the GEMM launch (um_gemm_acc_fused): src slice
 * (local, peer or IPC-mapped) -> dst slice (a staging buffer on the launching
 * device), same dtype and shape.  Replaces get_tile_async + PendingTileCopy
 * (distmatrix.py:42-59,161-168 -> fabric.py:177-201) on the hot path.      */
typedef struct {
  um_view src, dst;
} um_get_desc;

/* Max pulls per fused launch. */
#define UM_GEMM_MAX_GETS 64
/* Max distinct done_flags per launch. */
#define UM_GEMM_MAX_SIGNALS 64

/* Ops per grouped launch that travel inside the kernel parameters; longer
 * lists are staged through a stream-ordered device allocation.            */
#define UM_GEMM_MAX_INLINE_OPS 40

/* c += a @ b for a single op on `stream` (device = c.device unless remote). */
UM_API int um_gemm_acc(const um_view* a, const um_view* b, const um_view* c, void* stream);

/* Grouped persistent launch over a list of ops on one device.  All ops'
 * operands must be readable from `device`.  Equivalent to calling
 * um_gemm_acc for each op in order (accumulates commute).  Ops whose C views
 * are identical (same base, slice, pitch and epilogue) form a k-chain: their
 * products are accumulated in TMEM in list order and each output tile is
 * reduced into C once (UM_GEMM_CHAIN=0 turns this off).                    */
UM_API int um_gemm_acc_batch(const um_gemm_op* ops, int32_t nops, int32_t device, void* stream);

/* Fused get -> GEMM: ONE persistent launch that pulls `gets` with dedicated
 * get warps on every SM (chunks handed out in the order the launch first needs each get) while the tensor
 * cores run the ops; an op whose get_mask names pulls starts loading
 * only after every chunk of that pull has landed (device-side acquire), so
 * the reference's ordering rule "a compute depends on completion of its input
 * fetches" (runtime.py:219-236) holds without host round trips.
 * Deadlock-free: the get warps depend on nothing but their own loads.      */
UM_API int um_gemm_acc_fused(const um_gemm_op* ops, int32_t nops, const um_get_desc* gets, int32_t ngets,
                             int32_t device, void* stream);

/* Prepared launches: resolve an op/get list once (tensor maps encoded, work
 * list in the parameter block, persistent device buffers) and replay it with
 * one call per step.  The views' memory must stay allocated and in place
 * until um_gemm_destroy (which waits for the device if it owns buffers).
 * Replay semantics equal um_gemm_acc_fused on the same lists.              */
UM_API int um_gemm_prepare(const um_gemm_op* ops, int32_t nops, const um_get_desc* gets, int32_t ngets,
                           int32_t device, void** handle);
UM_API int um_gemm_launch(void* handle, void* stream);
UM_API int um_gemm_destroy(void* handle);

/* Cap the persistent grid of K1 launches on `device` to `max_clusters` CTA
 * pairs (0 = no cap): ranks sharing one GPU then run their launches side by
 * side instead of one after the other.  Read at launch time.               */
UM_API int um_gemm_set_grid_limit(int32_t device, int32_t max_clusters);

/* Tile/stage knobs of the GEMM (bench/profiling): returns 0 and fills.    */
UM_API int um_gemm_config(int32_t* bm, int32_t* bn, int32_t* bk, int32_t* stages, int32_t* cta_group);

/* ======================================================================== */
/* K2: one-sided get engine (fabric.py:156-201, distmatrix.py:151-168)        */
/* ======================================================================== */

/* dst <- src slice copy (same dtype and shape).  src may live on another
 * device (peer access) or another process (IPC-mapped); the copy runs on the
 * copy engines of the launching stream's device (the paper's transport,
 * PAPER.md:69).                                                            */
UM_API int um_get(const um_view* src, const um_view* dst, void* stream);
/* The same pull as one plain copy (2-D, or 1-D for a contiguous slice) that
 * the driver runs on the copy engines for peer sources: the SM-free transport for pulls a
 * running K1 waits for through um_signal / um_gemm_op.wait_flag (the
 * reference's get_async + PendingCopy.wait, fabric.py:177-201,
 * runtime.py:233-236).  Only used where um_ce_probe holds for the pair.     */
UM_API int um_get_ce(const um_view* src, const um_view* dst, void* stream);
/* *ok = 1 when a um_get_ce pull from src_device into dst_device completes
 * while a persistent kernel holds every SM of dst_device (copy engines, not
 * SM copy kernels), measured once per pair by doing exactly that with a
 * 0.5 s timeout.  get_engine "auto" / "ce" use flagged copy-engine pulls only
 * where this holds (same-device 2-D copies on the test box do NOT: the
 * driver runs them on SMs, and a K1 spinning on their flag would starve them). */
UM_API int um_ce_probe(int32_t dst_device, int32_t src_device, int32_t* ok);

/* Arrival flag of a get: write `value` to the device word `flag` in stream
 * order (after everything enqueued before it on `stream`), without using an
 * SM (stream memory operation), so a running K1 launch waiting on the flag
 * cannot starve it.  Replaces PendingTileCopy/PendingCopy.wait()
 * (distmatrix.py:42-59, fabric.py:41-58) as the device-side completion signal.
 * Returns UM_ECUDA if the device does not support stream memory operations. */
UM_API int um_signal(uint32_t* flag, uint32_t value, void* stream);
/* 1 if um_signal is usable on `device` (stream memory operations), else 0. */
UM_API int um_signal_supported(int32_t device, int32_t* out);
/* Stream-ordered wait: work enqueued on `stream` after this call starts only
 * once *flag >= value (32-bit, stream memory operation: no SM is held, so it
 * cannot starve the kernel that will produce the value).  The consumer side
 * of um_gemm_op.done_flag (K4 waiting for every replica's slice).          */
UM_API int um_wait_geq(const uint32_t* flag, uint32_t value, void* stream);

/* ======================================================================== */
/* Whole-multiply launch (runtime.execute_multiply, runtime.py:339-387)       */
/* ======================================================================== */

/* The reference's ExecConfig (runtime.py:26-40) as the C caller states it;
 * um_execute validates the counts (ValueError there, UM_EVALUE here).  The
 * schedule knobs themselves are applied when the plan is built.             */
typedef struct um_exec_cfg {
  int32_t stationarity;         /* UM_STATIONARY_A | _B | _C                 */
  int32_t prefetch_depth;       /* >= 1                                       */
  int32_t max_inflight_gemms;   /* >= 1                                       */
  int32_t max_inflight_accums;  /* >= 1                                       */
  int32_t accumulate_mode;      /* 0 PEER_ATOMIC, 1 LOCK_GET_PUT              */
  int32_t pool_capacity;        /* 0 = None (fetch-once pool), else >= 3      */
  int32_t reduce_mode;          /* UM_REDUCE_PEER | UM_REDUCE_NVLS            */
  int32_t reserved;
} um_exec_cfg;

#define UM_ACT_LAUNCH    0   /* um_gemm_launch(handle) on the rank's compute stream */
#define UM_ACT_WAIT_COPY 1   /* compute stream waits for copy `arg` to land           */
#define UM_ACT_WAIT_FLAG 2   /* compute stream waits until *(uint32*)handle >= arg     */
typedef struct um_exec_action {
  int32_t kind;
  int32_t arg;
  void* handle;
} um_exec_action;

/* One rank's serialised issue plan (what run_direct does for a rank,
 * runtime.py:193-256): copy-engine pulls (um_get, issued first on the rank's
 * get stream in first-use order) and an ordered action list.  Handles are
 * um_gemm_prepare'd launches; the caller owns them and every buffer the plan
 * names until um_sync_all (or the caller's own wait) after the last use.     */
typedef struct um_rank_plan {
  int32_t rank;
  int32_t device;
  int32_t ncopies;
  int32_t nactions;
  const um_get_desc* copies;
  const um_exec_action* actions;
} um_rank_plan;

/* One replica-reduction step: um_reduce_replicas(dst, srcs, nsrc, mode) on
 * `device`, after every rank's plan has completed (the run-level barrier,
 * runtime.py:376-386).                                                      */
typedef struct um_reduce_step {
  um_view dst;
  const um_view* srcs;
  int32_t nsrc;
  int32_t mode;
  int32_t device;
  int32_t reserved;
} um_reduce_step;

/* Issue a whole multiply asynchronously: every rank's plan on library-owned
 * streams (one compute + one get stream per rank), then the reduction steps.
 * Ordered after the previous um_execute on the same devices; returns without
 * host synchronisation.  Replaces execute_multiply's loop over ranks.       */
UM_API int um_execute(const um_rank_plan* ranks, int32_t nranks, const um_reduce_step* reduces, int32_t nreduce,
                      const um_exec_cfg* cfg);
/* Host barrier: wait until everything um_execute issued has completed.     */
UM_API int um_sync_all(void);
/* Stream interop: `stream` waits for um_execute's work on `device`
 * (um_execute_wait), or the next um_execute on `device` starts after the
 * work queued on `stream` (um_execute_after).                               */
UM_API int um_execute_wait(void* stream, int32_t device);
UM_API int um_execute_after(void* stream, int32_t device);

/* ======================================================================== */
/* K3: one-sided accumulate (fabric.py:203-234, distmatrix.py:170-209)        */
/* ======================================================================== */

/* dst += src (fp32, same shape); dst may be a peer pointer.  Element-wise
 * atomic (red.global.add), so concurrent accumulates never tear.           */
UM_API int um_accumulate(const um_view* src, const um_view* dst, void* stream);

/* ======================================================================== */
/* K4: replica reduction (distmatrix.py:211-232)                             */
/* ======================================================================== */

/* Replaces DistributedMatrix.reduce_replicas (distmatrix.py:211-232) for one
 * slice of one C tile.  mode:
 *   UM_REDUCE_PEER  dst += (srcs[0] + ... + srcs[n-1]), summed in array order
 *                   as the reference's `acc` (distmatrix.py:224-232); srcs may
 *                   be peer / IPC-mapped pointers (P2P loads over NVLink).
 *                   Views share the slice shape; a caller splits a tile into
 *                   row slices to distribute the reduction over devices.
 *   UM_REDUCE_NCCL  a collective over the replica owners: not callable on one
 *                   caller's pointers (returns UM_ECONFIG); the host drives it
 *                   with its NCCL communicator (ncclReduce per slice).
 *   UM_REDUCE_NVLS  nsrc == 1 and srcs[0] is the slice in a multicast team's
 *                   address space (um_nvls_team_create over the replicas'
 *                   um_sym_alloc blocks, dst's own replica a member): dst =
 *                   multimem.ld_reduce sum over the team (replica 0 included,
 *                   added in the switch; order is the hardware's, so real
 *                   inputs may round differently from PEER).
 * Non-origin replicas keep their partials in every mode.     */
#define UM_REDUCE_PEER 0
#define UM_REDUCE_NCCL 1
#define UM_REDUCE_NVLS 2
UM_API int um_reduce_replicas(const um_view* dst, const um_view* srcs, int32_t nsrc, int32_t mode, void* stream);

/* dst <- src (whole slice), used by broadcast_replica (distmatrix.py:234-250). */
UM_API int um_copy(const um_view* src, const um_view* dst, void* stream);

/* ======================================================================== */
/* K5: synthetic fill at global coordinates (distmatrix.py:95-101)           */
/* ======================================================================== */

#define UM_FILL_ZERO 0   /* C = 0 (cli.py:200)                               */
#define UM_FILL_INT  1   /* integers in [-8,8]  (cli.py:188-189 semantics)  */
#define UM_FILL_REAL 2   /* uniform(-1,1) rounded to the storage dtype      */
/* Fill the slice with value(seed, grow0 + r, gcol0 + c) (counter-based hash
 * at GLOBAL coordinates so replicas are identical; oracle/um_oracle.py
 * restates it).                                                            */
UM_API int um_fill(const um_view* dst, int64_t grow0, int64_t gcol0, uint64_t seed,
            int32_t mode, void* stream);

/* ======================================================================== */
/* Runtime: devices, symmetric memory, IPC (fabric.py:135-150)               */
/* ======================================================================== */

/* Enable peer access between all listed devices (single-process mode).    */
UM_API int um_init(int32_t ndev, const int32_t* devices);
/* Device allocation for the symmetric heap (one chunk).                   */
UM_API int um_device_alloc(int32_t device, uint64_t bytes, void** ptr);
UM_API int um_device_free(int32_t device, void* ptr);
/* CUDA IPC for multi-process (one process per GPU) symmetric heaps.        */
#define UM_IPC_HANDLE_BYTES 64
UM_API int um_ipc_get_handle(void* ptr, void* handle_out);
UM_API int um_ipc_open_handle(const void* handle, int32_t device, void** ptr_out);
UM_API int um_ipc_close_handle(void* ptr);
/* Symmetric memory through the CUDA VMM API (cuMemCreate + cuMemMap, mapped
 * read/write on every device that can reach the owner; POSIX-fd exportable
 * where the driver allows; sized to the multicast granularity) -- the
 * paper's pre-registered pool, and the only memory an
 * NVLS team can bind.  Replaces fabric.alloc (fabric.py:147-150) for such
 * segments.                                                                  */
UM_API int um_sym_granularity(int32_t device, uint64_t* bytes);
UM_API int um_sym_alloc(int32_t device, uint64_t bytes, void** ptr);
UM_API int um_sym_free(void* ptr);
/* NVLS (NVSwitch in-switch reduction) capability: *ok = 1 when the device
 * reports CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED AND a trial multicast
 * object can be created (a fabric not configured for multicast refuses
 * cuMulticastCreate although the attribute is set).                         */
UM_API int um_nvls_supported(int32_t device, int32_t* ok);
/* A multicast team over ndev DISTINCT devices, binding sym_ptrs[i] (a
 * um_sym_alloc base on devices[i]) at offset 0 for `bytes`; mc_ptrs_out[i]
 * receives the team's multicast address as mapped on devices[i].  Used by
 * UM_REDUCE_NVLS.  UM_ECONFIG when multicast is unsupported.                 */
UM_API int um_nvls_team_create(int32_t ndev, const int32_t* devices, void* const* sym_ptrs, uint64_t bytes,
                               void** mc_ptrs_out, void** team_out);
UM_API int um_nvls_team_destroy(void* team);
/* Device count / SM count helpers.                                          */
UM_API int um_device_count(int32_t* n);
UM_API int um_sm_count(int32_t device, int32_t* n);

/* Version and last error (thread-local).                                    */
UM_API const char* um_version(void);
UM_API const char* um_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* UNIMUL_B200_H */
