// K1: persistent bf16 x bf16 -> fp32 tile GEMM for sm_100a, C += A @ B.
//
// Replaces the reference's local multiply-accumulate
//   runtime.local_gemm            (/root/reference/pkg/src/unimul/runtime.py:96-107)
//   kernels.gemm_accumulate       (kernels.py:13-28)
//   _gemmcore.gemm_accumulate     (_gemmcore.pyx:10-25: c[i,j] += a[i,l] * b[l,j])
// and fuses the remote accumulate of Stationary A/B
//   fabric.accumulate PEER_ATOMIC (fabric.py:203-234) via distmatrix.accumulate_tile
// into the epilogue.
//
// and, in the same launch, the one-sided gets of run_direct
//   distmatrix.get_tile_async -> fabric.get_async (distmatrix.py:161-168,
//   fabric.py:177-201), PendingTileCopy.wait before local_gemm (runtime.py:219-236)
// as get warps that pull remote slices while the tensor cores work.
//
// Design (B200-first):
//  * warp-specialised persistent kernel: warp 0 = TMA producer, warp 1 = MMA
//    issuer (one thread issues tcgen05.mma), warps 2..5 = epilogue, warps
//    6..9 = get engine (pull chunks of remote slices into a staging pool; the
//    producer waits per band, per tile rows of A or per k-block rows of B).
//  * a dynamic tile scheduler (atomic counter, tile queue broadcast to both
//    CTAs of a pair) hands out tiles in raster order over the launch's ops.
//  * ops with the same C region form a k-chain: their k-segments accumulate
//    in one TMEM accumulator and the tile is reduced into C once.
//  * completion signals: when all tiles of the ops naming a done_flag are in
//    C, the epilogue adds their count to the flag (red.release.sys), which a
//    replica reducer's stream waits on (overlapped K4).
//  * operands are consumed IN PLACE from strided tile slices: each operand's
//    TMA tensor map is based at the tile base with dims (col_hi,row_hi) and the
//    loads start at (col_lo,row_lo), so arbitrary row offsets and ragged edges
//    need no copy (OOB zero-fill on load, clipping on the reduce).  TMA needs
//    the innermost start coordinate 16-byte aligned; the rare slices that
//    violate it (misaligned partitionings) are staged (see launch_batch).
//  * A is row-major m x k -> K-major SW128; B is row-major k x n -> MN-major SW128.
//  * CG == 2: a CTA pair (cluster of 2) issues cta_group::2 UMMA with M = 256;
//    each CTA stages its 128 rows of A and its half of every B column block.
//  * tile width NT per CTA pair: 256 (one N=256 accumulator, TMEM double
//    buffered so the epilogue of tile i overlaps the main loop of tile i+1) or
//    512 (two N=256 accumulators filling TMEM: 25% fewer operand bytes per
//    flop through L2; the MMA issuer runs the first k-blocks of a tile on
//    accumulator 0 while the epilogue still drains accumulator 1, so most of
//    the drain stays hidden), or 128 for latency-bound launches with few tiles
//    (one N=128 accumulator: half the per-SM drain, twice the SMs).
//  * epilogue: tcgen05.ld -> registers -> swizzled smem -> TMA reduce-add
//    (cp.reduce.async.bulk.tensor ... add) into the local C tile, or
//    red.global.add.v4.f32 straight into a peer C tile (fused K3).
//  * L2: tiles are walked in groups of 4 n-tiles so a wave of clusters shares
//    A and B panels; per-operand eviction hints are available as knobs.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <queue>
#include <vector>

#include "um_internal.h"
#include "um_ptx.cuh"

namespace um {

namespace gemm {

constexpr int BM = 128;       // rows per CTA (UMMA M = BM * CG)
constexpr int UMMA_N = 256;   // columns per tcgen05.mma (one accumulator), NT = 128: 128
// k per stage: 64 (A rows are one 128-byte swizzle row of bf16, SWIZZLE_128B)
// or 32 (A rows 64 bytes, SWIZZLE_64B; twice the stages in the same smem)
#ifndef UM_BK
#define UM_BK 64
#endif
constexpr int BK = UM_BK;
static_assert(BK == 64 || BK == 32, "BK is 64 or 32");
constexpr int A_SW_BYTES = BK * 2;            // A's swizzle span: one row of the stage's A tile
constexpr uint32_t A_LAYOUT = BK == 64 ? 2u : 4u;   // UMMA smem layout: SWIZZLE_128B / SWIZZLE_64B
constexpr int UMMA_K = 16;    // k per tcgen05.mma (kind::f16)
// epilogue warps: 4 (each drains a 32-lane quarter of TMEM, 2 smem boxes) or
// 8 (two warps per quarter, each owning half the columns; the warp loads its
// 128 columns of an accumulator into registers in one go and hands TMEM back
// before the reduce-adds, so the MMA issuer stops waiting on L2 reduce bandwidth)
// + GET_WARPS warps of the in-kernel get engine (fused K2, see below)
#ifndef UM_GET_WARPS
#define UM_GET_WARPS 4
#endif
constexpr int GET_WARPS = UM_GET_WARPS;
// launches without pulls are instantiated without get warps (GW = 0)
constexpr int num_threads(int ew, int gw) { return 64 + ew * 32 + gw * 32; }
// default rasterisation group: 4 n-tiles (negative = group along n), i.e. a
// 4-panel slice of B stays hot while A streams; measured best of {-4,4,8,16,32}
// on cfg2 / 16384^3 / cfg3 shapes with the dynamic scheduler. UM_GEMM_GROUP overrides.
constexpr int GROUP_M = -4;
constexpr int EPI_BOX_BYTES = 32 * 32 * 4;  // 32 rows x 32 fp32
constexpr int SUB_BYTES = BK * 128;          // one 64-column B sub-tile of a stage (8 KiB)
// launches of at most SMEM_WORKS works whose list sits in the parameter block
// copy it into shared memory during setup (before the programmatic-launch
// wait: kernel parameters are immutable), so no role's first tile waits on a
// chain of dependent parameter-block loads
constexpr int SMEM_WORKS = 8;

template <int CG, int NT, int EW = 4, int GW = GET_WARPS>
struct Cfg {
  static constexpr int EPI_WARPS = EW;
  static constexpr int NUM_THREADS = num_threads(EW, GW);
  static constexpr int EPI_BOXES = EW == 4 ? 2 : 1;           // smem boxes per epilogue warp
  static constexpr int UN = NT < UMMA_N ? NT : UMMA_N;       // columns per tcgen05.mma
  static constexpr int NACC = NT / UN;                       // accumulators per tile
  static constexpr int NBUF = 2 / NACC;                      // TMEM tile buffers
  static constexpr int STAGES = ((CG == 2 && NT == 256) ? 6 : (CG == 2 && NT == 128) ? 8 : 4) * (64 / BK);
  static constexpr int SUB_PER_ACC = UN / CG / 64;           // 64-col B sub-tiles per accumulator per CTA
  static constexpr int B_SUBS = NACC * SUB_PER_ACC;
  static constexpr int A_BYTES = BM * BK * 2;                // 16 KiB
  static constexpr int B_BYTES = B_SUBS * SUB_BYTES;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_BYTES = EW * EPI_BOXES * EPI_BOX_BYTES;
#if defined(UM_PROFILE) && UM_PROFILE
  static constexpr int BAR_BYTES = 512;   // + per-stage issue timestamps
#else
  static constexpr int BAR_BYTES = 256;
#endif
  static constexpr int WORKS_BYTES = SMEM_WORKS * 160;       // first works copied at setup (sizeof(Work) == 160)
  static constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + EPI_BYTES + BAR_BYTES + WORKS_BYTES;
  static constexpr uint32_t TMEM_COLS = 512;
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
};

struct alignas(16) Work {   // sizeof is a multiple of 16 (setup copies it as uint4)
  int32_t m, n, k;
  int32_t tiles_m, tiles_n, num_kb;
  int32_t tile_start, c_remote;
  int32_t a_row0, a_col0;
  int32_t b_row0, b_col0;
  int32_t c_row0, c_col0;
  int32_t c_vec_ok, group;
  int32_t a_pol, b_pol;     // L2 policy: 0 normal, 1 evict_first, 2 evict_last
  int32_t c_pol, prefetch;  // L2 policy of the C reduce-add (-1: no hint); L2 prefetch distance (k-blocks)
  int32_t sched_static, no_end_stagger;  // profiling A/B knobs: static round-robin tiles; no end stagger
  int32_t nseg, seg_kb;     // k-chain: head has nseg segments (itself + nseg-1 continuations that follow
                            // it in the work list, same C region); seg_kb = k-blocks of this segment
  int64_t c_pitch;
  float* c_ptr;
  const uint32_t* wait_flag;  // non-null: operands are staged by a get; wait for *wait_flag >= wait_value
  uint32_t wait_value;
  int32_t slot;               // completion-signal slot (-1: none)
  uint64_t wait_mask;         // bit i: wait until in-kernel get i has fully landed
  int32_t a_fine, b_fine;     // 1-based get whose chunks A (per tile rows) / B (per k-block rows) wait for
  int32_t c_prefetch, stagger;  // C L2 prefetch distance (k-blocks); accumulator stagger depth (0 = STAGES-1)
  int32_t debug_halfb;          // profiling only: skip half of the B loads (wrong results)
  int32_t debug_mma;            // profiling only: 1 = no operand loads (MMAs on stale smem), 2 = also B as K-major
};
static_assert(sizeof(Work) == 160, "Work layout (Cfg::WORKS_BYTES)");

// One slice pull of the in-kernel get engine: rows x row_bytes from src (local,
// peer or IPC-mapped memory) into a local staging buffer, cut into chunks of
// rows_per_chunk rows that the get warps of all CTAs take from a counter.
struct alignas(16) GetDesc {
  const uint8_t* src;
  uint8_t* dst;
  int64_t src_pitch, dst_pitch;   // bytes
  int32_t rows, row_bytes;
  int32_t rows_per_chunk, nchunks;
  int32_t chunk_start, vec;       // vec: 16-byte aligned rows (vector path)
  int32_t row0, pad_;             // first row of the band in its staging buffer (fine-grained waits)
};

// the work whose tile range holds tile t: the last work with tile_start <= t
// (binary search: a launch can carry > 100 works, e.g. row-sliced ops)
__device__ __forceinline__ int find_work(const Work* works, int nwork, int t) {
  int lo = 0, hi = nwork - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (works[mid].tile_start <= t) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Rasterisation: tiles are walked in groups of `group` consecutive m-tiles
// (group > 0) or n-tiles (group < 0), the other dimension sweeping inside a
// group, so a wave of clusters shares operand panels in L2.
__device__ __forceinline__ void tile_coords(const Work& wk, int lt, int& mb, int& nb) {
  if (wk.group >= 0) {
    const int G = wk.group;
    const int span = G * wk.tiles_n;
    const int g = lt / span;
    const int first = g * G;
    const int gm = min(wk.tiles_m - first, G);
    const int r = lt - g * span;
    mb = first + r % gm;
    nb = r / gm;
  } else {
    const int G = -wk.group;
    const int span = G * wk.tiles_m;
    const int g = lt / span;
    const int first = g * G;
    const int gn = min(wk.tiles_n - first, G);
    const int r = lt - g * span;
    nb = first + r % gn;
    mb = r / gn;
  }
}

// Staggered start (stream-K start, `nstag` > 0): work unit u < total_tiles is
// tile u, except that the first nstag tiles run only a prefix [0, L) of their
// k-blocks, L growing from 1 to num_kb - 1 across them; units total_tiles ..
// total_tiles + nstag - 1 are those tiles' remainders [L, num_kb).  The first
// wave's pairs thus finish their first unit at evenly spread times, so tile
// ends (and their C read-modify-write bursts) stay spread over the whole run
// instead of every pair draining at once each wave, and the remainders fill
// the last wave (list scheduling then ends within one k-block-sized piece of
// the ideal T / pairs).  Both pieces reduce-add into C (atomic), so they need
// no ordering.  Returns the tile index; [kb0, kb1) is the unit's k range.
//
// Split-k (`nsplit` > 1, launches with fewer tiles than CTA pairs): unit u is
// piece u / total_tiles of tile u % total_tiles, the pieces cutting the tile's
// k-blocks evenly, so a small launch spreads over nsplit x more SMs.
__device__ __forceinline__ int unit_span(const Work* works, int nwork, int total_tiles, int nstag, int nsplit, int u,
                                         int& w, int& kb0, int& kb1) {
  if (nsplit > 1) {
    const int t = u % total_tiles, piece = u / total_tiles;
    w = find_work(works, nwork, t);
    const int kb = works[w].num_kb;
    kb0 = (int)(((long long)piece * kb) / nsplit);
    kb1 = (int)(((long long)(piece + 1) * kb) / nsplit);
    return t;
  }
  const int t = u >= total_tiles ? u - total_tiles : u;
  w = find_work(works, nwork, t);
  const int kb = works[w].num_kb;
  kb0 = 0;
  kb1 = kb;
  if (t < nstag) {
    const int L = 1 + (int)(((long long)t * (kb - 1)) / nstag);
    if (u >= total_tiles) kb0 = L;
    else kb1 = L;
  }
  return t;
}

// Dynamic tile scheduling: the leader producer of each cluster takes the next
// tile index from a global atomic counter and broadcasts it through a small
// ring in shared memory (written into both CTAs of the pair) to every role.
// Concurrently running tiles are therefore always a sliding window of
// consecutive raster tiles, so tiles that share an operand panel run close in
// time and reuse it from L2 (a static persistent schedule lets clusters drift
// apart by whole tiles and the panels get re-read from DRAM).
constexpr int TQ = 4;  // tile-queue depth (producer runs <= 3 tiles ahead of the epilogue)

// up to 40 ops travel in the kernel parameters (CUDA >= 12.1 allows 32764
// bytes of parameters), so a whole rank's op list is normally ONE launch
constexpr int MAX_INLINE_OPS = UM_GEMM_MAX_INLINE_OPS;
constexpr int MAX_GETS = UM_GEMM_MAX_GETS;
constexpr int GET_CHUNK_BYTES = 32 * 1024;
constexpr int MAX_SLOTS = UM_GEMM_MAX_SIGNALS;
constexpr int MAX_CHUNK_FLAGS = 1 << 16;  // per-chunk landed flags (fine-grained waits)
#ifndef UM_B_WAIT_KB
#define UM_B_WAIT_KB 8
#endif
constexpr int B_WAIT_KB = UM_B_WAIT_KB;   // k-blocks of B rows waited for at once (fine waits)
// UM_PROFILE=1 (the separate libunimul_b200_prof.so, `make prof`) compiles in
// the MMA-thread wait accounting and the block-0 timeline behind UM_GEMM_STALLS.
// The default library has none of it: even untaken checks in the MMA issuer's
// loop cost ~10 % on mid-size launches (measured, 4096^3).
#ifndef UM_PROFILE
#define UM_PROFILE 0
#endif
// UM_VARIANTS=1 (`make variant`): the rejected kernel variants (cta_group::1,
// B multicast, 8 epilogue warps) without the profiling code, for A/B timing
#ifndef UM_VARIANTS
#define UM_VARIANTS 0
#endif
constexpr int TRACE_OFF = 4 * 512 - 16;   // profiling timeline stamps inside the prof buffer
// UM_GEMM_TIMELINE=<csv> (profiling build): per-pair tile spans and per-chunk
// landing times of the in-kernel pulls, after the stall counters
constexpr int TL_TILES = 96;                          // tiles recorded per pair
constexpr int TL_OFF = 4 * 512;                       // [pair][tile][3] = tile, start, end (ns)
constexpr int TL_CHUNKS = 32768;                      // chunk landing times recorded
constexpr int TL_CHUNK_OFF = TL_OFF + 128 * TL_TILES * 3;
constexpr int PS_OFF = TL_CHUNK_OFF + TL_CHUNKS;        // per CTA: producer cycles, producer waits for a free
                                                      // stage, load latency sum (issue -> full), count, max
constexpr int PS_WORDS = 8;
// (profiling) CTAs 0 and 1: per k-block of their first unit, when the producer
// issued the loads (after its stage and operand waits), and when its A rows landed
constexpr int KB_OFF = PS_OFF + 160 * PS_WORDS;
constexpr int KB_MAX = 512;
constexpr int PROF_WORDS = KB_OFF + 2 * (KB_MAX + 1);
// per-stream counter words: [0] next tile, [1] finished pairs, [2] next get chunk,
// [3, 3 + MAX_GETS) chunks landed per get, then completion-slot tallies, the
// CTA exit count, and the per-chunk landed flags
constexpr int EXIT_OFF = 3 + UM_GEMM_MAX_GETS + UM_GEMM_MAX_SIGNALS;
constexpr int CHUNK_FLAGS_OFF = EXIT_OFF + 1;

// Completion signal: once every tile of every op naming this slot has been
// written (all epilogue warps of both CTAs of each tile arrive), the kernel
// adds 1 to *flag with release semantics at system scope (flag may be a peer
// or IPC-mapped word: the replica reducer on another GPU waits on it).
struct alignas(16) SignalSlot {
  uint32_t* flag;
  int32_t expected;    // epilogue-warp arrivals (tiles x warps x CTAs) that complete the slot
  uint32_t increment;  // added to *flag: the number of ops of this launch naming the flag
};
struct alignas(64) LaunchArgs {
  const Work* works;          // null: use inl_works
  const CUtensorMap* maps;    // null: use inl_maps
  int nwork, total_tiles;
  int* counters;              // per-stream {tile, done clusters, get chunk, get done[MAX_GETS]}
  int ngets, total_chunks;
  int nslots;
  int nstag;                  // staggered start: the first nstag tiles run a k-prefix, their rest comes last
  int stag_ok;                // host: this launch may use a staggered start (set at prepare)
  int ext_waits;              // host: some op waits on an external arrival flag (copy-engine pull)
  int nsplit;                 // split-k pieces per tile (small launches), 1 = off
  int smem_works;             // host: the work list (inline, <= SMEM_WORKS works) is read from a shared-memory copy
  uint32_t get_ns_per_chunk;  // > 0: pace the pulls to one chunk per this many ns (link-rate emulation)
  unsigned long long* prof;   // (profiling, UM_GEMM_STALLS) per cluster: MMA-thread cycles total / waiting
                              // for operands / for the epilogue to free TMEM / for the next tile
  SignalSlot slots[MAX_SLOTS];
  CUtensorMap inl_maps[3 * MAX_INLINE_OPS];
  Work inl_works[MAX_INLINE_OPS];
  GetDesc gets[MAX_GETS];
  int32_t get_order[MAX_GETS];  // pull order: the i-th get pulled is gets[get_order[i]] (chunk_start ascending)
};
static_assert(sizeof(LaunchArgs) <= 32764, "kernel parameter block");

template <int CG, int NT, int EW, int GW, int NP>
__global__ void __launch_bounds__(num_threads(EW, GW), 1)
    gemm_bf16_kernel(const __grid_constant__ LaunchArgs args) {
  using C = Cfg<CG, NT, EW, GW>;
  constexpr int EPI_WARPS = EW;
  // NP pairs per cluster (NP == 2: a cluster of 4 CTAs computes a 512 x NT
  // super-tile; the two pairs share the B k-panel through TMA multicast)
  static_assert(NP == 1 || ((NP == 2 || NP == 4) && CG == 2), "B multicast needs CTA pairs");
  constexpr int CS = CG * NP;   // cluster size
  // small op lists travel inside the kernel parameters (no per-launch device
  // allocation or host->device copy); larger ones in a global-memory block
  const Work* __restrict__ works = args.works ? args.works : args.inl_works;   // (shared-memory copy below)
  const CUtensorMap* __restrict__ maps = args.maps ? args.maps : args.inl_maps;
  const int nwork = args.nwork;
  const int total_tiles = args.total_tiles;
  const int nstag = args.nstag;
  const int nsplit = args.nsplit;
  // work units handed out by the tile scheduler
  const int total_units = nsplit > 1 ? total_tiles * nsplit : total_tiles + nstag;
  int* const tile_counter = args.counters;       // [0] next tile, [1] finished clusters
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + C::STAGES * C::A_BYTES;
  uint8_t* smem_epi = smem + C::STAGES * C::STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_epi + C::EPI_BYTES);
  uint64_t* full = bars;                            // [STAGES]
  uint64_t* empty = bars + C::STAGES;               // [STAGES]
  uint64_t* tmem_full = bars + 2 * C::STAGES;       // [NBUF]
  uint64_t* tmem_empty = bars + 2 * C::STAGES + 2;  // [2]: per buffer (NACC=1) or per accumulator (NACC=2)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::STAGES + 4);
  uint64_t* tq_full = bars + 2 * C::STAGES + 5;     // [TQ]
  uint64_t* tq_empty = tq_full + TQ;                // [TQ] (leader CTA)
  volatile int* tq = reinterpret_cast<volatile int*>(tq_empty + TQ);  // [TQ]
  Work* smem_wk = reinterpret_cast<Work*>(reinterpret_cast<uint8_t*>(bars) + C::BAR_BYTES);   // [SMEM_WORKS]
#if UM_PROFILE
  // (profiling) clock64 at which the leader's producer issued each stage's loads
  volatile unsigned long long* issue_ts = reinterpret_cast<volatile unsigned long long*>(tq_empty + TQ + TQ / 2);
  static_assert((2 * C::STAGES + 5 + 2 * TQ + TQ / 2 + C::STAGES) * 8 <= C::BAR_BYTES, "barrier area");
#endif

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  // NP > 1 launches with a preferred cluster of 2*NP CTAs and a regular one of
  // 2: the hardware forms the big clusters where a GPC has room and pairs
  // elsewhere, so the cluster size (cs) and its pair count (np) are runtime values
  const uint32_t crank = (CS > 1) ? ptx::cluster_ctarank() : 0u;   // rank in the cluster
  const int cs = NP > 1 ? (int)ptx::cluster_nctarank() : CS;        // this cluster's size
  const int np = cs / CG;                                           // pairs in this cluster
  const uint32_t cta_rank = crank % CG;                             // rank in the CTA pair
  const int pair = (int)(crank / CG);
  const bool leader = cta_rank == 0;                                // pair leader (issues the MMAs)
  const bool cleader = crank == 0;                                  // cluster leader (takes tiles)
  const int TQ_CONSUMERS = (cs - 1) /*peer producers*/ + np /*MMA*/ + EPI_WARPS * cs;
  // tile-queue entries: the tile index, or for NP > 1 (tile * NP + part) where
  // a lone pair runs the NP 256-row parts of a tile one after the other
  auto decode = [&](int q, int& t, int& row_off) {
    int sub = 0;
    if constexpr (NP > 1) {
      t = q / NP;
      sub = np == NP ? pair : (q % NP);
    } else {
      t = q;
    }
    row_off = sub * BM * CG + (int)cta_rank * BM;   // this CTA's rows in the tile
  };

  // profiling (UM_GEMM_STALLS): block 0 stamps the globaltimer at milestones of
  // its first tile, to see where a small launch's fixed latency goes
  auto stamp = [&](int i) {
#if UM_PROFILE
    if (args.prof && blockIdx.x == 0) args.prof[TRACE_OFF + i] = ptx::globaltimer();
#else
    (void)i;
#endif
  };
  if (threadIdx.x == 0) stamp(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], np);   // every pair's MMAs release the stage (multicast B)
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tmem_full[s], 1);
      ptx::mbar_init(&tmem_empty[s], EPI_WARPS * CG);
    }
    for (int s = 0; s < TQ; ++s) {
      ptx::mbar_init(&tq_full[s], 1);
      ptx::mbar_init(&tq_empty[s], TQ_CONSUMERS);
    }
    ptx::fence_mbar_init();
  }
  // consumer side of the tile queue (one thread): i-th tile of this cluster
  auto next_tile = [&](int i) -> int {
    const int slot = i % TQ;
    ptx::mbar_wait_cluster(&tq_full[slot], (uint32_t)(i / TQ) & 1u);
    const int t = tq[slot];
    if constexpr (CG == 1) ptx::mbar_arrive(&tq_empty[slot]);
    else ptx::mbar_arrive_cluster(&tq_empty[slot], 0);
    return t;
  };
  if (args.smem_works && threadIdx.x >= 64) {
    const int v = threadIdx.x - 64;
    if (v < nwork * (int)(sizeof(Work) / 16))
      reinterpret_cast<uint4*>(smem_wk)[v] = reinterpret_cast<const uint4*>(args.inl_works)[v];
  }
  if (warp == 1) ptx::tmem_alloc<CG>(tmem_slot, C::TMEM_COLS);
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (args.smem_works) works = smem_wk;
  // Programmatic dependent launch: the setup above touches only this CTA's
  // shared memory and TMEM, so it may overlap the previous kernel's tail on
  // the stream (launched with programmatic stream serialization); every
  // global access comes after the wait for that kernel's completion.
  ptx::griddep_wait();
  // a launch that waits on copy-engine arrivals keeps its dependents out until
  // it exits: their CTAs, resident early, would take the SMs left free for
  // copies the driver runs with SMs (same-device 2-D copies)
  if (!args.ext_waits) ptx::griddep_launch_dependents();
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int s = 0; s < args.nslots; ++s)   // a slot whose ops have no tile is complete at once
      if (args.slots[s].expected == 0) ptx::red_release_sys_add_u32(args.slots[s].flag, args.slots[s].increment);
  // warm the descriptors of the first works while the CTA sets up (the first
  // TMA otherwise waits for its tensor map: ~1 us of a small launch)
  if (warp == 0 && lane < 3 * 8 && lane / 3 < nwork) ptx::prefetch_tmap(&maps[lane]);
  // ... and the first works themselves: every role's first tile reads them
  // through a chain of dependent scalar loads, each a cold miss (~1 us) when
  // the work list sits in the parameter block; one parallel touch here (32
  // lanes x 16 B) brings them into the SM's caches during setup
  if (!args.smem_works && (warp == 2 || warp == 3)) {
    const int nvec = min(nwork, 8) * (int)(sizeof(Work) / 16);
    const int v = (warp - 2) * 32 + lane;
    if (v < nvec) {
      const volatile uint4* wv = reinterpret_cast<const volatile uint4*>(works) + v;
      (void)wv->x;
    }
  }
  if (threadIdx.x == 0) stamp(1);

  if (warp == 0) {
    // ===================== TMA producer (warp 0; one elected lane issues) =====================
    // The whole warp runs the k-block loop so the TMA operands (tensor-map
    // address, coordinates, smem and barrier addresses) are warp-uniform: a
    // single-thread loop paid a per-instruction uniform-register waterfall and
    // its dependent chain (~1.5k cycles per k-block, measured) became the
    // operand-feed limit.  Tile-queue and get/flag waits stay on lane 0.
    {
      const bool issuer = ptx::elect_one();
      const uint64_t pols[3] = {ptx::policy_evict_normal(), ptx::policy_evict_first(), ptx::policy_evict_last()};
      int stage = 0;
      uint32_t phase = 0;
      uint64_t landed = 0;   // (lane 0) in-kernel gets whose every chunk this producer has observed
      // fine-grained waits: rows [r0, r1) of get g's band.  Fast path: the
      // band's chunk count says it has fully landed (then never checked
      // again); otherwise the flags of the chunks holding those rows, loaded
      // 8 at a time so their latencies overlap.
      auto wait_rows = [&](int g, int r0, int r1) {
        if ((landed >> g) & 1ull) return;
        const GetDesc& gd = args.gets[g];
        if (ptx::ld_relaxed_gpu_s32(&args.counters[3 + g]) >= gd.nchunks) {
          landed |= 1ull << g;
        } else {
          const int lo = max(r0 - gd.row0, 0), hi = min(r1 - gd.row0, gd.rows);
          if (hi <= lo) return;
          const int c_lo = gd.chunk_start + lo / gd.rows_per_chunk;
          const int c_hi = gd.chunk_start + (hi - 1) / gd.rows_per_chunk;
          const uint64_t t0 = ptx::globaltimer();
          uint32_t spins = 0;
          for (int c = c_lo; c <= c_hi; c += 8) {
            const int n = min(8, c_hi - c + 1);
            for (;;) {
              int ok = 1;
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (i < n) ok &= ptx::ld_relaxed_gpu_s32(&args.counters[CHUNK_FLAGS_OFF + c + i]) != 0;
              if (ok) break;
              __nanosleep(64);
              if ((++spins & 0x3FFFu) == 0 && ptx::globaltimer() - t0 > 20000000000ull) {
                printf("unimul_b200: chunk watchdog fired (block %d, get %d, chunk %d)\n", blockIdx.x, g, c);
                __trap();
              }
            }
          }
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        ptx::fence_proxy_async_global();
      };
      int flag_ok = -1;      // (lane 0) highest work index whose external arrival flag has been observed
      int q = 0;
#if UM_PROFILE
      unsigned long long p_empty = 0, p_issue = 0, p_t_issue = 0, p_tma = 0, p_loop = 0;
      const unsigned long long p_begin = clock64();
#endif
      for (int i = 0;; ++i) {
        if (lane == 0) {
          if (cleader) {
            // take the next tile and publish it to every CTA of the cluster
            const int slot = i % TQ;
            ptx::mbar_wait_cluster(&tq_empty[slot], ((uint32_t)(i / TQ) & 1u) ^ 1u);
            if (i == 0) stamp(11);
            if (NP > 1 && np == 1 && (i % NP) != 0) {
              q += 1;   // next part of the tile taken NP entries ago
            } else {
              // (a static first unit per cluster, i.e. no atomic on the launch's
              // critical path, was measured: no gain at 256^3..2048^3, -15 % at
              // 4096^3 with the staggered start, so every unit is dynamic)
              int t = (NP == 1 && works[0].sched_static) ? (int)(blockIdx.x / CS) + i * (int)(gridDim.x / CS)  // A/B knob
                                                         : atomicAdd(tile_counter, 1);
              if (t > total_units) t = total_units;
              q = t * NP;
            }
            if (i == 0) stamp(12);
            tq[slot] = q;
            if constexpr (CS > 1) {
              for (int r = 1; r < cs; ++r) ptx::st_shared_cluster_u32((const void*)&tq[slot], r, (uint32_t)q);
              for (int r = 0; r < cs; ++r) ptx::mbar_arrive_cluster(&tq_full[slot], r);
            } else {
              ptx::mbar_arrive_cluster(&tq_full[slot], 0);
            }
          } else {
            q = next_tile(i);
          }
        }
        q = __shfl_sync(0xffffffffu, q, 0);
        int t, row_off;
        decode(q, t, row_off);
        if (i == 0 && lane == 0) stamp(2);
        if (t >= total_units) {
          if (leader && lane == 0) {
            // this pair is done with the counter (its cluster leader took its
            // last tile); the last pair out re-zeroes it for the next launch
            __threadfence();
            if (atomicAdd(&tile_counter[1], 1) == (int)(gridDim.x / CG) - 1) {
              atomicExch(&tile_counter[0], 0);
              atomicExch(&tile_counter[1], 0);
            }
          }
#if UM_PROFILE
          if (args.prof && blockIdx.x < 160 && lane == 0) {
            args.prof[PS_OFF + PS_WORDS * blockIdx.x + 0] = clock64() - p_begin;
            args.prof[PS_OFF + PS_WORDS * blockIdx.x + 1] = p_empty;
            args.prof[PS_OFF + PS_WORDS * blockIdx.x + 5] = p_issue;
            args.prof[PS_OFF + PS_WORDS * blockIdx.x + 6] = p_tma;
            args.prof[PS_OFF + PS_WORDS * blockIdx.x + 7] = p_loop;
          }
#endif
          break;
        }
        int w0, ukb0, ukb1;
        t = unit_span(works, nwork, total_tiles, nstag, nsplit, t, w0, ukb0, ukb1);
        // the head work by value: independent vector loads instead of a chain
        // of dependent scalar ones through the parameter block
        const Work W0 = works[w0];
        int mb, nb;
        tile_coords(W0, t - W0.tile_start, mb, nb);
        if (i == 0 && lane == 0) stamp(13);
        // a k-chain: the segments (ops with the same C region) are loaded one
        // after the other into the same accumulator, one epilogue per tile
        int kbg = 0;   // k-block index over the whole chain (C prefetch trigger)
        const int cpf_at = W0.c_prefetch > 0 && W0.c_remote == 0 ? max(0, W0.num_kb - W0.c_prefetch) : -1;
        const int nseg = W0.nseg;
        // loop-invariant knobs read once per tile (the work list lives in the
        // parameter block or global memory: no reloads inside the k loop)
        const bool halfb = NP == 1 && C::NACC == 2 && works[0].debug_halfb;
#if UM_PROFILE
        const bool mma_only = works[0].debug_mma != 0;
#endif
        for (int w = w0; w < w0 + nseg; ++w) {
        const Work wk = w == w0 ? W0 : works[w];
        const int a_col0 = wk.a_col0, b_row0 = wk.b_row0, a_fine = wk.a_fine, b_fine = wk.b_fine;
        // fused get -> GEMM: this segment reads operand slices a get is still
        // delivering; wait until every chunk of those gets has landed
        if (lane == 0) {
          if (wk.wait_flag && w > flag_ok) {
            ptx::wait_flag_geq(wk.wait_flag, wk.wait_value);
            flag_ok = w;
          }
          for (uint64_t msk = wk.wait_mask & ~landed; msk; msk &= msk - 1) {
            const int gi = __ffsll((long long)msk) - 1;
            ptx::wait_count_geq(&args.counters[3 + gi], args.gets[gi].nchunks);
          }
          landed |= wk.wait_mask;
        }
        const CUtensorMap* ma = &maps[3 * w + 0];
        const CUtensorMap* mbm = &maps[3 * w + 1];
        const uint64_t pa = pols[wk.a_pol], pb = pols[wk.b_pol];
        const int arow = wk.a_row0 + mb * BM * CG * NP + row_off;
        const int bcol = wk.b_col0 + nb * NT + (int)cta_rank * (C::UN / CG);
        if (a_fine && lane == 0) wait_rows(a_fine - 1, arow, arow + BM);   // this CTA's A rows, all k
#if UM_PROFILE
        if (args.prof && i == 0 && w == w0 && blockIdx.x < 2 && lane == 0)
          args.prof[KB_OFF + blockIdx.x * (KB_MAX + 1) + KB_MAX] = ptx::globaltimer();
#endif
        __syncwarp();
        // optional L2 prefetch `pf` k-blocks ahead of the loads (UM_GEMM_PF; off by
        // default: measured slower, 1437 -> 1143..1292 TFLOP/s on cfg2)
        auto prefetch = [&](int kb) {
          if (!issuer) return;
          ptx::tma_prefetch_2d(ma, a_col0 + kb * BK, arow);
#pragma unroll
          for (int j = 0; j < C::NACC; ++j)
#pragma unroll
            for (int s = 0; s < C::SUB_PER_ACC; ++s)
              ptx::tma_prefetch_2d(mbm, bcol + j * C::UN + s * 64, b_row0 + kb * BK);
        };
        const int pf = wk.prefetch;
        // k-blocks of this segment; a staggered or split-k unit (single-segment
        // works only) covers [ukb0, ukb1) of its tile
        const bool piece = nstag > 0 || nsplit > 1;
        const int kbs = piece ? ukb0 : 0, kbe = piece ? ukb1 : wk.seg_kb;
        if (pf > 0)
          for (int kb = kbs; kb < min(kbs + pf, kbe); ++kb) prefetch(kb);
        if (i == 0 && lane == 0) stamp(14);
#if UM_PROFILE
        const unsigned long long p_t_loop = clock64();
#endif
        for (int kb = kbs; kb < kbe; ++kb) {
          if (pf > 0 && kb + pf < kbe) prefetch(kb + pf);
#if UM_PROFILE
          {
            const unsigned long long e0 = clock64();
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            const unsigned long long e1 = clock64();
            p_empty += e1 - e0;
            p_t_issue = e1;
            if (leader && lane == 0) issue_ts[stage] = e1;
          }
          if (mma_only) {   // (profiling) MMA-issue bound: no loads at all
            if (leader && issuer) ptx::mbar_arrive(&full[stage]);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
#else
          ptx::mbar_wait(&empty[stage], phase ^ 1);
#endif
          constexpr uint32_t MC_MASK = NP == 4 ? 0x55u : 0x5u;   // pair rank 0 of every pair
          const bool mcast = NP > 1 && np == NP;
          const uint32_t sa = ptx::smem_u32(smem_a + stage * C::A_BYTES);
          const uint32_t sb = ptx::smem_u32(smem_b + stage * C::B_BYTES);
          const int kcol = a_col0 + kb * BK;
          const int krow = b_row0 + kb * BK;
          if (b_fine && ((kb - kbs) % B_WAIT_KB) == 0) {
            // the B rows of the next B_WAIT_KB k-blocks: one flag poll + acquire
            // fence per batch (per k-block, the fences and polls of a band still
            // landing cost ~1.7 us per k-block: 2.4 instead of 0.7 us)
            if (lane == 0) wait_rows(b_fine - 1, krow, b_row0 + min(kb + B_WAIT_KB, kbe) * BK);
            __syncwarp();
          }
          if (kbg++ == cpf_at && issuer) {
            // bring this CTA's 128 x NT block of C into L2 ahead of the reduce-adds
            const Work& hd = works[w0];
            const CUtensorMap* mcp = &maps[3 * w0 + 2];
            const int crow = hd.c_row0 + mb * BM * CG * NP + row_off;
            for (int r = 0; r < BM; r += 32)
              for (int c = 0; c < NT; c += 32) ptx::tma_prefetch_2d(mcp, hd.c_col0 + nb * NT + c, crow + r);
          }
#if UM_PROFILE
          const unsigned long long p_t_tma = clock64();
#endif
          if (issuer) {
            // (profiling only, UM_GEMM_DEBUG_HALFB: wrong results) skip the second
            // accumulator's B sub-tiles -> bound on what halving B traffic can buy
            if (leader) ptx::mbar_arrive_expect_tx(&full[stage], (C::STAGE_BYTES - (halfb ? C::B_BYTES / 2 : 0)) * CG);
            if constexpr (CG == 1) {
              ptx::tma_load_2d_s(sa, ma, &full[stage], kcol, arow, pa);
            } else {
              ptx::tma_load_2d_cg2_s(sa, ma, &full[stage], kcol, arow, pa);
            }
#pragma unroll
            for (int j = 0; j < C::NACC; ++j)
#pragma unroll
              for (int s = 0; s < C::SUB_PER_ACC; ++s) {
                if (halfb && j == 1) continue;
                const int qsub = j * C::SUB_PER_ACC + s;
                const uint32_t dst = sb + qsub * SUB_BYTES;
                const int col = bcol + j * C::UN + s * 64;
                if (mcast) {
                  // the CTAs with this pair rank in the other pairs need the same B
                  // sub-tiles: each loads 1/NP of them into all (multicast)
                  if ((qsub * NP) / C::B_SUBS != pair) continue;
                  ptx::tma_load_2d_cg2_mc_s(dst, mbm, &full[stage], col, krow, (uint16_t)(MC_MASK << cta_rank), pb);
                } else if constexpr (CG == 1) {
                  ptx::tma_load_2d_s(dst, mbm, &full[stage], col, krow, pb);
                } else {
                  ptx::tma_load_2d_cg2_s(dst, mbm, &full[stage], col, krow, pb);
                }
              }
          }
          if (i == 0 && kb == 0 && lane == 0) stamp(3);
#if UM_PROFILE
          if (args.prof && i == 0 && blockIdx.x < 2 && lane == 0 && kb - kbs < KB_MAX)
            args.prof[KB_OFF + blockIdx.x * (KB_MAX + 1) + (kb - kbs)] = ptx::globaltimer();
#endif
#if UM_PROFILE
          {
            const unsigned long long p_now = clock64();
            p_issue += p_now - p_t_issue;
            p_tma += p_now - p_t_tma;
          }
#endif
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
#if UM_PROFILE
        p_loop += clock64() - p_t_loop;
#endif
        }  // k-chain segments
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA; one elected lane issues) =====================
    // The whole warp runs the loop (barrier waits, descriptor arithmetic) so
    // every operand of tcgen05.mma is warp-uniform; one elected lane issues.
    if (leader) {
      const bool issuer = ptx::elect_one();
      constexpr uint32_t idesc = ptx::make_idesc_bf16(BM * CG, C::UN, 0, 1);
      // a stage is free once every pair sharing its B (multicast) has consumed it
      const uint16_t EMPTY_MASK = (uint16_t)((1u << cs) - 1);
      const uint16_t PAIR_MASK = (uint16_t)(0x3u << (pair * CG));
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      unsigned long long c_full = 0, c_tmem = 0, c_tile = 0;
      const unsigned long long c_begin = clock64();
#if UM_PROFILE
      unsigned long long l_sum = 0, l_cnt = 0, l_max = 0;
#endif
      // (profiling) wait for a stage's operands and account the issue -> landed latency
      auto wait_full = [&](int stg, uint32_t ph) {
#if UM_PROFILE
        if (args.prof) {
          const unsigned long long t0 = clock64();
          ptx::mbar_wait(&full[stg], ph);
          const unsigned long long t1 = clock64();
          c_full += t1 - t0;
          const unsigned long long lat = t1 - issue_ts[stg];
          l_sum += lat;
          ++l_cnt;
          l_max = lat > l_max ? lat : l_max;
          return;
        }
#endif
        ptx::mbar_wait(&full[stg], ph);
      };
      auto timed = [&](unsigned long long& acc, auto&& fn) {
#if UM_PROFILE
        if (args.prof) {
          const unsigned long long t0 = clock64();
          fn();
          acc += clock64() - t0;
        } else {
          fn();
        }
#else
        (void)acc;
        fn();
#endif
      };
      // all MMAs of one k-block into accumulator `acc_col`
      auto issue = [&](int stg, uint32_t acc_col, int j, bool first_kb) {
        const uint32_t sa = ptx::smem_u32(smem_a + stg * C::A_BYTES);
        const uint32_t sb = ptx::smem_u32(smem_b + stg * C::B_BYTES) + j * C::SUB_PER_ACC * SUB_BYTES;
#if UM_PROFILE
        if (BK == 64 && works[0].debug_mma == 2) {   // (profiling) B read as K-major SW128: UMMA rate vs operand major-ness
          constexpr uint32_t idesc_k = ptx::make_idesc_bf16(BM * CG, C::UN, 0, 0);
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; ++kk) {
            const uint64_t adesc = ptx::make_smem_desc(sa + kk * (UMMA_K * 2), 16, 1024);
            const uint64_t bdesc = ptx::make_smem_desc(sb + kk * (UMMA_K * 2), 16, 1024);
            if (issuer) ptx::umma_f16<CG>(tmem_base + acc_col, adesc, bdesc, idesc_k, (!first_kb || kk) ? 1u : 0u);
          }
          return;
        }
#endif
#pragma unroll
        for (int kk = 0; kk < BK / UMMA_K; ++kk) {
          // A: K-major, swizzled rows of BK bf16; 8-row groups 8 * A_SW_BYTES apart;
          // advance 32 B per UMMA_K inside the swizzle row.
          const uint64_t adesc = ptx::make_smem_desc(sa + kk * (UMMA_K * 2), 16, 8 * A_SW_BYTES, A_LAYOUT);
          // B: MN-major SW128; 64-column blocks SUB_BYTES apart (LBO), 8-k groups
          // 1024 B apart (SBO); advance 16 k-rows = 2048 B per UMMA_K.
          const uint64_t bdesc = ptx::make_smem_desc(sb + kk * (UMMA_K * 128), SUB_BYTES, 1024);
          if (issuer) ptx::umma_f16<CG>(tmem_base + acc_col, adesc, bdesc, idesc, (!first_kb || kk) ? 1u : 0u);
        }
      };
      for (;; ++it) {
        int t = 0, row_off_unused;
        if (lane == 0) timed(c_tile, [&] { t = next_tile(it); });
        t = __shfl_sync(0xffffffffu, t, 0);
        decode(t, t, row_off_unused);
        if (t >= total_units) break;
#if UM_PROFILE
        const int tl_pair = (int)(blockIdx.x / CG);
        if (args.prof && it < TL_TILES && tl_pair < 128 && lane == 0) {
          unsigned long long* e = args.prof + TL_OFF + (tl_pair * TL_TILES + it) * 3;
          e[0] = (unsigned long long)t + 1;
          e[1] = ptx::globaltimer();
        }
#endif
        int w, ukb0, ukb1;
        t = unit_span(works, nwork, total_tiles, nstag, nsplit, t, w, ukb0, ukb1);
        const int num_kb = ukb1 - ukb0;    // k-blocks of this unit (the whole chain's, unstaggered)
        const int buf = it % C::NBUF;
        const uint32_t tph = (uint32_t)(it / C::NBUF) & 1u;
        if constexpr (C::NACC == 1) {
          timed(c_tmem, [&] { ptx::mbar_wait(&tmem_empty[buf], tph ^ 1); });
          ptx::tc_fence_after();
          for (int kb = 0; kb < num_kb; ++kb) {
            wait_full(stage, phase);
            if (it == 0 && kb == 0 && lane == 0) stamp(4);
            ptx::tc_fence_after();
            issue(stage, buf * C::UN, 0, kb == 0);
            if (issuer) ptx::umma_commit<CG>(&empty[stage], EMPTY_MASK);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
        } else {
          // accumulator 0 runs ahead by D k-blocks while the epilogue drains accumulator 1
          // no_end_stagger == 2: no stagger at all (both accumulators per k-block)
          const int SG = works[0].stagger > 0 ? min(works[0].stagger, C::STAGES - 1) : C::STAGES - 1;
          const int D = works[0].no_end_stagger == 2 ? 0 : min(SG, num_kb);
          timed(c_tmem, [&] { ptx::mbar_wait(&tmem_empty[0], tph ^ 1); });
          ptx::tc_fence_after();
          const int stage0 = stage;
          for (int kb = 0; kb < D; ++kb) {
            wait_full(stage, phase);
            ptx::tc_fence_after();
            issue(stage, 0, 0, kb == 0);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
          timed(c_tmem, [&] { ptx::mbar_wait(&tmem_empty[1], tph ^ 1); });
          ptx::tc_fence_after();
          int st = stage0;
          for (int kb = 0; kb < D; ++kb) {
            issue(st, C::UN, 1, kb == 0);
            if (issuer) ptx::umma_commit<CG>(&empty[st], EMPTY_MASK);
            if (++st == C::STAGES) st = 0;
          }
          // accumulator 0 also finishes E k-blocks early, so its drain overlaps
          // accumulator 1's tail
          const int E = works[0].no_end_stagger ? 0 : min(SG, num_kb - D);
          for (int kb = D; kb < num_kb - E; ++kb) {
            wait_full(stage, phase);
            ptx::tc_fence_after();
            issue(stage, 0, 0, kb == 0);          // kb == 0 only without a leading stagger (D == 0)
            issue(stage, C::UN, 1, kb == 0);
            if (issuer) ptx::umma_commit<CG>(&empty[stage], EMPTY_MASK);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
          const int stageE = stage;
          for (int kb = num_kb - E; kb < num_kb; ++kb) {
            wait_full(stage, phase);
            ptx::tc_fence_after();
            issue(stage, 0, 0, false);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
          if (issuer) ptx::umma_commit<CG>(&tmem_full[0], PAIR_MASK);
          st = stageE;
          for (int kb = num_kb - E; kb < num_kb; ++kb) {
            issue(st, C::UN, 1, false);
            if (issuer) ptx::umma_commit<CG>(&empty[st], EMPTY_MASK);
            if (++st == C::STAGES) st = 0;
          }
          if (issuer) ptx::umma_commit<CG>(&tmem_full[1], PAIR_MASK);
        }
        if constexpr (C::NACC == 1) if (issuer) ptx::umma_commit<CG>(&tmem_full[buf], PAIR_MASK);
        if (it == 0 && lane == 0) stamp(5);
#if UM_PROFILE
        if (args.prof && it < TL_TILES && tl_pair < 128 && lane == 0)   // all MMAs of the tile issued
          args.prof[TL_OFF + (tl_pair * TL_TILES + it) * 3 + 2] = ptx::globaltimer();
#endif
      }
      if (args.prof && lane == 0) {
        unsigned long long* o = args.prof + 4 * (blockIdx.x / CG);
        o[0] = clock64() - c_begin;
        o[1] = c_full;
        o[2] = c_tmem;
        o[3] = c_tile | ((unsigned long long)cs << 56);   // + this cluster's size
#if UM_PROFILE
        if (blockIdx.x < 160) {
          args.prof[PS_OFF + PS_WORDS * blockIdx.x + 2] = l_sum;
          args.prof[PS_OFF + PS_WORDS * blockIdx.x + 3] = l_cnt;
          args.prof[PS_OFF + PS_WORDS * blockIdx.x + 4] = l_max;
        }
#endif
      }
    }
  } else if (warp < 2 + EW) {
    // ===================== Epilogue (EW warps) =====================
    const int e = warp - 2;
    const int q = warp & 3;  // TMEM lane quarter this warp may access (hardware: warp % 4)
    constexpr int CHUNKS = C::UN / 32;                       // 32-column chunks per accumulator
    constexpr int WCH = EW == 4 ? CHUNKS : CHUNKS / 2;        // chunks per warp per accumulator
    const int ch0 = EW == 4 ? 0 : (e / 4) * WCH;              // EW == 8: column half of this warp
    const uint64_t cpols[3] = {ptx::policy_evict_normal(), ptx::policy_evict_first(), ptx::policy_evict_last()};
    uint64_t cpol = cpols[0];
    uint8_t* ebuf = smem_epi + e * C::EPI_BOXES * EPI_BOX_BYTES;
    const uint32_t ebuf_u32 = ptx::smem_u32(ebuf);
    const bool issuer = ptx::elect_one();   // issues this warp's bulk (TMA) ops; uniform operands
    int it = 0;
    int sbuf = 0;
    for (;; ++it) {
      int t = 0, row_off;
      if (lane == 0) t = next_tile(it);
      decode(__shfl_sync(0xffffffffu, t, 0), t, row_off);
      if (t >= total_units) break;
      int w, ukb0_unused, ukb1_unused;
      t = unit_span(works, nwork, total_tiles, nstag, nsplit, t, w, ukb0_unused, ukb1_unused);
      const Work& wk = works[w];
      const CUtensorMap* mc = &maps[3 * w + 2];
      const int c_remote = wk.c_remote, c_col0 = wk.c_col0, c_row0 = wk.c_row0, c_pol = wk.c_pol;
      if (c_pol >= 0) cpol = cpols[c_pol];
      int mb, nb;
      tile_coords(wk, t - wk.tile_start, mb, nb);
      const int buf = it % C::NBUF;
      const uint32_t tph = (uint32_t)(it / C::NBUF) & 1u;
      const int row_in_op = mb * BM * CG * NP + row_off + q * 32;   // first row of this warp

      // one 32x32 fp32 chunk (lane = row) from registers into C
      auto emit = [&](const uint32_t (&r)[32], int col0) {
        if (c_remote == 3) return;  // (profiling only) accumulator dropped: isolates the main loop's cost
        if (issuer) ptx::bulk_wait_read<C::EPI_BOXES - 1>();   // box no longer read by an earlier TMA op
        __syncwarp();
        const uint32_t base = ebuf_u32 + sbuf * EPI_BOX_BYTES;
        if (c_remote != 1) {
          // registers -> swizzled smem box -> TMA reduce-add into C
#pragma unroll
          for (int i = 0; i < 8; ++i)
            ptx::st_shared_v4(base + lane * 128 + ((i ^ (lane & 7)) << 4), r[4 * i], r[4 * i + 1], r[4 * i + 2],
                              r[4 * i + 3]);
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (issuer) {
            uint8_t* box = ebuf + sbuf * EPI_BOX_BYTES;
            if (c_remote == 2)  // (profiling only) plain store instead of reduce
              ptx::tma_store_2d(mc, box, c_col0 + col0, c_row0 + row_in_op);
            else if (c_pol >= 0)
              ptx::tma_reduce_add_2d_hint(mc, box, c_col0 + col0, c_row0 + row_in_op, cpol);
            else
              ptx::tma_reduce_add_2d(mc, box, c_col0 + col0, c_row0 + row_in_op);
            ptx::bulk_commit();
          }
        } else {
          // fused remote accumulate (K3): red.global.add into the (peer) C tile.
          // The 32x32 chunk is transposed through swizzled smem so that each
          // warp-wide red.v4 covers 4 full 128-byte row segments (coalesced
          // over NVLink / into L2); no async buffer to wait for.
#pragma unroll
          for (int i = 0; i < 8; ++i)
            ptx::st_shared_v4(base + lane * 128 + ((i ^ (lane & 7)) << 4), r[4 * i], r[4 * i + 1], r[4 * i + 2],
                              r[4 * i + 3]);
          __syncwarp();
          const int c4 = lane & 7;          // 16-byte column group of this lane
          const int col = col0 + 4 * c4;
          if (c_remote == 4 && wk.c_vec_ok && col0 + 32 <= wk.n && row_in_op + 32 <= wk.m) {
            // exclusive writer: plain read-modify-write through the load/store
            // units (the TMA unit stays free for the producer's operand loads);
            // 8 independent 16-byte loads in flight per lane
            float4 cv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int rr = i * 4 + (lane >> 3);
              cv[i] = *reinterpret_cast<const float4*>(wk.c_ptr + (int64_t)(wk.c_row0 + row_in_op + rr) * wk.c_pitch +
                                                       wk.c_col0 + col);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int rr = i * 4 + (lane >> 3);
              const float4 v = ptx::ld_shared_v4f(base + rr * 128 + ((c4 ^ (rr & 7)) << 4));
              cv[i].x += v.x; cv[i].y += v.y; cv[i].z += v.z; cv[i].w += v.w;
              *reinterpret_cast<float4*>(wk.c_ptr + (int64_t)(wk.c_row0 + row_in_op + rr) * wk.c_pitch + wk.c_col0 +
                                         col) = cv[i];
            }
          } else
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = i * 4 + (lane >> 3);   // row within the warp's 32
            const int row = row_in_op + rr;
            float4 v = ptx::ld_shared_v4f(base + rr * 128 + ((c4 ^ (rr & 7)) << 4));
            if (row < wk.m && col < wk.n) {
              float* dst = wk.c_ptr + (int64_t)(wk.c_row0 + row) * wk.c_pitch + wk.c_col0 + col;
              if (wk.c_vec_ok && col + 4 <= wk.n) {
                ptx::red_add_v4_f32(dst, v.x, v.y, v.z, v.w);
              } else {
                ptx::red_add_f32(dst, v.x);
                if (col + 1 < wk.n) ptx::red_add_f32(dst + 1, v.y);
                if (col + 2 < wk.n) ptx::red_add_f32(dst + 2, v.z);
                if (col + 3 < wk.n) ptx::red_add_f32(dst + 3, v.w);
              }
            }
          }
          __syncwarp();
        }
        sbuf = (sbuf + 1) % C::EPI_BOXES;
      };
      // accumulator drained into registers: hand it back to the MMA warp
      auto release = [&](int j) {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          uint64_t* bar = &tmem_empty[C::NACC == 1 ? buf : j];
          if constexpr (CG == 1) ptx::mbar_arrive(bar);
          else ptx::mbar_arrive_cluster(bar, (uint32_t)(pair * CG));   // this pair's MMA issuer
        }
      };

#pragma unroll 1
      for (int j = 0; j < C::NACC; ++j) {
        // NACC == 1: one barrier per TMEM buffer; NACC == 2: one per accumulator
        ptx::mbar_wait(&tmem_full[C::NACC == 1 ? buf : j], tph);
        if (it == 0 && j == 0 && e == 0 && lane == 0) stamp(6);
        ptx::tc_fence_after();
        const uint32_t acc_col = (uint32_t)(buf * C::NACC + j) * C::UN;
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc_col;
        const int col_acc = nb * NT + j * C::UN;
        if constexpr (EW == 8) {
          // whole 128-column share in registers, TMEM released before any reduce
          uint32_t r[WCH][32];
#pragma unroll
          for (int c = 0; c < WCH; ++c) ptx::tmem_ld_32x32b_x32(taddr + (ch0 + c) * 32, r[c]);
          ptx::tmem_ld_wait();
          release(j);
#pragma unroll
          for (int c = 0; c < WCH; ++c) emit(r[c], col_acc + (ch0 + c) * 32);
        } else {
#pragma unroll 1
          for (int ch = 0; ch < CHUNKS; ++ch) {
            uint32_t r[32];
            ptx::tmem_ld_32x32b_x32(taddr + ch * 32, r);
            ptx::tmem_ld_wait();
            if (ch == CHUNKS - 1) release(j);
            emit(r, col_acc + ch * 32);
          }
        }
      }
      if (it == 0 && e == 0 && lane == 0) stamp(7);
      if (wk.slot >= 0) {
        // this warp's share of the tile is in C: complete its bulk writes, then
        // count it; the last arrival of the slot publishes the signal
        if (issuer) ptx::bulk_wait<0>();   // the bulk groups are the issuing lane's
        ptx::fence_proxy_async_global();
        __threadfence_system();
        __syncwarp();
        if (lane == 0) {
          const SignalSlot& sg = args.slots[wk.slot];
          if (atomicAdd(&args.counters[3 + MAX_GETS + wk.slot], 1) == sg.expected - 1) {
            __threadfence_system();
            ptx::red_release_sys_add_u32(sg.flag, sg.increment);
          }
        }
      }
    }
    if (issuer) ptx::bulk_wait<0>();
    if (e == 0 && lane == 0) stamp(8);
  } else if (args.ngets > 0) {
    // ===================== get engine (GET_WARPS warps per CTA) =====================
    // Pulls the launch's remote operand slices into local staging buffers while
    // the tensor cores work on ops whose operands are already here.  Chunks are
    // handed out in pull order (get_order: first need) from a global counter, so every resident CTA
    // helps and the first ops' operands land first.  No wait on anything but its
    // own loads: deadlock-free whatever the SMs are doing.
    int* const chunk_ctr = &args.counters[2];
    const uint64_t t_begin = ptx::globaltimer();
    int* const done = &args.counters[3];
    for (;;) {
      int c = 0;
      if (lane == 0) c = atomicAdd(chunk_ctr, 1);
      c = __shfl_sync(0xffffffffu, c, 0);
      if (c >= args.total_chunks) break;
      if (args.get_ns_per_chunk) {
        // profiling knob (UM_GET_GBPS): release chunk c no earlier than c chunk-times
        // after the launch, i.e. emulate a link of that bandwidth on one GPU
        const uint64_t due = t_begin + (uint64_t)c * args.get_ns_per_chunk;
        while (ptx::globaltimer() < due) __nanosleep(200);
      }
      int oi = 0;
      while (oi + 1 < args.ngets && args.gets[args.get_order[oi + 1]].chunk_start <= c) ++oi;
      const int j = args.get_order[oi];
      const GetDesc& g = args.gets[j];
      const int r0 = (c - g.chunk_start) * g.rows_per_chunk;
      const int r1 = min(g.rows, r0 + g.rows_per_chunk);
      constexpr int U = 16;  // 16-byte loads in flight per lane (4 warps: 32 KiB per SM)
      if (g.vec == 2) {
        // 32-byte rows: 256-bit loads / stores (half the instructions per byte
        // of the 16-byte path, twice the bytes in flight: 8 x 32 B per lane);
        // (row, column) advanced incrementally, no division per element
        constexpr int U2 = 8;
        const int n32 = g.row_bytes >> 5;
        const int total = (r1 - r0) * n32;
        int rr = lane / n32, cc = lane - rr * n32;
        for (int base = lane; base < total; base += 32 * U2) {
          uint32_t v[U2][8];
          int pr[U2], pc[U2];
#pragma unroll
          for (int u = 0; u < U2; ++u) {
            pr[u] = rr;
            pc[u] = cc;
            if (base + u * 32 < total) ptx::ld_nc_v8(g.src + (int64_t)(r0 + rr) * g.src_pitch + cc * 32, v[u]);
            cc += 32;
            while (cc >= n32) { cc -= n32; ++rr; }
          }
#pragma unroll
          for (int u = 0; u < U2; ++u)
            if (base + u * 32 < total) ptx::st_v8(g.dst + (int64_t)(r0 + pr[u]) * g.dst_pitch + pc[u] * 32, v[u]);
        }
      } else if (g.vec) {
        // flat (row, 16-byte column) walk of the chunk; the division by the row
        // width is a float reciprocal + one-step fix-up (exact: i < 2^24)
        const int n16 = g.row_bytes >> 4;
        const float inv = 1.0f / (float)n16;
        const int total = (r1 - r0) * n16;
        auto split = [&](int i, int& rr, int& cc) {
          rr = __float2int_rz((float)i * inv);
          cc = i - rr * n16;
          if (cc < 0) { --rr; cc += n16; } else if (cc >= n16) { ++rr; cc -= n16; }
        };
        for (int base = lane; base < total; base += 32 * U) {
          uint4 v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = base + u * 32;
            if (i < total) {
              int rr, cc;
              split(i, rr, cc);
              v[u] = ptx::ld_nc_v4(g.src + (int64_t)(r0 + rr) * g.src_pitch + cc * 16);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = base + u * 32;
            if (i < total) {
              int rr, cc;
              split(i, rr, cc);
              *reinterpret_cast<uint4*>(g.dst + (int64_t)(r0 + rr) * g.dst_pitch + cc * 16) = v[u];
            }
          }
        }
      } else {
        // unaligned rows (misaligned partitionings): 2-byte granules
        const int n2 = g.row_bytes >> 1;
        const int total = (r1 - r0) * n2;
        for (int i = lane; i < total; i += 32) {
          const int rr = i / n2, cc = i - rr * n2;
          *reinterpret_cast<uint16_t*>(g.dst + (int64_t)(r0 + rr) * g.dst_pitch + cc * 2) =
              *reinterpret_cast<const uint16_t*>(g.src + (int64_t)(r0 + rr) * g.src_pitch + cc * 2);
        }
      }
      ptx::fence_proxy_async_global();   // these generic writes precede later TMA (async-proxy) reads
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        atomicAdd(&done[j], 1);
#if UM_PROFILE
        if (args.prof && c < TL_CHUNKS) args.prof[TL_CHUNK_OFF + c] = ptx::globaltimer();
#endif
        if (c < MAX_CHUNK_FLAGS) ptx::st_release_gpu_s32(&args.counters[CHUNK_FLAGS_OFF + c], 1);
      }
    }
  }

  if (threadIdx.x == 0) stamp(9);
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<CG>(tmem_base, C::TMEM_COLS);
    if (lane == 0) stamp(10);
  }
  // Every warp of this CTA is done with the stream's get / completion-slot
  // counters and chunk flags: the last CTA out re-zeroes what this launch
  // used, so the next launch on the stream (stream order, or griddepcontrol.wait
  // under programmatic launch) finds them zero without a host memset.
  if (args.ngets > 0 || args.nslots > 0) {
    int* const ctr = args.counters;
    if (threadIdx.x == 0) {
      __threadfence();
      tq[0] = atomicAdd(&ctr[EXIT_OFF], 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (tq[0]) {
      __threadfence();
      const int nflags = min(args.total_chunks, MAX_CHUNK_FLAGS);
      for (int i = threadIdx.x; i < nflags; i += blockDim.x) ctr[CHUNK_FLAGS_OFF + i] = 0;
      for (int i = threadIdx.x; i < args.ngets; i += blockDim.x) ctr[3 + i] = 0;
      for (int i = threadIdx.x; i < args.nslots; i += blockDim.x) ctr[3 + MAX_GETS + i] = 0;
      if (threadIdx.x == 0) {
        ctr[2] = 0;
        ctr[EXIT_OFF] = 0;
      }
    }
  }
}

// ------------------------------------------------------------------ host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// L2 sector promotion of TMA loads: UM_GEMM_PROMO = 0 none | 1 64B | 2 128B | 3 256B (default none:
// measured 1459 vs 1427 TFLOP/s for 256B on cfg2, DRAM bytes unchanged)
static CUtensorMapL2promotion l2_promotion() {
  static int p = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = getenv("UM_GEMM_PROMO");
    p = (e && *e) ? atoi(e) : 0;
    if (p < 0 || p > 3) p = 0;
  });
  switch (p) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

static int encode_2d(CUtensorMap* map, const um_view& v, uint32_t box_cols, uint32_t box_rows, const char* what,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return fail(UM_ECUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  const CUtensorMapDataType dt = v.dtype == UM_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  cuuint64_t dims[2] = {(cuuint64_t)v.col_hi, (cuuint64_t)v.row_hi};
  cuuint64_t strides[1] = {(cuuint64_t)(v.pitch * esize(v.dtype))};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dt, 2, v.base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swz, l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(UM_ECUDA, std::string("cuTensorMapEncodeTiled failed for ") + what + " (code " +
                              std::to_string((int)r) + ")");
  return UM_OK;
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}

// Tuning knobs (read once): UM_GEMM_CG=1|2, UM_GEMM_NT=128|256|512 (0 = auto),
// UM_GEMM_GROUP=<m-tiles, negative: n-tiles>, UM_GEMM_APOL / UM_GEMM_BPOL
// = 0 normal | 1 evict_first | 2 evict_last (-1 = auto).
struct Knobs {
  int cg = 2, nt = 0, group = GROUP_M, apol = -1, bpol = -1, cpol = -1, prefetch = 0, sched_static = 0;
  int epi_warps = 4;
  int pairs = 1;
  int chain = 1;
  int chain_waves = 6;
  int pdl = 1;
  int pull_order = 1;
  int tail_split = 0;
  int cpf = 0;
  int stagger = 0;
  int skstart = 1;
  int splitk = 1;
  int smem_works = 1;   // short inline work lists read from a shared-memory copy (UM_GEMM_SMEM_WORKS=0: off)
};
static const Knobs& knobs() {
  static Knobs k;
  static std::once_flag once;
  std::call_once(once, [] {
#if UM_PROFILE || UM_VARIANTS
    // variants measured and rejected (cta_group::1, B multicast across pairs,
    // 8 epilogue warps) are instantiated in the profiling build only
    k.cg = env_int("UM_GEMM_CG", 2) == 1 ? 1 : 2;
#else
    k.cg = 2;
#endif
    k.nt = env_int("UM_GEMM_NT", 0);
    k.group = env_int("UM_GEMM_GROUP", GROUP_M);
    if (k.group == 0) k.group = GROUP_M;
    k.apol = env_int("UM_GEMM_APOL", -1);
    k.bpol = env_int("UM_GEMM_BPOL", -1);
    k.cpol = env_int("UM_GEMM_CPOL", -1);
    k.prefetch = std::max(0, env_int("UM_GEMM_PF", 0));
    k.sched_static = env_int("UM_GEMM_STATIC", 0) ? 1 : 0;
#if UM_PROFILE || UM_VARIANTS
    k.epi_warps = env_int("UM_GEMM_EPI_WARPS", 4) == 8 ? 8 : 4;
    k.pairs = env_int("UM_GEMM_PAIRS", 1);
    if (k.pairs != 2 && k.pairs != 4) k.pairs = 1;
#else
    k.epi_warps = 4;
    k.pairs = 1;
#endif
    k.chain = env_int("UM_GEMM_CHAIN", 1) ? 1 : 0;
    k.chain_waves = env_int("UM_GEMM_CHAIN_WAVES", 6);
    k.pdl = env_int("UM_GEMM_PDL", 1) ? 1 : 0;
    k.pull_order = env_int("UM_GEMM_PULL_ORDER", 1) ? 1 : 0;
    k.tail_split = env_int("UM_GEMM_TAIL_SPLIT", 0);
    k.cpf = std::max(0, env_int("UM_GEMM_CPF", 0));
    k.stagger = std::max(0, env_int("UM_GEMM_STAGGER", 0));
    k.skstart = env_int("UM_GEMM_SKSTART", 1) ? 1 : 0;
    k.splitk = env_int("UM_GEMM_SPLITK", 1) ? 1 : 0;
    k.smem_works = env_int("UM_GEMM_SMEM_WORKS", 1) ? 1 : 0;
  });
  return k;
}

// Per-(device, stream) scheduler counters (layout at EXIT_OFF): zeroed once at
// creation; the tile words are re-zeroed by the last pair to leave the tile
// scheduler and the get / slot words and chunk flags by the last CTA to exit,
// so launches on one stream (serialised) reuse them with no per-launch memset.
static int* stream_counters(int device, cudaStream_t stream) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, cudaStream_t>, int*>> table;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : table)
    if (e.first.first == device && e.first.second == stream) return e.second;
  int* p = nullptr;
  constexpr size_t bytes = (CHUNK_FLAGS_OFF + MAX_CHUNK_FLAGS) * sizeof(int);
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  // zero in stream order: torch's streams are non-blocking, so a plain
  // cudaMemset (legacy default stream) would race the first launch
  if (cudaMemsetAsync(p, 0, bytes, stream) != cudaSuccess) return nullptr;
  table.push_back({{device, stream}, p});
  return p;
}

static std::atomic<int> g_grid_limit[64];

static int grid_limit(int device) { return (device >= 0 && device < 64) ? g_grid_limit[device].load() : 0; }

template <int CG, int NT, int EW, int GW, int NP = 1>
static int launch(LaunchArgs& args, int device, cudaStream_t stream) {
  using C = Cfg<CG, NT, EW, GW>;
  const int total_tiles = args.total_tiles;
  static bool attr_set[64] = {false};
  if (device < 0 || device >= 64) return fail(UM_EVALUE, "device index out of range");
  if (!attr_set[device]) {
    UM_CUDA_CHECK(cudaFuncSetAttribute(gemm_bf16_kernel<CG, NT, EW, GW, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       C::SMEM_BYTES));
    attr_set[device] = true;
  }
  int sms = 0;
  UM_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  // the persistent grid, in CTA pairs (CG == 2) or CTAs: one per SM.  NP == 2
  // asks for clusters of 4 (two pairs sharing B by multicast) where a GPC has
  // room for them and falls back to plain pairs elsewhere (a GPC's SM count is
  // not a multiple of 4: clusters of 4 alone would leave ~16 of 148 SMs idle);
  // a lone pair runs the two halves of a 512-row tile in turn
  int units = sms / CG;
  const int tile_units = NP * total_tiles;
  // with in-kernel gets every SM joins (its get warps pull even when it gets no tile)
  if (args.ngets == 0) units = std::min(units, tile_units);
  // co-resident ranks share the device: cap each launch's persistent grid so
  // their launches (and the pulls inside them) run side by side
  const int cap = grid_limit(device);
  if (cap > 0) units = std::max(1, std::min(units, cap));
  // ops waiting on external arrival flags (copy-engine pulls): keep two CTA
  // pairs' SMs free, so the transfer always makes progress even where the
  // driver runs a copy on SMs rather than copy engines (a persistent grid
  // holding every SM would starve it: observed for same-device copies)
  if (args.ext_waits) units = std::max(1, std::min(units, sms / CG - 2));
  if (NP > 1) units = std::max(NP, units - units % NP);   // the grid must divide into big clusters
  static int occ[64] = {0};
  static const bool fixed = getenv("UM_GEMM_PAIRS_FIXED") && atoi(getenv("UM_GEMM_PAIRS_FIXED")) == 1;
  if (NP > 1 && !occ[device]) {
    // how many of the big clusters can be resident at once (A/B knob
    // UM_GEMM_PAIRS_FIXED=1 launches only big clusters, sized by this)
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(units * CG, 1, 1);
    q.blockDim = dim3(C::NUM_THREADS, 1, 1);
    q.dynamicSmemBytes = C::SMEM_BYTES;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = CG * NP;
    qa[0].val.clusterDim.y = 1;
    qa[0].val.clusterDim.z = 1;
    q.attrs = qa;
    q.numAttrs = 1;
    int n = -1;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, gemm_bf16_kernel<CG, NT, EW, GW, NP>, &q);
    if (args.prof) fprintf(stderr, "[um_gemm stalls] max resident clusters of %d: %d (%s)\n", CG * NP, n, cudaGetErrorString(e));
    cudaGetLastError();
    occ[device] = (e == cudaSuccess && n > 0) ? n : 1;
  }
  if (NP > 1 && fixed) units = std::min(units, occ[device] * NP);
  // staggered start over the first wave (one prefix per launched pair) only
  // where the last wave would otherwise leave > 10 % of the launch idle: the
  // split tiles cost an extra epilogue and pipeline refill each (measured on
  // one B200: 4096^3 +9 %, but 8192^3 -2 %, 16384^3 -3 %, 6144^3 -8 % when
  // applied everywhere; tools/k1_ab.py, profiles/r2_ab_skstart.json)
  {
    const int waves = (total_tiles + units - 1) / max(1, units);
    const double idle = waves > 0 ? 1.0 - (double)total_tiles / ((double)waves * units) : 0.0;
    args.nstag = (NP == 1 && args.stag_ok && !args.ext_waits && total_tiles > units && idle > 0.10) ? units : 0;
  }
  // split-k for launches with fewer tiles than pairs: each piece keeps >= 4
  // k-blocks (its mainloop then still covers the pipeline fill); the grid
  // grows to the pieces
  args.nsplit = 1;
  if (NP == 1 && args.stag_ok && !args.ext_waits && knobs().splitk && total_tiles < sms / CG) {
    int min_kb = 1 << 30;
    const Work* ws = args.works ? nullptr : args.inl_works;
    if (ws) for (int i = 0; i < args.nwork; ++i) min_kb = std::min(min_kb, ws[i].num_kb);
    const int s = ws ? std::min((sms / CG) / std::max(1, total_tiles), min_kb / 4) : 1;
    if (s >= 2) {
      args.nsplit = s;
      args.nstag = 0;
      units = std::min(sms / CG, total_tiles * s);
      if (cap > 0) units = std::max(1, std::min(units, cap));
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(units * CG, 1, 1);
  cfg.blockDim = dim3(C::NUM_THREADS, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[3];
  int na = 0;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = (NP > 1 && fixed) ? CG * NP : CG;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  if (NP > 1 && !fixed) {
    attr[na].id = cudaLaunchAttributePreferredClusterDimension;
    attr[na].val.preferredClusterDim.x = CG * NP;
    attr[na].val.preferredClusterDim.y = 1;
    attr[na].val.preferredClusterDim.z = 1;
    ++na;
  }
  // programmatic dependent launch (the kernel waits with griddepcontrol.wait
  // before its first global access): back-to-back launches overlap one's
  // setup with the previous one's drain.  UM_GEMM_PDL=0 turns it off.
  if (knobs().pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  UM_CUDA_CHECK(cudaLaunchKernelEx(&cfg, gemm_bf16_kernel<CG, NT, EW, GW, NP>, args));
  return UM_OK;
}

// TMA requires the innermost start coordinate of a box to be 16-byte aligned
// (measured: an unaligned column offset raises an illegal-instruction fault;
// row offsets are free), and a 16-byte aligned base and row pitch.  Slices of
// misaligned partitionings (e.g. 3x4 tiles, cli.py:151-152) therefore get
// their A/B slice staged into an aligned scratch and their C update routed
// through the pointer-based red.global epilogue.
static inline bool inner_aligned(const um_view& v) {
  const int64_t es = esize(v.dtype);
  return (v.col_lo * es) % 16 == 0 && (v.pitch * es) % 16 == 0 && (reinterpret_cast<uintptr_t>(v.base) & 15) == 0;
}
static inline int64_t aligned_pitch(int64_t cols, int32_t dtype) {
  const int64_t per16 = 16 / esize(dtype);
  return (cols + per16 - 1) / per16 * per16;
}

// Pick the kernel variant for a launch: 256x512 pair tiles when there is
// enough work for at least two waves of them, else 256x256 (or 128x256).
static void pick_variant(const std::vector<um_gemm_op>& ops, int sms, int& cg, int& nt) {
  const Knobs& kn = knobs();
  cg = kn.cg;
  if (cg == 1) {
    nt = 256;
    return;
  }
  if (kn.nt == 128 || kn.nt == 256 || kn.nt == 512) {
    nt = kn.nt;
    return;
  }
  // tiles per distinct C region (k-chains share their tiles), for both widths
  int64_t t512 = 0, t256 = 0;
  std::vector<const um_view*> seen;
  for (const auto& op : ops) {
    const int64_t m = view_rows(op.a), n = view_cols(op.b);
    if (!m || !n || !view_cols(op.a)) continue;
    if (kn.chain) {
      bool dup = false;
      for (const um_view* c : seen)
        if (c->base == op.c.base && c->row_lo == op.c.row_lo && c->col_lo == op.c.col_lo && c->row_hi == op.c.row_hi &&
            c->col_hi == op.c.col_hi && c->pitch == op.c.pitch) {
          dup = true;
          break;
        }
      if (dup) continue;
      seen.push_back(&op.c);
    }
    t512 += ((m + 255) / 256) * ((n + 511) / 512);
    t256 += ((m + 255) / 256) * ((n + 255) / 256);
  }
  // the wider tile moves ~25 % fewer operand bytes per flop and measured 7-14 %
  // faster per tile; only when there are too few tiles for two waves does the
  // narrower one win (measured: cfg5 p=8's 256 tiles still run best at 512).
  // A launch whose 256-wide tiles fill at most half the pairs is latency
  // bound, and its tail is the drain of each CTA's fp32 accumulator (one SM
  // moves ~25-45 B/clk of it into C, tools/debug/drain_probe.cu): 128-wide
  // tiles halve the drain per SM and spread it over twice the SMs
  const int64_t pairs = std::max(1, sms / 2);
  nt = t512 >= 2 * pairs ? 512 : (2 * t256 <= pairs ? 128 : 256);
}

// A launch with everything host-side resolved: tensor maps encoded, work
// list and get descriptors in the parameter block, misaligned operands'
// staging copies listed.  One-shot calls build, launch and drop it; the
// runtime keeps one per (rank, schedule) and replays it (um_gemm_prepare /
// um_gemm_launch), so a repeated multiply costs one launch call on the host.
struct StageCopy {
  void* dst;
  size_t dpitch;
  const void* src;
  size_t spitch, width, height;
};
struct Prepared {
  int device = 0, CG = 2, NT = 256, EW = 4, NP = 1, ngets = 0, nslots = 0;
  bool persistent = false, empty = true;
  void* scratch = nullptr;    // aligned copies of misaligned operand slices
  void* dbuf = nullptr;       // work list + tensor maps of > MAX_INLINE_OPS ops
  std::vector<StageCopy> copies;
  LaunchArgs args;
};

static void release(Prepared* P, cudaStream_t stream) {
  if (!P) return;
  if (P->persistent) {
    if (P->scratch) cudaFree(P->scratch);
    if (P->dbuf) cudaFree(P->dbuf);
  } else {
    if (P->scratch) cudaFreeAsync(P->scratch, stream);
    if (P->dbuf) cudaFreeAsync(P->dbuf, stream);
  }
  delete P;
}

// persistent: device-side buffers are cudaMalloc'd and filled synchronously
// (kept until um_gemm_destroy); else they are stream-ordered on `stream`.
static int prepare(const um_gemm_op* ops_in, int nops, const um_get_desc* gets_in, int ngets, int device,
                   bool persistent, cudaStream_t stream, Prepared* P) {
  if (ngets < 0 || ngets > MAX_GETS || (ngets > 0 && !gets_in))
    return fail(UM_EVALUE, "in-kernel get list must hold 0.." + std::to_string(MAX_GETS) + " entries");
  DeviceGuard guard(device);
  P->device = device;
  P->persistent = persistent;
  memset(&P->args, 0, sizeof(P->args));
  // ---- stage misaligned operand slices
  std::vector<um_gemm_op> ops(ops_in, ops_in + nops);
  size_t scratch_bytes = 0;
  for (auto& op : ops) {
    for (um_view* v : {&op.a, &op.b})
      if (!inner_aligned(*v) && view_rows(*v) > 0 && view_cols(*v) > 0)
        scratch_bytes += (size_t)(view_rows(*v) * aligned_pitch(view_cols(*v), v->dtype) * esize(v->dtype) + 256);
    if (!inner_aligned(op.c)) op.c_remote = 1;
    if (ngets < 64 && (op.get_mask >> ngets) != 0)
      return fail(UM_EVALUE, "op waits on an in-kernel get outside the launch's list");
    if (op.a_get < 0 || op.a_get > ngets || op.b_get < 0 || op.b_get > ngets)
      return fail(UM_EVALUE, "a_get / b_get name a get outside the launch's list");
    if ((op.a_get && !inner_aligned(op.a)) || (op.b_get && !inner_aligned(op.b)))
      return fail(UM_ECONTRACT, "an operand delivered by an in-kernel get must be TMA-aligned (16-byte column start)");
  }
  void* scratch = nullptr;
  if (scratch_bytes) {
    if (persistent) UM_CUDA_CHECK(cudaMalloc(&scratch, scratch_bytes));
    else UM_CUDA_CHECK(cudaMallocAsync(&scratch, scratch_bytes, stream));
    P->scratch = scratch;
    size_t off = 0;
    for (auto& op : ops)
      for (um_view* v : {&op.a, &op.b}) {
        if (inner_aligned(*v) || view_rows(*v) == 0 || view_cols(*v) == 0) continue;
        int rc;
        if ((rc = check_view(v, "operand", false))) return rc;
        um_view dst = {};
        dst.base = static_cast<char*>(scratch) + off;
        dst.row_lo = 0;
        dst.row_hi = view_rows(*v);
        dst.col_lo = 0;
        dst.col_hi = view_cols(*v);
        dst.pitch = aligned_pitch(view_cols(*v), v->dtype);
        dst.dtype = v->dtype;
        dst.device = device;
        const int64_t es = esize(v->dtype);
        P->copies.push_back({dst.base, (size_t)(dst.pitch * es),
                             static_cast<const char*>(v->base) + (v->row_lo * v->pitch + v->col_lo) * es,
                             (size_t)(v->pitch * es), (size_t)(view_cols(*v) * es), (size_t)view_rows(*v)});
        off += (size_t)(dst.row_hi * dst.pitch * es + 255) / 256 * 256;
        *v = dst;
      }
  }

  int sms = 0;
  UM_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  int CG = 2, NT = 256;
  pick_variant(ops, sms, CG, NT);
  const Knobs& kn = knobs();
  P->CG = CG;
  P->NT = NT;
  P->EW = (CG == 2 && kn.epi_warps == 8 && NT != 128) ? 8 : 4;
  // experimental: clusters of 2 pairs sharing B by TMA multicast (UM_GEMM_PAIRS=2)
  P->NP = (CG == 2 && NT == 512 && P->EW == 4) ? kn.pairs : 1;
  const int NPAIR = P->NP;

  std::vector<Work> works;
  std::vector<CUtensorMap> maps;
  works.reserve(nops);
  maps.reserve(3 * nops);
  int total = 0;
  // completion-signal slots: one per distinct done_flag
  std::vector<uint32_t*> slot_flags;
  std::vector<int> slot_expected;
  std::vector<uint32_t> slot_inc;
  for (int i = 0; i < nops; ++i) {
    uint32_t* f = ops[i].done_flag;
    if (!f) continue;
    auto it = std::find(slot_flags.begin(), slot_flags.end(), f);
    if (it == slot_flags.end()) {
      if ((reinterpret_cast<uintptr_t>(f) & 3) != 0) return fail(UM_EVALUE, "done_flag must be 4-byte aligned");
      slot_flags.push_back(f);
      slot_expected.push_back(0);
      slot_inc.push_back(ops[i].done_piece ? 0 : 1);
    } else if (!ops[i].done_piece) {
      ++slot_inc[it - slot_flags.begin()];
    }
  }
  if ((int)slot_flags.size() > MAX_SLOTS)
    return fail(UM_EVALUE, "more than " + std::to_string(MAX_SLOTS) + " distinct done_flags in one launch");
  const int epi_arrivals = (CG == 2 ? 2 : 1) * P->EW * NPAIR;
  for (int i = 0; i < nops; ++i) {
    const um_gemm_op& op = ops[i];
    if (op.c_remote && op.c.dtype == UM_F32 && (reinterpret_cast<uintptr_t>(op.c.base) & 3))
      return fail(UM_ECONTRACT, "fp32 C base must be 4-byte aligned");
    int rc;
    if ((rc = check_view(&op.a, "a", true)) || (rc = check_view(&op.b, "b", true)) ||
        (rc = check_view(&op.c, "c", !op.c_remote)))
      return rc;
    if (op.a.dtype != UM_BF16 || op.b.dtype != UM_BF16 || op.c.dtype != UM_F32)
      return fail(UM_ECONTRACT, "gemm expects bf16 A/B and fp32 C");
    const int64_t m = view_rows(op.a), k = view_cols(op.a), n = view_cols(op.b);
    if (view_rows(op.b) != k || view_rows(op.c) != m || view_cols(op.c) != n)
      return fail(UM_ECONTRACT, "gemm shape mismatch: a " + std::to_string(m) + "x" + std::to_string(k) + ", b " +
                                    std::to_string(view_rows(op.b)) + "x" + std::to_string(n) + ", c " +
                                    std::to_string(view_rows(op.c)) + "x" + std::to_string(view_cols(op.c)));
    if (m == 0 || n == 0 || k == 0) continue;  // c += 0
    if (op.a.row_hi > INT32_MAX || op.a.col_hi > INT32_MAX || op.b.row_hi > INT32_MAX ||
        op.b.col_hi > INT32_MAX || op.c.row_hi > INT32_MAX || op.c.col_hi > INT32_MAX)
      return fail(UM_EVALUE, "tile extent exceeds int32 TMA coordinates");
    Work w = {};
    w.m = (int32_t)m;
    w.n = (int32_t)n;
    w.k = (int32_t)k;
    w.tiles_m = (int32_t)((m + BM * CG * NPAIR - 1) / (BM * CG * NPAIR));
    w.tiles_n = (int32_t)((n + NT - 1) / NT);
    w.num_kb = (int32_t)((k + BK - 1) / BK);
    w.seg_kb = w.num_kb;
    w.nseg = 1;
    w.tile_start = total;
    w.c_remote = op.c_remote;
    if (!op.c_remote) {
      static const char* dbg = getenv("UM_GEMM_EPI_DEBUG");
      if (dbg && !strcmp(dbg, "red")) w.c_remote = 1;  // A/B: coalesced red.global epilogue for local C
#if UM_PROFILE
      // profiling build only (results not C += A.B): store|none replace the
      // reduce-add, rmw assumes an exclusive writer of each C tile
      if (dbg && !strcmp(dbg, "store")) w.c_remote = 2;
      if (dbg && !strcmp(dbg, "none")) w.c_remote = 3;
      if (dbg && !strcmp(dbg, "rmw")) w.c_remote = 4;
#endif
    }
    w.a_row0 = (int32_t)op.a.row_lo;
    w.a_col0 = (int32_t)op.a.col_lo;
    w.b_row0 = (int32_t)op.b.row_lo;
    w.b_col0 = (int32_t)op.b.col_lo;
    w.c_row0 = (int32_t)op.c.row_lo;
    w.c_col0 = (int32_t)op.c.col_lo;
    w.c_pitch = op.c.pitch;
    w.c_ptr = reinterpret_cast<float*>(op.c.base);
    w.wait_flag = op.wait_flag;
    w.wait_value = op.wait_value;
    w.wait_mask = op.get_mask;
    w.c_prefetch = kn.cpf;
    w.stagger = kn.stagger;
#if UM_PROFILE
    w.debug_halfb = env_int("UM_GEMM_DEBUG_HALFB", 0) ? 1 : 0;   // profiling build only: wrong results
    w.debug_mma = env_int("UM_GEMM_DEBUG_MMA", 0);                // profiling build only: wrong results
#else
    w.debug_halfb = 0;
    w.debug_mma = 0;
#endif
    w.a_fine = op.a_get;
    w.b_fine = op.b_get;
    w.group = kn.group;
    // L2 eviction hints default to normal: measured on the box, evict_last on
    // the group-reused operand + evict_first on the streamed one lowered the
    // sustained rate (1144 vs 1211 TFLOP/s at group 16); kept as knobs.
    w.a_pol = kn.apol >= 0 ? kn.apol : 0;   // auto: set below
    w.b_pol = kn.bpol >= 0 ? kn.bpol : 0;
    w.c_pol = kn.cpol >= 0 && kn.cpol <= 2 ? kn.cpol : -1;
    w.prefetch = kn.prefetch;
    w.sched_static = kn.sched_static;
    w.no_end_stagger = std::min(2, std::max(0, env_int("UM_GEMM_NO_END_STAGGER", 0)));
    if (w.a_pol > 2) w.a_pol = 0;
    if (w.b_pol > 2) w.b_pol = 0;
    w.c_vec_ok = ((reinterpret_cast<uintptr_t>(op.c.base) & 15) == 0) && (op.c.pitch % 4 == 0) && (op.c.col_lo % 4 == 0);
    total += w.tiles_m * w.tiles_n;
    w.slot = -1;
    if (op.done_flag)
      w.slot = (int)(std::find(slot_flags.begin(), slot_flags.end(), op.done_flag) - slot_flags.begin());
    CUtensorMap ma, mbm, mc;
    if ((rc = encode_2d(&ma, op.a, BK, BM, "A", BK == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B)) ||
        (rc = encode_2d(&mbm, op.b, 64, BK, "B")))
      return rc;
    if (!op.c_remote) {
      if ((rc = encode_2d(&mc, op.c, 32, 32, "C"))) return rc;
    } else {
      memset(&mc, 0, sizeof(mc));
    }
    works.push_back(w);
    maps.push_back(ma);
    maps.push_back(mbm);
    maps.push_back(mc);
  }
  // ---- k-chains: ops writing the same C region (Stationary C: the k-chunks of
  // one C tile) become one work whose segments accumulate in TMEM, so each
  // output tile is drained and reduced into C once instead of once per op
  if (kn.chain && works.size() > 1) {
    auto same_c = [](const Work& x, const Work& y) {
      return x.c_ptr == y.c_ptr && x.c_row0 == y.c_row0 && x.c_col0 == y.c_col0 && x.m == y.m && x.n == y.n &&
             x.c_pitch == y.c_pitch && x.c_remote == y.c_remote && x.slot == y.slot && x.c_pol == y.c_pol;
    };
    std::vector<std::vector<size_t>> groups;
    std::vector<char> used(works.size(), 0);
    for (size_t i = 0; i < works.size(); ++i) {
      if (used[i]) continue;
      std::vector<size_t> grp = {i};
      used[i] = 1;
      for (size_t j = i + 1; j < works.size(); ++j)
        if (!used[j] && same_c(works[i], works[j])) {
          grp.push_back(j);
          used[j] = 1;
        }
      groups.push_back(grp);
    }
    // long chains make long tiles: too few of them leave the last wave of the
    // persistent grid half empty (cfg5 p=8: 8 chains x 32 tiles of k = 16384
    // on 74 pairs = 3.5 waves of 0.2 ms).  Cap the chain length so the launch
    // has >= chain_waves x pairs tiles (sub-chains of one C region accumulate
    // into it with the same reduce-add).
    int max_len = 1;
    for (const auto& g : groups) max_len = std::max(max_len, (int)g.size());
    if (kn.chain_waves > 0) {
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
      const long target = (long)kn.chain_waves * (sms / CG);
      auto tiles_at = [&](int L) {
        long t = 0;
        for (const auto& g : groups)
          t += (long)works[g[0]].tiles_m * works[g[0]].tiles_n * (((int)g.size() + L - 1) / L);
        return t;
      };
      while (max_len > 1 && tiles_at(max_len) < target) max_len = (max_len + 1) / 2;
    }
    std::vector<Work> cw;
    std::vector<CUtensorMap> cm;
    int tot = 0;
    for (const auto& grp_all : groups)
      for (size_t s0 = 0; s0 < grp_all.size(); s0 += max_len) {
      const std::vector<size_t> grp(grp_all.begin() + s0, grp_all.begin() + std::min(grp_all.size(), s0 + max_len));
      const size_t i = grp[0];
      int kb = 0;
      for (size_t g : grp) kb += works[g].seg_kb;
      Work head = works[i];
      head.nseg = (int32_t)grp.size();
      head.num_kb = kb;
      head.tile_start = tot;
      tot += head.tiles_m * head.tiles_n;
      cw.push_back(head);
      for (int q = 0; q < 3; ++q) cm.push_back(maps[3 * i + q]);
      for (size_t g = 1; g < grp.size(); ++g) {
        Work c = works[grp[g]];
        c.nseg = 0;
        c.tile_start = tot;       // continuation: never the target of a tile index
        cw.push_back(c);
        for (int q = 0; q < 3; ++q) cm.push_back(maps[3 * grp[g] + q]);
      }
    }
    works.swap(cw);
    maps.swap(cm);
    total = tot;
  }
  // the last wave of a fused launch (whose tail waits for the last pull) runs
  // on short tiles: works issued last, about one wave of tiles, are split
  // along k -- a chain into its segments, a single op into the two halves of
  // its k range.  Every piece reduce-adds into C (an atomic C +=), so the
  // pieces need no ordering among themselves.
  if (ngets > 0 && kn.tail_split && !works.empty()) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const long wave = sms / CG;
    std::vector<char> split(works.size(), 0);
    long tail = 0;
    for (size_t i = works.size(); i-- > 0 && tail < wave;) {
      const Work& w = works[i];
      if (w.nseg == 0) continue;                       // continuation: handled with its head
      tail += (long)w.tiles_m * w.tiles_n;
      split[i] = w.nseg > 1 ? 2 : (w.num_kb >= 8 ? 1 : 0);
    }
    std::vector<Work> cw;
    std::vector<CUtensorMap> cm;
    int tot = 0;
    bool unchain = false;                              // inside a chain being split into its segments
    auto emit = [&](Work x, size_t src, bool head) {
      x.tile_start = tot;                              // continuation: the next head's start, never a target
      if (head) tot += x.tiles_m * x.tiles_n;
      cw.push_back(x);
      for (int q = 0; q < 3; ++q) cm.push_back(maps[3 * src + q]);
    };
    for (size_t i = 0; i < works.size(); ++i) {
      Work w = works[i];
      if (w.nseg > 0) unchain = split[i] == 2;
      if (split[i] == 1) {
        const int h = w.num_kb / 2;
        Work a = w, b = w;
        a.num_kb = a.seg_kb = h;
        b.num_kb = b.seg_kb = w.num_kb - h;
        b.a_col0 += h * BK;
        b.b_row0 += h * BK;
        emit(a, i, true);
        emit(b, i, true);
      } else if (unchain) {
        w.nseg = 1;                                    // every segment of the chain becomes a work
        w.num_kb = w.seg_kb;
        emit(w, i, true);
      } else {
        emit(w, i, w.nseg > 0);
      }
    }
    works.swap(cw);
    maps.swap(cm);
    total = tot;
  }
  // default L2 policies for a launch that is ONE large work on an unshared
  // device: A evict_first (each A panel is read by the 4 concurrent tiles of a
  // raster group, then done), B evict_last (a group's B panels are reused over
  // the whole m sweep).  cfg2: DRAM reads 8.25 -> 7.9 GB per launch, +2-3 % on
  // cfg2 / 16384^3 / cfg3 shapes in power-capped runs.  Multi-op launches and
  // ranks sharing a GPU keep evict_normal (A slices reused across ops: cfg5
  // p=8 co-resident -3 % with the hints).
  {
    int heads = 0;
    for (const Work& w : works) heads += w.nseg > 0;
    const bool streaming = heads == 1 && grid_limit(device) == 0;
    for (Work& w : works) {
      if (kn.apol < 0 && streaming) w.a_pol = 1;
      if (kn.bpol < 0 && streaming) w.b_pol = 2;
    }
  }
  // completion-signal arrivals: every epilogue warp of both CTAs, once per tile of each work head
  for (const Work& w : works)
    if (w.nseg > 0 && w.slot >= 0) slot_expected[w.slot] += w.tiles_m * w.tiles_n * epi_arrivals;
  LaunchArgs& args = P->args;
  args.nwork = (int)works.size();
  args.total_tiles = total;
  args.nslots = (int)slot_flags.size();
  args.ext_waits = 0;
  for (const Work& w : works) args.ext_waits |= w.wait_flag != nullptr;
  // staggered start (unit_span): plain launches only -- no in-kernel gets, no
  // completion slots (a split tile is written twice), no k-chains, and tiles
  // long enough (>= 8 k-blocks) that a prefix/remainder pair stays mainloop-bound
  {
    bool ok = kn.skstart && ngets == 0 && args.nslots == 0 && !works.empty();
    for (const Work& w : works) ok = ok && w.nseg == 1 && w.num_kb >= 8;
    args.stag_ok = ok ? 1 : 0;
  }
  for (int s = 0; s < args.nslots; ++s) args.slots[s] = {slot_flags[s], slot_expected[s], slot_inc[s]};
  // ---- in-kernel gets (fused K2)
  // Pull order: by the time the launch first needs each get.  The tiles are
  // list-scheduled on the CTA pairs in work order with no waits (a segment's
  // time ~ its k-blocks); a get's need time is the earliest start of a
  // segment that waits on it.  The first-use order of the work list would
  // pull the second segments of the first wave's tiles before the first
  // segments of later first-wave tiles (UM_GEMM_PULL_ORDER=0 keeps it).
  std::vector<int> gorder(std::max(0, ngets));
  for (int i = 0; i < ngets; ++i) gorder[i] = i;
  if (ngets > 1 && kn.pull_order) {
    std::vector<double> need_t(ngets, 1e300);
    int pairs = 148;
    cudaDeviceGetAttribute(&pairs, cudaDevAttrMultiProcessorCount, device);
    pairs = std::max(1, pairs / CG);
    if (grid_limit(device) > 0) pairs = std::max(1, std::min(pairs, grid_limit(device)));
    std::priority_queue<double, std::vector<double>, std::greater<double>> free_at;
    for (int q = 0; q < pairs; ++q) free_at.push(0.0);
    for (size_t h = 0; h < works.size(); ++h) {
      if (works[h].nseg <= 0) continue;
      const long ntiles = (long)works[h].tiles_m * works[h].tiles_n;
      for (long tl = 0; tl < ntiles; ++tl) {
        double tt = free_at.top();
        free_at.pop();
        for (size_t w = h; w < h + (size_t)works[h].nseg && w < works.size(); ++w) {
          const Work& x = works[w];
          auto use = [&](int g) { if (g >= 0 && g < ngets) need_t[g] = std::min(need_t[g], tt); };
          use(x.a_fine - 1);
          use(x.b_fine - 1);
          for (int g = 0; g < ngets && g < 64; ++g)
            if ((x.wait_mask >> g) & 1ull) use(g);
          tt += (double)std::max(1, x.seg_kb);
        }
        free_at.push(tt);
      }
    }
    std::stable_sort(gorder.begin(), gorder.end(), [&](int a, int b) { return need_t[a] < need_t[b]; });
  }
  for (int i = 0; i < ngets; ++i) args.get_order[i] = gorder[i];
  int chunks = 0;
  for (int i = 0; i < ngets; ++i) {
    const um_get_desc& gd = gets_in[i];
    int rc;
    if ((rc = check_view(&gd.src, "get src", false)) || (rc = check_view(&gd.dst, "get dst", false))) return rc;
    if (gd.src.dtype != gd.dst.dtype || view_rows(gd.src) != view_rows(gd.dst) || view_cols(gd.src) != view_cols(gd.dst))
      return fail(UM_ECONTRACT, "get: src and dst slices differ in dtype or shape");
    const int64_t es = esize(gd.src.dtype);
    GetDesc& g = args.gets[i];
    g.src = static_cast<const uint8_t*>(gd.src.base) + (gd.src.row_lo * gd.src.pitch + gd.src.col_lo) * es;
    g.dst = static_cast<uint8_t*>(gd.dst.base) + (gd.dst.row_lo * gd.dst.pitch + gd.dst.col_lo) * es;
    g.src_pitch = gd.src.pitch * es;
    g.dst_pitch = gd.dst.pitch * es;
    if (view_rows(gd.src) > INT32_MAX || view_cols(gd.src) * es > INT32_MAX)
      return fail(UM_EVALUE, "get slice too large");
    g.rows = (int32_t)view_rows(gd.src);
    g.row_bytes = (int32_t)(view_cols(gd.src) * es);
    g.rows_per_chunk = std::max(1, GET_CHUNK_BYTES / std::max(1, g.row_bytes));
    g.nchunks = g.rows && g.row_bytes ? (g.rows + g.rows_per_chunk - 1) / g.rows_per_chunk : 0;
    g.row0 = (int32_t)gd.dst.row_lo;
    {
      const uintptr_t al = reinterpret_cast<uintptr_t>(g.src) | reinterpret_cast<uintptr_t>(g.dst) |
                           (uintptr_t)g.src_pitch | (uintptr_t)g.dst_pitch | (uintptr_t)g.row_bytes;
      // 2: 32-byte rows (256-bit loads / stores), 1: 16-byte rows, 0: 2-byte granules.
      // The 256-bit path is used only for sources in this device's own memory
      // (measured here); peer / IPC-mapped sources (NVLink) keep 16-byte loads.
      bool local_src = false;
      cudaPointerAttributes pa = {};
      if (cudaPointerGetAttributes(&pa, g.src) == cudaSuccess)
        local_src = pa.type == cudaMemoryTypeDevice && pa.device == device;
      cudaGetLastError();
      g.vec = ((al & 31) == 0 && local_src) ? 2 : (al & 15) == 0 ? 1 : 0;
    }
  }
  for (int oi = 0; oi < ngets; ++oi) {   // chunk ranges in pull order
    GetDesc& g = args.gets[gorder[oi]];
    g.chunk_start = chunks;
    chunks += g.nchunks;
  }
  args.ngets = ngets;
  args.total_chunks = chunks;
  if (chunks > MAX_CHUNK_FLAGS)   // too many chunks for per-chunk flags: whole-band waits instead
    for (Work& w : works) {
      if (w.a_fine) w.wait_mask |= 1ull << (w.a_fine - 1);
      if (w.b_fine) w.wait_mask |= 1ull << (w.b_fine - 1);
      w.a_fine = w.b_fine = 0;
    }
  // UM_GET_GBPS=<GB/s>: pace the in-kernel pulls to that rate (profiling: a
  // one-GPU run with pulls at NVLink speed)
  static const double get_gbps = [] {
    const char* e = getenv("UM_GET_GBPS");
    return (e && *e) ? atof(e) : 0.0;
  }();
  args.get_ns_per_chunk = get_gbps > 0 ? (uint32_t)(GET_CHUNK_BYTES / get_gbps + 0.5) : 0u;
  P->ngets = ngets;
  P->nslots = args.nslots;
  // gets only / signals only: still one launch (get warps; slots with no tile
  // are signalled at kernel start)
  P->empty = total == 0 && ngets == 0 && args.nslots == 0;
  void* dbuf = nullptr;
  // UM_GEMM_MAPS_GLOBAL=1 (A/B knob): work list + tensor maps in a global
  // buffer even for short lists (tests whether the first TMA's descriptor
  // fetch from the parameter bank delays small launches)
  static const bool maps_global = env_int("UM_GEMM_MAPS_GLOBAL", 0) != 0;
  if (works.size() <= (size_t)MAX_INLINE_OPS && !maps_global) {
    memcpy(args.inl_maps, maps.data(), maps.size() * sizeof(CUtensorMap));
    memcpy(args.inl_works, works.data(), works.size() * sizeof(Work));
    // (launches waiting on copy-engine arrival flags keep the parameter-block
    // list: with the shared-memory copy they hung under compute-sanitizer
    // racecheck, which serialises the device; plain, memcheck and synccheck
    // runs pass either way -- profiles/r2_sanitizer.md, session 4)
    args.smem_works = knobs().smem_works && works.size() <= (size_t)SMEM_WORKS && !args.ext_waits ? 1 : 0;
  } else {
    // large op lists: one stream-ordered allocation carries work list + tensor maps
    args.smem_works = 0;
    const size_t maps_bytes = maps.size() * sizeof(CUtensorMap);
    const size_t works_bytes = works.size() * sizeof(Work);
    std::vector<uint8_t> host(maps_bytes + works_bytes);
    memcpy(host.data(), maps.data(), maps_bytes);
    memcpy(host.data() + maps_bytes, works.data(), works_bytes);
    if (persistent) {
      UM_CUDA_CHECK(cudaMalloc(&dbuf, host.size()));
      P->dbuf = dbuf;
      UM_CUDA_CHECK(cudaMemcpy(dbuf, host.data(), host.size(), cudaMemcpyHostToDevice));
    } else {
      UM_CUDA_CHECK(cudaMallocAsync(&dbuf, host.size(), stream));
      P->dbuf = dbuf;
      UM_CUDA_CHECK(cudaMemcpyAsync(dbuf, host.data(), host.size(), cudaMemcpyHostToDevice, stream));
    }
    args.maps = reinterpret_cast<const CUtensorMap*>(dbuf);
    args.works = reinterpret_cast<const Work*>(reinterpret_cast<uint8_t*>(dbuf) + maps_bytes);
  }
  return UM_OK;
}

static int launch_prepared(Prepared* P, cudaStream_t stream) {
  if (P->empty) return UM_OK;
  DeviceGuard guard(P->device);
  for (const StageCopy& c : P->copies)
    UM_CUDA_CHECK(cudaMemcpy2DAsync(c.dst, c.dpitch, c.src, c.spitch, c.width, c.height, cudaMemcpyDefault, stream));
  LaunchArgs& args = P->args;
  // zero at creation and re-zeroed by the last CTA of every launch (kernel exit)
  args.counters = stream_counters(P->device, stream);
  if (!args.counters) return fail(UM_ECUDA, "could not allocate the scheduler counters");
  // profiling (UM_GEMM_STALLS=1): MMA-thread stall breakdown, synchronous, printed to stderr
  static const bool stalls = env_int("UM_GEMM_STALLS", 0) != 0;
  unsigned long long* prof = nullptr;
  if (stalls) {
    UM_CUDA_CHECK(cudaMallocAsync(&prof, PROF_WORDS * sizeof(unsigned long long), stream));
    UM_CUDA_CHECK(cudaMemsetAsync(prof, 0, PROF_WORDS * sizeof(unsigned long long), stream));
  }
  args.prof = prof;
  int rc;
  const bool g = P->ngets > 0;
#if UM_PROFILE || UM_VARIANTS
  if (P->CG == 1) rc = g ? launch<1, 256, 4, GET_WARPS>(args, P->device, stream) : launch<1, 256, 4, 0>(args, P->device, stream);
  else if (P->NT == 512 && P->NP == 2)
    rc = g ? launch<2, 512, 4, GET_WARPS, 2>(args, P->device, stream) : launch<2, 512, 4, 0, 2>(args, P->device, stream);
  else if (P->NT == 512 && P->NP == 4)
    rc = g ? launch<2, 512, 4, GET_WARPS, 4>(args, P->device, stream) : launch<2, 512, 4, 0, 4>(args, P->device, stream);
  else if (P->NT == 512 && P->EW == 8)
    rc = g ? launch<2, 512, 8, GET_WARPS>(args, P->device, stream) : launch<2, 512, 8, 0>(args, P->device, stream);
  else if (P->EW == 8 && P->NT != 512)
    rc = g ? launch<2, 256, 8, GET_WARPS>(args, P->device, stream) : launch<2, 256, 8, 0>(args, P->device, stream);
  else
#endif
  if (P->NT == 512)
    rc = g ? launch<2, 512, 4, GET_WARPS>(args, P->device, stream) : launch<2, 512, 4, 0>(args, P->device, stream);
  else if (P->NT == 128)
    rc = g ? launch<2, 128, 4, GET_WARPS>(args, P->device, stream) : launch<2, 128, 4, 0>(args, P->device, stream);
  else
    rc = g ? launch<2, 256, 4, GET_WARPS>(args, P->device, stream) : launch<2, 256, 4, 0>(args, P->device, stream);
  args.prof = nullptr;
  if (prof) {
    std::vector<unsigned long long> h(PROF_WORDS);
    cudaMemcpyAsync(h.data(), prof, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    cudaFreeAsync(prof, stream);
    double tot = 0, full = 0, tmem = 0, tile = 0;
    int n = 0, n4 = 0;
    for (int c = 0; c < TRACE_OFF / 4; ++c)
      if (h[4 * c]) {
        const unsigned long long t3 = h[4 * c + 3] & ((1ull << 56) - 1);
        tot += h[4 * c]; full += h[4 * c + 1]; tmem += h[4 * c + 2]; tile += t3; ++n;
        n4 += (h[4 * c + 3] >> 56) > 2;
      }
    if (const char* tl = getenv("UM_GEMM_TIMELINE")) {
      // append this launch's tile spans and chunk landings, ns after its first event
      static int launch_no = 0;
      unsigned long long t0 = ~0ull;
      for (int i = 0; i < 128 * TL_TILES; ++i)
        if (h[TL_OFF + 3 * i]) t0 = std::min(t0, h[TL_OFF + 3 * i + 1]);
      for (int c = 0; c < TL_CHUNKS; ++c)
        if (h[TL_CHUNK_OFF + c]) t0 = std::min(t0, h[TL_CHUNK_OFF + c]);
      if (FILE* f = fopen(tl, launch_no == 0 ? "w" : "a")) {
        if (launch_no == 0) fprintf(f, "launch,kind,pair,index,id,start_ns,end_ns\n");
        for (int pr = 0; pr < 128; ++pr)
          for (int i = 0; i < TL_TILES; ++i) {
            const unsigned long long* e = &h[TL_OFF + (pr * TL_TILES + i) * 3];
            if (e[0])
              fprintf(f, "%d,tile,%d,%d,%llu,%llu,%llu\n", launch_no, pr, i, e[0] - 1, e[1] - t0,
                      e[2] ? e[2] - t0 : 0ull);
          }
        for (int c = 0; c < TL_CHUNKS; ++c)
          if (h[TL_CHUNK_OFF + c])
            fprintf(f, "%d,chunk,-1,%d,%d,%llu,%llu\n", launch_no, c, c, h[TL_CHUNK_OFF + c] - t0,
                    h[TL_CHUNK_OFF + c] - t0);
        // CTA b's first unit: loads issued for k-block kb (index kb), A rows landed (index -1)
        for (int b = 0; b < 2; ++b)
          for (int kb = 0; kb <= KB_MAX; ++kb) {
            const unsigned long long v = h[KB_OFF + b * (KB_MAX + 1) + kb];
            if (v && v >= t0)
              fprintf(f, "%d,kb,%d,%d,%d,%llu,%llu\n", launch_no, b, kb == KB_MAX ? -1 : kb, b, v - t0, v - t0);
          }
        fclose(f);
      }
      ++launch_no;
    }
    if (h[TRACE_OFF]) {
      fprintf(stderr, "[um_gemm stalls] block 0 timeline (us after entry): setup %.2f, first tile %.2f, first loads "
                      "issued %.2f, first operands landed %.2f, first tile's MMAs committed %.2f, epilogue got TMEM "
                      "%.2f, epilogue issued C %.2f, C writes complete %.2f, loops done %.2f, exit %.2f\n",
              (h[TRACE_OFF + 1] - h[TRACE_OFF]) * 1e-3, (h[TRACE_OFF + 2] - h[TRACE_OFF]) * 1e-3,
              (h[TRACE_OFF + 3] - h[TRACE_OFF]) * 1e-3, (h[TRACE_OFF + 4] - h[TRACE_OFF]) * 1e-3,
              (h[TRACE_OFF + 5] - h[TRACE_OFF]) * 1e-3, (h[TRACE_OFF + 6] - h[TRACE_OFF]) * 1e-3,
              (h[TRACE_OFF + 7] - h[TRACE_OFF]) * 1e-3, (h[TRACE_OFF + 8] - h[TRACE_OFF]) * 1e-3,
              (h[TRACE_OFF + 9] - h[TRACE_OFF]) * 1e-3, (h[TRACE_OFF + 10] - h[TRACE_OFF]) * 1e-3);
      fprintf(stderr, "[um_gemm stalls] block 0 producer (us): tile-queue slot free %.2f, unit taken %.2f, coordinates "
                      "%.2f, segment set up %.2f\n", (h[TRACE_OFF + 11] - h[TRACE_OFF]) * 1e-3,
              (h[TRACE_OFF + 12] - h[TRACE_OFF]) * 1e-3, (h[TRACE_OFF + 13] - h[TRACE_OFF]) * 1e-3,
              (h[TRACE_OFF + 14] - h[TRACE_OFF]) * 1e-3);
    }
    {
      double pt = 0, pe = 0, pi = 0, ptm = 0, pl = 0, ls = 0, lc = 0, lm = 0;
      int np_ = 0;
      for (int b = 0; b < 160; ++b) {
        const unsigned long long* e = &h[PS_OFF + PS_WORDS * b];
        if (e[0]) { pt += e[0]; pe += e[1]; pi += e[5]; ptm += e[6]; pl += e[7]; ++np_; }
        if (e[3]) { ls += e[2]; lc += e[3]; lm = std::max(lm, (double)e[4]); }
      }
      if (np_ && lc)
        fprintf(stderr, "[um_gemm stalls] producers wait for a free stage %.1f %% and issue loads %.1f %% of their "
                        "cycles (of which the TMA instructions %.1f %%; the k-block loops %.1f %%); operand load latency "
                        "(leader issue -> stage full) mean %.0f, max %.0f cycles over %.0f stages\n",
                100 * pe / pt, 100 * pi / pt, 100 * ptm / pt, 100 * pl / pt, ls / lc, lm, lc);
    }
    if (n)
      fprintf(stderr, "[um_gemm stalls] %d pairs (%d in clusters > 2), MMA thread: waiting for operands %.1f %%, for TMEM (epilogue) "
                      "%.1f %%, for the next tile %.1f %% of %.0f cycles\n", n, n4, 100 * full / tot, 100 * tmem / tot,
              100 * tile / tot, tot / n);
  }
  return rc;
}

int launch_batch(const um_gemm_op* ops, int nops, const um_get_desc* gets, int ngets, int device,
                 cudaStream_t stream) {
  // A one-shot launch keeps its work list in the kernel's parameter block: a
  // longer op list without in-kernel gets runs as consecutive launches of at
  // most MAX_INLINE_OPS ops (stream order keeps C += exact).  The descriptor
  // block of a longer list would otherwise be a device buffer filled from a
  // stack-local host vector, which a CUDA-graph capture cannot record safely.
  if (nops > MAX_INLINE_OPS && ngets == 0) {
    for (int i = 0; i < nops; i += MAX_INLINE_OPS) {
      int rc = launch_batch(ops + i, std::min(MAX_INLINE_OPS, nops - i), nullptr, 0, device, stream);
      if (rc != UM_OK) return rc;
    }
    return UM_OK;
  }
  if (nops > MAX_INLINE_OPS) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    UM_CUDA_CHECK(cudaStreamIsCapturing(stream, &cs));
    if (cs != cudaStreamCaptureStatusNone)
      return fail(UM_ECONTRACT, "a captured one-shot fused launch holds at most " + std::to_string(MAX_INLINE_OPS) +
                                    " ops (use um_gemm_prepare for longer lists)");
  }
  Prepared* P = new Prepared();
  int rc = prepare(ops, nops, gets, ngets, device, false, stream, P);
  if (rc == UM_OK) rc = launch_prepared(P, stream);
  release(P, stream);
  return rc;
}

}  // namespace gemm
}  // namespace um

extern "C" int um_gemm_acc(const um_view* a, const um_view* b, const um_view* c, void* stream) {
  if (!a || !b || !c) return um::fail(UM_EVALUE, "null view");
  um_gemm_op op = {};
  op.a = *a;
  op.b = *b;
  op.c = *c;
  op.c_remote = 0;
  return um::gemm::launch_batch(&op, 1, nullptr, 0, c->device, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int um_gemm_acc_batch(const um_gemm_op* ops, int32_t nops, int32_t device, void* stream) {
  if (nops < 0 || (nops > 0 && !ops)) return um::fail(UM_EVALUE, "bad op list");
  return um::gemm::launch_batch(ops, nops, nullptr, 0, device, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int um_gemm_acc_fused(const um_gemm_op* ops, int32_t nops, const um_get_desc* gets, int32_t ngets,
                                 int32_t device, void* stream) {
  if (nops < 0 || (nops > 0 && !ops)) return um::fail(UM_EVALUE, "bad op list");
  return um::gemm::launch_batch(ops, nops, gets, ngets, device, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int um_gemm_prepare(const um_gemm_op* ops, int32_t nops, const um_get_desc* gets, int32_t ngets,
                               int32_t device, void** handle) {
  if (!handle) return um::fail(UM_EVALUE, "null handle pointer");
  if (nops < 0 || (nops > 0 && !ops)) return um::fail(UM_EVALUE, "bad op list");
  auto* P = new um::gemm::Prepared();
  int rc = um::gemm::prepare(ops, nops, gets, ngets, device, true, nullptr, P);
  if (rc != UM_OK) {
    um::gemm::release(P, nullptr);
    *handle = nullptr;
    return rc;
  }
  *handle = P;
  return UM_OK;
}

extern "C" int um_gemm_launch(void* handle, void* stream) {
  if (!handle) return um::fail(UM_EVALUE, "null launch handle");
  return um::gemm::launch_prepared(static_cast<um::gemm::Prepared*>(handle), reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int um_gemm_destroy(void* handle) {
  if (handle) {
    auto* P = static_cast<um::gemm::Prepared*>(handle);
    um::DeviceGuard guard(P->device);
    if (P->scratch || P->dbuf) cudaDeviceSynchronize();   // buffers may still be read by a launch
    um::gemm::release(P, nullptr);
  }
  return UM_OK;
}

extern "C" int um_gemm_set_grid_limit(int32_t device, int32_t max_clusters) {
  if (device < 0 || device >= 64) return um::fail(UM_EVALUE, "device index out of range");
  um::gemm::g_grid_limit[device].store(std::max(0, max_clusters));
  return UM_OK;
}

extern "C" int um_gemm_config(int32_t* bm, int32_t* bn, int32_t* bk, int32_t* stages, int32_t* cta_group) {
  const auto& kn = um::gemm::knobs();
  const int cg = kn.cg;
  const int nt = cg == 1 ? 256 : (kn.nt == 256 ? 256 : 512);
  if (bm) *bm = um::gemm::BM * cg;
  if (bn) *bn = nt;
  if (bk) *bk = um::gemm::BK;
  if (stages) *stages = cg == 1 ? um::gemm::Cfg<1, 256>::STAGES
                                : (nt == 512 ? um::gemm::Cfg<2, 512>::STAGES : um::gemm::Cfg<2, 256>::STAGES);
  if (cta_group) *cta_group = cg;
  return UM_OK;
}
