/*
 * include/guardian.h -- C ABI of libguardian.so, a B200-native (sm_100a)
 * implementation of Guardian's per-access address fencing
 * (Guardian: Safe GPU Sharing in Multi-Tenant Environments, arXiv 2401.09290).
 *
 * Citations: PAPER.md:<line> (§section / Listing / Table); SPEC.md:<line>;
 * SURVEY.md §8 rows (a1..a11) and readings (A1..A16).  DESIGN.md holds the
 * full design and the readings of the paper this library follows.
 *
 * Conventions (all entry points):
 *  - extern "C"; every call returns gd_status; out-parameters come last.
 *  - Device addresses are uint64_t; host buffers are plain pointers.
 *  - `stream` is a cudaStream_t / CUstream handle owned by the caller
 *    (e.g. torch.cuda.Stream().cuda_stream); NULL is the legacy default stream.
 *  - Launches are asynchronous on `stream`.  gd_stats() synchronises.
 *  - Structural errors (unknown tenant, bad mode, misaligned pointer, an
 *    unsupported shape, size overflow) are returned BEFORE any launch and no
 *    work is done.  Launchers do NOT range-check pointer arguments: the
 *    device fence does that (PAPER.md:171 checks host transfers on the host,
 *    PAPER.md:230 fences kernel accesses on the device).
 *  - Asynchronous CUDA faults surface as GD_ERR_CUDA at the next synchronising
 *    call; gd_last_cuda_error() returns the cudaError_t behind GD_ERR_CUDA.
 *  - n = 0 launches are GD_OK and do nothing.
 *  - Size limits (GD_ERR_INVALID_ARG beyond them; every grid stays below
 *    2^31 CTAs): copy n <= 2^44 bytes; saxpy, scatter n <= 2^42 elements;
 *    gather n * row_elems <= 2^41; stencil H * pitch <= 2^58 floats, and
 *    the LSU stencil H <= 2^19 rows (GD_ERR_UNSUPPORTED; the TMA stencil has
 *    no such limit).
 *  - Thread safety: arena mutations (partition alloc/free, malloc/free) are
 *    serialised by an internal mutex; launches read an immutable snapshot of
 *    the partition bounds entry and may be issued from several threads.
 *    Partition alloc/free wait until no launch, checked transfer, fill or
 *    graph replay is between its bounds snapshot and its enqueue, and free
 *    synchronises the device before it unmaps: work is never enqueued with
 *    bounds of a partition that no longer exists.
 */
#ifndef GUARDIAN_H
#define GUARDIAN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GD_OK = 0,
    GD_ERR_INVALID_ARG = 1,
    GD_ERR_NOT_POW2 = 2,           /* arena size not a power of two     */
    GD_ERR_DEVICE_OOM = 3,         /* no free buddy block / no device memory (SPEC DeviceOom) */
    GD_ERR_PARTITION_OOM = 4,      /* gd_malloc: partition full (SPEC PartitionOom)     */
    GD_ERR_UNKNOWN_PARTITION = 5,  /* no such tenant id (SPEC UnknownApp)               */
    GD_ERR_UNKNOWN_ALLOC = 6,      /* gd_free of an address that is not a live allocation */
    GD_ERR_ALIGN = 7,              /* pointer misaligned for the kernel's access width  */
    GD_ERR_OOB_RANGE = 8,          /* host transfer outside the partition (SPEC OOB_TRANSFER) */
    GD_ERR_UNSUPPORTED = 9,        /* shape/arena a kernel cannot take                 */
    GD_ERR_CUDA = 10               /* a CUDA runtime/driver call failed                */
} gd_status;

/* Fence modes, chosen per launch at run time ("can be
 * dynamically utilized at runtime").
 *  NONE  : the native kernel ("issues a native kernel") -- the
 *          unfenced twin every overhead is measured against.
 *  MASK  : address fencing, fenced = (addr & mask_w) | base, with
 *          mask_w = (size-1) & ~(w-1) for a w-byte access (Listing 1 lines
 *          26-28; reading A3).  Out-of-partition addresses
 *          wrap into the own partition; nothing is detected.
 *  CHECK : address checking: an access is allowed iff its
 *          w bytes lie in [base, base+size) and it is w-aligned; a refused
 *          load reads 0, a refused store / atomic is dropped, and the
 *          tenant's violation counter is incremented (reading A1).
 *  MODULO: address fencing with modulo (§4.4), fenced =
 *          base + (((addr - base) mod size) & ~(w-1)), the 64-bit modulo
 *          inline with the reciprocal parameter floor(2^64/size) ("an extra
 *          parameter holding the 1/partition_size").  Needs no
 *          alignment and no power-of-two size: it is the mode for exact-size
 *          partitions (gd_partition_alloc_exact).  Nothing is detected.
 *  MASK_COUNT: MASK plus detection ("an optional
 *          GD_FLAG_COUNT adds detection"): every access goes where MASK puts
 *          it, and each access CHECK would refuse is counted.
 *  CLAMP : north_star's check mode "compare, clamp and set a violation flag"
 *          (reading A1's saturating variant): the access goes to the largest
 *          w-aligned address of the partition at or below it (the base when
 *          there is none) and each access CHECK would refuse is counted.
 *          Every out-of-partition store lands on an edge word, so results
 *          are deterministic only on inputs whose clamped stores do not
 *          collide (reading R-race).
 *  MASK and MASK_COUNT require a power-of-two, size-aligned partition
 *  (GD_ERR_NOT_POW2 otherwise); the others take any partition.
 *  Counted accesses (CHECK, MASK_COUNT, CLAMP) are equal in number for the
 *  same launch: one per logical access outside the partition.               */
typedef enum {
    GD_MODE_NONE = 0, GD_MODE_MASK = 1, GD_MODE_CHECK = 2, GD_MODE_MODULO = 3,
    GD_MODE_MASK_COUNT = 4, GD_MODE_CLAMP = 5
} gd_mode;

/* Per-access flag, OR-ed into the mode of any launch (gd_launch_fenced_*,
 * gd_work.mode): fence every access one by one, as the paper's instrumented
 * kernels do ("before every load and store"; §4.3), instead of
 * the default hoisting: a CHECK / MODULO / MASK_COUNT / CLAMP launch of copy,
 * saxpy or stencil v1 whose whole footprint lies in the partition runs the
 * unfenced twin (decided on the host from the launch's bounds snapshot,
 * DESIGN.md reading R-hoist-launch), and inside other launches a tile-level
 * range test runs the unfenced body on tiles wholly inside the partition
 * (reading R-hoist).  Results and
 * violation counts are identical either way; only the cost differs.  The
 * descriptor-fenced TMA kernels (GEMM, K5 v2) have no per-access fence and
 * ignore it; MASK is always per access.  Setting GD_CHECK_PER_ACCESS=1 in the
 * environment forces it for every launch of the process.  Any other bit
 * above the mode is GD_ERR_INVALID_ARG.                                      */
#define GD_FENCE_PER_ACCESS 0x100u

/* Kernel kinds (index of the per-kind statistics).                            */
typedef enum {
    GD_KIND_COPY = 0, GD_KIND_SAXPY = 1, GD_KIND_GATHER = 2,
    GD_KIND_SCATTER = 3, GD_KIND_STENCIL = 4, GD_KIND_GEMM = 5,
    GD_NUM_KINDS = 6
} gd_kind;

#define GD_MAX_TENANTS 64u
#define GD_ALL_TENANTS 0xFFFFFFFFu
#define GD_MIN_PARTITION 4096u        /* SPEC.md:217 minimum partition size     */

/* gd_arena_create flags */
#define GD_ARENA_VMM 0u               /* default: CUDA VMM reservation aligned to its size */

typedef struct gd_arena gd_arena;     /* opaque, library-owned */

/* One row of the partition bounds table ("the application id,
 * the base address, and the partition size"); mask and end are derived
 * (PAPER.md:230).  For GD_PART_POW2 partitions base is aligned to size and
 * size is a power of two; exact-size partitions carry only base and size.   */
#define GD_PART_POW2 1u
typedef struct {
    uint32_t id;
    uint32_t flags;                   /* GD_PART_POW2 or 0          */
    uint64_t base;
    uint64_t size;
    uint64_t mask;                    /* size - 1                  */
    uint64_t end;                     /* base + size (exclusive)   */
} gd_partition_info;

/* Per-tenant statistics.  violations come from the device counters (check
 * mode); launches / bytes / flops are host-side accounting of algorithmic
 * work (SURVEY.md §8(d) "Algorithmic work per unit").                         */
typedef struct {
    uint64_t violations;
    uint64_t launches;
    uint64_t bytes;
    uint64_t flops;
    uint64_t violations_by_kind[GD_NUM_KINDS];
    uint64_t launches_by_kind[GD_NUM_KINDS];
} gd_stats_t;

/* ---- arena and partitions ------ */

/* Reserve a power-of-two device arena of arena_bytes on `device`, aligned to
 * its own size (CUDA VMM reservation; physical memory is mapped per partition
 * at gd_partition_alloc).  Errors: NOT_POW2 (size not a power of two or below
 * 4 KiB), DEVICE_OOM, CUDA.                                                  */
gd_status gd_arena_create(int device, uint64_t arena_bytes, uint32_t flags, gd_arena **out);
/* Use caller-owned device memory [dev_ptr, dev_ptr+bytes) as the arena (the
 * caller keeps it alive and fully backed; the library never frees it).
 * dev_ptr must be aligned to bytes (ALIGN), bytes a power of two (NOT_POW2).
 * device < 0 creates a VIRTUAL arena: bookkeeping only, no CUDA calls, every
 * launch returns UNSUPPORTED (host-logic tests on machines without a GPU).  */
gd_status gd_arena_wrap(int device, uint64_t dev_ptr, uint64_t bytes, gd_arena **out);
gd_status gd_arena_destroy(gd_arena *a);
/* base, size and device of an arena (device = -1 for a virtual arena).       */
gd_status gd_arena_info(const gd_arena *a, uint64_t *base, uint64_t *size, int *device);

/* Carve a partition: size = next_pow2(max(requested, 4 KiB)), base = a free
 * buddy block of that size, so base % size == 0.
 * The partition is physically backed in full (every fenced address is
 * mapped) and scrubbed to zero before it is returned (reading A15).
 * Errors: INVALID_ARG (requested 0 or > arena), DEVICE_OOM (no free block,
 * or all GD_MAX_TENANTS ids in use), CUDA.                                    */
gd_status gd_partition_alloc(gd_arena *a, uint64_t requested_bytes, gd_partition_info *out);
/* Exact-size partition (removes the power-of-two
 * utilisation limit PAPER.md:246 names): size = requested rounded up to the
 * physical backing granule (2 MiB for VMM arenas, 4 KiB otherwise); placed at
 * a block of next_pow2(size) whose unused tail goes straight back to the
 * buddy allocator.  Usable with NONE, CHECK and MODULO launches; a MASK
 * launch on it returns GD_ERR_NOT_POW2 (unless size happens to be a power
 * of two).  Errors as gd_partition_alloc.                                   */
gd_status gd_partition_alloc_exact(gd_arena *a, uint64_t requested_bytes, gd_partition_info *out);
/* Return a partition to the buddy allocator (coalescing). UNKNOWN_PARTITION. */
gd_status gd_partition_free(gd_arena *a, uint32_t id);
gd_status gd_partition_get(const gd_arena *a, uint32_t id, gd_partition_info *out);

/* Sub-allocation inside a partition: first
 * fit over the partition's free extents, 256-byte aligned.  bytes = 0 is
 * INVALID_ARG; a full partition is PARTITION_OOM.  gd_free takes the exact
 * address gd_malloc returned (UNKNOWN_ALLOC otherwise).                      */
gd_status gd_malloc(gd_arena *a, uint32_t id, uint64_t bytes, uint64_t *dev_addr);
gd_status gd_free(gd_arena *a, uint32_t id, uint64_t dev_addr);

/* Host-transfer validation (§4.2.2):
 * *ok = 1 iff [addr, addr+len) lies inside the partition with no 64-bit
 * wraparound (len = 0: base <= addr <= end).                                 */
gd_status gd_check_range(const gd_arena *a, uint32_t id, uint64_t addr, uint64_t len, int *ok);
/* Checked transfers: OOB_RANGE (nothing copied) when the device range fails
 * gd_check_range.  Asynchronous on `stream` (host memory should be pinned).  */
gd_status gd_memcpy_h2d(gd_arena *a, uint32_t id, uint64_t dst, const void *src, uint64_t n, void *stream);
gd_status gd_memcpy_d2h(gd_arena *a, uint32_t id, void *dst, uint64_t src, uint64_t n, void *stream);
/* Device-to-device transfer inside one partition ("within the GPU memory
 * (e.g., cudaMemcpyD2D())"): both ranges are checked.         */
gd_status gd_memcpy_d2d(gd_arena *a, uint32_t id, uint64_t dst, uint64_t src, uint64_t n, void *stream);

/* Trusted fill of [base+offset, base+offset+nbytes) of a partition (K7):
 * pattern 0 = zeros (the scrub), 1 = the address-revealing word pattern
 * P(o) = (o >> 2) ^ 0x9E3779B9 of the byte offset o from the partition base
 * (SURVEY.md §8(d) C3).  offset and nbytes must be multiples of 16 (ALIGN);
 * the range must lie in the partition (OOB_RANGE).                          */
gd_status gd_partition_fill(gd_arena *a, uint32_t id, uint32_t pattern, uint64_t offset, uint64_t nbytes, void *stream);

/* ---- fenced kernels (§8(b)) --------------------------
 * Every global address each kernel computes passes through the fence of
 * `mode` with the partition's base and mask passed by value as a
 * __grid_constant__ kernel parameter (constant bank; §4.2.3
 * parameter augmentation, reading A12).  Check-mode refusals are counted
 * per logical access with warp/CTA aggregation into the tenant's counter.   */

/* dst[0:nbytes) = src[0:nbytes): 16-byte units, then a byte tail.
 * dst, src 16-byte aligned (ALIGN).  Overlapping buffers: unspecified.       */
gd_status gd_launch_fenced_copy(gd_arena *a, uint32_t id, gd_mode mode, uint64_t dst, uint64_t src,
                                uint64_t nbytes, void *stream);
/* y[i] = fmaf(alpha, x[i], y[i]) for i < n, fp32, one rounding.
 * x, y 16-byte aligned (ALIGN).                                              */
gd_status gd_launch_fenced_saxpy(gd_arena *a, uint32_t id, gd_mode mode, float alpha, uint64_t x,
                                 uint64_t y, uint64_t n, void *stream);
/* out[i*D+d] = table[sext(idx[i])*D + d] for i < n, d < D = row_elems (u32
 * words; int32 indices sign-extended and scaled in 64 bits, Listing 1 line
 * 22 mul.wide.s32).  out, idx 16-byte aligned; table 4-byte aligned.        */
gd_status gd_launch_fenced_gather(gd_arena *a, uint32_t id, gd_mode mode, uint64_t out, uint64_t table,
                                  uint64_t idx, uint64_t n, uint32_t row_elems, void *stream);
/* table[sext(idx[i])] += src[i] (u32, wrapping; device atomics, so the
 * result is order-independent).  idx, src 16-byte aligned; table 4-byte.    */
gd_status gd_launch_fenced_scatter(gd_arena *a, uint32_t id, gd_mode mode, uint64_t table, uint64_t idx,
                                   uint64_t src, uint64_t n, void *stream);
/* 5-point Jacobi sweep over the interior of an H x W fp32 grid with row
 * pitch `pitch_elems`: out = fmaf(c1, (N+S)+(W+E), c0*C); boundary rows and
 * columns of out are not written.  in, out 16-byte aligned, pitch % 4 == 0. */
gd_status gd_launch_fenced_stencil(gd_arena *a, uint32_t id, gd_mode mode, uint64_t out, uint64_t in,
                                   uint32_t H, uint32_t W, uint64_t pitch_elems, float c0, float c1,
                                   void *stream);
/* K5 v2: the same sweep with both operands
 * staged by TMA and fenced in their tensor maps (reading R-TMA) instead of
 * per access: `in` is H rows x W floats, `out` the rows 0..H-2 x columns
 * 0..W-2 that hold interior points.  Each map's base is fenced like a
 * 16-byte access (check: an illegal base gives no rows) and its row count
 * clamped so that its last row ends inside the partition; rows of `in` past
 * it read as 0, interior points in rows of `out` past it are not stored (no
 * wrap-around of rows, unlike v1's per-access mask).  The counting modes
 * count, once per operand, the rows check would refuse.  Same alignment
 * rules as gd_launch_fenced_stencil.                                         */
gd_status gd_launch_fenced_stencil_tma(gd_arena *a, uint32_t id, gd_mode mode, uint64_t out, uint64_t in,
                                       uint32_t H, uint32_t W, uint64_t pitch_elems, float c0, float c1,
                                       void *stream);
/* C[M,N] = A[M,K] . B[N,K]^T, bf16 inputs (K-major, row strides lda/ldb in
 * elements), fp32 accumulation on the tcgen05 tensor cores, bf16 output
 * (row stride ldc).  The fence is applied to the TMA tensor maps: each
 * operand's global address is fenced and its row extent clamped to the
 * partition (reading of O2).  Shape limits: K % 64 == 0,
 * N % 16 == 0, strides % 8 == 0 (UNSUPPORTED otherwise).                     */
gd_status gd_launch_fenced_gemm(gd_arena *a, uint32_t id, gd_mode mode, uint64_t C, uint64_t A, uint64_t B,
                                uint32_t M, uint32_t N, uint32_t K, uint64_t lda, uint64_t ldb, uint64_t ldc,
                                void *stream);

/* ---- multi-tenant launcher -------- */
/* One queued launch.  Field use per kind:
 *   COPY   : ptr = {dst, src},        u64[0] = nbytes
 *   SAXPY  : ptr = {x, y},            u64[0] = n,  f32[0] = alpha
 *   GATHER : ptr = {out, table, idx}, u64[0] = n,  u32[0] = row_elems
 *   SCATTER: ptr = {table, idx, src}, u64[0] = n
 *   STENCIL: ptr = {out, in},         u64[0] = pitch, u32 = {H, W}, f32 = {c0, c1}
 *   GEMM   : ptr = {C, A, B},         u64 = {lda, ldb, ldc}, u32 = {M, N, K}     */
typedef struct {
    uint32_t tenant;
    uint32_t kind;                    /* gd_kind */
    uint32_t mode;                    /* gd_mode */
    uint32_t u32[3];
    uint64_t ptr[3];
    uint64_t u64[3];
    float f32[2];
} gd_work;

/* Issue order of the launcher, without launching (pure host logic): work
 * items keep FIFO order within a tenant; tenants take turns round-robin in
 * order of first appearance ("selects GPU calls from different
 * applications in a round-robin fashion"; SPEC.md:398 a1,b1,a2).
 * order_out[k] = index into items of the k-th launch.                       */
gd_status gd_schedule_round_robin(const gd_work *items, uint32_t n_items, uint32_t *order_out);
/* Validate every item (nothing is issued if any is invalid), then issue them
 * in gd_schedule_round_robin order, each on streams[s] where s is the rank
 * of its tenant in order of first appearance modulo n_streams (one stream
 * per tenant in one context: PAPER.md:177).  order_out may be NULL.         */
gd_status gd_launcher_run(gd_arena *a, const gd_work *items, uint32_t n_items, void *const *streams,
                          uint32_t n_streams, uint32_t *order_out);

/* Issue policies (gd_launcher_run_policy).
 *  ROUND_ROBIN : gd_launcher_run, the paper's launcher:
 *                every tenant's stream free-running, the hardware overlaps.
 *  NO_TENSOR_RANDOM : the same order and streams, plus cross-stream event
 *                waits so that a tensor-core kernel (GEMM) never runs
 *                concurrently with a random-access kernel (gather, scatter):
 *                each waits for every such kernel of the other class issued
 *                before it.  Streaming kernels (copy, saxpy, stencil) stay
 *                free.  Measured on B200 (tools/c5_policies.py): GEMM with a
 *                concurrent gather is 22 % slower than the two serialised
 *                (the gather's random DRAM traffic stalls the GEMM's TMA
 *                pipeline), while GEMM with a copy is 13 % faster, and
 *                copy / gather pairs are neutral.  Results are identical
 *                (different tenants never share memory); only overlap changes.
 *  MEMORY_LANE : NO_TENSOR_RANDOM, and the memory-bound kernels (all but
 *                GEMM) run one after another in issue order on a single
 *                "HBM lane" (event chain across the tenant streams), so only
 *                tensor-core work overlaps them.                             */
typedef enum { GD_POLICY_ROUND_ROBIN = 0, GD_POLICY_NO_TENSOR_RANDOM = 1, GD_POLICY_MEMORY_LANE = 2 } gd_policy;
gd_status gd_launcher_run_policy(gd_arena *a, const gd_work *items, uint32_t n_items, void *const *streams,
                                 uint32_t n_streams, uint32_t policy, uint32_t *order_out);

/* ---- captured steps (CUDA graphs) ------------------------------------------ */
typedef struct gd_graph gd_graph;     /* opaque, library-owned */
/* Capture one gd_launcher_run of `items` over n_streams library-owned tenant
 * streams (fork / join through an origin stream) into a CUDA graph, every
 * kernel with its partition descriptor baked in.  Items are validated first
 * (nothing is captured if any is invalid).  Errors as gd_launcher_run.     */
gd_status gd_graph_create(gd_arena *a, const gd_work *items, uint32_t n_items, uint32_t n_streams, gd_graph **out);
/* Replay the captured step on `stream` with one host call.  Refuses with
 * UNKNOWN_PARTITION (nothing launched) if any partition the graph fences was
 * freed or re-allocated since capture: stale bounds are never used; and, for
 * a graph that captured unfenced solo launches (gd_arena_set_native_when_solo),
 * if the arena's partition set or that switch changed since capture.        */
gd_status gd_graph_launch(gd_graph *g, void *stream);
gd_status gd_graph_destroy(gd_graph *g);

/* ---- statistics --------------------------------- */
/* Synchronises the device, then returns tenant id's counters, or the sum over
 * all tenants for GD_ALL_TENANTS.                                            */
gd_status gd_stats(gd_arena *a, uint32_t id, gd_stats_t *out);
gd_status gd_stats_reset(gd_arena *a, uint32_t id);
/* Device address of the trusted violation counters (u64[GD_MAX_TENANTS][GD_NUM_KINDS]),
 * allocated outside the arena; 0 for virtual arenas.          */
gd_status gd_stats_device_ptr(const gd_arena *a, uint64_t *dev_ptr);

const char *gd_status_str(gd_status s);
int gd_last_cuda_error(void);
/* Native kernel for a tenant alone ("When an application runs
 * alone, the manager issues a native kernel"; SPEC.md:418 --native-when-solo,
 * default off).  While on and exactly one partition of the arena is live,
 * every launch is validated in its requested mode and then run as
 * GD_MODE_NONE: no fence and nothing counted.  A second live partition
 * restores fencing for the next launch: the decision is taken and the kernel
 * enqueued while partition changes are held off, and a new partition is
 * scrubbed only after every enqueued kernel has finished.  A graph captured
 * while a tenant ran alone is refused at replay (UNKNOWN_PARTITION) once any
 * partition was allocated or freed, or this switch changed, since capture.  */
gd_status gd_arena_set_native_when_solo(gd_arena *a, int on);

/* Synchronises, then reports (and clears) device-side health flags:
 * bit 0 = a tensor-core (GEMM) pipeline wait timed out, bit 1 = a TMA load
 * wait of the K5 v2 stencil timed out (the kernel gave up after ~2 s instead
 * of hanging the shared context; the tile was not stored).                   */
gd_status gd_device_flags(gd_arena *a, uint32_t *flags);
/* Library build identification, e.g. "guardian sm_100a <git>".               */
const char *gd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GUARDIAN_H */
