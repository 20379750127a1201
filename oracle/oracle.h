/*
 * oracle/oracle.h -- CPU oracle for Guardian's per-access address fencing.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2401_09290_b200/csrc/); neither includes or imports the other.
 *
 * What it is: a plain, slow, sequential simulation of one tenant's kernel
 * running over a byte array that stands for a range of device virtual
 * addresses.  Every global access of every simulated kernel goes through the
 * fence of the selected mode, exactly as the paper places the fence "before
 * every load/store" (§4.3, Listing 1 lines 26-28 at
 * PAPER.md:211-214).  Logical elements are processed in ascending order.
 *
 * Citations: PAPER.md:<line> (§section / Listing / Table);
 *            SPEC.md:<line> ([MODULE]/[OP]);  SURVEY.md §8(c) readings A1..A16.
 *
 * Parity pins: every function below is pinned by tests/test_oracle_pins.py
 * against values the paper prints, closed forms, brute force, or a library
 * routine.  No function is "parity unpinned".
 */
#ifndef GUARDIAN_ORACLE_H
#define GUARDIAN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Fence modes: none = native kernel ("issues a native kernel"),
 * mask = address fencing with bitwise operations,
 * check = address checking.          */
enum { OR_NONE = 0, OR_MASK = 1, OR_CHECK = 2, OR_MODULO = 3, OR_MASK_COUNT = 4, OR_CLAMP = 5 };
/* OR_MASK_COUNT: mask mode plus detection ("an optional
 *   GD_FLAG_COUNT adds detection"): the access goes where the mask fence puts
 *   it and is counted when the check predicate refuses it.
 * OR_CLAMP: north_star's check mode "compare, clamp and set a violation
 *   flag" (the GD_CHECK_SATURATE variant): the access goes
 *   to the nearest w-aligned address of the partition at or below it
 *   (or_fence_clamp) and is counted when the check predicate refuses it.   */

/* One simulated tenant launch context.
 *   va, len, bytes : the simulated device memory; byte bytes[k] stands for
 *                    device address va + k.  Caller-owned.
 *   base, size     : the tenant's partition ("the base address,
 *                    and the partition size"); size is a power of two and
 *                    base is size-aligned.
 *   mode           : OR_NONE / OR_MASK / OR_CHECK / OR_MODULO / OR_MASK_COUNT /
 *                    OR_CLAMP.
 * Outputs (accumulated, caller zeroes them):
 *   violations     : accesses outside the partition in the counting modes
 *                    (check: refused; mask-count, clamp: performed at the
 *                    fenced address), one per logical access (§8(c) A1).
 *   faults         : accesses whose final address lies outside the simulated
 *                    memory; they are skipped ("DeviceFault").
 *   accesses       : logical accesses attempted.                               */
typedef struct {
    uint64_t va;
    uint64_t len;
    uint8_t *bytes;
    uint64_t base;
    uint64_t size;
    int32_t mode;
    int32_t pad_;
    uint64_t violations;
    uint64_t faults;
    uint64_t accesses;
} or_ctx;

/* ---- the fence itself ---------------------------------------------------- */
/* mask = size - 1 (16 MB partition -> mask 0x000000FFFFFF).   */
uint64_t or_mask(uint64_t size);
/* Mask-mode fence of a w-byte access at a: AND with the mask, then OR with the
 * base (Listing 1 lines 26-28).  The mask additionally clears the low log2(w)
 * bits so a fenced access stays w-aligned.             */
uint64_t or_fence_mask(uint64_t a, uint64_t base, uint64_t size, uint32_t w);
/* Modulo-mode fence (§4.4): partition_base +
 * ((arbitrary_addr - partition_base) % partition_size), with the 64-bit
 * unsigned remainder (reading A10: a - base wraps mod 2^64 for a < base),
 * rounded down to a multiple of w (reading A3; size is a multiple of 16).   */
uint64_t or_fence_modulo(uint64_t a, uint64_t base, uint64_t size, uint32_t w);
/* Check-mode predicate: the w bytes [a, a+w) all lie in [base, base+size) and
 * a is w-aligned ("partition base and ending addresses";
 * SURVEY.md §8(c) A2, A3).  Returns 1 for an allowed access.                */
int or_check_ok(uint64_t a, uint64_t base, uint64_t size, uint32_t w);
/* Host-transfer range check (§4.2.2):
 * [addr, addr+len) inside [base, base+size) with no 64-bit wraparound;
 * len = 0 is allowed iff base <= addr <= base+size.                          */
int or_check_range(uint64_t base, uint64_t size, uint64_t addr, uint64_t len);
/* Clamp fence: the largest w-aligned address x of the partition with x <= a,
 * or base when there is none: base for a < base, base+size-w for
 * a > base+size-w, a rounded down to w otherwise (north_star "clamp").    */
uint64_t or_fence_clamp(uint64_t a, uint64_t base, uint64_t size, uint32_t w);
/* The address a fenced access really touches in ctx's mode, or 0 with *ok=0
 * when check mode refuses it.  Does not touch memory or counters.           */
uint64_t or_resolve(const or_ctx *c, uint64_t a, uint32_t w, int *ok);
/* 1 when the access counts as a violation in ctx's mode: check, mask-count
 * and clamp modes count exactly the accesses the check predicate refuses.   */
int or_counted(const or_ctx *c, uint64_t a, uint32_t w);
/* Element-wise loops over the two functions above (brute-force pins only).   */
void or_fence_mask_n(const uint64_t *a, uint64_t n, uint64_t base,
                     uint64_t size, uint32_t w, uint64_t *out);
void or_check_ok_n(const uint64_t *a, uint64_t n, uint64_t base,
                   uint64_t size, uint32_t w, uint8_t *out);
void or_fence_modulo_n(const uint64_t *a, uint64_t n, uint64_t base,
                       uint64_t size, uint32_t w, uint64_t *out);
void or_fence_clamp_n(const uint64_t *a, uint64_t n, uint64_t base,
                      uint64_t size, uint32_t w, uint64_t *out);

/* ---- simulated kernels -------------------------------- */
/* copy: 16-byte units, then the byte tail.                                   */
void or_copy(or_ctx *c, uint64_t dst, uint64_t src, uint64_t nbytes);
/* saxpy: y[i] = fmaf(a, x[i], y[i]) (one rounding).                          */
void or_saxpy(or_ctx *c, float a, uint64_t x, uint64_t y, uint64_t n);
/* gather: out[i*D+d] = table[sext(idx[i])*D + d], int64 address arithmetic
 * (Listing 1 line 22 `mul.wide.s32`).                          */
void or_gather(or_ctx *c, uint64_t out, uint64_t table, uint64_t idx,
               uint64_t n, uint32_t D);
/* scatter-add: table[sext(idx[i])] += src[i] (u32, wrapping).               */
void or_scatter_add(or_ctx *c, uint64_t table, uint64_t idx, uint64_t src,
                    uint64_t n);
/* 5-point Jacobi sweep over interior points (fp32):
 * out = fmaf(c1, (N+S)+(W+E), c0*C).                                         */
void or_stencil(or_ctx *c, uint64_t out, uint64_t in, uint32_t H, uint32_t W,
                uint64_t pitch, float c0, float c1);

/* ---- descriptor-fenced operands (TMA paths) - */
/* Number of rows (of `rowbytes` bytes each, `stride` bytes apart, starting at
 * operand address p) that a descriptor-fenced operand may touch in ctx's
 * mode; *p_fenced receives the start address after fencing.                  */
uint64_t or_desc_rows(const or_ctx *c, uint64_t p, uint64_t rows,
                      uint64_t rowbytes, uint64_t stride, uint64_t *p_fenced);
/* C[i][j] = sum_k A[i][k] * B[j][k]; A: M x K bf16 (row stride lda elements),
 * B: N x K bf16 (ldb), C: M x N bf16 (ldc).  Accumulate in fp64, round to
 * fp32, round to bf16 (RNE).  Rows of an operand at or past its descriptor
 * row count read as zero / are not stored.  If rows != NULL only the listed
 * rows of C are computed and stored (sampling at full size).                */
void or_gemm(or_ctx *c, uint64_t C, uint64_t A, uint64_t B, uint32_t M,
             uint32_t N, uint32_t K, uint64_t lda, uint64_t ldb, uint64_t ldc,
             const uint32_t *rows, uint32_t nrows);

/* K5 v2: the stencil with both operands descriptor-fenced (TMA staging).
 * in: H rows x W floats; out: rows 0..H-2 x columns 0..W-2 (interior points
 * only are stored).  Rows of in past its descriptor row count read as 0;
 * interior points in out rows past its row count are not stored.             */
void or_stencil_tma(or_ctx *c, uint64_t out, uint64_t in, uint32_t H, uint32_t W,
                    uint64_t pitch, float c0, float c1);

/* bf16 helpers used by or_gemm (exposed for pins).                           */
uint16_t or_f32_to_bf16(float f);
float or_bf16_to_f32(uint16_t h);

#ifdef __cplusplus
}
#endif
#endif
