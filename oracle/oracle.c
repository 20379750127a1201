/*
 * oracle/oracle.c -- CPU oracle for Guardian's per-access address fencing.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain C11, compiled with
 * -O2 -ffp-contract=off so that every float operation is rounded exactly as
 * written (one rounding per + and *, fmaf() is the single fused rounding).
 *
 * Each function follows the definition it cites, in the paper's order:
 *   - mask fence: AND with the mask, then OR with the base (Listing 1 lines
 *     26-28; §4.3).
 *   - check mode: conditional check against the partition base and end
 *     (§4.2.3, §4.4); an access that fails the
 *     check is not performed (loads read 0, stores are dropped) and is
 *     counted.
 *   - modulo: partition_base + ((addr - partition_base) % partition_size)
 *     (§4.4; u64 remainder, reading A10).
 *   - mask-count / clamp: the mask fence plus detection (SURVEY.md §8(c)
 *     A14) / north_star's "compare, clamp and set a violation flag" (A1):
 *     both count exactly the accesses check mode refuses.
 *   - none: the native kernel.
 *   - descriptor-fenced operands (TMA kernels, §8(c) O2): the operand base is
 *     fenced like a 16-byte access and its row count clamped to the
 *     partition (or_desc_rows; or_gemm, or_stencil_tma).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* The fence                                                                  */
/* ------------------------------------------------------------------------- */

uint64_t or_mask(uint64_t size) {
    /* "partition size is 16 MB ... the mask is 0x000000FFFFFF" */
    return size - 1u;
}

uint64_t or_fence_mask(uint64_t a, uint64_t base, uint64_t size, uint32_t w) {
    /* Listing 1 line 26: and.b64 %rd4, %rd4, %grdreg2   (mask)
     * Listing 1 line 28: or.b64  %rd4, %rd4, %grdreg1   (base)
     * The mask also clears the low log2(w) address bits (reading A3).       */
    uint64_t mask = or_mask(size) & ~((uint64_t)w - 1u);
    uint64_t r = a & mask;
    r = r | base;
    return r;
}

uint64_t or_fence_modulo(uint64_t a, uint64_t base, uint64_t size, uint32_t w) {
    /* fenced_addr = partition_base +
     * ((arbitrary_addr - partition_base) % partition_size)                 */
    uint64_t off = a - base;                 /* u64: wraps for a < base (A10) */
    uint64_t r = off % size;
    r = r - r % w;                           /* keep the access w-aligned (A3) */
    return base + r;
}

int or_check_ok(uint64_t a, uint64_t base, uint64_t size, uint32_t w) {
    /* Every byte of [a, a+w) inside [base, base+size), a w-aligned.         */
    if (a % w != 0) return 0;
    if (a < base) return 0;
    uint64_t off = a - base;
    if (off >= size) return 0;
    if (off + w > size) return 0;   /* off < size <= 2^63: no overflow */
    return 1;
}

int or_check_range(uint64_t base, uint64_t size, uint64_t addr, uint64_t len) {
    /* ok iff [addr, addr+len) is inside [base, base+size)
     * with no wraparound; len = 0 ok iff base <= addr <= base + size.       */
    uint64_t end = base + size;
    if (len == 0) return addr >= base && addr <= end;
    if (addr < base) return 0;
    if (addr > UINT64_MAX - len) return 0;          /* addr + len wraps */
    if (addr + len > end) return 0;
    return 1;
}

uint64_t or_fence_clamp(uint64_t a, uint64_t base, uint64_t size, uint32_t w) {
    /* north_star: check mode may "compare, clamp and set a violation flag".
     * Clamp to the partition's w-aligned addresses [base, base+size-w].     */
    uint64_t last = base + size - w;
    if (a < base) return base;
    if (a > last) return last;
    return a - a % w;                        /* base is w-aligned: stays >= base */
}

uint64_t or_resolve(const or_ctx *c, uint64_t a, uint32_t w, int *ok) {
    *ok = 1;
    if (c->mode == OR_MASK || c->mode == OR_MASK_COUNT) return or_fence_mask(a, c->base, c->size, w);
    if (c->mode == OR_MODULO) return or_fence_modulo(a, c->base, c->size, w);
    if (c->mode == OR_CLAMP) return or_fence_clamp(a, c->base, c->size, w);
    if (c->mode == OR_CHECK) {
        if (!or_check_ok(a, c->base, c->size, w)) {
            *ok = 0;
            return 0;
        }
        return a;
    }
    return a;
}

int or_counted(const or_ctx *c, uint64_t a, uint32_t w) {
    if (c->mode == OR_CHECK || c->mode == OR_MASK_COUNT || c->mode == OR_CLAMP)
        return !or_check_ok(a, c->base, c->size, w);
    return 0;
}

void or_fence_clamp_n(const uint64_t *a, uint64_t n, uint64_t base,
                      uint64_t size, uint32_t w, uint64_t *out) {
    for (uint64_t i = 0; i < n; i++) out[i] = or_fence_clamp(a[i], base, size, w);
}

void or_fence_mask_n(const uint64_t *a, uint64_t n, uint64_t base,
                     uint64_t size, uint32_t w, uint64_t *out) {
    for (uint64_t i = 0; i < n; i++) out[i] = or_fence_mask(a[i], base, size, w);
}

void or_check_ok_n(const uint64_t *a, uint64_t n, uint64_t base,
                   uint64_t size, uint32_t w, uint8_t *out) {
    for (uint64_t i = 0; i < n; i++) out[i] = (uint8_t)or_check_ok(a[i], base, size, w);
}

/* ------------------------------------------------------------------------- */
/* Simulated memory                                                           */
/* ------------------------------------------------------------------------- */

/* Host pointer for [r, r+w) of simulated memory, or NULL (a fault).          */
static uint8_t *mem_at(or_ctx *c, uint64_t r, uint32_t w) {
    if (r < c->va || r - c->va > c->len || c->len - (r - c->va) < w) {
        c->faults++;
        return NULL;
    }
    return c->bytes + (r - c->va);
}

/* One fenced access of w bytes at a: returns the host pointer it reaches, or
 * NULL when check mode refuses it (counted) or it leaves simulated memory.  */
static uint8_t *fenced(or_ctx *c, uint64_t a, uint32_t w) {
    int ok;
    c->accesses++;
    uint64_t r = or_resolve(c, a, w, &ok);
    if (or_counted(c, a, w)) c->violations++;
    if (!ok) return NULL;
    return mem_at(c, r, w);
}

static void ld(or_ctx *c, uint64_t a, uint32_t w, void *v) {
    uint8_t *p = fenced(c, a, w);
    if (p) memcpy(v, p, w);
    else memset(v, 0, w);            /* refused load reads 0 (reading A1) */
}

static void st(or_ctx *c, uint64_t a, uint32_t w, const void *v) {
    uint8_t *p = fenced(c, a, w);
    if (p) memcpy(p, v, w);          /* refused store is dropped (A1) */
}

/* ------------------------------------------------------------------------- */
/* Kernels                                               */
/* ------------------------------------------------------------------------- */

void or_copy(or_ctx *c, uint64_t dst, uint64_t src, uint64_t nbytes) {
    uint8_t v[16];
    uint64_t units = nbytes / 16;
    for (uint64_t u = 0; u < units; u++) {
        ld(c, src + 16 * u, 16, v);
        st(c, dst + 16 * u, 16, v);
    }
    for (uint64_t b = units * 16; b < nbytes; b++) {
        ld(c, src + b, 1, v);
        st(c, dst + b, 1, v);
    }
}

void or_saxpy(or_ctx *c, float a, uint64_t x, uint64_t y, uint64_t n) {
    for (uint64_t i = 0; i < n; i++) {
        float xv, yv;
        ld(c, x + 4 * i, 4, &xv);
        ld(c, y + 4 * i, 4, &yv);
        float r = fmaf(a, xv, yv);
        st(c, y + 4 * i, 4, &r);
    }
}

void or_gather(or_ctx *c, uint64_t out, uint64_t table, uint64_t idx,
               uint64_t n, uint32_t D) {
    for (uint64_t i = 0; i < n; i++) {
        int32_t j;
        ld(c, idx + 4 * i, 4, &j);
        for (uint32_t d = 0; d < D; d++) {
            /* Listing 1 line 22: mul.wide.s32 -- sign-extend, multiply in
             * 64 bits; then add to the table address (mod 2^64).          */
            int64_t e = (int64_t)j * (int64_t)D + (int64_t)d;
            uint64_t a = table + (uint64_t)e * 4u;
            uint32_t v;
            ld(c, a, 4, &v);
            st(c, out + 4 * (i * (uint64_t)D + d), 4, &v);
        }
    }
}

void or_scatter_add(or_ctx *c, uint64_t table, uint64_t idx, uint64_t src,
                    uint64_t n) {
    for (uint64_t i = 0; i < n; i++) {
        int32_t j;
        uint32_t v;
        ld(c, idx + 4 * i, 4, &j);
        ld(c, src + 4 * i, 4, &v);
        uint64_t a = table + (uint64_t)((int64_t)j * 4);
        /* one read-modify-write access, fenced like a store */
        uint8_t *p = fenced(c, a, 4);
        if (p) {
            uint32_t t;
            memcpy(&t, p, 4);
            t = t + v;               /* mod 2^32 */
            memcpy(p, &t, 4);
        }
    }
}

void or_stencil(or_ctx *c, uint64_t out, uint64_t in, uint32_t H, uint32_t W,
                uint64_t pitch, float c0, float c1) {
    for (uint64_t r = 1; r + 1 < H; r++) {
        for (uint64_t col = 1; col + 1 < W; col++) {
            uint64_t e = r * pitch + col;
            float C, N, S, Wv, E;
            ld(c, in + 4 * e, 4, &C);
            ld(c, in + 4 * (e - pitch), 4, &N);
            ld(c, in + 4 * (e + pitch), 4, &S);
            ld(c, in + 4 * (e - 1), 4, &Wv);
            ld(c, in + 4 * (e + 1), 4, &E);
            float ns = N + S;
            float we = Wv + E;
            float s = ns + we;
            float t = c0 * C;
            float o = fmaf(c1, s, t);
            st(c, out + 4 * e, 4, &o);
        }
    }
}

/* ------------------------------------------------------------------------- */
/* Descriptor-fenced operands and the GEMM                                    */
/* ------------------------------------------------------------------------- */

uint64_t or_desc_rows(const or_ctx *c, uint64_t p, uint64_t rows,
                      uint64_t rowbytes, uint64_t stride, uint64_t *p_fenced) {
    *p_fenced = p;
    if (c->mode == OR_NONE) return rows;
    uint64_t pf;
    if (c->mode == OR_MASK) {
        /* the descriptor's global address is fenced like a 16-byte access
         * (tensor-map addresses must be 16-byte aligned)                   */
        pf = or_fence_mask(p, c->base, c->size, 16);
    } else if (c->mode == OR_MASK_COUNT) {
        pf = or_fence_mask(p, c->base, c->size, 16);
    } else if (c->mode == OR_MODULO) {
        pf = or_fence_modulo(p, c->base, c->size, 16);
    } else if (c->mode == OR_CLAMP) {
        pf = or_fence_clamp(p, c->base, c->size, 16);
    } else {
        /* check: the start must itself be a legal 16-byte-aligned address */
        if (!or_check_ok(p, c->base, c->size, 16)) return 0;
        pf = p;
    }
    *p_fenced = pf;
    uint64_t end = c->base + c->size;
    if (end - pf < rowbytes) return 0;
    uint64_t valid = (end - pf - rowbytes) / stride + 1;   /* last byte < end */
    return valid < rows ? valid : rows;
}

/* K5 v2, the TMA-staged stencil:
 * both operands are descriptor-fenced.  `in` is H rows of W floats (`pitch`
 * floats apart), `out` the H-1 rows of W-1 floats that can hold interior
 * points (rows 0..H-2, columns 0..W-2; row 0 and column 0 are never stored).
 * Rows of `in` at or past its descriptor row count read as 0 (TMA OOB fill),
 * interior points of `out` rows at or past its row count are not stored (TMA
 * store clipping).  Arithmetic and order exactly as or_stencil.  The counting
 * modes count the rows check would refuse, once per operand.                */
void or_stencil_tma(or_ctx *c, uint64_t out, uint64_t in, uint32_t H, uint32_t W,
                    uint64_t pitch, float c0, float c1) {
    if (H < 3 || W < 3) return;
    uint64_t inf, outf;
    uint64_t rin = or_desc_rows(c, in, H, 4ull * W, 4ull * pitch, &inf);
    uint64_t rout = or_desc_rows(c, out, H - 1, 4ull * (W - 1), 4ull * pitch, &outf);
    if (c->mode == OR_CHECK || c->mode == OR_MASK_COUNT || c->mode == OR_CLAMP) {
        or_ctx chk = *c;
        uint64_t pf;
        chk.mode = OR_CHECK;
        c->violations += (H - or_desc_rows(&chk, in, H, 4ull * W, 4ull * pitch, &pf)) +
                         ((H - 1) - or_desc_rows(&chk, out, H - 1, 4ull * (W - 1), 4ull * pitch, &pf));
    }
    for (uint64_t r = 1; r + 1 < H; r++) {
        for (uint64_t col = 1; col + 1 < W; col++) {
            float v[5] = {0.f, 0.f, 0.f, 0.f, 0.f};          /* C, N, S, W, E */
            const uint64_t rr[5] = {r, r - 1, r + 1, r, r};
            const uint64_t cc[5] = {col, col, col, col - 1, col + 1};
            for (int k = 0; k < 5; k++) {
                if (rr[k] >= rin) continue;                   /* past the descriptor: zero fill */
                uint8_t *p = mem_at(c, inf + 4 * (rr[k] * pitch + cc[k]), 4);
                if (p) memcpy(&v[k], p, 4);
            }
            float ns = v[1] + v[2];
            float we = v[3] + v[4];
            float s = ns + we;
            float t = c0 * v[0];
            float o = fmaf(c1, s, t);
            if (r < rout) {
                uint8_t *p = mem_at(c, outf + 4 * (r * pitch + col), 4);
                if (p) memcpy(p, &o, 4);
            }
        }
    }
}

uint16_t or_f32_to_bf16(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu))
        return (uint16_t)((u >> 16) | 0x0040u);            /* quiet NaN */
    uint32_t lsb = (u >> 16) & 1u;
    u = u + 0x7fffu + lsb;                                 /* round to nearest even */
    return (uint16_t)(u >> 16);
}

float or_bf16_to_f32(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

void or_gemm(or_ctx *c, uint64_t C, uint64_t A, uint64_t B, uint32_t M,
             uint32_t N, uint32_t K, uint64_t lda, uint64_t ldb, uint64_t ldc,
             const uint32_t *rows, uint32_t nrows) {
    uint64_t Af, Bf, Cf;
    uint64_t rA = or_desc_rows(c, A, M, 2ull * K, 2ull * lda, &Af);
    uint64_t rB = or_desc_rows(c, B, N, 2ull * K, 2ull * ldb, &Bf);
    uint64_t rC = or_desc_rows(c, C, M, 2ull * N, 2ull * ldc, &Cf);
    if (c->mode == OR_CHECK || c->mode == OR_MASK_COUNT || c->mode == OR_CLAMP) {
        /* counted as check mode would refuse them: rows of each operand that
         * are not wholly inside the partition at their unfenced address    */
        or_ctx chk = *c;
        uint64_t pf;
        chk.mode = OR_CHECK;
        c->violations += (M - or_desc_rows(&chk, A, M, 2ull * K, 2ull * lda, &pf)) +
                         (N - or_desc_rows(&chk, B, N, 2ull * K, 2ull * ldb, &pf)) +
                         (M - or_desc_rows(&chk, C, M, 2ull * N, 2ull * ldc, &pf));
    }

    double *arow = (double *)malloc(sizeof(double) * (K ? K : 1));
    double *brow = (double *)malloc(sizeof(double) * (K ? K : 1));
    uint32_t count = rows ? nrows : M;
    for (uint32_t t = 0; t < count; t++) {
        uint32_t i = rows ? rows[t] : t;
        if (i >= rC) continue;                       /* store dropped */
        for (uint32_t k = 0; k < K; k++) {
            arow[k] = 0.0;
            if (i < rA) {
                uint8_t *p = mem_at(c, Af + 2ull * (i * lda + k), 2);
                if (p) { uint16_t h; memcpy(&h, p, 2); arow[k] = or_bf16_to_f32(h); }
            }
        }
        for (uint32_t j = 0; j < N; j++) {
            double acc = 0.0;
            if (j < rB) {
                for (uint32_t k = 0; k < K; k++) {
                    uint8_t *p = mem_at(c, Bf + 2ull * (j * ldb + k), 2);
                    uint16_t h = 0;
                    if (p) memcpy(&h, p, 2);
                    brow[k] = or_bf16_to_f32(h);
                }
                for (uint32_t k = 0; k < K; k++) acc += arow[k] * brow[k];
            }
            float r32 = (float)acc;
            uint16_t out = or_f32_to_bf16(r32);
            uint8_t *p = mem_at(c, Cf + 2ull * (i * ldc + j), 2);
            if (p) memcpy(p, &out, 2);
        }
    }
    free(arow);
    free(brow);
}

void or_fence_modulo_n(const uint64_t *a, uint64_t n, uint64_t base, uint64_t size, uint32_t w, uint64_t *out) {
    for (uint64_t i = 0; i < n; i++) out[i] = or_fence_modulo(a[i], base, size, w);
}
