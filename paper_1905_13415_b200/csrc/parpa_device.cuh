// parpa_device.cuh — device primitives of the ParPaRaw hot path on sm_100a.
//
// Citations: P:n = PAPER.md line n.  DESIGN.md §Kernels describes the data layouts.
//
//   * Device state numbering.  The DFA's non-invalid states are renumbered 0..k-1 (k <= 8) and
//     the absorbing invalid state becomes nibble 0xF.  A state-transition vector τ
//      over the k live states is kept in BYTE form in two registers (byte j =
//     0x80 | τ_j, INV = 0x8F or 0xFF) and in NIBBLE form in one register (nibble j = τ_j).
//     The composite operator (a∘b)_j = b_{a_j} is one PRMT per four entries: b in
//     byte form is the PRMT source, a in nibble form the selector.  A selector nibble 0xF
//     (= INV) makes PRMT replicate the sign bit of byte 7, which is set in every byte-form
//     entry, so INV maps to INV without a 9th lane: 9 states fit the 8-lane form because INV is
//     absorbing.  This replaces the paper's MFIRA + BFE/BFI per instance.
//   * Per-byte LUT in shared memory (64 KB, replicated per lane group so that random byte values
//     never bank-conflict).  Row b (256 B) holds for 16 lane slots {sel_lo, sel_hi} — the
//     nibble-form transition row of b's symbol group split in two 16-bit PRMT selectors — and,
//     at +128 B, the pass-2 step row: byte j = 0x80 | next(j) | flags(j) << 4.  One PRMT builds
//     the LDS address (b << 8 | lane slot) straight from the input word.  The byte -> symbol
//     group map of P:725-731 / tab:twiddling is folded into this table at DFA-compile time.
//   * Segment summary (SegT within a tile, Seg globally): record count (POPCNT),
//     field count, the abs/rel column offset with the ⊕ operator of P:408-414, and the carries
//     of the field left open at the segment end (first / last DATA byte, control-byte flags)
//     so that spans can be trimmed across chunk and tile boundaries.
#pragma once
#include <stdint.h>

namespace parpa {

constexpr int CHUNK = 64;                  // bytes per thread ("chunk")
constexpr int WT = CHUNK * 32;             // one warp tile = 2 KB (a lane per 64-byte chunk)
constexpr int LUT_BYTES = 256 * 256;       // 64 KB shared-memory LUT
constexpr uint32_t NIB_IDENT = 0x76543210u;
constexpr uint32_t INV_DEV = 0xFu;
constexpr unsigned long long NONE = 0xFFFFFFFFFFFFFFFFull;
constexpr uint32_t NONE16 = 0xFFFFu;

// emission kind in bits 4-5 of a pass-2 step byte, coded so that 0xFF (produced for INV by PRMT's sign
// replication) reads as CTRL: DATA 00, FIELD 01, RECORD 10, CTRL 11.  Two gathered bits per byte give the
// masks: DATA = ~(b4 | b5), DELIM = b4 ^ b5, RECORD = b5 & ~b4.
constexpr uint32_t KC_DATA = 0u, KC_FIELD = 1u, KC_RECORD = 2u, KC_CTRL = 3u, KC_MASK = 0x30u;
__device__ __host__ __forceinline__ uint32_t step_kind_code(uint32_t x) { return (x >> 4) & 3u; }

// SegT / Seg flag bits
constexpr uint32_t F_ABS = 1, F_HD = 2, F_IC = 4, F_PC = 8, F_PRE = 16;

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// ---- τ representations ------------------------------------------------------------------
__device__ __forceinline__ uint32_t pack_nib(uint32_t t0, uint32_t t1) {   // byte form -> nibble form
  uint32_t x = t0 & 0x0F0F0F0Fu, y = t1 & 0x0F0F0F0Fu;
  x |= x >> 4;
  y |= y >> 4;
  return prmt(x, y, 0x6420);
}
__device__ __forceinline__ uint32_t spread16(uint32_t h) {                // 4 nibbles -> 4 bytes | 0x80
  uint32_t x = h & 0xFFFFu;
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  return x | 0x80808080u;
}
// (a∘b) with both in nibble form: c_j = b[a_j]
__device__ __forceinline__ uint32_t compose_nib(uint32_t a, uint32_t b) {
  uint32_t b0 = spread16(b), b1 = spread16(b >> 16);
  return pack_nib(prmt(b0, b1, a), prmt(b0, b1, a >> 16));
}
__device__ __host__ __forceinline__ uint32_t nib_at(uint32_t t, uint32_t s) {      // τ[s], s in 0..7 or 0xF
  return s == INV_DEV ? INV_DEV : (t >> (4 * s)) & 0xFu;
}

// ---- tile-local segment summary (3 words) ------------------------------------------------
struct SegT {
  uint32_t cnt;     // recs (low 16) | delimiters (high 16)          — counts within one tile
  uint32_t colf;    // column value (low 16) | flags (high 16)
  uint32_t pos;     // first DATA (low 16) | last DATA (high 16), tile-local, 0xFFFF = none
};
__device__ __forceinline__ SegT segt_ident() { return SegT{0u, 0u, 0xFFFFFFFFu}; }

// a then b
__device__ __forceinline__ SegT segt_op(SegT a, SegT b) {
  SegT c;
  c.cnt = a.cnt + b.cnt;                                   // both halves < 2^16 within a tile
  uint32_t fa = a.colf >> 16, fb = b.colf >> 16;
  uint32_t col = (fb & F_ABS) ? (b.colf & 0xFFFFu) : ((a.colf + b.colf) & 0xFFFFu);
  uint32_t fl = ((fa | fb) & (F_ABS | F_HD));
  uint32_t afd = a.pos & 0xFFFFu, bfd = b.pos & 0xFFFFu;
  uint32_t pos;
  if (fb & F_HD) {
    pos = b.pos;
    fl |= fb & (F_IC | F_PC | F_PRE);
  } else if (afd == NONE16) {
    pos = b.pos;
    fl |= (fb & (F_IC | F_PC)) | ((fa | fb) & F_PRE);
  } else if (bfd == NONE16) {
    pos = a.pos;
    fl |= (fa & (F_IC | F_PRE)) | ((fa & F_PC) || (fb & F_PRE) ? F_PC : 0);
  } else {
    pos = afd | (b.pos & 0xFFFF0000u);
    fl |= (fa & F_PRE) | (fb & F_PC) | (((fa & (F_IC | F_PC)) || (fb & (F_PRE | F_IC))) ? F_IC : 0);
  }
  c.colf = col | (fl << 16);
  c.pos = pos;
  return c;
}

// ---- global segment summary ---------------------------------------------------------------
struct Seg {
  unsigned long long recs, nflds, fd, ld;
  uint32_t col, flags;
};
__device__ __host__ __forceinline__ Seg seg_ident() { return Seg{0ull, 0ull, NONE, NONE, 0u, 0u}; }

__device__ __host__ __forceinline__ Seg seg_op(const Seg &a, const Seg &b) {
  Seg c;
  c.recs = a.recs + b.recs;
  c.nflds = a.nflds + b.nflds;
  c.col = (b.flags & F_ABS) ? b.col : a.col + b.col;
  uint32_t fl = (a.flags | b.flags) & (F_ABS | F_HD);
  if (b.flags & F_HD) {
    c.fd = b.fd; c.ld = b.ld;
    fl |= b.flags & (F_IC | F_PC | F_PRE);
  } else if (a.fd == NONE) {
    c.fd = b.fd; c.ld = b.ld;
    fl |= (b.flags & (F_IC | F_PC)) | ((a.flags | b.flags) & F_PRE);
  } else if (b.fd == NONE) {
    c.fd = a.fd; c.ld = a.ld;
    fl |= (a.flags & (F_IC | F_PRE)) | (((a.flags & F_PC) || (b.flags & F_PRE)) ? F_PC : 0);
  } else {
    c.fd = a.fd; c.ld = b.ld;
    fl |= (a.flags & F_PRE) | (b.flags & F_PC) |
          (((a.flags & (F_IC | F_PC)) || (b.flags & (F_PRE | F_IC))) ? F_IC : 0);
  }
  c.flags = fl;
  return c;
}

__device__ __forceinline__ Seg segt_to_seg(SegT t, unsigned long long tile_base) {
  Seg s;
  s.recs = t.cnt & 0xFFFFu;
  s.nflds = t.cnt >> 16;
  s.col = t.colf & 0xFFFFu;
  s.flags = t.colf >> 16;
  uint32_t fd = t.pos & 0xFFFFu, ld = t.pos >> 16;
  s.fd = fd == NONE16 ? NONE : tile_base + fd;
  s.ld = ld == NONE16 ? NONE : tile_base + ld;
  return s;
}

// ---- 64-bit mask helpers (bit i = chunk byte i) -------------------------------------------
__device__ __forceinline__ int msb64(unsigned long long x) { return 63 - __clzll(x); }
__device__ __forceinline__ int lsb64(unsigned long long x) { return __ffsll(x) - 1; }
__device__ __forceinline__ unsigned long long below(int p) {          // bits [0, p)
  return p >= 64 ? ~0ull : ((1ull << p) - 1ull);
}
__device__ __forceinline__ unsigned long long above(int p) {          // bits (p, 63]
  return p >= 63 ? 0ull : (~0ull << (p + 1));
}

// Open-field summary of a byte range given its DATA / CTRL masks (range already applied).
// Returns flags (IC, PC, PRE) and fd / ld (chunk-local, -1 = none).
__device__ __forceinline__ uint32_t open_summary(unsigned long long Dm, unsigned long long Km, int &fd, int &ld) {
  if (Dm == 0ull) {
    fd = ld = -1;
    return Km ? F_PRE : 0u;
  }
  fd = lsb64(Dm);
  ld = msb64(Dm);
  uint32_t fl = 0;
  if (Km & below(fd)) fl |= F_PRE;
  if (Km & above(ld)) fl |= F_PC;
  if (Km & above(fd) & below(ld)) fl |= F_IC;
  return fl;
}

// Chunk summary from its masks (positions chunk-local, offset by `off` into the tile).
__device__ __forceinline__ SegT chunk_segt(unsigned long long Dm, unsigned long long Fm,
                                           unsigned long long Rm, unsigned long long Vm, uint32_t off) {
  unsigned long long Km = Vm & ~Dm & ~Fm;
  SegT s;
  uint32_t recs = __popcll(Rm), nd = __popcll(Fm);
  s.cnt = recs | (nd << 16);
  uint32_t col, fl = 0;
  if (Rm) {
    col = __popcll(Fm & above(msb64(Rm)));
    fl |= F_ABS;
  } else {
    col = nd;
  }
  unsigned long long open = Vm;
  if (Fm) {
    fl |= F_HD;
    open &= above(msb64(Fm));
  }
  int fd, ld;
  fl |= open_summary(Dm & open, Km & open, fd, ld);
  s.pos = fd < 0 ? 0xFFFFFFFFu : ((uint32_t)(fd + off) | ((uint32_t)(ld + off) << 16));
  s.colf = col | (fl << 16);
  return s;
}

// ---- warp shuffles ----------------------------------------------------------------------
__device__ __forceinline__ SegT shfl_up_segt(SegT s, int d) {
  return SegT{__shfl_up_sync(0xffffffffu, s.cnt, d), __shfl_up_sync(0xffffffffu, s.colf, d),
              __shfl_up_sync(0xffffffffu, s.pos, d)};
}
__device__ __forceinline__ SegT shfl_down_segt(SegT s, int d) {
  return SegT{__shfl_down_sync(0xffffffffu, s.cnt, d), __shfl_down_sync(0xffffffffu, s.colf, d),
              __shfl_down_sync(0xffffffffu, s.pos, d)};
}
__device__ __forceinline__ SegT shfl_segt(SegT s, int l) {
  return SegT{__shfl_sync(0xffffffffu, s.cnt, l), __shfl_sync(0xffffffffu, s.colf, l),
              __shfl_sync(0xffffffffu, s.pos, l)};
}

// ---- memory-model helpers for the decoupled look-back --------------------------------------
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Programmatic dependent launch (the parse's kernels after the first are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): a kernel runs its prologue (LUT build, descriptor
// copies) while its predecessor drains, then waits for the predecessor's completion and memory before
// touching its outputs.  Every CTA signals its dependents only when it leaves (PdlTrigger), so a
// dependent grid never takes SM resources from unfinished CTAs of its predecessor (the ticket-ordered
// look-back scans need every block to get an SM).  Both are no-ops for a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
struct PdlTrigger {
  __device__ __forceinline__ ~PdlTrigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
};

}  // namespace parpa

namespace parpa {
__device__ __forceinline__ uint32_t smem_u32(const void *p) {            // shared-window address
  return (uint32_t)__cvta_generic_to_shared(p);
}
}  // namespace parpa
