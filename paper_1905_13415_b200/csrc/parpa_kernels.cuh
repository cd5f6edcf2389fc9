// parpa_kernels.cuh — the hot-path kernels of libparpa (sm_100a) and their device building blocks.
//
//   building blocks  LUT build, chunk load, S1+S2 τ of a chunk (chunk_tau4: four 16-byte chains),
//                    S4 re-simulation masks (chunk_masks), warp ∘-scan of τ, look-back over τ
//                    descriptors (lookback_tau), field emission helpers, conversion glue.
//   k_pass1 .. k_seg_scan   the scan half (parpa_passes.cuh): S1-S5, chain-free passes + two
//                    single-pass decoupled look-back scans over warp-tile aggregates.
//   k_emit           S6+S7 per 2 KB warp tile from the stored chunk masks and tile prefixes: one lane
//                    per field (E1), column-major coalesced writes with int64 / float64 conversion (E2)
//                    (P:432-469).
//   k_finalize       end-of-input action, implicit last record, missing columns, status.
//   k_deferred       device-tier conversion of typed fields the thread tier deferred: fields with
//                    control bytes inside their span (re-simulated from the chunk entry state to
//                    drop them) and floats outside the exact fast path (exact decimal algorithm).
//   k_debug_trace    per-byte states / emission kinds from the per-chunk entry states (tests only).
#pragma once
#include <cooperative_groups.h>
#include "parpa_convert.cuh"
#include "parpa_device.cuh"

namespace parpa {

// column stores of the emission kernels (streaming by default; PARPA_COL_STORE_WB: write-back)
template <class T>
__device__ __forceinline__ void st_col(T *p, T v) {
#ifdef PARPA_COL_STORE_WB
  *p = v;
#else
  __stcs(p, v);
#endif
}

enum { MODE_TAU = 0, MODE_COUNT = 1 };
enum { T_SPAN = 0, T_INT64 = 1, T_FLOAT64 = 2, T_TIMESTAMP = 3, T_SKIP = 4 };   // T_SKIP: internal
// TS = the schema has timestamp columns: the emission kernels are instantiated with and without
// them so that schemas without timestamps carry none of that code (registers, stack).
template <bool TS, class Src>
__device__ __forceinline__ int conv_typed(Src &s, uint32_t type, long long &v) {
  if (TS && type == T_TIMESTAMP) return conv_timestamp(s, v);
  return type == T_INT64 ? conv_int64(s, v) : conv_float64_fast(s, v);
}
// device tier: exact for every type
template <bool TS, class Src>
__device__ __forceinline__ int conv_typed_exact(Src &s, uint32_t type, long long &v) {
  if (TS && type == T_TIMESTAMP) return conv_timestamp(s, v);
  return type == T_INT64 ? conv_int64(s, v) : conv_float64_exact(s, v);
}
enum { EOI_NONE = 0, EOI_RECORD = 1, EOI_ERROR = 2 };
enum { ST_OK = 0, ST_EFORMAT = -4, ST_ECOLUMNS = -5, ST_EUNSUPPORTED = -6, ST_ENEEDMORE = -7 };

// Device states are CLASSES of live DFA states with identical transition and emission rows (they may
// differ only in their end-of-input action, e.g. CSV's EOR and EOF): CSV's five live states become
// four, so pass 1 composes τ with one PRMT per byte instead of two.  Where the exact member matters
// (the end-of-input action, reported states) it is recovered from the byte before: members of a class
// share their rows, so the state after a byte is exact (next_exact) whatever member the class stood for.
struct DfaK {                       // compiled DFA, passed by value (kernel parameter space)
  uint32_t lut[256][4];             // per byte: {sel_lo, sel_hi, step_lo, step_hi}
  uint8_t hmap[16];                 // device state -> DFA state (its first member; index 15 = INV)
  uint8_t eoi[16];                  // EOI action by device state (of its first member)
  uint8_t gob[256];                 // byte -> symbol group
  uint8_t next_exact[16][16];       // [device state][group] -> exact DFA state after the byte
  uint8_t eoi_state[16];            // EOI action by DFA state
  uint32_t nlive, merged, inv_state, pad;   // device states in use; 1 if some class has > 1 member
  const uint4 *img;                 // prebuilt shared-memory LUT images in device memory (on device img_dev), or
  int img_dev, pad2;                // null: [PRMT layout LUT_BYTES][DP4A step layout 32 KB] (see build_lut)
};

struct ColDesc {
  unsigned long long *off;
  uint32_t *len;
  void *val;
  uint8_t *valid;
  uint32_t type, has_def;
  long long def_bits;
};

struct DeferItem {
  unsigned long long fd, ld, row;
  uint32_t col, ic;
};

constexpr int MAX_COLS = 64;
struct ColsK {                      // column descriptors, passed by value (kernel parameter space)
  ColDesc c[MAX_COLS];
};

struct Ctrl {
  unsigned int ticket;               // block tickets of k_tau_scan
  unsigned int ticket2;              // block tickets of k_seg_scan
  unsigned int n_defer;
  unsigned int defer_overflow;
  unsigned int unsupported;
  unsigned int n_long;               // fields queued for the block tier (parpa_collab.cuh)
  unsigned int n_huge;               // fields queued for the device tier
  unsigned int pad1;
  unsigned long long inv_neg;        // ~(first invalid byte position), 0 = none (atomicMax)
  unsigned long long n_missing;
  unsigned long long n_extra;
  unsigned int deferred_done;        // k_deferred blocks finished (the last one settles the status)
  unsigned int emit_ticket;          // k_emit: next warp tile to take (reset by the last warp out)
  unsigned int emit_done;            // k_emit: warps finished
  unsigned int last_cls;             // 0x100 | device class before the range's last byte (pass 2), 0 = unknown
};

struct TileInfo {
  Seg excl;                          // prefix of everything before the tile (seed included)
  uint32_t entry;                    // device entry state
  uint32_t pad;
};

struct Stats {                       // mirrors parpa_stats
  unsigned long long records, fields, first_invalid, missing_records, extra_fields, deferred_fields;
  int status;
  uint32_t final_state;
  uint32_t block_fields, device_fields;
};

struct CollabAcc {                   // per long field: reductions over its bytes (parpa_collab.cuh)
  unsigned long long first_dot, first_e, p0, plast, pexp;   // NONE = no such position
  uint32_t n_dot, n_e, bad, pad;
};

struct KArgs {
  const uint8_t *in;
  unsigned long long len, base;      // bytes of this range, global offset of in[0]
  const uint8_t *left;               // bytes preceding the range (multi-GPU halo), may be null
  unsigned long long left_len;
  uint32_t left_state;               // device state before left[0] (the halo's entry state), 0xFF unknown
  const unsigned long long *skip;    // sorted record indices not to write (skip records), may be null
  unsigned long long nskip;
  uint32_t pad_ls;
  uint32_t ntiles, seed_dev, is_last, C;
  uint32_t seed_exact, pad_se;       // the DFA state seed_dev stands for (exact; for an empty range's EOI)
  Seg seed;                          // composed prefix of everything before the range
  unsigned long long row_base;       // global record index of local row 0
  unsigned long long cap;            // rows per column
  // ntiles = warp tiles (WT bytes each); nblk = scan blocks (SCAN_TILE warp tiles each)
  uint32_t *lex;                     // [ntiles * 32] lane-exclusive τ within its warp tile (nibble form)
  uint32_t *wtau;                    // [ntiles] warp-tile τ aggregate
  uint32_t *wpre;                    // [ntiles] τ of everything before the warp tile in this range (unseeded)
  uint4 *wseg;                       // [ntiles] warp-tile SegT aggregate {cnt, colf, pos, 0}
  unsigned long long *tau_desc;      // [nblk] decoupled look-back descriptors (flag << 32) | nibble τ
  uint32_t *bflag;                   // [nblk] Seg look-back flags
  Seg *bagg, *bincl;                 // [nblk] block aggregate / inclusive prefix (valid once flagged)
  uint32_t *tot_tau;                 // τ of the whole range (nibble form, seed not applied)
  Seg *tot_seg;                      // Seg of the whole range (unseeded; the seed is applied on use)
  TileInfo *tinfo;                   // [ntiles]
  uint8_t *chunk_state;              // [ntiles * 32] device entry state of each chunk
  unsigned long long *masks;         // [ntiles][3][32] DATA / DELIM / RECORD masks of each chunk
  Ctrl *ctrl;
  DeferItem *dq;
  uint32_t dq_cap, strict;
  uint32_t emit_k, pad_ek;           // k_emit unit: 0 = by field density, 1 = warp tiles, SPARSE_K = super tiles
  unsigned long long *lq, *hq;       // block- / device-tier queues: row | column << 56 (parpa_collab.cuh)
  CollabAcc *hacc;                   // [hq_cap] device-tier accumulators
  uint32_t lq_cap, hq_cap;
  Stats *stats;
  unsigned long long *prof;          // optional [gridDim][16] cycle counters (PARPA_DEBUG)
};

constexpr uint32_t FLAG_AGG = 1, FLAG_INCL = 2;

// ---- shared-memory LUT ------------------------------------------------------------------------
// The pass kernels place the LUT at a 64 KB-aligned shared-window address S, so that one PRMT builds
// the whole 32-bit LDS address of an input byte: (S >> 16) << 16 | b << 8 | lane slot  ("laneaddr"
// holds the lane slot in byte 0 and S >> 16 in byte 2; selector 0x56k4).
template <int OFF>
__device__ __forceinline__ uint2 lds_u2(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2+%3];" : "=r"(v.x), "=r"(v.y) : "r"(addr), "n"(OFF));
  return v;
}
__device__ __forceinline__ uint32_t lds_u1(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
// LUT layouts.  PRMT layout (pass 1, k_small): 256-byte rows, the τ row of byte b at b * 256 (16 eight-byte
// slots, or 32 four-byte slots with at most four device states) and its step row at b * 256 + 128; the
// LUT sits at a 64 KB-aligned shared address so one PRMT forms the LDS address (b << 8 | slot).
// DP4A layout (pass 2): the step rows alone, 128 bytes per byte value (32 KB); the address is one IDP4A
// on the FMA pipe, dp4a(v, 128 << 8k, base + slot) — pass 2 is bound by the ALU pipe, which then keeps
// only the step and gather instructions (pass 1 with one compose PRMT per byte measured faster with the
// PRMT address).
template <bool DP>
__device__ __forceinline__ uint32_t lut_addr(uint32_t v, uint32_t k, uint32_t lbase) {
  if (DP) return __dp4a(v, 128u << (8u * k), lbase);
  return prmt(v, lbase, 0x5604u | (k << 4));
}
constexpr uint32_t STEP_ROW_DP = 128;
// With a prebuilt image (DfaK::img) the LUTs are plain coalesced 16-byte copies from L2 instead of per-entry
// constant-bank reads (which serialise over the warp's distinct addresses).
__device__ __forceinline__ void build_lut_step_dp(uint8_t *lut, const DfaK &d) {    // DP4A layout
  if (d.img) {
    const uint4 *src = d.img + LUT_BYTES / 16;
    for (int i = threadIdx.x; i < 256 * STEP_ROW_DP / 16; i += blockDim.x) reinterpret_cast<uint4 *>(lut)[i] = __ldg(src + i);
    return;
  }
  const bool ns4 = d.nlive <= 4;
  for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) {
    const int b = i >> 4, slot = i & 15;
    *reinterpret_cast<uint2 *>(lut + b * STEP_ROW_DP + slot * 8) = make_uint2(d.lut[b][2], ns4 ? d.lut[b][2] : d.lut[b][3]);
  }
}
__device__ __forceinline__ void build_lut(uint8_t *lut, const DfaK &d) {
  if (d.img) {
    for (int i = threadIdx.x; i < LUT_BYTES / 16; i += blockDim.x) reinterpret_cast<uint4 *>(lut)[i] = __ldg(d.img + i);
    return;
  }
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
    int b = i >> 5, half = (i >> 4) & 1, slot = i & 15;
    // (at most four device states: the τ half holds sel_lo in 32 four-byte slots, one per lane, so the
    // 32-bit loads of chunk_tau4<NS4> never share a bank between lanes l and l + 16)
    const bool ns4 = d.nlive <= 4;
    uint2 v = half ? make_uint2(d.lut[b][2], ns4 ? d.lut[b][2] : d.lut[b][3])
                   : make_uint2(d.lut[b][0], ns4 ? d.lut[b][0] : d.lut[b][1]);
    *reinterpret_cast<uint2 *>(lut + b * 256 + half * 128 + slot * 8) = v;
  }
}

// ---- chunk load ------------------------------------------------------------------------------
__device__ __forceinline__ void load_chunk(const uint8_t *p, int nvalid, uint32_t (&v)[16]) {
  if (nvalid == CHUNK) {
    const uint4 *q = reinterpret_cast<const uint4 *>(p);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      uint4 x = __ldg(q + k);
      v[4 * k] = x.x; v[4 * k + 1] = x.y; v[4 * k + 2] = x.z; v[4 * k + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      uint32_t w = 0;
#pragma unroll
      for (int j = 0; j < 4; j++)
        if (4 * k + j < nvalid) w |= (uint32_t)p[4 * k + j] << (8 * j);
      v[k] = w;
    }
  }
}

// ---- S1+S2: state-transition vector of a chunk (right to left: τ <- row(b_i) ∘ τ) -------------
// ---- S4: re-simulation from the entry state -> DATA / DELIM / RECORD masks --------------------
// multipliers that gather bit (4+k) of each byte into bits 32..35 of the 64-bit product
__device__ __forceinline__ uint32_t gather4(uint32_t x, uint32_t bitmask, uint32_t mul) {
  return __umulhi(x & bitmask, mul) & 0xFu;
}

// NS4 (at most four device states): the step row fits one word (per-lane 4-byte slots, see build_lut)
// and the step is PRMT(row, row, x) — an INV selector replicates the sign of byte 3.
template <bool FULL, bool NS4 = false, bool DP = false>
__device__ __forceinline__ uint32_t chunk_masks(uint32_t laneaddr, const uint32_t (&v)[16], int nvalid, uint32_t entry,
                                                unsigned long long &Dm, unsigned long long &Fm,
                                                unsigned long long &Rm, uint32_t &xprev) {
  uint32_t x = 0x80u | entry;
  xprev = x;
  uint32_t g4[2] = {0, 0}, g5[2] = {0, 0};                // kind-code bits 4 / 5 of every byte
#pragma unroll
  for (int w = 0; w < 16; w++) {
    uint32_t xs[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      int i = 4 * w + k;
      if (FULL || i < nvalid) {
        if (FULL ? i == CHUNK - 1 : i == nvalid - 1) xprev = x;   // the class before the chunk's last byte
        const uint32_t ad = lut_addr<DP>(v[w], (uint32_t)k, laneaddr) + (DP ? 0u : 128u);
        if (NS4) {
          const uint32_t st = lds_u1(ad);
          x = prmt(st, st, x);
        } else {
          const uint2 st = lds_u2<0>(ad);
          x = prmt(st.x, st.y, x);
        }
        xs[k] = x;
      } else {
        xs[k] = 0xFFu;                                    // outside the chunk: not data / delimiter
      }
    }
    uint32_t pk = prmt(prmt(xs[0], xs[1], 0x0040u), prmt(xs[2], xs[3], 0x0040u), 0x5410u);
    int h = w >> 3, sh = 4 * (w & 7);
    g4[h] |= gather4(pk, 0x10101010u, 0x10204080u) << sh;
    g5[h] |= gather4(pk, 0x20202020u, 0x08102040u) << sh;
  }
  const unsigned long long b4 = (unsigned long long)g4[0] | ((unsigned long long)g4[1] << 32);
  const unsigned long long b5 = (unsigned long long)g5[0] | ((unsigned long long)g5[1] << 32);
  Dm = ~(b4 | b5);
  Fm = b4 ^ b5;
  Rm = b5 & ~b4;
  return x & 0xFu;
}

// The same masks with a strided pack: the step result of byte i (i = 32h + 8p + s) goes into byte p of word
// W[s] (one PRMT), so that bit-plane k of the 32 bytes is  sum_s ((W[s] >> k) & 0x01010101) << s  — bit
// 8p + s = byte i, already in input order: one shift and one LOP3 per word and plane (the shifts on the FMA
// pipe as multiplies), instead of a 4-byte pack plus a multiply-gather per 4 bytes.
template <int SH>
__device__ __forceinline__ uint32_t plane_bits(uint32_t w) {   // (w >> 4 | 5) & 0x01010101, moved up by s
  if constexpr (SH >= 0) return w * (1u << SH);                // IMAD.SHL (FMA pipe)
  else return __umulhi(w, 1u << (32 + SH));                    // w >> -SH (FMA pipe)
}
template <bool FULL, bool NS4 = false, bool DP = false>
__device__ __forceinline__ uint32_t chunk_masks_t(uint32_t laneaddr, const uint32_t (&v)[16], int nvalid, uint32_t entry,
                                                  unsigned long long &Dm, unsigned long long &Fm,
                                                  unsigned long long &Rm, uint32_t &xprev) {
  uint32_t x = 0x80u | entry;
  xprev = x;
  uint32_t g4[2], g5[2];
#pragma unroll
  for (int h = 0; h < 2; h++) {
    uint32_t W[8];
#pragma unroll
    for (int s = 0; s < 8; s++) W[s] = 0u;
#pragma unroll
    for (int j = 0; j < 32; j++) {
      const int i = 32 * h + j, p = j >> 3, sidx = j & 7;
      uint32_t r = 0xFFu;                                    // outside the chunk: not data / delimiter
      if (FULL || i < nvalid) {
        if (FULL ? i == CHUNK - 1 : i == nvalid - 1) xprev = x;   // the class before the chunk's last byte
        const uint32_t ad = lut_addr<DP>(v[i >> 2], (uint32_t)(i & 3), laneaddr) + (DP ? 0u : 128u);
        if (NS4) {
          const uint32_t st = lds_u1(ad);
          x = prmt(st, st, x);
        } else {
          const uint2 st = lds_u2<0>(ad);
          x = prmt(st.x, st.y, x);
        }
        r = x;
      }
      W[sidx] = prmt(W[sidx], r, p == 0 ? 0x3214u : p == 1 ? 0x3240u : p == 2 ? 0x3410u : 0x4210u);
    }
    uint32_t a4 = 0u, a5 = 0u;
#pragma unroll
    for (int sidx = 0; sidx < 8; sidx++) {
      const uint32_t m = 0x01010101u << sidx;
      // bit 4 (5) of byte p of W[s] -> bit 8p + s
      uint32_t u4, u5;
      switch (sidx) {
        case 0: u4 = plane_bits<-4>(W[0]); u5 = plane_bits<-5>(W[0]); break;
        case 1: u4 = plane_bits<-3>(W[1]); u5 = plane_bits<-4>(W[1]); break;
        case 2: u4 = plane_bits<-2>(W[2]); u5 = plane_bits<-3>(W[2]); break;
        case 3: u4 = plane_bits<-1>(W[3]); u5 = plane_bits<-2>(W[3]); break;
        case 4: u4 = W[4]; u5 = plane_bits<-1>(W[4]); break;
        case 5: u4 = plane_bits<1>(W[5]); u5 = W[5]; break;
        case 6: u4 = plane_bits<2>(W[6]); u5 = plane_bits<1>(W[6]); break;
        default: u4 = plane_bits<3>(W[7]); u5 = plane_bits<2>(W[7]); break;
      }
      a4 |= u4 & m;
      a5 |= u5 & m;
    }
    g4[h] = a4;
    g5[h] = a5;
  }
  const unsigned long long b4 = (unsigned long long)g4[0] | ((unsigned long long)g4[1] << 32);
  const unsigned long long b5 = (unsigned long long)g5[0] | ((unsigned long long)g5[1] << 32);
  Dm = ~(b4 | b5);
  Fm = b4 ^ b5;
  Rm = b5 & ~b4;
  return x & 0xFu;
}
#ifdef PARPA_MASK_GATHER
#define CHUNK_MASKS chunk_masks
#else
#define CHUNK_MASKS chunk_masks_t
#endif

// ---- 4-way ILP τ: the chunk is cut into four 16-byte quarters with independent PRMT chains, composed
// at the end.  qt[q] = nibble τ of quarter q (q = 0..2).
// NS4: at most four device states (+ INV): τ in byte form fits one register, and one PRMT per byte
// composes it (selector nibbles 0-3 pick bytes 0-3; an INV nibble 0xF replicates the sign of byte 7,
// which is byte 3 of the same register — set, so INV stays INV).
template <bool FULL, bool NS4 = false>
__device__ __forceinline__ void chunk_tau4(uint32_t laneaddr, const uint32_t (&v)[16], int nvalid,
                                           uint32_t &t0, uint32_t &t1, uint32_t (&qt)[3]) {
  uint32_t a0[4], a1[4];
#pragma unroll
  for (int q = 0; q < 4; q++) { a0[q] = 0x83828180u; a1[q] = 0x87868584u; }
#pragma unroll
  for (int i = 15; i >= 0; --i) {
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int b = 16 * q + i;
      if (!FULL && b >= nvalid) continue;
      const uint32_t ad = lut_addr<false>(v[b >> 2], (uint32_t)(b & 3), laneaddr);
      if (NS4) {
        a0[q] = prmt(a0[q], a0[q], lds_u1(ad));
      } else {
        const uint2 e = lds_u2<0>(ad);
        uint32_t n0 = prmt(a0[q], a1[q], e.x);
        uint32_t n1 = prmt(a0[q], a1[q], e.y);
        a0[q] = n0;
        a1[q] = n1;
      }
    }
  }
  uint32_t n[4];
#pragma unroll
  for (int q = 0; q < 4; q++) n[q] = pack_nib(a0[q], a1[q]);
  qt[0] = n[0]; qt[1] = n[1]; qt[2] = n[2];
  // chunk τ = n0 ∘ n1 ∘ n2 ∘ n3 (byte form for the warp scan): source = later, selector = earlier
  uint32_t x0 = prmt(a0[3], a1[3], n[2]), x1 = prmt(a0[3], a1[3], n[2] >> 16);      // n2 ∘ n3
  uint32_t y0 = prmt(a0[1], a1[1], n[0]), y1 = prmt(a0[1], a1[1], n[0] >> 16);      // n0 ∘ n1
  uint32_t y = pack_nib(y0, y1);
  t0 = prmt(x0, x1, y);                                                               // (n0∘n1)∘(n2∘n3)
  t1 = prmt(x0, x1, y >> 16);
}

// scalar re-walk (rare): position of the first byte whose transition enters INV
// (step rows at lut + b * row + laneoff: row = 256 with lut at the step half, or STEP_ROW_DP)
__device__ int first_inv_in_chunk(const uint8_t *lut, const uint8_t *p, int nvalid, uint32_t laneoff,
                                  uint32_t entry, uint32_t row = 256) {
  uint32_t x = 0x80u | entry;
  for (int i = 0; i < nvalid; i++) {
    uint32_t b = p[i];
    uint2 st = *reinterpret_cast<const uint2 *>(lut + b * row + laneoff);
    x = prmt(st.x, st.y, x);
    if ((x & 0xFu) == INV_DEV) return i;
  }
  return -1;
}

// ---- warp-level τ scan (a warp tile = 32 chunks) ------------------------------------------------
// returns the lane's exclusive prefix; *agg = the warp tile's aggregate
__device__ __forceinline__ uint32_t warp_scan_tau(uint32_t t0, uint32_t t1, uint32_t &agg) {
  const int lane = threadIdx.x & 31;
  uint32_t inc = pack_nib(t0, t1), b0 = t0, b1 = t1;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) {                         // inc <- o ∘ inc  (o is the earlier prefix)
      uint32_t n0 = prmt(b0, b1, o), n1 = prmt(b0, b1, o >> 16);
      b0 = n0; b1 = n1;
      inc = pack_nib(n0, n1);
    }
  }
  agg = __shfl_sync(0xffffffffu, inc, 31);
  uint32_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
  return lane == 0 ? NIB_IDENT : ex;
}

// At most four device states (chunk_tau4<NS4>): t0 = τ in byte form (entries 0-3; INV = 0xFF); entries 4-7
// stay the identity, so each step is one PRMT with the earlier prefix's nibbles as selector (an INV nibble
// replicates the sign of byte 3: INV stays INV) and a 3-instruction repack of four nibbles.
__device__ __forceinline__ uint32_t nib4(uint32_t b) {        // byte form (entries 0-3) -> nibble form
  uint32_t x = b & 0x0F0F0F0Fu;
  x |= x >> 4;
  return prmt(x, 0x7654u, 0x5420u);
}
__device__ __forceinline__ uint32_t warp_scan_tau4(uint32_t t0, uint32_t &agg) {
  const int lane = threadIdx.x & 31;
  uint32_t b = t0, inc = nib4(t0);
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) {                         // inc <- o ∘ inc
      b = prmt(b, b, o);
      inc = nib4(b);
    }
  }
  agg = __shfl_sync(0xffffffffu, inc, 31);
  const uint32_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
  return lane == 0 ? NIB_IDENT : ex;
}

// ---- warp-level SegT scan -----------------------------------------------------------------------
__device__ __forceinline__ SegT warp_scan_segt(SegT s, SegT &agg) {            // exclusive
  const int lane = threadIdx.x & 31;
  SegT inc = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    SegT o = shfl_up_segt(inc, d);
    if (lane >= d) inc = segt_op(o, inc);
  }
  agg = shfl_segt(inc, 31);
  SegT ex = shfl_up_segt(inc, 1);
  return lane == 0 ? segt_ident() : ex;
}

// ---- decoupled look-back over τ (one warp) -----------------------------------------------------
// Window = 8 descriptors per lane = 256 tiles per memory round trip (all loads in flight at once),
// combined per lane as a depth-3 tree and across lanes with shuffles.  Returns τ_0 ∘ ... ∘ τ_{t-1}.
constexpr int LB_PER_LANE = 8;
__device__ uint32_t lookback_tau(const KArgs &a, uint32_t t) {
  const int lane = threadIdx.x & 31;
  uint32_t acc = NIB_IDENT;
  long long base = (long long)t - 1;
  unsigned long long nwin = 0, nspin = 0;
  while (true) {
    unsigned long long d[LB_PER_LANE];
#pragma unroll
    for (int k = 0; k < LB_PER_LANE; k++) {                  // all loads in flight at once
      long long j = base - (long long)lane * LB_PER_LANE - k;
      d[k] = j >= 0 ? ld_relaxed_u64(a.tau_desc + j) : (((unsigned long long)FLAG_INCL << 32) | NIB_IDENT);
    }
    nwin++;
    while (true) {                                            // re-poll only the unpublished ones
      bool missing = false;
#pragma unroll
      for (int k = 0; k < LB_PER_LANE; k++) {
        long long j = base - (long long)lane * LB_PER_LANE - k;
        if ((d[k] >> 32) == 0u) {
          d[k] = ld_relaxed_u64(a.tau_desc + j);
          missing = true;
        }
      }
      if (!__any_sync(0xffffffffu, missing)) break;
      nspin++;
      __nanosleep(64);
    }
    uint32_t v[LB_PER_LANE];
    bool incl = false;
    int kstar = LB_PER_LANE - 1;
#pragma unroll
    for (int k = 0; k < LB_PER_LANE; k++) {
      v[k] = (uint32_t)d[k];
      if (!incl && (d[k] >> 32) == FLAG_INCL) { incl = true; kstar = k; }
    }
#pragma unroll
    for (int k = 0; k < LB_PER_LANE; k++)
      if (k > kstar) v[k] = NIB_IDENT;
    uint32_t p0 = compose_nib(v[1], v[0]), p1 = compose_nib(v[3], v[2]);
    uint32_t p2 = compose_nib(v[5], v[4]), p3 = compose_nib(v[7], v[6]);
    uint32_t w = compose_nib(compose_nib(p3, p2), compose_nib(p1, p0));
    unsigned m = __ballot_sync(0xffffffffu, incl);
    int L = m ? __ffs(m) - 1 : 31;
    if (lane > L) w = NIB_IDENT;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      uint32_t o = __shfl_down_sync(0xffffffffu, w, dd);
      if (lane + dd < 32) w = compose_nib(o, w);
    }
    w = __shfl_sync(0xffffffffu, w, 0);
    acc = compose_nib(w, acc);
    if (m) break;
    base -= 32 * LB_PER_LANE;
  }
  if (a.prof && lane == 0) {
    atomicAdd(a.prof + blockIdx.x * 16 + 11, nwin);
    atomicAdd(a.prof + blockIdx.x * 16 + 12, nspin);
  }
  return acc;
}

// ---- decoupled look-back over Seg (one warp) ---------------------------------------------------------
__device__ __forceinline__ Seg shfl_down_seg(const Seg &s, int d) {
  Seg o;
  o.recs = __shfl_down_sync(0xffffffffu, s.recs, d);
  o.nflds = __shfl_down_sync(0xffffffffu, s.nflds, d);
  o.fd = __shfl_down_sync(0xffffffffu, s.fd, d);
  o.ld = __shfl_down_sync(0xffffffffu, s.ld, d);
  o.col = __shfl_down_sync(0xffffffffu, s.col, d);
  o.flags = __shfl_down_sync(0xffffffffu, s.flags, d);
  return o;
}
__device__ __forceinline__ Seg shfl_seg(const Seg &s, int l) {
  Seg o;
  o.recs = __shfl_sync(0xffffffffu, s.recs, l);
  o.nflds = __shfl_sync(0xffffffffu, s.nflds, l);
  o.fd = __shfl_sync(0xffffffffu, s.fd, l);
  o.ld = __shfl_sync(0xffffffffu, s.ld, l);
  o.col = __shfl_sync(0xffffffffu, s.col, l);
  o.flags = __shfl_sync(0xffffffffu, s.flags, l);
  return o;
}
__device__ __forceinline__ Seg ldcg_seg(const Seg *p) {
  Seg s;
  s.recs = __ldcg(&p->recs);
  s.nflds = __ldcg(&p->nflds);
  s.fd = __ldcg(&p->fd);
  s.ld = __ldcg(&p->ld);
  s.col = __ldcg(&p->col);
  s.flags = __ldcg(&p->flags);
  return s;
}
__device__ __forceinline__ void stcg_seg(Seg *p, const Seg &s) {
  __stcg(&p->recs, s.recs);
  __stcg(&p->nflds, s.nflds);
  __stcg(&p->fd, s.fd);
  __stcg(&p->ld, s.ld);
  __stcg(&p->col, s.col);
  __stcg(&p->flags, s.flags);
}

// ---- S6+S7: field emission ---------------------------------------------------------------------
struct EmitCounters {
  unsigned long long missing, extra;
  uint32_t unsupported;
};

__device__ __forceinline__ uint8_t fetch_byte(const KArgs &a, unsigned long long pos, bool &ok) {
  if (pos >= a.base) return __ldg(a.in + (pos - a.base));
  unsigned long long back = a.base - pos;
  if (a.left && back <= a.left_len) return a.left[a.left_len - back];
  ok = false;
  return 0;
}

struct RawSrc {                       // the raw span [pos, end] of a field without inner control bytes
  const KArgs *a;
  unsigned long long pos, end;
  bool ok;
  __device__ __forceinline__ bool next(uint8_t &c) {
    if (pos > end) return false;
    c = fetch_byte(*a, pos++, ok);
    return true;
  }
};

// The device tier's queue holds dq_cap items (len / 512, at least 4096).  A field that finds it full marks
// its valid byte (VALID_REDO_IC / VALID_REDO) and k_deferred, seeing defer_overflow, converts every marked
// row of the typed columns from its span: any number of deferred fields parses.
constexpr uint8_t VALID_REDO = 0xFF, VALID_REDO_IC = 0xFE;
#include "parpa_collab.cuh"
__device__ __forceinline__ void push_defer(const KArgs &a, const ColDesc *cd, unsigned long long fd,
                                           unsigned long long ld, unsigned long long row, uint32_t c, uint32_t ic) {
  uint32_t idx = atomicAdd(&a.ctrl->n_defer, 1u);
  if (idx < a.dq_cap) {
    cd->valid[row] = 0;              // k_deferred's overflow sweep must only see markers of this launch
    a.dq[idx] = DeferItem{fd, ld, row, c, ic};
  } else {
    cd->valid[row] = ic ? VALID_REDO_IC : VALID_REDO;
    atomicOr(&a.ctrl->defer_overflow, 1u);
  }
}

// Output row of record r: r - row_base, minus the skipped records before it; NONE for a skipped record
// (every writer tests row < cap, so a skipped record is simply not written).
__device__ __forceinline__ unsigned long long skipped_before(const KArgs &a, unsigned long long r) {
  unsigned long long lo = 0, hi = a.nskip;
  while (lo < hi) {
    const unsigned long long mid = (lo + hi) >> 1;
    if (a.skip[mid] < r) lo = mid + 1; else hi = mid;
  }
  return lo;
}
// SK = false: the emission kernel instantiated for parses without skipped records (no skip-list code).
template <bool SK = true>
__device__ __forceinline__ unsigned long long out_row(const KArgs &a, unsigned long long r) {
  if (!SK || a.nskip == 0) return r - a.row_base;
  const unsigned long long k = skipped_before(a, r);
  if (k < a.nskip && a.skip[k] == r) return NONE;
  return r - k - a.row_base;
}

template <bool TS, bool SK = true>
__device__ void emit_field(const KArgs &a, const ColDesc *cols, unsigned long long r, uint32_t c, unsigned long long fd,
                           unsigned long long ld, uint32_t fl, unsigned long long dpos, EmitCounters &cnt) {
  if (c >= a.C) { cnt.extra++; return; }
  unsigned long long row = out_row<SK>(a, r);
  if (row >= a.cap) return;                         // capacity exceeded (reported by k_finalize) or skipped
  const ColDesc *cd = cols + c;
  if (cd->type == T_SKIP) return;
  unsigned long long off;
  uint32_t len;
  if (fd == NONE) {
    off = dpos; len = 0;
  } else {
    off = fd;
    unsigned long long L = ld + 1 - fd;
    if (L >= 0xFFFFFFFFull) { cnt.unsupported = 1; L = 0xFFFFFFFEull; }
    len = (uint32_t)L;
  }
  st_col(cd->off + row, off);
  st_col(cd->len + row, len);
  uint32_t type = cd->type;
  if (type == T_SPAN) return;
  long long v = 0;
  int ok = 0;
  if (fd == NONE) {
    if (cd->has_def) { v = cd->def_bits; ok = 1; }
  } else if (fl & F_IC) {
    push_defer(a, cd, fd, ld, row, c, 1u);
    return;
  } else {
    RawSrc src{&a, fd, ld, true};
    // long fields skip the one-thread attempt: push_defer hands them to the block / device tier
    int res = ld + 1 - fd < COLLAB_MIN ? conv_typed<TS>(src, type, v) : 2;
    if (!src.ok) res = 2;                           // bytes outside this range: device tier
    if (res == 2) { push_defer(a, cd, fd, ld, row, c, 0u); return; }
    ok = res;
    if (!ok) v = 0;
  }
  reinterpret_cast<long long *>(cd->val)[row] = v;
  cd->valid[row] = (uint8_t)ok;
}

template <bool SK = true>
__device__ void fill_missing(const KArgs &a, const ColDesc *cols, unsigned long long r, uint32_t from, unsigned long long dpos,
                             EmitCounters &cnt) {
  if (from >= a.C) return;
  unsigned long long row = out_row<SK>(a, r);
  if (row == NONE) return;                          // a skipped record
  cnt.missing++;
  if (row >= a.cap) return;
  for (uint32_t k = from; k < a.C; k++) {
    const ColDesc *cd = cols + k;
    if (cd->type == T_SKIP) continue;
    cd->off[row] = dpos;
    cd->len[row] = 0xFFFFFFFFu;
    if (cd->type != T_SPAN) {
      reinterpret_cast<long long *>(cd->val)[row] = cd->has_def ? cd->def_bits : 0;
      cd->valid[row] = (uint8_t)(cd->has_def ? 1 : 0);
    }
  }
}

// open-field carry: a then b, where b holds no delimiter
__device__ __forceinline__ void open_combine(unsigned long long &fd, unsigned long long &ld, uint32_t &fl,
                                             unsigned long long bfd, unsigned long long bld, uint32_t bfl) {
  if (fd == NONE) {
    fd = bfd; ld = bld;
    fl = (bfl & (F_IC | F_PC)) | ((fl | bfl) & F_PRE);
  } else if (bfd != NONE) {
    uint32_t ic = ((fl & (F_IC | F_PC)) || (bfl & (F_PRE | F_IC))) ? F_IC : 0;
    fl = (fl & F_PRE) | (bfl & F_PC) | ic;
    ld = bld;
  } else {
    fl = (fl & (F_IC | F_PRE)) | (((fl & F_PC) || (bfl & F_PRE)) ? F_PC : 0);
  }
}

template <bool TS, bool SK = true>
__device__ void emit_chunk(const KArgs &a, const ColDesc *cols, const Seg &st, unsigned long long Dm, unsigned long long Fm,
                           unsigned long long Rm, unsigned long long Vm, unsigned long long cbase,
                           EmitCounters &cnt) {
  unsigned long long Km = Vm & ~Dm & ~Fm;
  unsigned long long r = st.recs;
  uint32_t c = st.col;
  unsigned long long cfd = st.fd, cld = st.ld;
  uint32_t cfl = st.flags & (F_IC | F_PC | F_PRE);
  int prev = -1;
  unsigned long long fm = Fm;
  while (fm) {
    int p = lsb64(fm);
    fm &= fm - 1ull;
    unsigned long long rng = below(p) & above(prev);
    int fd, ld;
    uint32_t fl = open_summary(Dm & rng, Km & rng, fd, ld);
    unsigned long long sfd = fd < 0 ? NONE : cbase + (unsigned)fd;
    unsigned long long sld = fd < 0 ? NONE : cbase + (unsigned)ld;
    if (prev >= 0) { cfd = sfd; cld = sld; cfl = fl; }
    else open_combine(cfd, cld, cfl, sfd, sld, fl);
    emit_field<TS, SK>(a, cols, r, c, cfd, cld, cfl, cbase + (unsigned)p, cnt);
    if ((Rm >> p) & 1ull) {
      fill_missing<SK>(a, cols, r, c + 1, cbase + (unsigned)p, cnt);
      r++;
      c = 0;
    } else {
      c++;
    }
    prev = p;
  }
}

__device__ __forceinline__ void flush_counters(const KArgs &a, EmitCounters &cnt) {
  if (cnt.missing) atomicAdd(&a.ctrl->n_missing, cnt.missing);
  if (cnt.extra) atomicAdd(&a.ctrl->n_extra, cnt.extra);
  if (cnt.unsupported) atomicOr(&a.ctrl->unsupported, 1u);
}

// ---- per-warp emission (S6+S7): field list in shared memory, then column-wise writes -------------
// E1: every lane walks its delimiters and appends (first-DATA offset, length | IC) of each field to
//     the warp's field list at its tile-local field index, and the end index / delimiter position of
//     each record it closes to the row list.
// E2: the warp sweeps (column, row) pairs column by column: lanes hold consecutive rows of ONE column,
//     so the column-major stores coalesce and every lane runs the same converter (no type
//     divergence).  Digits come from the warp's shared-memory copy of its tile.  This is the paper's
//     "partition by column, then convert per column" at warp-tile granularity.
constexpr int FCAP = 512;                   // fields per warp tile handled by E1/E2
constexpr int RCAP = 128;                   // records per warp tile handled by E1/E2
// K = warp tiles per emission unit: 1 (the tile's bytes staged in shared memory), or SPARSE_K for inputs
// with few fields per byte (a super tile of K consecutive warp tiles per warp: the per-tile work — delimiter
// list, field-0 carry, E2 set-up — is paid once per K tiles, and the few typed fields read their bytes from
// global memory instead of a staged copy).
template <int K>
struct alignas(16) WarpScratchT {
  uint32_t bytes[K == 1 ? WT / 4 + 8 : 4];  // the tile (plain layout) + a tail pad for 16-byte windows (K = 1)
  uint32_t fields[FCAP];                    // unit offset | length << POS_BITS | IC << 31
  uint2 f0;                                 // field 0 when it starts before the unit: {rel, len | IC << 31}
  uint32_t rows[RCAP];                      // end field index (low 16) | record delimiter position (high 16)
  uint16_t dlist[FCAP];                     // delimiter positions (unit-local) | record bit << 15
  uint32_t dmask[WT * K / 32], kmask[WT * K / 32];  // DATA / CTRL bits of the unit, 32 per word
  uint16_t kpre[WT * K / 32];               // CTRL bits before each word
  uint16_t segpre[K == 1 ? 2 : WT * K / 32];  // super tiles, E1a: delimiters before each lane's 32-bit segments
  uint32_t e1_nf, e1_nrec, e1_plain;        // E1 -> E2 when several warps share a tile (k_small)
};
using WarpScratch = WarpScratchT<1>;
#ifndef PARPA_SPARSE_K
#define PARPA_SPARSE_K 4
#endif
constexpr int SPARSE_K = PARPA_SPARSE_K;    // super tiles of SPARSE_K * 2 KB
template <int K> struct UnitBits {          // unit-local positions: POS_BITS bits; field lengths: LEN_MASK
  static constexpr uint32_t POS_BITS = K == 1 ? 11u : K == 2 ? 12u : 13u;
  static constexpr uint32_t POS_MASK = (1u << POS_BITS) - 1u;
  static constexpr uint32_t LEN_MASK = K == 1 ? 0xFFFu : (1u << (31u - POS_BITS)) - 1u;
};
static_assert(SPARSE_K == 2 || SPARSE_K == 4, "UnitBits covers K = 1, 2, 4");
template <int K> struct Masks {             // a lane's K chunks (chunk lane * K + j of the unit)
  unsigned long long D[K], F[K], R[K], V[K];
};
#ifndef PARPA_E2_ROWS_MIN
#define PARPA_E2_ROWS_MIN 16
#endif
constexpr uint32_t E2_ROWS_MIN = PARPA_E2_ROWS_MIN;  // tiles with at least this many rows: column-uniform E2
constexpr int E2_ROWS_MIN_MAX = 32;
static_assert(E2_ROWS_MIN <= E2_ROWS_MIN_MAX, "c_rcp16 covers nrows < 32");
constexpr uint32_t E1A_SELECT_MAX = 32;              // tiles with at most this many delimiters: one select round
// 65536/d + 1: (n * c_rcp16[d]) >> 16 == n / d exactly for every d < 32 and n < 1024 (the numerators are < 128)
__constant__ uint32_t c_rcp16[E2_ROWS_MIN_MAX] = {0u, 65537u, 32769u, 21846u, 16385u, 13108u, 10923u, 9363u, 8193u,
                                                   7282u, 6554u, 5958u, 5462u, 5042u, 4682u, 4370u, 4097u, 3856u, 3641u,
                                                   3450u, 3277u, 3121u, 2979u, 2850u, 2731u, 2622u, 2521u, 2428u, 2341u,
                                                   2260u, 2185u, 2115u};
constexpr uint32_t FIELD_WRITTEN = 0xFFFFFFFFu;   // E1 already wrote this field
constexpr uint32_t FIELD_FAR = 0xFFFFFFFEu;       // field 0 began before the tile: see WarpScratch::f0

__device__ __forceinline__ void stash_chunk(uint32_t *buf, int lane, const uint32_t (&v)[16]) {
  uint4 *b = reinterpret_cast<uint4 *>(buf) + lane * 4;
#pragma unroll
  for (int u = 0; u < 4; u++) b[u] = make_uint4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
}

struct TileSrc {                       // raw field bytes: shared-memory tile copy, global before it
  const KArgs *a;
  const uint8_t *tb;                   // scratch bytes
  unsigned long long tbase;            // global position of tile byte 0
  unsigned long long pos, end;
  bool ok;
  __device__ __forceinline__ bool next(uint8_t &c) {
    if (pos > end) return false;
    unsigned long long p = pos++;
    c = p >= tbase ? tb[p - tbase] : fetch_byte(*a, p, ok);
    return true;
  }
};

template <bool TS>
__device__ __forceinline__ void write_value(const KArgs &a, const ColDesc *cd, uint32_t c, unsigned long long row,
                                            unsigned long long fd, unsigned long long ld, bool ic, bool empty,
                                            const uint8_t *tb, unsigned long long tbase,
                                            unsigned long long tb_lim = ~0ull) {
  long long v = 0;
  int ok = 0;
  if (empty) {
    if (cd->has_def) { v = cd->def_bits; ok = 1; }
  } else if (ic) {
    push_defer(a, cd, fd, ld, row, c, 1u);
    return;
  } else {
    int res = 2;
    const unsigned long long L = ld + 1 - fd;
    // the field's first bytes as a register window from the tile copy in shared memory (a field that
    // began in an earlier tile — at most field 0 of the tile — takes the byte-wise path below)
    const bool is_ts = TS && cd->type == T_TIMESTAMP;
#ifdef PARPA_BISECT_A
    if (fd >= tbase && L <= (is_ts ? 26ull : 16ull)) {
#else
    if (fd >= tbase && L <= (is_ts ? 26ull : 16ull) && fd - tbase + 36u <= tb_lim) {
#endif
      const uint32_t o = (uint32_t)(fd - tbase), sh = (o & 3u) * 8u;
      const uint32_t *w = reinterpret_cast<const uint32_t *>(tb) + (o >> 2);
      const bool isf = cd->type == T_FLOAT64;
      if (is_ts) {
        uint32_t x[7] = {0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < 7; k++) x[k] = __funnelshift_r(w[k], w[k + 1], sh);
        res = conv_timestamp_words(x, (int)L, v);
      } else if (L <= 4ull) {
        res = conv_window4(__funnelshift_r(w[0], w[1], sh), (uint32_t)L, isf, v);
      } else if (L <= 8ull) {
        const uint32_t w0 = w[0], w1 = w[1], w2 = w[2];
        const unsigned long long x8 = (unsigned long long)__funnelshift_r(w0, w1, sh) |
                                      ((unsigned long long)__funnelshift_r(w1, w2, sh) << 32);
        res = conv_window8(x8, (uint32_t)L, isf, v);
      } else {
        const uint32_t w0 = w[0], w1 = w[1], w2 = w[2], w3 = w[3], w4 = w[4];
        res = conv_window(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh), __funnelshift_r(w2, w3, sh),
                          __funnelshift_r(w3, w4, sh), (uint32_t)L, isf, v);
      }
    }
    if (res == 2 && L < COLLAB_MIN) {                // (long fields: push_defer -> block / device tier)
      TileSrc src{&a, tb, tbase, fd, ld, true};
      res = conv_typed<TS>(src, cd->type, v);
      if (!src.ok) res = 2;
    }
    if (res == 2) { push_defer(a, cd, fd, ld, row, c, 0u); return; }
    ok = res;
    if (!ok) v = 0;
  }
  st_col(reinterpret_cast<long long *>(cd->val) + row, v);
  st_col(cd->valid + row, (uint8_t)ok);
}

// The common case of write_value, inline: a non-empty field inside the tile copy, without inner control
// bytes, of at most 8 characters (26 for a timestamp), converted from a register window.  o = tile offset
// of its first byte.  Everything else goes to write_value (empty / default, deferred, long fields).
template <bool TS>
__device__ __forceinline__ void write_value_tile(const KArgs &a, const ColDesc *cd, uint32_t type, uint32_t c,
                                                 unsigned long long row, uint32_t o, uint32_t len, bool ic, bool far,
                                                 unsigned long long off, const uint8_t *tb, unsigned long long tbase,
                                                 unsigned long long tb_lim = ~0ull) {
  long long v = 0;
  int res = 2;
  // (tb_lim: bytes readable from tb — the staged tile's pad, or the input's end for a global-memory unit)
#ifdef PARPA_BISECT_A
  if (!(ic || far) && len - 1u < (TS && type == T_TIMESTAMP ? 26u : 8u)) {
#else
  if (!(ic || far) && len - 1u < (TS && type == T_TIMESTAMP ? 26u : 8u) && o + 36u <= tb_lim) {
#endif
    const uint32_t sh = (o & 3u) * 8u;
    const uint32_t *w = reinterpret_cast<const uint32_t *>(tb) + (o >> 2);
    const bool isf = type == T_FLOAT64;
    if (TS && type == T_TIMESTAMP) {
      uint32_t x[7] = {0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int k = 0; k < 7; k++) x[k] = __funnelshift_r(w[k], w[k + 1], sh);
      res = conv_timestamp_words(x, (int)len, v);
#ifndef PARPA_CONV8_ONLY
    } else if (len <= 4u) {
      res = conv_window4(__funnelshift_r(w[0], w[1], sh), len, isf, v);
#endif
    } else {
      const uint32_t w0 = w[0], w1 = w[1], w2 = w[2];
      const unsigned long long x8 = (unsigned long long)__funnelshift_r(w0, w1, sh) |
                                    ((unsigned long long)__funnelshift_r(w1, w2, sh) << 32);
      res = conv_window8(x8, len, isf, v);
    }
  }
  if (res == 2) {
    write_value<TS>(a, cd, c, row, off, off + len - 1, ic, len == 0, tb, tbase, tb_lim);
    return;
  }
  st_col(reinterpret_cast<long long *>(cd->val) + row, v);
  st_col(cd->valid + row, (uint8_t)res);
}

// Per-warp emission of one tile (S6+S7).  prefix = everything before the tile (seed included).
// E1a: each lane appends its delimiters (tile position | record bit) to the warp's delimiter list at
//      its exclusive delimiter count, and publishes its DATA / CTRL words and CTRL prefix counts.
// E1b: one lane per field: the first / last DATA byte between the two delimiters from the DATA words
//      (ffs / clz, usually one word), inner control bytes from the CTRL prefix counts, record and
//      column from ballots over the record bits.  Only field 0 can have begun in an earlier tile; it
//      is combined with the prefix's open-field carry (P:408-414 extended with the carries).
// E2:  column-major writes (below).
template <class WS>
__device__ __forceinline__ uint32_t kcount(const WS *ws, uint32_t x) {   // CTRL bytes before x
  return ws->kpre[x >> 5] + __popc(ws->kmask[x >> 5] & ((1u << (x & 31u)) - 1u));
}
// NP > 1 (k_small): NP warps share one tile — part 0 runs E0/E1 into its scratch `ws`, a named barrier
// (bar, NP warps) publishes it, and every part writes the columns c = part, part + NP, ... in E2 (the
// column-uniform path) or every NP-th item (the flattened path).  NP == 1 is the one-warp-per-tile path.
template <bool TS, int NP = 1, bool SK = true, int K = 1>
__device__ __forceinline__ void emit_tile(const KArgs &a, const ColDesc *cols, WarpScratchT<K> *ws, const Seg &prefix,
                          const Masks<K> &m, unsigned long long tbase_g, unsigned long long cbase,
                          EmitCounters &cnt, uint32_t part = 0, int bar = 0) {
  static_assert(K == 1 || NP == 1, "super tiles are one warp per unit");
  constexpr uint32_t POSM = UnitBits<K>::POS_MASK, LSH = UnitBits<K>::POS_BITS, LENM = UnitBits<K>::LEN_MASK;
  const int lane = threadIdx.x & 31;
  uint32_t nf = 0, nrec = 0;
  bool plain = false, need_e1b = false;
  if (NP == 1 || part == 0) {
  unsigned long long Kmj[K];
  // per-lane (delimiters << 16 | records) and CTRL counts -> exclusive offsets, tile totals
  uint32_t mine = 0, kmine = 0;
#pragma unroll
  for (int j = 0; j < K; j++) {
    Kmj[j] = m.V[j] & ~m.D[j] & ~m.F[j];
    mine += (uint32_t)__popcll(m.R[j]) | ((uint32_t)__popcll(m.F[j]) << 16);
    kmine += (uint32_t)__popcll(Kmj[j]);
  }
  uint32_t inc = mine, kinc = kmine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d), ko = __shfl_up_sync(0xffffffffu, kinc, d);
    if (lane >= d) { inc += o; kinc += ko; }
  }
  const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
  nf = tot >> 16;
  nrec = tot & 0xFFFFu;
  if (nf > (uint32_t)FCAP || nrec >= (uint32_t)RCAP) {       // warp-uniform: dense tile, direct path
    SegT sagg;
    if constexpr (K == 1) {
      const SegT sex = warp_scan_segt(chunk_segt(m.D[0], m.F[0], m.R[0], m.V[0], (uint32_t)lane * CHUNK), sagg);
      emit_chunk<TS, SK>(a, cols, seg_op(prefix, segt_to_seg(sex, tbase_g)), m.D[0], m.F[0], m.R[0], m.V[0], cbase, cnt);
    } else {
      SegT ls = segt_ident();
#pragma unroll
      for (int j = 0; j < K; j++)
        ls = segt_op(ls, chunk_segt(m.D[j], m.F[j], m.R[j], m.V[j], ((uint32_t)lane * K + (uint32_t)j) * CHUNK));
      SegT run = warp_scan_segt(ls, sagg);
#pragma unroll
      for (int j = 0; j < K; j++) {
        emit_chunk<TS, SK>(a, cols, seg_op(prefix, segt_to_seg(run, tbase_g)), m.D[j], m.F[j], m.R[j], m.V[j],
                           cbase + (unsigned long long)j * CHUNK, cnt);
        if (j + 1 < K) run = segt_op(run, chunk_segt(m.D[j], m.F[j], m.R[j], m.V[j], ((uint32_t)lane * K + (uint32_t)j) * CHUNK));
      }
    }
    if (NP == 1) return;
    nf = 0u;                                                  // the other parts have nothing to write
    nrec = 0u;
  } else {
  // ---- E1a ----
  if (K == 1 && nf <= E1A_SELECT_MAX) {
    const unsigned long long Fm = m.F[0], Rm = m.R[0];
    // few delimiters (long fields, e.g. yelp text): lane k selects the k-th delimiter of the tile — the
    // owning chunk by a shuffle binary search over the lanes' exclusive counts, the bit by a popcount
    // binary search — instead of every lane walking its own mask with most lanes idle.
    const uint32_t ex = (inc - mine) >> 16;
    const uint32_t flo = (uint32_t)Fm, fhi = (uint32_t)(Fm >> 32), rlo = (uint32_t)Rm, rhi = (uint32_t)(Rm >> 32);
    const unsigned lt = (1u << lane) - 1u;
    {
      const uint32_t k = (uint32_t)lane;
      uint32_t o = 0;
#pragma unroll
      for (uint32_t st = 16; st; st >>= 1)
        if (__shfl_sync(0xffffffffu, ex, o + st) <= k) o += st;
      const uint32_t r = k - __shfl_sync(0xffffffffu, ex, o);
      const uint32_t ol = __shfl_sync(0xffffffffu, flo, o), oh = __shfl_sync(0xffffffffu, fhi, o);
      const uint32_t rl = __shfl_sync(0xffffffffu, rlo, o), rh = __shfl_sync(0xffffffffu, rhi, o);
      const uint32_t cl = (uint32_t)__popc(ol);
      const bool upper = r >= cl;
      uint32_t word = upper ? oh : ol, rr = upper ? r - cl : r, q = 0;
#pragma unroll
      for (uint32_t sh = 16; sh; sh >>= 1) {
        const uint32_t c = (uint32_t)__popc(word & ((1u << sh) - 1u));
        if (rr >= c) { rr -= c; word >>= sh; q += sh; }
      }
      const bool act = k < nf;
      const uint32_t pos = o * CHUNK + (upper ? 32u : 0u) + q;
      const uint32_t isrec = act ? (((upper ? rh : rl) >> q) & 1u) : 0u;
      const unsigned recm = __ballot_sync(0xffffffffu, isrec != 0u);
      if (act) ws->dlist[k] = (uint16_t)(pos | (isrec << 15));
      if (isrec) ws->rows[__popc(recm & lt)] = (k + 1u) | (pos << 16);
    }
  } else if (K > 1) {
    // Super tiles: the warp selects delimiters cooperatively instead of each lane walking its 256 bytes (the
    // walk ran at ~3 active lanes of 32 on yelp).  The DATA / CTRL words go to shared memory first (the masks
    // then die: register pressure), the lanes' delimiter / record words to `fields` (free until E1b) and the
    // delimiters before each 32-bit segment to `segpre`; lane t then takes the unit's delimiters t, t + 32, ...:
    // owning lane by a shuffle binary search over the lanes' exclusive counts, segment by a binary search over
    // that lane's 2K segment counts, bit by a popcount search.
    constexpr int NS = 2 * K;                                   // 32-bit segments per lane
    uint32_t kex = kinc - kmine, seg = 0;
#pragma unroll
    for (int j = 0; j < K; j++) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const uint32_t si = (uint32_t)lane * NS + (uint32_t)(2 * j + h);
        const uint32_t kw = (uint32_t)(Kmj[j] >> (32 * h)), fw = (uint32_t)(m.F[j] >> (32 * h));
        ws->dmask[si] = (uint32_t)(m.D[j] >> (32 * h));
        ws->kmask[si] = kw;
        ws->kpre[si] = (uint16_t)kex;
        kex += (uint32_t)__popc(kw);
        ws->fields[si] = fw;
        ws->fields[WT * K / 32 + si] = (uint32_t)(m.R[j] >> (32 * h));
        ws->segpre[si] = (uint16_t)seg;
        seg += (uint32_t)__popc(fw);
      }
    }
    __syncwarp();
    const uint32_t ex = (inc - mine) >> 16;                   // this lane's first delimiter index
    const unsigned lt = (1u << lane) - 1u;
    uint32_t jcarry = 0;
    for (uint32_t kb = 0; kb < nf; kb += 32) {                 // warp-uniform rounds
      const uint32_t k = kb + (uint32_t)lane;
      uint32_t o = 0;
#pragma unroll
      for (uint32_t st = 16; st; st >>= 1)
        if (__shfl_sync(0xffffffffu, ex, o + st) <= k) o += st;
      const uint32_t r = k - __shfl_sync(0xffffffffu, ex, o);
      const bool act = k < nf;
      uint32_t s = 0;                                           // segment of lane o holding rank r
#pragma unroll
      for (uint32_t st = NS / 2; st; st >>= 1)
        if (act && ws->segpre[o * NS + s + st] <= r) s += st;
      const uint32_t wi = o * NS + s;
      uint32_t word = act ? ws->fields[wi] : 0u, rr = act ? r - ws->segpre[wi] : 0u, q = 0;
#pragma unroll
      for (uint32_t sh = 16; sh; sh >>= 1) {
        const uint32_t c = (uint32_t)__popc(word & ((1u << sh) - 1u));
        if (rr >= c) { rr -= c; word >>= sh; q += sh; }
      }
      const uint32_t pos = (o * K + (s >> 1)) * CHUNK + (s & 1u) * 32u + q;
      const uint32_t isrec = act ? ((ws->fields[WT * K / 32 + wi] >> q) & 1u) : 0u;
      const unsigned recm = __ballot_sync(0xffffffffu, isrec != 0u);
      if (act) ws->dlist[k] = (uint16_t)(pos | (isrec << 15));
      if (isrec) ws->rows[jcarry + __popc(recm & lt)] = (k + 1u) | (pos << 16);
      jcarry += (uint32_t)__popc(recm);
    }
    __syncwarp();                                               // `fields` is rewritten by E1b
  } else {
    uint32_t k = (inc - mine) >> 16, jr = (inc - mine) & 0xFFFFu;
#pragma unroll
    for (int j = 0; j < K; j++) {
      const uint32_t base = ((uint32_t)lane * K + (uint32_t)j) * CHUNK;
#pragma unroll
      for (int h = 0; h < 2; h++) {                      // 32-bit halves: no 64-bit bit arithmetic per step
        uint32_t fm = (uint32_t)(m.F[j] >> (32 * h));
        const uint32_t rm = (uint32_t)(m.R[j] >> (32 * h)), hb = base + 32u * (uint32_t)h;
        while (fm) {
          const uint32_t p = (uint32_t)__ffs(fm) - 1u;
          fm &= fm - 1u;
          const uint32_t pos = hb + p, isrec = (rm >> p) & 1u;
          ws->dlist[k++] = (uint16_t)(pos | (isrec << 15));
          if (isrec) ws->rows[jr++] = k | (pos << 16);   // end field index | record delimiter position
        }
      }
    }
  }
  if constexpr (K > 1) {
    // (written before the select above)
  } else if constexpr (K == 1) {
    ws->dmask[2 * lane] = (uint32_t)m.D[0];
    ws->dmask[2 * lane + 1] = (uint32_t)(m.D[0] >> 32);
    ws->kmask[2 * lane] = (uint32_t)Kmj[0];
    ws->kmask[2 * lane + 1] = (uint32_t)(Kmj[0] >> 32);
    const uint32_t kex = kinc - kmine;
    ws->kpre[2 * lane] = (uint16_t)kex;
    ws->kpre[2 * lane + 1] = (uint16_t)(kex + __popc((uint32_t)Kmj[0]));
  } else {
    uint32_t kex = kinc - kmine;
#pragma unroll
    for (int j = 0; j < K; j++) {
      const uint32_t wi = 2u * ((uint32_t)lane * K + (uint32_t)j);
      ws->dmask[wi] = (uint32_t)m.D[j];
      ws->dmask[wi + 1] = (uint32_t)(m.D[j] >> 32);
      ws->kmask[wi] = (uint32_t)Kmj[j];
      ws->kmask[wi + 1] = (uint32_t)(Kmj[j] >> 32);
      ws->kpre[wi] = (uint16_t)kex;
      kex += __popc((uint32_t)Kmj[j]);
      ws->kpre[wi + 1] = (uint16_t)kex;
      kex += __popc((uint32_t)(Kmj[j] >> 32));
    }
  }
  __syncwarp();
  const uint32_t ktot = __shfl_sync(0xffffffffu, kinc, 31);    // CTRL bytes in the tile (warp-uniform)
  plain = ktot == 0u;
  if (plain) {
    // E1b' (no CTRL byte in the tile): field k is the byte range between delimiters k-1 and k, all DATA,
    // so E2 reads it straight from the delimiter list.  Only field 0 (which may continue a field of an
    // earlier tile) needs an entry; extra fields (column >= C) are counted per row.
    const uint32_t c0 = prefix.col;
    uint32_t extra = 0;
    const uint32_t last_end = nrec ? (ws->rows[nrec - 1] & 0xFFFFu) : 0u;
    const uint32_t nrows = nrec + (nf > last_end ? 1u : 0u);
    for (uint32_t j = lane; j < nrows; j += 32) {
      const uint32_t start = j ? (ws->rows[j - 1] & 0xFFFFu) : 0u, end = j < nrec ? (ws->rows[j] & 0xFFFFu) : nf;
      const uint32_t cs = j ? 0u : c0, hi = cs + (end - start), lo = max(a.C, cs);
      if (hi > lo) extra += hi - lo;
    }
    if (lane == 0 && nf) {
      const uint32_t p = ws->dlist[0] & POSM;
      unsigned long long cfd = prefix.fd, cld = prefix.ld;
      uint32_t cfl = prefix.flags & (F_IC | F_PC | F_PRE);
      open_combine(cfd, cld, cfl, p ? tbase_g : NONE, p ? tbase_g + p - 1u : NONE, 0u);
      uint32_t e;
      if (cfd == NONE) {
        e = p;
      } else {
        const unsigned long long L = cld + 1 - cfd;
        const long long rel = (long long)cfd - (long long)tbase_g;
        const uint32_t icf = (cfl & F_IC) ? 0x80000000u : 0u;
        if (rel >= 0 && L <= (unsigned long long)WT * K) {
          e = (uint32_t)rel | ((uint32_t)L << LSH) | icf;
        } else if (L >= 0x7FFFFFFFull || rel < -0x7FFFFFFFll) {   // huge / far-away: write it here
          emit_field<TS, SK>(a, cols, prefix.recs, c0, cfd, cld, cfl, tbase_g + p, cnt);
          e = FIELD_WRITTEN;
          if (c0 >= a.C) cnt.extra--;                           // emit_field counted it already
        } else {
          ws->f0 = make_uint2((uint32_t)(int32_t)rel, (uint32_t)L | icf);
          e = FIELD_FAR;
        }
      }
      ws->fields[0] = e;
    }
    cnt.extra += extra;
  } else {
  // ---- E1b ----
  if (NP == 1) {
  {
    const uint32_t c0 = prefix.col;
    uint32_t jcarry = 0, extra = 0;
    int lastrec = -1;
    const unsigned lt = (1u << lane) - 1u;
    for (uint32_t kb = 0; kb < nf; kb += 32) {
      const uint32_t k = kb + (uint32_t)lane;
      const bool act = k < nf;
      const uint32_t dl = act ? ws->dlist[k] : 0u;
      const uint32_t p = dl & POSM;
      const bool isrec = act && (dl >> 15);
      const unsigned recm = __ballot_sync(0xffffffffu, isrec);
      const uint32_t jr = jcarry + __popc(recm & lt);
      const unsigned before = recm & lt;
      const int lr = before ? (int)(kb + 31u - __clz(before)) : lastrec;
      const uint32_t c = lr >= 0 ? k - (uint32_t)lr - 1u : c0 + k;
      extra += (uint32_t)__popc(__ballot_sync(0xffffffffu, act && c >= a.C));
      if (act) {
        const uint32_t x = k ? (ws->dlist[k - 1] & POSM) + 1u : 0u;   // field bytes [x, p)
        // inner / surrounding control bytes only matter for converted columns (a span is [first, last DATA])
        const uint32_t ty = c < a.C ? cols[c].type : (uint32_t)T_SKIP;
        const bool typed = ty != T_SPAN && ty != T_SKIP;
        int fd = -1, ld = -1;
        uint32_t ic = 0;
        if (ktot == 0u) {                                     // no CTRL byte: [x, p) is all DATA
          if (x < p) { fd = (int)x; ld = (int)p - 1; }
        } else {
          if (x < p) {
            uint32_t w = x >> 5;
            uint32_t bits = ws->dmask[w] & (0xFFFFFFFFu << (x & 31u));
            const uint32_t wp = p >> 5;
            while (!bits && w < wp) bits = ws->dmask[++w];
            if (bits) {
              const uint32_t f = (w << 5) + (uint32_t)__ffs(bits) - 1u;
              if (f < p) fd = (int)f;
            }
          }
          if (fd >= 0) {
            const uint32_t y = p - 1u;
            uint32_t w = y >> 5;
            uint32_t bits = ws->dmask[w] & (0xFFFFFFFFu >> (31u - (y & 31u)));
            while (!bits) bits = ws->dmask[--w];
            ld = (int)((w << 5) + 31u - (uint32_t)__clz(bits));
            if (typed && ld > fd && kcount(ws, (uint32_t)ld) > kcount(ws, (uint32_t)fd + 1u)) ic = 0x80000000u;
          }
        }
        uint32_t e = fd < 0 ? p : ((uint32_t)fd | ((uint32_t)(ld + 1 - fd) << LSH) | ic);  // empty: (delim, 0)
        if (K > 1 && typed && fd >= 0)    // super tiles read typed bytes from global memory in E2: start the load now
#ifdef PARPA_PREF_L2
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a.in + (tbase_g - a.base) + (unsigned)fd));
#else
          asm volatile("prefetch.global.L1 [%0];" ::"l"(a.in + (tbase_g - a.base) + (unsigned)fd));
#endif
        if (k == 0) {                                         // may continue a field of an earlier tile
          uint32_t fl = ic ? F_IC : 0u;
          if (ktot && typed) {
            if (fd >= 0) {
              if (kcount(ws, (uint32_t)fd) > 0u) fl |= F_PRE;
              if (kcount(ws, p) > kcount(ws, (uint32_t)ld + 1u)) fl |= F_PC;
            } else if (kcount(ws, p) > 0u) {
              fl |= F_PRE;
            }
          }
          unsigned long long cfd = prefix.fd, cld = prefix.ld;
          uint32_t cfl = prefix.flags & (F_IC | F_PC | F_PRE);
          open_combine(cfd, cld, cfl, fd >= 0 ? tbase_g + (unsigned)fd : NONE, fd >= 0 ? tbase_g + (unsigned)ld : NONE,
                       fl);
          if (cfd == NONE) {
            e = p;
          } else {
            const unsigned long long L = cld + 1 - cfd;
            const long long rel = (long long)cfd - (long long)tbase_g;
            const uint32_t icf = (cfl & F_IC) ? 0x80000000u : 0u;
            if (rel >= 0 && L <= (unsigned long long)WT * K) {
              e = (uint32_t)rel | ((uint32_t)L << LSH) | icf;
            } else if (L >= 0x7FFFFFFFull || rel < -0x7FFFFFFFll) {   // huge / far-away: write it here
              emit_field<TS, SK>(a, cols, prefix.recs + jr, c, cfd, cld, cfl, tbase_g + p, cnt);
              e = FIELD_WRITTEN;
              if (c >= a.C) cnt.extra--;                      // emit_field counted it already
            } else {
              ws->f0 = make_uint2((uint32_t)(int32_t)rel, (uint32_t)L | icf);
              e = FIELD_FAR;
            }
          }
        }
        ws->fields[k] = e;
      }
      jcarry += (uint32_t)__popc(recm);
      if (recm) lastrec = (int)(kb + 31u - __clz(recm));
    }
    if (lane == 0) cnt.extra += extra;
  }
  } else {
    need_e1b = true;                                        // split over the NP parts after the barrier
  }
  }
  }                                                         // (not dense)
  }                                                         // (E0 / E1: the whole tile or part 0)
  __syncwarp();
  if (NP > 1) {                                             // part 0's E1 -> every part
    if (part == 0 && lane == 0) { ws->e1_nf = nf; ws->e1_nrec = nrec; ws->e1_plain = plain ? 1u : 0u; }
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(NP * 32) : "memory");
    nf = ws->e1_nf;
    nrec = ws->e1_nrec;
    plain = ws->e1_plain != 0u;
    (void)need_e1b;
    if (!plain && nf > 0u) {
      // E1b split over the NP parts (k_small: the tile's E1 latency is on the critical path): part p takes the
      // 32-field blocks p, p + NP, ..., its record / column carries recomputed from the delimiter list
      const uint32_t c0 = prefix.col;
      const unsigned lt = (1u << lane) - 1u;
      uint32_t extra = 0;
      for (uint32_t kb = 32u * part; kb < nf; kb += 32u * NP) {
        uint32_t jcarry = 0;                                // records before kb, and the last of them
        int lastrec = -1;
        for (uint32_t b = 0; b < kb; b += 32) {
          const uint32_t kk = b + (uint32_t)lane;
          const unsigned mr = __ballot_sync(0xffffffffu, kk < nf && (ws->dlist[kk] >> 15));
          jcarry += (uint32_t)__popc(mr);
          if (mr) lastrec = (int)(b + 31u - __clz(mr));
        }
      const uint32_t k = kb + (uint32_t)lane;
      const bool act = k < nf;
      const uint32_t dl = act ? ws->dlist[k] : 0u;
      const uint32_t p = dl & POSM;
      const bool isrec = act && (dl >> 15);
      const unsigned recm = __ballot_sync(0xffffffffu, isrec);
      const uint32_t jr = jcarry + __popc(recm & lt);
      const unsigned before = recm & lt;
      const int lr = before ? (int)(kb + 31u - __clz(before)) : lastrec;
      const uint32_t c = lr >= 0 ? k - (uint32_t)lr - 1u : c0 + k;
      extra += (uint32_t)__popc(__ballot_sync(0xffffffffu, act && c >= a.C));
      if (act) {
        const uint32_t x = k ? (ws->dlist[k - 1] & POSM) + 1u : 0u;   // field bytes [x, p)
        // inner / surrounding control bytes only matter for converted columns (a span is [first, last DATA])
        const uint32_t ty = c < a.C ? cols[c].type : (uint32_t)T_SKIP;
        const bool typed = ty != T_SPAN && ty != T_SKIP;
        int fd = -1, ld = -1;
        uint32_t ic = 0;
        if (false) {                                          // (the tile has CTRL bytes)                                     // no CTRL byte: [x, p) is all DATA
          if (x < p) { fd = (int)x; ld = (int)p - 1; }
        } else {
          if (x < p) {
            uint32_t w = x >> 5;
            uint32_t bits = ws->dmask[w] & (0xFFFFFFFFu << (x & 31u));
            const uint32_t wp = p >> 5;
            while (!bits && w < wp) bits = ws->dmask[++w];
            if (bits) {
              const uint32_t f = (w << 5) + (uint32_t)__ffs(bits) - 1u;
              if (f < p) fd = (int)f;
            }
          }
          if (fd >= 0) {
            const uint32_t y = p - 1u;
            uint32_t w = y >> 5;
            uint32_t bits = ws->dmask[w] & (0xFFFFFFFFu >> (31u - (y & 31u)));
            while (!bits) bits = ws->dmask[--w];
            ld = (int)((w << 5) + 31u - (uint32_t)__clz(bits));
            if (typed && ld > fd && kcount(ws, (uint32_t)ld) > kcount(ws, (uint32_t)fd + 1u)) ic = 0x80000000u;
          }
        }
        uint32_t e = fd < 0 ? p : ((uint32_t)fd | ((uint32_t)(ld + 1 - fd) << LSH) | ic);  // empty: (delim, 0)
        if (K > 1 && typed && fd >= 0)    // super tiles read typed bytes from global memory in E2: start the load now
#ifdef PARPA_PREF_L2
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a.in + (tbase_g - a.base) + (unsigned)fd));
#else
          asm volatile("prefetch.global.L1 [%0];" ::"l"(a.in + (tbase_g - a.base) + (unsigned)fd));
#endif
        if (k == 0) {                                         // may continue a field of an earlier tile
          uint32_t fl = ic ? F_IC : 0u;
          if (typed) {
            if (fd >= 0) {
              if (kcount(ws, (uint32_t)fd) > 0u) fl |= F_PRE;
              if (kcount(ws, p) > kcount(ws, (uint32_t)ld + 1u)) fl |= F_PC;
            } else if (kcount(ws, p) > 0u) {
              fl |= F_PRE;
            }
          }
          unsigned long long cfd = prefix.fd, cld = prefix.ld;
          uint32_t cfl = prefix.flags & (F_IC | F_PC | F_PRE);
          open_combine(cfd, cld, cfl, fd >= 0 ? tbase_g + (unsigned)fd : NONE, fd >= 0 ? tbase_g + (unsigned)ld : NONE,
                       fl);
          if (cfd == NONE) {
            e = p;
          } else {
            const unsigned long long L = cld + 1 - cfd;
            const long long rel = (long long)cfd - (long long)tbase_g;
            const uint32_t icf = (cfl & F_IC) ? 0x80000000u : 0u;
            if (rel >= 0 && L <= (unsigned long long)WT * K) {
              e = (uint32_t)rel | ((uint32_t)L << LSH) | icf;
            } else if (L >= 0x7FFFFFFFull || rel < -0x7FFFFFFFll) {   // huge / far-away: write it here
              emit_field<TS, SK>(a, cols, prefix.recs + jr, c, cfd, cld, cfl, tbase_g + p, cnt);
              e = FIELD_WRITTEN;
              if (c >= a.C) cnt.extra--;                      // emit_field counted it already
            } else {
              ws->f0 = make_uint2((uint32_t)(int32_t)rel, (uint32_t)L | icf);
              e = FIELD_FAR;
            }
          }
        }
        ws->fields[k] = e;
      }
      }
      if (lane == 0) cnt.extra += extra;
      __syncwarp();
      asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(NP * 32) : "memory");   // every field entry written
    }
  }
  // ---- E2 ----
  // the unit's bytes: the staged copy (K = 1), or global memory (super tiles: few typed fields)
  const uint8_t *tb = K == 1 ? reinterpret_cast<const uint8_t *>(ws->bytes) : a.in + (tbase_g - a.base);
  const unsigned long long tb_lim = K == 1 ? ~0ull : a.len - (tbase_g - a.base);
  const uint32_t last_end = nrec ? (ws->rows[nrec - 1] & 0xFFFFu) : 0u;
  const uint32_t nrows = nrec + (nf > last_end ? 1u : 0u);
  if (nrows == 0) {                                         // no delimiter: the open field continues
    __syncwarp();
    if (NP > 1) asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(NP * 32) : "memory");
    return;
  }
  const uint32_t c0 = prefix.col;
  const unsigned long long r0 = prefix.recs;
  if (nrows >= E2_ROWS_MIN) {
    // Column-uniform writes (tiles with many short records, e.g. taxi / clf): lanes = tile rows, one
    // column per step.  The row bookkeeping is done once per lane, the column descriptor and type are
    // warp-uniform (no type divergence, span columns skip conversion as a whole warp), and each store
    // covers consecutive rows of one column.
    for (uint32_t jb = 0; jb < nrows; jb += 32) {
      const uint32_t ji = jb + (uint32_t)lane;
      const bool closed = ji < nrec;
      uint32_t start = 0u, end = 0u, cs = 0u, dpos = 0u;
      unsigned long long row = 0ull;
      bool live = ji < nrows;
      if (live) {
        start = ji == 0 ? 0u : (ws->rows[ji - 1] & 0xFFFFu);
        const uint32_t rw = closed ? ws->rows[ji] : 0u;
        end = closed ? (rw & 0xFFFFu) : nf;
        dpos = rw >> 16;
        cs = ji == 0 ? c0 : 0u;
        row = out_row<SK>(a, r0 + ji);
        live = row < a.cap;
      }
      if ((NP == 1 || part == 0) && live && closed && end - start + cs < a.C) cnt.missing++;   // short record
      for (uint32_t c = (NP == 1 ? 0u : part); c < a.C; c += NP) {   // warp-uniform
        const ColDesc *cd = cols + c;
        const uint32_t type = cd->type;
        if (type == T_SKIP) continue;
        if (!live || c < cs) continue;                        // c < cs: written by an earlier tile
        const uint32_t k = start + (c - cs);
        if (k < end) {
          if (plain && k) {                                    // the common case: [x, p), all DATA, in the tile
            const uint32_t x = (ws->dlist[k - 1] & POSM) + 1u, len = (ws->dlist[k] & POSM) - x;
            const unsigned long long off = tbase_g + x;        // empty (x == p): (delimiter position, 0)
            st_col(cd->off + row, off);
            st_col(cd->len + row, len);
            if (type != T_SPAN) write_value_tile<TS>(a, cd, type, c, row, x, len, false, false, off, tb, tbase_g, tb_lim);
            continue;
          }
          const uint32_t e = ws->fields[k];
          if (k) {                                             // only field 0 can carry a special entry
            const uint32_t o = e & POSM, len = (e >> LSH) & LENM;
            const unsigned long long off = tbase_g + o;
            st_col(cd->off + row, off);
            st_col(cd->len + row, len);
            if (type != T_SPAN) write_value_tile<TS>(a, cd, type, c, row, o, len, (e >> 31) != 0, false, off, tb, tbase_g, tb_lim);
            continue;
          }
          if (e == FIELD_WRITTEN) continue;
          uint32_t len, o;
          unsigned long long off;
          bool ic;
          const bool far = e == FIELD_FAR;
          if (far) {
            const uint2 f = ws->f0;
            off = tbase_g + (unsigned long long)(long long)(int32_t)f.x;
            len = f.y & 0x7FFFFFFFu;
            ic = (f.y >> 31) != 0;
            o = 0u;
          } else {
            o = e & POSM;
            off = tbase_g + o;
            len = (e >> LSH) & LENM;
            ic = (e >> 31) != 0;
          }
          st_col(cd->off + row, off);
          st_col(cd->len + row, len);
          if (type != T_SPAN) write_value_tile<TS>(a, cd, type, c, row, o, len, ic, far, off, tb, tbase_g, tb_lim);
        } else if (closed) {
          st_col(cd->off + row, tbase_g + dpos);
          st_col(cd->len + row, 0xFFFFFFFFu);
          if (type != T_SPAN) {
            st_col(reinterpret_cast<long long *>(cd->val) + row, cd->has_def ? cd->def_bits : 0ll);
            st_col(cd->valid + row, (uint8_t)(cd->has_def ? 1 : 0));
          }
        }
      }
    }
    __syncwarp();
    if (NP > 1) asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(NP * 32) : "memory");
    return;
  }
  // Column-major writes: (column, tile row) items flattened over the lanes, rows fastest, so a warp
  // step stores consecutive rows of one or two columns (coalesced) with every lane busy; numeric
  // columns share one converter, so mixed int / float steps do not diverge.
  const uint32_t total = a.C * nrows;
  const uint32_t it0 = (uint32_t)lane + 32u * (NP == 1 ? 0u : part), step = 32u * NP;
  // division by nrows (< E2_ROWS_MIN here) as a multiply by a 16-bit reciprocal (exact, see c_rcp16)
  const uint32_t rcp = c_rcp16[nrows];
  uint32_t c = (it0 * rcp) >> 16, jr = it0 - c * nrows;
  const uint32_t dc = (step * rcp) >> 16, djr = step - dc * nrows;
  for (uint32_t it = it0; it < total; it += step) {
    const uint32_t ci = c, ji = jr;
    jr += djr;
    c += dc;
    if (jr >= nrows) { jr -= nrows; c++; }
    const uint32_t start = ji == 0 ? 0u : (ws->rows[ji - 1] & 0xFFFFu);
    const uint32_t end = ji < nrec ? (ws->rows[ji] & 0xFFFFu) : nf;
    const uint32_t cs = ji == 0 ? c0 : 0u;
    if (ci < cs) continue;                                  // written by an earlier tile
    const unsigned long long row = out_row<SK>(a, r0 + ji);
    if (row >= a.cap) continue;
    const uint32_t k = start + (ci - cs);
    const ColDesc *cd = cols + ci;
    const bool skip = cd->type == T_SKIP;
    if (k < end) {
      uint32_t e;
      if (plain && k) {                                     // [x, p) between two delimiters, all DATA
        const uint32_t x = (ws->dlist[k - 1] & POSM) + 1u, p = ws->dlist[k] & POSM;
        e = x < p ? x | ((p - x) << LSH) : p;
      } else {
        e = ws->fields[k];
      }
      if (e == FIELD_WRITTEN || skip) continue;
      uint32_t len, o;
      unsigned long long off;
      bool ic;
      const bool far = e == FIELD_FAR;
      if (far) {
        const uint2 f = ws->f0;
        off = tbase_g + (unsigned long long)(long long)(int32_t)f.x;
        len = f.y & 0x7FFFFFFFu;
        ic = (f.y >> 31) != 0;
        o = 0u;
      } else {
        o = e & POSM;
        off = tbase_g + o;
        len = (e >> LSH) & LENM;
        ic = (e >> 31) != 0;
      }
      st_col(cd->off + row, off);
      st_col(cd->len + row, len);
      if (cd->type != T_SPAN) write_value_tile<TS>(a, cd, cd->type, ci, row, o, len, ic, far, off, tb, tbase_g, tb_lim);
    } else if (ji < nrec) {                                 // record closed with fewer fields
      if (k == end) cnt.missing++;
      if (skip) continue;
      st_col(cd->off + row, tbase_g + (ws->rows[ji] >> 16));
      st_col(cd->len + row, 0xFFFFFFFFu);
      if (cd->type != T_SPAN) {
        st_col(reinterpret_cast<long long *>(cd->val) + row, cd->has_def ? cd->def_bits : 0ll);
        st_col(cd->valid + row, (uint8_t)(cd->has_def ? 1 : 0));
      }
    }
  }
  __syncwarp();
  if (NP > 1) asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(NP * 32) : "memory");   // scratch reusable
}

}  // namespace parpa
#include "parpa_passes.cuh"
namespace parpa {

// ---- two-phase emit kernel (per warp tile, from the stored prefixes; no look-back) ------------------
#ifndef PARPA_EMIT_WARPS
#define PARPA_EMIT_WARPS 16
#define PARPA_EMIT_MINB 2
#endif
constexpr int EMIT_WARPS = PARPA_EMIT_WARPS;
constexpr size_t EMIT_SMEM = EMIT_WARPS * (sizeof(WarpScratchT<1>) > sizeof(WarpScratchT<SPARSE_K>)
                                                ? sizeof(WarpScratchT<1>) : sizeof(WarpScratchT<SPARSE_K>));

// S6+S7 per warp tile from what the scan half stored: the DATA / DELIM / RECORD masks of every chunk
// (k_pass2) and the tile prefix (k_seg_scan).  No LUT, no re-simulation: 2 CTAs per SM.
// Emission of sparse inputs (on average >= 32 bytes per field, e.g. yelp's long text): super tiles of SPARSE_K
// warp tiles per warp.  A kernel of its own, launched next to k_emit (each returns at once when the range is
// not its kind: the decision reads the range's field count, so both agree): in one kernel the 4-chunk masks
// raised the register pressure of the per-tile path until it spilled (taxi +2%, CLF +9%).
__device__ __forceinline__ bool emit_is_sparse(const KArgs &a) {
  const unsigned long long nfl = a.tot_seg ? a.tot_seg->nflds : 0ull;
  return a.emit_k == (uint32_t)SPARSE_K || (a.emit_k == 0u && a.len >= 32ull * (nfl + 1ull));
}
#ifndef PARPA_SPARSE_MINB
#define PARPA_SPARSE_MINB PARPA_EMIT_MINB
#endif
#ifndef PARPA_SPARSE_WARPS
#define PARPA_SPARSE_WARPS 14     // 2 x 14 warps per SM, 72 registers: at 16 x 2 (64 registers) the 4-chunk masks
#endif                            // spill (measured on yelp: 16 -> 2.06 ms, 14 -> 1.81, 12 -> 1.85, 10 -> 1.82)
constexpr int SPARSE_WARPS = PARPA_SPARSE_WARPS;
constexpr size_t SPARSE_SMEM = SPARSE_WARPS * sizeof(WarpScratchT<SPARSE_K>);
template <bool TS, bool SK>
__global__ void __launch_bounds__(SPARSE_WARPS * 32, PARPA_SPARSE_MINB) k_emit_sparse(const KArgs a, const ColsK colsk) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ ColDesc s_cols[MAX_COLS];
  PdlTrigger pdl_trigger;
  for (int c = threadIdx.x; c < (int)a.C; c += blockDim.x) s_cols[c] = colsk.c[c];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  EmitCounters cnt{0ull, 0ull, 0u};
  __syncthreads();
  pdl_wait();
  if (!emit_is_sparse(a)) return;
  const uint32_t nw = gridDim.x * SPARSE_WARPS;
  WarpScratchT<SPARSE_K> *ws4 = reinterpret_cast<WarpScratchT<SPARSE_K> *>(smem) + warp;
  const uint32_t nunits = (a.ntiles + SPARSE_K - 1) / SPARSE_K;
  while (true) {
    uint32_t u = 0;
    if (lane == 0) u = atomicAdd(&a.ctrl->emit_ticket, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= nunits) break;
    const uint32_t t0 = u * SPARSE_K;
    const unsigned long long ustart = (unsigned long long)t0 * WT;
#ifndef PARPA_NO_SPARSE_PREFETCH
    {                                                    // the unit this warp will take about one round later:
      const uint32_t un = u + nw;                        // its masks (3 KB) and tile prefixes into L2
      if (un < nunits) {
        const unsigned long long tn = (unsigned long long)un * SPARSE_K;
        if (lane < 24) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.masks + tn * 96 + (unsigned)lane * 16));
        else if (lane == 24) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.tinfo + tn));
      }
    }
#endif
    Masks<SPARSE_K> mm;
    // chunk lane * K + j of the unit: tile t0 + (lane * K + j) / 32, lane (lane * K + j) % 32 of its masks
    const unsigned long long *mk0 = a.masks + (unsigned long long)t0 * 96;
    if (ustart + (unsigned long long)SPARSE_K * WT <= a.len) {   // every unit but the last: all chunks full
#pragma unroll
      for (int j = 0; j < SPARSE_K; j++) {
        const uint32_t ci = (uint32_t)lane * SPARSE_K + (uint32_t)j;
        const unsigned long long *mk = mk0 + (ci >> 5) * 96 + (ci & 31u);
        mm.D[j] = mk[0]; mm.F[j] = mk[32]; mm.R[j] = mk[64];
        mm.V[j] = ~0ull;
      }
    } else {
#pragma unroll
      for (int j = 0; j < SPARSE_K; j++) {
        const uint32_t ci = (uint32_t)lane * SPARSE_K + (uint32_t)j;
        const unsigned long long cs = ustart + (unsigned long long)ci * CHUNK;
        const int nv = cs >= a.len ? 0 : (int)min((unsigned long long)CHUNK, a.len - cs);
        if (nv > 0) {
          const unsigned long long *mk = mk0 + (ci >> 5) * 96 + (ci & 31u);
          mm.D[j] = mk[0]; mm.F[j] = mk[32]; mm.R[j] = mk[64];
        } else {
          mm.D[j] = mm.F[j] = mm.R[j] = 0ull;
        }
        mm.V[j] = nv >= 64 ? ~0ull : ((1ull << nv) - 1ull);
      }
    }
    emit_tile<TS, 1, SK, SPARSE_K>(a, s_cols, ws4, seg_op(a.seed, a.tinfo[t0].excl), mm, a.base + ustart,
                                   a.base + ustart + (unsigned long long)lane * SPARSE_K * CHUNK, cnt);
  }
  if (lane == 0 && atomicAdd(&a.ctrl->emit_done, 1u) == nw - 1u) {   // last warp out: ready for the next launch
    a.ctrl->emit_done = 0u;
    a.ctrl->emit_ticket = 0u;
  }
  flush_counters(a, cnt);
}

template <bool TS, bool SK>
__global__ void __launch_bounds__(EMIT_WARPS * 32, PARPA_EMIT_MINB) k_emit(const KArgs a, const ColsK colsk) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ ColDesc s_cols[MAX_COLS];
  PdlTrigger pdl_trigger;
  for (int c = threadIdx.x; c < (int)a.C; c += blockDim.x) s_cols[c] = colsk.c[c];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpScratch *ws = reinterpret_cast<WarpScratch *>(smem) + warp;
  EmitCounters cnt{0ull, 0ull, 0u};
  __syncthreads();
  pdl_wait();
  const uint32_t nw = gridDim.x * EMIT_WARPS;
  const uint32_t ntiles = emit_is_sparse(a) ? 0u : a.ntiles;   // k_emit_sparse's range: no tiles here
#ifdef PARPA_EMIT_STATIC
  const uint32_t gw = blockIdx.x * EMIT_WARPS + warp;
  for (uint32_t t = gw; t < ntiles; t += nw) {
#else
  // Tiles are taken in input order from one atomic counter, so the warps writing adjacent tiles (which
  // share the boundary sectors of every output column) stay together in time: with a static grid stride
  // the warps drift apart over ~500 tiles each and the boundary sectors leave L2 half written (DRAM
  // read-modify-write; measured at 4.8 GB of taxi).
#ifdef PARPA_EMIT_TICKET2
  // Tickets are taken one tile ahead: the atomic for the tile after next is in flight while this tile is
  // processed, and the next tile's bytes, masks and prefix are prefetched into L2 as soon as it is known.
  uint32_t tk = 0;
  if (lane == 0) tk = atomicAdd(&a.ctrl->emit_ticket, 2u);
  tk = __shfl_sync(0xffffffffu, tk, 0);
  uint32_t t = tk, tn = tk + 1;
  while (true) {
    if (t >= ntiles) break;
    uint32_t tnn = 0;
    if (lane == 0 && tn < ntiles) tnn = atomicAdd(&a.ctrl->emit_ticket, 1u);
    if (tn < ntiles) {                                   // the warp's next tile into L2
      const unsigned long long tb = (unsigned long long)tn;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a.in + tb * WT + (unsigned long long)lane * CHUNK));
      if (lane < 6) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.masks + tb * 96 + lane * 16));
      if (lane == 6) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.tinfo + tb));
    }
#else
  while (true) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(&a.ctrl->emit_ticket, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= ntiles) break;
#endif
#endif
    const unsigned long long tstart = (unsigned long long)t * WT;
    const unsigned long long cstart = tstart + (unsigned long long)lane * CHUNK;
    const int nvalid = cstart >= a.len ? 0 : (int)min((unsigned long long)CHUNK, a.len - cstart);
    {
      uint32_t v[16];
      load_chunk(a.in + cstart, nvalid, v);
      stash_chunk(ws->bytes, lane, v);
    }
#if defined(PARPA_EMIT_STATIC) || !defined(PARPA_EMIT_TICKET2)
    if (t + nw < ntiles) {                              // the warp's next tile into L2 (2 KB + 768 B masks):
      const unsigned long long tn = (unsigned long long)(t + nw);   // its loads then wait on L2, not DRAM
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a.in + tn * WT + (unsigned long long)lane * CHUNK));
      if (lane < 6) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.masks + tn * 96 + lane * 16));
      else if (lane == 6) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.tinfo + tn));   // and its prefix
    }
#endif
    const unsigned long long *mk = a.masks + (unsigned long long)t * 96 + lane;
    const unsigned long long Dm = mk[0], Fm = mk[32], Rm = mk[64];
    const unsigned long long Vm = nvalid >= 64 ? ~0ull : ((1ull << nvalid) - 1ull);
    const Masks<1> mm{{Dm}, {Fm}, {Rm}, {Vm}};
    emit_tile<TS, 1, SK>(a, s_cols, ws, seg_op(a.seed, a.tinfo[t].excl), mm, a.base + tstart, a.base + cstart, cnt);
#if !defined(PARPA_EMIT_STATIC) && defined(PARPA_EMIT_TICKET2)
    t = tn;
    tn = __shfl_sync(0xffffffffu, tnn, 0);
#endif
  }
#ifndef PARPA_EMIT_STATIC
  if (lane == 0 && atomicAdd(&a.ctrl->emit_done, 1u) == nw - 1u) {   // last warp out: ready for the next launch
    a.ctrl->emit_done = 0u;
    a.ctrl->emit_ticket = 0u;
  }
#endif
  flush_counters(a, cnt);
}

// ---- finalize ---------------------------------------------------------------------------------------
__device__ void finalize_one(const KArgs &a, const DfaK &dfa, const ColsK &colsk) {   // one thread
  Seg tot = a.ntiles ? seg_op(a.seed, *a.tot_seg) : a.seed;
  uint32_t tau = a.ntiles ? *a.tot_tau : NIB_IDENT;
  const uint32_t fin = nib_at(tau, a.seed_dev);
  // the exact final DFA state: the class's member if it has one member, else from the last byte
  uint32_t fin_exact = dfa.hmap[fin];
  if (a.len == 0) {
    fin_exact = a.seed_exact;
  } else if (dfa.merged && (ld_volatile_u32(&a.ctrl->last_cls) & 0x100u)) {   // recorded by pass 2
    const uint32_t cb = ld_volatile_u32(&a.ctrl->last_cls) & 0xFu;
    fin_exact = cb == INV_DEV ? dfa.inv_state : dfa.next_exact[cb][dfa.gob[a.in[a.len - 1]]];
  } else if (dfa.merged) {
    const unsigned long long kc = (a.len - 1) / CHUNK;
    uint32_t x = 0x80u | a.chunk_state[kc];
    for (unsigned long long p = kc * CHUNK; p + 1 < a.len; p++) {
      const uint8_t b = a.in[p];
      x = prmt(dfa.lut[b][2], dfa.lut[b][3], x);
    }
    const uint32_t cb = x & 0xFu;
    fin_exact = cb == INV_DEV ? dfa.inv_state : dfa.next_exact[cb][dfa.gob[a.in[a.len - 1]]];
  }
  EmitCounters cnt{0ull, 0ull, 0u};
  unsigned long long R = tot.recs, nf = tot.nflds;
  unsigned long long first_inv = a.ctrl->inv_neg ? ~a.ctrl->inv_neg : NONE;
  if (a.is_last) {
    uint32_t act = dfa.eoi_state[fin_exact];
    unsigned long long end = a.base + a.len;
    if (act == EOI_RECORD) {                               // implicit record delimiter at EOI
      emit_field<true>(a, colsk.c, R, tot.col, tot.fd, tot.ld, tot.flags & (F_IC | F_PC | F_PRE), end, cnt);
      fill_missing(a, colsk.c, R, tot.col + 1, end, cnt);
      R++;
      nf++;
    } else if (act == EOI_ERROR && first_inv == NONE) {
      first_inv = end;
    }
  }
  unsigned long long missing = a.ctrl->n_missing + cnt.missing;
  unsigned long long extra = a.ctrl->n_extra + cnt.extra;
  unsigned int n_defer = a.ctrl->n_defer;
  const unsigned long long nskipped = a.nskip ? skipped_before(a, R) : 0ull;   // skipped records < R
  int status = ST_OK;
  if (first_inv != NONE) status = ST_EFORMAT;
  else if (a.ctrl->unsupported || cnt.unsupported) status = ST_EUNSUPPORTED;
  else if (R - a.row_base - nskipped > a.cap) status = ST_ENEEDMORE;
  else if ((missing || extra) && a.strict) status = ST_ECOLUMNS;
  if (a.stats) {
    a.stats->records = R - a.row_base - nskipped;
    a.stats->fields = nf - a.seed.nflds;
    a.stats->first_invalid = first_inv;
    a.stats->missing_records = missing;
    a.stats->extra_fields = extra;
    a.stats->deferred_fields = n_defer;              // (of which the block / device tiers: set by k_deferred)
    a.stats->block_fields = 0u;
    a.stats->device_fields = 0u;
    a.stats->status = status;
    a.stats->final_state = fin_exact;
  }
}
__global__ void k_finalize(const __grid_constant__ KArgs a, const __grid_constant__ DfaK dfa,
                           const __grid_constant__ ColsK colsk) {
  PdlTrigger pdl_trigger;
  pdl_wait();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  finalize_one(a, dfa, colsk);
}

// ---- device-tier conversion of deferred fields ------------------------------------------------------
struct DfaDataSrc {                   // DATA bytes of [fd, ld], re-simulated from the chunk entry state
  const KArgs *a;
  const DfaK *d;
  unsigned long long pos, end;
  uint32_t x;
  bool ok;
  __device__ bool next(uint8_t &c) {
    while (pos <= end) {
      const uint8_t b = fetch_byte(*a, pos, ok);       // the left context (halo) before the range
      pos++;
      uint32_t step_lo = d->lut[b][2], step_hi = d->lut[b][3];
      uint32_t prev = x;
      x = prmt(step_lo, step_hi, prev);
      if ((x & KC_MASK) == 0u) { c = b; return true; }
    }
    return false;
  }
};

// one deferred field: the exact device-tier conversion of its DATA bytes
template <bool TS>
__device__ void convert_deferred(const KArgs &a, const DfaK &dfa, const ColDesc *cd, unsigned long long fd,
                                 unsigned long long ld, unsigned long long row, uint32_t ic) {
  long long v = 0;
  int ok = 0;
  if (ic) {
    unsigned long long from;                         // a position whose state is known, and the state
    uint32_t x;
    bool known = true;
    if (fd >= a.base) {
      const unsigned long long k = (fd - a.base) / CHUNK;
      from = a.base + k * CHUNK;
      x = 0x80u | a.chunk_state[k];
    } else if (a.left && a.left_state != 0xFFu && fd >= a.base - a.left_len) {
      from = a.base - a.left_len;                    // the halo's first byte, whose state the sender gave
      x = 0x80u | a.left_state;
    } else {
      known = false;                                 // a span crossing into a previous range with inner
      from = fd;                                     // control bytes and no left context: unsupported
      x = 0u;
      atomicOr(&a.ctrl->unsupported, 1u);
    }
    if (known) {
      bool okb = true;
      for (unsigned long long p = from; p < fd; p++) {
        const uint8_t b = fetch_byte(a, p, okb);
        x = prmt(dfa.lut[b][2], dfa.lut[b][3], x);
      }
      DfaDataSrc src{&a, &dfa, fd, ld, x, true};
      ok = conv_typed_exact<TS>(src, cd->type, v);
      if (!src.ok || !okb) { ok = 0; atomicOr(&a.ctrl->unsupported, 1u); }
    }
  } else {
    RawSrc src{&a, fd, ld, true};
    ok = conv_typed_exact<TS>(src, cd->type, v);
    if (!src.ok) { ok = 0; atomicOr(&a.ctrl->unsupported, 1u); }
  }
  if (ok != 1) { ok = 0; v = 0; }
  reinterpret_cast<long long *>(cd->val)[row] = v;
  cd->valid[row] = (uint8_t)ok;
}

// every thread of the grid (tid of nth): the queued fields, then (after an overflow) the marked rows
template <bool TS>
__device__ __forceinline__ void deferred_all(const KArgs &a, const DfaK &dfa, const ColsK &colsk, unsigned long long tid,
                             unsigned long long nth) {
  unsigned int n = min(a.ctrl->n_defer, a.dq_cap);
  for (unsigned long long i = tid; i < n; i += nth) {
    const DeferItem it = a.dq[i];
    // long numeric fields without inner control bytes: queued for the block / device tier (the emission
    // kernels only test the length; the routing lives here, out of their code)
    if (!it.ic && push_collab(a, colsk.c + it.col, it.fd, it.ld, it.row, it.col)) continue;
    convert_deferred<TS>(a, dfa, colsk.c + it.col, it.fd, it.ld, it.row, it.ic);
  }
  if (a.ctrl->defer_overflow) {                     // the queue was full: convert the marked rows
    const unsigned long long R = a.stats ? min((unsigned long long)a.stats->records, a.cap) : a.cap;
    for (uint32_t c = 0; c < a.C; c++) {
      const ColDesc *cd = colsk.c + c;
      if (cd->type == T_SPAN || cd->type == T_SKIP) continue;
      for (unsigned long long r = tid; r < R; r += nth) {
        const uint8_t m = cd->valid[r];
        if (m == VALID_REDO || m == VALID_REDO_IC) {
          const unsigned long long fd = cd->off[r], ld = fd + cd->len[r] - 1;
          if (m == VALID_REDO && push_collab(a, cd, fd, ld, r, c)) continue;
          convert_deferred<TS>(a, dfa, cd, fd, ld, r, m == VALID_REDO_IC ? 1u : 0u);
        }
      }
    }
  }
}
template <bool TS>
__global__ void k_deferred(const __grid_constant__ KArgs a, const __grid_constant__ DfaK dfa,
                           const __grid_constant__ ColsK colsk) {
  PdlTrigger pdl_trigger;
  pdl_wait();
  const unsigned long long nth = (unsigned long long)gridDim.x * blockDim.x;
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  deferred_all<TS>(a, dfa, colsk, tid, nth);
  __shared__ CollabSmem s_collab;                  // long numeric fields: block tier, then device tier
  collab_tiers<TS>(a, colsk, s_collab);            // (cooperative launch)
  // the last block to finish settles the status (every block's conversions are done by then)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    // (modulo the grid: a plan emitted more than once keeps counting)
    if ((atomicAdd(&a.ctrl->deferred_done, 1u) + 1u) % gridDim.x == 0u && a.stats) {
      collab_stats(a);
      if (*reinterpret_cast<volatile unsigned int *>(&a.ctrl->unsupported) && a.stats->status != ST_EFORMAT)
        a.stats->status = ST_EUNSUPPORTED;           // k_finalize's order: EFORMAT > EUNSUPPORTED > the rest
    }
  }
}

// ---- debug trace (tests): per-byte state-before and emission kind ---------------------------------
__global__ void k_debug_trace(const __grid_constant__ KArgs a, const __grid_constant__ DfaK dfa,
                              uint8_t *chunk_states_out, uint8_t *kinds, uint8_t *states) {
  // exact DFA states: the state before byte p is next_exact[class before byte p-1][group of byte p-1]
  // (the class before the first byte of a chunk comes from re-simulating the chunk before it)
  unsigned long long nchunks = (a.len + CHUNK - 1) / CHUNK;
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < nchunks;
       k += (unsigned long long)gridDim.x * blockDim.x) {
    uint32_t prev_cls = 0xFFu, prev_b = 0u;                  // class before / value of the byte before chunk k
    if (k > 0) {
      uint32_t y = 0x80u | a.chunk_state[k - 1];
      for (unsigned long long p = (k - 1) * CHUNK; p + 1 < k * CHUNK; p++) {
        const uint8_t b = a.in[p];
        y = prmt(dfa.lut[b][2], dfa.lut[b][3], y);
      }
      prev_cls = y & 0xFu;
      prev_b = a.in[k * CHUNK - 1];
    }
    auto exact = [&](uint32_t cls_before_prev, uint32_t bprev) -> uint32_t {
      return cls_before_prev == INV_DEV ? dfa.inv_state : dfa.next_exact[cls_before_prev][dfa.gob[bprev]];
    };
    const uint32_t st = a.chunk_state[k];
    const uint32_t e0 = k == 0 ? a.seed_exact : exact(prev_cls, prev_b);
    if (chunk_states_out) chunk_states_out[k] = (uint8_t)e0;
    if (!kinds && !states) continue;
    uint32_t x = 0x80u | st;
    unsigned long long end = min(a.len, (k + 1) * CHUNK);
    for (unsigned long long p = k * CHUNK; p < end; p++) {
      uint8_t b = a.in[p];
      if (states) states[p] = (uint8_t)(p == k * CHUNK ? e0 : exact(prev_cls, prev_b));
      prev_cls = x & 0xFu;
      prev_b = b;
      x = prmt(dfa.lut[b][2], dfa.lut[b][3], x);
      const uint32_t kc = step_kind_code(x);
      uint8_t kind = kc == KC_RECORD ? 3 : kc == KC_FIELD ? 2 : kc == KC_DATA ? 0 : 1;   // parpa_emit codes
      if (kinds) kinds[p] = kind;
    }
  }
}

}  // namespace parpa
#include "parpa_small.cuh"
