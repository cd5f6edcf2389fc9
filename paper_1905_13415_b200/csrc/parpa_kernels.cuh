// parpa_kernels.cuh — the hot-path kernels of libparpa (sm_100a).
//
//   k_scan<MODE>   persistent CTAs take 16 KB tiles in ticket order.  Per tile:
//                  S1+S2  each thread classifies its 64-byte chunk through the shared-memory LUT and
//                         builds its state-transition vector right-to-left with PRMT;
//                  S3     warp-shuffle scan of the vectors with ∘ + decoupled look-back
//                         over tile aggregates (single-pass scan after Merrill);
//                  S4     re-simulation from the now known entry state -> DATA / DELIM / RECORD
//                         masks (the paper's three bitmap indexes);
//                  S5     record counts by POPCNT and the abs/rel column offset plus the
//                         open-field carries, reduced (MODE_COUNT) or scanned (MODE_EMIT) over the
//                         CTA and chained across tiles by a second decoupled look-back;
//                  S6+S7  (MODE_EMIT) each thread walks its delimiters and writes every field's span
//                         column-major, converting int64 / float64 fields in place.
//   k_emit         S4-S7 for the two-phase path, from the per-chunk entry states and per-tile
//                  prefixes that k_scan<MODE_COUNT> stored (input read a second time).
//   k_finalize     end-of-input action, implicit last record, missing columns, status.
//   k_deferred     device-tier conversion of typed fields the thread tier deferred: fields with
//                  control bytes inside their span (re-simulated from the chunk entry state to
//                  drop them) and floats outside the exact fast path (exact decimal algorithm).
//   k_debug_trace  per-byte states / emission kinds from the per-chunk entry states (tests only).
#pragma once
#include "parpa_convert.cuh"
#include "parpa_device.cuh"

namespace parpa {

enum { MODE_TAU = 0, MODE_COUNT = 1, MODE_EMIT = 2 };
enum { T_SPAN = 0, T_INT64 = 1, T_FLOAT64 = 2 };
enum { EOI_NONE = 0, EOI_RECORD = 1, EOI_ERROR = 2 };
enum { ST_OK = 0, ST_EFORMAT = -4, ST_ECOLUMNS = -5, ST_EUNSUPPORTED = -6, ST_ENEEDMORE = -7 };

struct DfaK {                       // compiled DFA, passed by value (kernel parameter space)
  uint32_t lut[256][4];             // per byte: {sel_lo, sel_hi, step_lo, step_hi}
  uint8_t hmap[16];                 // device state -> DFA state (index 15 = INV)
  uint8_t eoi[16];                  // EOI action by device state
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
  unsigned int ticket;
  unsigned int n_defer;
  unsigned int defer_overflow;
  unsigned int unsupported;
  unsigned long long inv_neg;        // ~(first invalid byte position), 0 = none (atomicMax)
  unsigned long long n_missing;
  unsigned long long n_extra;
  unsigned long long pad[3];
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
};

struct KArgs {
  const uint8_t *in;
  unsigned long long len, base;      // bytes of this range, global offset of in[0]
  const uint8_t *left;               // bytes preceding the range (multi-GPU halo), may be null
  unsigned long long left_len;
  uint32_t ntiles, seed_dev, is_last, C;
  Seg seed;                          // composed prefix of everything before the range
  unsigned long long row_base;       // global record index of local row 0
  unsigned long long cap;            // rows per column
  unsigned long long *tau_desc;      // [ntiles] (flag << 32) | nibble τ
  uint32_t *seg_flag;                // [ntiles]
  Seg *seg_agg, *seg_incl;           // [ntiles]
  TileInfo *tinfo;                   // [ntiles]
  uint8_t *chunk_state;              // [ntiles * THREADS] device entry state of each chunk
  Ctrl *ctrl;
  DeferItem *dq;
  uint32_t dq_cap, strict;
  Stats *stats;
};

constexpr uint32_t FLAG_AGG = 1, FLAG_INCL = 2;

// ---- shared-memory LUT ------------------------------------------------------------------------
__device__ __forceinline__ void build_lut(uint8_t *lut, const DfaK &d) {
  for (int i = threadIdx.x; i < 256 * 32; i += THREADS) {
    int b = i >> 5, half = (i >> 4) & 1, slot = i & 15;
    uint2 v = half ? make_uint2(d.lut[b][2], d.lut[b][3]) : make_uint2(d.lut[b][0], d.lut[b][1]);
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
template <bool FULL>
__device__ __forceinline__ void chunk_tau(const uint8_t *lut, const uint32_t (&v)[16], int nvalid,
                                          uint32_t laneoff, uint32_t &t0, uint32_t &t1) {
  t0 = 0x83828180u;
  t1 = 0x87868584u;
#pragma unroll
  for (int i = CHUNK - 1; i >= 0; --i) {
    if (!FULL && i >= nvalid) continue;
    uint32_t addr = prmt(v[i >> 2], laneoff, 0x5504u | ((uint32_t)(i & 3) << 4));
    uint2 e = *reinterpret_cast<const uint2 *>(lut + addr);
    uint32_t n0 = prmt(t0, t1, e.x);
    uint32_t n1 = prmt(t0, t1, e.y);
    t0 = n0;
    t1 = n1;
  }
}

// ---- S4: re-simulation from the entry state -> DATA / DELIM / RECORD masks --------------------
// multipliers that gather bit (4+k) of each byte into bits 32..35 of the 64-bit product
__device__ __forceinline__ uint32_t gather4(uint32_t x, uint32_t bitmask, uint32_t mul) {
  return __umulhi(x & bitmask, mul) & 0xFu;
}

template <bool FULL>
__device__ __forceinline__ uint32_t chunk_masks(const uint8_t *lut, const uint32_t (&v)[16], int nvalid,
                                                uint32_t laneoff, uint32_t entry,
                                                unsigned long long &Dm, unsigned long long &Fm,
                                                unsigned long long &Rm) {
  uint32_t x = 0x80u | entry;
  uint32_t d[2] = {0, 0}, f[2] = {0, 0}, r[2] = {0, 0};
#pragma unroll
  for (int w = 0; w < 16; w++) {
    uint32_t xs[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      int i = 4 * w + k;
      if (FULL || i < nvalid) {
        uint32_t addr = prmt(v[w], laneoff, 0x5504u | ((uint32_t)k << 4));
        uint2 st = *reinterpret_cast<const uint2 *>(lut + addr + 128);
        x = prmt(st.x, st.y, x);
        xs[k] = x;
      } else {
        xs[k] = 0xFFu;                                    // outside the chunk: not data / delimiter
      }
    }
    uint32_t pk = prmt(prmt(xs[0], xs[1], 0x0040u), prmt(xs[2], xs[3], 0x0040u), 0x5410u);
    uint32_t npk = ~pk;
    int h = w >> 3, sh = 4 * (w & 7);
    d[h] |= gather4(npk, 0x10101010u, 0x10204080u) << sh;
    f[h] |= gather4(npk, 0x20202020u, 0x08102040u) << sh;
    r[h] |= gather4(npk, 0x40404040u, 0x04081020u) << sh;
  }
  Dm = (unsigned long long)d[0] | ((unsigned long long)d[1] << 32);
  Fm = (unsigned long long)f[0] | ((unsigned long long)f[1] << 32);
  Rm = (unsigned long long)r[0] | ((unsigned long long)r[1] << 32);
  return x & 0xFu;
}

// scalar re-walk (rare): position of the first byte whose transition enters INV
__device__ int first_inv_in_chunk(const uint8_t *lut, const uint8_t *p, int nvalid, uint32_t laneoff,
                                  uint32_t entry) {
  uint32_t x = 0x80u | entry;
  for (int i = 0; i < nvalid; i++) {
    uint32_t b = p[i];
    uint2 st = *reinterpret_cast<const uint2 *>(lut + (b << 8) + laneoff + 128);
    x = prmt(st.x, st.y, x);
    if ((x & 0xFu) == INV_DEV) return i;
  }
  return -1;
}

// ---- CTA-level τ scan (exclusive per thread, aggregate per tile) ---------------------------------
struct TauScanSmem {
  uint32_t wtot[WARPS];
  uint32_t wpre[WARPS];
  uint32_t agg;
  uint32_t prefix;
  uint32_t tile;
};

__device__ __forceinline__ uint32_t cta_scan_tau(uint32_t t0, uint32_t t1, TauScanSmem &sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
  uint32_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) ex = NIB_IDENT;
  if (lane == 31) sm.wtot[warp] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t p = NIB_IDENT;
    for (int w = 0; w < WARPS; w++) {
      sm.wpre[w] = p;
      p = compose_nib(p, sm.wtot[w]);
    }
    sm.agg = p;
  }
  __syncthreads();
  return compose_nib(sm.wpre[warp], ex);
}

// ---- decoupled look-back over τ (warp 0) ---------------------------------------------------------
// returns the exclusive prefix τ_0 ∘ ... ∘ τ_{t-1} of tile t (identity for t == 0)
__device__ uint32_t lookback_tau(const KArgs &a, uint32_t t) {
  const int lane = threadIdx.x & 31;
  uint32_t acc = NIB_IDENT;
  long long base = (long long)t - 1;
  while (true) {
    long long j = base - lane;
    uint32_t val = NIB_IDENT, flag = FLAG_INCL;
    if (j >= 0) {
      unsigned long long dsc;
      do {
        dsc = ld_relaxed_u64(a.tau_desc + j);
      } while ((dsc >> 32) == 0u);
      flag = (uint32_t)(dsc >> 32);
      val = (uint32_t)dsc;
    }
    unsigned m = __ballot_sync(0xffffffffu, flag == FLAG_INCL);
    int k = m ? __ffs(m) - 1 : 31;
    uint32_t w = lane <= k ? val : NIB_IDENT;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {       // w <- w_{lane+d..} ∘ w   (farther tiles first)
      uint32_t o = __shfl_down_sync(0xffffffffu, w, d);
      if (lane + d < 32) w = compose_nib(o, w);
    }
    w = __shfl_sync(0xffffffffu, w, 0);
    acc = compose_nib(w, acc);
    if (m) break;
    base -= 32;
  }
  return acc;
}

// ---- CTA-level SegT reduce / scan --------------------------------------------------------------
struct SegScanSmem {
  SegT wtot[WARPS];
  SegT wpre[WARPS];
  SegT agg;
};

__device__ __forceinline__ SegT cta_reduce_segt(SegT s, SegScanSmem &sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    SegT o = shfl_down_segt(s, d);
    if (lane + d < 32) s = segt_op(s, o);
  }
  if (lane == 0) sm.wtot[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    SegT p = segt_ident();
    for (int w = 0; w < WARPS; w++) p = segt_op(p, sm.wtot[w]);
    sm.agg = p;
  }
  __syncthreads();
  return sm.agg;
}

__device__ __forceinline__ SegT cta_scan_segt(SegT s, SegScanSmem &sm) {     // exclusive
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  SegT inc = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    SegT o = shfl_up_segt(inc, d);
    if (lane >= d) inc = segt_op(o, inc);
  }
  SegT ex = shfl_up_segt(inc, 1);
  if (lane == 0) ex = segt_ident();
  if (lane == 31) sm.wtot[warp] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    SegT p = segt_ident();
    for (int w = 0; w < WARPS; w++) {
      sm.wpre[w] = p;
      p = segt_op(p, sm.wtot[w]);
    }
    sm.agg = p;
  }
  __syncthreads();
  return segt_op(sm.wpre[warp], ex);
}

// ---- decoupled look-back over Seg (warp 0) ---------------------------------------------------------
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

// returns seed ∘ Seg_0 ∘ ... ∘ Seg_{t-1}
__device__ Seg lookback_seg(const KArgs &a, uint32_t t) {
  const int lane = threadIdx.x & 31;
  Seg acc = seg_ident();
  long long base = (long long)t - 1;
  while (true) {
    long long j = base - lane;
    Seg val = seg_ident();
    uint32_t flag = FLAG_INCL;
    if (j >= 0) {
      do {
        flag = ld_acquire_u32(a.seg_flag + j);
      } while (flag == 0u);
      val = ldcg_seg(flag == FLAG_INCL ? a.seg_incl + j : a.seg_agg + j);
    } else if (j == -1) {
      val = a.seed;
    }
    unsigned m = __ballot_sync(0xffffffffu, flag == FLAG_INCL);
    int k = m ? __ffs(m) - 1 : 31;
    Seg w = lane <= k ? val : seg_ident();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      Seg o = shfl_down_seg(w, d);
      if (lane + d < 32) w = seg_op(o, w);
    }
    w = shfl_seg(w, 0);
    acc = seg_op(w, acc);
    if (m) break;
    base -= 32;
  }
  return acc;
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

__device__ __forceinline__ void push_defer(const KArgs &a, unsigned long long fd, unsigned long long ld,
                                           unsigned long long row, uint32_t c, uint32_t ic) {
  uint32_t idx = atomicAdd(&a.ctrl->n_defer, 1u);
  if (idx < a.dq_cap) a.dq[idx] = DeferItem{fd, ld, row, c, ic};
  else atomicOr(&a.ctrl->defer_overflow, 1u);
}

__device__ void emit_field(const KArgs &a, const ColDesc *cols, unsigned long long r, uint32_t c, unsigned long long fd,
                           unsigned long long ld, uint32_t fl, unsigned long long dpos, EmitCounters &cnt) {
  if (c >= a.C) { cnt.extra++; return; }
  unsigned long long row = r - a.row_base;
  if (row >= a.cap) return;                         // capacity exceeded: reported by k_finalize
  const ColDesc *cd = cols + c;
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
  __stcs(cd->off + row, off);
  __stcs(cd->len + row, len);
  uint32_t type = cd->type;
  if (type == T_SPAN) return;
  long long v = 0;
  int ok = 0;
  if (fd == NONE) {
    if (cd->has_def) { v = cd->def_bits; ok = 1; }
  } else if (fl & F_IC) {
    push_defer(a, fd, ld, row, c, 1u);
    return;
  } else {
    RawSrc src{&a, fd, ld, true};
    int res = type == T_INT64 ? conv_int64(src, v) : conv_float64_fast(src, v);
    if (!src.ok) res = 2;                           // bytes outside this range: device tier
    if (res == 2) { push_defer(a, fd, ld, row, c, 0u); return; }
    ok = res;
    if (!ok) v = 0;
  }
  reinterpret_cast<long long *>(cd->val)[row] = v;
  cd->valid[row] = (uint8_t)ok;
}

__device__ void fill_missing(const KArgs &a, const ColDesc *cols, unsigned long long r, uint32_t from, unsigned long long dpos,
                             EmitCounters &cnt) {
  if (from >= a.C) return;
  cnt.missing++;
  unsigned long long row = r - a.row_base;
  if (row >= a.cap) return;
  for (uint32_t k = from; k < a.C; k++) {
    const ColDesc *cd = cols + k;
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
    emit_field(a, cols, r, c, cfd, cld, cfl, cbase + (unsigned)p, cnt);
    if ((Rm >> p) & 1ull) {
      fill_missing(a, cols, r, c + 1, cbase + (unsigned)p, cnt);
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

// ---- the fused scan kernel -------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(THREADS) k_scan(const KArgs a, const DfaK dfa, const ColsK colsk) {
  extern __shared__ __align__(16) uint8_t lut[];
  __shared__ TauScanSmem tsm;
  __shared__ SegScanSmem ssm;
  __shared__ Seg s_prefix;
  __shared__ ColDesc s_cols[MODE == MODE_EMIT ? MAX_COLS : 1];
  build_lut(lut, dfa);
  if (MODE == MODE_EMIT)
    for (int c = threadIdx.x; c < (int)a.C; c += THREADS) s_cols[c] = colsk.c[c];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t laneoff = (uint32_t)(lane & 15) * 8u;
  EmitCounters cnt{0ull, 0ull, 0u};
  __syncthreads();
  while (true) {
    if (tid == 0) tsm.tile = atomicAdd(&a.ctrl->ticket, 1u);
    __syncthreads();
    const uint32_t t = tsm.tile;
    if (t >= a.ntiles) break;
    const unsigned long long tstart = (unsigned long long)t * TILE;
    const unsigned long long cstart = tstart + (unsigned long long)tid * CHUNK;
    int nvalid = cstart >= a.len ? 0 : (int)min((unsigned long long)CHUNK, a.len - cstart);
    uint32_t v[16];
    load_chunk(a.in + cstart, nvalid, v);
    uint32_t t0, t1;
    if (nvalid == CHUNK) chunk_tau<true>(lut, v, nvalid, laneoff, t0, t1);
    else chunk_tau<false>(lut, v, nvalid, laneoff, t0, t1);
    uint32_t ex = cta_scan_tau(t0, t1, tsm);
    // publish the tile aggregate, look back, publish the inclusive prefix
    if (tid < 32) {
      uint32_t prefix = NIB_IDENT;
      if (t == 0) {
        if (tid == 0) st_relaxed_u64(a.tau_desc, ((unsigned long long)FLAG_INCL << 32) | tsm.agg);
      } else {
        if (tid == 0) st_relaxed_u64(a.tau_desc + t, ((unsigned long long)FLAG_AGG << 32) | tsm.agg);
        prefix = lookback_tau(a, t);
        if (tid == 0)
          st_relaxed_u64(a.tau_desc + t, ((unsigned long long)FLAG_INCL << 32) | compose_nib(prefix, tsm.agg));
      }
      if (tid == 0) tsm.prefix = prefix;
    }
    __syncthreads();
    if (MODE == MODE_TAU) continue;
    const uint32_t tile_entry = nib_at(tsm.prefix, a.seed_dev);
    const uint32_t entry = nib_at(ex, tile_entry);
    a.chunk_state[(unsigned long long)t * THREADS + tid] = (uint8_t)entry;
    unsigned long long Dm, Fm, Rm;
    uint32_t fin;
    if (nvalid == CHUNK) fin = chunk_masks<true>(lut, v, nvalid, laneoff, entry, Dm, Fm, Rm);
    else fin = chunk_masks<false>(lut, v, nvalid, laneoff, entry, Dm, Fm, Rm);
    if (fin == INV_DEV && entry != INV_DEV && nvalid > 0) {
      int p = first_inv_in_chunk(lut, a.in + cstart, nvalid, laneoff, entry);
      if (p >= 0) atomicMax(&a.ctrl->inv_neg, ~(a.base + cstart + (unsigned)p));
    }
    const unsigned long long Vm = nvalid >= 64 ? ~0ull : ((1ull << nvalid) - 1ull);
    SegT s = chunk_segt(Dm, Fm, Rm, Vm, (uint32_t)tid * CHUNK);
    SegT sex;
    if (MODE == MODE_EMIT) sex = cta_scan_segt(s, ssm);
    else cta_reduce_segt(s, ssm);
    if (tid < 32) {
      Seg agg = segt_to_seg(ssm.agg, a.base + tstart);
      Seg prefix;
      if (t == 0) {
        prefix = a.seed;
        if (tid == 0) {
          stcg_seg(a.seg_incl, seg_op(prefix, agg));
          st_release_u32(a.seg_flag, FLAG_INCL);
        }
      } else {
        if (tid == 0) {
          stcg_seg(a.seg_agg + t, agg);
          st_release_u32(a.seg_flag + t, FLAG_AGG);
        }
        prefix = lookback_seg(a, t);
        if (tid == 0) {
          stcg_seg(a.seg_incl + t, seg_op(prefix, agg));
          st_release_u32(a.seg_flag + t, FLAG_INCL);
        }
      }
      if (tid == 0) {
        s_prefix = prefix;
        a.tinfo[t].excl = prefix;
        a.tinfo[t].entry = tile_entry;
      }
    }
    __syncthreads();
    if (MODE == MODE_EMIT) {
      Seg st = seg_op(s_prefix, segt_to_seg(sex, a.base + tstart));
      emit_chunk(a, s_cols, st, Dm, Fm, Rm, Vm, a.base + cstart, cnt);
    }
  }
  flush_counters(a, cnt);
}

// ---- two-phase emit kernel -------------------------------------------------------------------------
__global__ void __launch_bounds__(THREADS) k_emit(const KArgs a, const DfaK dfa, const ColsK colsk) {
  extern __shared__ __align__(16) uint8_t lut[];
  __shared__ SegScanSmem ssm;
  __shared__ ColDesc s_cols[MAX_COLS];
  build_lut(lut, dfa);
  for (int c = threadIdx.x; c < (int)a.C; c += THREADS) s_cols[c] = colsk.c[c];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t laneoff = (uint32_t)(lane & 15) * 8u;
  EmitCounters cnt{0ull, 0ull, 0u};
  __syncthreads();
  for (uint32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    const unsigned long long tstart = (unsigned long long)t * TILE;
    const unsigned long long cstart = tstart + (unsigned long long)tid * CHUNK;
    int nvalid = cstart >= a.len ? 0 : (int)min((unsigned long long)CHUNK, a.len - cstart);
    uint32_t v[16];
    load_chunk(a.in + cstart, nvalid, v);
    const uint32_t entry = a.chunk_state[(unsigned long long)t * THREADS + tid];
    unsigned long long Dm, Fm, Rm;
    if (nvalid == CHUNK) chunk_masks<true>(lut, v, nvalid, laneoff, entry, Dm, Fm, Rm);
    else chunk_masks<false>(lut, v, nvalid, laneoff, entry, Dm, Fm, Rm);
    const unsigned long long Vm = nvalid >= 64 ? ~0ull : ((1ull << nvalid) - 1ull);
    SegT s = chunk_segt(Dm, Fm, Rm, Vm, (uint32_t)tid * CHUNK);
    SegT sex = cta_scan_segt(s, ssm);
    Seg st = seg_op(a.tinfo[t].excl, segt_to_seg(sex, a.base + tstart));
    emit_chunk(a, s_cols, st, Dm, Fm, Rm, Vm, a.base + cstart, cnt);
    __syncthreads();
  }
  flush_counters(a, cnt);
}

// ---- finalize ---------------------------------------------------------------------------------------
__global__ void k_finalize(const KArgs a, const DfaK dfa, const ColsK colsk) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Seg tot = a.ntiles ? a.seg_incl[a.ntiles - 1] : a.seed;
  uint32_t tau = a.ntiles ? (uint32_t)a.tau_desc[a.ntiles - 1] : NIB_IDENT;
  uint32_t fin = nib_at(tau, a.seed_dev);
  EmitCounters cnt{0ull, 0ull, 0u};
  unsigned long long R = tot.recs, nf = tot.nflds;
  unsigned long long first_inv = a.ctrl->inv_neg ? ~a.ctrl->inv_neg : NONE;
  if (a.is_last) {
    uint32_t act = dfa.eoi[fin];
    unsigned long long end = a.base + a.len;
    if (act == EOI_RECORD) {                               // implicit record delimiter at EOI
      emit_field(a, colsk.c, R, tot.col, tot.fd, tot.ld, tot.flags & (F_IC | F_PC | F_PRE), end, cnt);
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
  int status = ST_OK;
  if (first_inv != NONE) status = ST_EFORMAT;
  else if (a.ctrl->unsupported || cnt.unsupported || a.ctrl->defer_overflow) status = ST_EUNSUPPORTED;
  else if (R - a.row_base > a.cap) status = ST_ENEEDMORE;
  else if ((missing || extra) && a.strict) status = ST_ECOLUMNS;
  if (a.stats) {
    a.stats->records = R - a.row_base;
    a.stats->fields = nf - a.seed.nflds;
    a.stats->first_invalid = first_inv;
    a.stats->missing_records = missing;
    a.stats->extra_fields = extra;
    a.stats->deferred_fields = n_defer;
    a.stats->status = status;
    a.stats->final_state = dfa.hmap[fin];
  }
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
      uint8_t b = a->in[pos - a->base];
      pos++;
      uint32_t step_lo = d->lut[b][2], step_hi = d->lut[b][3];
      uint32_t prev = x;
      x = prmt(step_lo, step_hi, prev);
      if ((x & NOT_DATA) == 0) { c = b; return true; }
    }
    return false;
  }
};

__global__ void k_deferred(const KArgs a, const DfaK dfa, const ColsK colsk) {
  unsigned int n = min(a.ctrl->n_defer, a.dq_cap);
  for (unsigned int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    DeferItem it = a.dq[i];
    const ColDesc *cd = colsk.c + it.col;
    long long v = 0;
    int ok = 0;
    if (it.ic) {
      if (it.fd < a.base) {
        atomicOr(&a.ctrl->unsupported, 1u);          // a span crossing into a previous range with inner
      } else {                                        // control bytes (multi-GPU) is not handled
        unsigned long long local = it.fd - a.base;
        unsigned long long k = local / CHUNK;
        uint32_t x = 0x80u | a.chunk_state[k];
        for (unsigned long long p = k * CHUNK; p < local; p++) {
          uint8_t b = a.in[p];
          x = prmt(dfa.lut[b][2], dfa.lut[b][3], x);
        }
        DfaDataSrc src{&a, &dfa, it.fd, it.ld, x, true};
        ok = cd->type == T_INT64 ? conv_int64(src, v) : conv_float64_exact(src, v);
      }
    } else {
      RawSrc src{&a, it.fd, it.ld, true};
      ok = cd->type == T_INT64 ? conv_int64(src, v) : conv_float64_exact(src, v);
      if (!src.ok) { ok = 0; atomicOr(&a.ctrl->unsupported, 1u); }
    }
    if (ok != 1) { ok = 0; v = 0; }
    reinterpret_cast<long long *>(cd->val)[it.row] = v;
    cd->valid[it.row] = (uint8_t)ok;
  }
  if (a.stats && blockIdx.x == 0 && threadIdx.x == 0 && (a.ctrl->unsupported || a.ctrl->defer_overflow) &&
      a.stats->status == ST_OK)
    a.stats->status = ST_EUNSUPPORTED;
}

// ---- debug trace (tests): per-byte state-before and emission kind ---------------------------------
__global__ void k_debug_trace(const KArgs a, const DfaK dfa, uint8_t *chunk_states_out, uint8_t *kinds,
                              uint8_t *states) {
  unsigned long long nchunks = (a.len + CHUNK - 1) / CHUNK;
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < nchunks;
       k += (unsigned long long)gridDim.x * blockDim.x) {
    uint32_t st = a.chunk_state[k];
    if (chunk_states_out) chunk_states_out[k] = dfa.hmap[st];
    if (!kinds && !states) continue;
    uint32_t x = 0x80u | st;
    unsigned long long end = min(a.len, (k + 1) * CHUNK);
    for (unsigned long long p = k * CHUNK; p < end; p++) {
      uint8_t b = a.in[p];
      if (states) states[p] = dfa.hmap[x & 0xFu];
      x = prmt(dfa.lut[b][2], dfa.lut[b][3], x);
      uint32_t f = x & 0x70u;
      uint8_t kind = !(f & NOT_REC) ? 3 : !(f & NOT_DELIM) ? 2 : !(f & NOT_DATA) ? 0 : 1;
      if (kinds) kinds[p] = kind;
    }
  }
}

}  // namespace parpa
