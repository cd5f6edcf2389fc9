// parpa_fused.cuh — S4+S5+S6+S7 in one persistent kernel: the delimiter-emitting re-simulation, the
// record / field / column prefix scan and the column partition with conversion, per tile, without the
// chunk masks or the tile bytes ever leaving shared memory / registers.
//
//   k_fused     one CTA per SM = FG_GROUPS independent warp groups sharing the 64 KB LUT.  A group
//               (FG_CW compute warps + 1 scan warp) takes a GROUP TILE (FG_CW warp tiles = 14 KB) in
//               ticket order, and
//                 1. each compute warp loads its 2 KB warp tile into its shared-memory scratch (the copy
//                    E2 reads digits from) and re-simulates it from its entry state (lex ∘ wpre, from
//                    k_pass1 / k_tau_scan) -> DATA / DELIM / RECORD masks in registers and
//                    the warp tile's SegT (POPCNT record count, ⊕ column offset, open-field carries,
//                    P:391-414);
//                 2. the scan warp ⊕-scans the group's SegTs, publishes the group aggregate and runs a
//                    decoupled look-back over the earlier group tiles (Merrill & Garland) -> the
//                    prefix of everything before every warp tile, while the compute warps build their
//                    tile-local field lists (E1, no prefix needed);
//                 3. every compute warp partitions its fields by column and converts them (E2,
//                    P:439-469).
// Replaces k_pass2 + k_seg_scan + k_emit of the staged path for parse_into / parse_range: the input is
// read once more after pass 1 (instead of twice), the 24 B of masks per 64-byte chunk are neither
// written nor read back, and the per-warp-tile prefixes never touch memory.
#pragma once

namespace parpa {

constexpr int FG_CW = 7;                        // compute warps per group (a group tile = 7 warp tiles)
constexpr int FG_WARPS = FG_CW + 1;             // + the group's scan warp
constexpr int FG_GROUPS = 2;                    // groups per CTA
constexpr int F_WARPS = FG_WARPS * FG_GROUPS;   // 16 warps, one CTA per SM
constexpr uint32_t F_PREFETCH = 640;            // L2 prefetch distance in group tiles (≈ 2 × in flight)
constexpr int F_CWARPS = FG_CW * FG_GROUPS;     // warps with a scratch slot
constexpr size_t F_SMEM = LUT_BYTES + (F_CWARPS + 1) * sizeof(WarpScratch) + 256;

struct FusedSmem {
  WarpScratch *ws;
  uint32_t laneaddr, laneoff;
  uint8_t *lut;
};
// LUT at the first 64 KB-aligned shared address of the dynamic region (one PRMT forms LDS addresses,
// see lds_u2), the per-warp scratch slots packed before and after it.
__device__ __forceinline__ FusedSmem fused_smem(uint8_t *smem, int warp, int lane) {
  const uint32_t sb0 = smem_u32(smem);
  const uint32_t sb = (sb0 + 15u) & ~15u;
  uint8_t *base = smem + (sb - sb0);
  const uint32_t lut_off = ((sb + 0xFFFFu) & ~0xFFFFu) - sb;
  const uint32_t nfirst = lut_off / (uint32_t)sizeof(WarpScratch);
  const uint32_t off = (uint32_t)warp < nfirst
                           ? (uint32_t)warp * (uint32_t)sizeof(WarpScratch)
                           : lut_off + LUT_BYTES + ((uint32_t)warp - nfirst) * (uint32_t)sizeof(WarpScratch);
  FusedSmem f;
  f.lut = base + lut_off;
  f.ws = reinterpret_cast<WarpScratch *>(base + off);
  f.laneoff = (uint32_t)(lane & 15) * 8u;
  f.laneaddr = f.laneoff | (((sb + lut_off) >> 16) << 16);
  return f;
}

// named barriers of a group (all FG_WARPS warps take part; the producer side arrives, the consumer side
// waits): 1+4g previous tile done (compute -> scan), 2+4g ticket posted (scan -> compute), 3+4g SegTs
// posted (compute -> scan), 4+4g prefixes posted (scan -> compute)
__device__ __forceinline__ void nbar_sync(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(FG_WARPS * 32) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "n"(FG_WARPS * 32) : "memory");
}

// Group-tile descriptors, structure of arrays in a.gdesc ([7][a.gstride] 64-bit words, zeroed per call):
// words 0-1 the AGGREGATE of group tile j in compact tile-relative form, words 2-6 its INCLUSIVE prefix.
// Every word carries a tag in bit 63 and is written with a relaxed store; a reader accepts a descriptor
// once all its words carry the tag, so no release / acquire pair (MEMBAR + L1 invalidation per load on
// sm_100a) is on the look-back path.  Lane l of a look-back round reads descriptor base - l (then
// base - 32 - l, ...), so each load instruction covers 32 consecutive words.
constexpr unsigned long long GD_TAG = 1ull << 63, GD_VAL = GD_TAG - 1ull;
constexpr uint32_t GD_NONE16 = 0xFFFFu;
__device__ __forceinline__ unsigned long long *gword(const KArgs &a, int w, unsigned long long j) {
  return a.gdesc + (unsigned long long)w * a.gstride + j;
}
// aggregate of a group tile (counts < 2^14, positions relative to the tile start)
__device__ __forceinline__ void gagg_store(const KArgs &a, unsigned long long j, const Seg &s, unsigned long long tb) {
  const unsigned long long w0 = GD_TAG | s.recs | (s.nflds << 14) | ((unsigned long long)s.col << 28) |
                                ((unsigned long long)(s.flags & 0x1Fu) << 42);
  const uint32_t fr = s.fd == NONE ? GD_NONE16 : (uint32_t)(s.fd - tb), lr = s.ld == NONE ? GD_NONE16 : (uint32_t)(s.ld - tb);
  st_relaxed_u64(gword(a, 0, j), w0);
  st_relaxed_u64(gword(a, 1, j), GD_TAG | fr | ((unsigned long long)lr << 16));
}
__device__ __forceinline__ Seg gagg_seg(unsigned long long w0, unsigned long long w1, unsigned long long tb) {
  Seg s;
  s.recs = w0 & 0x3FFFull;
  s.nflds = (w0 >> 14) & 0x3FFFull;
  s.col = (uint32_t)(w0 >> 28) & 0x3FFFu;
  s.flags = (uint32_t)(w0 >> 42) & 0x1Fu;
  const uint32_t fr = (uint32_t)w1 & 0xFFFFu, lr = (uint32_t)(w1 >> 16) & 0xFFFFu;
  s.fd = fr == GD_NONE16 ? NONE : tb + fr;
  s.ld = lr == GD_NONE16 ? NONE : tb + lr;
  return s;
}
__device__ __forceinline__ void gincl_store(const KArgs &a, unsigned long long j, const Seg &s) {
  st_relaxed_u64(gword(a, 2, j), GD_TAG | s.recs);
  st_relaxed_u64(gword(a, 3, j), GD_TAG | s.nflds);
  st_relaxed_u64(gword(a, 4, j), GD_TAG | ((s.fd + 1ull) & GD_VAL));        // NONE -> 0
  st_relaxed_u64(gword(a, 5, j), GD_TAG | ((s.ld + 1ull) & GD_VAL));
  st_relaxed_u64(gword(a, 6, j), GD_TAG | ((unsigned long long)s.flags << 32) | s.col);
}
__device__ __forceinline__ Seg gincl_seg(const unsigned long long (&w)[7]) {
  Seg s;
  s.recs = w[2] & GD_VAL;
  s.nflds = w[3] & GD_VAL;
  s.fd = (w[4] & GD_VAL) - 1ull;
  s.ld = (w[5] & GD_VAL) - 1ull;
  s.col = (uint32_t)w[6];
  s.flags = (uint32_t)(w[6] >> 32) & 0xFFu;
  return s;
}
__device__ __forceinline__ unsigned long long gtile_base(const KArgs &a, unsigned long long j) {
  return a.base + j * (unsigned long long)(FG_CW * WT);
}
// descriptor state: 2 inclusive, 1 aggregate, 0 not published
__device__ __forceinline__ uint32_t gdesc_read(const KArgs &a, long long j, Seg &d) {
  if (j < 0) { d = seg_ident(); return FLAG_INCL; }
  unsigned long long w[7];
#pragma unroll
  for (int k = 0; k < 7; k++) w[k] = ld_relaxed_u64(gword(a, k, (unsigned long long)j));
  if ((w[2] & w[3] & w[4] & w[5] & w[6]) >> 63) { d = gincl_seg(w); return FLAG_INCL; }
  if ((w[0] & w[1]) >> 63) { d = gagg_seg(w[0], w[1], gtile_base(a, (unsigned long long)j)); return FLAG_AGG; }
  d = seg_ident();
  return 0u;
}

// decoupled look-back over the group-tile descriptors (one warp): returns G_0 ⊕ ... ⊕ G_{T-1}.
// 32 descriptors per round trip, lane l = tile base - l (lower lane = later tile).
__device__ Seg lookback_gseg(const KArgs &a, uint32_t T) {
  const int lane = threadIdx.x & 31;
  Seg acc = seg_ident();
  long long base = (long long)T - 1;
  while (true) {
    const long long j = base - lane;
    Seg d;
    uint32_t st = gdesc_read(a, j, d);
    int L;
    unsigned im;
    while (true) {
      im = __ballot_sync(0xffffffffu, st == FLAG_INCL);
      L = im ? __ffs(im) - 1 : 31;                           // the latest tile with an inclusive prefix
      const bool missing = lane <= L && st == 0u;
      if (!__any_sync(0xffffffffu, missing)) break;
      if (a.prof && lane == 0) atomicAdd(a.prof + blockIdx.x * 16 + 8, 1ull);
      __nanosleep(32);
      if (st != FLAG_INCL) st = gdesc_read(a, j, d);
    }
    Seg v = lane <= L ? d : seg_ident();
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {                    // higher lane = earlier tiles
      Seg o = shfl_down_seg(v, dd);
      if (lane + dd < 32) v = seg_op(o, v);
    }
    acc = seg_op(shfl_seg(v, 0), acc);
    if (a.prof && lane == 0) atomicAdd(a.prof + blockIdx.x * 16 + 7, 1ull);
    if (im) break;
    base -= 32;
  }
  return acc;
}

// PARPA_FPROF=1 (debug): per-CTA cycle counters of the phases (a.prof[blockIdx][0..15])
#define FP_MARK(var) const long long var = a.prof ? clock64() : 0
#define FP_ADD(idx, v) do { if (a.prof && lane == 0) atomicAdd(a.prof + blockIdx.x * 16 + (idx), (unsigned long long)(v)); } while (0)

template <bool TS>
__global__ void __launch_bounds__(F_WARPS * 32, 1) k_fused(const KArgs a, const DfaK dfa, const ColsK colsk) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ ColDesc s_cols[MAX_COLS];
  __shared__ uint4 s_wseg[FG_GROUPS][FG_CW];
  __shared__ Seg s_wpre[FG_GROUPS][FG_CW];
  __shared__ uint32_t s_tile[FG_GROUPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = warp / FG_WARPS, gw = warp % FG_WARPS;
  const bool scan_warp = gw == FG_CW;
  const int bar_done = 1 + 4 * grp, bar_tile = 2 + 4 * grp, bar_seg = 3 + 4 * grp, bar_pre = 4 + 4 * grp;
  const FusedSmem fs = fused_smem(smem, scan_warp ? 0 : grp * FG_CW + gw, lane);
  WarpScratch *ws = fs.ws;
  PdlTrigger pdl_trigger;
  build_lut(fs.lut, dfa);
  for (int c = threadIdx.x; c < (int)a.C; c += blockDim.x) s_cols[c] = colsk.c[c];
  __syncthreads();
  pdl_wait();
  EmitCounters cnt{0ull, 0ull, 0u};
  const uint32_t ngt = (a.ntiles + FG_CW - 1) / FG_CW;
  while (true) {
    // the ticket is taken only when the group's previous tile is finished (no tile waits behind another)
    if (scan_warp) {
      nbar_sync(bar_done);
      if (lane == 0) s_tile[grp] = atomicAdd(&a.ctrl->gticket, 1u);
      nbar_arrive(bar_tile);
    } else {
      nbar_arrive(bar_done);
      nbar_sync(bar_tile);
    }
    const uint32_t T = s_tile[grp];
    if (T >= ngt) break;
    if (scan_warp) {
      // ---- the group's scan: ⊕ over its warp tiles, aggregate first, then the look-back ----
      FP_MARK(s0);
      nbar_sync(bar_seg);                                      // the compute warps' SegTs are posted
      FP_MARK(s1);
      Seg e = seg_ident();
      const uint32_t tl = T * FG_CW + (uint32_t)lane;
      if (lane < FG_CW && tl < a.ntiles) {
        const uint4 w = s_wseg[grp][lane];
        e = segt_to_seg(SegT{w.x, w.y, w.z}, a.base + (unsigned long long)tl * WT);
      }
      Seg inc = e;
#pragma unroll
      for (int d = 1; d < 8; d <<= 1) {
        const Seg o = shfl_up_seg(inc, d);
        if (lane >= d) inc = seg_op(o, inc);
      }
      const Seg agg = shfl_seg(inc, FG_CW - 1);
      Seg ex = shfl_up_seg(inc, 1);
      if (lane == 0) ex = seg_ident();
      Seg prefix = seg_ident();
      if (T == 0) {
        if (lane == 0) gincl_store(a, 0, agg);
      } else {
        if (lane == 0) gagg_store(a, T, agg, gtile_base(a, T));
        prefix = lookback_gseg(a, T);
        if (lane == 0) gincl_store(a, T, seg_op(prefix, agg));
      }
      if (lane == 0 && T == ngt - 1) *a.tot_seg = seg_op(prefix, agg);
      if (lane < FG_CW) s_wpre[grp][lane] = seg_op(a.seed, seg_op(prefix, ex));
      FP_MARK(s2);
      nbar_arrive(bar_pre);
      if (gw == FG_CW) { FP_ADD(4, s2 - s1); FP_ADD(9, s1 - s0); }
      continue;
    }
    FP_MARK(t0);
    const uint32_t t = T * FG_CW + (uint32_t)gw;               // this warp's warp tile
    {                                                          // L2 prefetch of a tile a later group takes
      const unsigned long long tp = (unsigned long long)(T + F_PREFETCH) * FG_CW + gw;
      if (tp < a.ntiles && (lane & 1) == 0)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.in + tp * WT + (unsigned long long)lane * CHUNK));
    }
    const bool live = t < a.ntiles;
    const unsigned long long tstart = (unsigned long long)t * WT;
    const unsigned long long cstart = tstart + (unsigned long long)lane * CHUNK;
    const int nv = (!live || cstart >= a.len) ? 0 : (int)min((unsigned long long)CHUNK, a.len - cstart);
    unsigned long long Dm = 0ull, Fm = 0ull, Rm = 0ull;
    const unsigned long long Vm = nv >= 64 ? ~0ull : ((1ull << nv) - 1ull);
    SegT sg = segt_ident();
    if (live) {
      uint32_t v[16];
      load_chunk(a.in + cstart, nv, v);
      stash_chunk(ws->bytes, lane, v);
      const uint32_t entry = nib_at(a.lex[(unsigned long long)t * 32 + lane], nib_at(a.wpre[t], a.seed_dev));
      a.chunk_state[(unsigned long long)t * 32 + lane] = (uint8_t)entry;
      uint32_t fin;
      if (nv == CHUNK) fin = chunk_masks<true>(fs.laneaddr, v, nv, entry, Dm, Fm, Rm);
      else fin = chunk_masks<false>(fs.laneaddr, v, nv, entry, Dm, Fm, Rm);
      if (fin == INV_DEV && entry != INV_DEV && nv > 0) {
        const int p = first_inv_in_chunk(fs.lut, a.in + cstart, nv, fs.laneoff, entry);
        if (p >= 0) atomicMax(&a.ctrl->inv_neg, ~(a.base + cstart + (unsigned)p));
      }
      sg = warp_tile_segt(Dm, Fm, Rm, Vm);
    }
    if (lane == 0) s_wseg[grp][gw] = make_uint4(sg.cnt, sg.colf, sg.pos, 0u);
    FP_MARK(t1);
    nbar_arrive(bar_seg);
    if (live) emit_tile_local(a, ws, Dm, Fm, Rm, Vm);          // E1 while the scan warp looks back
    FP_MARK(t3);
    nbar_sync(bar_pre);
    FP_MARK(t6);
    if (live) emit_tile_global<TS>(a, s_cols, ws, s_wpre[grp][gw], Dm, Fm, Rm, Vm, a.base + tstart, a.base + cstart, cnt);
    FP_MARK(t7);
    if (gw == 1) {
      FP_ADD(0, 1); FP_ADD(1, t1 - t0); FP_ADD(3, t3 - t1); FP_ADD(5, t6 - t3); FP_ADD(6, t7 - t6);
    }
  }
  flush_counters(a, cnt);
}

}  // namespace parpa
