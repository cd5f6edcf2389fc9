// parpa_small.cuh — the whole parse of a SMALL input (<= SMALL_MAX_TILES warp tiles, 2 MB) in one
// cooperative launch: the paper's small-input regime ("several kernel launches per column"
// dominate 1 MB inputs) answered by one kernel whose phases are separated by grid-wide barriers.
//
//   k_small   grid = ceil(tiles / SMALL_WARPS) CTAs (<= #SMs, all co-resident: cooperative launch),
//             SMALL_WARPS warps per CTA, one warp per warp tile per phase:
//     1. pass 1 (S1-S2): the chunk τ and the warp ∘-scan -> lane-exclusive τ, warp-tile τ (global)
//     -- grid barrier --
//     2. τ scan (S3): every CTA scans all warp-tile τ itself (<= 1024 of them) into shared memory, so no
//        second barrier is needed; CTA 0 writes the range's τ
//     3. pass 2 (S4-S5a): masks and warp-tile SegT (global)
//     -- grid barrier --
//     4. ⊕ scan (S5b): every CTA scans all warp-tile SegTs and keeps the prefixes of its own tiles
//     5. emission (S6-S7): emit_tile per warp tile
//     -- grid barrier --
//     6. end-of-input action and status (one thread), then the device tier over the whole grid and the
//        status it settles.
// The same device functions as the large-input kernels: results are identical by construction, and the
// GPU tests run both (PARPA_SMALL=0 forces the multi-kernel path).
#pragma once
#include <cooperative_groups.h>

namespace parpa {

constexpr int SMALL_WARPS = 16;
constexpr int SMALL_NP = 4;                            // warps sharing one tile in the emission phase
constexpr uint32_t SMALL_MAX_TILES = 1024;             // 2 MB
constexpr size_t SMALL_SMEM = LUT_BYTES + (SMALL_WARPS + 2) * sizeof(WarpScratch) + 256;   // 16 + spare + split slack

__device__ __forceinline__ void small_smem(uint8_t *smem, int warp, int lane, uint8_t *&lut, WarpScratch *&ws,
                                           uint32_t &laneaddr, uint32_t &laneoff, uint8_t *&spare) {
  const uint32_t sb0 = smem_u32(smem);
  const uint32_t sb = (sb0 + 15u) & ~15u;
  uint8_t *base = smem + (sb - sb0);
  const uint32_t lut_off = ((sb + 0xFFFFu) & ~0xFFFFu) - sb;
  const uint32_t nfirst = lut_off / (uint32_t)sizeof(WarpScratch);
  auto slot = [&](uint32_t w) -> uint32_t {
    return w < nfirst ? w * (uint32_t)sizeof(WarpScratch)
                      : lut_off + LUT_BYTES + (w - nfirst) * (uint32_t)sizeof(WarpScratch);
  };
  lut = base + lut_off;
  ws = reinterpret_cast<WarpScratch *>(base + slot((uint32_t)warp));
  spare = base + slot(SMALL_WARPS);                     // one more slot: the scan arrays (<= 4 KB)
  laneoff = (uint32_t)(lane & 15) * 8u;
  laneaddr = laneoff | (((sb + lut_off) >> 16) << 16);       // PRMT layout
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SMALL_MARK(i) do { if (a.prof && blockIdx.x == 0 && threadIdx.x == 0) a.prof[i] = gtimer(); } while (0)

template <bool TS>
__global__ void __launch_bounds__(SMALL_WARPS * 32, 1) k_small(const __grid_constant__ KArgs a, const __grid_constant__ DfaK dfa,
                                                           const __grid_constant__ ColsK colsk) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ ColDesc s_cols[MAX_COLS];
  __shared__ uint32_t s_w32[SMALL_WARPS];
  __shared__ Seg s_wseg[SMALL_WARPS];
  __shared__ Seg s_carry, s_seg_all;
  __shared__ uint32_t s_tau_all;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t *lut, *spare;
  WarpScratch *ws;
  uint32_t laneaddr, laneoff;
  small_smem(smem, warp, lane, lut, ws, laneaddr, laneoff, spare);
  uint32_t *s_pre = reinterpret_cast<uint32_t *>(spare);          // [SMALL_MAX_TILES] exclusive τ per warp tile
  SMALL_MARK(0);
  build_lut(lut, dfa);
  for (int c = threadIdx.x; c < (int)a.C; c += blockDim.x) s_cols[c] = colsk.c[c];
  __syncthreads();
  SMALL_MARK(1);
  const uint32_t nt = a.ntiles, nwarps = gridDim.x * SMALL_WARPS, gw = blockIdx.x * SMALL_WARPS + warp;
  const uint32_t ngroups = nwarps / SMALL_NP, grp = gw / SMALL_NP, part = gw % SMALL_NP;
  WarpScratch *gws = ws;                               // the group's shared scratch: its part-0 warp's slot
  {
    uint8_t *l2; uint8_t *sp2; uint32_t la2, lo2;
    small_smem(smem, warp - (int)part, lane, l2, gws, la2, lo2, sp2);
  }

  // ---- 1. pass 1 ----
  for (uint32_t t = gw; t < nt; t += nwarps) {
    const unsigned long long cstart = (unsigned long long)t * WT + (unsigned long long)lane * CHUNK;
    const int nv = chunk_valid(a, cstart);
    uint32_t v[16], t0, t1, qt[3];
    load_chunk(a.in + cstart, nv, v);
    if (dfa.nlive <= 4) {
      const uint32_t la4 = laneaddr - laneoff + (uint32_t)lane * 4u;   // one 4-byte slot per lane
      if (nv == CHUNK) chunk_tau4<true, true>(la4, v, nv, t0, t1, qt);
      else chunk_tau4<false, true>(la4, v, nv, t0, t1, qt);
    } else {
      if (nv == CHUNK) chunk_tau4<true>(laneaddr, v, nv, t0, t1, qt);
      else chunk_tau4<false>(laneaddr, v, nv, t0, t1, qt);
    }
    uint32_t agg;
    const uint32_t ex = warp_scan_tau(t0, t1, agg);
    a.lex[(unsigned long long)t * 32 + lane] = ex;
    if (lane == 0) a.wtau[t] = agg;
  }
  SMALL_MARK(2);
  grid.sync();
  SMALL_MARK(3);

  // ---- 2. τ scan: exclusive ∘-prefix of every warp tile, in shared memory ----
  {
    uint32_t carry = NIB_IDENT;
    for (uint32_t b = 0; b < nt; b += blockDim.x) {
      const uint32_t i = b + threadIdx.x;
      const uint32_t e = i < nt ? __ldcg(a.wtau + i) : NIB_IDENT;
      uint32_t inc = e;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc = compose_nib(o, inc);
      }
      if (lane == 31) s_w32[warp] = inc;
      __syncthreads();
      if (warp == 0) {                                 // exclusive scan of the warp aggregates (in place)
        uint32_t w = lane < SMALL_WARPS ? s_w32[lane] : NIB_IDENT;
#pragma unroll
        for (int d = 1; d < SMALL_WARPS; d <<= 1) {
          const uint32_t o = __shfl_up_sync(0xffffffffu, w, d);
          if (lane >= d) w = compose_nib(o, w);
        }
        const uint32_t ex = __shfl_up_sync(0xffffffffu, w, 1);
        if (lane < SMALL_WARPS) s_w32[lane] = lane == 0 ? NIB_IDENT : ex;
        if (lane == SMALL_WARPS - 1) s_tau_all = w;
      }
      __syncthreads();
      uint32_t lex = __shfl_up_sync(0xffffffffu, inc, 1);
      if (lane == 0) lex = NIB_IDENT;
      if (i < nt) s_pre[i] = compose_nib(compose_nib(carry, s_w32[warp]), lex);
      carry = compose_nib(carry, s_tau_all);
      __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.tot_tau = carry;
  }
  __syncthreads();
  SMALL_MARK(4);

  // ---- 3. pass 2 ----
  for (uint32_t t = gw; t < nt; t += nwarps) {
    const unsigned long long cstart = (unsigned long long)t * WT + (unsigned long long)lane * CHUNK;
    const int nv = chunk_valid(a, cstart);
    uint32_t v[16];
    load_chunk(a.in + cstart, nv, v);
    const uint32_t entry = nib_at(__ldcg(a.lex + (unsigned long long)t * 32 + lane), nib_at(s_pre[t], a.seed_dev));
    a.chunk_state[(unsigned long long)t * 32 + lane] = (uint8_t)entry;
    unsigned long long Dm, Fm, Rm;
    uint32_t fin, xprev;
    if (dfa.nlive <= 4) {
      const uint32_t la4 = laneaddr - laneoff + (uint32_t)lane * 4u;   // one 4-byte slot per lane
      if (nv == CHUNK) fin = chunk_masks<true, true>(la4, v, nv, entry, Dm, Fm, Rm, xprev);
      else fin = chunk_masks<false, true>(la4, v, nv, entry, Dm, Fm, Rm, xprev);
    } else {
      if (nv == CHUNK) fin = chunk_masks<true>(laneaddr, v, nv, entry, Dm, Fm, Rm, xprev);
      else fin = chunk_masks<false>(laneaddr, v, nv, entry, Dm, Fm, Rm, xprev);
    }
    if (fin == INV_DEV && entry != INV_DEV && nv > 0) {
      const int p = first_inv_in_chunk(lut + 128, a.in + cstart, nv, laneoff, entry);
      if (p >= 0) atomicMax(&a.ctrl->inv_neg, ~(a.base + cstart + (unsigned)p));
    }
    if (nv > 0 && cstart + (unsigned)nv == a.len) a.ctrl->last_cls = 0x100u | (xprev & 0xFu);   // for the EOI action
    unsigned long long *mk = a.masks + (unsigned long long)t * 96 + lane;
    mk[0] = Dm;
    mk[32] = Fm;
    mk[64] = Rm;
    const unsigned long long Vm = nv >= 64 ? ~0ull : ((1ull << nv) - 1ull);
    const SegT sg = warp_tile_segt(Dm, Fm, Rm, Vm);
    if (lane == 0) a.wseg[t] = make_uint4(sg.cnt, sg.colf, sg.pos, 0u);
  }
  SMALL_MARK(5);
  grid.sync();
  SMALL_MARK(6);

  // ---- 4. ⊕ scan: the prefix of each of this CTA's tiles (every CTA scans all tiles) ----
  {
    Seg carry = seg_ident();
    for (uint32_t b = 0; b < nt; b += blockDim.x) {
      const uint32_t i = b + threadIdx.x;
      Seg e = seg_ident();
      if (i < nt) {
        const uint4 w = __ldcg(a.wseg + i);
        e = segt_to_seg(SegT{w.x, w.y, w.z}, a.base + (unsigned long long)i * WT);
      }
      Seg inc = e;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const Seg o = shfl_up_seg(inc, d);
        if (lane >= d) inc = seg_op(o, inc);
      }
      if (lane == 31) s_wseg[warp] = inc;
      __syncthreads();
      if (warp == 0) {                                 // exclusive scan of the warp aggregates (in place)
        Seg w = lane < SMALL_WARPS ? s_wseg[lane] : seg_ident();
#pragma unroll
        for (int d = 1; d < SMALL_WARPS; d <<= 1) {
          const Seg o = shfl_up_seg(w, d);
          if (lane >= d) w = seg_op(o, w);
        }
        const Seg ex = shfl_up_seg(w, 1);
        if (lane < SMALL_WARPS) s_wseg[lane] = lane == 0 ? seg_ident() : ex;
        if (lane == SMALL_WARPS - 1) s_seg_all = w;
      }
      __syncthreads();
      Seg lex = shfl_up_seg(inc, 1);
      if (lane == 0) lex = seg_ident();
      // tile i is emitted by warp group (i mod ngroups) -> block (i mod ngroups) * SMALL_NP / SMALL_WARPS
      if (i < nt && (i % ngroups) * SMALL_NP / SMALL_WARPS == blockIdx.x) a.tinfo[i].excl = seg_op(seg_op(carry, s_wseg[warp]), lex);
      carry = seg_op(carry, s_seg_all);
      __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *a.tot_seg = carry;
      s_carry = carry;
    }
  }
  __syncthreads();                                     // this CTA's tinfo entries are visible to its warps
  SMALL_MARK(7);

  // ---- 5. emission ----
  EmitCounters cnt{0ull, 0ull, 0u};
  for (uint32_t t = grp; t < nt; t += ngroups) {       // SMALL_NP warps per tile (emit_tile NP > 1)
    const unsigned long long tstart = (unsigned long long)t * WT;
    const unsigned long long cstart = tstart + (unsigned long long)lane * CHUNK;
    const int nv = chunk_valid(a, cstart);
    const unsigned long long *mk = a.masks + (unsigned long long)t * 96 + lane;
    unsigned long long Dm = 0ull, Fm = 0ull, Rm = 0ull;
    if (part == 0) {
      uint32_t v[16];
      load_chunk(a.in + cstart, nv, v);
      stash_chunk(gws->bytes, lane, v);
      Dm = __ldcg(mk); Fm = __ldcg(mk + 32); Rm = __ldcg(mk + 64);
    }
    const unsigned long long Vm = nv >= 64 ? ~0ull : ((1ull << nv) - 1ull);
    const Masks<1> mm{{Dm}, {Fm}, {Rm}, {Vm}};
    emit_tile<TS, SMALL_NP>(a, s_cols, gws, seg_op(a.seed, a.tinfo[t].excl), mm, a.base + tstart,
                            a.base + cstart, cnt, part, 1 + warp / SMALL_NP);
  }
  flush_counters(a, cnt);
  SMALL_MARK(8);
  grid.sync();
  SMALL_MARK(9);

  // ---- 6. end of input and status (block 0), the device tier (every block; it needs the record count
  // only after a queue overflow), and the status the last block to finish settles ----
  if (blockIdx.x == 0 && threadIdx.x == 0) finalize_one(a, dfa, colsk);
  SMALL_MARK(10);
  grid.sync();           // the end-of-input field may have been queued; the sweep reads stats->records
  SMALL_MARK(11);
  deferred_all<TS>(a, dfa, colsk, (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x,
                   (unsigned long long)gridDim.x * blockDim.x);
  {
    __shared__ CollabSmem s_collab;                // long numeric fields: block tier, then device tier
    collab_tiers<TS>(a, colsk, s_collab);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&a.ctrl->deferred_done, 1u) + 1u == gridDim.x) {   // the last block out
      if (a.stats) collab_stats(a);
      if (a.stats && *reinterpret_cast<volatile unsigned int *>(&a.ctrl->unsupported) &&
          *reinterpret_cast<volatile int *>(&a.stats->status) != ST_EFORMAT)
        a.stats->status = ST_EUNSUPPORTED;
      // leave the control words zeroed: a reused workspace (parpa_parse_into_ws) needs no memset per parse
      volatile unsigned int *c = reinterpret_cast<volatile unsigned int *>(a.ctrl);
      for (int i = 0; i < (int)(sizeof(Ctrl) / 4); i++) c[i] = 0u;
    }
  }
  SMALL_MARK(12);
}

}  // namespace parpa
