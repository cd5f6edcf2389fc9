// parpa_passes.cuh — the scan half of the hot path as four chain-free / single-pass kernels.
//
//   k_pass1     S1+S2+S3a  per warp tile (2 KB, one 64-byte chunk per lane): the chunk's
//               state-transition vector through the shared-memory LUT, a warp ∘-scan
//               with shuffles -> lane-exclusive τ (lex) and the warp-tile aggregate.
//               No inter-CTA dependency: persistent grid, high occupancy.
//   k_tau_scan  S3b  single-pass scan of the warp-tile aggregates with decoupled look-back
//               (Merrill & Garland, the paper's P:250 reference): blocks of SCAN_TILE aggregates in
//               ticket order, block aggregate published before the look-back -> the τ of everything
//               before every warp tile; k_pass2 applies the range's entry state to it.
//   k_pass2     S4+S5a  per warp tile: lane entry = lex applied to the tile entry, re-simulation
//               -> DATA / DELIM / RECORD masks (the paper's bitmap indexes), record
//               count by POPCNT and the abs/rel column offset plus the open-field
//               carries, reduced over the warp -> one SegT per warp tile.
//   k_seg_scan  S5b  single-pass decoupled look-back scan of the warp-tile SegTs (⊕ of P:408-414,
//               64-bit positions) -> the prefix (records, fields, column, open field) of every warp
//               tile within the range; k_emit / k_finalize compose it after the range's seed.
//
// Every kernel is bounded by its own DRAM stream or ALU work; nothing spins on another CTA except the
// two small scans, whose look-backs cover SCAN_TILE warp tiles (4 MB of input) per block.
#pragma once

namespace parpa {

constexpr int PASS_WARPS = 32;                       // k_pass1 / k_pass2: one 1024-thread CTA per SM
constexpr size_t PASS_SMEM = LUT_BYTES + (PASS_WARPS + 1) * 2 * WT;   // LUT + two tile buffers per warp (+1 slack)

// Shared-memory layout of the pass kernels: the LUT at the first 64 KB-aligned shared address of the
// dynamic region (so a PRMT yields full LDS addresses, see lds_u2), the per-warp tile buffers in the
// space before and after it.
struct PassSmem {
  uint8_t *lut;
  uint4 *bufs;
  uint32_t laneaddr, laneoff;
};
__device__ __forceinline__ PassSmem pass_smem(uint8_t *smem, int warp, int lane) {
  const uint32_t sb = smem_u32(smem);
  const uint32_t lut_off = ((sb + 0xFFFFu) & ~0xFFFFu) - sb;
  const uint32_t nfirst = lut_off / (2 * WT);
  const uint32_t boff = (uint32_t)warp < nfirst ? (uint32_t)warp * 2 * WT
                                                : lut_off + LUT_BYTES + ((uint32_t)warp - nfirst) * 2 * WT;
  PassSmem p;
  p.lut = smem + lut_off;
  p.bufs = reinterpret_cast<uint4 *>(smem + boff);
  p.laneoff = (uint32_t)(lane & 15) * 8u;
  p.laneaddr = p.laneoff | (((sb + lut_off) >> 16) << 16);   // PRMT layout (pass 1)
  return p;
}
#ifndef PARPA_SCAN_ITEMS
#define PARPA_SCAN_ITEMS 8
#endif
constexpr int SCAN_THREADS = 256, SCAN_ITEMS = PARPA_SCAN_ITEMS;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS; // warp tiles per scan block (4 MB of input at 8 items)
// k_seg_scan: fewer items per thread (more, shorter blocks: its look-back chain is the cost; measured 4 vs 8
// items: 0.162 -> 0.143 ms on yelp 4.8 GB).  The look-back arrays are sized by its (larger) block count.
#ifndef PARPA_SEG_ITEMS
#define PARPA_SEG_ITEMS 4
#endif
constexpr int SEG_ITEMS = PARPA_SEG_ITEMS;
constexpr int SEG_TILE = SCAN_THREADS * SEG_ITEMS;
static_assert(SEG_TILE <= SCAN_TILE, "the workspace's look-back arrays are sized by k_seg_scan's blocks");

__device__ __forceinline__ int chunk_valid(const KArgs &a, unsigned long long cstart) {
  return cstart >= a.len ? 0 : (int)min((unsigned long long)CHUNK, a.len - cstart);
}

// ---- per-warp double-buffered tile staging (cp.async, no registers held across the wait) ----------
// Each lane copies its own 64-byte chunk as four 16-byte units and reads back only those, so a lane's
// own cp.async.wait_group orders everything it reads (no warp barrier needed).  Units are XOR-swizzled
// so that the 128-bit reads of eight consecutive lanes hit distinct banks.
__device__ __forceinline__ uint32_t pswz(int lane, int u) { return (uint32_t)lane * 4u + (uint32_t)(u ^ ((lane >> 1) & 3)); }
__device__ __forceinline__ void cp_async16(void *dst, const void *src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
// nfull = tiles entirely inside the input (a 32-bit compare per tile: the pass kernels are ALU-bound)
__device__ __forceinline__ void stage_chunk(const KArgs &a, uint4 *buf, uint32_t t, int lane, uint32_t nfull) {
  const unsigned long long cstart = (unsigned long long)t * WT + (unsigned long long)lane * CHUNK;
  if (t < nfull) {                                                     // whole tile in range (all but the last):
    const uint8_t *src = a.in + cstart;                                // no per-unit clamps
#pragma unroll
    for (int u = 0; u < 4; u++) cp_async16(buf + pswz(lane, u), src + 16 * u, 16u);
    return;
  }
  const int nv = chunk_valid(a, cstart);
#pragma unroll
  for (int u = 0; u < 4; u++) {
    const int nb = max(0, min(16, nv - 16 * u));                     // tail: zero-filled
    cp_async16(buf + pswz(lane, u), nb ? (const void *)(a.in + cstart + 16 * u) : (const void *)a.in, (uint32_t)nb);
  }
}
__device__ __forceinline__ void read_chunk(const uint4 *buf, int lane, uint32_t (&v)[16]) {
#pragma unroll
  for (int u = 0; u < 4; u++) {
    const uint4 x = buf[pswz(lane, u)];
    v[4 * u] = x.x; v[4 * u + 1] = x.y; v[4 * u + 2] = x.z; v[4 * u + 3] = x.w;
  }
}

// ---- K1: pass 1 ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(PASS_WARPS * 32, 1) k_pass1(const KArgs a, const DfaK dfa) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const PassSmem ps = pass_smem(smem, warp, lane);
  PdlTrigger pdl_trigger;
  build_lut(ps.lut, dfa);
  __syncthreads();
  pdl_wait();
  uint4 *bufs = ps.bufs;
  const uint32_t nw = gridDim.x * PASS_WARPS;
  const uint32_t nfull = (uint32_t)(a.len / WT);
  uint32_t t = blockIdx.x * PASS_WARPS + warp;
  if (t < a.ntiles) stage_chunk(a, bufs, t, lane, nfull);
  cp_async_commit();
  for (uint32_t i = 0; t < a.ntiles; t += nw, i ^= 1u) {
    if (t + nw < a.ntiles) stage_chunk(a, bufs + (i ^ 1u) * (WT / 16), t + nw, lane, nfull);
    cp_async_commit();
    cp_async_wait1();
    uint32_t v[16], t0, t1, qt[3], agg, ex;
    read_chunk(bufs + i * (WT / 16), lane, v);
    if (dfa.nlive <= 4) {                                   // warp-uniform (kernel parameter)
      const uint32_t la4 = ps.laneaddr - ps.laneoff + (uint32_t)lane * 4u;   // one 4-byte slot per lane
      if (t < nfull) {
        chunk_tau4<true, true>(la4, v, CHUNK, t0, t1, qt);
      } else {
        const int nv = chunk_valid(a, (unsigned long long)t * WT + (unsigned long long)lane * CHUNK);
        chunk_tau4<false, true>(la4, v, nv, t0, t1, qt);
      }
      ex = warp_scan_tau4(t0, agg);
    } else {
      if (t < nfull) {
        chunk_tau4<true>(ps.laneaddr, v, CHUNK, t0, t1, qt);
      } else {
        const int nv = chunk_valid(a, (unsigned long long)t * WT + (unsigned long long)lane * CHUNK);
        chunk_tau4<false>(ps.laneaddr, v, nv, t0, t1, qt);
      }
      ex = warp_scan_tau(t0, t1, agg);
    }
    a.lex[(unsigned long long)t * 32 + lane] = ex;
    if (lane == 0) a.wtau[t] = agg;
  }
}

// ---- K2: τ scan over warp tiles -----------------------------------------------------------------
__global__ void __launch_bounds__(SCAN_THREADS) k_tau_scan(const KArgs a) {
  __shared__ uint32_t s_bid, s_prefix;
  __shared__ uint32_t s_warp[SCAN_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  PdlTrigger pdl_trigger;
  pdl_wait();
  if (threadIdx.x == 0) s_bid = atomicAdd(&a.ctrl->ticket, 1u);   // ticket order: look-backs only
  __syncthreads();                                                   // wait on started blocks
  const uint32_t b = s_bid;
  const unsigned long long t0 = (unsigned long long)b * SCAN_TILE + (unsigned long long)threadIdx.x * SCAN_ITEMS;
  uint32_t e[SCAN_ITEMS];
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; k++) e[k] = t0 + k < a.ntiles ? a.wtau[t0 + k] : NIB_IDENT;
  uint32_t loc = e[0];
#pragma unroll
  for (int k = 1; k < SCAN_ITEMS; k++) loc = compose_nib(loc, e[k]);
  uint32_t inc = loc;                                                // warp inclusive ∘-scan
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc = compose_nib(o, inc);
  }
  uint32_t wex = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) wex = NIB_IDENT;
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < SCAN_THREADS / 32 ? s_warp[lane] : NIB_IDENT;
#pragma unroll
    for (int d = 1; d < SCAN_THREADS / 32; d <<= 1) {
      uint32_t o = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w = compose_nib(o, w);
    }
    const uint32_t bagg = __shfl_sync(0xffffffffu, w, SCAN_THREADS / 32 - 1);
    uint32_t bex = __shfl_up_sync(0xffffffffu, w, 1);
    if (lane < SCAN_THREADS / 32) s_warp[lane] = lane == 0 ? NIB_IDENT : bex;
    uint32_t prefix = NIB_IDENT;
    if (b == 0) {
      if (lane == 0) st_relaxed_u64(a.tau_desc, ((unsigned long long)FLAG_INCL << 32) | bagg);
    } else {
      if (lane == 0) st_relaxed_u64(a.tau_desc + b, ((unsigned long long)FLAG_AGG << 32) | bagg);
      prefix = lookback_tau(a, b);
      if (lane == 0) st_relaxed_u64(a.tau_desc + b, ((unsigned long long)FLAG_INCL << 32) | compose_nib(prefix, bagg));
    }
    if (lane == 0) {
      s_prefix = prefix;
      if ((unsigned long long)(b + 1) * SCAN_TILE >= a.ntiles) *a.tot_tau = compose_nib(prefix, bagg);
    }
  }
  __syncthreads();
  uint32_t cur = compose_nib(compose_nib(s_prefix, s_warp[warp]), wex);
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; k++) {
    if (t0 + k < a.ntiles) a.wpre[t0 + k] = cur;
    cur = compose_nib(cur, e[k]);
  }
}

// ---- the warp tile's SegT directly from the lanes' masks (ballots + warp reductions) ----------------
// Same value as the ordered ∘-reduction of the 32 chunk summaries (segt_op over chunk_segt): record and
// delimiter counts, the column after the last record delimiter, and the open field after
// the last delimiter (first / last DATA byte, control bytes before / inside / after).
__device__ __forceinline__ SegT warp_tile_segt(unsigned long long Dm, unsigned long long Fm, unsigned long long Rm,
                                               unsigned long long Vm) {
  // Branch-free form: every per-lane quantity is a select on the lane's position relative to the lane of
  // the last record / last delimiter / first and last open DATA byte (no divergent single-lane paths).
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  const uint32_t nrec = __reduce_add_sync(FULL, (uint32_t)__popcll(Rm));
  const uint32_t nd = __reduce_add_sync(FULL, (uint32_t)__popcll(Fm));
  // bits strictly after the last record / delimiter of this lane (all bits if it has none)
  const unsigned long long aftR = Rm ? (~0ull << (63 - __clzll(Rm))) << 1 : ~0ull;
  const unsigned long long aftF = Fm ? (~0ull << (63 - __clzll(Fm))) << 1 : ~0ull;
  const unsigned rb = __ballot_sync(FULL, Rm != 0ull), fb = __ballot_sync(FULL, Fm != 0ull);
  const int L = rb ? 31 - __clz(rb) : -1, Lf = fb ? 31 - __clz(fb) : -1;
  const uint32_t col = __reduce_add_sync(FULL, lane >= L ? (uint32_t)__popcll(Fm & aftR) : 0u);
  uint32_t fl = (rb ? F_ABS : 0u) | (fb ? F_HD : 0u);
  const unsigned long long open = lane >= Lf ? (Vm & aftF) : 0ull;     // the field left open at the end
  const unsigned long long Km = Vm & ~Dm & ~Fm;
  const unsigned long long Do = Dm & open, Ko = Km & open;
  const unsigned db = __ballot_sync(FULL, Do != 0ull);
  uint32_t pos = 0xFFFFFFFFu, pf;
  if (db) {
    const int f0 = __ffs(db) - 1, f1 = 31 - __clz(db);
    const int fdloc = __shfl_sync(FULL, Do ? __ffsll((long long)Do) - 1 : 0, f0);
    const int ldloc = __shfl_sync(FULL, Do ? 63 - __clzll(Do) : 0, f1);
    const unsigned long long belowF = (1ull << fdloc) - 1ull, aboveF = (~0ull << fdloc) << 1;
    const unsigned long long belowL = (1ull << ldloc) - 1ull, aboveL = (~0ull << ldloc) << 1;
    const unsigned long long pre_m = lane < f0 ? ~0ull : lane == f0 ? belowF : 0ull;
    const unsigned long long pc_m = lane > f1 ? ~0ull : lane == f1 ? aboveL : 0ull;
    const unsigned long long in_m = (lane > f0 ? ~0ull : lane == f0 ? aboveF : 0ull) &
                                    (lane < f1 ? ~0ull : lane == f1 ? belowL : 0ull);
    pf = ((Ko & pre_m) ? F_PRE : 0u) | ((Ko & pc_m) ? F_PC : 0u) | ((Ko & in_m) ? F_IC : 0u);
    pos = (uint32_t)(f0 * CHUNK + fdloc) | ((uint32_t)(f1 * CHUNK + ldloc) << 16);
  } else {
    pf = Ko ? F_PRE : 0u;
  }
  fl |= __reduce_or_sync(FULL, pf);
  return SegT{nrec | (nd << 16), col | (fl << 16), pos};
}

// ---- K3: pass 2 ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(PASS_WARPS * 32, 1) k_pass2(const KArgs a, const DfaK dfa) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const PassSmem ps = pass_smem(smem, warp, lane);
  PdlTrigger pdl_trigger;
  build_lut_step_dp(ps.lut, dfa);                          // DP4A layout: step rows only
  const uint32_t lbase = smem_u32(ps.lut) + ps.laneoff;
  __syncthreads();
  pdl_wait();
  uint4 *bufs = ps.bufs;
  const uint32_t nw = gridDim.x * PASS_WARPS;
  const uint32_t nfull = (uint32_t)(a.len / WT);
  uint32_t t = blockIdx.x * PASS_WARPS + warp;
  if (t < a.ntiles) stage_chunk(a, bufs, t, lane, nfull);
  cp_async_commit();
  // each tile's lane-exclusive τ and tile prefix are loaded one iteration ahead (their latency was exposed
  // right before the re-simulation: -3 to -4% on pass 2)
  uint32_t lex_n = t < a.ntiles ? a.lex[(unsigned long long)t * 32 + lane] : 0u, wpre_n = t < a.ntiles ? a.wpre[t] : 0u;
  for (uint32_t i = 0; t < a.ntiles; t += nw, i ^= 1u) {
    if (t + nw < a.ntiles) stage_chunk(a, bufs + (i ^ 1u) * (WT / 16), t + nw, lane, nfull);
    cp_async_commit();
    const uint32_t lex_c = lex_n, wpre_c = wpre_n;
    if (t + nw < a.ntiles) { lex_n = a.lex[(unsigned long long)(t + nw) * 32 + lane]; wpre_n = a.wpre[t + nw]; }
    cp_async_wait1();
    const unsigned long long cstart = (unsigned long long)t * WT + (unsigned long long)lane * CHUNK;
    const int nv = t < nfull ? CHUNK : chunk_valid(a, cstart);
    uint32_t v[16];
    read_chunk(bufs + i * (WT / 16), lane, v);
    const uint32_t entry = nib_at(lex_c, nib_at(wpre_c, a.seed_dev));
    a.chunk_state[(unsigned long long)t * 32 + lane] = (uint8_t)entry;
    unsigned long long Dm, Fm, Rm;
    uint32_t fin, xprev;
    if (dfa.nlive <= 4) {
      const uint32_t la4 = lbase - ps.laneoff + (uint32_t)lane * 4u;   // one 4-byte slot per lane
      if (nv == CHUNK) fin = CHUNK_MASKS<true, true, true>(la4, v, nv, entry, Dm, Fm, Rm, xprev);
      else fin = CHUNK_MASKS<false, true, true>(la4, v, nv, entry, Dm, Fm, Rm, xprev);
    } else {
      if (nv == CHUNK) fin = CHUNK_MASKS<true, false, true>(lbase, v, nv, entry, Dm, Fm, Rm, xprev);
      else fin = CHUNK_MASKS<false, false, true>(lbase, v, nv, entry, Dm, Fm, Rm, xprev);
    }
    if (fin == INV_DEV && entry != INV_DEV && nv > 0) {
      int p = first_inv_in_chunk(ps.lut, a.in + cstart, nv, ps.laneoff, entry, STEP_ROW_DP);
      if (p >= 0) atomicMax(&a.ctrl->inv_neg, ~(a.base + cstart + (unsigned)p));
    }
    if (t + 1u == a.ntiles && nv > 0 && cstart + (unsigned)nv == a.len)
      a.ctrl->last_cls = 0x100u | (xprev & 0xFu);                            // for the EOI action
    unsigned long long *mk = a.masks + (unsigned long long)t * 96 + lane;   // for k_emit
    mk[0] = Dm;
    mk[32] = Fm;
    mk[64] = Rm;
    const unsigned long long Vm = t < nfull ? ~0ull : nv >= 64 ? ~0ull : ((1ull << nv) - 1ull);
    const SegT s = warp_tile_segt(Dm, Fm, Rm, Vm);
    if (lane == 0) a.wseg[t] = make_uint4(s.cnt, s.colf, s.pos, 0u);
  }
}

// ---- K4: record / column scan over warp tiles ---------------------------------------------------
__device__ __forceinline__ Seg shfl_up_seg(const Seg &s, int d) {
  Seg o;
  o.recs = __shfl_up_sync(0xffffffffu, s.recs, d);
  o.nflds = __shfl_up_sync(0xffffffffu, s.nflds, d);
  o.fd = __shfl_up_sync(0xffffffffu, s.fd, d);
  o.ld = __shfl_up_sync(0xffffffffu, s.ld, d);
  o.col = __shfl_up_sync(0xffffffffu, s.col, d);
  o.flags = __shfl_up_sync(0xffffffffu, s.flags, d);
  return o;
}
__device__ __forceinline__ Seg wseg_at(const KArgs &a, unsigned long long t) {
  const uint4 w = a.wseg[t];
  return segt_to_seg(SegT{w.x, w.y, w.z}, a.base + t * WT);
}

// returns B_0 ∘ ... ∘ B_{b-1} over the block aggregates; one descriptor per lane per round trip
__device__ Seg lookback_bseg(const KArgs &a, uint32_t b) {
  const int lane = threadIdx.x & 31;
  Seg acc = seg_ident();
  long long base = (long long)b - 1;
  while (true) {
    const long long j = base - lane;
    uint32_t f = j >= 0 ? ld_acquire_u32(a.bflag + j) : FLAG_INCL;
    unsigned incl, zero;
    int L;
    while (true) {
      incl = __ballot_sync(0xffffffffu, f == FLAG_INCL);
      zero = __ballot_sync(0xffffffffu, f == 0u);
      L = incl ? __ffs(incl) - 1 : 31;
      const unsigned need = L == 31 ? 0xFFFFFFFFu : ((2u << L) - 1u);
      if (!(zero & need)) break;
      __nanosleep(32);
      if (f == 0u) f = ld_acquire_u32(a.bflag + j);
    }
    Seg v = seg_ident();
    if (lane <= L && j >= 0) v = f == FLAG_INCL ? ldcg_seg(a.bincl + j) : ldcg_seg(a.bagg + j);
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {                            // higher lane = earlier block
      Seg o = shfl_down_seg(v, dd);
      if (lane + dd < 32) v = seg_op(o, v);
    }
    acc = seg_op(shfl_seg(v, 0), acc);
    if (incl) break;
    base -= 32;
  }
  return acc;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_seg_scan(const KArgs a) {
  __shared__ uint32_t s_bid;
  __shared__ Seg s_prefix;
  __shared__ Seg s_warp[SCAN_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  PdlTrigger pdl_trigger;
  pdl_wait();
  if (threadIdx.x == 0) s_bid = atomicAdd(&a.ctrl->ticket2, 1u);
  __syncthreads();
  const uint32_t b = s_bid;
  const unsigned long long t0 = (unsigned long long)b * SEG_TILE + (unsigned long long)threadIdx.x * SEG_ITEMS;
  Seg loc = seg_ident();
#pragma unroll
  for (int k = 0; k < SEG_ITEMS; k++)
    if (t0 + k < a.ntiles) loc = seg_op(loc, wseg_at(a, t0 + k));
  Seg inc = loc;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    Seg o = shfl_up_seg(inc, d);
    if (lane >= d) inc = seg_op(o, inc);
  }
  Seg wex = shfl_up_seg(inc, 1);
  if (lane == 0) wex = seg_ident();
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    Seg w = lane < SCAN_THREADS / 32 ? s_warp[lane] : seg_ident();
#pragma unroll
    for (int d = 1; d < SCAN_THREADS / 32; d <<= 1) {
      Seg o = shfl_up_seg(w, d);
      if (lane >= d) w = seg_op(o, w);
    }
    const Seg bagg = shfl_seg(w, SCAN_THREADS / 32 - 1);
    Seg bex = shfl_up_seg(w, 1);
    if (lane < SCAN_THREADS / 32) s_warp[lane] = lane == 0 ? seg_ident() : bex;
    Seg prefix = seg_ident();                       // unseeded: k_emit / k_finalize apply a.seed
    if (b == 0) {
      if (lane == 0) {
        stcg_seg(a.bincl, bagg);
        st_release_u32(a.bflag, FLAG_INCL);
      }
    } else {
      if (lane == 0) {
        stcg_seg(a.bagg + b, bagg);
        st_release_u32(a.bflag + b, FLAG_AGG);
      }
      prefix = lookback_bseg(a, b);
      if (lane == 0) {
        stcg_seg(a.bincl + b, seg_op(prefix, bagg));
        st_release_u32(a.bflag + b, FLAG_INCL);
      }
    }
    if (lane == 0) {
      s_prefix = prefix;
      if ((unsigned long long)(b + 1) * SEG_TILE >= a.ntiles) *a.tot_seg = seg_op(prefix, bagg);
    }
  }
  __syncthreads();
  Seg cur = seg_op(seg_op(s_prefix, s_warp[warp]), wex);
#pragma unroll
  for (int k = 0; k < SEG_ITEMS; k++) {
    if (t0 + k >= a.ntiles) break;
    a.tinfo[t0 + k].excl = cur;
    cur = seg_op(cur, wseg_at(a, t0 + k));
  }
}

}  // namespace parpa

// ---- string materialisation (the paper's CSS P:439-457) ---------------------------------
// From a completed parse of the same bytes: for row r of a column (span offset / length), the DATA
// bytes inside the span (control bytes such as the escaping quote of "" dropped), concatenated in row
// order: offsets[R + 1] (Arrow layout) and the bytes.  The DATA bytes are located with the chunk
// masks that k_pass2 stores.
namespace parpa {

constexpr uint32_t MISSING_LEN_DEV = 0xFFFFFFFFu;

__device__ __forceinline__ unsigned long long dmask_of_chunk(const KArgs &a, unsigned long long k) {
  return a.masks[(k >> 5) * 96 + (k & 31)];                  // [tile][D,F,R][lane]
}
// number of DATA bytes in [p, p + n) of the range
__device__ unsigned long long data_bytes_in(const KArgs &a, unsigned long long p, unsigned long long n) {
  unsigned long long cnt = 0, end = p + n;
  while (p < end) {
    const unsigned long long k = p >> 6, lo = p & 63, hi = min(64ull, end - (k << 6));
    unsigned long long m = dmask_of_chunk(a, k) >> lo;
    const unsigned long long w = hi - lo;
    if (w < 64) m &= (1ull << w) - 1ull;
    cnt += __popcll(m);
    p = (k + 1) << 6;
  }
  return cnt;
}

// CSS layouts: ARROW = the DATA bytes of every field concatenated (offsets index);
// INLINE = each field followed by a terminator byte (inline-terminated CSS); VECTOR = ARROW bytes plus an
// auxiliary byte vector, nonzero at the last symbol of every non-empty field (vector-delimited CSS).
enum { CSS_ARROW = 0, CSS_INLINE = 1, CSS_VECTOR = 2 };

// extra = 1 for the inline-terminated layout (one terminator per field, missing / empty fields included)
__global__ void k_str_len(const KArgs a, const unsigned long long *off, const uint32_t *len, unsigned long long rows,
                          unsigned long long *lens, uint32_t extra) {
  for (unsigned long long r = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; r < rows;
       r += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t L = len[r];
    lens[r] = ((L == MISSING_LEN_DEV || L == 0) ? 0ull : data_bytes_in(a, off[r] - a.base, L)) + extra;
  }
}

// in-place exclusive scan of v[0, n) (unsigned 64-bit), v[n] = total: single pass, decoupled look-back
// over blocks of SCAN_TILE elements (flags: 1 aggregate, 2 inclusive; payload then release-flag)
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_u64(unsigned long long *v, unsigned long long n,
                                                          unsigned int *ticket, uint32_t *flag,
                                                          unsigned long long *agg, unsigned long long *incl) {
  __shared__ uint32_t s_bid;
  __shared__ unsigned long long s_warp[SCAN_THREADS / 32], s_prefix;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_bid = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t b = s_bid;
  const unsigned long long i0 = (unsigned long long)b * SCAN_TILE + (unsigned long long)threadIdx.x * SCAN_ITEMS;
  unsigned long long x[SCAN_ITEMS], loc = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; k++) {
    x[k] = i0 + k < n ? v[i0 + k] : 0ull;
    loc += x[k];
  }
  unsigned long long inc = loc;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < SCAN_THREADS / 32 ? s_warp[lane] : 0ull;
#pragma unroll
    for (int d = 1; d < SCAN_THREADS / 32; d <<= 1) {
      const unsigned long long o = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += o;
    }
    const unsigned long long bagg = __shfl_sync(0xffffffffu, w, SCAN_THREADS / 32 - 1);
    const unsigned long long bex = __shfl_up_sync(0xffffffffu, w, 1);
    if (lane < SCAN_THREADS / 32) s_warp[lane] = lane == 0 ? 0ull : bex;
    unsigned long long prefix = 0;
    if (b == 0) {
      if (lane == 0) { __stcg(incl, bagg); st_release_u32(flag, FLAG_INCL); }
    } else {
      if (lane == 0) { __stcg(agg + b, bagg); st_release_u32(flag + b, FLAG_AGG); }
      long long base = (long long)b - 1;
      while (true) {                                          // look-back, one block per lane
        const long long j = base - lane;
        uint32_t f = j >= 0 ? ld_acquire_u32(flag + j) : FLAG_INCL;
        unsigned incm, zero;
        int L;
        while (true) {
          incm = __ballot_sync(0xffffffffu, f == FLAG_INCL);
          zero = __ballot_sync(0xffffffffu, f == 0u);
          L = incm ? __ffs(incm) - 1 : 31;
          const unsigned need = L == 31 ? 0xFFFFFFFFu : ((2u << L) - 1u);
          if (!(zero & need)) break;
          __nanosleep(32);
          if (f == 0u) f = ld_acquire_u32(flag + j);
        }
        unsigned long long val = 0;
        if (lane <= L && j >= 0) val = f == FLAG_INCL ? __ldcg(incl + j) : __ldcg(agg + j);
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) val += __shfl_down_sync(0xffffffffu, val, d);
        prefix += __shfl_sync(0xffffffffu, val, 0);
        if (incm) break;
        base -= 32;
      }
      if (lane == 0) { __stcg(incl + b, prefix + bagg); st_release_u32(flag + b, FLAG_INCL); }
    }
    if (lane == 0) {
      s_prefix = prefix;
      if ((unsigned long long)(b + 1) * SCAN_TILE >= n) v[n] = prefix + bagg;   // total
    }
  }
  __syncthreads();
  const unsigned long long wex = __shfl_up_sync(0xffffffffu, inc, 1);
  unsigned long long cur = s_prefix + s_warp[warp] + (lane == 0 ? 0ull : wex) ;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; k++) {
    if (i0 + k < n) v[i0 + k] = cur;
    cur += x[k];
  }
}

// one warp per row: copy the DATA bytes of the span to data[offsets[r] ...]; INLINE: the terminator after
// them (a DATA byte equal to the terminator sets *clash: the layout needs it absent); VECTOR:
// aux (zeroed by the caller) gets a 1 at the field's last symbol
__global__ void k_str_copy(const KArgs a, const unsigned long long *off, const uint32_t *len, unsigned long long rows,
                           const unsigned long long *offsets, uint8_t *data, uint32_t mode, uint32_t term,
                           uint8_t *aux, unsigned int *clash) {
  const int lane = threadIdx.x & 31;
  const unsigned long long nw = (unsigned long long)gridDim.x * (blockDim.x >> 5);
  const uint32_t extra = mode == CSS_INLINE ? 1u : 0u;
  bool hit = false;
  for (unsigned long long r = blockIdx.x * (unsigned long long)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
       r += nw) {
    const uint32_t L = len[r];
    const unsigned long long o0 = offsets[r], n = offsets[r + 1] - o0 - extra;   // DATA bytes of the field
    if (extra && lane == 0) data[o0 + n] = (uint8_t)term;
    if (L == MISSING_LEN_DEV || L == 0 || n == 0) continue;
    if (mode == CSS_VECTOR && lane == 0) aux[o0 + n - 1] = 1;
    const unsigned long long p0 = off[r] - a.base;
    const bool all = n == L;                                   // no control byte inside: plain copy
    unsigned long long o = o0;
    for (unsigned long long q = 0; q < L; q += 32) {
      const unsigned long long p = p0 + q + lane;
      const bool in = q + lane < L;
      const uint8_t c = in ? a.in[p] : 0;
      bool keep = in;
      if (!all && in) keep = (dmask_of_chunk(a, p >> 6) >> (p & 63)) & 1ull;
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        data[o + __popc(m & ((1u << lane) - 1u))] = c;
        hit |= extra && c == (uint8_t)term;
      }
      o += __popc(m);
    }
  }
  if (hit) atomicOr(clash, 1u);
}

// ---- CSS index generation: the positions of the terminators (INLINE: data[k] == term) or of the
// nonzero auxiliary entries (VECTOR), in order.  Per 2 KB tile a count, an exclusive scan, then the writes.
__device__ __forceinline__ bool css_mark(uint32_t mode, const uint8_t *data, const uint8_t *aux, uint32_t term,
                                         unsigned long long k) {
  return mode == CSS_INLINE ? data[k] == (uint8_t)term : aux[k] != 0;
}
__global__ void k_css_count(uint32_t mode, const uint8_t *data, const uint8_t *aux, uint32_t term, unsigned long long n,
                            unsigned long long *cnt) {
  const int lane = threadIdx.x & 31;
  const unsigned long long ntile = (n + WT - 1) / WT;
  for (unsigned long long t = blockIdx.x * (unsigned long long)(blockDim.x >> 5) + (threadIdx.x >> 5); t < ntile;
       t += (unsigned long long)gridDim.x * (blockDim.x >> 5)) {
    uint32_t c = 0;
    for (unsigned long long k = t * WT + lane; k < min(n, (t + 1) * WT); k += 32) c += css_mark(mode, data, aux, term, k);
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) cnt[t] = c;
  }
}
__global__ void k_css_write(uint32_t mode, const uint8_t *data, const uint8_t *aux, uint32_t term, unsigned long long n,
                            const unsigned long long *base, unsigned long long *idx) {
  const int lane = threadIdx.x & 31;
  const unsigned long long ntile = (n + WT - 1) / WT;
  for (unsigned long long t = blockIdx.x * (unsigned long long)(blockDim.x >> 5) + (threadIdx.x >> 5); t < ntile;
       t += (unsigned long long)gridDim.x * (blockDim.x >> 5)) {
    unsigned long long o = base[t];
    for (unsigned long long k0 = t * WT; k0 < min(n, (t + 1) * WT); k0 += 32) {
      const unsigned long long k = k0 + lane;
      const bool m = k < n && css_mark(mode, data, aux, term, k);
      const unsigned b = __ballot_sync(0xffffffffu, m);
      if (m) idx[o + __popc(b & ((1u << lane) - 1u))] = k;
      o += __popc(b);
    }
  }
}

}  // namespace parpa

// ---- column-count inference (reading R13's NEXT) ------------------------------------------
// Fields per record over the whole input: each lane walks its delimiters from its exact starting
// column (the tile prefix composed with the lane-exclusive chunk summaries), and every record
// delimiter contributes column + 1.  Warp min / max, then one atomic per warp.
namespace parpa {
__global__ void k_infer_cols(const KArgs a, unsigned int *minmax) {
  const int lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  uint32_t mn = 0xFFFFFFFFu, mx = 0;
  for (uint32_t t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < a.ntiles; t += nw) {
    const unsigned long long cstart = (unsigned long long)t * WT + (unsigned long long)lane * CHUNK;
    const int nv = chunk_valid(a, cstart);
    const unsigned long long *mk = a.masks + (unsigned long long)t * 96 + lane;
    const unsigned long long Dm = mk[0], Fm = mk[32], Rm = mk[64];
    const unsigned long long Vm = nv >= 64 ? ~0ull : ((1ull << nv) - 1ull);
    SegT sagg;
    const SegT sex = warp_scan_segt(chunk_segt(Dm, Fm, Rm, Vm, (uint32_t)lane * CHUNK), sagg);
    const Seg st = seg_op(seg_op(a.seed, a.tinfo[t].excl), segt_to_seg(sex, a.base + (unsigned long long)t * WT));
    uint32_t c = st.col;
    unsigned long long fm = Fm;
    while (fm) {
      const int p = lsb64(fm);
      fm &= fm - 1ull;
      if ((Rm >> p) & 1ull) {
        mn = min(mn, c + 1u);
        mx = max(mx, c + 1u);
        c = 0;
      } else {
        c++;
      }
    }
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) {
    if (mn != 0xFFFFFFFFu) atomicMin(minmax, mn);
    atomicMax(minmax + 1, mx);
  }
}
}  // namespace parpa

// ---- type inference (reading R31) -------------------------------------------
// "threads identify the minimum numerical type being required to back their field value.  A subsequent
// parallel reduction over the minimum type yields the inferred type of a column", extended to
// temporal types as P:574 suggests.  Class of one field's DATA bytes: INT8 / INT16 / INT32 / INT64 by the
// range of an R14 integer, FLOAT64 for the R15 grammar (incl. integers beyond int64), TIMESTAMP for a valid
// R29 datetime, else STRING; empty / missing fields have no class.  The reduction is a bitwise OR of
// 1 << class (associative and commutative), resolved on the host (parpa_infer_types).
namespace parpa {
enum { TC_EMPTY = 0, TC_INT8 = 1, TC_INT16 = 2, TC_INT32 = 3, TC_INT64 = 4, TC_FLOAT64 = 5, TC_TIMESTAMP = 6,
       TC_STRING = 7 };

struct DataSrc {                       // the DATA bytes of the raw span [pos, end) (control bytes dropped)
  const KArgs *a;
  unsigned long long pos, end;
  bool all;                            // the span holds no control byte
  __device__ __forceinline__ bool next(uint8_t &c) {
    while (pos < end) {
      const unsigned long long p = pos++;
      if (all || ((dmask_of_chunk(*a, p >> 6) >> (p & 63)) & 1ull)) {
        c = a->in[p];
        return true;
      }
    }
    return false;
  }
};

template <class Src>
__device__ uint32_t field_class(const Src &src) {
  Src s = src;
  uint8_t c;
  if (!s.next(c)) return TC_EMPTY;
  bool neg = false, isint = true, over = false;
  if (c == '+' || c == '-') {
    neg = c == '-';
    if (!s.next(c)) isint = false;
  }
  unsigned long long acc = 0;
  const unsigned long long lim = neg ? 0x8000000000000000ull : 0x7FFFFFFFFFFFFFFFull;
  while (isint) {
    const unsigned d = (unsigned)c - '0';
    if (d > 9u) { isint = false; break; }
    if (!over) {
      if (acc > (lim - d) / 10ull) over = true;
      else acc = acc * 10ull + d;
    }
    if (!s.next(c)) break;
  }
  if (isint) {
    if (over) return TC_FLOAT64;                     // a digit string beyond int64: the float grammar
    const unsigned long long m = neg ? acc - (acc ? 1ull : 0ull) : acc;   // |v| - 1 for negatives
    return m <= 0x7Full ? TC_INT8 : m <= 0x7FFFull ? TC_INT16 : m <= 0x7FFFFFFFull ? TC_INT32 : TC_INT64;
  }
  long long v;
  Src f = src;
  if (conv_float64_fast(f, v) != 0) return TC_FLOAT64;   // 0 = not the R15 grammar
  Src t = src;
  if (conv_timestamp(t, v) == 1) return TC_TIMESTAMP;
  return TC_STRING;
}

__global__ void k_field_class(const KArgs a, const unsigned long long *off, const uint32_t *len,
                              unsigned long long rows, unsigned int *mask) {
  unsigned int m = 0;
  for (unsigned long long r = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; r < rows;
       r += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t L = len[r];
    if (L == MISSING_LEN_DEV || L == 0) continue;
    const unsigned long long p0 = off[r] - a.base;
    const DataSrc src{&a, p0, p0 + L, data_bytes_in(a, p0, L) == L};
    m |= 1u << field_class(src);
  }
  m = __reduce_or_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0 && m) atomicOr(mask, m);
}
}  // namespace parpa

// ---- skipping rows ("ignores a set of rows by performing an initial parallel
// pass over the input, pruning symbols of ignored rows (i.e., parallel stream compaction)") ----------
// A row is a raw line: the bytes up to and including a '\n' (rows ignore quoting: "some records may span
// multiple rows").  Per warp tile (32 lanes x 64 bytes): k_rows_count counts '\n'; a scan gives each
// tile its first row; k_rows_keep counts the bytes of rows not in the sorted skip list; a scan gives each
// tile its output offset; k_rows_write compacts them.  Both passes walk the skip list with a pointer
// that only moves forward (rows increase along a chunk).
namespace parpa {

__device__ __forceinline__ uint32_t nl_count_word(uint32_t w) {        // bytes equal to '\n' in a word
  const uint32_t t = w ^ 0x0A0A0A0Au;
  return (uint32_t)__popc(~(((t & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | t) & 0x80808080u);
}
__global__ void k_rows_count(const uint8_t *in, unsigned long long len, uint32_t ntiles, unsigned long long *lines) {
  const int lane = threadIdx.x & 31;
  for (uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntiles; t += (gridDim.x * blockDim.x) >> 5) {
    const unsigned long long cstart = (unsigned long long)t * WT + (unsigned long long)lane * CHUNK;
    const int nv = cstart >= len ? 0 : (int)min((unsigned long long)CHUNK, len - cstart);
    uint32_t v[16];
    load_chunk(in + cstart, nv, v);
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < 16; k++) c += nl_count_word(v[k]);     // zero-filled tails count nothing
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) lines[t] = c;
  }
}
// WRITE = false: kept bytes per tile into kept[t]; WRITE = true: the kept bytes to out[obase[t] + ...]
template <bool WRITE>
__global__ void k_rows_keep(const uint8_t *in, unsigned long long len, uint32_t ntiles, const unsigned long long *lbase,
                            const unsigned long long *skip, unsigned long long nskip, unsigned long long *kept,
                            const unsigned long long *obase, uint8_t *out) {
  const int lane = threadIdx.x & 31;
  for (uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntiles; t += (gridDim.x * blockDim.x) >> 5) {
    const unsigned long long cstart = (unsigned long long)t * WT + (unsigned long long)lane * CHUNK;
    const int nv = cstart >= len ? 0 : (int)min((unsigned long long)CHUNK, len - cstart);
    uint32_t v[16];
    load_chunk(in + cstart, nv, v);
    uint32_t nl = 0;
#pragma unroll
    for (int k = 0; k < 16; k++) nl += nl_count_word(v[k]);
    uint32_t inc = nl;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += o;
    }
    unsigned long long row = lbase[t] + (inc - nl);           // row of the chunk's first byte
    unsigned long long lo = 0, hi = nskip;                     // first skip entry >= row
    while (lo < hi) {
      const unsigned long long mid = (lo + hi) >> 1;
      if (skip[mid] < row) lo = mid + 1; else hi = mid;
    }
    bool drop = lo < nskip && skip[lo] == row;
    uint32_t keepmask[2] = {0u, 0u};
    for (int i = 0; i < nv; i++) {
      const uint32_t b = (v[i >> 2] >> (8 * (i & 3))) & 0xFFu;
      if (!drop) keepmask[i >> 5] |= 1u << (i & 31);
      if (b == 0x0Au) {                                        // the next byte starts the next row
        row++;
        while (lo < nskip && skip[lo] < row) lo++;
        drop = lo < nskip && skip[lo] == row;
      }
    }
    const uint32_t mine = (uint32_t)(__popc(keepmask[0]) + __popc(keepmask[1]));
    uint32_t kinc = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, kinc, d);
      if (lane >= d) kinc += o;
    }
    if (!WRITE) {
      if (lane == 31) kept[t] = kinc;
    } else {
      unsigned long long o = obase[t] + (kinc - mine);
      for (int i = 0; i < nv; i++)
        if ((keepmask[i >> 5] >> (i & 31)) & 1u) out[o++] = (uint8_t)((v[i >> 2] >> (8 * (i & 3))) & 0xFFu);
    }
  }
}

}  // namespace parpa
