// parpa_collab.cuh — block- and device-level collaborative conversion of long numeric fields (P:459-469:
// "If, during lookup, a thread detects that its string of symbols exceeds a certain threshold, it will defer
// generating that field value for the block- or device-level collaboration ... all threads of a thread-block
// collaborate on generating a field value.  Fields that exceed the on-chip memory available to a thread-block
// ... are addressed by the device-level collaboration.")
//
// Scope: int64 / float64 fields without inner control bytes (their DATA bytes are the raw span [fd, ld],
// reading R11) of at least COLLAB_MIN bytes.  Fields with inner control bytes keep the thread device tier,
// which re-simulates the DFA and stops at the first byte outside the number grammar (in the CSV / CLF
// dialects their DATA bytes always hold a '"' or '\', so it stops early).
//
// With the DATA bytes contiguous, every quantity the exact conversion needs is a position, found by
// min / max / count reductions over the bytes in two sweeps (no scan, no order between workers):
//   sweep A   count and first position of '.' and of 'e' / 'E'; any byte outside [0-9.eE+-] -> invalid
//   sweep C   (the exponent position now known) first / last nonzero significand digit, first nonzero
//             exponent digit, signs anywhere but at fd or right after the 'e' -> invalid
//   finish    grammar (R15) from the positions; int64: at most 19 significant digits, accumulated exactly;
//             float64: the first 800 significant digits gathered in parallel into a shared Decimal, the
//             "truncated nonzero" flag from the last nonzero digit, the decimal point from the positions,
//             the exponent from its first significant digits (the thread tier's saturation at 10^11), then the same
//             exact decimal -> binary rounding as the thread device tier (dec_float_bits).
// Block tier: one CTA runs the sweeps over one field with shared-memory reductions.  Device tier (fields of
// at least DEVICE_MIN bytes): every CTA of the (cooperative) grid sweeps a slice of every such field and
// reduces into the field's global accumulator; grid barriers separate the sweeps; CTA h % grid finishes
// field h.  The result equals the thread tier's conv_int64 / conv_float64_exact on the same bytes.
#pragma once

// (included by parpa_kernels.cuh after fetch_byte, inside namespace parpa; cooperative_groups.h is
// included at the top of parpa_kernels.cuh)

constexpr uint32_t COLLAB_MIN = 1024;          // raw numeric fields of >= 1 KB: block tier
constexpr uint32_t DEVICE_MIN = 256u * 1024u;  // raw numeric fields of >= 256 KB: device tier
constexpr int COLLAB_DIGITS = DEC_MAX + 2;     // bytes gathered from the first significant digit

__device__ __forceinline__ void collab_init(CollabAcc &c) {
  c.first_dot = c.first_e = c.p0 = c.pexp = NONE;
  c.plast = 0ull;
  c.n_dot = c.n_e = c.bad = c.pad = 0u;
}

// a collab queue item: output row (56 bits) | column (7 bits) << 56; the span comes from the column's
// offset / length, which the emitter wrote before it queued the field
__device__ __forceinline__ unsigned long long collab_item(unsigned long long row, uint32_t c) {
  return row | ((unsigned long long)c << 56);
}

// The emitter's router: true if the field went to a collaborative queue.  Capacity cannot run out: spans are
// disjoint, so a range of len bytes holds at most len / COLLAB_MIN such fields (+1 reaching into the halo).
__device__ __forceinline__ bool push_collab_slow(const KArgs &a, const ColDesc *cd, unsigned long long fd,
                                              unsigned long long ld, unsigned long long row, uint32_t c) {
  const unsigned long long L = ld + 1 - fd;
  if (!a.lq || (cd->type != T_INT64 && cd->type != T_FLOAT64)) return false;
  if (L >= DEVICE_MIN) {
    const uint32_t h = atomicAdd(&a.ctrl->n_huge, 1u);
    if (h < a.hq_cap) {
      collab_init(a.hacc[h]);
      a.hq[h] = collab_item(row, c);
      cd->valid[row] = 0;
      return true;
    }
  }
  const uint32_t i = atomicAdd(&a.ctrl->n_long, 1u);
  if (i >= a.lq_cap) return false;
  a.lq[i] = collab_item(row, c);
  cd->valid[row] = 0;
  return true;
}
// (the emission kernels keep only the length test inline: long fields are rare)
__device__ __forceinline__ bool push_collab(const KArgs &a, const ColDesc *cd, unsigned long long fd,
                                            unsigned long long ld, unsigned long long row, uint32_t c) {
#ifdef PARPA_NO_COLLAB_CODE
  return false;
#else
  return ld + 1 - fd >= COLLAB_MIN && push_collab_slow(a, cd, fd, ld, row, c);
#endif
}

__device__ __forceinline__ uint32_t ld_volatile_u32(const unsigned int *p) {
  return *reinterpret_cast<const volatile unsigned int *>(p);
}
__device__ __forceinline__ uint8_t collab_byte(const KArgs &a, unsigned long long p, bool &ok) {
  return fetch_byte(a, p, ok);
}

// ---- the two sweeps over bytes [fd + first, ld] with stride `step` (per-thread partial accumulators) ------
__device__ __forceinline__ void sweep_a(const KArgs &a, unsigned long long fd, unsigned long long ld,
                                        unsigned long long first, unsigned long long step, CollabAcc &t, bool &ok) {
  for (unsigned long long p = fd + first; p <= ld; p += step) {
    const uint8_t c = collab_byte(a, p, ok);
    if ((unsigned)(c - '0') <= 9u) continue;
    if (c == '.') { t.n_dot++; t.first_dot = min(t.first_dot, p); }
    else if ((c | 0x20) == 'e') { t.n_e++; t.first_e = min(t.first_e, p); }
    else if (c != '+' && c != '-') t.bad = 1u;
  }
}
__device__ __forceinline__ void sweep_c(const KArgs &a, unsigned long long fd, unsigned long long ld,
                                        unsigned long long first, unsigned long long step,
                                        unsigned long long first_e, CollabAcc &t, bool &ok) {
  const unsigned long long e_end = first_e == NONE ? ld + 1 : first_e;
  for (unsigned long long p = fd + first; p <= ld; p += step) {
    const uint8_t c = collab_byte(a, p, ok);
    if (c >= '1' && c <= '9') {
      if (p < e_end) { t.p0 = min(t.p0, p); t.plast = max(t.plast, p); }
      else t.pexp = min(t.pexp, p);
    } else if (c == '+' || c == '-') {
      if (p != fd && !(first_e != NONE && p == first_e + 1)) t.bad = 1u;
    }
  }
}

// shared / global reduction of a thread's partial accumulator
__device__ __forceinline__ void acc_reduce(CollabAcc *dst, const CollabAcc &t, bool phase_c) {
  if (!phase_c) {
    if (t.n_dot) { atomicAdd(&dst->n_dot, t.n_dot); atomicMin(&dst->first_dot, t.first_dot); }
    if (t.n_e) { atomicAdd(&dst->n_e, t.n_e); atomicMin(&dst->first_e, t.first_e); }
  } else {
    if (t.p0 != NONE) { atomicMin(&dst->p0, t.p0); atomicMax(&dst->plast, t.plast); }
    if (t.pexp != NONE) atomicMin(&dst->pexp, t.pexp);
  }
  if (t.bad) atomicOr(&dst->bad, 1u);
}

// the global accumulator after a grid barrier: L2 loads (this SM's L1 may hold the line from before)
__device__ __forceinline__ CollabAcc load_acc_cg(const CollabAcc *p) {
  CollabAcc c;
  c.first_dot = __ldcg(&p->first_dot); c.first_e = __ldcg(&p->first_e); c.p0 = __ldcg(&p->p0);
  c.plast = __ldcg(&p->plast); c.pexp = __ldcg(&p->pexp);
  c.n_dot = __ldcg(&p->n_dot); c.n_e = __ldcg(&p->n_e); c.bad = __ldcg(&p->bad); c.pad = 0u;
  return c;
}

struct CollabSmem {
  CollabAcc acc;
  Decimal dec;
  uint8_t dig[COLLAB_DIGITS];
  unsigned long long fd, ld, row;
  uint32_t col, ok_all;
};

// One CTA: the exact value of field [fd, ld] from its reductions `acc` (shared or global, final).  Writes the
// column's value / valid.  Every thread of the CTA calls it.
template <bool TS>
__device__ void collab_finish(const KArgs &a, const ColDesc *cd, CollabSmem &sm, const CollabAcc &acc,
                              unsigned long long fd, unsigned long long ld, unsigned long long row) {
  bool ok = true;
  // gather the bytes from the first nonzero significand digit (at most DEC_MAX digits + the '.')
  const unsigned long long p0 = acc.p0;
  if (p0 != NONE)
    for (int i = threadIdx.x; i < COLLAB_DIGITS; i += blockDim.x)
      sm.dig[i] = p0 + (unsigned)i <= ld ? collab_byte(a, p0 + (unsigned)i, ok) : (uint8_t)0;
  if (!ok) atomicAnd(&sm.ok_all, 0u);
  __syncthreads();
  if (threadIdx.x == 0) {
    bool okb = sm.ok_all != 0u;
    long long v = 0;
    int valid = 0;
    const uint8_t c0 = collab_byte(a, fd, okb);
    const bool sgn = c0 == '+' || c0 == '-', neg = c0 == '-';
    const unsigned long long ss = fd + (sgn ? 1u : 0u);
    const bool has_e = acc.n_e != 0u, has_dot = acc.n_dot != 0u;
    const unsigned long long se = has_e ? acc.first_e : ld + 1;
    bool gram = !acc.bad && acc.n_dot <= 1u && acc.n_e <= 1u && !(has_dot && has_e && acc.first_dot > acc.first_e) &&
                se > ss && (se - ss) - (has_dot ? 1u : 0u) >= 1u;
    unsigned long long es = 0;
    if (gram && has_e) {
      es = acc.first_e + 1;
      if (es <= ld) {
        const uint8_t ce = collab_byte(a, es, okb);
        if (ce == '+' || ce == '-') es++;
      }
      gram = es <= ld;                                            // at least one exponent digit
    }
    if (cd->type == T_INT64) {
      if (gram && !has_e && !has_dot) {
        if (p0 == NONE) {
          valid = 1;                                              // all zeros
        } else if (se - p0 <= 19u) {
          unsigned long long accv = 0;
          for (unsigned i = 0; i < (unsigned)(se - p0); i++) accv = accv * 10ull + (sm.dig[i] - '0');
          const unsigned long long lim = neg ? 0x8000000000000000ull : 0x7FFFFFFFFFFFFFFFull;
          if (accv <= lim) { v = neg ? (long long)(0ull - accv) : (long long)accv; valid = 1; }
        }
      }
    } else if (gram) {
      Decimal &d = sm.dec;
      d.nd = 0; d.dp = 0; d.neg = neg; d.trunc = false;
      if (p0 != NONE) {
        // digits from p0 up to the exponent (skipping the '.'), the first DEC_MAX of them stored
        unsigned long long q = p0;                                // position of the last stored digit
        for (int i = 0; i < COLLAB_DIGITS && p0 + (unsigned)i < se && d.nd < DEC_MAX; i++) {
          const uint8_t c = sm.dig[i];
          if (c == '.') continue;
          d.d[d.nd++] = (uint8_t)(c - '0');
          q = p0 + (unsigned)i;
        }
        if (acc.plast > q) d.trunc = true;                        // a nonzero digit beyond the stored ones
        long long dp = (has_dot && acc.first_dot < p0) ? -(long long)(p0 - acc.first_dot - 1)
                                                       : (long long)((has_dot ? acc.first_dot : se) - p0);
        if (has_e) {
          long long ex = 0;
          if (acc.pexp != NONE)
            for (unsigned long long p = acc.pexp; p <= ld && ex < EXP_SAT; p++) ex = ex * 10 + (collab_byte(a, p, okb) - '0');
          const bool eneg = collab_byte(a, acc.first_e + 1, okb) == '-';
          dp += eneg ? -ex : ex;
        }
        if (dp > 100000) dp = 100000;
        if (dp < -100000) dp = -100000;
        d.dp = (int)dp;
        dec_trim(d);
      }
      v = (long long)dec_float_bits(d);
      valid = 1;
    }
    if (!okb) { valid = 0; atomicOr(&a.ctrl->unsupported, 1u); }
    if (valid != 1) v = 0;
    reinterpret_cast<long long *>(cd->val)[row] = v;
    cd->valid[row] = (uint8_t)valid;
  }
  __syncthreads();
}

// Block tier: CTA b converts the long-queue items b, b + grid, ...  (every thread of the CTA calls it)
template <bool TS>
__device__ void collab_block_tier(const KArgs &a, const ColsK &colsk, CollabSmem &sm) {
  // (L2 loads throughout: in k_small the queue and the spans were written by other CTAs of this launch)
  const uint32_t n = a.lq ? min(ld_volatile_u32(&a.ctrl->n_long), a.lq_cap) : 0u;
  for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
    if (threadIdx.x == 0) {
      const unsigned long long it = __ldcg(a.lq + i);
      sm.row = it & ((1ull << 56) - 1ull);
      sm.col = (uint32_t)(it >> 56);
      const ColDesc *cd = colsk.c + sm.col;
      sm.fd = __ldcg(cd->off + sm.row);
      sm.ld = sm.fd + __ldcg(cd->len + sm.row) - 1;
      collab_init(sm.acc);
      sm.ok_all = 1u;
    }
    __syncthreads();
    const unsigned long long fd = sm.fd, ld = sm.ld;
    bool ok = true;
    CollabAcc t;
    collab_init(t);
    sweep_a(a, fd, ld, threadIdx.x, blockDim.x, t, ok);
    acc_reduce(&sm.acc, t, false);
    __syncthreads();
    const unsigned long long fe = sm.acc.n_e ? sm.acc.first_e : NONE;
    collab_init(t);
    sweep_c(a, fd, ld, threadIdx.x, blockDim.x, fe, t, ok);
    acc_reduce(&sm.acc, t, true);
    if (!ok) atomicAnd(&sm.ok_all, 0u);
    __syncthreads();
    const CollabAcc acc = sm.acc;
    collab_finish<TS>(a, colsk.c + sm.col, sm, acc, fd, ld, sm.row);
  }
}

// Device tier: every CTA sweeps its slice of every huge field; needs a cooperative launch (grid barriers).
// Only entered when n_huge > 0 (a value every CTA reads the same: it was final before this kernel started).
template <bool TS>
__device__ void collab_device_tier(const KArgs &a, const ColsK &colsk, CollabSmem &sm) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const uint32_t n = min(ld_volatile_u32(&a.ctrl->n_huge), a.hq_cap);
  const unsigned long long gt = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long gs = (unsigned long long)gridDim.x * blockDim.x;
  bool ok = true;
  for (int phase = 0; phase < 2; phase++) {
    for (uint32_t h = 0; h < n; h++) {
      const unsigned long long it = __ldcg(a.hq + h);
      const unsigned long long row = it & ((1ull << 56) - 1ull);
      const ColDesc *cd = colsk.c + (uint32_t)(it >> 56);
      const unsigned long long fd = __ldcg(cd->off + row), ld = fd + __ldcg(cd->len + row) - 1;
      if (threadIdx.x == 0) collab_init(sm.acc);
      __syncthreads();
      CollabAcc t;
      collab_init(t);
      if (phase == 0) {
        sweep_a(a, fd, ld, gt, gs, t, ok);
      } else {
        const CollabAcc g = load_acc_cg(&a.hacc[h]);
        sweep_c(a, fd, ld, gt, gs, g.n_e ? g.first_e : NONE, t, ok);
      }
      acc_reduce(&sm.acc, t, phase == 1);                         // CTA partial in shared memory,
      __syncthreads();
      if (threadIdx.x == 0) acc_reduce(&a.hacc[h], sm.acc, phase == 1);   // one global update per CTA
      __syncthreads();
    }
    __threadfence();
    grid.sync();
  }
  if (!ok) atomicOr(&a.ctrl->unsupported, 1u);
  for (uint32_t h = blockIdx.x; h < n; h += gridDim.x) {
    const unsigned long long it = __ldcg(a.hq + h);
    const unsigned long long row = it & ((1ull << 56) - 1ull);
    const ColDesc *cd = colsk.c + (uint32_t)(it >> 56);
    const unsigned long long fd = __ldcg(cd->off + row), ld = fd + __ldcg(cd->len + row) - 1;
    if (threadIdx.x == 0) sm.ok_all = 1u;
    __syncthreads();
    const CollabAcc acc = load_acc_cg(&a.hacc[h]);
    collab_finish<TS>(a, cd, sm, acc, fd, ld, row);
  }
}


// After the thread tier (which routes the long fields): a grid barrier, then the block tier and, if any field
// is huge, the device tier.  Entered by every thread of every CTA; the decision reads n_defer, which is final
// before the tiers start (every CTA sees the same value), so either all CTAs meet the barriers or none does.
template <bool TS>
__device__ __forceinline__ void collab_tiers(const KArgs &a, const ColsK &colsk, CollabSmem &sm) {
  if (!a.lq || ld_volatile_u32(&a.ctrl->n_defer) == 0u) return;
  __threadfence();
  cooperative_groups::this_grid().sync();          // the queues are complete
  collab_block_tier<TS>(a, colsk, sm);
  if (ld_volatile_u32(&a.ctrl->n_huge)) collab_device_tier<TS>(a, colsk, sm);
}
// (the last CTA out) the block- / device-tier counts into the stats
__device__ __forceinline__ void collab_stats(const KArgs &a) {
  a.stats->block_fields = a.lq ? min(ld_volatile_u32(&a.ctrl->n_long), a.lq_cap) : 0u;
  a.stats->device_fields = a.lq ? min(ld_volatile_u32(&a.ctrl->n_huge), a.hq_cap) : 0u;
}
