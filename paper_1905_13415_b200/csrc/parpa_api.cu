// parpa_api.cu — host side of libparpa: DFA compilation, workspace, kernel launches, the C ABI of
// include/parpa.h.  Build: see paper_1905_13415_b200/build.py (nvcc -gencode arch=compute_100a,
// code=sm_100a -lineinfo -O3 -shared).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "../../include/parpa.h"
#include "parpa_kernels.cuh"

using namespace parpa;

struct parpa_dfa {
  uint32_t S, G, start, inv;
  uint8_t gob[256];
  uint8_t trans[16][16], emit[16][16], eoi[16];
  uint8_t dmap[16];       // DFA state -> device state (0..7, 0xF = INV)
  DfaK k;                 // compiled tables (kernel parameter)
};

namespace {

constexpr size_t ALIGN = 256;
size_t align_up(size_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }

thread_local char t_last_error[256] = "";
int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return PARPA_OK;
  snprintf(t_last_error, sizeof(t_last_error), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  if (e == cudaErrorMemoryAllocation) return PARPA_ENOMEM;
  return PARPA_ECUDA;
}
#define CK(x)                                  \
  do {                                         \
    cudaError_t _e = (x);                      \
    if (_e != cudaSuccess) return cuda_status(_e); \
  } while (0)

// ---- per-device launch configuration -----------------------------------------------------
struct DevCfg {
  bool init = false;
  int sms = 0;
  int occ_pass1 = 0, occ_pass2 = 0, occ_emit = 0, occ_sparse = 0, occ_small = 0;
};
std::mutex g_mu;
DevCfg g_dev[64];

int dev_cfg(DevCfg **out) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return PARPA_ECUDA;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCfg &c = g_dev[dev];
  if (!c.init) {
    CK(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaFuncSetAttribute(k_pass1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PASS_SMEM));
    CK(cudaFuncSetAttribute(k_pass2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PASS_SMEM));
    CK(cudaFuncSetAttribute(k_emit<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)EMIT_SMEM));
    CK(cudaFuncSetAttribute(k_emit<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)EMIT_SMEM));
    CK(cudaFuncSetAttribute(k_emit<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)EMIT_SMEM));
    CK(cudaFuncSetAttribute(k_emit<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)EMIT_SMEM));
    CK(cudaFuncSetAttribute(k_emit_sparse<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SPARSE_SMEM));
    CK(cudaFuncSetAttribute(k_emit_sparse<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SPARSE_SMEM));
    CK(cudaFuncSetAttribute(k_emit_sparse<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SPARSE_SMEM));
    CK(cudaFuncSetAttribute(k_emit_sparse<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SPARSE_SMEM));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ_pass1, k_pass1, PASS_WARPS * 32, PASS_SMEM));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ_pass2, k_pass2, PASS_WARPS * 32, PASS_SMEM));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ_emit, k_emit<false, false>, EMIT_WARPS * 32, EMIT_SMEM));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ_sparse, k_emit_sparse<false, false>, SPARSE_WARPS * 32, SPARSE_SMEM));
    CK(cudaFuncSetAttribute(k_small<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMALL_SMEM));
    CK(cudaFuncSetAttribute(k_small<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMALL_SMEM));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ_small, k_small<false>, SMALL_WARPS * 32, SMALL_SMEM));
    if (getenv("PARPA_DEBUG")) {
      auto show = [](const char *n, const void *f) {
        cudaFuncAttributes fa;
        if (cudaFuncGetAttributes(&fa, f) == cudaSuccess)
          fprintf(stderr, "[parpa] %s: regs=%d maxThreads=%d static_smem=%zu local=%zu maxDynSmem=%d\n", n, fa.numRegs,
                  fa.maxThreadsPerBlock, fa.sharedSizeBytes, fa.localSizeBytes, fa.maxDynamicSharedSizeBytes);
      };
      show("k_pass1", (const void *)k_pass1);
      show("k_tau_scan", (const void *)k_tau_scan);
      show("k_pass2", (const void *)k_pass2);
      show("k_seg_scan", (const void *)k_seg_scan);
      show("k_emit", (const void *)k_emit<false, false>);
      show("k_emit<ts>", (const void *)k_emit<true, false>);
      fprintf(stderr, "[parpa] occ pass1=%d pass2=%d emit=%d sms=%d\n", c.occ_pass1, c.occ_pass2, c.occ_emit, c.sms);
    }
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    c.init = true;
  }
  *out = &c;
  return PARPA_OK;
}

// ---- profiling ----------------------------------------------------------------------------
struct ProfRec {
  const char *name;
  cudaEvent_t a, b;
};
bool g_prof = false;
thread_local std::vector<ProfRec> t_prof;
thread_local std::vector<ProfRec> t_prof_done;

struct Launch {
  cudaStream_t s;
  const char *name;
  cudaEvent_t a = nullptr, b = nullptr;
  Launch(cudaStream_t st, const char *n) : s(st), name(n) {
    if (g_prof) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, s);
    }
  }
  ~Launch() {
    if (g_prof) {
      cudaEventRecord(b, s);
      t_prof.push_back(ProfRec{name, a, b});
    }
  }
};
void prof_begin() {}
void prof_end() {
  if (!g_prof) return;
  t_prof_done.insert(t_prof_done.end(), t_prof.begin(), t_prof.end());
  t_prof.clear();
}
void prof_clear() {
  for (auto &r : t_prof) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto &r : t_prof_done) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  t_prof.clear();
  t_prof_done.clear();
}

// ---- workspace ------------------------------------------------------------------------------
struct Work {
  void *block = nullptr;
  unsigned long long *tau_desc = nullptr;
  uint32_t *bflag = nullptr;
  Ctrl *ctrl = nullptr;
  uint32_t *lex = nullptr, *wtau = nullptr, *tot_tau = nullptr;
  uint32_t *wpre = nullptr;
  uint4 *wseg = nullptr;
  Seg *bagg = nullptr, *bincl = nullptr, *tot_seg = nullptr;
  TileInfo *tinfo = nullptr;
  uint8_t *chunk_state = nullptr;
  unsigned long long *masks = nullptr;
  DeferItem *dq = nullptr;
  unsigned long long *lq = nullptr, *hq = nullptr;   // block- / device-tier queues (parpa_collab.cuh)
  CollabAcc *hacc = nullptr;
  Stats *stats = nullptr;
  uint8_t *aligned_in = nullptr;
  uint32_t ntiles = 0, nblk = 0, dq_cap = 0, lq_cap = 0, hq_cap = 0;
};

// One cudaMallocAsync block per call: the look-back descriptors and control words (zeroed), then the
// per-warp-tile and per-chunk arrays (written before they are read; no clearing needed).
int work_alloc(Work &w, uint64_t len, uint32_t /*C*/, bool need_aligned_copy, cudaStream_t s) {
  uint64_t nt64 = (len + WT - 1) / WT;
  if (nt64 > 0x07FFFFFFull) return PARPA_EUNSUPPORTED;       // chunk index must fit 32 bits
  w.ntiles = (uint32_t)nt64;
  w.nblk = (uint32_t)((nt64 + SEG_TILE - 1) / SEG_TILE);     // k_seg_scan's blocks (>= k_tau_scan's)
  size_t nt = std::max<size_t>(w.ntiles, 1), nb = std::max<size_t>(w.nblk, 1);
  w.dq_cap = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(4096, len / 512), 1u << 24);
  size_t o = 0;
  size_t o_tau = o; o = align_up(o + nb * 8);
  size_t o_flag = o; o = align_up(o + nb * 4);
  size_t o_ctrl = o; o = align_up(o + sizeof(Ctrl));
  size_t zero = o;
  size_t o_lex = o; o = align_up(o + nt * 32 * 4);
  size_t o_wtau = o; o = align_up(o + nt * 4);
  size_t o_went = o; o = align_up(o + nt * 4);
  size_t o_wseg = o; o = align_up(o + nt * 16);
  size_t o_bagg = o; o = align_up(o + nb * sizeof(Seg));
  size_t o_binc = o; o = align_up(o + nb * sizeof(Seg));
  size_t o_tot = o; o = align_up(o + sizeof(Seg) + 16);
  size_t o_tinfo = o; o = align_up(o + nt * sizeof(TileInfo));
  size_t o_cs = o; o = align_up(o + nt * 32);
  size_t o_mk = o; o = align_up(o + nt * 96 * 8);
  size_t o_dq = o; o = align_up(o + (size_t)w.dq_cap * sizeof(DeferItem));
  // spans are disjoint: at most len / COLLAB_MIN fields of >= COLLAB_MIN bytes (+ one reaching into a halo)
  w.lq_cap = (uint32_t)std::min<uint64_t>(len / COLLAB_MIN + 4, 0xFFFFFFF0ull);
  w.hq_cap = (uint32_t)(len / DEVICE_MIN + 4);
  size_t o_lq = o; o = align_up(o + (size_t)w.lq_cap * 8);
  size_t o_hq = o; o = align_up(o + (size_t)w.hq_cap * 8);
  size_t o_ha = o; o = align_up(o + (size_t)w.hq_cap * sizeof(CollabAcc));
  size_t o_st = o; o = align_up(o + sizeof(Stats));
  size_t o_in = o; if (need_aligned_copy) o = align_up(o + len);
  CK(cudaMallocAsync(&w.block, o, s));
  uint8_t *b = (uint8_t *)w.block;
  w.tau_desc = (unsigned long long *)(b + o_tau);
  w.bflag = (uint32_t *)(b + o_flag);
  w.ctrl = (Ctrl *)(b + o_ctrl);
  w.lex = (uint32_t *)(b + o_lex);
  w.wtau = (uint32_t *)(b + o_wtau);
  w.wpre = (uint32_t *)(b + o_went);
  w.wseg = (uint4 *)(b + o_wseg);
  w.bagg = (Seg *)(b + o_bagg);
  w.bincl = (Seg *)(b + o_binc);
  w.tot_seg = (Seg *)(b + o_tot);
  w.tot_tau = (uint32_t *)(b + o_tot + sizeof(Seg));
  w.tinfo = (TileInfo *)(b + o_tinfo);
  w.chunk_state = b + o_cs;
  w.masks = (unsigned long long *)(b + o_mk);
  w.dq = (DeferItem *)(b + o_dq);
  w.lq = (unsigned long long *)(b + o_lq);
  w.hq = (unsigned long long *)(b + o_hq);
  w.hacc = (CollabAcc *)(b + o_ha);
  w.stats = (Stats *)(b + o_st);
  w.aligned_in = need_aligned_copy ? b + o_in : nullptr;
  CK(cudaMemsetAsync(w.block, 0, zero, s));
  return PARPA_OK;
}
void work_free(Work &w, cudaStream_t s) {
  if (w.block) cudaFreeAsync(w.block, s);
  w.block = nullptr;
}

Seg seg_identity() { return Seg{0ull, 0ull, NONE, NONE, 0u, 0u}; }

Seg counts_to_seg(const parpa_counts &c) {
  return Seg{c.records, c.fields, c.open_first, c.open_last, c.column, c.flags};
}
parpa_counts seg_to_counts(const Seg &s, uint64_t first_inv) {
  parpa_counts c;
  c.records = s.recs; c.fields = s.nflds; c.open_first = s.fd; c.open_last = s.ld;
  c.column = s.col; c.flags = s.flags; c.first_invalid = first_inv;
  return c;
}

void make_args(KArgs &a, const Work &w, const uint8_t *in, uint64_t len) {
  memset(&a, 0, sizeof(a));
  a.in = in;
  a.len = len;
  a.ntiles = w.ntiles;
  a.seed = seg_identity();
  a.lex = w.lex;
  a.wtau = w.wtau;
  a.wpre = w.wpre;
  a.wseg = w.wseg;
  a.tau_desc = w.tau_desc;
  a.bflag = w.bflag;
  a.bagg = w.bagg;
  a.bincl = w.bincl;
  a.tot_tau = w.tot_tau;
  a.tot_seg = w.tot_seg;
  a.tinfo = w.tinfo;
  a.chunk_state = w.chunk_state;
  a.masks = w.masks;
  a.ctrl = w.ctrl;
  a.dq = w.dq;
  a.dq_cap = w.dq_cap;
  static const bool collab = !(getenv("PARPA_NO_COLLAB") && getenv("PARPA_NO_COLLAB")[0] == '1');   // A/B, tests
  a.lq = collab ? w.lq : nullptr;
  a.hq = w.hq;
  a.hacc = w.hacc;
  a.lq_cap = w.lq_cap;
  a.hq_cap = w.hq_cap;
  const char *ek = getenv("PARPA_EMIT_K");                   // A/B and tests: force the emission unit
  a.emit_k = ek ? (uint32_t)atoi(ek) : 0u;
  a.is_last = 1;
  a.cap = 0;
  a.left_state = 0xFFu;                                     // no halo state known
}

int prepare_input(Work &w, const uint8_t *&in, uint64_t len, cudaStream_t s) {
  if (w.aligned_in) {
    CK(cudaMemcpyAsync(w.aligned_in, in, len, cudaMemcpyDeviceToDevice, s));
    in = w.aligned_in;
  }
  return PARPA_OK;
}
bool misaligned(const void *p) { return ((uintptr_t)p & 15u) != 0; }

int set_columns(const parpa_schema *sch, const parpa_column *cols, uint32_t C, ColsK &ck) {
  memset(&ck, 0, sizeof(ck));
  if (C > MAX_COLS) return PARPA_EUNSUPPORTED;
  for (uint32_t c = 0; c < C; c++) {
    ColDesc &d = ck.c[c];
    d.off = (unsigned long long *)cols[c].offset;
    d.len = cols[c].length;
    d.val = cols[c].value;
    d.valid = cols[c].valid;
    d.type = sch->types ? sch->types[c] : PARPA_SPAN;
    d.has_def = sch->has_default ? sch->has_default[c] : 0;
    d.def_bits = sch->default_bits ? sch->default_bits[c] : 0;
    if (d.type > PARPA_TIMESTAMP) return PARPA_EINVAL;
    if (!d.off && !d.len && !d.val && !d.valid) {            // skipped column: counted, not written
      d.type = T_SKIP;
      continue;
    }
    if (!d.off || !d.len) return PARPA_EINVAL;
    if (d.type != PARPA_SPAN && (!d.val || !d.valid)) return PARPA_EINVAL;
  }
  return PARPA_OK;
}

// Launch with programmatic stream serialisation (PDL, see PdlTrigger): the kernel may start its prologue
// while its stream predecessor drains.  PARPA_NO_PDL=1 in the environment launches normally (A/B).
static bool pdl_enabled() {
  static const bool on = !(getenv("PARPA_NO_PDL") && getenv("PARPA_NO_PDL")[0] == '1');
  return on;
}
template <typename... P, typename... A>
cudaError_t launch_k(void (*k)(P...), unsigned grid, unsigned block, size_t smem, cudaStream_t s, bool pdl,
                     A &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl && pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}
// the same with the cooperative attribute (co-resident CTAs: grid barriers are allowed)
template <typename... P, typename... A>
cudaError_t launch_coop(void (*k)(P...), unsigned grid, unsigned block, size_t smem, cudaStream_t s, bool pdl,
                        A &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl && pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

// The DFA as the LUT-building kernels see it: the prebuilt image only on the device it lives on.
const DfaK &dfa_for_device(const DfaK &k, DfaK &tmp) {
  int dev = -1;
  if (!k.img || (cudaGetDevice(&dev) == cudaSuccess && dev == k.img_dev)) return k;
  tmp = k;
  tmp.img = nullptr;
  return tmp;
}

int grid_for(int occ, int sms, uint32_t ntiles, int warps_per_cta) {
  long long g = (long long)std::max(occ, 1) * sms;
  long long need = ((long long)ntiles + warps_per_cta - 1) / warps_per_cta;
  return (int)std::max<long long>(1, std::min<long long>(g, need));
}

// S1-S3: pass 1 and the τ scan (unseeded); S4-S5: pass 2 (seeded by a.seed_dev) and the
// record/column scan (unseeded; a.seed is applied by k_emit / k_finalize).
int launch_half2(const KArgs &a, const DfaK &k, cudaStream_t s, uint32_t *launches);
int launch_passes(int mode, const KArgs &a, const DfaK &k0, cudaStream_t s, uint32_t *launches) {
  if (a.ntiles == 0) return PARPA_OK;
  DfaK tmp;
  const DfaK &k = dfa_for_device(k0, tmp);
  DevCfg *dc;
  int rc = dev_cfg(&dc);
  if (rc) return rc;
  const uint32_t nblk = (a.ntiles + SCAN_TILE - 1) / SCAN_TILE;
  {
    Launch L(s, "k_pass1");
    CK(launch_k(k_pass1, grid_for(dc->occ_pass1, dc->sms, a.ntiles, PASS_WARPS), PASS_WARPS * 32, PASS_SMEM, s, false, a, k));
  }
  CK(cudaGetLastError());
  {
    Launch L(s, "k_tau_scan");
    CK(launch_k(k_tau_scan, nblk, SCAN_THREADS, 0, s, true, a));
  }
  CK(cudaGetLastError());
  if (launches) *launches += 2;
  return mode == MODE_TAU ? PARPA_OK : launch_half2(a, k, s, launches);
}

int launch_half2(const KArgs &a, const DfaK &k0, cudaStream_t s, uint32_t *launches) {
  if (a.ntiles == 0) return PARPA_OK;
  DfaK tmp;
  const DfaK &k = dfa_for_device(k0, tmp);
  DevCfg *dc;
  int rc = dev_cfg(&dc);
  if (rc) return rc;
  const uint32_t nblk = (a.ntiles + SEG_TILE - 1) / SEG_TILE;
  {
    Launch L(s, "k_pass2");
    CK(launch_k(k_pass2, grid_for(dc->occ_pass2, dc->sms, a.ntiles, PASS_WARPS), PASS_WARPS * 32, PASS_SMEM, s, true, a, k));
  }
  CK(cudaGetLastError());
  {
    Launch L(s, "k_seg_scan");
    CK(launch_k(k_seg_scan, nblk, SCAN_THREADS, 0, s, true, a));
  }
  CK(cudaGetLastError());
  if (launches) *launches += 2;
  return PARPA_OK;
}

bool has_timestamps(const KArgs &a, const ColsK &ck) {
  for (uint32_t c = 0; c < a.C && c < (uint32_t)MAX_COLS; c++)
    if (ck.c[c].type == T_TIMESTAMP) return true;
  return false;
}

int launch_emit(const KArgs &a, const DfaK &k, const ColsK &ck, cudaStream_t s, uint32_t *launches) {
  if (a.ntiles == 0) return PARPA_OK;
  DevCfg *dc;
  int rc = dev_cfg(&dc);
  if (rc) return rc;
  {
    Launch L(s, "k_emit");
    const int g = grid_for(dc->occ_emit, dc->sms, a.ntiles, EMIT_WARPS);
    const bool ts = has_timestamps(a, ck), sk = a.nskip > 0;
    if (ts && sk) CK(launch_k(k_emit<true, true>, g, EMIT_WARPS * 32, EMIT_SMEM, s, true, a, ck));
    else if (ts) CK(launch_k(k_emit<true, false>, g, EMIT_WARPS * 32, EMIT_SMEM, s, true, a, ck));
    else if (sk) CK(launch_k(k_emit<false, true>, g, EMIT_WARPS * 32, EMIT_SMEM, s, true, a, ck));
    else CK(launch_k(k_emit<false, false>, g, EMIT_WARPS * 32, EMIT_SMEM, s, true, a, ck));
  }
  CK(cudaGetLastError());
  {
    // sparse ranges (>= 32 bytes per field): super tiles; k_emit above returned at once for them, this one
    // returns at once for the others (both read the range's field count on the device)
    Launch L(s, "k_emit_sparse");
    const int g = grid_for(dc->occ_sparse, dc->sms, (a.ntiles + SPARSE_K - 1) / SPARSE_K, SPARSE_WARPS);
    const bool ts = has_timestamps(a, ck), sk = a.nskip > 0;
#ifdef PARPA_SPARSE_NOPDL
    const bool pdl = false;
#else
    const bool pdl = true;
#endif
    if (ts && sk) CK(launch_k(k_emit_sparse<true, true>, g, SPARSE_WARPS * 32, SPARSE_SMEM, s, pdl, a, ck));
    else if (ts) CK(launch_k(k_emit_sparse<true, false>, g, SPARSE_WARPS * 32, SPARSE_SMEM, s, pdl, a, ck));
    else if (sk) CK(launch_k(k_emit_sparse<false, true>, g, SPARSE_WARPS * 32, SPARSE_SMEM, s, pdl, a, ck));
    else CK(launch_k(k_emit_sparse<false, false>, g, SPARSE_WARPS * 32, SPARSE_SMEM, s, pdl, a, ck));
  }
  CK(cudaGetLastError());
  if (launches) *launches += 2;
  return PARPA_OK;
}

// Small inputs (<= SMALL_MAX_TILES warp tiles): the whole parse as one cooperative launch (k_small).
// PARPA_SMALL=0 in the environment forces the multi-kernel path (A/B, tests).
static bool small_enabled() {
  static const bool on = !(getenv("PARPA_SMALL") && getenv("PARPA_SMALL")[0] == '0');
  return on;
}
bool use_small(const KArgs &a) {
  if (!small_enabled() || a.ntiles == 0 || a.ntiles > SMALL_MAX_TILES) return false;
  DevCfg *dc;
  if (dev_cfg(&dc)) return false;
  return dc->occ_small >= 1;
}
int launch_small(const KArgs &a, const DfaK &k0, const ColsK &ck, cudaStream_t s, uint32_t *launches) {
  DfaK tmp;
  const DfaK &k = dfa_for_device(k0, tmp);
  DevCfg *dc;
  int rc0 = dev_cfg(&dc);
  if (rc0) return rc0;
  // one warp per tile in the passes, SMALL_NP warps per tile in the emission phase
  const unsigned grid = (unsigned)std::min<long long>((long long)dc->occ_small * dc->sms,
                                                       ((long long)a.ntiles * SMALL_NP + SMALL_WARPS - 1) / SMALL_WARPS);
  void *args[] = {(void *)&a, (void *)&k, (void *)&ck};
  static const bool sprof = getenv("PARPA_SPROF") && getenv("PARPA_SPROF")[0] == '1';
  KArgs ap = a;
  if (sprof) {
    CK(cudaMallocAsync(&ap.prof, 16 * 8, s));
    CK(cudaMemsetAsync(ap.prof, 0, 16 * 8, s));
    args[0] = (void *)&ap;
  }
  {
    Launch L(s, "k_small");
    if (has_timestamps(a, ck))
      CK(cudaLaunchCooperativeKernel((const void *)k_small<true>, dim3(grid), dim3(SMALL_WARPS * 32), args, SMALL_SMEM, s));
    else
      CK(cudaLaunchCooperativeKernel((const void *)k_small<false>, dim3(grid), dim3(SMALL_WARPS * 32), args, SMALL_SMEM, s));
  }
  CK(cudaGetLastError());
  if (sprof) {
    unsigned long long h[16];
    CK(cudaMemcpyAsync(h, ap.prof, 16 * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    fprintf(stderr, "[parpa sprof] us: lut %.1f pass1 %.1f sync %.1f tauscan %.1f pass2 %.1f sync %.1f segscan %.1f emit %.1f "
            "sync %.1f fin %.1f sync %.1f deferred+sync %.1f total %.1f\n", (h[1] - h[0]) / 1e3, (h[2] - h[1]) / 1e3,
            (h[3] - h[2]) / 1e3, (h[4] - h[3]) / 1e3, (h[5] - h[4]) / 1e3, (h[6] - h[5]) / 1e3, (h[7] - h[6]) / 1e3,
            (h[8] - h[7]) / 1e3, (h[9] - h[8]) / 1e3, (h[10] - h[9]) / 1e3, (h[11] - h[10]) / 1e3, (h[12] - h[11]) / 1e3,
            (h[12] - h[0]) / 1e3);
    cudaFreeAsync(ap.prof, s);
  }
  if (launches) (*launches)++;
  return PARPA_OK;
}

int launch_tail(const KArgs &a, const DfaK &k, const ColsK &ck, cudaStream_t s, uint32_t *launches) {
  DevCfg *dc;
  int rc = dev_cfg(&dc);
  if (rc) return rc;
  {
    Launch L(s, "k_finalize");
    CK(launch_k(k_finalize, 1, 32, 0, s, a.ntiles != 0, a, k, ck));
  }
  CK(cudaGetLastError());
  {
    Launch L(s, "k_deferred");
    // cooperative: the device tier of parpa_collab.cuh separates its sweeps by grid barriers
    if (has_timestamps(a, ck)) CK(launch_coop(k_deferred<true>, dc->sms * 2, 128, 0, s, true, a, k, ck));
    else CK(launch_coop(k_deferred<false>, dc->sms * 2, 128, 0, s, true, a, k, ck));
  }
  CK(cudaGetLastError());
  if (launches) *launches += 2;
  return PARPA_OK;
}

void host_tau_dfa(const parpa_dfa *d, uint32_t nib, parpa_tau *out) {
  for (int i = 0; i < 16; i++) out->tau[i] = 0xFF;
  for (uint32_t i = 0; i < d->S; i++) {
    uint32_t di = d->dmap[i];
    uint32_t r = di == INV_DEV ? INV_DEV : (nib >> (4 * di)) & 0xF;
    out->tau[i] = d->k.hmap[r];
  }
}

// ---- exact states where device classes merged DFA states (see DfaK) ----------------------------------
uint32_t host_class_step(const parpa_dfa *d, uint32_t c, uint8_t b) {
  return c == INV_DEV ? INV_DEV : d->dmap[d->trans[d->gob[b]][d->k.hmap[c]]];
}
uint32_t host_exact_after(const parpa_dfa *d, uint32_t cls_before_last, uint8_t last) {
  return cls_before_last == INV_DEV ? d->inv : d->trans[d->gob[last]][d->k.hmap[cls_before_last]];
}
// The range's transition vector in DFA numbering with exact entries: the class vector over all but the
// last byte (tile prefix ∘ lane prefix, then the last chunk's bytes on the host), then the last byte's
// exact row.  Needs lex / wpre of a completed pass 1 + τ scan.
int host_tau_exact(const parpa_dfa *d, const Work &w, const uint8_t *in, uint64_t len, uint32_t tot_nib,
                   cudaStream_t s, parpa_tau *out) {
  if (!d->k.merged || len == 0) { host_tau_dfa(d, tot_nib, out); return PARPA_OK; }
  const uint64_t kc = (len - 1) / CHUNK, t = kc / 32;
  uint32_t lex = 0, wpre = 0;
  uint8_t bytes[CHUNK];
  const uint64_t nb = len - kc * CHUNK;
  CK(cudaMemcpyAsync(&lex, w.lex + kc, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&wpre, w.wpre + t, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(bytes, in + kc * CHUNK, nb, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int i = 0; i < 16; i++) out->tau[i] = 0xFF;
  for (uint32_t st = 0; st < d->S; st++) {
    uint32_t c = nib_at(lex, nib_at(wpre, d->dmap[st]));
    for (uint64_t q = 0; q + 1 < nb; q++) c = host_class_step(d, c, bytes[q]);
    out->tau[st] = (uint8_t)host_exact_after(d, c, bytes[nb - 1]);
  }
  return PARPA_OK;
}
// The exact DFA state after a scanned range (for its end-of-input action on the host): the class
// before the last byte from the last chunk's entry state, then the last byte's exact row.
int host_final_exact(const parpa_dfa *d, const Work &w, const uint8_t *in, uint64_t len, uint32_t fin_class,
                     uint32_t seed_exact, cudaStream_t s, uint32_t &exact) {
  if (len == 0) { exact = seed_exact; return PARPA_OK; }
  if (!d->k.merged) { exact = d->k.hmap[fin_class]; return PARPA_OK; }
  const uint64_t kc = (len - 1) / CHUNK, nb = len - kc * CHUNK;
  uint8_t st = 0, bytes[CHUNK];
  CK(cudaMemcpyAsync(&st, w.chunk_state + kc, 1, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(bytes, in + kc * CHUNK, nb, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  uint32_t c = st & 0xFu;
  for (uint64_t q = 0; q + 1 < nb; q++) c = host_class_step(d, c, bytes[q]);
  exact = host_exact_after(d, c, bytes[nb - 1]);
  return PARPA_OK;
}

}  // namespace

struct parpa_plan {
  const parpa_dfa *dfa;
  const uint8_t *in;
  uint64_t len;
  Work w;
  KArgs a;
  uint64_t records;
  cudaStream_t s;
};

// Allocator of result-owned buffers (parpa_set_allocator; default stream-ordered cudaMallocAsync / cudaFreeAsync).
struct Allocator {
  parpa_alloc_fn alloc = nullptr;
  parpa_free_fn free = nullptr;
  void *ctx = nullptr;
};
static std::mutex g_alloc_mu;
static Allocator g_alloc;
static Allocator current_allocator() {
  std::lock_guard<std::mutex> g(g_alloc_mu);
  return g_alloc;
}

struct parpa_result {
  uint32_t C;
  std::vector<parpa_column> cols;
  std::vector<void *> allocs;
  Allocator al;                       // the allocator the buffers came from (freed with its free)
  cudaStream_t s = nullptr;
  parpa_stats stats;
};

// A plan may be counted / emitted more than once: each call first clears the control words and look-back
// flags its kernels accumulate into (a repeated call used to run on stale tickets and flags).
static int reset_scan_state(parpa_plan *p) {
  Ctrl *c = p->w.ctrl;
  CK(cudaMemsetAsync(&c->ticket2, 0, sizeof(c->ticket2), p->s));
  CK(cudaMemsetAsync(&c->inv_neg, 0, sizeof(c->inv_neg), p->s));
  if (p->w.nblk) CK(cudaMemsetAsync(p->w.bflag, 0, (size_t)p->w.nblk * 4, p->s));
  return PARPA_OK;
}
static int reset_emit_state(parpa_plan *p, cudaStream_t s) {
  Ctrl *c = p->w.ctrl;
  CK(cudaMemsetAsync(&c->n_defer, 0, offsetof(Ctrl, inv_neg) - offsetof(Ctrl, n_defer), s));
  CK(cudaMemsetAsync(&c->n_missing, 0, sizeof(Ctrl) - offsetof(Ctrl, n_missing), s));
  return PARPA_OK;
}


extern "C" {

const char *parpa_last_error(void) { return t_last_error; }
const char *parpa_version(void) { return "parpa 0.1 (sm_100a, dense LUT path)"; }
uint32_t parpa_chunk_bytes(void) { return CHUNK; }
uint32_t parpa_tile_bytes(void) { return WT; }

const char *parpa_status_string(int st) {
  switch (st) {
  case PARPA_OK: return "ok";
  case PARPA_EINVAL: return "invalid argument";
  case PARPA_ENOMEM: return "out of memory";
  case PARPA_ECUDA: return "CUDA error";
  case PARPA_EFORMAT: return "format error (invalid state reached or non-accepting end state)";
  case PARPA_ECOLUMNS: return "record with a number of fields != number of columns (strict)";
  case PARPA_EUNSUPPORTED: return "unsupported (DFA too large, field too long, or device-tier overflow)";
  case PARPA_ENEEDMORE: return "output capacity too small";
  default: return "unknown status";
  }
}

// The shared-memory LUT images of a DFA (the layouts build_lut / build_lut_step_dp write), in device memory of
// the current device: the pass kernels and k_small copy them instead of building entry by entry.
static bool have_device() {                              // probed once (no device: no runtime re-probing per DFA)
  static const bool yes = [] {
    int n = 0;
    const bool ok = cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
    cudaGetLastError();
    return ok;
  }();
  return yes;
}
static void make_lut_image(parpa_dfa *d) {
  int dev = -1;
  if (!have_device() || cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  const bool ns4 = d->k.nlive <= 4;
  std::vector<uint32_t> h((LUT_BYTES + 256 * STEP_ROW_DP) / 4);
  for (int b = 0; b < 256; b++)
    for (int half = 0; half < 2; half++)
      for (int slot = 0; slot < 16; slot++) {
        const size_t o = ((size_t)b * 256 + half * 128 + slot * 8) / 4;
        h[o] = half ? d->k.lut[b][2] : d->k.lut[b][0];
        h[o + 1] = half ? (ns4 ? d->k.lut[b][2] : d->k.lut[b][3]) : (ns4 ? d->k.lut[b][0] : d->k.lut[b][1]);
      }
  for (int b = 0; b < 256; b++)
    for (int slot = 0; slot < 16; slot++) {
      const size_t o = (LUT_BYTES + (size_t)b * STEP_ROW_DP + slot * 8) / 4;
      h[o] = d->k.lut[b][2];
      h[o + 1] = ns4 ? d->k.lut[b][2] : d->k.lut[b][3];
    }
  void *p = nullptr;
  if (cudaMalloc(&p, h.size() * 4) != cudaSuccess) { cudaGetLastError(); return; }
  if (cudaMemcpy(p, h.data(), h.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(p);
    return;
  }
  d->k.img = (const uint4 *)p;
  d->k.img_dev = dev;
}

int parpa_create_dfa(uint32_t S, uint32_t start, uint32_t inv, uint32_t G, const uint8_t *gob,
                     const uint8_t *trans, const uint8_t *emit, const uint8_t *eoi, parpa_dfa **out) {
  if (!out || !gob || !trans || !emit || !eoi) return PARPA_EINVAL;
  if (S < 2 || S > 16 || G < 1 || G > 16 || start >= S || inv >= S || start == inv) return PARPA_EINVAL;
  for (int b = 0; b < 256; b++)
    if (gob[b] >= G) return PARPA_EINVAL;
  for (uint32_t g = 0; g < G; g++)
    for (uint32_t s = 0; s < S; s++) {
      if (trans[g * S + s] >= S || emit[g * S + s] > PARPA_RECORD) return PARPA_EINVAL;
    }
  for (uint32_t g = 0; g < G; g++)
    if (trans[g * S + inv] != inv || emit[g * S + inv] != PARPA_CTRL) return PARPA_EINVAL;
  for (uint32_t s = 0; s < S; s++)
    if (eoi[s] > PARPA_EOI_ERROR) return PARPA_EINVAL;
  parpa_dfa *d = new (std::nothrow) parpa_dfa;
  if (!d) return PARPA_ENOMEM;
  memset(d, 0, sizeof(*d));
  d->S = S; d->G = G; d->start = start; d->inv = inv;
  memcpy(d->gob, gob, 256);
  for (uint32_t g = 0; g < G; g++)
    for (uint32_t s = 0; s < S; s++) {
      d->trans[g][s] = trans[g * S + s];
      d->emit[g][s] = emit[g * S + s];
    }
  memcpy(d->eoi, eoi, S);
  // device states = classes of live states with identical transition and emission rows (in order of
  // their first member); INV -> 0xF
  uint32_t rep[16], k = 0;
  for (uint32_t s = 0; s < S; s++) {
    if (s == inv) { d->dmap[s] = INV_DEV; continue; }
    uint32_t j = 0;
    for (; j < k; j++) {
      bool same = true;
      for (uint32_t g = 0; g < G && same; g++)
        same = d->trans[g][s] == d->trans[g][rep[j]] && d->emit[g][s] == d->emit[g][rep[j]];
      if (same) break;
    }
    if (j == k) rep[k++] = s;
    d->dmap[s] = (uint8_t)j;
  }
  if (k > 8) { delete d; return PARPA_EUNSUPPORTED; }
  d->k.nlive = k;
  d->k.merged = k < S - 1 ? 1u : 0u;
  d->k.inv_state = inv;
  memcpy(d->k.gob, gob, 256);
  for (uint32_t s = 0; s < S; s++) d->k.eoi_state[s] = eoi[s];
  for (int j = 0; j < 16; j++) { d->k.hmap[j] = (uint8_t)inv; d->k.eoi[j] = eoi[inv]; }
  for (uint32_t j = 0; j < k; j++) { d->k.hmap[j] = (uint8_t)rep[j]; d->k.eoi[j] = eoi[rep[j]]; }
  for (uint32_t j = 0; j < 16; j++)
    for (uint32_t g = 0; g < 16; g++)
      d->k.next_exact[j][g] = (uint8_t)(j < k && g < G ? d->trans[g][rep[j]] : inv);
  for (int b = 0; b < 256; b++) {
    uint32_t g = gob[b];
    uint32_t sel = 0;
    uint8_t step[8];
    for (uint32_t j = 0; j < 8; j++) {
      uint32_t nd = INV_DEV, kind = PARPA_CTRL;
      if (j < k) {
        uint32_t s = rep[j];
        nd = d->dmap[d->trans[g][s]];
        kind = d->emit[g][s];
      }
      sel |= nd << (4 * j);
      const uint32_t fl = (kind == PARPA_DATA ? KC_DATA : kind == PARPA_FIELD ? KC_FIELD
                           : kind == PARPA_RECORD ? KC_RECORD : KC_CTRL) << 4;
      step[j] = (uint8_t)(0x80u | nd | fl);
    }
    d->k.lut[b][0] = sel & 0xFFFFu;
    d->k.lut[b][1] = sel >> 16;
    d->k.lut[b][2] = step[0] | (step[1] << 8) | (step[2] << 16) | ((uint32_t)step[3] << 24);
    d->k.lut[b][3] = step[4] | (step[5] << 8) | (step[6] << 16) | ((uint32_t)step[7] << 24);
  }
  d->k.img = nullptr;
  d->k.img_dev = -1;
  make_lut_image(d);                                     // (no device: the kernels build the LUTs themselves)
  *out = d;
  return PARPA_OK;
}

void parpa_destroy_dfa(parpa_dfa *d) {
  if (!d) return;
  if (d->k.img) cudaFree((void *)d->k.img);
  delete d;
}

int parpa_set_profiling(int enable) {
  prof_clear();
  g_prof = enable != 0;
  return PARPA_OK;
}

int parpa_last_kernel_times(const char **names, float *ms, int cap) {
  int n = 0;
  for (auto &r : t_prof_done) {
    if (n >= cap) break;
    float t = 0;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) t = -1;
    if (names) names[n] = r.name;
    if (ms) ms[n] = t;
    n++;
  }
  return n;
}

// ---- plan: scan pass -------------------------------------------------------------------------
static int plan_scan(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, uint32_t seed_state,
                     const Seg &seed, uint64_t base, uint32_t C, cudaStream_t s, parpa_plan *p) {
  p->dfa = dfa;
  p->len = len;
  p->s = s;
  int rc = work_alloc(p->w, len, C, len && misaligned(d_bytes), s);
  if (rc) return rc;
  const uint8_t *in = d_bytes;
  if ((rc = prepare_input(p->w, in, len, s))) return rc;
  p->in = in;
  make_args(p->a, p->w, in, len);
  p->a.seed_dev = dfa->dmap[seed_state];
  p->a.seed_exact = seed_state;
  p->a.seed = seed;
  p->a.base = base;
  p->a.row_base = seed.recs;
  return launch_passes(MODE_COUNT, p->a, dfa->k, s, nullptr);
}

static int plan_totals(parpa_plan *p, Seg &tot, uint32_t &tau, uint64_t &first_inv) {
  cudaStream_t s = p->s;
  tot = p->a.seed;
  tau = NIB_IDENT;
  Ctrl ctrl;
  if (p->w.ntiles) {
    CK(cudaMemcpyAsync(&tot, p->w.tot_seg, sizeof(Seg), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&tau, p->w.tot_tau, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&ctrl, p->w.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    tot = seg_op(p->a.seed, tot);                      // the device total is unseeded
    first_inv = ctrl.inv_neg ? ~ctrl.inv_neg : NONE;
  } else {
    first_inv = NONE;
  }
  return PARPA_OK;
}

int parpa_plan_create(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, void *stream,
                      parpa_plan **out) {
  if (!dfa || !out || (len && !d_bytes)) return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  parpa_plan *p = new (std::nothrow) parpa_plan;
  if (!p) return PARPA_ENOMEM;
  prof_begin();
  int rc = plan_scan(dfa, d_bytes, len, dfa->start, seg_identity(), 0, 1024, s, p);
  if (rc) { work_free(p->w, s); delete p; return rc; }
  Seg tot;
  uint32_t tau;
  uint64_t fi;
  if ((rc = plan_totals(p, tot, tau, fi))) { work_free(p->w, s); delete p; return rc; }
  uint32_t fin = 0;
  if ((rc = host_final_exact(dfa, p->w, p->in, len, nib_at(tau, p->a.seed_dev), p->a.seed_exact, s, fin))) {
    work_free(p->w, s); delete p; return rc;
  }
  p->records = tot.recs + (dfa->eoi[fin] == EOI_RECORD ? 1 : 0);
  *out = p;
  return PARPA_OK;
}

int parpa_plan_records(const parpa_plan *p, uint64_t *records) {
  if (!p || !records) return PARPA_EINVAL;
  *records = p->records;
  return PARPA_OK;
}

int parpa_plan_emit(parpa_plan *p, const parpa_schema *sch, const parpa_column *cols, parpa_stats *d_stats,
                    void *stream) {
  if (!p || !sch || (sch->num_columns && !cols)) return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  ColsK ck;
  int rc = set_columns(sch, cols, sch->num_columns, ck);
  if (rc) return rc;
  KArgs a = p->a;
  a.C = sch->num_columns;
  a.strict = sch->strict;
  a.cap = p->records;
  a.stats = d_stats ? (Stats *)d_stats : p->w.stats;
  if ((rc = reset_emit_state(p, s))) return rc;
  rc = launch_emit(a, p->dfa->k, ck, s, nullptr);
  if (!rc) rc = launch_tail(a, p->dfa->k, ck, s, nullptr);
  prof_end();
  return rc;
}

void parpa_plan_destroy(parpa_plan *p) {
  if (!p) return;
  work_free(p->w, p->s);
  delete p;
}

// ---- one-call parse -------------------------------------------------------------------------------
int parpa_parse(const parpa_dfa *dfa, const parpa_schema *sch, const uint8_t *d_bytes, uint64_t len,
                void *stream, parpa_result **out) {
  if (!dfa || !sch || !out) return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  parpa_plan *p = nullptr;
  int rc = parpa_plan_create(dfa, d_bytes, len, stream, &p);
  if (rc) return rc;
  parpa_result *r = new (std::nothrow) parpa_result;
  if (!r) { parpa_plan_destroy(p); return PARPA_ENOMEM; }
  uint32_t C = sch->num_columns;
  r->C = C;
  r->cols.resize(C);
  uint64_t R = std::max<uint64_t>(p->records, 1);
  r->al = current_allocator();
  r->s = s;
  for (uint32_t c = 0; c < C; c++) {
    uint8_t type = sch->types ? sch->types[c] : PARPA_SPAN;
    void *a = nullptr;
    size_t per = 8 + 4 + (type != PARPA_SPAN ? 9 : 0);
    if (r->al.alloc) a = r->al.alloc(R * per + 64, stream, r->al.ctx);
    else if (cudaMallocAsync(&a, R * per + 64, s) != cudaSuccess) a = nullptr;
    if (!a) { rc = PARPA_ENOMEM; break; }
    r->allocs.push_back(a);
    uint8_t *b = (uint8_t *)a;
    r->cols[c].offset = (uint64_t *)b;
    r->cols[c].value = type != PARPA_SPAN ? (void *)(b + R * 8) : nullptr;
    r->cols[c].length = (uint32_t *)(b + R * (type != PARPA_SPAN ? 16 : 8));
    r->cols[c].valid = type != PARPA_SPAN ? b + R * 20 : nullptr;
  }
  if (!rc) rc = parpa_plan_emit(p, sch, r->cols.data(), nullptr, stream);
  if (!rc) {
    Stats st;
    if (cudaMemcpyAsync(&st, p->w.stats, sizeof(Stats), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      rc = PARPA_ECUDA;
    memcpy(&r->stats, &st, sizeof(st));
  }
  parpa_plan_destroy(p);
  if (rc) { parpa_result_free(r); return rc; }
  *out = r;
  return PARPA_OK;
}

int parpa_result_stats(const parpa_result *r, parpa_stats *out) {
  if (!r || !out) return PARPA_EINVAL;
  *out = r->stats;
  return PARPA_OK;
}
int parpa_result_records(const parpa_result *r, uint64_t *records) {
  if (!r || !records) return PARPA_EINVAL;
  *records = r->stats.records;
  return PARPA_OK;
}
int parpa_result_status(const parpa_result *r, int *status, uint64_t *first_invalid, uint64_t *n_missing_records,
                        uint64_t *n_extra_fields) {
  if (!r || !status) return PARPA_EINVAL;
  *status = r->stats.status;
  if (first_invalid) *first_invalid = r->stats.first_invalid;
  if (n_missing_records) *n_missing_records = r->stats.missing_records;
  if (n_extra_fields) *n_extra_fields = r->stats.extra_fields;
  return PARPA_OK;
}
int parpa_result_column(const parpa_result *r, uint32_t c, parpa_column *out) {
  if (!r || !out || c >= r->C) return PARPA_EINVAL;
  *out = r->cols[c];
  return PARPA_OK;
}
int parpa_result_copy_column(const parpa_result *r, uint32_t c, const parpa_column *dst, void *stream) {
  if (!r || !dst || c >= r->C) return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t R = r->stats.records;
  if (!R) return PARPA_OK;
  const parpa_column &src = r->cols[c];
  if (dst->offset) CK(cudaMemcpyAsync(dst->offset, src.offset, R * 8, cudaMemcpyDeviceToDevice, s));
  if (dst->length) CK(cudaMemcpyAsync(dst->length, src.length, R * 4, cudaMemcpyDeviceToDevice, s));
  if (dst->value && src.value) CK(cudaMemcpyAsync(dst->value, src.value, R * 8, cudaMemcpyDeviceToDevice, s));
  if (dst->valid && src.valid) CK(cudaMemcpyAsync(dst->valid, src.valid, R, cudaMemcpyDeviceToDevice, s));
  return PARPA_OK;
}

void parpa_result_free(parpa_result *r) {
  if (!r) return;
  for (void *a : r->allocs) {
    if (r->al.free) r->al.free(a, (void *)r->s, r->al.ctx);
    else cudaFreeAsync(a, r->s);
  }
  if (!r->al.free && !r->allocs.empty()) cudaStreamSynchronize(r->s);
  delete r;
}

int parpa_set_allocator(parpa_alloc_fn alloc, parpa_free_fn free_fn, void *ctx) {
  if ((alloc == nullptr) != (free_fn == nullptr)) return PARPA_EINVAL;
  std::lock_guard<std::mutex> g(g_alloc_mu);
  g_alloc.alloc = alloc;
  g_alloc.free = free_fn;
  g_alloc.ctx = ctx;
  return PARPA_OK;
}

// ---- single-pass capacity path ------------------------------------------------------------------
static int parse_into_impl(const parpa_dfa *dfa, const parpa_schema *sch, const uint8_t *d_bytes, uint64_t len,
                           const parpa_column *cols, uint64_t cap, parpa_stats *d_stats, cudaStream_t s,
                           uint32_t seed_state, const Seg &seed, uint64_t base, const uint8_t *left,
                           uint64_t left_len, int is_last, uint32_t *launches,
                           const uint64_t *d_skip = nullptr, uint64_t nskip = 0) {
  if (!dfa || !sch || !d_stats || (len && !d_bytes) || (sch->num_columns && !cols)) return PARPA_EINVAL;
  ColsK ck;
  int rc = set_columns(sch, cols, sch->num_columns, ck);
  if (rc) return rc;
  prof_begin();
  Work w;
  rc = work_alloc(w, len, sch->num_columns, len && misaligned(d_bytes), s);
  if (rc) return rc;
  const uint8_t *in = d_bytes;
  if (!rc) rc = prepare_input(w, in, len, s);
  if (!rc) {
    KArgs a;
    make_args(a, w, in, len);
    a.C = sch->num_columns;
    a.strict = sch->strict;
    a.cap = cap;
    a.stats = (Stats *)d_stats;
    a.seed_dev = dfa->dmap[seed_state];
    a.seed_exact = seed_state;
    a.seed = seed;
    a.base = base;
    a.row_base = seed.recs;
    a.left = left;
    a.left_len = left_len;
    a.is_last = is_last;
    a.skip = (const unsigned long long *)d_skip;
    a.nskip = d_skip ? nskip : 0;
    uint32_t n = 0;
    if (use_small(a)) {
      rc = launch_small(a, dfa->k, ck, s, &n);
    } else {
      rc = launch_passes(MODE_COUNT, a, dfa->k, s, &n);
      if (!rc) rc = launch_emit(a, dfa->k, ck, s, &n);
      if (!rc) rc = launch_tail(a, dfa->k, ck, s, &n);
    }
    if (launches) *launches = n;
  }
  work_free(w, s);
  prof_end();
  return rc;
}

int parpa_parse_into(const parpa_dfa *dfa, const parpa_schema *sch, const uint8_t *d_bytes, uint64_t len,
                     const parpa_column *cols, uint64_t cap, parpa_stats *d_stats, void *stream,
                     uint32_t *gpu_launches) {
  if (!dfa) return PARPA_EINVAL;
  return parse_into_impl(dfa, sch, d_bytes, len, cols, cap, d_stats, (cudaStream_t)stream,
                         dfa->start, seg_identity(), 0, nullptr, 0, 1, gpu_launches);
}

// ---- caller-owned workspace: parse_into without allocation, memset or host synchronisation --------------
struct parpa_workspace {
  Work w;
  uint64_t max_len = 0;
  size_t zero_bytes = 0;                // the look-back descriptors + control words (zeroed before a staged parse)
  bool clean = true;                    // control words zero (k_small leaves them so; the staged kernels do not)
};

int parpa_workspace_create(uint64_t max_len, void *stream, parpa_workspace **out) {
  if (!out) return PARPA_EINVAL;
  parpa_workspace *ws = new (std::nothrow) parpa_workspace;
  if (!ws) return PARPA_ENOMEM;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = work_alloc(ws->w, std::max<uint64_t>(max_len, 1), 0, false, s);
  if (rc) { delete ws; return rc; }
  ws->max_len = max_len;
  ws->zero_bytes = (size_t)((uint8_t *)ws->w.lex - (uint8_t *)ws->w.block);
  *out = ws;
  return PARPA_OK;
}

void parpa_workspace_destroy(parpa_workspace *ws) {
  if (!ws) return;
  if (ws->w.block) cudaFree(ws->w.block);
  delete ws;
}

int parpa_parse_into_ws(parpa_workspace *ws, const parpa_dfa *dfa, const parpa_schema *sch, const uint8_t *d_bytes,
                        uint64_t len, const parpa_column *cols, uint64_t cap, parpa_stats *d_stats, void *stream,
                        uint32_t *gpu_launches) {
  if (!ws || !dfa || !sch || !d_stats || (len && !d_bytes) || (sch->num_columns && !cols) || len > ws->max_len ||
      (len && misaligned(d_bytes)))
    return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  ColsK ck;
  int rc = set_columns(sch, cols, sch->num_columns, ck);
  if (rc) return rc;
  prof_begin();
  KArgs a;
  make_args(a, ws->w, d_bytes, len);
  a.ntiles = (uint32_t)((len + WT - 1) / WT);
  a.C = sch->num_columns;
  a.strict = sch->strict;
  a.cap = cap;
  a.stats = (Stats *)d_stats;
  a.seed_dev = dfa->dmap[dfa->start];
  a.seed_exact = dfa->start;
  uint32_t n = 0;
  if (use_small(a)) {
    if (!ws->clean) CK(cudaMemsetAsync(ws->w.block, 0, ws->zero_bytes, s));
    rc = launch_small(a, dfa->k, ck, s, &n);
    ws->clean = true;
  } else {
    CK(cudaMemsetAsync(ws->w.block, 0, ws->zero_bytes, s));
    rc = launch_passes(MODE_COUNT, a, dfa->k, s, &n);
    if (!rc) rc = launch_emit(a, dfa->k, ck, s, &n);
    if (!rc) rc = launch_tail(a, dfa->k, ck, s, &n);
    ws->clean = false;
  }
  if (gpu_launches) *gpu_launches = n;
  prof_end();
  return rc;
}

int parpa_parse_into_skip(const parpa_dfa *dfa, const parpa_schema *sch, const uint8_t *d_bytes, uint64_t len,
                          const uint64_t *d_skip_records, uint64_t nskip, const parpa_column *cols, uint64_t cap,
                          parpa_stats *d_stats, void *stream, uint32_t *gpu_launches) {
  if (!dfa || (nskip && !d_skip_records)) return PARPA_EINVAL;
  return parse_into_impl(dfa, sch, d_bytes, len, cols, cap, d_stats, (cudaStream_t)stream,
                         dfa->start, seg_identity(), 0, nullptr, 0, 1, gpu_launches, d_skip_records, nskip);
}

int parpa_parse_range(const parpa_dfa *dfa, const parpa_schema *sch, const uint8_t *d_bytes, uint64_t len,
                      const parpa_context *ctx, const uint8_t *left, uint64_t left_len, int is_last,
                      const parpa_column *cols, uint64_t cap, parpa_stats *d_stats, void *stream) {
  if (!dfa || !ctx || ctx->entry_state >= dfa->S) return PARPA_EINVAL;
  return parse_into_impl(dfa, sch, d_bytes, len, cols, cap, d_stats, (cudaStream_t)stream,
                         ctx->entry_state, counts_to_seg(ctx->prefix), ctx->base, left, left_len,
                         is_last, nullptr);
}

// ---- end-to-end from host memory ---------------------------------------------------------------------
// Streaming (the paper's §4.4): the input is cut into partitions of P bytes;
// partition i+1 is copied host->device on one stream while partition i is parsed on the caller's
// stream and partition i-1's columns are copied back on a third.  The context carry between
// partitions is the staged range plan (τ -> entry state, counts -> ⊕-prefix); a record straddling a
// cut has its first columns in partition i-1's last local row and the rest in partition i's row 0,
// and each partition copies back only its own columns of those rows.  Each partition sees a 1 MB
// left context (the "halo") for typed fields that straddle the cut.
static uint64_t stream_partition_bytes() {
  const char *e = getenv("PARPA_STREAM_PARTITION");
  if (e) {
    unsigned long long v = strtoull(e, nullptr, 10);
    if (v >= 4096) return v;
  }
  return 512ull << 20;
}

static int parse_host_stream(const parpa_dfa *dfa, const parpa_schema *sch, const uint8_t *h_bytes, uint64_t len,
                             const parpa_column *h_cols, uint64_t cap, parpa_stats *stats, cudaStream_t s,
                             uint64_t P) {
  const uint32_t C = sch->num_columns;
  const uint64_t HALO = 1ull << 20;
  const uint64_t np = (len + P - 1) / P;
  cudaStream_t sc = nullptr, sd = nullptr;
  cudaEvent_t evH[2] = {nullptr, nullptr}, evC[2] = {nullptr, nullptr}, evA = nullptr;
  uint8_t *inbuf[2] = {nullptr, nullptr};
  Stats *d_pst = nullptr;
  std::vector<Stats> pst(np);
  int rc = PARPA_OK;
  auto ck = [&](cudaError_t e) { if (e != cudaSuccess && rc == PARPA_OK) rc = cuda_status(e); return rc == PARPA_OK; };
  ck(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
  ck(cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking));
  for (int b = 0; b < 2; b++) {
    ck(cudaEventCreateWithFlags(&evH[b], cudaEventDisableTiming));
    ck(cudaEventCreateWithFlags(&evC[b], cudaEventDisableTiming));
    ck(cudaMallocAsync(&inbuf[b], HALO + P + 64, s));
  }
  ck(cudaEventCreateWithFlags(&evA, cudaEventDisableTiming));
  ck(cudaMallocAsync(&d_pst, np * sizeof(Stats), s));
  ck(cudaEventRecord(evA, s));                           // allocations visible to the copy streams
  ck(cudaStreamWaitEvent(sc, evA, 0));
  ck(cudaStreamWaitEvent(sd, evA, 0));
  auto h2d = [&](uint64_t i) {
    const uint64_t base = i * P, n = std::min(P, len - base), halo = std::min(HALO, base);
    const int b = (int)(i & 1);
    ck(cudaStreamWaitEvent(sc, evC[b], 0));             // partition i-2 is done with this buffer
    ck(cudaMemcpyAsync(inbuf[b] + HALO - halo, h_bytes + base - halo, halo + n, cudaMemcpyHostToDevice, sc));
    ck(cudaEventRecord(evH[b], sc));
  };
  Seg prefix = seg_identity();
  uint32_t state = dfa->start;
  uint64_t total_rows = 0;
  if (rc == PARPA_OK) h2d(0);
  for (uint64_t i = 0; i < np && rc == PARPA_OK; i++) {
    const uint64_t base = i * P, n = std::min(P, len - base), halo = std::min(HALO, base);
    const int b = (int)(i & 1);
    const bool last = i + 1 == np;
    if (!last) h2d(i + 1);                               // overlaps this partition's parse
    if (!ck(cudaStreamWaitEvent(s, evH[b], 0))) break;
    parpa_plan *p = nullptr;
    parpa_tau tau;
    if ((rc = parpa_range_begin(dfa, inbuf[b] + HALO, n, base, s, &p, &tau))) break;
    parpa_counts cnt;
    if ((rc = parpa_range_count(p, state, &cnt))) { parpa_plan_destroy(p); break; }
    const uint32_t next_state = tau.tau[state];
    const uint64_t nloc = cnt.records + ((last && dfa->eoi[next_state] == PARPA_EOI_RECORD) ? 1 : 0);
    const Seg after = seg_op(prefix, counts_to_seg(cnt));
    const uint64_t rows_alloc = nloc + 2;
    std::vector<parpa_column> dcols(C);
    void *blk = nullptr;
    size_t tot = 0;
    for (uint32_t c = 0; c < C; c++) {
      const uint8_t type = sch->types ? sch->types[c] : PARPA_SPAN;
      tot += align_up(rows_alloc * 8) + align_up(rows_alloc * 4) + (type != PARPA_SPAN ? align_up(rows_alloc * 8) + align_up(rows_alloc) : 0);
    }
    if (!ck(cudaMallocAsync(&blk, std::max<size_t>(tot, 256), s))) { parpa_plan_destroy(p); break; }
    uint8_t *q = (uint8_t *)blk;
    for (uint32_t c = 0; c < C; c++) {
      const uint8_t type = sch->types ? sch->types[c] : PARPA_SPAN;
      dcols[c].offset = (uint64_t *)q; q += align_up(rows_alloc * 8);
      dcols[c].length = (uint32_t *)q; q += align_up(rows_alloc * 4);
      if (type != PARPA_SPAN) {
        dcols[c].value = q; q += align_up(rows_alloc * 8);
        dcols[c].valid = q; q += align_up(rows_alloc);
      } else {
        dcols[c].value = nullptr;
        dcols[c].valid = nullptr;
      }
    }
    parpa_context ctx;
    memset(&ctx, 0, sizeof(ctx));
    ctx.entry_state = state;
    ctx.base = base;
    ctx.prefix = seg_to_counts(prefix, NONE);
    rc = parpa_range_emit(p, sch, &ctx, halo ? inbuf[b] + HALO - halo : nullptr, halo, last ? 1 : 0, dcols.data(),
                          rows_alloc, (parpa_stats *)(d_pst + i), s);
    parpa_plan_destroy(p);
    if (rc) { cudaFreeAsync(blk, s); break; }
    ck(cudaEventRecord(evC[b], s));
    ck(cudaStreamWaitEvent(sd, evC[b], 0));
    // this partition's rows: local row 0 = global row prefix.recs; columns before the partition's
    // start column belong to the previous partition, those after its end column to the next
    const uint64_t row0 = prefix.recs;
    for (uint32_t c = 0; c < C && rc == PARPA_OK; c++) {
      const uint64_t lo = c < prefix.col ? 1 : 0;
      const uint64_t hi = nloc + ((!last && c < after.col) ? 1 : 0);
      const uint64_t glo = row0 + lo, ghi = std::min<uint64_t>(row0 + hi, cap);
      if (glo >= ghi) continue;
      const uint64_t m = ghi - glo;
      if (h_cols[c].offset) ck(cudaMemcpyAsync(h_cols[c].offset + glo, dcols[c].offset + lo, m * 8, cudaMemcpyDeviceToHost, sd));
      if (h_cols[c].length) ck(cudaMemcpyAsync(h_cols[c].length + glo, dcols[c].length + lo, m * 4, cudaMemcpyDeviceToHost, sd));
      if (dcols[c].value && h_cols[c].value)
        ck(cudaMemcpyAsync((uint8_t *)h_cols[c].value + glo * 8, (uint8_t *)dcols[c].value + lo * 8, m * 8, cudaMemcpyDeviceToHost, sd));
      if (dcols[c].valid && h_cols[c].valid) ck(cudaMemcpyAsync(h_cols[c].valid + glo, dcols[c].valid + lo, m, cudaMemcpyDeviceToHost, sd));
    }
    ck(cudaMemcpyAsync(&pst[i], d_pst + i, sizeof(Stats), cudaMemcpyDeviceToHost, sd));
    ck(cudaFreeAsync(blk, sd));
    total_rows += nloc;
    state = next_state;
    prefix = after;
  }
  if (sd) cudaStreamSynchronize(sd);
  if (sc) cudaStreamSynchronize(sc);
  cudaStreamSynchronize(s);
  if (rc == PARPA_OK) {                                   // combine the partitions' statistics
    Stats t;
    memset(&t, 0, sizeof(t));
    t.first_invalid = NONE;
    int st = ST_OK;
    for (uint64_t i = 0; i < np; i++) {
      t.fields += pst[i].fields;
      t.missing_records += pst[i].missing_records;
      t.extra_fields += pst[i].extra_fields;
      t.deferred_fields += pst[i].deferred_fields;
      t.block_fields += pst[i].block_fields;
      t.device_fields += pst[i].device_fields;
      t.first_invalid = std::min(t.first_invalid, pst[i].first_invalid);
      const int ps = pst[i].status;
      if (ps == ST_EFORMAT) st = ST_EFORMAT;
      else if (ps == ST_EUNSUPPORTED && st != ST_EFORMAT) st = ST_EUNSUPPORTED;
      else if (ps == ST_ECOLUMNS && st == ST_OK) st = ST_ECOLUMNS;
    }
    t.records = total_rows;
    if (st == ST_OK || st == ST_ECOLUMNS) {
      if (total_rows > cap) st = ST_ENEEDMORE;
    }
    t.status = st;
    t.final_state = pst[np - 1].final_state;
    memcpy(stats, &t, sizeof(t));
  }
  for (int b = 0; b < 2; b++) {
    if (inbuf[b]) cudaFreeAsync(inbuf[b], s);
    if (evH[b]) cudaEventDestroy(evH[b]);
    if (evC[b]) cudaEventDestroy(evC[b]);
  }
  if (d_pst) cudaFreeAsync(d_pst, s);
  if (evA) cudaEventDestroy(evA);
  cudaStreamSynchronize(s);
  if (sc) cudaStreamDestroy(sc);
  if (sd) cudaStreamDestroy(sd);
  return rc;
}

int parpa_parse_host(const parpa_dfa *dfa, const parpa_schema *sch, const uint8_t *h_bytes, uint64_t len,
                     const parpa_column *h_cols, uint64_t cap, parpa_stats *stats, void *stream) {
  if (!dfa || !sch || !stats || (len && !h_bytes)) return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t P = stream_partition_bytes();
  if (len > P) return parse_host_stream(dfa, sch, h_bytes, len, h_cols, cap, stats, s, P);
  uint32_t C = sch->num_columns;
  std::vector<parpa_column> dcols(C);
  std::vector<size_t> per(C);
  void *blk = nullptr;
  size_t total = align_up(len + 16) + align_up(sizeof(Stats));
  for (uint32_t c = 0; c < C; c++) {
    uint8_t type = sch->types ? sch->types[c] : PARPA_SPAN;
    per[c] = align_up(cap * 8) + align_up(cap * 4) + (type != PARPA_SPAN ? align_up(cap * 8) + align_up(cap) : 0);
    total += per[c];
  }
  CK(cudaMallocAsync(&blk, total, s));
  uint8_t *b = (uint8_t *)blk;
  uint8_t *d_in = b;
  b += align_up(len + 16);
  parpa_stats *d_stats = (parpa_stats *)b;
  b += align_up(sizeof(Stats));
  for (uint32_t c = 0; c < C; c++) {
    uint8_t type = sch->types ? sch->types[c] : PARPA_SPAN;
    dcols[c].offset = (uint64_t *)b; b += align_up(cap * 8);
    dcols[c].length = (uint32_t *)b; b += align_up(cap * 4);
    if (type != PARPA_SPAN) {
      dcols[c].value = b; b += align_up(cap * 8);
      dcols[c].valid = b; b += align_up(cap);
    } else {
      dcols[c].value = nullptr;
      dcols[c].valid = nullptr;
    }
  }
  int rc = PARPA_OK;
  if (len && cudaMemcpyAsync(d_in, h_bytes, len, cudaMemcpyHostToDevice, s) != cudaSuccess) rc = PARPA_ECUDA;
  if (!rc) rc = parpa_parse_into(dfa, sch, d_in, len, dcols.data(), cap, d_stats, stream, nullptr);
  Stats hs;
  if (!rc && cudaMemcpyAsync(&hs, d_stats, sizeof(Stats), cudaMemcpyDeviceToHost, s) != cudaSuccess) rc = PARPA_ECUDA;
  if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = PARPA_ECUDA;
  if (!rc) {
    uint64_t R = std::min<uint64_t>(hs.records, cap);
    for (uint32_t c = 0; c < C && !rc; c++) {
      if (!R) break;
      if (h_cols[c].offset && cudaMemcpyAsync(h_cols[c].offset, dcols[c].offset, R * 8, cudaMemcpyDeviceToHost, s)) rc = PARPA_ECUDA;
      if (h_cols[c].length && cudaMemcpyAsync(h_cols[c].length, dcols[c].length, R * 4, cudaMemcpyDeviceToHost, s)) rc = PARPA_ECUDA;
      if (dcols[c].value && h_cols[c].value && cudaMemcpyAsync(h_cols[c].value, dcols[c].value, R * 8, cudaMemcpyDeviceToHost, s)) rc = PARPA_ECUDA;
      if (dcols[c].valid && h_cols[c].valid && cudaMemcpyAsync(h_cols[c].valid, dcols[c].valid, R, cudaMemcpyDeviceToHost, s)) rc = PARPA_ECUDA;
    }
    if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = PARPA_ECUDA;
    memcpy(stats, &hs, sizeof(hs));
  }
  cudaFreeAsync(blk, s);
  cudaStreamSynchronize(s);
  return rc;
}

// ---- range summaries -------------------------------------------------------------------------------
int parpa_summarize(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, void *stream, parpa_tau *out) {
  if (!dfa || !out || (len && !d_bytes)) return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  Work w;
  int rc = work_alloc(w, len, 1, len && misaligned(d_bytes), s);
  if (rc) return rc;
  const uint8_t *in = d_bytes;
  rc = prepare_input(w, in, len, s);
  KArgs a;
  make_args(a, w, in, len);
  if (!rc) rc = launch_passes(MODE_TAU, a, dfa->k, s, nullptr);
  uint32_t desc = NIB_IDENT;
  if (!rc && w.ntiles) {
    if (cudaMemcpyAsync(&desc, w.tot_tau, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess) rc = PARPA_ECUDA;
  }
  if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = PARPA_ECUDA;
  if (!rc) rc = host_tau_exact(dfa, w, in, len, (uint32_t)desc, s, out);
  work_free(w, s);
  return rc;
}

int parpa_count(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, uint64_t base, uint32_t entry,
                void *stream, parpa_counts *out, parpa_tau *tau_out) {
  if (!dfa || !out || entry >= dfa->S || (len && !d_bytes)) return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  parpa_plan p;
  int rc = plan_scan(dfa, d_bytes, len, entry, seg_identity(), base, 1, s, &p);
  Seg tot;
  uint32_t tau = NIB_IDENT;
  uint64_t fi = NONE;
  if (!rc) rc = plan_totals(&p, tot, tau, fi);
  if (!rc) {
    *out = seg_to_counts(tot, fi);
    if (tau_out) rc = host_tau_exact(dfa, p.w, p.in, len, tau, s, tau_out);
  }
  work_free(p.w, s);
  return rc;
}

int parpa_compose_tau(const parpa_dfa *dfa, const parpa_tau *a, const parpa_tau *b, parpa_tau *out) {
  if (!dfa || !a || !b || !out) return PARPA_EINVAL;
  parpa_tau r;
  for (int i = 0; i < 16; i++) r.tau[i] = 0xFF;
  for (uint32_t i = 0; i < dfa->S; i++) {
    if (a->tau[i] >= dfa->S) return PARPA_EINVAL;
    r.tau[i] = b->tau[a->tau[i]];                 // (a∘b)_i = b_{a_i}
  }
  *out = r;
  return PARPA_OK;
}

int parpa_compose_counts(const parpa_counts *a, const parpa_counts *b, parpa_counts *out) {
  if (!a || !b || !out) return PARPA_EINVAL;
  Seg c = seg_op(counts_to_seg(*a), counts_to_seg(*b));
  *out = seg_to_counts(c, std::min(a->first_invalid, b->first_invalid));
  return PARPA_OK;
}

// ---- staged range plan (multi-GPU exchange with every pass run once) ------------------------------
int parpa_range_begin(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, uint64_t base, void *stream,
                      parpa_plan **out, parpa_tau *tau_out) {
  if (!dfa || !out || !tau_out || (len && !d_bytes)) return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  parpa_plan *p = new (std::nothrow) parpa_plan;
  if (!p) return PARPA_ENOMEM;
  p->dfa = dfa;
  p->len = len;
  p->s = s;
  p->records = 0;
  int rc = work_alloc(p->w, len, 1, len && misaligned(d_bytes), s);
  if (rc) { delete p; return rc; }
  const uint8_t *in = d_bytes;
  if (!rc) rc = prepare_input(p->w, in, len, s);
  p->in = in;
  make_args(p->a, p->w, in, len);
  p->a.base = base;
  p->a.seed_dev = INV_DEV + 1;                            // not known yet: set by parpa_range_count
  if (!rc) rc = launch_passes(MODE_TAU, p->a, dfa->k, s, nullptr);
  uint32_t tau = NIB_IDENT;
  if (!rc && p->w.ntiles && cudaMemcpyAsync(&tau, p->w.tot_tau, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    rc = PARPA_ECUDA;
  if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = PARPA_ECUDA;
  prof_end();
  if (!rc) rc = host_tau_exact(dfa, p->w, p->in, len, tau, s, tau_out);
  if (rc) { work_free(p->w, s); delete p; return rc; }
  *out = p;
  return PARPA_OK;
}

int parpa_range_count(parpa_plan *p, uint32_t entry_state, parpa_counts *out) {
  if (!p || !out || entry_state >= p->dfa->S) return PARPA_EINVAL;
  if (int rc0 = reset_scan_state(p)) return rc0;
  p->a.seed_dev = p->dfa->dmap[entry_state];
  p->a.seed_exact = entry_state;
  int rc = launch_half2(p->a, p->dfa->k, p->s, nullptr);
  prof_end();
  if (rc) return rc;
  Seg tot;
  uint32_t tau;
  uint64_t fi;
  if ((rc = plan_totals(p, tot, tau, fi))) return rc;        // a.seed is the identity here
  *out = seg_to_counts(tot, fi);
  return PARPA_OK;
}

int parpa_range_emit(parpa_plan *p, const parpa_schema *sch, const parpa_context *ctx, const uint8_t *left,
                     uint64_t left_len, int is_last, const parpa_column *cols, uint64_t cap, parpa_stats *d_stats,
                     void *stream) {
  return parpa_range_emit_halo(p, sch, ctx, left, left_len, PARPA_STATE_UNKNOWN, is_last, cols, cap, d_stats, stream);
}

int parpa_range_state_at(const parpa_plan *p, uint64_t pos, uint32_t *state) {
  if (!p || !state || pos < p->a.base || pos >= p->a.base + p->len || ((pos - p->a.base) % CHUNK) != 0 ||
      p->a.seed_dev > INV_DEV)
    return PARPA_EINVAL;
  uint8_t d = 0;
  CK(cudaMemcpyAsync(&d, p->w.chunk_state + (pos - p->a.base) / CHUNK, 1, cudaMemcpyDeviceToHost, p->s));
  CK(cudaStreamSynchronize(p->s));
  *state = p->dfa->k.hmap[d & 0xF];
  return PARPA_OK;
}

int parpa_range_emit_halo(parpa_plan *p, const parpa_schema *sch, const parpa_context *ctx, const uint8_t *left,
                          uint64_t left_len, uint32_t left_state, int is_last, const parpa_column *cols, uint64_t cap,
                          parpa_stats *d_stats, void *stream) {
  if (!p || !sch || !ctx || !d_stats || (sch->num_columns && !cols)) return PARPA_EINVAL;
  if (left_state != PARPA_STATE_UNKNOWN && (left_state >= p->dfa->S || !left || !left_len)) return PARPA_EINVAL;
  if (ctx->entry_state >= p->dfa->S || p->dfa->dmap[ctx->entry_state] != p->a.seed_dev) return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  ColsK ck;
  int rc = set_columns(sch, cols, sch->num_columns, ck);
  if (rc) return rc;
  KArgs a = p->a;
  a.C = sch->num_columns;
  a.strict = sch->strict;
  a.cap = cap;
  a.stats = (Stats *)d_stats;
  a.seed = counts_to_seg(ctx->prefix);
  a.row_base = a.seed.recs;
  a.left = left;
  a.left_len = left_len;
  a.left_state = left_state == PARPA_STATE_UNKNOWN ? 0xFFu : p->dfa->dmap[left_state];
  a.is_last = is_last;
  if ((rc = reset_emit_state(p, s))) return rc;
  rc = launch_emit(a, p->dfa->k, ck, s, nullptr);
  if (!rc) rc = launch_tail(a, p->dfa->k, ck, s, nullptr);
  prof_end();
  return rc;
}

// ---- column-count inference ---------------------------------------------------------------
int parpa_infer_columns(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, void *stream,
                        uint32_t *min_fields, uint32_t *max_fields, uint64_t *records) {
  if (!dfa || !min_fields || !max_fields || !records || (len && !d_bytes)) return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  parpa_plan p;
  int rc = plan_scan(dfa, d_bytes, len, dfa->start, seg_identity(), 0, 1, s, &p);
  unsigned int *d_mm = nullptr;
  unsigned int mm[2] = {0xFFFFFFFFu, 0u};
  if (!rc && cudaMallocAsync(&d_mm, 8, s) != cudaSuccess) rc = PARPA_ENOMEM;
  if (!rc && cudaMemcpyAsync(d_mm, mm, 8, cudaMemcpyHostToDevice, s) != cudaSuccess) rc = PARPA_ECUDA;
  if (!rc && p.w.ntiles) {
    DevCfg *dc;
    if (!(rc = dev_cfg(&dc))) {
      k_infer_cols<<<dc->sms * 4, 256, 0, s>>>(p.a, d_mm);
      if (cudaGetLastError() != cudaSuccess) rc = PARPA_ECUDA;
    }
  }
  if (!rc && cudaMemcpyAsync(mm, d_mm, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess) rc = PARPA_ECUDA;
  Seg tot;
  uint32_t tau;
  uint64_t fi;
  if (!rc) rc = plan_totals(&p, tot, tau, fi);               // synchronises
  uint32_t fin = 0;
  if (!rc) rc = host_final_exact(dfa, p.w, p.in, len, nib_at(tau, p.a.seed_dev), p.a.seed_exact, s, fin);
  if (d_mm) cudaFreeAsync(d_mm, s);
  work_free(p.w, s);
  if (rc) return rc;
  uint64_t R = tot.recs;
  if (dfa->eoi[fin] == EOI_RECORD) {                         // the implicit last record
    const uint32_t n = tot.col + 1;
    mm[0] = std::min(mm[0], n);
    mm[1] = std::max(mm[1], n);
    R++;
  }
  *records = R;
  *min_fields = R ? mm[0] : 0;
  *max_fields = mm[1];
  return fi != NONE ? PARPA_EFORMAT : PARPA_OK;
}

// ---- type inference (reading R31) ---------------------------------------------
static uint8_t resolve_class(uint32_t m) {
  m &= ~1u;                                                   // empty fields carry no type
  if (!m) return PARPA_CLASS_EMPTY;
  if (m & (1u << PARPA_CLASS_STRING)) return PARPA_CLASS_STRING;
  if (m & (1u << PARPA_CLASS_TIMESTAMP)) return m == (1u << PARPA_CLASS_TIMESTAMP) ? PARPA_CLASS_TIMESTAMP : PARPA_CLASS_STRING;
  return (uint8_t)(31 - __builtin_clz(m));                     // the widest numeric class
}

int parpa_infer_types(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, uint32_t num_columns,
                      void *stream, uint32_t *class_masks, uint8_t *types, uint64_t *records) {
  if (!dfa || (len && !d_bytes) || (num_columns && (!class_masks || !types)) || num_columns > MAX_COLS)
    return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  parpa_plan *p = nullptr;
  int rc = parpa_plan_create(dfa, d_bytes, len, stream, &p);
  if (rc) return rc;
  const uint64_t R = p->records, Rc = std::max<uint64_t>(R, 1);
  void *blk = nullptr;
  unsigned int *d_mask = nullptr;
  const size_t len_off = (Rc * 8 + 255) / 256 * 256, col_bytes = (len_off + Rc * 4 + 255) / 256 * 256;
  if (cudaMallocAsync(&blk, num_columns * col_bytes + 4 * (size_t)std::max(num_columns, 1u) + 16, s) != cudaSuccess)
    rc = PARPA_ENOMEM;
  std::vector<parpa_column> cols(num_columns);
  std::vector<uint8_t> tspan(num_columns, PARPA_SPAN);
  if (!rc) {
    uint8_t *b = (uint8_t *)blk;
    for (uint32_t c = 0; c < num_columns; c++) {
      cols[c].offset = (uint64_t *)(b + c * col_bytes);
      cols[c].length = (uint32_t *)(b + c * col_bytes + len_off);
      cols[c].value = nullptr;
      cols[c].valid = nullptr;
    }
    d_mask = (unsigned int *)(b + num_columns * col_bytes);
    if (cudaMemsetAsync(d_mask, 0, 4 * (size_t)std::max(num_columns, 1u), s) != cudaSuccess) rc = PARPA_ECUDA;
  }
  parpa_schema sch{num_columns, tspan.data(), nullptr, nullptr, 0};
  if (!rc && num_columns) rc = parpa_plan_emit(p, &sch, cols.data(), nullptr, stream);   // spans of every column
  DevCfg *dc = nullptr;
  if (!rc && R) rc = dev_cfg(&dc);
  for (uint32_t c = 0; !rc && R && c < num_columns; c++) {
    k_field_class<<<dc->sms * 8, 256, 0, s>>>(p->a, (const unsigned long long *)cols[c].offset, cols[c].length, R,
                                              d_mask + c);
    if (cudaGetLastError() != cudaSuccess) rc = PARPA_ECUDA;
  }
  parpa_stats st{};
  if (!rc && num_columns && cudaMemcpyAsync(class_masks, d_mask, 4 * num_columns, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    rc = PARPA_ECUDA;
  if (!rc && cudaMemcpyAsync(&st, p->w.stats, sizeof(st), cudaMemcpyDeviceToHost, s) != cudaSuccess) rc = PARPA_ECUDA;
  if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = PARPA_ECUDA;
  if (blk) cudaFreeAsync(blk, s);
  parpa_plan_destroy(p);
  if (rc) return rc;
  for (uint32_t c = 0; c < num_columns; c++) types[c] = resolve_class(class_masks[c]);
  if (records) *records = R;
  return st.status == PARPA_EFORMAT || st.status == PARPA_EUNSUPPORTED ? st.status : PARPA_OK;
}

// ---- string materialisation ---------------------------------------------------------------
// The CSS of one column (layouts P:493-502) from a completed scan half over the same bytes (a.masks).
// Sizes (d_data null): per-row DATA counts (+1 per field for the inline terminator), exclusive scan -> d_offsets,
// total.  Copy: the bytes, the terminators (INLINE) or the auxiliary vector (VECTOR).  Synchronous.
static int strings_core(const KArgs &a, const parpa_column *col, uint64_t rows, uint32_t mode, uint32_t term,
                        int64_t *d_offsets, uint64_t *total, uint8_t *d_data, uint8_t *d_aux, cudaStream_t s) {
  DevCfg *dc = nullptr;
  int rc = dev_cfg(&dc);
  if (rc) return rc;
  const unsigned long long *off = (const unsigned long long *)col->offset;
  unsigned long long *v = (unsigned long long *)d_offsets;
  if (!d_data) {
    if (!rows) {
      CK(cudaMemsetAsync(d_offsets, 0, 8, s));
      CK(cudaStreamSynchronize(s));
      if (total) *total = 0;
      return PARPA_OK;
    }
    k_str_len<<<dc->sms * 8, 256, 0, s>>>(a, off, col->length, rows, v, mode == CSS_INLINE ? 1u : 0u);
    CK(cudaGetLastError());
    const uint64_t nb = (rows + SCAN_TILE - 1) / SCAN_TILE;
    void *sb = nullptr;
    const size_t o_agg = (16 + nb * 4 + 15) / 16 * 16;                  // 8-byte payloads stay aligned
    const size_t bytes = o_agg + 2 * nb * 8;
    CK(cudaMallocAsync(&sb, bytes, s));
    if (cudaMemsetAsync(sb, 0, bytes, s) != cudaSuccess) rc = PARPA_ECUDA;
    if (!rc) {
      uint8_t *b = (uint8_t *)sb;
      k_scan_u64<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(v, rows, (unsigned int *)b, (uint32_t *)(b + 16),
                                                        (unsigned long long *)(b + o_agg),
                                                        (unsigned long long *)(b + o_agg + nb * 8));
      if (cudaGetLastError() != cudaSuccess) rc = PARPA_ECUDA;
    }
    cudaFreeAsync(sb, s);
    if (!rc && total && cudaMemcpyAsync(total, v + rows, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess) rc = PARPA_ECUDA;
    if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = PARPA_ECUDA;
    return rc;
  }
  if (!rows) return PARPA_OK;
  unsigned int *clash = nullptr;
  CK(cudaMallocAsync(&clash, 4, s));
  if (cudaMemsetAsync(clash, 0, 4, s) != cudaSuccess) rc = PARPA_ECUDA;
  if (!rc && mode == CSS_VECTOR) {                                      // the auxiliary vector starts zeroed
    uint64_t n = 0;
    if (cudaMemcpyAsync(&n, v + rows, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
      rc = PARPA_ECUDA;
    if (!rc && n && cudaMemsetAsync(d_aux, 0, n, s) != cudaSuccess) rc = PARPA_ECUDA;
  }
  if (!rc) {
    k_str_copy<<<dc->sms * 8, 256, 0, s>>>(a, off, col->length, rows, v, d_data, mode, term, d_aux, clash);
    if (cudaGetLastError() != cudaSuccess) rc = PARPA_ECUDA;
  }
  unsigned int h = 0;
  if (!rc && (cudaMemcpyAsync(&h, clash, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess))
    rc = PARPA_ECUDA;
  cudaFreeAsync(clash, s);
  if (!rc && h) rc = PARPA_EUNSUPPORTED;                                // the terminator occurs in the CSS
  return rc;
}

static int strings_impl(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, const parpa_column *col,
                        uint64_t rows, int64_t *d_offsets, uint64_t *total, uint8_t *d_data, cudaStream_t s) {
  Work w;
  int rc = work_alloc(w, len, 1, len && misaligned(d_bytes), s);
  if (rc) return rc;
  const uint8_t *in = d_bytes;
  rc = prepare_input(w, in, len, s);
  KArgs a;
  make_args(a, w, in, len);
  a.seed_dev = dfa->dmap[dfa->start];
  a.seed_exact = dfa->start;
  if (!rc) rc = launch_passes(MODE_COUNT, a, dfa->k, s, nullptr);       // the chunk masks
  if (!rc) rc = strings_core(a, col, rows, CSS_ARROW, 0u, d_offsets, total, d_data, nullptr, s);
  work_free(w, s);
  if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = PARPA_ECUDA;
  return rc;
}

int parpa_strings_size(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, const parpa_column *column,
                       uint64_t rows, int64_t *d_offsets, uint64_t *total, void *stream) {
  if (!dfa || !column || !d_offsets || !total || (len && !d_bytes) || (rows && (!column->offset || !column->length)))
    return PARPA_EINVAL;
  return strings_impl(dfa, d_bytes, len, column, rows, d_offsets, total, nullptr, (cudaStream_t)stream);
}

int parpa_strings_copy(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, const parpa_column *column,
                       uint64_t rows, const int64_t *d_offsets, uint8_t *d_data, void *stream) {
  if (!dfa || !column || !d_offsets || !d_data || (len && !d_bytes) || (rows && (!column->offset || !column->length)))
    return PARPA_EINVAL;
  return strings_impl(dfa, d_bytes, len, column, rows, const_cast<int64_t *>(d_offsets), nullptr, d_data,
                      (cudaStream_t)stream);
}

// ---- CSS from a plan (reuses the plan's chunk masks: no second scan half) -----------------------------
int parpa_plan_strings_size(parpa_plan *plan, const parpa_column *column, uint64_t rows, uint32_t mode,
                            int64_t *d_offsets, uint64_t *total, void *stream) {
  if (!plan || !column || !d_offsets || !total || mode > CSS_VECTOR || (rows && (!column->offset || !column->length)))
    return PARPA_EINVAL;
  return strings_core(plan->a, column, rows, mode, 0u, d_offsets, total, nullptr, nullptr, (cudaStream_t)stream);
}
int parpa_plan_strings_copy(parpa_plan *plan, const parpa_column *column, uint64_t rows, uint32_t mode,
                            uint32_t terminator, const int64_t *d_offsets, uint8_t *d_data, uint8_t *d_aux,
                            void *stream) {
  if (!plan || !column || !d_offsets || !d_data || mode > CSS_VECTOR || terminator > 255 ||
      (mode == CSS_VECTOR && !d_aux) || (rows && (!column->offset || !column->length)))
    return PARPA_EINVAL;
  return strings_core(plan->a, column, rows, mode, terminator, const_cast<int64_t *>(d_offsets), nullptr, d_data,
                      d_aux, (cudaStream_t)stream);
}

int parpa_css_index(uint32_t mode, uint32_t terminator, const uint8_t *d_data, const uint8_t *d_aux, uint64_t n,
                    uint64_t *d_index, uint64_t *count, void *stream) {
  if ((mode != CSS_INLINE && mode != CSS_VECTOR) || terminator > 255 || !count || (n && !d_index) ||
      (n && mode == CSS_INLINE && !d_data) || (n && mode == CSS_VECTOR && !d_aux))
    return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  *count = 0;
  if (n == 0) return PARPA_OK;
  DevCfg *dc;
  int rc = dev_cfg(&dc);
  if (rc) return rc;
  const uint64_t nt = (n + WT - 1) / WT, nb = (nt + SCAN_TILE - 1) / SCAN_TILE;
  const size_t o_scan = align_up((nt + 1) * 8), o_agg = (16 + nb * 4 + 15) / 16 * 16, scan_bytes = o_agg + 2 * nb * 8;
  void *blk = nullptr;
  CK(cudaMallocAsync(&blk, o_scan + scan_bytes, s));
  uint8_t *b = (uint8_t *)blk;
  unsigned long long *cnt = (unsigned long long *)b;
  uint8_t *sc = b + o_scan;
  if (cudaMemsetAsync(sc, 0, scan_bytes, s) != cudaSuccess) rc = PARPA_ECUDA;
  const unsigned grid = (unsigned)std::min<uint64_t>((uint64_t)dc->sms * 8, (nt + 7) / 8);
  if (!rc) {
    k_css_count<<<grid, 256, 0, s>>>(mode, d_data, d_aux, terminator, n, cnt);
    k_scan_u64<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(cnt, nt, (unsigned int *)sc, (uint32_t *)(sc + 16),
                                                      (unsigned long long *)(sc + o_agg),
                                                      (unsigned long long *)(sc + o_agg + nb * 8));
    k_css_write<<<grid, 256, 0, s>>>(mode, d_data, d_aux, terminator, n, cnt, (unsigned long long *)d_index);
    if (cudaGetLastError() != cudaSuccess) rc = PARPA_ECUDA;
  }
  if (!rc && (cudaMemcpyAsync(count, cnt + nt, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
              cudaStreamSynchronize(s) != cudaSuccess))
    rc = PARPA_ECUDA;
  cudaFreeAsync(blk, s);
  return rc;
}

// ---- skipping rows (stream compaction) ---------------------------------------------------
int parpa_compact_rows(const uint8_t *d_in, uint64_t len, const uint64_t *d_skip_rows, uint64_t nskip, uint8_t *d_out,
                       uint64_t *out_len, void *stream) {
  if ((len && (!d_in || !d_out)) || !out_len || (nskip && !d_skip_rows)) return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (len == 0) { *out_len = 0; return PARPA_OK; }
  DevCfg *dc;
  int rc = dev_cfg(&dc);
  if (rc) return rc;
  const uint64_t nt64 = (len + WT - 1) / WT;
  if (nt64 > 0x07FFFFFFull) return PARPA_EUNSUPPORTED;
  const uint32_t nt = (uint32_t)nt64;
  const uint64_t nb = (nt + SCAN_TILE - 1) / SCAN_TILE;
  // [lines / first row per tile : nt + 1][kept / output offset per tile : nt + 1][scan scratch]
  const size_t o_lines = 0, o_kept = align_up((nt + 1) * 8), o_scan = o_kept + align_up((nt + 1) * 8);
  const size_t o_agg = (16 + nb * 4 + 15) / 16 * 16, scan_bytes = o_agg + 2 * nb * 8;
  void *blk = nullptr;
  CK(cudaMallocAsync(&blk, o_scan + 2 * scan_bytes, s));
  uint8_t *b = (uint8_t *)blk;
  unsigned long long *lines = (unsigned long long *)(b + o_lines), *kept = (unsigned long long *)(b + o_kept);
  uint8_t *sc0 = b + o_scan, *sc1 = b + o_scan + scan_bytes;
  if (!rc && cudaMemsetAsync(sc0, 0, 2 * scan_bytes, s) != cudaSuccess) rc = PARPA_ECUDA;
  const unsigned grid = (unsigned)std::min<uint64_t>((uint64_t)dc->sms * 8, (nt + 7) / 8);
  const unsigned long long *skip = (const unsigned long long *)d_skip_rows;
  if (!rc) {
    k_rows_count<<<grid, 256, 0, s>>>(d_in, len, nt, lines);
    k_scan_u64<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(lines, nt, (unsigned int *)sc0, (uint32_t *)(sc0 + 16),
                                                      (unsigned long long *)(sc0 + o_agg),
                                                      (unsigned long long *)(sc0 + o_agg + nb * 8));
    k_rows_keep<false><<<grid, 256, 0, s>>>(d_in, len, nt, lines, skip, nskip, kept, nullptr, nullptr);
    k_scan_u64<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(kept, nt, (unsigned int *)sc1, (uint32_t *)(sc1 + 16),
                                                      (unsigned long long *)(sc1 + o_agg),
                                                      (unsigned long long *)(sc1 + o_agg + nb * 8));
    k_rows_keep<true><<<grid, 256, 0, s>>>(d_in, len, nt, lines, skip, nskip, nullptr, kept, d_out);
    if (cudaGetLastError() != cudaSuccess) rc = PARPA_ECUDA;
  }
  unsigned long long total = 0;
  if (!rc && cudaMemcpyAsync(&total, kept + nt, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess) rc = PARPA_ECUDA;
  cudaFreeAsync(blk, s);
  if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = PARPA_ECUDA;
  if (!rc) *out_len = total;
  return rc;
}

// ---- debug ----------------------------------------------------------------------------------------
int parpa_debug_masks(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, uint64_t *d_masks, void *stream) {
  if (!dfa || (len && (!d_bytes || !d_masks))) return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  parpa_plan p;
  int rc = plan_scan(dfa, d_bytes, len, dfa->start, seg_identity(), 0, 1, s, &p);
  if (!rc && p.w.ntiles &&
      cudaMemcpyAsync(d_masks, p.w.masks, (size_t)p.w.ntiles * 96 * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    rc = PARPA_ECUDA;
  work_free(p.w, s);
  if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = PARPA_ECUDA;
  return rc;
}

int parpa_debug_trace(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, uint8_t *d_chunk_states,
                      uint8_t *d_kinds, uint8_t *d_states, void *stream) {
  if (!dfa || (len && !d_bytes)) return PARPA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  parpa_plan p;
  int rc = plan_scan(dfa, d_bytes, len, dfa->start, seg_identity(), 0, 1, s, &p);
  if (!rc && len) {
    k_debug_trace<<<1024, 128, 0, s>>>(p.a, dfa->k, d_chunk_states, d_kinds, d_states);
    if (cudaGetLastError() != cudaSuccess) rc = PARPA_ECUDA;
  }
  work_free(p.w, s);
  if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = PARPA_ECUDA;
  return rc;
}

}  // extern "C"
