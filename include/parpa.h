/*
 * parpa.h — C ABI of libparpa, the B200-native (sm_100a) implementation of the data-parallel
 * hot path of ParPaRaw (arXiv 1905.13415, "ParPaRaw: Massively Parallel Parsing of
 * Delimiter-Separated Raw Data").  Citations: P:n = line n of the paper's PAPER.md;
 * DESIGN.md lists the readings R1..R28 taken where the paper is silent.
 *
 * What the library computes (all on the GPU, hand-written CUDA kernels; no CPU fallback):
 *   S1 symbol-group lookup        P:725-731, P:865-884 (tab:twiddling)
 *   S2 multi-state DFA simulation  P:340-347 (one DFA instance per state -> state-transition vector)
 *   S3 composite-operator scan     P:349-364 (exclusive scan with (a∘b)_i = b_{a_i}, identity seed)
 *   S4 delimiter-emitting re-simulation P:368-375 (record / field / control per symbol)
 *   S5 record / column offset scans P:386-414 (POPCNT record counts, abs/rel column operator ⊕)
 *   S6 column partition            P:439-457 (here: field spans scattered column-major)
 *   S7 type conversion             P:459-469 (int64 exact, float64 correctly rounded), defaults
 *   S8 validation                  P:540-543 (invalid transitions, non-accepting end state)
 *
 * Conventions for every function:
 *   - Returns a status (PARPA_OK or a negative PARPA_E*).  Out-parameters are untouched on error.
 *   - "device pointer" = CUDA global memory of the current device; "host pointer" = ordinary
 *     (pinned or pageable) host memory.  Streams are passed as `void *` holding a cudaStream_t
 *     (NULL = legacy default stream).
 *   - Work is enqueued on the given stream.  Functions documented as "synchronous" wait for the
 *     stream before returning.
 *   - A parpa_dfa is immutable after creation and may be shared across threads and streams.
 */
#ifndef PARPA_H
#define PARPA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------------------------- */
enum {
  PARPA_OK = 0,
  PARPA_EINVAL = -1,        /* bad argument / DFA tables violating the validation rules */
  PARPA_ENOMEM = -2,        /* device or host allocation failed */
  PARPA_ECUDA = -3,         /* CUDA runtime error (also: no usable device) */
  PARPA_EFORMAT = -4,       /* input reached the invalid state, or EOI action = error */
  PARPA_ECOLUMNS = -5,      /* strict schema: some record has != C fields */
  PARPA_EUNSUPPORTED = -6,  /* DFA too large for this build, field length >= 2^32-1 */
  PARPA_ENEEDMORE = -7      /* caller capacity too small; the required record count is reported */
};

/* ---- emission kinds, EOI actions, column types ---------------------------------------- */
/* The paper's three bitmap indexes (record delimiter, field delimiter, control)
 * collapse to one 2-bit kind per symbol: RECORD => FIELD => control (reading R2). */
enum { PARPA_DATA = 0, PARPA_CTRL = 1, PARPA_FIELD = 2, PARPA_RECORD = 3 };
/* End-of-input action per final state (reading R6, "non-accepting end state"). */
enum { PARPA_EOI_NONE = 0, PARPA_EOI_RECORD = 1, PARPA_EOI_ERROR = 2 };
/* Column types: SPAN = raw field span only (strings, datetimes); INT64 / FLOAT64 converted. */
enum { PARPA_SPAN = 0, PARPA_INT64 = 1, PARPA_FLOAT64 = 2, PARPA_TIMESTAMP = 3 };

#define PARPA_MISSING_LENGTH 0xFFFFFFFFu   /* length of a missing field (record had fewer fields) */
#define PARPA_NONE 0xFFFFFFFFFFFFFFFFull   /* "no position" */

typedef struct parpa_dfa parpa_dfa;
typedef struct parpa_plan parpa_plan;
typedef struct parpa_result parpa_result;

/* ---- DFA ------------------------------------------------------------------------------- *
 * parpa_create_dfa — compile a parsing DFA ("uses a DFA while parsing"; P:727:
 * "collapse all the transition table's symbols that have identical state transitions into
 * symbol groups"; tab:ttable row-per-group layout).
 *   num_states      |S|, 2..16.  The device works on classes of non-invalid states with identical
 *                   transition and emission rows (states that differ only in their eoi action, such as
 *                   CSV's EOR / EOF, share a class; the exact state is recovered wherever it is reported
 *                   or decides the end-of-input action).  This build runs up to 8 classes (else
 *                   PARPA_EUNSUPPORTED); with at most 4 — CSV — pass 1 composes with one PRMT per byte.
 *   start_state     the sequential parser's starting state (reading R1)
 *   invalid_state   the INV state; must be absorbing: transition[g][inv] == inv for all g,
 *                   and emit[g][inv] == PARPA_CTRL
 *   num_groups      G, 1..16
 *   group_of_byte   host uint8[256]: symbol group of each byte value
 *   transition      host uint8[G][S] row per group: next state from state s on group g
 *   emit            host uint8[G][S] row per group: emission kind of the symbol, by SOURCE state
 *   eoi             host uint8[S]: end-of-input action of each final state
 * On success *out owns a heap object; free it with parpa_destroy_dfa.  Validation failures
 * return PARPA_EINVAL (SPEC S:32-36 invariants).  Synchronous.  When a device is present the DFA's two
 * shared-memory LUT images (96 KB) are also placed in the current device's memory (the kernels copy them
 * instead of building them; on another device, or without one, the kernels build them). */
int parpa_create_dfa(uint32_t num_states, uint32_t start_state, uint32_t invalid_state,
                     uint32_t num_groups, const uint8_t *group_of_byte, const uint8_t *transition,
                     const uint8_t *emit, const uint8_t *eoi, parpa_dfa **out);
void parpa_destroy_dfa(parpa_dfa *dfa);

/* ---- schema ------------------------------------------------------------------------------ *
 * C columns; types[c] in {PARPA_SPAN, PARPA_INT64, PARPA_FLOAT64, PARPA_TIMESTAMP}
 * (PARPA_TIMESTAMP: int64 seconds since 1970-01-01T00:00:00Z of an ISO "YYYY-MM-DD HH:MM:SS" or
 * Common-Log-Format "DD/Mon/YYYY:HH:MM:SS +HHMM" field; DESIGN reading R29); has_default[c] / default_bits[c]
 * give the column default for empty AND missing typed fields (reading R16: without a
 * default such fields are null, valid = 0).  default_bits holds the int64 value or the IEEE-754
 * bits of the double.  strict != 0 turns records with != C fields into PARPA_ECOLUMNS.
 * All arrays are host memory, read during the call only; has_default / default_bits may be NULL. */
typedef struct {
  uint32_t num_columns;
  const uint8_t *types;
  const uint8_t *has_default;
  const int64_t *default_bits;
  uint32_t strict;
} parpa_schema;

/* Column storage (device pointers).  Row r of column c is the field of record r (0-based):
 *   offset[r]  uint64: byte offset of the field's first DATA byte in the input (reading R11;
 *              for an empty field the position of its terminating delimiter or of EOI; for a
 *              missing field the position of the record delimiter that ended the record)
 *   length[r]  uint32: last DATA byte + 1 - offset; 0 if empty; PARPA_MISSING_LENGTH if missing
 *   value[r]   int64 / double (typed columns only; NULL for spans); 0 when invalid
 *   valid[r]   uint8: 1 if value holds a converted or default value (typed columns only)
 * A column whose four pointers are all NULL is skipped: it still counts as a column of
 * the record (missing / extra accounting unchanged) but nothing is converted or written for it. */
typedef struct {
  uint64_t *offset;
  uint32_t *length;
  void *value;
  uint8_t *valid;
} parpa_column;

/* Scalar outcome of a parse. */
typedef struct {
  uint64_t records;           /* R */
  uint64_t fields;            /* number of fields closed (incl. the implicit EOI one) */
  uint64_t first_invalid;     /* byte offset of the first symbol whose transition entered INV, or of
                                 EOI when the end state's action is error; PARPA_NONE if valid */
  uint64_t missing_records;   /* records with fewer than C fields */
  uint64_t extra_fields;      /* fields beyond column C-1 (dropped) */
  uint64_t deferred_fields;   /* typed fields converted by the device tiers (thread, block, grid) */
  int32_t status;             /* PARPA_OK / EFORMAT / ECOLUMNS / EUNSUPPORTED / ENEEDMORE */
  uint32_t final_state;       /* DFA state after the last byte */
  uint32_t block_fields;      /* of deferred_fields: int64 / float64 fields of >= 1 KB without inner control
                                 bytes, converted by one thread block each */
  uint32_t device_fields;     /* of deferred_fields: such fields of >= 256 KB, converted by the whole grid
                                 (device-level collaboration) */
} parpa_stats;

/* ---- one-call parse (library-sized outputs) --------------------------------------------- *
 * parpa_parse — parse len bytes at device pointer d_bytes (input stays caller-owned and must
 * remain valid until the call returns).  Runs the scan kernel (S1-S5, one input read), reads the
 * record count back (one host sync), allocates exact [C][R] column storage owned by the result,
 * then runs the emit kernel (S4-S7, second read), finalize and the deferred-conversion kernel.
 * Synchronous.  Format errors do not fail the call: *out is produced and its stats carry
 * PARPA_EFORMAT (outputs are then unspecified). */
int parpa_parse(const parpa_dfa *dfa, const parpa_schema *schema, const uint8_t *d_bytes,
                uint64_t len, void *stream, parpa_result **out);

/* Accessors of a parpa_result (host-side handles; column pointers are device memory owned by the
 * result and freed by parpa_result_free). */
int parpa_result_stats(const parpa_result *res, parpa_stats *out);
/* the same, field by field: the record count; the status with the first invalid byte offset
 * and the missing-record / extra-field counts (each out-pointer but `status` may be NULL) */
int parpa_result_records(const parpa_result *res, uint64_t *records);
int parpa_result_status(const parpa_result *res, int *status, uint64_t *first_invalid, uint64_t *n_missing_records,
                        uint64_t *n_extra_fields);
int parpa_result_column(const parpa_result *res, uint32_t c, parpa_column *out);
/* copy column c (records rows) into caller device columns `dst` on `stream` (asynchronous) */
int parpa_result_copy_column(const parpa_result *res, uint32_t c, const parpa_column *dst, void *stream);
void parpa_result_free(parpa_result *res);
/* Allocator hook for result-owned buffers (SURVEY §8(b) ownership): alloc(bytes, stream, ctx) returns device
 * memory usable on `stream` (NULL = out of memory -> PARPA_ENOMEM); free(ptr, stream, ctx) releases it.  Both
 * NULL restores the default (cudaMallocAsync / cudaFreeAsync on the parse's stream).  A result keeps the
 * allocator it was created with; the hook is process-wide (mutex-protected).  PARPA_EINVAL if exactly one is
 * NULL.  Workspaces are internal and always stream-ordered cudaMallocAsync. */
typedef void *(*parpa_alloc_fn)(size_t bytes, void *stream, void *ctx);
typedef void (*parpa_free_fn)(void *ptr, void *stream, void *ctx);
int parpa_set_allocator(parpa_alloc_fn alloc, parpa_free_fn free_fn, void *ctx);

/* ---- two-phase parse into caller-owned columns ---------------------------------------- *
 * parpa_plan_create — run the scan kernel over the input and keep its per-tile prefixes
 * (entry state, record/column offsets) in a plan.  Synchronous (one host sync to read R).
 * parpa_plan_records — the number of rows the emit phase will produce.
 * parpa_plan_emit — run emit + finalize + deferred conversion into caller columns (each with
 * room for parpa_plan_records rows); d_stats (device pointer to a parpa_stats, may be NULL) is
 * written on the stream.  Asynchronous.  The input must still be valid.  The plan refers to `dfa`: the DFA
 * must outlive it (destroy the plan first). */
int parpa_plan_create(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, void *stream,
                      parpa_plan **out);
int parpa_plan_records(const parpa_plan *plan, uint64_t *records);
int parpa_plan_emit(parpa_plan *plan, const parpa_schema *schema, const parpa_column *columns,
                    parpa_stats *d_stats, void *stream);
void parpa_plan_destroy(parpa_plan *plan);

/* ---- parse into caller-owned columns without a host round trip (capacity path) ---------- *
 * parpa_parse_into — enqueues the whole parse: pass 1 (S1-S2, warp ∘-scan), the single-pass
 * decoupled look-back scan of warp-tile transition vectors (S3), pass 2 (S4, warp-tile record /
 * column summaries), the look-back scan of those (S5), emission (S6-S7) straight into the
 * caller's columns (capacity rows each), then finalize and deferred conversion (7 launches).  Rows >= capacity are not written; d_stats->status is then PARPA_ENEEDMORE and
 * d_stats->records the number required.  Asynchronous; d_stats is a device pointer (required).
 * gpu_launches (host, may be NULL) receives the number of kernels enqueued. */
int parpa_parse_into(const parpa_dfa *dfa, const parpa_schema *schema, const uint8_t *d_bytes,
                     uint64_t len, const parpa_column *columns, uint64_t capacity,
                     parpa_stats *d_stats, void *stream, uint32_t *gpu_launches);

/* ---- end-to-end from host memory (streaming: the paper's §4.4) ---------------- *
 * parpa_parse_host — h_bytes (host) -> device -> parse -> columns copied back into the caller's
 * host columns (capacity rows each) -> *stats (host).  Synchronous.  Inputs longer than one
 * partition (512 MB, or the byte count in the environment variable PARPA_STREAM_PARTITION) are
 * streamed: partition i+1 is copied in while partition i is parsed and partition i-1's columns are
 * copied out (three streams, double-buffered input), with the context carried between partitions
 * by the staged range plan; results are identical to a single-shot parse.  Pinned host buffers
 * give full PCIe overlap.  Errors as parpa_parse_into; PARPA_ENEEDMORE if capacity is short
 * (stats->records = the number required, the first `capacity` rows are written). */
int parpa_parse_host(const parpa_dfa *dfa, const parpa_schema *schema, const uint8_t *h_bytes,
                     uint64_t len, const parpa_column *h_columns, uint64_t capacity,
                     parpa_stats *stats, void *stream);

/* ---- range summaries: windows and multi-GPU (context carry; reading R27) ----- *
 * A byte range [0, len) at global offset `base` of a larger input is reduced to a summary:
 *   parpa_tau      the range's state-transition vector: tau[i] = state after the range
 *                  when entered in state i (PARPA entries for i >= num_states are 0xFF)
 *   parpa_counts   record / field counts, the abs/rel column offset and the carries of
 *                  the field left open at the range end, for a given entry state
 * parpa_compose_tau(a, b) = a∘b.  parpa_compose_counts(a, b) = a⊕b on every field.
 * parpa_parse_range parses a range given the composed summary of everything before it; a typed
 * field that starts before the range reads its leading bytes from `left_context` (host-visible
 * device pointer to the `left_len` bytes preceding the range; may be NULL / 0). */
typedef struct { uint8_t tau[16]; } parpa_tau;
typedef struct {
  uint64_t records, fields;
  uint64_t open_first, open_last;   /* first / last DATA byte (global offsets) of the open field */
  uint32_t column;                  /* column offset value */
  uint32_t flags;                   /* bit0 abs, bit1 has delimiter, bit2-4 control-byte carries */
  uint64_t first_invalid;
} parpa_counts;
typedef struct {
  uint32_t entry_state;             /* DFA state at the range start */
  uint32_t _pad;
  uint64_t base;                    /* global byte offset of the range start */
  parpa_counts prefix;              /* composed counts of all bytes before the range */
} parpa_context;

int parpa_summarize(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, void *stream,
                    parpa_tau *out);                                  /* synchronous */
int parpa_count(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, uint64_t base,
                uint32_t entry_state, void *stream, parpa_counts *out, parpa_tau *tau_out);
int parpa_compose_tau(const parpa_dfa *dfa, const parpa_tau *a, const parpa_tau *b, parpa_tau *out);
int parpa_compose_counts(const parpa_counts *a, const parpa_counts *b, parpa_counts *out);
/* ---- column-count inference ------------------------------------------------ *
 * parpa_infer_columns — the number of records and the minimum / maximum number of fields per record
 * of the device bytes under the DFA (host outputs; synchronous on `stream`): what a schema's C
 * should be (reading R13 takes C from the schema).  Returns PARPA_EFORMAT (outputs still set for
 * the bytes before the first invalid one is reached) if the input reaches the invalid state. */
int parpa_infer_columns(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, void *stream,
                        uint32_t *min_fields, uint32_t *max_fields, uint64_t *records);

/* ---- type inference ("Type inference", reading R31) --------------- *
 * parpa_infer_types — the type each of the first num_columns columns needs, from the device bytes
 * alone ("threads identify the minimum numerical type being required to back their field value. A
 * subsequent parallel reduction over the minimum type yields the inferred type of a column", P:571-572;
 * extended to temporal types as P:574 allows).  Class of one field's DATA bytes (control bytes
 * dropped): PARPA_CLASS_INT8 / _INT16 / _INT32 / _INT64 for an R14 integer by its range, _FLOAT64 for
 * the R15 grammar (an integer beyond int64 included), _TIMESTAMP for a valid R29 datetime, else
 * _STRING; empty and missing fields have no class.
 *   class_masks  host uint32[num_columns]: OR over the column's fields of (1 << class)
 *   types        host uint8[num_columns]: the resolved type — _EMPTY if no field has a class, _STRING
 *                if any field is a string or timestamps mix with numbers, _TIMESTAMP if all are
 *                timestamps, else the widest numeric class present
 *   records      host, optional: R
 * Parses the input with num_columns span columns (library-owned, freed before returning) and is
 * synchronous on `stream`.  Errors: PARPA_EINVAL (null pointers, num_columns > 64), PARPA_ENOMEM;
 * PARPA_EFORMAT / PARPA_EUNSUPPORTED as the parse reports them (outputs set). */
enum { PARPA_CLASS_EMPTY = 0, PARPA_CLASS_INT8 = 1, PARPA_CLASS_INT16 = 2, PARPA_CLASS_INT32 = 3,
       PARPA_CLASS_INT64 = 4, PARPA_CLASS_FLOAT64 = 5, PARPA_CLASS_TIMESTAMP = 6, PARPA_CLASS_STRING = 7 };
int parpa_infer_types(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, uint32_t num_columns,
                      void *stream, uint32_t *class_masks, uint8_t *types, uint64_t *records);

/* ---- string materialisation (the paper's CSS) ------------------ *
 * For one column of a completed parse of the same device bytes (column->offset / ->length, device
 * arrays of `rows` entries): the DATA bytes of every field — control bytes such as the escaping
 * quote of "" or CLF's brackets and quotes dropped — concatenated in row order, Arrow layout.
 * parpa_strings_size fills d_offsets (device, rows + 1 int64; d_offsets[0] = 0, d_offsets[rows] =
 * total) and *total (host).  parpa_strings_copy then writes the bytes to d_data (device, >= total).
 * Missing fields are empty strings.  Both re-run the scan half to locate DATA bytes and are
 * synchronous on `stream`.  Errors: PARPA_EINVAL on null pointers. */
int parpa_strings_size(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len,
                       const parpa_column *column, uint64_t rows, int64_t *d_offsets, uint64_t *total,
                       void *stream);
int parpa_strings_copy(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len,
                       const parpa_column *column, uint64_t rows, const int64_t *d_offsets,
                       uint8_t *d_data, void *stream);

/* ---- the CSS from a plan, three layouts (alternative tagging modes P:493-502) --------- *
 * The same string materialisation as above, but from a parpa_plan of the same bytes (its chunk masks are
 * reused: no second scan half).  column / rows: a column emitted from this plan (device offset / length).
 * mode PARPA_CSS_ARROW  : d_data = the DATA bytes of every field in row order; d_offsets[r] = start of
 *                         field r, d_offsets[rows] = total.
 * mode PARPA_CSS_INLINE : inline-terminated CSS: each field's bytes followed by `terminator`
 *                         (e.g. 0x1F, unit separator); d_offsets[r] = start of field r, its terminator at
 *                         d_offsets[r + 1] - 1; total = Arrow total + rows.  The terminator must not occur
 *                         in the column's CSS: if it does the copy returns PARPA_EUNSUPPORTED (bytes written).
 * mode PARPA_CSS_VECTOR : vector-delimited CSS: d_data as ARROW, plus d_aux (device, total
 *                         bytes): 1 at the last symbol of every non-empty field, else 0.
 * parpa_plan_strings_size fills d_offsets (rows + 1 int64) and *total; parpa_plan_strings_copy writes d_data
 * (>= total bytes) and, for VECTOR, d_aux.  Both synchronous on `stream`.  Errors: PARPA_EINVAL (null
 * pointers, mode > 2, terminator > 255, VECTOR without d_aux).
 * parpa_css_index — the CSS's index the way the paper builds it: the positions, in order,
 * of every terminator (INLINE: d_data[k] == terminator) or nonzero auxiliary entry (VECTOR: d_aux[k] != 0)
 * among n bytes, written to d_index (device, room for the number of fields); *count = how many.  Stream
 * compaction (per-tile counts, exclusive scan, ordered writes); synchronous.  Errors: PARPA_EINVAL. */
enum { PARPA_CSS_ARROW = 0, PARPA_CSS_INLINE = 1, PARPA_CSS_VECTOR = 2 };
int parpa_plan_strings_size(parpa_plan *plan, const parpa_column *column, uint64_t rows, uint32_t mode,
                            int64_t *d_offsets, uint64_t *total, void *stream);
int parpa_plan_strings_copy(parpa_plan *plan, const parpa_column *column, uint64_t rows, uint32_t mode,
                            uint32_t terminator, const int64_t *d_offsets, uint8_t *d_data, uint8_t *d_aux,
                            void *stream);
int parpa_css_index(uint32_t mode, uint32_t terminator, const uint8_t *d_data, const uint8_t *d_aux, uint64_t n,
                    uint64_t *d_index, uint64_t *count, void *stream);

/* ---- caller-owned workspace (latency: no allocation, memset or host sync per parse) ------------ *
 * parpa_workspace_create allocates (stream-ordered on `stream`) the device workspace of parses of up to max_len
 * bytes (about 0.45 * max_len bytes) and zeroes its control words.  parpa_parse_into_ws is parpa_parse_into
 * using it: nothing is allocated or synchronised, so a CUDA graph of it is a single kernel node for inputs up
 * to 2 MB (the cooperative k_small leaves the control words zeroed for the next parse; larger inputs add one
 * memset).  One parse at a time per workspace (stream order).  d_bytes must be 16-byte aligned.  Errors:
 * PARPA_EINVAL (len > max_len, misaligned input, null pointers), else as parpa_parse_into.
 * parpa_workspace_destroy frees it (synchronous). */
typedef struct parpa_workspace parpa_workspace;
int parpa_workspace_create(uint64_t max_len, void *stream, parpa_workspace **out);
void parpa_workspace_destroy(parpa_workspace *ws);
int parpa_parse_into_ws(parpa_workspace *ws, const parpa_dfa *dfa, const parpa_schema *schema, const uint8_t *d_bytes,
                        uint64_t len, const parpa_column *columns, uint64_t capacity, parpa_stats *d_stats,
                        void *stream, uint32_t *gpu_launches);

/* ---- staged range plan: the same exchange with every pass run once per rank ------------- *
 * parpa_range_begin  runs S1-S3 on the device range [d_bytes, d_bytes+len) at global offset
 *                    `base` and returns the range's transition vector (host *tau_out) — the
 *                    summary the first allgather exchanges.  The plan keeps the device state.
 * parpa_range_count  runs S4-S5 from `entry_state` (the composition of the other ranks' vectors,
 *                    P:361-364) and returns the range's counts (host *out; unseeded, base-relative
 *                    positions are global) — the summary the second allgather exchanges.
 * parpa_range_emit   writes the range's columns given ctx (entry_state as passed to
 *                    parpa_range_count, prefix = ⊕ of the earlier ranks' counts), with the same
 *                    left-context / is_last / capacity semantics as parpa_parse_range.
 *                    Asynchronous; d_stats is a device pointer.
 * Release with parpa_plan_destroy.  Errors: PARPA_EINVAL on a null argument, an entry state out of
 * range or an emit whose entry state differs from the count's. */
int parpa_range_begin(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, uint64_t base,
                      void *stream, parpa_plan **plan, parpa_tau *tau_out);
int parpa_range_count(parpa_plan *plan, uint32_t entry_state, parpa_counts *out);
int parpa_range_emit(parpa_plan *plan, const parpa_schema *schema, const parpa_context *ctx,
                     const uint8_t *left_context, uint64_t left_len, int is_last,
                     const parpa_column *columns, uint64_t capacity, parpa_stats *d_stats,
                     void *stream);

/* ---- the cross-rank halo (the multi-GPU analogue of the paper's partition carry-over) --- *
 * A field whose DATA begins on an earlier rank (its first DATA byte = the composed prefix's open_first
 * < base) needs those bytes to be converted; if control bytes lie inside it, also the DFA state at
 * some earlier position (the device tier re-simulates to drop them).
 * parpa_range_state_at   *state = the DFA state before the byte at global offset `pos` of this range (a
 *                        member of its class, which parses identically),
 *                        for pos - base a multiple of parpa_chunk_bytes() (after parpa_range_count;
 *                        synchronous).  The rank holding the start of a straddling field sends the bytes
 *                        from that chunk boundary on, with this state, to the ranks that need them.
 * parpa_range_emit_halo  parpa_range_emit with `left_state` = the DFA state before left_context[0]
 *                        (PARPA_STATE_UNKNOWN: as parpa_range_emit, where a straddling typed field with
 *                        inner control bytes is PARPA_EUNSUPPORTED).
 * Errors: PARPA_EINVAL (pos not chunk-aligned / outside the range / before the count; a known
 * left_state without left bytes or >= num_states). */
#define PARPA_STATE_UNKNOWN 0xFFFFFFFFu
int parpa_range_state_at(const parpa_plan *plan, uint64_t pos, uint32_t *state);
int parpa_range_emit_halo(parpa_plan *plan, const parpa_schema *schema, const parpa_context *ctx,
                          const uint8_t *left_context, uint64_t left_len, uint32_t left_state, int is_last,
                          const parpa_column *columns, uint64_t capacity, parpa_stats *d_stats,
                          void *stream);

/* ---- skipping records ("PARPA is able to ignore a user-specified set of records and
 * columns") ------------------------------------------------------------------------- *
 * parpa_parse_into_skip — parpa_parse_into that does not write the records whose indices (0-based,
 * over the whole input) are listed in d_skip_records (device uint64[nskip], sorted ascending, unique):
 * record r is written to row r - (number of skipped records before r), stats->records counts the
 * records written.  Columns are skipped by passing NULL pointers (see parpa_column).  Skipped records
 * take no part in the missing-field count; their extra fields are still counted.  Errors as
 * parpa_parse_into; PARPA_EINVAL if nskip > 0 and d_skip_records is NULL. */
int parpa_parse_into_skip(const parpa_dfa *dfa, const parpa_schema *schema, const uint8_t *d_bytes,
                          uint64_t len, const uint64_t *d_skip_records, uint64_t nskip,
                          const parpa_column *columns, uint64_t capacity, parpa_stats *d_stats,
                          void *stream, uint32_t *gpu_launches);

/* parpa_compact_rows — skipping rows ("rows are different from records, as some records may span
 * multiple rows ... PARPA ignores a set of rows by performing an initial parallel pass over the input,
 * pruning symbols of ignored rows (i.e., parallel stream compaction)").  A row is a raw line:
 * the bytes up to and including a '\n' (quoting is not considered), rows numbered from 0.  Copies the
 * bytes of every row not listed in d_skip_rows (device uint64[nskip], sorted ascending, unique) from
 * d_in (device, len bytes) to d_out (device, >= len bytes) in order and sets *out_len (host) to their
 * count; parse d_out afterwards (offsets then refer to the compacted bytes).  Synchronous.  Errors:
 * PARPA_EINVAL on null pointers, PARPA_ENOMEM, PARPA_ECUDA. */
int parpa_compact_rows(const uint8_t *d_in, uint64_t len, const uint64_t *d_skip_rows, uint64_t nskip,
                       uint8_t *d_out, uint64_t *out_len, void *stream);

int parpa_parse_range(const parpa_dfa *dfa, const parpa_schema *schema, const uint8_t *d_bytes,
                      uint64_t len, const parpa_context *ctx, const uint8_t *left_context,
                      uint64_t left_len, int is_last, const parpa_column *columns,
                      uint64_t capacity, parpa_stats *d_stats, void *stream);

/* ---- debug export for parity tests ------------------------------------------------------ *
 * parpa_debug_trace — per-thread-chunk entry states as computed by the scan kernel's S2-S3 path
 * (d_chunk_states: uint8 per chunk of parpa_chunk_bytes() bytes, DFA state numbering), and, if
 * d_kinds / d_states are non-NULL, each byte's emission kind and state-before-byte re-simulated on
 * the GPU from those entry states.  Synchronous. */
int parpa_debug_trace(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len,
                      uint8_t *d_chunk_states, uint8_t *d_kinds, uint8_t *d_states, void *stream);
/* parpa_debug_masks — the emission masks exactly as pass 2 (k_pass2, the production kernel) stores them
 * for the emission kernel: d_masks (device, ceil(len / parpa_tile_bytes()) * 96 uint64) in the layout
 * [warp tile][DATA, DELIM, RECORD][lane], bit i of lane l's word = byte i of chunk (tile * 32 + l).
 * Synchronous.  Errors: PARPA_EINVAL on null pointers. */
int parpa_debug_masks(const parpa_dfa *dfa, const uint8_t *d_bytes, uint64_t len, uint64_t *d_masks,
                      void *stream);
uint32_t parpa_chunk_bytes(void);
uint32_t parpa_tile_bytes(void);   /* bytes per warp tile (the unit of the scans and of emission) */

/* ---- profiling hooks ----------------------------------------------------------------------- *
 * parpa_set_profiling(1) clears the history and starts recording a CUDA event pair around every
 * kernel this thread launches (on the launching stream); parpa_last_kernel_times fills names[i]
 * (static strings) and ms[i] for up to cap recorded launches, oldest first (synchronises on them). */
int parpa_set_profiling(int enable);
int parpa_last_kernel_times(const char **names, float *ms, int cap);

const char *parpa_status_string(int status);
/* text of the last CUDA runtime error seen by this thread ("" if none) */
const char *parpa_last_error(void);
const char *parpa_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PARPA_H */
