/*
 * parpa_oracle.c — the sequential CPU oracle for the ParPaRaw hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` legs may load this library.  It shares no
 * source, header, table or constant with the CUDA path (paper_1905_13415_b200/):
 * the dialects below are written as explicit control flow and never read the
 * transition/emission tables the GPU consumes.
 *
 * What it computes (§3, "Massively Parallel Parsing"):
 *   P:310  "A sequential approach would simply set the starting state of its DFA and
 *           read the symbols of the input beginning to end" — this file IS that
 *           sequential approach.  Everything the parallel method produces (the three
 *           bitmap indexes P:369-375, record/column offsets P:386-418, the columnar
 *           partition P:439-457 and type conversion P:459-469) is a function of the
 *           per-byte (state, symbol) sequence, so the oracle derives it directly.
 *   Emission per byte is one of DATA / CTRL / FIELD / RECORD (the three bitmaps of
 *   P:371-374 collapsed; RECORD => FIELD => control), decided by the
 *   state BEFORE the byte and the byte (reading R2).
 *   Span of a field = [first DATA byte, last DATA byte] in the raw input (reading R11);
 *   typed value = conversion of the field's DATA bytes (the paper's CSS holds only
 *   non-control symbols).
 *
 * Readings of the paper taken here (all listed in DESIGN.md §Readings):
 *   R1 start state index 0 (EOR); R4 LF only; R5 blank line = one record with one
 *   empty field; R6 per-state end-of-input action; R7 INV => EFORMAT with
 *   first_invalid = first byte entering INV; R11 spans; R12 missing / extra fields;
 *   R14/R15 int64 / float64 grammars (float64 correctly rounded via glibc strtod);
 *   R16 defaults for empty and missing fields; R19 '#' comments only at
 *   record start; R20 Common Log Format grammar.
 *
 * Parity: pinned by tests/test_oracle_*.py (paper fixtures, brute force, Python csv,
 * Python int()/float()).  The CSV+comment and CLF dialects are invented (the paper
 * gives no table for them) — "parity unpinned by the paper"; they are pinned only by
 * hand-written fixtures and by equality with the table walker below.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <errno.h>

enum { K_DATA = 0, K_CTRL = 1, K_FIELD = 2, K_RECORD = 3 };
enum { EOI_NONE = 0, EOI_RECORD = 1, EOI_ERROR = 2 };
enum { T_SPAN = 0, T_INT64 = 1, T_FLOAT64 = 2, T_TIMESTAMP = 3 };
enum { ST_OK = 0, ST_EFORMAT = -4, ST_ECOLUMNS = -5, ST_EUNSUPPORTED = -6 };
enum { D_CSV = 0, D_CSV_COMMENT = 1, D_CLF = 2, D_TABLES = 3 };
#define NONE64 0xFFFFFFFFFFFFFFFFull
#define MISSING_LEN 0xFFFFFFFFu

/* ------------------------------------------------------------------------- */
/* Dialect 1: RFC 4180 CSV, LF only — tab:ttable, six states incl.  */
/* INV.  States in the column order of tab:ttable.                  */
/* ------------------------------------------------------------------------- */
enum { CSV_EOR = 0, CSV_ENC = 1, CSV_FLD = 2, CSV_EOF = 3, CSV_ESC = 4, CSV_INV = 5 };

static int csv_step(int st, uint8_t b, int *kind) {
  switch (st) {
  case CSV_EOR: case CSV_FLD: case CSV_EOF:          /* outside quotes */
    if (b == '\n') { *kind = K_RECORD; return CSV_EOR; }     /* row "\n": EOR EOR EOR */
    if (b == ',')  { *kind = K_FIELD;  return CSV_EOF; }     /* row ",":  EOF EOF EOF */
    if (b == '"') {                                           /* row "\"": ENC INV ENC */
      *kind = K_CTRL;
      return st == CSV_FLD ? CSV_INV : CSV_ENC;               /* quote in FLD is invalid */
    }
    *kind = K_DATA; return CSV_FLD;                           /* row "*":  FLD FLD FLD */
  case CSV_ENC:                                               /* inside quotes: column ENC */
    if (b == '"') { *kind = K_CTRL; return CSV_ESC; }         /* first quote of a pair: control */
    *kind = K_DATA; return CSV_ENC;                           /* , \n * stay enclosed, are data */
  case CSV_ESC:                                               /* after a quote inside quotes */
    if (b == '"')  { *kind = K_DATA;   return CSV_ENC; }      /* "" -> literal quote (reading R3) */
    if (b == ',')  { *kind = K_FIELD;  return CSV_EOF; }
    if (b == '\n') { *kind = K_RECORD; return CSV_EOR; }
    *kind = K_CTRL; return CSV_INV;                           /* "x"y : invalid */
  default:                                                    /* INV is absorbing */
    *kind = K_CTRL; return CSV_INV;
  }
}
static int csv_eoi(int st) {                                  /* reading R6 */
  switch (st) {
  case CSV_EOR: return EOI_NONE;
  case CSV_FLD: case CSV_EOF: case CSV_ESC: return EOI_RECORD;
  default: return EOI_ERROR;                                  /* ENC (unterminated quote), INV */
  }
}

/* ------------------------------------------------------------------------- */
/* Dialect 2: CSV + '#' comment lines (reading R19: '#' opens a comment only at */
/* record start; comment bytes and their terminating '\n' are control). */
/* ------------------------------------------------------------------------- */
enum { CC_EOR = 0, CC_ENC = 1, CC_FLD = 2, CC_EOF = 3, CC_ESC = 4, CC_CMT = 5, CC_INV = 6 };

static int csvc_step(int st, uint8_t b, int *kind) {
  switch (st) {
  case CC_EOR:
    if (b == '#') { *kind = K_CTRL; return CC_CMT; }
    /* fallthrough: otherwise like any other outside-quotes state */
  case CC_FLD: case CC_EOF:
    if (b == '\n') { *kind = K_RECORD; return CC_EOR; }
    if (b == ',')  { *kind = K_FIELD;  return CC_EOF; }
    if (b == '"') { *kind = K_CTRL; return st == CC_FLD ? CC_INV : CC_ENC; }
    *kind = K_DATA; return CC_FLD;                           /* includes '#' inside a field */
  case CC_ENC:
    if (b == '"') { *kind = K_CTRL; return CC_ESC; }
    *kind = K_DATA; return CC_ENC;
  case CC_ESC:
    if (b == '"')  { *kind = K_DATA;   return CC_ENC; }
    if (b == ',')  { *kind = K_FIELD;  return CC_EOF; }
    if (b == '\n') { *kind = K_RECORD; return CC_EOR; }
    *kind = K_CTRL; return CC_INV;
  case CC_CMT:
    *kind = K_CTRL;
    return b == '\n' ? CC_EOR : CC_CMT;                       /* comment ends at its newline */
  default:
    *kind = K_CTRL; return CC_INV;
  }
}
static int csvc_eoi(int st) {
  switch (st) {
  case CC_EOR: case CC_CMT: return EOI_NONE;
  case CC_FLD: case CC_EOF: case CC_ESC: return EOI_RECORD;
  default: return EOI_ERROR;
  }
}

/* ------------------------------------------------------------------------- */
/* Dialect 3: Common Log Format (reading R20; CLF/ELF are the paper's motivating */
/* log formats).  Space delimits fields; "..." and [...] enclose   */
/* (enclosing bytes are control); inside quotes '\' escapes the next byte (both */
/* kept as data, raw); '#' at line start opens a directive/comment line.         */
/* ------------------------------------------------------------------------- */
enum { CL_EOR = 0, CL_FLD = 1, CL_EOF = 2, CL_QUO = 3, CL_QES = 4, CL_CLS = 5,
       CL_BRK = 6, CL_CMT = 7, CL_INV = 8 };

static int clf_step(int st, uint8_t b, int *kind) {
  switch (st) {
  case CL_EOR: case CL_EOF:                 /* at the start of a field */
    if (st == CL_EOR && b == '#') { *kind = K_CTRL; return CL_CMT; }
    if (b == '\n') { *kind = K_RECORD; return CL_EOR; }
    if (b == ' ')  { *kind = K_FIELD;  return CL_EOF; }
    if (b == '"')  { *kind = K_CTRL;   return CL_QUO; }
    if (b == '[')  { *kind = K_CTRL;   return CL_BRK; }
    *kind = K_DATA; return CL_FLD;          /* ] \ # and every other byte start a bare field */
  case CL_FLD:                              /* inside a bare field */
    if (b == '\n') { *kind = K_RECORD; return CL_EOR; }
    if (b == ' ')  { *kind = K_FIELD;  return CL_EOF; }
    *kind = K_DATA; return CL_FLD;
  case CL_QUO:                              /* inside "..." */
    if (b == '"')  { *kind = K_CTRL; return CL_CLS; }
    if (b == '\\') { *kind = K_DATA; return CL_QES; }
    if (b == '\n') { *kind = K_CTRL; return CL_INV; }
    *kind = K_DATA; return CL_QUO;
  case CL_QES:                              /* byte after a backslash inside quotes */
    if (b == '\n') { *kind = K_CTRL; return CL_INV; }
    *kind = K_DATA; return CL_QUO;
  case CL_CLS:                              /* right after a closing quote or bracket */
    if (b == '\n') { *kind = K_RECORD; return CL_EOR; }
    if (b == ' ')  { *kind = K_FIELD;  return CL_EOF; }
    *kind = K_CTRL; return CL_INV;
  case CL_BRK:                              /* inside [...] */
    if (b == ']')  { *kind = K_CTRL; return CL_CLS; }
    if (b == '\n') { *kind = K_CTRL; return CL_INV; }
    *kind = K_DATA; return CL_BRK;
  case CL_CMT:
    *kind = K_CTRL;
    return b == '\n' ? CL_EOR : CL_CMT;
  default:
    *kind = K_CTRL; return CL_INV;
  }
}
static int clf_eoi(int st) {
  switch (st) {
  case CL_EOR: case CL_CMT: return EOI_NONE;
  case CL_FLD: case CL_EOF: case CL_CLS: return EOI_RECORD;
  default: return EOI_ERROR;                /* QUO, QES, BRK (unterminated), INV */
  }
}

/* ------------------------------------------------------------------------- */
/* Generic sequential table walker (used only for random-DFA brute force and to */
/* prove that the tables handed to the GPU encode the dialects above).          */
/* transition / emit are row-per-group [G][S]; emission by SOURCE state. */
/* ------------------------------------------------------------------------- */
typedef struct {
  const uint8_t *group_of_byte;   /* [256] */
  const uint8_t *trans;           /* [G][S] */
  const uint8_t *emit;            /* [G][S] */
  const uint8_t *eoi;             /* [S] */
  uint32_t S, G, start, inv;
} walker;

/* ------------------------------------------------------------------------- */
/* Result container.                                                           */
/* ------------------------------------------------------------------------- */
typedef struct {
  uint32_t C;
  uint64_t R, cap;
  uint64_t **off;
  uint32_t **len;
  int64_t **val;       /* int64 value, or the IEEE-754 bits of the float64 */
  uint8_t **valid;
  uint64_t nfields, first_invalid, n_missing, n_extra;
  int status, final_state, eoi_action;
  /* schema */
  uint8_t *types, *has_def;
  int64_t *def_bits;
  /* open field's DATA bytes */
  uint8_t *fbuf;
  uint64_t fcap, flen;
  /* string capture (the paper's CSS P:439-457): the DATA bytes of every field of one
   * column, concatenated in row order; soff[r] = start of row r (soff[R] = total) */
  int64_t str_col;
  uint8_t *sbuf;
  uint64_t scap, slen, *soff, socap;
} or_result;
static int64_t g_str_col = -1;          /* set by oracle_parse_strings for the duration of one call */
static void *xrealloc(void *p, size_t n);

static void str_row(or_result *r, const uint8_t *b, uint64_t n) {   /* append row R's string */
  if (r->R + 2 > r->socap) {
    r->socap = r->socap ? r->socap * 2 : 1024;
    r->soff = (uint64_t *)xrealloc(r->soff, r->socap * 8);
  }
  r->soff[r->R] = r->slen;
  if (r->slen + n > r->scap) {
    while (r->slen + n > r->scap) r->scap = r->scap ? r->scap * 2 : 4096;
    r->sbuf = (uint8_t *)xrealloc(r->sbuf, r->scap);
  }
  if (n) memcpy(r->sbuf + r->slen, b, n);
  r->slen += n;
}

static void *xrealloc(void *p, size_t n) {
  void *q = realloc(p, n ? n : 1);
  if (!q) abort();
  return q;
}

static void grow_rows(or_result *r) {
  if (r->R < r->cap) return;
  uint64_t nc = r->cap ? r->cap * 2 : 1024;
  for (uint32_t c = 0; c < r->C; c++) {
    r->off[c] = xrealloc(r->off[c], nc * sizeof(uint64_t));
    r->len[c] = xrealloc(r->len[c], nc * sizeof(uint32_t));
    r->val[c] = xrealloc(r->val[c], nc * sizeof(int64_t));
    r->valid[c] = xrealloc(r->valid[c], nc);
  }
  r->cap = nc;
}

/* R14: int64 grammar [+-]?[0-9]+, exact, overflow => invalid. */
static int conv_int64(const uint8_t *s, uint64_t n, int64_t *out) {
  uint64_t i = 0;
  int neg = 0;
  if (n == 0) return 0;
  if (s[0] == '+' || s[0] == '-') { neg = s[0] == '-'; i = 1; }
  if (i == n) return 0;
  uint64_t limit = neg ? 9223372036854775808ull : 9223372036854775807ull;
  uint64_t acc = 0;
  for (; i < n; i++) {
    if (s[i] < '0' || s[i] > '9') return 0;
    uint64_t d = (uint64_t)(s[i] - '0');
    if (acc > (limit - d) / 10) return 0;          /* acc*10 + d > limit */
    acc = acc * 10 + d;
  }
  *out = neg ? (int64_t)(0 - acc) : (int64_t)acc;
  return 1;
}

/* R15: float64 grammar [+-]?([0-9]+(\.[0-9]*)?|\.[0-9]+)([eE][+-]?[0-9]+)?,
 * value = the exact decimal rounded to nearest, ties to even (glibc strtod, "C" locale). */
static int float_grammar(const uint8_t *s, uint64_t n) {
  uint64_t i = 0, nd = 0;
  if (i < n && (s[i] == '+' || s[i] == '-')) i++;
  while (i < n && s[i] >= '0' && s[i] <= '9') { i++; nd++; }
  if (i < n && s[i] == '.') {
    i++;
    while (i < n && s[i] >= '0' && s[i] <= '9') { i++; nd++; }
  }
  if (nd == 0) return 0;
  if (i < n && (s[i] == 'e' || s[i] == 'E')) {
    uint64_t ne = 0;
    i++;
    if (i < n && (s[i] == '+' || s[i] == '-')) i++;
    while (i < n && s[i] >= '0' && s[i] <= '9') { i++; ne++; }
    if (ne == 0) return 0;
  }
  return i == n;
}
static int conv_float64(const uint8_t *s, uint64_t n, int64_t *bits) {
  if (!float_grammar(s, n)) return 0;
  char stackbuf[256];
  char *buf = n < sizeof(stackbuf) ? stackbuf : (char *)xrealloc(NULL, n + 1);
  memcpy(buf, s, n);
  buf[n] = 0;
  errno = 0;
  double v = strtod(buf, NULL);         /* ERANGE (overflow -> +-inf, underflow -> 0/subnormal) is kept */
  if (buf != stackbuf) free(buf);
  memcpy(bits, &v, 8);
  return 1;
}

/* N2 / reading R29: timestamp = int64 seconds since 1970-01-01T00:00:00Z, proleptic Gregorian
 * calendar, no leap seconds.  Accepted shapes, exact lengths only:
 *   ISO  "YYYY-MM-DD HH:MM:SS" (19 bytes; 'T' also accepted between date and time), read as UTC
 *        (the taxi and yelp datetime columns);
 *   CLF  "DD/Mon/YYYY:HH:MM:SS +HHMM" (26 bytes; Mon = Jan..Dec), local time minus the offset
 *        (the Common Log Format %t field).
 * Month 1-12, day 1..days in that month, hour 0-23, minute 0-59, second 0-59, offset hours 0-23 and
 * minutes 0-59; anything else is invalid (null).  Days from the civil date by the textbook
 * era / year-of-era / day-of-year decomposition (400-year cycles of 146097 days). */
static int64_t days_from_civil(int64_t y, int64_t m, int64_t d) {
  y -= m <= 2;
  const int64_t era = (y >= 0 ? y : y - 399) / 400;
  const int64_t yoe = y - era * 400;
  const int64_t doy = (153 * (m > 2 ? m - 3 : m + 9) + 2) / 5 + d - 1;
  const int64_t doe = yoe * 365 + yoe / 4 - yoe / 100 + doy;
  return era * 146097 + doe - 719468;
}
static int is_leap(int64_t y) { return (y % 4 == 0 && y % 100 != 0) || y % 400 == 0; }
static int digits_at(const uint8_t *s, int n, int64_t *v) {
  int64_t a = 0;
  for (int i = 0; i < n; i++) {
    if (s[i] < '0' || s[i] > '9') return 0;
    a = a * 10 + (s[i] - '0');
  }
  *v = a;
  return 1;
}
static int civil_seconds(int64_t Y, int64_t M, int64_t D, int64_t h, int64_t mi, int64_t sec, int64_t *out) {
  static const int mdays[12] = {31, 28, 31, 30, 31, 30, 31, 31, 30, 31, 30, 31};
  if (M < 1 || M > 12 || D < 1) return 0;
  if (D > mdays[M - 1] + (M == 2 && is_leap(Y))) return 0;
  if (h > 23 || mi > 59 || sec > 59) return 0;
  *out = days_from_civil(Y, M, D) * 86400 + h * 3600 + mi * 60 + sec;
  return 1;
}
static int conv_timestamp(const uint8_t *s, uint64_t n, int64_t *out) {
  int64_t Y, M, D, h, mi, sec;
  if (n == 19) {
    if (s[4] != '-' || s[7] != '-' || (s[10] != ' ' && s[10] != 'T') || s[13] != ':' || s[16] != ':') return 0;
    if (!digits_at(s, 4, &Y) || !digits_at(s + 5, 2, &M) || !digits_at(s + 8, 2, &D) || !digits_at(s + 11, 2, &h) ||
        !digits_at(s + 14, 2, &mi) || !digits_at(s + 17, 2, &sec))
      return 0;
    return civil_seconds(Y, M, D, h, mi, sec, out);
  }
  if (n == 26) {
    static const char *mon = "JanFebMarAprMayJunJulAugSepOctNovDec";
    int64_t zh, zm;
    if (s[2] != '/' || s[6] != '/' || s[11] != ':' || s[14] != ':' || s[17] != ':' || s[20] != ' ') return 0;
    if (s[21] != '+' && s[21] != '-') return 0;
    M = 0;
    for (int k = 0; k < 12; k++)
      if (memcmp(s + 3, mon + 3 * k, 3) == 0) M = k + 1;
    if (!M) return 0;
    if (!digits_at(s, 2, &D) || !digits_at(s + 7, 4, &Y) || !digits_at(s + 12, 2, &h) || !digits_at(s + 15, 2, &mi) ||
        !digits_at(s + 18, 2, &sec) || !digits_at(s + 22, 2, &zh) || !digits_at(s + 24, 2, &zm))
      return 0;
    if (zh > 23 || zm > 59) return 0;
    int64_t t;
    if (!civil_seconds(Y, M, D, h, mi, sec, &t)) return 0;
    const int64_t off = zh * 3600 + zm * 60;
    *out = s[21] == '+' ? t - off : t + off;
    return 1;
  }
  return 0;
}

static void close_field(or_result *r, uint32_t c, uint64_t pos, uint64_t first, uint64_t last) {
  r->nfields++;
  if (c >= r->C) { r->n_extra++; r->flen = 0; return; }
  grow_rows(r);
  uint64_t row = r->R;
  uint64_t off, len;
  if (first == NONE64) { off = pos; len = 0; }
  else { off = first; len = last + 1 - first; }
  if (len >= MISSING_LEN) { r->status = ST_EUNSUPPORTED; len = MISSING_LEN - 1; }
  r->off[c][row] = off;
  r->len[c][row] = (uint32_t)len;
  int64_t v = 0;
  int ok = 0;
  if (r->flen == 0) {                                   /* R16: empty -> default or null */
    if (r->types[c] != T_SPAN && r->has_def[c]) { v = r->def_bits[c]; ok = 1; }
  } else if (r->types[c] == T_INT64) {
    ok = conv_int64(r->fbuf, r->flen, &v);
  } else if (r->types[c] == T_FLOAT64) {
    ok = conv_float64(r->fbuf, r->flen, &v);
  } else if (r->types[c] == T_TIMESTAMP) {
    ok = conv_timestamp(r->fbuf, r->flen, &v);
  }
  if (!ok) v = 0;
  r->val[c][row] = v;
  r->valid[c][row] = (uint8_t)(r->types[c] == T_SPAN ? 0 : ok);
  if ((int64_t)c == r->str_col) str_row(r, r->fbuf, r->flen);
  r->flen = 0;
}

static void close_record(or_result *r, uint32_t c_next, uint64_t pos) {
  /* c_next = number of fields this record had.  R12: missing columns are null /
   * default, with span (record-terminating position, 0xFFFFFFFF). */
  if (c_next < r->C) {
    grow_rows(r);
    r->n_missing++;
    for (uint32_t k = c_next; k < r->C; k++) {
      r->off[k][r->R] = pos;
      r->len[k][r->R] = MISSING_LEN;
      int def = r->types[k] != T_SPAN && r->has_def[k];
      r->val[k][r->R] = def ? r->def_bits[k] : 0;
      r->valid[k][r->R] = (uint8_t)def;
      if ((int64_t)k == r->str_col) str_row(r, NULL, 0);       /* missing field: empty string */
    }
  }
  r->R++;
}

/* The sequential parse (SURVEY §8c algorithm).  trace_state[i] = state BEFORE byte i,
 * trace_kind[i] = emission of byte i (debug parity); either may be NULL. */
static or_result *run(int dialect, const walker *w, const uint8_t *in, uint64_t n, uint32_t C,
                      const uint8_t *types, const uint8_t *has_def, const int64_t *def_bits,
                      int strict, uint8_t *trace_state, uint8_t *trace_kind) {
  or_result *r = (or_result *)calloc(1, sizeof(or_result));
  r->C = C;
  r->str_col = g_str_col < (int64_t)C ? g_str_col : -1;
  r->off = calloc(C ? C : 1, sizeof(void *));
  r->len = calloc(C ? C : 1, sizeof(void *));
  r->val = calloc(C ? C : 1, sizeof(void *));
  r->valid = calloc(C ? C : 1, sizeof(void *));
  r->types = calloc(C ? C : 1, 1);
  r->has_def = calloc(C ? C : 1, 1);
  r->def_bits = calloc(C ? C : 1, 8);
  for (uint32_t c = 0; c < C; c++) {
    r->types[c] = types ? types[c] : T_SPAN;
    r->has_def[c] = has_def ? has_def[c] : 0;
    r->def_bits[c] = def_bits ? def_bits[c] : 0;
  }
  r->first_invalid = NONE64;
  int inv = dialect == D_CSV ? CSV_INV : dialect == D_CSV_COMMENT ? CC_INV
          : dialect == D_CLF ? CL_INV : (int)w->inv;
  int st = dialect == D_TABLES ? (int)w->start : 0;          /* R1: start state EOR = 0 */
  uint32_t c = 0;                                           /* column of the open field */
  uint64_t first = NONE64, last = NONE64;                   /* DATA span of the open field */
  for (uint64_t i = 0; i < n; i++) {
    uint8_t b = in[i];
    int kind, nx;
    switch (dialect) {
    case D_CSV: nx = csv_step(st, b, &kind); break;
    case D_CSV_COMMENT: nx = csvc_step(st, b, &kind); break;
    case D_CLF: nx = clf_step(st, b, &kind); break;
    default: {
      uint32_t g = w->group_of_byte[b];
      nx = w->trans[g * w->S + (uint32_t)st];
      kind = w->emit[g * w->S + (uint32_t)st];
    }
    }
    if (trace_state) trace_state[i] = (uint8_t)st;
    if (trace_kind) trace_kind[i] = (uint8_t)kind;
    if (nx == inv && st != inv && r->first_invalid == NONE64) r->first_invalid = i;
    if (kind == K_DATA) {
      if (first == NONE64) first = i;
      last = i;
      if (r->flen == r->fcap) {
        r->fcap = r->fcap ? r->fcap * 2 : 256;
        r->fbuf = xrealloc(r->fbuf, r->fcap);
      }
      r->fbuf[r->flen++] = b;
    } else if (kind == K_FIELD || kind == K_RECORD) {
      close_field(r, c, i, first, last);
      first = last = NONE64;
      c++;
      if (kind == K_RECORD) { close_record(r, c, i); c = 0; }
    }
    st = nx;
  }
  r->final_state = st;
  int act = dialect == D_CSV ? csv_eoi(st) : dialect == D_CSV_COMMENT ? csvc_eoi(st)
          : dialect == D_CLF ? clf_eoi(st) : w->eoi[st];
  r->eoi_action = act;
  if (act == EOI_RECORD) {                                  /* implicit last record delimiter at N */
    close_field(r, c, n, first, last);
    c++;
    close_record(r, c, n);
  }
  if (act == EOI_ERROR || r->first_invalid != NONE64) {
    r->status = ST_EFORMAT;
    if (r->first_invalid == NONE64) r->first_invalid = n;
  } else if (r->status == ST_OK && strict && (r->n_missing || r->n_extra)) {
    r->status = ST_ECOLUMNS;
  }
  free(r->fbuf);
  r->fbuf = NULL;
  return r;
}

/* ------------------------------------------------------------------------- */
/* exported API (loaded by oracle/__init__.py via ctypes)                       */
/* ------------------------------------------------------------------------- */
or_result *oracle_parse(int dialect, const uint8_t *in, uint64_t n, uint32_t C, const uint8_t *types,
                        const uint8_t *has_def, const int64_t *def_bits, int strict,
                        uint8_t *trace_state, uint8_t *trace_kind) {
  return run(dialect, NULL, in, n, C, types, has_def, def_bits, strict, trace_state, trace_kind);
}

or_result *oracle_parse_tables(const uint8_t *group_of_byte, uint32_t S, uint32_t G, const uint8_t *trans,
                               const uint8_t *emit, const uint8_t *eoi, uint32_t start, uint32_t inv,
                               const uint8_t *in, uint64_t n, uint32_t C, const uint8_t *types,
                               const uint8_t *has_def, const int64_t *def_bits, int strict,
                               uint8_t *trace_state, uint8_t *trace_kind) {
  walker w = {group_of_byte, trans, emit, eoi, S, G, start, inv};
  return run(D_TABLES, &w, in, n, C, types, has_def, def_bits, strict, trace_state, trace_kind);
}

/* scalar results: R, nfields, first_invalid, n_missing, n_extra, status, final_state, eoi_action */
void oracle_stats(const or_result *r, uint64_t *out8) {
  out8[0] = r->R;
  out8[1] = r->nfields;
  out8[2] = r->first_invalid;
  out8[3] = r->n_missing;
  out8[4] = r->n_extra;
  out8[5] = (uint64_t)(int64_t)r->status;
  out8[6] = (uint64_t)r->final_state;
  out8[7] = (uint64_t)r->eoi_action;
}

/* copy column c into caller arrays of length >= R (any pointer may be NULL) */
void oracle_column(const or_result *r, uint32_t c, uint64_t *off, uint32_t *len, int64_t *val, uint8_t *valid) {
  if (c >= r->C || r->R == 0) return;
  if (off) memcpy(off, r->off[c], r->R * 8);
  if (len) memcpy(len, r->len[c], r->R * 4);
  if (val) memcpy(val, r->val[c], r->R * 8);
  if (valid) memcpy(valid, r->valid[c], r->R);
}

void oracle_free(or_result *r) {
  if (!r) return;
  for (uint32_t c = 0; c < r->C; c++) {
    free(r->off[c]); free(r->len[c]); free(r->val[c]); free(r->valid[c]);
  }
  free(r->off); free(r->len); free(r->val); free(r->valid);
  free(r->types); free(r->has_def); free(r->def_bits);
  free(r->sbuf); free(r->soff);
  free(r);
}

/* parse with string capture of column str_col (then oracle_strings_size / oracle_strings) */
or_result *oracle_parse_strings(int dialect, const uint8_t *in, uint64_t n, uint32_t C, const uint8_t *types,
                                uint32_t str_col) {
  g_str_col = str_col;
  or_result *r = run(dialect, NULL, in, n, C, types, NULL, NULL, 0, NULL, NULL);
  g_str_col = -1;
  return r;
}
uint64_t oracle_strings_size(const or_result *r) { return r->slen; }
/* offsets[R + 1] (int64) and data[slen] */
void oracle_strings(const or_result *r, int64_t *offsets, uint8_t *data) {
  for (uint64_t i = 0; i < r->R; i++) offsets[i] = (int64_t)r->soff[i];
  offsets[r->R] = (int64_t)r->slen;
  if (r->slen) memcpy(data, r->sbuf, r->slen);
}

/* Conversion routines exposed for the number pins (R14/R15). */
int oracle_conv_int64(const uint8_t *s, uint64_t n, int64_t *out) { return conv_int64(s, n, out); }
int oracle_conv_float64(const uint8_t *s, uint64_t n, int64_t *bits) { return conv_float64(s, n, bits); }
int oracle_conv_timestamp(const uint8_t *s, uint64_t n, int64_t *out) { return conv_timestamp(s, n, out); }
