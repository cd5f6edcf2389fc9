/*
 * parpa_gen.c — seeded synthetic inputs shaped like the paper's workloads.
 *
 * Shared by the oracle side and the CUDA side as INPUT only: it holds none of the
 * method's arithmetic (no DFA, no scan, no conversion).  Records are generated
 * independently from (seed, record index) with splitmix64, so any record range can
 * be produced on any thread / rank and the byte stream is identical.
 *
 * Workload recipes (after SURVEY §8d):
 *   cfg1  1 MB RFC-4180 CSV, 8 columns (3 int64, 2 float64, 3 string), ~10% quoted
 *         fields with embedded ',' '\n' and "" escapes (BASELINE configs[0]).
 *   taxi  NYC-yellow-taxi-shaped CSV, 18 columns (6 int64, 9 float64, 3 span),
 *         unquoted, ~90 B/record (configs[1], configs[4]).
 *   yelp  yelp-review-shaped CSV, 9 columns all quoted, long multi-line text with
 *         escaped quotes and some UTF-8, mean record ~721 B (configs[2]).
 *   clf   Common Log Format lines with bracketed time, quoted request (\" escapes,
 *         '#' inside), and '#' directive lines (configs[3]).
 * Ground truth (pin G1): record count and the wrapping sum / null count of every
 * int64 column, as printed by the generator.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { G_CFG1 = 0, G_TAXI = 1, G_YELP = 2, G_CLF = 3 };
#define MAX_INT_COLS 8
#define MAX_REC 65536

typedef struct { uint64_t s; } rng_t;

static inline uint64_t next64(rng_t *r) {            /* splitmix64 */
  uint64_t z = (r->s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static inline rng_t rng_for(uint64_t seed, uint64_t rec) {
  rng_t r = {seed * 0xD1B54A32D192ED03ull ^ (rec + 1) * 0x9E3779B97F4A7C15ull};
  next64(&r);
  return r;
}
static inline uint64_t urange(rng_t *r, uint64_t lo, uint64_t hi) {   /* inclusive */
  unsigned __int128 m = (unsigned __int128)next64(r) * (hi - lo + 1);
  return lo + (uint64_t)(m >> 64);
}
static inline double unit(rng_t *r) { return (double)(next64(r) >> 11) * (1.0 / 9007199254740992.0); }
static inline int chance(rng_t *r, double p) { return unit(r) < p; }

typedef struct {
  uint8_t *p;
  int64_t ints[MAX_INT_COLS];     /* int64 values printed in this record (ground truth) */
  uint8_t isnull[MAX_INT_COLS];
  int nint;
} out_t;

static inline void put(out_t *o, char c) { *o->p++ = (uint8_t)c; }
static inline void puts_(out_t *o, const char *s) { while (*s) *o->p++ = (uint8_t)*s++; }
static void put_u64(out_t *o, uint64_t v) {
  char t[24];
  int n = 0;
  do { t[n++] = (char)('0' + v % 10); v /= 10; } while (v);
  while (n) *o->p++ = (uint8_t)t[--n];
}
static void put_i64(out_t *o, int64_t v) {
  if (v < 0) { put(o, '-'); put_u64(o, (uint64_t)0 - (uint64_t)v); }
  else put_u64(o, (uint64_t)v);
}
static void put_pad(out_t *o, uint64_t v, int width) {
  char t[24];
  for (int i = width - 1; i >= 0; i--) { t[i] = (char)('0' + v % 10); v /= 10; }
  for (int i = 0; i < width; i++) put(o, t[i]);
}
static void gt_int(out_t *o, int64_t v, int isnull) {
  o->ints[o->nint] = isnull ? 0 : v;
  o->isnull[o->nint] = (uint8_t)isnull;
  o->nint++;
}
static void put_int_field(out_t *o, int64_t v) { put_i64(o, v); gt_int(o, v, 0); }

/* money-like decimal from an integer count of hundredths; trailing zeros sometimes dropped */
static void put_cents(out_t *o, rng_t *r, int64_t cents) {
  if (cents < 0) { put(o, '-'); cents = -cents; }
  put_u64(o, (uint64_t)(cents / 100));
  int64_t f = cents % 100;
  if (f == 0) {
    if (chance(r, 0.5)) puts_(o, ".0");
  } else if (f % 10 == 0) {
    put(o, '.'); put(o, (char)('0' + f / 10));
    if (chance(r, 0.5)) put(o, '0');
  } else {
    put(o, '.'); put_pad(o, (uint64_t)f, 2);
  }
}

static const char ALNUM[] = "abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ0123456789";
static const char B64[] = "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789-_";

static void put_words(out_t *o, rng_t *r, int len) {   /* ~len chars of lowercase words */
  uint8_t *end = o->p + len;
  while (o->p < end) {
    int wl = (int)urange(r, 1, 9);
    for (int i = 0; i < wl && o->p < end; i++) put(o, (char)('a' + urange(r, 0, 25)));
    if (o->p < end) put(o, ' ');
  }
}

/* a string field; quoted with probability pq, then with embedded ',' '\n' '""' (cfg1) */
static void put_cfg1_string(out_t *o, rng_t *r, int minl, int maxl, int alnum, double pq) {
  if (chance(r, 0.02)) return;                              /* empty field */
  int len = (int)urange(r, (uint64_t)minl, (uint64_t)maxl);
  int quoted = chance(r, pq);
  if (quoted) put(o, '"');
  uint8_t *start = o->p;
  if (alnum) for (int i = 0; i < len; i++) put(o, ALNUM[urange(r, 0, 61)]);
  else put_words(o, r, len);
  if (quoted) {
    int n = (int)(o->p - start);
    const char *ins[3] = {",", "\n", "\"\""};
    double pr[3] = {0.5, 0.3, 0.3};
    for (int k = 0; k < 3; k++) {
      if (!chance(r, pr[k])) continue;
      int at = (int)urange(r, 0, (uint64_t)n);
      int il = (int)strlen(ins[k]);
      memmove(start + at + il, start + at, (size_t)(n - at));
      memcpy(start + at, ins[k], (size_t)il);
      o->p += il;
      n += il;
    }
    put(o, '"');
  }
}

static void gen_cfg1(out_t *o, rng_t *r, uint64_t rec) {
  put_int_field(o, (int64_t)rec);                              /* c0 row id */
  put(o, ',');
  { int64_t v = (int64_t)urange(r, 0, 2000000) - 1000000;      /* c1 int, quoted 5% */
    int q = chance(r, 0.05);
    if (q) put(o, '"');
    put_int_field(o, v);
    if (q) put(o, '"'); }
  put(o, ',');
  { int d = (int)urange(r, 1, 6);                              /* c2 float, 1-6 decimals */
    uint64_t scale = 1; for (int i = 0; i < d; i++) scale *= 10;
    int64_t m = (int64_t)urange(r, 0, 20000 * scale) - (int64_t)(10000 * scale);
    if (m < 0) put(o, '-');
    uint64_t a = (uint64_t)(m < 0 ? -m : m);
    put_u64(o, a / scale); put(o, '.'); put_pad(o, a % scale, d); }
  put(o, ',');
  put_cfg1_string(o, r, 3, 12, 1, 0.27);                       /* c3 alnum */
  put(o, ',');
  { if (chance(r, 0.5)) put(o, '-');                           /* c4 %.3e in [-1, 1] */
    put(o, (char)('1' + urange(r, 0, 8))); put(o, '.'); put_pad(o, urange(r, 0, 999), 3);
    puts_(o, "e-0"); put(o, (char)('1' + urange(r, 0, 4))); }
  put(o, ',');
  put_cfg1_string(o, r, 0, 40, 0, 0.27);                       /* c5 text */
  put(o, ',');
  put_int_field(o, (int64_t)urange(r, 0, 100));                /* c6 int */
  put(o, ',');
  put_cfg1_string(o, r, 0, 60, 0, 0.27);                       /* c7 text */
  put(o, '\n');
}

static void put_datetime(out_t *o, rng_t *r, int y0, int y1) {
  put_u64(o, urange(r, (uint64_t)y0, (uint64_t)y1)); put(o, '-');
  put_pad(o, urange(r, 1, 12), 2); put(o, '-');
  put_pad(o, urange(r, 1, 28), 2); put(o, ' ');
  put_pad(o, urange(r, 0, 23), 2); put(o, ':');
  put_pad(o, urange(r, 0, 59), 2); put(o, ':');
  put_pad(o, urange(r, 0, 59), 2);
}

static void gen_taxi(out_t *o, rng_t *r) {
  put_int_field(o, chance(r, 0.6) ? 1 : 2);                    /* VendorID */
  put(o, ','); put_datetime(o, r, 2019, 2019);                /* pickup */
  put(o, ','); put_datetime(o, r, 2019, 2019);                /* dropoff */
  put(o, ',');
  if (chance(r, 0.01)) gt_int(o, 0, 1);                        /* passenger_count (1% empty) */
  else put_int_field(o, chance(r, 0.7) ? 1 : (int64_t)urange(r, 2, 6));
  put(o, ',');
  { int64_t h = (int64_t)(-log(1.0 - unit(r)) * 300.0);        /* trip_distance ~ Exp(mean 3) */
    put_cents(o, r, h); }
  put(o, ',');
  if (chance(r, 0.01)) gt_int(o, 0, 1);                        /* RatecodeID */
  else { static const int rc[6] = {1, 2, 3, 4, 5, 99};
         put_int_field(o, chance(r, 0.95) ? 1 : rc[urange(r, 1, 5)]); }
  put(o, ','); put(o, chance(r, 0.99) ? 'N' : 'Y');           /* store_and_fwd_flag */
  put(o, ','); put_int_field(o, (int64_t)urange(r, 1, 265));  /* PULocationID */
  put(o, ','); put_int_field(o, (int64_t)urange(r, 1, 265));  /* DOLocationID */
  put(o, ',');
  { uint64_t u = urange(r, 0, 99);                             /* payment_type */
    put_int_field(o, u < 70 ? 1 : u < 95 ? 2 : u < 98 ? 3 : 4); }
  int64_t fare = 250 + (int64_t)(-log(1.0 - unit(r)) * 1200.0);
  static const int64_t extras[5] = {0, 50, 100, 250, 300};
  int64_t extra = extras[urange(r, 0, 4)];
  int64_t mta = chance(r, 0.95) ? 50 : 0;
  int64_t tip = chance(r, 0.3) ? 0 : (int64_t)urange(r, 1, 2000);
  int64_t tolls = chance(r, 0.9) ? 0 : (chance(r, 0.5) ? 576 : 612);
  int64_t impr = 30;
  int64_t cong = chance(r, 0.8) ? 250 : 0;
  int64_t total = fare + extra + mta + tip + tolls + impr + cong;
  put(o, ','); put_cents(o, r, fare);
  put(o, ','); put_cents(o, r, extra);
  put(o, ','); put_cents(o, r, mta);
  put(o, ','); put_cents(o, r, tip);
  put(o, ','); put_cents(o, r, tolls);
  put(o, ','); put_cents(o, r, impr);
  put(o, ','); put_cents(o, r, total);
  put(o, ','); put_cents(o, r, cong);
  put(o, '\n');
}

static void put_id22(out_t *o, rng_t *r) {
  put(o, '"');
  for (int i = 0; i < 22; i++) put(o, B64[urange(r, 0, 63)]);
  put(o, '"');
}
static int64_t geometric(rng_t *r, double p) {            /* P(k) = (1-p)^k p */
  int64_t k = 0;
  while (!chance(r, p) && k < 1000) k++;
  return k;
}

static void gen_yelp(out_t *o, rng_t *r) {
  put_id22(o, r); put(o, ',');                                /* review_id */
  put_id22(o, r); put(o, ',');                                /* user_id */
  put_id22(o, r); put(o, ',');                                /* business_id */
  { uint64_t u = urange(r, 0, 99);                             /* stars */
    int64_t s = u < 40 ? 5 : u < 65 ? 4 : u < 77 ? 3 : u < 87 ? 2 : 1;
    put(o, '"'); put_int_field(o, s); put(o, '"'); }
  put(o, ',');
  put(o, '"'); put_int_field(o, geometric(r, 0.5)); put(o, '"'); put(o, ',');   /* useful */
  put(o, '"'); put_int_field(o, geometric(r, 2.0 / 3.0)); put(o, '"'); put(o, ',');  /* funny */
  put(o, '"'); put_int_field(o, geometric(r, 2.0 / 3.0)); put(o, '"'); put(o, ',');  /* cool */
  /* text: lognormal length (sigma 0.8), words with ',' breaks "" and UTF-8 */
  { double z = 0;
    for (int i = 0; i < 12; i++) z += unit(r);
    z -= 6.0;                                                   /* ~N(0,1) (Irwin-Hall) */
    double L = exp(6.09 + 0.8 * z);
    int len = (int)L;
    if (len < 1) len = 1;
    if (len > 20000) len = 20000;
    put(o, '"');
    uint8_t *end = o->p + len;
    while (o->p < end) {
      int wl = (int)urange(r, 1, 10);
      int q = chance(r, 0.01);
      if (q) { put(o, '"'); put(o, '"'); }
      for (int i = 0; i < wl; i++) put(o, (char)('a' + urange(r, 0, 25)));
      if (chance(r, 0.005)) {
        static const char *u8[4] = {"\xC3\xA9", "\xC3\xBC", "\xE2\x82\xAC", "\xF0\x9F\x98\x80"};
        puts_(o, u8[urange(r, 0, 3)]);
      }
      if (q) { put(o, '"'); put(o, '"'); }
      if (chance(r, 0.1)) put(o, ',');
      if (chance(r, 0.02)) { put(o, '\n'); if (chance(r, 0.5)) put(o, '\n'); }
      else put(o, ' ');
    }
    put(o, '"'); }
  put(o, ',');
  put(o, '"'); put_datetime(o, r, 2005, 2019); put(o, '"');    /* date */
  put(o, '\n');
}

static const char *MONTHS[12] = {"Jan", "Feb", "Mar", "Apr", "May", "Jun",
                                 "Jul", "Aug", "Sep", "Oct", "Nov", "Dec"};

static void gen_clf(out_t *o, rng_t *r, uint64_t rec) {
  if (rec == 0) {
    puts_(o, "#Version: 1.0\n");
    puts_(o, "#Fields: host ident authuser [date] \"request\" status bytes\n");
  }
  if (chance(r, 0.001)) puts_(o, "#Remark: rotated [x] \"y\" log, see #Fields\n");
  for (int i = 0; i < 4; i++) {                                /* host */
    put_u64(o, urange(r, 1, 254));
    if (i < 3) put(o, '.');
  }
  puts_(o, " - ");                                            /* ident */
  if (chance(r, 0.9)) put(o, '-');                            /* user */
  else { int n = (int)urange(r, 3, 8); for (int i = 0; i < n; i++) put(o, (char)('a' + urange(r, 0, 25))); }
  puts_(o, " [");                                             /* time */
  put_pad(o, urange(r, 1, 28), 2); put(o, '/'); puts_(o, MONTHS[urange(r, 0, 11)]); put(o, '/');
  put_u64(o, urange(r, 2000, 2019)); put(o, ':');
  put_pad(o, urange(r, 0, 23), 2); put(o, ':'); put_pad(o, urange(r, 0, 59), 2); put(o, ':');
  put_pad(o, urange(r, 0, 59), 2);
  { static const char *zones[5] = {" -0700", " +0000", " +0100", " -0500", " +0530"};
    puts_(o, zones[urange(r, 0, 4)]); }
  puts_(o, "] \"");                                           /* request */
  uint64_t m = urange(r, 0, 99);
  int head = 0;
  if (m < 85) puts_(o, "GET");
  else if (m < 93) puts_(o, "POST");
  else if (m < 97) { puts_(o, "HEAD"); head = 1; }
  else puts_(o, "PUT");
  put(o, ' ');
  int segs = (int)urange(r, 1, 5);
  for (int s = 0; s < segs; s++) {
    put(o, '/');
    int n = (int)urange(r, 1, 10);
    for (int i = 0; i < n; i++) put(o, ALNUM[urange(r, 0, 35) < 26 ? urange(r, 0, 25) : 52 + urange(r, 0, 9)]);
  }
  if (chance(r, 0.3)) { puts_(o, "?id="); put_u64(o, urange(r, 0, 99999)); puts_(o, "&p=1"); }
  if (chance(r, 0.01)) puts_(o, "?q=\\\"x y\\\"");                /* escaped quotes */
  if (chance(r, 0.01)) puts_(o, "#frag");
  put(o, ' ');
  puts_(o, chance(r, 0.5) ? "HTTP/1.0" : "HTTP/1.1");
  puts_(o, "\" ");
  uint64_t su = urange(r, 0, 99);                               /* status */
  int64_t status = su < 80 ? 200 : su < 88 ? 304 : su < 95 ? 404 : su < 98 ? 301 : 500;
  put_int_field(o, status);
  put(o, ' ');
  if (status == 304 || head) { put(o, '-'); gt_int(o, 0, 1); }   /* bytes: '-' -> null */
  else put_int_field(o, (int64_t)urange(r, 0, 50000));
  put(o, '\n');
}

/* one record; returns its length */
static size_t gen_record(int cfg, uint64_t seed, uint64_t rec, uint8_t *buf, out_t *o) {
  rng_t r = rng_for(seed, rec);
  o->p = buf;
  o->nint = 0;
  switch (cfg) {
  case G_CFG1: gen_cfg1(o, &r, rec); break;
  case G_TAXI: gen_taxi(o, &r); break;
  case G_YELP: gen_yelp(o, &r); break;
  default: gen_clf(o, &r, rec); break;
  }
  return (size_t)(o->p - buf);
}

/* ------------------------------------------------------------------------- */
typedef struct {
  int cfg;
  uint64_t seed, r0, nrec;
  uint8_t *buf;
  size_t cap, used;
  uint32_t *ends;              /* end offset of each record in buf */
  int64_t *ints;               /* [nrec][MAX_INT_COLS] */
  uint8_t *nulls;
} job_t;

static void *worker(void *arg) {
  job_t *j = (job_t *)arg;
  out_t o;
  j->used = 0;
  for (uint64_t k = 0; k < j->nrec; k++) {
    if (j->cap - j->used < MAX_REC) {
      j->cap = j->cap * 2 + MAX_REC;
      j->buf = (uint8_t *)realloc(j->buf, j->cap);
    }
    size_t n = gen_record(j->cfg, j->seed, j->r0 + k, j->buf + j->used, &o);
    j->used += n;
    j->ends[k] = (uint32_t)j->used;
    memcpy(j->ints + k * MAX_INT_COLS, o.ints, sizeof(o.ints));
    memcpy(j->nulls + k * MAX_INT_COLS, o.isnull, sizeof(o.isnull));
  }
  return NULL;
}

/*
 * Generate records r0, r0+1, ... into out[0..target) and stop at the last complete record
 * that fits (or after max_records).  Returns N; *R_out = records written;
 * gt_out[0..MAX_INT_COLS) = wrapping int64 sums, gt_out[MAX_INT_COLS..2*MAX_INT_COLS) = null counts.
 */
uint64_t gen_fill(int cfg, uint64_t seed, uint64_t r0, uint64_t target, uint64_t max_records,
                  uint8_t *out, int nthreads, uint64_t *R_out, int64_t *gt_out) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  const uint64_t B = 8192;
  job_t jobs[256];
  pthread_t th[256];
  memset(jobs, 0, sizeof(jobs));
  for (int t = 0; t < nthreads; t++) {
    jobs[t].ends = (uint32_t *)malloc(B * sizeof(uint32_t));
    jobs[t].ints = (int64_t *)malloc(B * MAX_INT_COLS * sizeof(int64_t));
    jobs[t].nulls = (uint8_t *)malloc(B * MAX_INT_COLS);
  }
  uint64_t pos = 0, R = 0, rec = r0;
  int64_t sums[MAX_INT_COLS] = {0}, nul[MAX_INT_COLS] = {0};
  int done = 0;
  while (!done) {
    for (int t = 0; t < nthreads; t++) {
      jobs[t].cfg = cfg; jobs[t].seed = seed; jobs[t].r0 = rec + (uint64_t)t * B; jobs[t].nrec = B;
      pthread_create(&th[t], NULL, worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    for (int t = 0; t < nthreads && !done; t++) {
      job_t *j = &jobs[t];
      uint64_t take = 0, bytes = 0;
      for (uint64_t k = 0; k < j->nrec; k++) {
        if (pos + j->ends[k] > target || R + k >= max_records) { done = 1; break; }
        take = k + 1;
        bytes = j->ends[k];
      }
      memcpy(out + pos, j->buf, bytes);
      for (uint64_t k = 0; k < take; k++)
        for (int c = 0; c < MAX_INT_COLS; c++) {
          sums[c] = (int64_t)((uint64_t)sums[c] + (uint64_t)j->ints[k * MAX_INT_COLS + c]);
          nul[c] += j->nulls[k * MAX_INT_COLS + c];
        }
      pos += bytes;
      R += take;
    }
    rec += (uint64_t)nthreads * B;
  }
  for (int t = 0; t < nthreads; t++) {
    free(jobs[t].buf); free(jobs[t].ends); free(jobs[t].ints); free(jobs[t].nulls);
  }
  if (R_out) *R_out = R;
  if (gt_out) for (int c = 0; c < MAX_INT_COLS; c++) { gt_out[c] = sums[c]; gt_out[MAX_INT_COLS + c] = nul[c]; }
  return pos;
}

/* one record (for tests): returns length written to buf (cap >= 65536) */
uint64_t gen_one(int cfg, uint64_t seed, uint64_t rec, uint8_t *buf) {
  out_t o;
  return gen_record(cfg, seed, rec, buf, &o);
}
