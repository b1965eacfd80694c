/*
 * husky_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU oracle for the Huskysort hot path
 * (Hillyard et al., arXiv 2012.00866).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2012_00866_b200/) never links, imports or executes it,
 * and this file shares no code, header, table or constant generator with it.
 *
 * Citations are "PAPER.md:<lines> (<section/algorithm>)" into the paper text.
 *
 * What it computes:
 *   1. encode  : a line-by-line transcription of Alg. 4 "stringToLong"
 *                 with the section-4.3 constants
 *                (PAPER.md:486-494), asciiToLong,
 *                unicodeToLong = stringToLong(...) >>> 1,
 *                and Alg. 3's `perfect` flag.
 *   2. sort    : Huskysort's end result is a full sort of xs (Alg. 1 last line
 *                "Arrays.sort(xs)").  The plain definition is
 *                a stable sort of indices under cmp(i,j): code units compared
 *                position by position as unsigned; a proper prefix sorts first;
 *                equal strings are ordered by original index (DESIGN.md reading
 *                R7, north_star "ties broken by original index").  Implemented
 *                as a textbook top-down merge sort.
 *   3. verify  : a linear uniqueness verifier (perm is a bijection and every
 *                adjacent pair is strictly increasing under cmp).  Because cmp
 *                is a strict total order, the sorted arrangement is unique, so
 *                verify(perm)==0  <=>  perm equals the merge-sort result.
 *   4. alg1    : a paper-literal cross-check for small n: encode -> introsort
 *                of (code, element) with co-swap
 *                -> full insertion-sort cleanup with cmp.
 *
 * Every function here is "pinned" by tests/test_oracle_pins.py against values
 * the paper / SPEC state, closed forms, brute force over all pairs on tiny
 * alphabets, and Python's library sort.  Nothing is parity-unpinned.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_CODER_ASCII 0
#define ORACLE_CODER_UNICODE 1
#define ORACLE_CODER_ENGLISH5 2
#define ORACLE_CODER_ENGLISH6 3

/* PAPER.md:486-494 (section 4.3, "Constants") */
#define BITS_LONG 64
#define BIT_WIDTH_UNICODE 16
#define MAX_LENGTH_UNICODE (BITS_LONG / BIT_WIDTH_UNICODE) /* 4 */
#define MASK_SHORT 0xFFFF
#define MASK_UNICODE MASK_SHORT
#define BIT_WIDTH_ASCII 7
#define MAX_LENGTH_ASCII (BITS_LONG / BIT_WIDTH_ASCII) /* 9 */
#define MASK_ASCII 0x7F
/* PAPER.md:218-219 (section 3.2): "5-bit ASCII, words of 12 (or fewer)
 * characters" and "case-dependent strings (6-bit ASCII) ... 10 characters or
 * less".  The paper prints only these capacities; width/length/mask follow the
 * section-4.3 pattern (MAX_LENGTH = 64 / BIT_WIDTH, mask = 2^BIT_WIDTH - 1),
 * as SPEC.md:224-240 concretises them (reading R15). */
#define BIT_WIDTH_ENGLISH5 5
#define MAX_LENGTH_ENGLISH5 (BITS_LONG / BIT_WIDTH_ENGLISH5) /* 12 */
#define MASK_ENGLISH5 0x1F
#define BIT_WIDTH_ENGLISH6 6
#define MAX_LENGTH_ENGLISH6 (BITS_LONG / BIT_WIDTH_ENGLISH6) /* 10 */
#define MASK_ENGLISH6 0x3F

static int byte_coder(int coder) { return coder != ORACLE_CODER_UNICODE; }
static int known_coder(int coder) { return coder >= ORACLE_CODER_ASCII && coder <= ORACLE_CODER_ENGLISH6; }

/* unit i of string s: u8 for the byte coders (ASCII, ENGLISH5/6), u16 for
 * UNICODE (reading R8: Java Strings are UTF-16 code units). */
static uint32_t unit_at(int coder, const void *units, int64_t pos) {
  if (byte_coder(coder)) return ((const uint8_t *)units)[pos];
  return ((const uint16_t *)units)[pos];
}

/* Alg. 4 "stringToLong", transcribed step by step.
 * str = units[start .. start+len).  Java's long shift masks its count to 6 bits
 * (reading R2); the only case where the count reaches 64 is the empty UNICODE
 * string, where result is 0 either way. */
static uint64_t string_to_long(int coder, const void *units, int64_t start, int64_t len,
                               int maxLength, int bitWidth, uint32_t mask) {
  int64_t length = len < maxLength ? len : maxLength; /* length = Math.min(str.length(), maxLength) */
  int64_t padding = maxLength - length;               /* padding = maxLength - length */
  uint64_t result = 0;                                /* result = 0 */
  if (mask == 0) {
    for (int64_t i = 0; i < length; i++) /* for i = 0 to length (exclusive, reading R3) */
      result = (result << bitWidth) | (uint64_t)unit_at(coder, units, start + i);
  } else {
    for (int64_t i = 0; i < length; i++)
      result = (result << bitWidth) | (uint64_t)(unit_at(coder, units, start + i) & mask);
  }
  result = result << ((bitWidth * padding) & 63); /* result = result << bitWidth * padding */
  return result;
}

/* asciiToLong */
static uint64_t ascii_to_long(const void *units, int64_t start, int64_t len) {
  return string_to_long(ORACLE_CODER_ASCII, units, start, len, MAX_LENGTH_ASCII,
                        BIT_WIDTH_ASCII, MASK_ASCII);
}

/* unicodeToLong: ">>> 1" is a logical shift. */
static uint64_t unicode_to_long(const void *units, int64_t start, int64_t len) {
  return string_to_long(ORACLE_CODER_UNICODE, units, start, len, MAX_LENGTH_UNICODE,
                        BIT_WIDTH_UNICODE, MASK_UNICODE) >> 1;
}

/* englishToLong: 5-bit letters, case folded by the mask */
static uint64_t english5_to_long(const void *units, int64_t start, int64_t len) {
  return string_to_long(ORACLE_CODER_ENGLISH5, units, start, len, MAX_LENGTH_ENGLISH5,
                        BIT_WIDTH_ENGLISH5, MASK_ENGLISH5);
}

/* case-dependent 6-bit letters */
static uint64_t english6_to_long(const void *units, int64_t start, int64_t len) {
  return string_to_long(ORACLE_CODER_ENGLISH6, units, start, len, MAX_LENGTH_ENGLISH6,
                        BIT_WIDTH_ENGLISH6, MASK_ENGLISH6);
}

/* perfectForLength: ASCII is exact up to MAX_LENGTH_ASCII = 9 chars;
 * UNICODE keeps only "the first 3 15/16ths characters" => 3
 * (reading R4); ENGLISH5 12 and ENGLISH6 10 characters. */
static int perfect_for_length(int coder, int64_t len) {
  if (coder == ORACLE_CODER_ASCII) return len <= MAX_LENGTH_ASCII;
  if (coder == ORACLE_CODER_ENGLISH5) return len <= MAX_LENGTH_ENGLISH5;
  if (coder == ORACLE_CODER_ENGLISH6) return len <= MAX_LENGTH_ENGLISH6;
  return len <= MAX_LENGTH_UNICODE - 1;
}

/* Alg. 3 "huskyEncode (for character sequence)".
 * Returns 0 on success, 1 on a bad argument. */
int oracle_encode(int coder, const void *units, const int64_t *offsets, uint64_t n,
                  uint64_t *codes, int32_t *perfect) {
  if (!known_coder(coder)) return 1;
  int isPerfect = 1; /* isPerfect = true */
  for (uint64_t i = 0; i < n; i++) {
    int64_t start = offsets[i], len = offsets[i + 1] - offsets[i];
    if (len < 0) return 1;
    if (isPerfect) isPerfect = perfect_for_length(coder, len);
    switch (coder) {
      case ORACLE_CODER_ASCII: codes[i] = ascii_to_long(units, start, len); break;
      case ORACLE_CODER_UNICODE: codes[i] = unicode_to_long(units, start, len); break;
      case ORACLE_CODER_ENGLISH5: codes[i] = english5_to_long(units, start, len); break;
      default: codes[i] = english6_to_long(units, start, len); break;
    }
  }
  if (perfect) *perfect = isPerfect;
  return 0;
}

/* ---------------------------------------------------------------- sort */

typedef struct {
  int coder;
  const void *units;
  const int64_t *offsets;
} ctx_t;

/* cmp(i, j): Java String.compareTo over code units, with the
 * original index as the final tie-break (reading R7).  <0, 0 (only i==j), >0. */
static int cmp_idx(const ctx_t *c, uint32_t i, uint32_t j) {
  int64_t ai = c->offsets[i], al = c->offsets[i + 1] - ai;
  int64_t bj = c->offsets[j], bl = c->offsets[j + 1] - bj;
  int64_t m = al < bl ? al : bl;
  for (int64_t k = 0; k < m; k++) {
    uint32_t ua = unit_at(c->coder, c->units, ai + k);
    uint32_t ub = unit_at(c->coder, c->units, bj + k);
    if (ua != ub) return ua < ub ? -1 : 1;
  }
  if (al != bl) return al < bl ? -1 : 1;
  return i < j ? -1 : (i > j ? 1 : 0);
}

/* textbook top-down merge sort of a[lo, hi) using tmp */
static void merge_sort(const ctx_t *c, uint32_t *a, uint32_t *tmp, uint64_t lo, uint64_t hi) {
  if (hi - lo < 2) return;
  uint64_t mid = lo + (hi - lo) / 2;
  merge_sort(c, a, tmp, lo, mid);
  merge_sort(c, a, tmp, mid, hi);
  uint64_t i = lo, j = mid, k = lo;
  while (i < mid && j < hi) {
    if (cmp_idx(c, a[j], a[i]) < 0) tmp[k++] = a[j++];
    else tmp[k++] = a[i++];
  }
  while (i < mid) tmp[k++] = a[i++];
  while (j < hi) tmp[k++] = a[j++];
  memcpy(a + lo, tmp + lo, (hi - lo) * sizeof(uint32_t));
}

/* perm[r] = original index of the r-th string in sorted order.  0 ok, 1 bad arg, 2 OOM. */
int oracle_sort(int coder, const void *units, const int64_t *offsets, uint64_t n, uint32_t *perm) {
  if (!known_coder(coder)) return 1;
  if (n > 0xFFFFFFFFull) return 1;
  ctx_t c = {coder, units, offsets};
  for (uint64_t i = 0; i < n; i++) perm[i] = (uint32_t)i;
  if (n < 2) return 0;
  uint32_t *tmp = (uint32_t *)malloc(n * sizeof(uint32_t));
  if (!tmp) return 2;
  merge_sort(&c, perm, tmp, 0, n);
  free(tmp);
  return 0;
}

/* T-thread variant of oracle_sort, for the CPU baseline at T = nproc
 * (SURVEY.md 8(d)): the same plain definition, split as T chunk merge sorts
 * (the textbook merge_sort above, one pthread per chunk) followed by rounds of
 * pairwise merges of adjacent chunks with the same cmp.  Merging adjacent,
 * individually sorted chunks with "take the right element only if strictly
 * smaller" is exactly the merge step of merge_sort, so the result equals
 * oracle_sort's (pinned in tests/test_oracle_pins_next.py).  0 ok, 1 bad arg,
 * 2 OOM / thread failure. */
typedef struct {
  const ctx_t *c;
  uint32_t *a, *tmp;
  uint64_t lo, mid, hi;
  int merge_only;
} mt_job_t;

static void merge_runs(const ctx_t *c, uint32_t *a, uint32_t *tmp, uint64_t lo, uint64_t mid, uint64_t hi) {
  uint64_t i = lo, j = mid, k = lo;
  while (i < mid && j < hi) {
    if (cmp_idx(c, a[j], a[i]) < 0) tmp[k++] = a[j++];
    else tmp[k++] = a[i++];
  }
  while (i < mid) tmp[k++] = a[i++];
  while (j < hi) tmp[k++] = a[j++];
  memcpy(a + lo, tmp + lo, (hi - lo) * sizeof(uint32_t));
}

static void *mt_worker(void *arg) {
  mt_job_t *j = (mt_job_t *)arg;
  if (j->merge_only) merge_runs(j->c, j->a, j->tmp, j->lo, j->mid, j->hi);
  else merge_sort(j->c, j->a, j->tmp, j->lo, j->hi);
  return NULL;
}

int oracle_sort_mt(int coder, const void *units, const int64_t *offsets, uint64_t n, uint32_t *perm, int threads) {
  if (!known_coder(coder) || threads < 1 || threads > 1024) return 1;
  if (n > 0xFFFFFFFFull) return 1;
  if (threads == 1 || n < 2 * (uint64_t)threads) return oracle_sort(coder, units, offsets, n, perm);
  ctx_t c = {coder, units, offsets};
  for (uint64_t i = 0; i < n; i++) perm[i] = (uint32_t)i;
  uint32_t *tmp = (uint32_t *)malloc(n * sizeof(uint32_t));
  uint64_t *bound = (uint64_t *)malloc((threads + 1) * sizeof(uint64_t));
  pthread_t *tid = (pthread_t *)malloc(threads * sizeof(pthread_t));
  mt_job_t *jobs = (mt_job_t *)malloc(threads * sizeof(mt_job_t));
  int rc = 0;
  if (!tmp || !bound || !tid || !jobs) { rc = 2; goto out; }
  for (int t = 0; t <= threads; t++) bound[t] = n * (uint64_t)t / (uint64_t)threads;
  int runs = threads;
  for (int t = 0; t < runs; t++) {
    jobs[t] = (mt_job_t){&c, perm, tmp, bound[t], 0, bound[t + 1], 0};
    if (pthread_create(&tid[t], NULL, mt_worker, &jobs[t])) { rc = 2; runs = t; break; }
  }
  for (int t = 0; t < runs; t++) pthread_join(tid[t], NULL);
  if (rc) goto out;
  /* rounds of pairwise merges: runs [bound[2k], bound[2k+1]) + [bound[2k+1], bound[2k+2]) */
  while (runs > 1) {
    int pairs = runs / 2, started = 0;
    for (int k = 0; k < pairs; k++) {
      jobs[k] = (mt_job_t){&c, perm, tmp, bound[2 * k], bound[2 * k + 1], bound[2 * k + 2], 1};
      if (pthread_create(&tid[k], NULL, mt_worker, &jobs[k])) { rc = 2; break; }
      started++;
    }
    for (int k = 0; k < started; k++) pthread_join(tid[k], NULL);
    if (rc) goto out;
    int m = 0;
    for (int k = 0; k < runs; k += 2) bound[m++] = bound[k];
    bound[m] = n;
    runs = m;
  }
out:
  free(tmp);
  free(bound);
  free(tid);
  free(jobs);
  return rc;
}

/* sorted_units = concatenation of strings in perm order; sorted_offsets[0] = 0. */
int oracle_gather(int coder, const void *units, const int64_t *offsets, uint64_t n,
                  const uint32_t *perm, void *sorted_units, int64_t *sorted_offsets) {
  size_t w = byte_coder(coder) ? 1 : 2;
  int64_t pos = 0;
  sorted_offsets[0] = 0;
  for (uint64_t r = 0; r < n; r++) {
    uint32_t i = perm[r];
    int64_t len = offsets[i + 1] - offsets[i];
    memcpy((char *)sorted_units + pos * w, (const char *)units + offsets[i] * w, len * w);
    pos += len;
    sorted_offsets[r + 1] = pos;
  }
  return 0;
}

/* Linear uniqueness verifier.  Returns 0 if perm is a bijection on [0,n) and
 * cmp(perm[r], perm[r+1]) < 0 for every r; 1 if not a bijection; 2 + r (as
 * int64) at the first out-of-order pair r; -1 on OOM. */
int64_t oracle_verify(int coder, const void *units, const int64_t *offsets, uint64_t n,
                      const uint32_t *perm) {
  ctx_t c = {coder, units, offsets};
  uint8_t *seen = (uint8_t *)calloc(n ? n : 1, 1);
  if (!seen) return -1;
  for (uint64_t r = 0; r < n; r++) {
    if (perm[r] >= n || seen[perm[r]]) { free(seen); return 1; }
    seen[perm[r]] = 1;
  }
  free(seen);
  for (uint64_t r = 0; r + 1 < n; r++)
    if (cmp_idx(&c, perm[r], perm[r + 1]) >= 0) return 2 + (int64_t)r;
  return 0;
}

/* ----------------------------------------- Alg. 1, paper-literal (small n) */

static int floor_lg(uint64_t n) {
  int r = -1;
  while (n) { n >>= 1; r++; }
  return r;
}

/* "when elements i, j of longs are exchanged, then elements i, j of xs are
 * also exchanged" */
static void co_swap(int64_t *longs, uint32_t *xs, uint64_t i, uint64_t j) {
  int64_t t = longs[i]; longs[i] = longs[j]; longs[j] = t;
  uint32_t u = xs[i]; xs[i] = xs[j]; xs[j] = u;
}

static void sift_down(int64_t *longs, uint32_t *xs, uint64_t lo, uint64_t root, uint64_t n) {
  for (;;) {
    uint64_t child = 2 * root + 1;
    if (child >= n) return;
    if (child + 1 < n && longs[lo + child + 1] > longs[lo + child]) child++;
    if (longs[lo + root] >= longs[lo + child]) return;
    co_swap(longs, xs, lo + root, lo + child);
    root = child;
  }
}

/* introsort on the Java-signed longs (reading R1) over [lo, hi) */
static void intro_sort(int64_t *longs, uint32_t *xs, uint64_t lo, uint64_t hi, int depth) {
  while (hi - lo > 16) {
    if (depth == 0) { /* heapsort fallback */
      uint64_t n = hi - lo;
      for (uint64_t s = n / 2; s-- > 0;) sift_down(longs, xs, lo, s, n);
      for (uint64_t e = n; e-- > 1;) { co_swap(longs, xs, lo, lo + e); sift_down(longs, xs, lo, 0, e); }
      return;
    }
    depth--;
    /* median of three -> pivot at hi-1, Lomuto partition */
    uint64_t mid = lo + (hi - lo) / 2;
    if (longs[mid] < longs[lo]) co_swap(longs, xs, mid, lo);
    if (longs[hi - 1] < longs[lo]) co_swap(longs, xs, hi - 1, lo);
    if (longs[mid] < longs[hi - 1]) co_swap(longs, xs, mid, hi - 1);
    int64_t pivot = longs[hi - 1];
    uint64_t store = lo;
    for (uint64_t i = lo; i < hi - 1; i++)
      if (longs[i] < pivot) co_swap(longs, xs, i, store++);
    co_swap(longs, xs, store, hi - 1);
    intro_sort(longs, xs, store + 1, hi, depth);
    hi = store;
  }
  for (uint64_t i = lo + 1; i < hi; i++)
    for (uint64_t j = i; j > lo && longs[j] < longs[j - 1]; j--) co_swap(longs, xs, j, j - 1);
}

/* Alg. 1 with the insertion-sort cleanup that section 3.2
 * allows: perm = xs after the full pass.  Returns the number of
 * inversions the cleanup had to remove through *residual (may be NULL). */
int oracle_huskysort_alg1(int coder, const void *units, const int64_t *offsets, uint64_t n,
                          uint32_t *perm, int32_t *perfect, uint64_t *residual) {
  ctx_t c = {coder, units, offsets};
  uint64_t moves = 0;
  for (uint64_t i = 0; i < n; i++) perm[i] = (uint32_t)i;
  if (n < 2) { if (perfect) *perfect = 1; if (residual) *residual = 0; return 0; }
  uint64_t *codes = (uint64_t *)malloc(n * sizeof(uint64_t));
  if (!codes) return 2;
  int32_t isPerfect = 1;
  int rc = oracle_encode(coder, units, offsets, n, codes, &isPerfect); /* coding = huskyEncode(xs) */
  if (rc) { free(codes); return rc; }
  intro_sort((int64_t *)codes, perm, 0, n, 2 * floor_lg(n)); /* Introsort(xs, longs, 0, n, 2*floor_lg(n)) */
  /* "If coding.perfect return" is NOT taken: with NUL units a length-perfect
   * coding is not injective (reading R4), so the cleanup always runs here. */
  for (uint64_t i = 1; i < n; i++) /* insertion-sort cleanup */
    for (uint64_t j = i; j > 0 && cmp_idx(&c, perm[j], perm[j - 1]) < 0; j--) {
      uint32_t t = perm[j]; perm[j] = perm[j - 1]; perm[j - 1] = t;
      moves++;
    }
  free(codes);
  if (perfect) *perfect = isPerfect;
  if (residual) *residual = moves;
  return 0;
}

/* ------------------------------------------------- numeric keys (perfect coding)
 * for a perfect encoding (p = 0) step 3 is skipped, so
 * Huskysort's result is the plain sort of the keys.  The plain definition is a
 * stable sort of indices under the key type's natural order (Java compareTo;
 * SPEC.md:264-275, reading R16), equal keys by original index:
 *   0 uint64 (unsigned), 1 int64 (Long.compare), 2 double (Double.compare:
 *   numeric order; -0.0 < +0.0; every NaN equal to every NaN and above +inf). */
typedef struct {
  int type;
  const uint64_t *keys;
} kctx_t;

static int cmp_double_java(uint64_t a, uint64_t b) {
  double x, y;
  memcpy(&x, &a, 8);
  memcpy(&y, &b, 8);
  if (x < y) return -1;
  if (x > y) return 1;
  /* equal or unordered: Double.compare falls back to doubleToLongBits, which
   * maps every NaN to one canonical NaN */
  int xn = x != x, yn = y != y;
  if (xn || yn) return xn == yn ? 0 : (xn ? 1 : -1);
  int64_t sa = (int64_t)a, sb = (int64_t)b; /* +-0.0: signed bit patterns */
  return sa < sb ? -1 : (sa > sb ? 1 : 0);
}

static int cmp_key(const kctx_t *c, uint32_t i, uint32_t j) {
  uint64_t a = c->keys[i], b = c->keys[j];
  int r;
  if (c->type == 0) r = a < b ? -1 : (a > b ? 1 : 0);
  else if (c->type == 1) r = (int64_t)a < (int64_t)b ? -1 : ((int64_t)a > (int64_t)b ? 1 : 0);
  else r = cmp_double_java(a, b);
  if (r) return r;
  return i < j ? -1 : (i > j ? 1 : 0);
}

static void merge_sort_keys(const kctx_t *c, uint32_t *a, uint32_t *tmp, uint64_t lo, uint64_t hi) {
  if (hi - lo < 2) return;
  uint64_t mid = lo + (hi - lo) / 2;
  merge_sort_keys(c, a, tmp, lo, mid);
  merge_sort_keys(c, a, tmp, mid, hi);
  uint64_t i = lo, j = mid, k = lo;
  while (i < mid && j < hi) {
    if (cmp_key(c, a[j], a[i]) < 0) tmp[k++] = a[j++];
    else tmp[k++] = a[i++];
  }
  while (i < mid) tmp[k++] = a[i++];
  while (j < hi) tmp[k++] = a[j++];
  memcpy(a + lo, tmp + lo, (hi - lo) * sizeof(uint32_t));
}

/* perm[r] = original index of the r-th key.  0 ok, 1 bad arg, 2 OOM. */
int oracle_sort_keys(int type, const uint64_t *keys, uint64_t n, uint32_t *perm) {
  if (type < 0 || type > 2 || n > 0xFFFFFFFFull) return 1;
  kctx_t c = {type, keys};
  for (uint64_t i = 0; i < n; i++) perm[i] = (uint32_t)i;
  if (n < 2) return 0;
  uint32_t *tmp = (uint32_t *)malloc(n * sizeof(uint32_t));
  if (!tmp) return 2;
  merge_sort_keys(&c, perm, tmp, 0, n);
  free(tmp);
  return 0;
}
