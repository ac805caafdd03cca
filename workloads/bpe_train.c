/* bpe_train.c -- WORKLOAD GENERATION ONLY (bench.py / tests): builds the
 * SURVEY.md §8(d) cfg4 table, "continue BPE training from GPT-2's 50k merges
 * on generator text, taking the most frequent adjacent pair each step; when
 * frequencies drop below 2, fill with random training-consistent merges whose
 * byte strings are unique (like tests/helpers.hpp:85-114)".
 *
 * Training runs on the text WITHOUT pre-tokenization (one token sequence per
 * text), so merges cross word boundaries: the adversarial case for the
 * encoder's piece decomposition. Nothing here is product code.
 *
 * Algorithm (standard incremental BPE training):
 *   - the text as a doubly linked token list (positions never move);
 *   - pair -> {count, occurrence list} in an open-addressing map; occurrence
 *     lists are append-only and validated lazily;
 *   - forced phase: the base table's merges in rank order, each applied to all
 *     its occurrences left to right (= BPE encoding of the text by the base
 *     table: the block engine's pass order, block_engine.hpp:286-307);
 *   - training phase: a max-heap of (count, pair) with lazy deletion picks the
 *     most frequent pair (ties: smallest (left, right)); pairs that already are
 *     merges of the table are skipped (add_merge needs unique pairs,
 *     merge_table.hpp:263-269); if left+right's bytes already are a token, the
 *     merge points at that token instead of minting a duplicate (§8d);
 *   - fill phase: random pairs of existing tokens (components predate the
 *     rank, so training-consistent), unique pair and unique bytes.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t key; /* l << 32 | r; UINT64_MAX = empty */
  int32_t count;
  int32_t head; /* occurrence list head (-1 = none) */
  int32_t is_merge;
} PairSlot;

typedef struct {
  PairSlot* s;
  uint64_t cap, used;
} PairMap;

static uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

static int pm_init(PairMap* m, uint64_t cap) {
  m->cap = cap;
  m->used = 0;
  m->s = (PairSlot*)malloc(cap * sizeof(PairSlot));
  if (!m->s) return -1;
  for (uint64_t i = 0; i < cap; ++i) {
    m->s[i].key = UINT64_MAX;
    m->s[i].count = 0;
    m->s[i].head = -1;
    m->s[i].is_merge = 0;
  }
  return 0;
}

static PairSlot* pm_get(PairMap* m, uint64_t key, int create);

static int pm_grow(PairMap* m) {
  PairMap n;
  if (pm_init(&n, m->cap * 2)) return -1;
  for (uint64_t i = 0; i < m->cap; ++i)
    if (m->s[i].key != UINT64_MAX) {
      PairSlot* d = pm_get(&n, m->s[i].key, 1);
      *d = m->s[i];
    }
  free(m->s);
  *m = n;
  return 0;
}

static PairSlot* pm_get(PairMap* m, uint64_t key, int create) {
  if (create && (m->used + 1) * 2 > m->cap && pm_grow(m)) return NULL;
  uint64_t i = mix64(key) & (m->cap - 1);
  for (;;) {
    PairSlot* s = &m->s[i];
    if (s->key == key) return s;
    if (s->key == UINT64_MAX) {
      if (!create) return NULL;
      s->key = key;
      m->used++;
      return s;
    }
    i = (i + 1) & (m->cap - 1);
  }
}

/* Token bytes: a (pointer, length) view per id; new tokens point into the text
 * (every trained token occurs there) or into the fill arena. */
typedef struct {
  const uint8_t** p;
  uint32_t* len;
  uint64_t* h; /* polynomial hash of the bytes */
  uint64_t* pw; /* B^len */
  uint32_t n, cap;
} Toks;

static const uint64_t kB = 0x100000001b3ULL;

static uint64_t pw_of(uint32_t len) {
  uint64_t r = 1, b = kB;
  while (len) {
    if (len & 1) r *= b;
    b *= b;
    len >>= 1;
  }
  return r;
}

typedef struct {
  uint64_t* key; /* bytes hash -> id */
  uint32_t* id;
  uint64_t cap;
} ByteMap;

static int bm_insert(ByteMap* b, uint64_t h, uint32_t id) {
  uint64_t i = mix64(h) & (b->cap - 1);
  while (b->id[i] != UINT32_MAX) i = (i + 1) & (b->cap - 1);
  b->key[i] = h;
  b->id[i] = id;
  return 0;
}

/* id of a token with exactly these bytes (l's bytes then r's), or UINT32_MAX. */
static uint32_t bm_find(const ByteMap* b, const Toks* T, uint64_t h, uint32_t l, uint32_t r) {
  uint64_t i = mix64(h) & (b->cap - 1);
  const uint32_t ll = T->len[l], lr = T->len[r];
  while (b->id[i] != UINT32_MAX) {
    if (b->key[i] == h) {
      const uint32_t c = b->id[i];
      if (T->len[c] == ll + lr && !memcmp(T->p[c], T->p[l], ll) && !memcmp(T->p[c] + ll, T->p[r], lr)) return c;
    }
    i = (i + 1) & (b->cap - 1);
  }
  return UINT32_MAX;
}

typedef struct {
  int32_t count;
  uint64_t key;
} HeapEnt;

typedef struct {
  HeapEnt* a;
  uint64_t n, cap;
} Heap;

static int he_less(HeapEnt x, HeapEnt y) { /* x has lower priority than y */
  if (x.count != y.count) return x.count < y.count;
  return x.key > y.key;
}

static int heap_push(Heap* h, int32_t count, uint64_t key) {
  if (h->n == h->cap) {
    uint64_t nc = h->cap ? h->cap * 2 : 1024;
    HeapEnt* na = (HeapEnt*)realloc(h->a, nc * sizeof(HeapEnt));
    if (!na) return -1;
    h->a = na;
    h->cap = nc;
  }
  uint64_t i = h->n++;
  HeapEnt e = {count, key};
  while (i > 0) {
    uint64_t p = (i - 1) / 2;
    if (!he_less(h->a[p], e)) break;
    h->a[i] = h->a[p];
    i = p;
  }
  h->a[i] = e;
  return 0;
}

static HeapEnt heap_pop(Heap* h) {
  HeapEnt top = h->a[0];
  HeapEnt e = h->a[--h->n];
  uint64_t i = 0;
  for (;;) {
    uint64_t c = 2 * i + 1;
    if (c >= h->n) break;
    if (c + 1 < h->n && he_less(h->a[c], h->a[c + 1])) ++c;
    if (!he_less(e, h->a[c])) break;
    h->a[i] = h->a[c];
    i = c;
  }
  if (h->n) h->a[i] = e;
  return top;
}

typedef struct {
  uint32_t* tok;
  int32_t *nxt, *prv;
  int32_t *occ_pos, *occ_next;
  uint64_t occ_n, occ_cap;
  PairMap pm;
  Heap heap;
  int track; /* push heap entries on count increments (training phase) */
} State;

static int occ_add(State* S, PairSlot* s, int32_t pos) {
  if (S->occ_n == S->occ_cap) {
    uint64_t nc = S->occ_cap * 2;
    int32_t* a = (int32_t*)realloc(S->occ_pos, nc * 4);
    if (!a) return -1;
    S->occ_pos = a;
    a = (int32_t*)realloc(S->occ_next, nc * 4);
    if (!a) return -1;
    S->occ_next = a;
    S->occ_cap = nc;
  }
  S->occ_pos[S->occ_n] = pos;
  S->occ_next[S->occ_n] = s->head;
  s->head = (int32_t)S->occ_n++;
  return 0;
}

static int pair_inc(State* S, uint32_t l, uint32_t r, int32_t pos) {
  const uint64_t key = ((uint64_t)l << 32) | r;
  PairSlot* s = pm_get(&S->pm, key, 1);
  if (!s) return -1;
  s->count++;
  if (occ_add(S, s, pos)) return -1;
  if (S->track && !s->is_merge && s->count >= 2) return heap_push(&S->heap, s->count, key);
  return 0;
}

static void pair_dec(State* S, uint32_t l, uint32_t r) {
  PairSlot* s = pm_get(&S->pm, ((uint64_t)l << 32) | r, 0);
  if (s) s->count--;
}

static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* Applies merge (l, r) -> m to every live occurrence, left to right. */
static int64_t apply_merge(State* S, uint32_t l, uint32_t r, uint32_t m, int32_t** scratch, uint64_t* scap) {
  const uint64_t key = ((uint64_t)l << 32) | r;
  PairSlot* s = pm_get(&S->pm, key, 0);
  if (!s) return 0;
  uint64_t k = 0;
  for (int32_t o = s->head; o >= 0; o = S->occ_next[o]) {
    if (k == *scap) {
      uint64_t nc = *scap ? *scap * 2 : 4096;
      int32_t* na = (int32_t*)realloc(*scratch, nc * 4);
      if (!na) return -1;
      *scratch = na;
      *scap = nc;
    }
    (*scratch)[k++] = S->occ_pos[o];
  }
  s->head = -1; /* the list is consumed; survivors of other pairs re-add */
  qsort(*scratch, k, 4, cmp_i32);
  int64_t done = 0;
  int32_t last = -1;
  for (uint64_t q = 0; q < k; ++q) {
    const int32_t i = (*scratch)[q];
    if (i == last) continue;
    last = i;
    const int32_t j = S->nxt[i];
    if (S->tok[i] != l || j < 0 || S->tok[j] != r) continue; /* stale */
    const int32_t p = S->prv[i], nn = S->nxt[j];
    if (p >= 0) pair_dec(S, S->tok[p], l);
    if (nn >= 0) pair_dec(S, r, S->tok[nn]);
    pair_dec(S, l, r);
    S->tok[i] = m;
    S->tok[j] = UINT32_MAX;
    S->nxt[i] = nn;
    if (nn >= 0) S->prv[nn] = i;
    if (p >= 0 && pair_inc(S, S->tok[p], m, p)) return -1;
    if (nn >= 0 && pair_inc(S, m, S->tok[nn], i)) return -1;
    ++done;
  }
  s = pm_get(&S->pm, key, 0);
  if (s && s->count > 0) { /* self-pair runs: rebuild this pair's list from scratch of survivors */
    for (uint64_t q = 0; q < k; ++q) {
      const int32_t i = (*scratch)[q];
      const int32_t j = S->nxt[i];
      if (S->tok[i] == l && j >= 0 && S->tok[j] == r && occ_add(S, s, i)) return -1;
    }
  }
  return done;
}

static uint64_t splitmix(uint64_t* x) {
  uint64_t z = (*x += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* Returns 0 on success, -1 on allocation failure, -2 on bad input.
 * tok_blob/tok_off: bytes of ids 0..n_tok-1 (dense ids).
 * forced: n_forced rows (l, r, m), applied in order.
 * out_merges: rows (l, r, m) of the NEW merges (trained, then filled).
 * out_blob/out_off: bytes of new token ids n_tok.. (out_off has room for
 *   target_new + 1 entries; out_off[0] = 0).
 * counts[0..3] = trained merges, filled merges, new tokens, last trained
 *   pair count. */
int bbt_train(const uint8_t* text, int64_t n, const uint8_t* tok_blob, const uint64_t* tok_off, int64_t n_tok,
              const uint32_t* forced, int64_t n_forced, int64_t target_new, int64_t fill_allowed, uint64_t seed,
              int32_t max_len, uint32_t* out_merges, uint8_t* out_blob, int64_t blob_cap, uint64_t* out_off,
              int64_t* counts) {
  if (n < 2 || n > INT32_MAX || n_tok < 256) return -2;
  State S;
  memset(&S, 0, sizeof(S));
  const uint64_t max_tok = (uint64_t)n_tok + (uint64_t)target_new;
  Toks T;
  T.cap = (uint32_t)max_tok;
  T.n = (uint32_t)n_tok;
  T.p = (const uint8_t**)malloc(max_tok * sizeof(void*));
  T.len = (uint32_t*)malloc(max_tok * 4);
  T.h = (uint64_t*)malloc(max_tok * 8);
  T.pw = (uint64_t*)malloc(max_tok * 8);
  ByteMap BM;
  BM.cap = 1;
  while (BM.cap < 2 * max_tok + 16) BM.cap <<= 1;
  BM.key = (uint64_t*)malloc(BM.cap * 8);
  BM.id = (uint32_t*)malloc(BM.cap * 4);
  S.tok = (uint32_t*)malloc((uint64_t)n * 4);
  S.nxt = (int32_t*)malloc((uint64_t)n * 4);
  S.prv = (int32_t*)malloc((uint64_t)n * 4);
  S.occ_cap = (uint64_t)n + 1024;
  S.occ_pos = (int32_t*)malloc(S.occ_cap * 4);
  S.occ_next = (int32_t*)malloc(S.occ_cap * 4);
  int32_t* scratch = NULL;
  uint64_t scap = 0;
  int rc = -1;
  uint32_t* byte_tok = NULL;
  if (!T.p || !T.len || !T.h || !T.pw || !BM.key || !BM.id || !S.tok || !S.nxt || !S.prv || !S.occ_pos ||
      !S.occ_next || pm_init(&S.pm, 1u << 22))
    goto out;
  memset(BM.id, 0xFF, BM.cap * 4);
  for (uint32_t t = 0; t < (uint32_t)n_tok; ++t) {
    T.p[t] = tok_blob + tok_off[t];
    T.len[t] = (uint32_t)(tok_off[t + 1] - tok_off[t]);
    uint64_t h = 0;
    for (uint32_t k = 0; k < T.len[t]; ++k) h = h * kB + T.p[t][k] + 1;
    T.h[t] = h;
    T.pw[t] = pw_of(T.len[t]);
    bm_insert(&BM, h, t);
  }
  byte_tok = (uint32_t*)malloc(256 * 4);
  if (!byte_tok) goto out;
  for (int b = 0; b < 256; ++b) byte_tok[b] = UINT32_MAX;
  for (uint32_t t = 0; t < (uint32_t)n_tok; ++t)
    if (T.len[t] == 1) byte_tok[T.p[t][0]] = t;
  for (int64_t i = 0; i < n; ++i) {
    S.tok[i] = byte_tok[text[i]];
    if (S.tok[i] == UINT32_MAX) {
      rc = -2;
      goto out;
    }
    S.nxt[i] = i + 1 < n ? (int32_t)(i + 1) : -1;
    S.prv[i] = (int32_t)i - 1;
  }
  for (int64_t i = 0; i + 1 < n; ++i)
    if (pair_inc(&S, S.tok[i], S.tok[i + 1], (int32_t)i)) goto out;
  /* forced phase */
  for (int64_t k = 0; k < n_forced; ++k) {
    const uint32_t l = forced[3 * k], r = forced[3 * k + 1], m = forced[3 * k + 2];
    PairSlot* s = pm_get(&S.pm, ((uint64_t)l << 32) | r, 1);
    if (!s) goto out;
    s->is_merge = 1;
    if (apply_merge(&S, l, r, m, &scratch, &scap) < 0) goto out;
  }
  /* training phase */
  S.track = 1;
  for (uint64_t i = 0; i < S.pm.cap; ++i) {
    PairSlot* s = &S.pm.s[i];
    if (s->key != UINT64_MAX && !s->is_merge && s->count >= 2 && heap_push(&S.heap, s->count, s->key)) goto out;
  }
  int64_t made = 0, new_tok = 0, last_count = 0;
  uint64_t blob_used = 0;
  out_off[0] = 0;
  while (made < target_new && S.heap.n) {
    HeapEnt e = heap_pop(&S.heap);
    PairSlot* s = pm_get(&S.pm, e.key, 0);
    if (!s || s->is_merge) continue;
    if (s->count != e.count) {
      if (s->count >= 2 && s->count < e.count && heap_push(&S.heap, s->count, e.key)) goto out;
      continue;
    }
    if (s->count < 2) break;
    const uint32_t l = (uint32_t)(e.key >> 32), r = (uint32_t)e.key;
    if (T.len[l] + T.len[r] > (uint32_t)max_len) {
      s->is_merge = 1; /* never pick it again */
      continue;
    }
    const uint64_t h = T.h[l] * T.pw[r] + T.h[r];
    uint32_t m = bm_find(&BM, &T, h, l, r);
    if (m == UINT32_MAX) {
      m = T.n++;
      /* bytes of the new token: the first occurrence in the text */
      int32_t pos = -1;
      for (int32_t o = s->head; o >= 0; o = S.occ_next[o]) {
        const int32_t i = S.occ_pos[o], j = S.nxt[i];
        if (S.tok[i] == l && j >= 0 && S.tok[j] == r) {
          pos = i;
          break;
        }
      }
      if (pos < 0) goto out;
      T.p[m] = text + pos;
      T.len[m] = T.len[l] + T.len[r];
      T.h[m] = h;
      T.pw[m] = T.pw[l] * T.pw[r];
      bm_insert(&BM, h, m);
      if (blob_used + T.len[m] > (uint64_t)blob_cap) goto out;
      memcpy(out_blob + blob_used, T.p[m], T.len[m]);
      blob_used += T.len[m];
      out_off[++new_tok] = blob_used;
    }
    s->is_merge = 1;
    last_count = s->count;
    out_merges[3 * made] = l;
    out_merges[3 * made + 1] = r;
    out_merges[3 * made + 2] = m;
    ++made;
    if (apply_merge(&S, l, r, m, &scratch, &scap) < 0) goto out;
  }
  const int64_t trained = made;
  /* fill phase: random consistent merges over all tokens */
  uint64_t rs = seed;
  int64_t attempts = 0;
  while (fill_allowed && made < target_new && attempts < 50 * target_new) {
    ++attempts;
    const uint32_t l = (uint32_t)(splitmix(&rs) % T.n), r = (uint32_t)(splitmix(&rs) % T.n);
    if (T.len[l] + T.len[r] > (uint32_t)max_len) continue;
    PairSlot* s = pm_get(&S.pm, ((uint64_t)l << 32) | r, 1);
    if (!s) goto out;
    if (s->is_merge) continue;
    const uint64_t h = T.h[l] * T.pw[r] + T.h[r];
    if (bm_find(&BM, &T, h, l, r) != UINT32_MAX) continue; /* unique bytes */
    const uint32_t m = T.n++;
    if (blob_used + T.len[l] + T.len[r] > (uint64_t)blob_cap) goto out;
    memcpy(out_blob + blob_used, T.p[l], T.len[l]);
    memcpy(out_blob + blob_used + T.len[l], T.p[r], T.len[r]);
    T.p[m] = out_blob + blob_used;
    T.len[m] = T.len[l] + T.len[r];
    T.h[m] = h;
    T.pw[m] = T.pw[l] * T.pw[r];
    bm_insert(&BM, h, m);
    blob_used += T.len[m];
    out_off[++new_tok] = blob_used;
    s->is_merge = 1;
    out_merges[3 * made] = l;
    out_merges[3 * made + 1] = r;
    out_merges[3 * made + 2] = m;
    ++made;
  }
  counts[0] = trained;
  counts[1] = made - trained;
  counts[2] = new_tok;
  counts[3] = last_count;
  rc = 0;
out:
  free(byte_tok);
  free(T.p);
  free(T.len);
  free(T.h);
  free(T.pw);
  free(BM.key);
  free(BM.id);
  free(S.tok);
  free(S.nxt);
  free(S.prv);
  free(S.occ_pos);
  free(S.occ_next);
  free(S.pm.s);
  free(S.heap.a);
  free(scratch);
  return rc;
}
