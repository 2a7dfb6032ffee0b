/* oracle/gmask_port.c — TEST INFRASTRUCTURE ONLY.  See gmask_port.h.
 *
 * Plain-C restatement of the reference runtime (/root/reference/proj):
 *   TokenTrie::Build          src/runtime.cpp:18-61
 *   Engine::InitialConfig     src/runtime.cpp:115-121
 *   ConditionMatches/Accepts  src/runtime.cpp:123-136
 *   Engine::FindEdge          src/runtime.cpp:138-146
 *   Engine::Apply/Undo        src/runtime.cpp:148-175
 *   Engine::Step              src/runtime.cpp:177-186
 *   Engine::AllowedTerminals  src/runtime.cpp:188-208 (+ kernels.cpp:12-38)
 *   Engine::WalkTrie/ComputeMask      src/runtime.cpp:261-287
 *   Engine::ComputeMaskNaive  src/runtime.cpp:289-307
 * over the flat automaton exported from `gmask::Dpda` (dpda.hpp:97-124).
 */
#define _POSIX_C_SOURCE 199309L
#include "gmask_port.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

struct gp_automaton {
  int32_t S, initial, accept, E;
  int32_t max_cond;
  int32_t* shift;      /* S*256, dpda.hpp:114-116 */
  int32_t* edge_begin; /* S+1 */
  uint64_t* acc;       /* E*4 */
  uint8_t* dollar;     /* E */
  uint8_t* dynamic;    /* E */
  int32_t* cond_off;   /* E */
  int32_t* cond_len;
  int32_t* push_off;
  int32_t* push_len;
  int32_t* cond;       /* pool, top first */
  int32_t* push;       /* pool, bottom first */
};

typedef struct {
  int32_t token, first_child, next_sibling;
  uint8_t byte;
} gp_node;

struct gp_trie {
  gp_node* nodes;
  int32_t n, cap, num_tokens;
};

/* ------------------------------------------------------------ loading */
typedef struct {
  const uint8_t* p;
  const uint8_t* end;
  int bad;
} rd;

static void rd_bytes(rd* r, void* dst, size_t n) {
  if (r->bad || (size_t)(r->end - r->p) < n) {
    r->bad = 1;
    memset(dst, 0, n);
    return;
  }
  memcpy(dst, r->p, n);
  r->p += n;
}
static int32_t rd_i32(rd* r) { int32_t v; rd_bytes(r, &v, 4); return v; }
static uint64_t rd_u64(rd* r) { uint64_t v; rd_bytes(r, &v, 8); return v; }
static uint8_t rd_u8(rd* r) { uint8_t v; rd_bytes(r, &v, 1); return v; }

gp_automaton* gp_automaton_load(const uint8_t* buf, int64_t n) {
  if (n < 8 || memcmp(buf, "P3DPDA01", 8) != 0) return NULL;
  rd r = {buf + 8, buf + n, 0};
  gp_automaton* a = (gp_automaton*)calloc(1, sizeof(gp_automaton));
  a->S = rd_i32(&r);
  a->initial = rd_i32(&r);
  a->accept = rd_i32(&r);
  (void)rd_u64(&r);
  int32_t tl = rd_i32(&r);
  if (tl < 0 || a->S <= 0) { free(a); return NULL; }
  r.p += tl;
  a->shift = (int32_t*)malloc(sizeof(int32_t) * (size_t)a->S * 256);
  for (int64_t i = 0; i < (int64_t)a->S * 256; ++i) a->shift[i] = rd_i32(&r);
  a->E = rd_i32(&r);
  a->edge_begin = (int32_t*)malloc(sizeof(int32_t) * (size_t)(a->S + 1));
  for (int32_t i = 0; i <= a->S; ++i) a->edge_begin[i] = rd_i32(&r);
  size_t E = (size_t)a->E;
  a->acc = (uint64_t*)malloc(8 * E * 4 + 8);
  a->dollar = (uint8_t*)malloc(E + 1);
  a->dynamic = (uint8_t*)malloc(E + 1);
  a->cond_off = (int32_t*)malloc(4 * E + 4);
  a->cond_len = (int32_t*)malloc(4 * E + 4);
  a->push_off = (int32_t*)malloc(4 * E + 4);
  a->push_len = (int32_t*)malloc(4 * E + 4);
  size_t ccap = 1024, pcap = 1024, nc = 0, np = 0;
  a->cond = (int32_t*)malloc(4 * ccap);
  a->push = (int32_t*)malloc(4 * pcap);
  a->max_cond = 1;
  for (size_t e = 0; e < E && !r.bad; ++e) {
    (void)rd_i32(&r); /* source */
    for (int k = 0; k < 4; ++k) a->acc[e * 4 + k] = rd_u64(&r);
    a->dollar[e] = rd_u8(&r);
    (void)rd_u8(&r); /* origin */
    a->dynamic[e] = rd_u8(&r);
    (void)rd_u8(&r);
    (void)rd_i32(&r); /* target */
    int32_t cl = rd_i32(&r), pl = rd_i32(&r);
    if (cl < 0 || pl < 0) { r.bad = 1; break; }
    while (nc + (size_t)cl > ccap) { ccap *= 2; a->cond = (int32_t*)realloc(a->cond, 4 * ccap); }
    while (np + (size_t)pl > pcap) { pcap *= 2; a->push = (int32_t*)realloc(a->push, 4 * pcap); }
    a->cond_off[e] = (int32_t)nc;
    a->cond_len[e] = cl;
    a->push_off[e] = (int32_t)np;
    a->push_len[e] = pl;
    for (int32_t i = 0; i < cl; ++i) a->cond[nc++] = rd_i32(&r);
    for (int32_t i = 0; i < pl; ++i) a->push[np++] = rd_i32(&r);
    if (cl > a->max_cond) a->max_cond = cl;
  }
  if (r.bad) { gp_automaton_free(a); return NULL; }
  return a;
}

void gp_automaton_free(gp_automaton* a) {
  if (!a) return;
  free(a->shift); free(a->edge_begin); free(a->acc); free(a->dollar); free(a->dynamic);
  free(a->cond_off); free(a->cond_len); free(a->push_off); free(a->push_len);
  free(a->cond); free(a->push); free(a);
}
int32_t gp_num_states(const gp_automaton* a) { return a->S; }
int32_t gp_num_edges(const gp_automaton* a) { return a->E; }

/* ------------------------------------------------------------ trie (runtime.cpp:18-61) */
static int32_t trie_new_node(gp_trie* t, uint8_t b, int32_t next) {
  if (t->n == t->cap) {
    t->cap = t->cap ? t->cap * 2 : 1024;
    t->nodes = (gp_node*)realloc(t->nodes, sizeof(gp_node) * (size_t)t->cap);
  }
  gp_node* nd = &t->nodes[t->n];
  nd->token = -1;
  nd->first_child = -1;
  nd->next_sibling = next;
  nd->byte = b;
  return t->n++;
}

gp_trie* gp_trie_build(const uint8_t* bytes, const int64_t* offs, int32_t n, int* err_kind) {
  gp_trie* t = (gp_trie*)calloc(1, sizeof(gp_trie));
  *err_kind = 0;
  trie_new_node(t, 0, -1); /* root */
  for (int32_t id = 0; id < n; ++id) {
    if (offs[id + 1] <= offs[id]) { *err_kind = 1; gp_trie_free(t); return NULL; }
    int32_t cur = 0;
    for (int64_t i = offs[id]; i < offs[id + 1]; ++i) {
      uint8_t b = bytes[i];
      int32_t prev = -1, child = t->nodes[cur].first_child;
      while (child != -1 && t->nodes[child].byte < b) {
        prev = child;
        child = t->nodes[child].next_sibling;
      }
      if (child == -1 || t->nodes[child].byte != b) {
        int32_t fresh = trie_new_node(t, b, child);
        if (prev == -1) t->nodes[cur].first_child = fresh;
        else t->nodes[prev].next_sibling = fresh;
        child = fresh;
      }
      cur = child;
    }
    if (t->nodes[cur].token != -1) { *err_kind = 2; gp_trie_free(t); return NULL; }
    t->nodes[cur].token = id;
  }
  t->num_tokens = n;
  return t;
}
void gp_trie_free(gp_trie* t) { if (t) { free(t->nodes); free(t); } }
int32_t gp_trie_nodes(const gp_trie* t) { return t->n; }

/* ------------------------------------------------------------ configs */
static void cfg_reserve(gp_config* c, int32_t need) {
  if (need <= c->cap) return;
  int32_t cap = c->cap ? c->cap : 16;
  while (cap < need) cap *= 2;
  c->stack = (int32_t*)realloc(c->stack, sizeof(int32_t) * (size_t)cap);
  c->cap = cap;
}

void gp_config_init(const gp_automaton* a, gp_config* c) {
  cfg_reserve(c, 16);
  c->state = a->initial;
  c->status = GP_ALIVE;
  c->depth = 1;
  c->stack[0] = a->initial;
}

void gp_config_copy(gp_config* dst, const gp_config* src) {
  cfg_reserve(dst, src->depth > 16 ? src->depth : 16);
  memcpy(dst->stack, src->stack, sizeof(int32_t) * (size_t)src->depth);
  dst->depth = src->depth;
  dst->state = src->state;
  dst->status = src->status;
}

void gp_config_free(gp_config* c) { free(c->stack); c->stack = NULL; c->cap = c->depth = 0; }

/* ------------------------------------------------------------ stepping */
/* runtime.cpp:123-131 */
static int cond_matches(const gp_automaton* a, const gp_config* c, int32_t e) {
  int32_t k = a->cond_len[e];
  if (c->depth < k) return 0;
  const int32_t* cond = a->cond + a->cond_off[e];
  for (int32_t i = 0; i < k; ++i) {
    if (c->stack[c->depth - 1 - i] != cond[i]) return 0;
  }
  return 1;
}

/* runtime.cpp:133-136 (terminal 256 = kEndMarker, grammar.hpp:28) */
static int accepts(const gp_automaton* a, int32_t e, int32_t terminal) {
  if (terminal == 256) return a->dollar[e];
  return (int)((a->acc[e * 4 + (terminal >> 6)] >> (terminal & 63)) & 1u);
}

/* runtime.cpp:138-146: first edge in arbitration order; -1 if none. */
static int32_t find_edge(const gp_automaton* a, const gp_config* c, int32_t terminal) {
  for (int32_t e = a->edge_begin[c->state]; e < a->edge_begin[c->state + 1]; ++e) {
    if (!accepts(a, e, terminal)) continue;
    if (!cond_matches(a, c, e)) continue;
    return e;
  }
  return -1;
}

/* runtime.cpp:148-168; returns the number of entries pushed. */
static int32_t apply_edge(const gp_automaton* a, gp_config* c, int32_t e, int32_t terminal) {
  int32_t k = a->cond_len[e];
  int32_t pl = a->push_len[e];
  cfg_reserve(c, c->depth - k + pl + 1);
  c->depth -= k;
  memcpy(c->stack + c->depth, a->push + a->push_off[e], sizeof(int32_t) * (size_t)pl);
  c->depth += pl;
  int32_t pushed = pl;
  if (a->dynamic[e]) {
    int32_t t = a->shift[(size_t)c->stack[c->depth - 1] * 256 + (uint8_t)terminal];
    c->stack[c->depth++] = t;
    ++pushed;
  }
  c->state = c->stack[c->depth - 1];
  if (terminal == 256) c->status = GP_ACCEPTED;
  return pushed;
}

/* runtime.cpp:177-186 */
int gp_step(const gp_automaton* a, gp_config* c, int32_t terminal) {
  if (c->status != GP_ALIVE) return 0;
  int32_t e = find_edge(a, c, terminal);
  if (e < 0) {
    c->status = GP_DEAD;
    return 0;
  }
  apply_edge(a, c, e, terminal);
  return 1;
}

/* runtime.cpp:188-208 with kernels.cpp:12-38: OR of accepted sets (and $)
 * over ALL condition-matching edges of the current state. */
void gp_allowed(const gp_automaton* a, const gp_config* c, uint64_t bytes[4], int* dollar) {
  bytes[0] = bytes[1] = bytes[2] = bytes[3] = 0;
  *dollar = 0;
  if (c->status != GP_ALIVE) return;
  for (int32_t e = a->edge_begin[c->state]; e < a->edge_begin[c->state + 1]; ++e) {
    if (!cond_matches(a, c, e)) continue;
    for (int k = 0; k < 4; ++k) bytes[k] |= a->acc[e * 4 + k];
    if (a->dollar[e]) *dollar = 1;
  }
}

/* ------------------------------------------------------------ masks */
typedef struct {
  const gp_automaton* a;
  const gp_trie* t;
  gp_config cfg;
  uint32_t* words;
} walk_ctx;

/* runtime.cpp:261-278: DFS with in-place Apply/Undo (runtime.cpp:148-175). */
static void walk_trie(walk_ctx* w, int32_t node) {
  const gp_node* nodes = w->t->nodes;
  int32_t token = nodes[node].token;
  if (token != -1) w->words[token >> 5] |= 1u << (token & 31);
  if (nodes[node].first_child == -1) return;
  uint64_t allowed[4];
  int dollar;
  gp_allowed(w->a, &w->cfg, allowed, &dollar);
  int32_t popped[w->a->max_cond > 0 ? w->a->max_cond : 1];
  for (int32_t child = nodes[node].first_child; child != -1; child = nodes[child].next_sibling) {
    uint8_t b = nodes[child].byte;
    if (!((allowed[b >> 6] >> (b & 63)) & 1u)) continue;
    int32_t e = find_edge(w->a, &w->cfg, b);
    if (e < 0) continue; /* unreachable: allowed set is exact */
    int32_t old_state = w->cfg.state, old_status = w->cfg.status;
    int32_t k = w->a->cond_len[e];
    memcpy(popped, w->cfg.stack + w->cfg.depth - k, sizeof(int32_t) * (size_t)k);
    int32_t pushed = apply_edge(w->a, &w->cfg, e, b);
    walk_trie(w, child);
    w->cfg.depth -= pushed;
    memcpy(w->cfg.stack + w->cfg.depth, popped, sizeof(int32_t) * (size_t)k);
    w->cfg.depth += k;
    w->cfg.state = old_state;
    w->cfg.status = old_status;
  }
}

/* runtime.cpp:280-287 */
void gp_mask(const gp_automaton* a, const gp_config* c, const gp_trie* t, uint32_t* words) {
  int32_t nw = (t->num_tokens + 1 + 31) / 32;
  memset(words, 0, sizeof(uint32_t) * (size_t)nw);
  if (c->status != GP_ALIVE) return;
  walk_ctx w = {a, t, {0, 0, 0, 0, NULL}, words};
  gp_config_copy(&w.cfg, c);
  walk_trie(&w, 0);
  uint64_t allowed[4];
  int dollar;
  gp_allowed(a, c, allowed, &dollar);
  if (dollar) words[t->num_tokens >> 5] |= 1u << (t->num_tokens & 31);
  gp_config_free(&w.cfg);
}

/* runtime.cpp:289-307 */
void gp_mask_naive(const gp_automaton* a, const gp_config* c, const uint8_t* bytes,
                   const int64_t* offs, int32_t n, uint32_t* words) {
  int32_t nw = (n + 1 + 31) / 32;
  memset(words, 0, sizeof(uint32_t) * (size_t)nw);
  if (c->status != GP_ALIVE) return;
  gp_config probe = {0, 0, 0, 0, NULL};
  for (int32_t id = 0; id < n; ++id) {
    gp_config_copy(&probe, c);
    int alive = 1;
    for (int64_t i = offs[id]; i < offs[id + 1]; ++i) {
      if (!gp_step(a, &probe, bytes[i])) { alive = 0; break; }
    }
    if (alive) words[id >> 5] |= 1u << (id & 31);
  }
  gp_config_copy(&probe, c);
  if (gp_step(a, &probe, 256)) words[n >> 5] |= 1u << (n & 31);
  gp_config_free(&probe);
}

/* ------------------------------------------------------------ samplers */
static uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t gp_stream_draw(uint64_t seed, uint64_t seq, uint64_t draw) {
  return mix64(mix64(seed ^ (seq * 0xD1B54A32D192ED03ull)) ^ draw);
}

static uint32_t limited(const uint32_t* w, const uint32_t* f, int32_t i, int32_t limit) {
  uint32_t x = w[i] & (f ? f[i] : ~0u);
  if (i == (limit - 1) / 32 && (limit & 31)) x &= (1u << (limit & 31)) - 1u;
  return x;
}

static int32_t count_bits(const uint32_t* w, const uint32_t* f, int32_t limit) {
  int32_t n = 0;
  for (int32_t i = 0; i < (limit + 31) / 32; ++i) n += __builtin_popcount(limited(w, f, i, limit));
  return n;
}

static int32_t select_bit(const uint32_t* w, const uint32_t* f, int32_t limit, uint32_t r) {
  for (int32_t i = 0; i < (limit + 31) / 32; ++i) {
    uint32_t x = limited(w, f, i, limit);
    uint32_t c = (uint32_t)__builtin_popcount(x);
    if (r < c) {
      while (r--) x &= x - 1u;
      return i * 32 + __builtin_ctz(x);
    }
    r -= c;
  }
  return -1;
}

int32_t gp_stream_pick(const uint32_t* mask, const uint32_t* structural, int32_t V, uint64_t u) {
  int32_t n_all = count_bits(mask, NULL, V);
  int eos = (int)((mask[V >> 5] >> (V & 31)) & 1u);
  if (n_all == 0) return eos ? V : -1;
  if (eos && ((u >> 32) & 3u) == 0) return V; /* EOS with probability 1/4 */
  uint32_t lo = (uint32_t)u;
  if ((u >> 34) & 1u) {
    int32_t n_s = structural ? count_bits(mask, structural, V) : 0;
    if (n_s > 0) return select_bit(mask, structural, V, (uint32_t)(((uint64_t)lo * (uint32_t)n_s) >> 32));
  }
  return select_bit(mask, NULL, V, (uint32_t)(((uint64_t)lo * (uint32_t)n_all) >> 32));
}

static uint32_t bf16_key(uint16_t h) {
  uint32_t bits = (uint32_t)h << 16;
  return (bits & 0x80000000u) ? ~bits : (bits | 0x80000000u);
}

int32_t gp_greedy_pick(const uint32_t* mask, const uint16_t* logits, int32_t V) {
  int32_t best = -1;
  uint32_t best_key = 0;
  for (int32_t t = 0; t <= V; ++t) {
    if (!((mask[t >> 5] >> (t & 31)) & 1u)) continue;
    uint32_t k = bf16_key(logits[t]);
    if (best < 0 || k > best_key) { best = t; best_key = k; }
  }
  return best;
}

/* ------------------------------------------------------------ sampler
 * Temperature / top-k / top-p sampling over the allowed tokens — the rule of
 * kernels.cu SampleKernel, restated with one full 16-bit key
 * histogram instead of the device's two-level one.  Compiled with
 * -ffp-contract=off: the weight is the same sequence of correctly rounded
 * fp32 operations as on the device. */
static uint32_t sample_key(uint32_t bits16) {
  return (bits16 & 0x8000u) ? (~bits16 & 0xFFFFu) : (bits16 | 0x8000u);
}

static float key_value(uint32_t key) {
  uint32_t bits = ((key & 0x8000u) ? (key & 0x7FFFu) : (~key & 0xFFFFu)) << 16;
  float f;
  memcpy(&f, &bits, 4);
  return f;
}

uint64_t gp_sample_weight(uint32_t key, float vmax, float temperature) {
  float v = key_value(key);
  float d = v - vmax;
  float x = d / temperature;
  float y = x * 1.44269502f;
  if (!(y >= -64.0f)) return 0;
  if (y > 0.0f) return 0;
  float fl = floorf(y);
  int n = (int)fl;
  float f = y - fl;
  float p = 1.54035304e-4f;
  p = fmaf(p, f, 1.33335581e-3f);
  p = fmaf(p, f, 9.61812911e-3f);
  p = fmaf(p, f, 5.55041087e-2f);
  p = fmaf(p, f, 2.40226507e-1f);
  p = fmaf(p, f, 6.93147181e-1f);
  p = fmaf(p, f, 1.0f);
  uint32_t sbits = (uint32_t)(n + 32 + 127) << 23;
  float scale;
  memcpy(&scale, &sbits, 4);
  return (uint64_t)llrintf(p * scale);
}

int32_t gp_sample_pick(const uint32_t* mask, const uint16_t* logits, int32_t V, float temperature, int32_t top_k,
                       uint32_t top_p24, uint64_t u) {
  int32_t v1 = V + 1;
  uint32_t* cnt = (uint32_t*)calloc(65536, sizeof(uint32_t));
  uint32_t n_allowed = 0, kmax = 0;
  for (int32_t t = 0; t < v1; ++t) {
    if (!((mask[t >> 5] >> (t & 31)) & 1u)) continue;
    uint32_t k = sample_key(logits[t]);
    cnt[k]++;
    n_allowed++;
    if (k > kmax) kmax = k;
  }
  int32_t tok = -1;
  if (n_allowed > 0) {
    float vmax = key_value(kmax);
    /* kept_k: keys >= the k-th largest key (ties kept) */
    uint32_t tau_k = 0;
    if (top_k > 0 && (uint32_t)top_k < n_allowed) {
      uint32_t cum = 0;
      for (int32_t k = 65535; k >= 0; --k) {
        cum += cnt[k];
        if (cum >= (uint32_t)top_k) { tau_k = (uint32_t)k; break; }
      }
    }
    unsigned __int128 s_k = 0;
    for (int32_t k = 65535; k >= (int32_t)tau_k; --k) {
      if (cnt[k]) s_k += (unsigned __int128)cnt[k] * gp_sample_weight((uint32_t)k, vmax, temperature);
    }
    uint32_t tau_p = tau_k;
    unsigned __int128 s_p = s_k;
    if (s_k > 0 && top_p24 < (1u << 24)) {
      unsigned __int128 prod = s_k * top_p24;
      unsigned __int128 target = (prod >> 24) + ((prod & 0xFFFFFFu) ? 1 : 0);
      unsigned __int128 cum = 0;
      for (int32_t k = 65535; k >= (int32_t)tau_k; --k) {
        if (!cnt[k]) continue;
        cum += (unsigned __int128)cnt[k] * gp_sample_weight((uint32_t)k, vmax, temperature);
        if (cum >= target) { tau_p = (uint32_t)k; s_p = cum; break; }
      }
    }
    uint32_t kappa = kmax;
    uint64_t jth = 0;
    if (s_p > 0) {
      uint64_t r = (uint64_t)((s_p * (uint32_t)u) >> 32);
      unsigned __int128 cum = 0;
      for (int32_t k = 65535; k >= (int32_t)tau_p; --k) {
        if (!cnt[k]) continue;
        uint64_t w = gp_sample_weight((uint32_t)k, vmax, temperature);
        unsigned __int128 wb = (unsigned __int128)cnt[k] * w;
        if ((unsigned __int128)r < cum + wb) {
          kappa = (uint32_t)k;
          jth = (uint64_t)(((unsigned __int128)r - cum) / w);
          break;
        }
        cum += wb;
      }
    }
    for (int32_t t = 0; t < v1; ++t) {
      if (!((mask[t >> 5] >> (t & 31)) & 1u)) continue;
      if (sample_key(logits[t]) != kappa) continue;
      if (jth == 0) { tok = t; break; }
      --jth;
    }
  }
  free(cnt);
  return tok;
}

/* ------------------------------------------------------------ workload restatements
 * Synthetic inputs restated here so the CPU arm of bench.py needs nothing
 * from the product library (tests check both generators agree byte for
 * byte, and make_golden.py checks the 32k vocabulary against the reference's
 * own WriteBenchVocab, tests/acceptance/acceptance_main.cpp:341-359). */

/* std::mt19937_64 (the reference's generator). */
typedef struct { uint64_t mt[312]; int i; } mt64;
static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i) g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->i = 312;
}
static uint64_t mt64_next(mt64* g) {
  if (g->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      uint64_t x = (g->mt[k] & 0xFFFFFFFF80000000ull) | (g->mt[(k + 1) % 312] & 0x7FFFFFFFull);
      uint64_t xa = x >> 1;
      if (x & 1u) xa ^= 0xB5026F5AA96619E9ull;
      g->mt[k] = g->mt[(k + 156) % 312] ^ xa;
    }
    g->i = 0;
  }
  uint64_t y = g->mt[g->i++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

typedef struct { char s[16]; int32_t n; } vtok;

static int vtok_cmp(const void* x, const void* y) {
  const vtok* a = (const vtok*)x;
  const vtok* b = (const vtok*)y;
  int32_t m = a->n < b->n ? a->n : b->n;
  int c = memcmp(a->s, b->s, (size_t)m);
  return c ? c : (a->n > b->n) - (a->n < b->n);
}

static uint64_t vtok_hash(const char* s, int32_t n) {
  uint64_t h = 1469598103934665603ull;
  for (int32_t i = 0; i < n; ++i) h = (h ^ (uint8_t)s[i]) * 1099511628211ull;
  return h | 1u;
}

/* WriteBenchVocab (acceptance_main.cpp:341-359), continued past 32,000 and
 * with the SQL flavour (flavor 1) of the product's workload generator:
 * fragments, then mt19937_64(424242) tokens until `n` distinct, sorted
 * (std::set order).  Returns the byte total; bytes/offs may be NULL. */
int64_t gp_synth_vocab(int32_t n, int32_t flavor, uint8_t* bytes, int64_t cap, int64_t* offs) {
  static const char* frags[] = {"true", "false", "null", "{\"", " \"", "\":", "\",", "\"}", "},", "],", "[{", "}}",
                                "]}", "0.", "e+", ", ", "\": \"", "0", "1", "2", "3", "4", "5", "6", "7", "8", "9"};
  static const char* sql[] = {"SELECT ", "FROM ", "WHERE ", "AND ", "OR ", "ORDER ", "BY ", "ASC", "DESC",
                              "COUNT", "SUM", "MAX", "MIN", "(", ")", "* ", "= ", "< ", "> ", ", "};
  char alphabet[128] = "abcdefghijklmnopqrstuvwxyz0123456789{}[],:\" .-+eE_";
  if (n < 27) return -1;
  if (flavor == 1) strcat(alphabet, "ABCDEFGHIJKLMNOPQRSTUVWXYZ()*=<>");
  const uint64_t na = (uint64_t)strlen(alphabet);
  size_t slots = 16;
  while (slots < (size_t)n * 2) slots <<= 1;
  uint64_t* hs = (uint64_t*)calloc(slots, sizeof(uint64_t));
  int32_t* hi = (int32_t*)malloc(sizeof(int32_t) * slots);
  vtok* toks = (vtok*)malloc(sizeof(vtok) * (size_t)n);
  int32_t count = 0;
  /* insert: returns 1 when new */
#define GP_INSERT(str, len)                                                              \
  do {                                                                                   \
    uint64_t h_ = vtok_hash((str), (len));                                               \
    size_t j_ = (size_t)h_ & (slots - 1);                                                \
    int dup_ = 0;                                                                        \
    while (hs[j_]) {                                                                     \
      if (hs[j_] == h_ && toks[hi[j_]].n == (len) && !memcmp(toks[hi[j_]].s, (str), (size_t)(len))) { \
        dup_ = 1;                                                                        \
        break;                                                                           \
      }                                                                                  \
      j_ = (j_ + 1) & (slots - 1);                                                       \
    }                                                                                    \
    if (!dup_ && count < n) {                                                            \
      hs[j_] = h_;                                                                       \
      hi[j_] = count;                                                                    \
      memcpy(toks[count].s, (str), (size_t)(len));                                       \
      toks[count].n = (len);                                                             \
      ++count;                                                                           \
    }                                                                                    \
  } while (0)
  for (size_t k = 0; k < sizeof(frags) / sizeof(frags[0]); ++k) GP_INSERT(frags[k], (int32_t)strlen(frags[k]));
  if (flavor == 1) {
    for (size_t k = 0; k < sizeof(sql) / sizeof(sql[0]); ++k) GP_INSERT(sql[k], (int32_t)strlen(sql[k]));
  }
  mt64 g;
  mt64_seed(&g, 424242u);
  static const int32_t lens[] = {1, 2, 2, 3, 3, 4, 5, 6, 8};
  while (count < n) {
    int32_t len = lens[mt64_next(&g) % 9u];
    char t[16];
    for (int32_t i = 0; i < len; ++i) t[i] = alphabet[mt64_next(&g) % na];
    GP_INSERT(t, len);
  }
#undef GP_INSERT
  qsort(toks, (size_t)n, sizeof(vtok), vtok_cmp);
  int64_t total = 0;
  for (int32_t i = 0; i < n; ++i) total += toks[i].n;
  if (bytes && offs) {
    if (cap < total) total = -2;
    else {
      int64_t o = 0;
      for (int32_t i = 0; i < n; ++i) {
        offs[i] = o;
        memcpy(bytes + o, toks[i].s, (size_t)toks[i].n);
        o += toks[i].n;
      }
      offs[n] = o;
    }
  }
  free(hs); free(hi); free(toks);
  return total;
}

/* Tokens holding any of {}[],:" (the stream sampler's structural set). */
int32_t gp_structural_words(const uint8_t* bytes, const int64_t* offs, int32_t n, uint32_t* words) {
  int32_t nw = (n + 1 + 31) / 32, c = 0;
  memset(words, 0, sizeof(uint32_t) * (size_t)nw);
  for (int32_t t = 0; t < n; ++t) {
    for (int64_t i = offs[t]; i < offs[t + 1]; ++i) {
      if (bytes[i] && strchr("{}[],:\"", bytes[i])) {
        words[t >> 5] |= 1u << (t & 31);
        ++c;
        break;
      }
    }
  }
  return c;
}

/* Synthetic bf16 logit of token t in row b of rotating buffer k (config 5's
 * greedy decode loop; the device bench fills its buffers with the same
 * function, kernels in workload.cu).  Values in (-2, 2), 2,048 distinct, so
 * ties (broken by the lowest id) are common. */
uint16_t gp_synth_logit(uint64_t seed, int32_t k, int32_t b, int32_t t) {
  uint64_t h = mix64(seed ^ 0x6C6F67697473ull ^ ((uint64_t)(uint32_t)k * 0xA24BAED4963EE407ull) ^
                     ((uint64_t)(uint32_t)b * 0xD1B54A32D192ED03ull));
  uint64_t x = mix64(h ^ (uint64_t)(uint32_t)t);
  return (uint16_t)((0x3C00u + (uint32_t)(x & 0x3FFu)) ^ (((x >> 20) & 1u) ? 0x8000u : 0u));
}

void gp_synth_logit_row(uint64_t seed, int32_t k, int32_t b, int32_t n, uint16_t* row) {
  for (int32_t t = 0; t < n; ++t) row[t] = gp_synth_logit(seed, k, b, t);
}

/* Polynomial hash of a mask row (sum of w_i * M^(i+1) mod 2^64): the
 * per-step mask digests of the decode loop, recomputed by the tests from
 * device bitmasks with numpy. */
uint64_t gp_mask_hash(const uint32_t* words, int32_t nw) {
  const uint64_t M = 0x9E3779B97F4A7C15ull;
  uint64_t h = 0, p = M;
  for (int32_t i = 0; i < nw; ++i) {
    h += (uint64_t)words[i] * p;
    p *= M;
  }
  return h;
}

/* ------------------------------------------------------------ decode loop */
int gp_decode_run(const gp_automaton* a, const gp_trie* t, const uint8_t* bytes,
                  const int64_t* offs, const uint32_t* structural, int32_t batch, int32_t steps,
                  uint64_t seed, int32_t stack_cap, double* stats, int32_t* tokens_out,
                  int32_t* final_stacks, const gp_run_opts* opts) {
  gp_run_opts o;
  memset(&o, 0, sizeof(o));
  if (opts) o = *opts;
  int32_t V = t->num_tokens;
  int32_t nw = (V + 1 + 31) / 32;
  uint32_t* mask = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)nw);
  uint16_t* row = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(V + 1));
  gp_config* cfgs = (gp_config*)calloc((size_t)batch, sizeof(gp_config));
  int32_t* chosen = (int32_t*)malloc(sizeof(int32_t) * (size_t)batch * (size_t)steps);
  for (int32_t b = 0; b < batch; ++b) gp_config_init(a, &cfgs[b]);
  int64_t restarts = 0, pops = 0, wpops = 0;
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (int32_t s = 0; s < steps; ++s) {
    for (int32_t b = 0; b < batch; ++b) {
      gp_config* c = &cfgs[b];
      gp_mask(a, c, t, mask);
      pops += count_bits(mask, NULL, V + 1);
      if (b < o.digest_seqs && s >= o.warmup) wpops += count_bits(mask, NULL, V);
      if (o.mask_hash) o.mask_hash[(int64_t)b * steps + s] = gp_mask_hash(mask, nw);
      int32_t tok;
      if (o.mode == 1) {
        gp_synth_logit_row(o.logit_seed, s % (o.rows > 0 ? o.rows : 1), b, V + 1, row);
        tok = gp_greedy_pick(mask, row, V);
      } else {
        for (int32_t i = 0; i <= V; ++i) {
          if (!((mask[i >> 5] >> (i & 31)) & 1u)) row[i] = 0xFF80u;
        }
        tok = gp_stream_pick(mask, structural, V, gp_stream_draw(seed, (uint64_t)b, (uint64_t)s));
      }
      chosen[(int64_t)b * steps + s] = tok;
      int overflow = 0;
      if (tok == V) {
        gp_step(a, c, 256);
      } else if (tok >= 0) {
        for (int64_t i = offs[tok]; i < offs[tok + 1]; ++i) {
          if (!gp_step(a, c, bytes[i])) break;
          if (c->depth > stack_cap) { overflow = 1; break; }
        }
      }
      if (tok < 0 || overflow || c->status != GP_ALIVE) {
        gp_config_init(a, c);
        ++restarts;
      }
    }
  }
  clock_gettime(CLOCK_MONOTONIC, &t1);
  uint64_t digest = 1469598103934665603ull, wdigest = 1469598103934665603ull;
  for (int64_t i = 0; i < (int64_t)batch * steps; ++i) {
    uint32_t v = (uint32_t)chosen[i];
    for (int k = 0; k < 4; ++k) digest = (digest ^ ((v >> (8 * k)) & 0xffu)) * 1099511628211ull;
    if (tokens_out) tokens_out[i] = chosen[i];
  }
  for (int32_t b = 0; b < batch && b < o.digest_seqs; ++b) {
    for (int32_t s = o.warmup; s < steps; ++s) {
      uint32_t v = (uint32_t)chosen[(int64_t)b * steps + s];
      for (int k = 0; k < 4; ++k) wdigest = (wdigest ^ ((v >> (8 * k)) & 0xffu)) * 1099511628211ull;
    }
  }
  stats[0] = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  stats[1] = (double)batch * steps;
  stats[2] = (double)restarts;
  stats[3] = (double)(digest >> 11);
  stats[4] = (double)pops;
  stats[5] = (double)(wdigest >> 11);
  stats[6] = (double)wpops;
  if (final_stacks) {
    for (int32_t b = 0; b < batch; ++b) {
      int32_t* r = final_stacks + (int64_t)b * (stack_cap + 2);
      r[0] = cfgs[b].depth;
      r[1] = cfgs[b].status;
      for (int32_t i = 0; i < cfgs[b].depth && i < stack_cap; ++i) r[2 + i] = cfgs[b].stack[i];
    }
  }
  for (int32_t b = 0; b < batch; ++b) gp_config_free(&cfgs[b]);
  free(cfgs); free(mask); free(row); free(chosen);
  return 0;
}
