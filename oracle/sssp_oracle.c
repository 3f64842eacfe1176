/*
 * sssp_oracle.c -- CPU restatement of the reference's matrix-scan Dijkstra.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity *checker* for the
 * B200 path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_2504_03667_b200/, libsssp_cuda.so) never links or calls it.
 *
 * Parity is pinned two ways (see tests/test_oracle.py):
 *   - against the known-answer tests of the reference's own unit suite
 *     (proj/tests/test_serial.cpp:11-38, test_dataparallel.cpp:60-80, 144-154,
 *     test_partitioned.cpp:194-246), and
 *   - against oracle/_ref/libref_sssp.so, the reference headers compiled
 *     unmodified from /root/reference/proj/include (oracle/Makefile), on
 *     golden vectors committed under tests/golden/.
 *
 * Every function cites the reference file:line it restates.  Paths are
 * relative to /root/reference/proj/include/sssp/ unless stated.
 *
 * Encoding (weight.hpp:9-21): Weight = uint64, kInfinity = UINT64_MAX,
 * kMaxWeight = UINT32_MAX, kNoVertex = SIZE_MAX (uint64 on LP64).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define O_INF UINT64_MAX
#define O_NOV UINT64_MAX
#define O_MAXW 0xFFFFFFFFull

enum { O_OK = 0, O_BAD_SOURCE = 1, O_BAD_ARG = 2, O_OOM = 3 };

/* ---------------------------------------------------------------- mt19937_64
 * std::mt19937_64 as fixed by [rand.predef]; the reference relies on its
 * output being standard-specified (generate.hpp:17-20). */
typedef struct {
  uint64_t mt[312];
  int idx;
} o_mt64;

void o_mt64_seed(o_mt64* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

uint64_t o_mt64_next(o_mt64* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ull) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

/* generate.hpp:21-29 -- unbiased draw from [0, bound). */
uint64_t o_uniform_below(o_mt64* r, uint64_t bound) {
  const uint64_t span = UINT64_MAX;
  const uint64_t limit = span - span % bound;
  uint64_t x;
  do {
    x = o_mt64_next(r);
  } while (x >= limit);
  return x % bound;
}

/* generate.hpp:31-33 -- weights uniform in [1, 100]. */
static uint64_t o_random_weight(o_mt64* r) { return 1 + o_uniform_below(r, 100); }

/* ------------------------------------------------------------------ graphs */

/* graph.hpp:37-44 (Graph::no_edges): INF everywhere, 0 on the diagonal. */
void o_no_edges(uint64_t n, uint64_t* adj) {
  for (uint64_t i = 0; i < n * n; ++i) adj[i] = O_INF;
  for (uint64_t i = 0; i < n; ++i) adj[i * n + i] = 0;
}

/* graph.hpp:73-88 (graph_from_edges): min over duplicates, mirror when
 * undirected.  edges = m triples (u, v, w).  Returns O_BAD_ARG on the same
 * inputs the reference rejects with std::invalid_argument. */
int o_graph_from_edges(uint64_t n, const uint64_t* edges, uint64_t m, int directed,
                       uint64_t* adj) {
  o_no_edges(n, adj);
  for (uint64_t i = 0; i < m; ++i) {
    const uint64_t u = edges[3 * i], v = edges[3 * i + 1], w = edges[3 * i + 2];
    if (u >= n || v >= n) return O_BAD_ARG;
    if (u == v) return O_BAD_ARG;
    if (w > O_MAXW) return O_BAD_ARG;
    if (w < adj[u * n + v]) adj[u * n + v] = w;
    if (!directed && w < adj[v * n + u]) adj[v * n + u] = w;
  }
  return O_OK;
}

/* generate.hpp:38-48 (generate_dense) followed by graph_from_edges, filled
 * straight into the matrix in the generator's draw order (u < v, row-major). */
int o_generate_dense(uint64_t n, uint64_t seed, int directed, uint64_t* adj) {
  if (n < 2) return O_BAD_ARG;
  o_mt64 r;
  o_mt64_seed(&r, seed);
  o_no_edges(n, adj);
  for (uint64_t u = 0; u < n; ++u)
    for (uint64_t v = u + 1; v < n; ++v) {
      const uint64_t w = o_random_weight(&r);
      adj[u * n + v] = w;
      if (!directed) adj[v * n + u] = w;
    }
  return O_OK;
}

/* open-addressing set of canonical pairs for generate_sparse's std::set. */
typedef struct {
  uint64_t* keys;
  uint64_t cap;
} o_pairset;

static int o_pairset_insert(o_pairset* s, uint64_t a, uint64_t b) {
  const uint64_t key = ((a < b ? a : b) << 32 | (a < b ? b : a)) + 1; /* 0 = empty */
  uint64_t h = key * 0x9E3779B97F4A7C15ull;
  for (uint64_t i = h & (s->cap - 1);; i = (i + 1) & (s->cap - 1)) {
    if (s->keys[i] == 0) {
      s->keys[i] = key;
      return 1;
    }
    if (s->keys[i] == key) return 0;
  }
}

/* generate.hpp:53-83 (generate_sparse): Fisher-Yates chain + 2n+1 distinct
 * random edges.  Writes 3n (u, v, w) triples into edges. */
int o_generate_sparse_edges(uint64_t n, uint64_t seed, uint64_t* edges) {
  if (n < 7 || n > 0xFFFFFFFFull) return O_BAD_ARG;
  o_mt64 r;
  o_mt64_seed(&r, seed);
  uint64_t* order = (uint64_t*)malloc(n * sizeof(uint64_t));
  o_pairset set;
  set.cap = 1;
  while (set.cap < 8 * n) set.cap <<= 1;
  set.keys = (uint64_t*)calloc(set.cap, sizeof(uint64_t));
  if (!order || !set.keys) {
    free(order);
    free(set.keys);
    return O_OOM;
  }
  for (uint64_t i = 0; i < n; ++i) order[i] = i;
  for (uint64_t i = n - 1; i > 0; --i) {
    uint64_t j = o_uniform_below(&r, i + 1);
    uint64_t t = order[i];
    order[i] = order[j];
    order[j] = t;
  }
  uint64_t m = 0;
  for (uint64_t i = 0; i + 1 < n; ++i) {
    o_pairset_insert(&set, order[i], order[i + 1]);
    edges[3 * m] = order[i];
    edges[3 * m + 1] = order[i + 1];
    edges[3 * m + 2] = o_random_weight(&r);
    ++m;
  }
  while (m < 3 * n) {
    uint64_t u = o_uniform_below(&r, n);
    uint64_t v = o_uniform_below(&r, n);
    if (u == v || !o_pairset_insert(&set, u, v)) continue;
    edges[3 * m] = u;
    edges[3 * m + 1] = v;
    edges[3 * m + 2] = o_random_weight(&r);
    ++m;
  }
  free(order);
  free(set.keys);
  return O_OK;
}

/* Bernoulli(p) random graph used by BASELINE configs 2 and 4 (SURVEY.md
 * §8d; not a reference generator).  Candidate pairs in row-major order
 * (u < v when undirected, u != v when directed); pair kept iff
 * (rng() >> 11) < p_q53, where p_q53 = p * 2^53; a kept pair then draws
 * 1 + uniform_below(100) as its weight. */
int o_generate_bernoulli(uint64_t n, uint64_t p_q53, uint64_t seed, int directed,
                         uint64_t* adj) {
  if (n < 1) return O_BAD_ARG;
  o_mt64 r;
  o_mt64_seed(&r, seed);
  o_no_edges(n, adj);
  for (uint64_t u = 0; u < n; ++u)
    for (uint64_t v = directed ? 0 : u + 1; v < n; ++v) {
      if (u == v) continue;
      if ((o_mt64_next(&r) >> 11) >= p_q53) continue;
      const uint64_t w = o_random_weight(&r);
      adj[u * n + v] = w;
      if (!directed) adj[v * n + u] = w;
    }
  return O_OK;
}

/* --------------------------------------------------------------- engines */

/* serial.hpp:26-63 (dijkstra_serial): n rounds of lowest-(dist, id)
 * election over unvisited vertices, then a strict-< relaxation of the
 * elected row.  visit_order (optional, n entries) receives the elected
 * vertex of every round (serial.hpp:49).  counters (optional, 2 entries)
 * receive extract_min_scans and relax_checks (serial.hpp:16-19). */
int o_dijkstra_serial(const uint64_t* adj, uint64_t n, uint64_t source, uint64_t* dist,
                      uint64_t* pred, uint64_t* visit_order, uint64_t* counters) {
  if (source >= n) return O_BAD_SOURCE; /* serial.hpp:30 */
  char* visited = (char*)calloc(n ? n : 1, 1);
  if (!visited) return O_OOM;
  uint64_t scans = 0, checks = 0;
  for (uint64_t v = 0; v < n; ++v) {
    dist[v] = O_INF;
    pred[v] = O_NOV;
  }
  dist[source] = 0;
  for (uint64_t round = 0; round < n; ++round) {
    uint64_t u = O_NOV;
    for (uint64_t v = 0; v < n; ++v) {
      ++scans;
      if (!visited[v] && (u == O_NOV || dist[v] < dist[u])) u = v;
    }
    visited[u] = 1;
    if (visit_order) visit_order[round] = u;
    const uint64_t du = dist[u];
    const uint64_t* row = adj + u * n;
    for (uint64_t v = 0; v < n; ++v) {
      ++checks;
      const uint64_t w = row[v];
      if (!visited[v] && w != O_INF && du != O_INF && du + w < dist[v]) {
        dist[v] = du + w;
        pred[v] = u;
      }
    }
  }
  if (counters) {
    counters[0] = scans;
    counters[1] = checks;
  }
  free(visited);
  return O_OK;
}

/* partition.hpp:25-29 (pad_vertex_count). */
uint64_t o_pad_vertex_count(uint64_t n, uint64_t p) {
  if (n < 1 || p < 1) return 0;
  if (p > n) return p;
  return n + (p - n % p) % p;
}

/* partitioned.hpp:184-225 in WorkerMode::sequential (:142-154), which the
 * reference proves bit-identical to the threaded mode.  Column block k owns
 * [k*loc_n, (k+1)*loc_n) of the padded matrix (partition.hpp:31-41,
 * pad_graph :46-54).  winners (optional, 2*padded_n entries) receives the
 * (dist, vertex) MinLocPair of every round (partitioned.hpp:94-101). */
int o_dijkstra_partitioned(const uint64_t* adj, uint64_t n, uint64_t source, uint64_t p,
                           uint64_t* dist, uint64_t* pred, uint64_t* winners) {
  if (p < 1) return O_BAD_ARG;
  if (source >= n) return O_BAD_SOURCE;
  const uint64_t pn = o_pad_vertex_count(n, p);
  const uint64_t loc_n = pn / p;
  uint64_t* ld = (uint64_t*)malloc(pn * sizeof(uint64_t));
  uint64_t* lp = (uint64_t*)malloc(pn * sizeof(uint64_t));
  char* vis = (char*)calloc(pn, 1);
  uint64_t* cd = (uint64_t*)malloc(p * sizeof(uint64_t));
  uint64_t* cv = (uint64_t*)malloc(p * sizeof(uint64_t));
  if (!ld || !lp || !vis || !cd || !cv) {
    free(ld); free(lp); free(vis); free(cd); free(cv);
    return O_OOM;
  }
  for (uint64_t v = 0; v < pn; ++v) {
    ld[v] = O_INF;
    lp[v] = O_NOV;
  }
  ld[source] = 0; /* partitioned.hpp:196 */
  for (uint64_t r = 0; r < pn; ++r) {
    /* local_min per block (partitioned.hpp:81-90): skip visited and INF,
     * sentinel (INF, padded_n); ties go to the lower global id. */
    for (uint64_t k = 0; k < p; ++k) {
      cd[k] = O_INF;
      cv[k] = pn;
      for (uint64_t j = k * loc_n; j < (k + 1) * loc_n; ++j) {
        if (vis[j] || ld[j] == O_INF) continue;
        if (ld[j] < cd[k] || (ld[j] == cd[k] && j < cv[k])) {
          cd[k] = ld[j];
          cv[k] = j;
        }
      }
    }
    /* allreduce_minloc (partitioned.hpp:94-101): lexicographic min. */
    uint64_t wd = cd[0], wv = cv[0];
    for (uint64_t k = 1; k < p; ++k)
      if (cd[k] < wd || (cd[k] == wd && cv[k] < wv)) {
        wd = cd[k];
        wv = cv[k];
      }
    if (winners) {
      winners[2 * r] = wd;
      winners[2 * r + 1] = wv;
    }
    /* relax_owned on every block (partitioned.hpp:106-119). */
    if (wv < pn) vis[wv] = 1;
    if (wd == O_INF) continue;
    for (uint64_t j = 0; j < pn; ++j) {
      if (vis[j]) continue;
      /* padding columns/rows are INF (pad_graph, partition.hpp:46-54). */
      const uint64_t w = (wv < n && j < n) ? adj[wv * n + j] : (wv == j ? 0 : O_INF);
      if (w != O_INF && wd + w < ld[j]) {
        ld[j] = wd + w;
        lp[j] = wv;
      }
    }
  }
  for (uint64_t v = 0; v < n; ++v) { /* gather, padding truncated (:208-223) */
    dist[v] = ld[v];
    pred[v] = lp[v];
  }
  free(ld); free(lp); free(vis); free(cd); free(cv);
  return O_OK;
}

/* oracle.hpp:27-46 (all_pairs_bruteforce, Floyd-Warshall).  d is n*n. */
int o_all_pairs(const uint64_t* adj, uint64_t n, uint64_t* d) {
  memcpy(d, adj, n * n * sizeof(uint64_t));
  for (uint64_t k = 0; k < n; ++k)
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t dik = d[i * n + k];
      if (dik == O_INF) continue;
      for (uint64_t j = 0; j < n; ++j) {
        const uint64_t dkj = d[k * n + j];
        if (dkj == O_INF) continue;
        if (dik + dkj < d[i * n + j]) d[i * n + j] = dik + dkj;
      }
    }
  return O_OK;
}

/* oracle.hpp:51-120 (validate_result): returns the number of violations
 * (0 = valid shortest-path tree with fixpoint distances). */
uint64_t o_validate(const uint64_t* adj, uint64_t n, uint64_t source, const uint64_t* dist,
                    const uint64_t* pred) {
  uint64_t bad = 0;
  if (source >= n) return 1;
  if (dist[source] != 0) ++bad;
  if (pred[source] != O_NOV) ++bad;
  for (uint64_t u = 0; u < n; ++u) {
    if (dist[u] == O_INF) continue;
    for (uint64_t v = 0; v < n; ++v) {
      const uint64_t w = adj[u * n + v];
      if (w != O_INF && dist[u] + w < dist[v]) ++bad;
    }
  }
  for (uint64_t v = 0; v < n; ++v) {
    if (v == source) continue;
    if (dist[v] == O_INF) {
      if (pred[v] != O_NOV) ++bad;
      continue;
    }
    const uint64_t u = pred[v];
    if (u == O_NOV || u >= n) {
      ++bad;
      continue;
    }
    const uint64_t w = adj[u * n + v];
    if (w == O_INF || (dist[u] == O_INF ? O_INF : dist[u] + w) != dist[v]) ++bad;
  }
  for (uint64_t v = 0; v < n; ++v) {
    if (v == source || dist[v] == O_INF) continue;
    uint64_t cur = v, hops = 0;
    while (cur != source && cur != O_NOV && cur < n && hops <= n) {
      cur = pred[cur];
      ++hops;
    }
    if (cur != source) ++bad;
  }
  return bad;
}

/* dataparallel.hpp:302-327 (dijkstra_dataparallel) with the sequential lane
 * schedule (:207-210), which the reference proves produces the same result as
 * the threaded one: relax_round (:184-217) until a round lowers nothing,
 * then reconstruct_predecessors (:221-264).  *rounds = rounds_executed. */
static const uint64_t* o_dp_dist;
static int o_dp_cmp(const void* a, const void* b) { /* (dist, id) ascending, :233-237 */
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  const uint64_t dx = o_dp_dist[x], dy = o_dp_dist[y];
  if (dx != dy) return dx < dy ? -1 : 1;
  return x < y ? -1 : (x > y ? 1 : 0);
}
int o_dijkstra_dataparallel(const uint64_t* adj, uint64_t n, uint64_t source, uint64_t* dist,
                            uint64_t* pred, uint64_t* rounds) {
  if (source >= n) return O_BAD_SOURCE; /* :305-306 */
  uint64_t* snap = (uint64_t*)malloc((n ? n : 1) * 8);
  uint64_t* order = (uint64_t*)malloc((n ? n : 1) * 8);
  char* attached = (char*)calloc(n ? n : 1, 1);
  if (!snap || !order || !attached) {
    free(snap);
    free(order);
    free(attached);
    return O_OOM;
  }
  for (uint64_t v = 0; v < n; ++v) { /* RelaxState, :44-52 */
    dist[v] = v == source ? 0 : O_INF;
    pred[v] = O_NOV;
  }
  uint64_t r = 0;
  int any;
  do { /* relax_round, :184-217; relax_cell, :67-79 */
    any = 0;
    memcpy(snap, dist, n * 8);
    for (uint64_t u = 0; u < n; ++u) {
      const uint64_t su = snap[u];
      if (su == O_INF) continue;
      for (uint64_t v = 0; v < n; ++v) {
        const uint64_t w = adj[u * n + v];
        if (w == O_INF) continue;
        if (su + w < dist[v]) {
          dist[v] = su + w;
          pred[v] = u;
          any = 1;
        }
      }
    }
    ++r;
  } while (any);
  /* reconstruct_predecessors, :221-264 */
  uint64_t m = 0;
  for (uint64_t v = 0; v < n; ++v) {
    pred[v] = O_NOV;
    if (v != source && dist[v] != O_INF) order[m++] = v;
  }
  o_dp_dist = dist;
  qsort(order, m, 8, o_dp_cmp);
  attached[source] = 1;
  int progress = 1;
  while (progress) {
    progress = 0;
    for (uint64_t i = 0; i < m; ++i) {
      const uint64_t v = order[i];
      if (attached[v]) continue;
      const uint64_t dv = dist[v];
      for (uint64_t u = 0; u < n; ++u) {
        if (u == v || !attached[u]) continue;
        const uint64_t w = adj[u * n + v];
        if (w == O_INF) continue;
        const uint64_t du = dist[u];
        if (du != O_INF && du + w == dv) {
          pred[v] = u;
          attached[v] = 1;
          progress = 1;
          break;
        }
      }
    }
  }
  if (rounds) *rounds = r;
  free(snap);
  free(order);
  free(attached);
  return O_OK;
}
