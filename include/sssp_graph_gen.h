/*
 * sssp_graph_gen.h -- host-side graph builders exported by libsssp_cuda.so.
 *
 * These produce the reference's Graph::adj layout (row-major uint64, INF =
 * UINT64_MAX, diagonal 0; graph.hpp:30-45) for the benchmark and test
 * inputs, restating the reference generators (generate.hpp:15-83) and
 * graph_from_edges (graph.hpp:73-88).  Every builder can emit a column
 * block [col_begin, col_begin+col_count) with leading dimension ld, so a
 * process that owns one shard (partition.hpp:31-41) never materialises the
 * whole matrix.  Pass col_begin = 0, col_count = ld = n for the full matrix.
 */
#ifndef SSSP_GRAPH_GEN_H
#define SSSP_GRAPH_GEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* graph_from_edges(generate_dense(n, seed), directed): complete graph,
 * weights 1 + uniform_below(100) drawn for u < v in row-major order. */
int sssp_gen_dense(uint64_t n, uint64_t seed, int directed, uint64_t col_begin,
                   uint64_t col_count, uint64_t ld, uint64_t* out);

/* graph_from_edges(generate_sparse(n, seed), directed): 3n distinct edges. */
int sssp_gen_sparse(uint64_t n, uint64_t seed, int directed, uint64_t col_begin,
                    uint64_t col_count, uint64_t ld, uint64_t* out);

/* Bernoulli graph of BASELINE configs 2 and 4: pairs in
 * row-major order (u < v undirected, u != v directed), kept iff
 * (rng() >> 11) < p_q53 (p = p_q53 / 2^53), weight 1 + uniform_below(100). */
int sssp_gen_bernoulli(uint64_t n, uint64_t p_q53, uint64_t seed, int directed,
                       uint64_t col_begin, uint64_t col_count, uint64_t ld, uint64_t* out);

/* graph_from_edges over m (u, v, w) triples; returns SSSP_ERR_BAD_ARG on
 * the inputs the reference rejects (endpoint >= n, self-loop, w > 2^32-1). */
int sssp_graph_from_edges(uint64_t n, const uint64_t* edges, uint64_t m, int directed,
                          uint64_t col_begin, uint64_t col_count, uint64_t ld, uint64_t* out);

/* parse_edge_list_text (graph.hpp:126-170) on all host threads: the '<n> <m>'
 * header then m '<u> <v> <w>' lines ('#' / blank lines skipped, CRLF
 * tolerated).  Call with edges == NULL to read n and m from the header, then
 * with a buffer of >= 3*m uint64.  On input the reference rejects, returns
 * SSSP_ERR_BAD_ARG with *err_line = the reference's ParseError line and err =
 * its what() text ("line N: ..."), the same first error a sequential scan
 * reports; *err_line = 0 when only the buffer was too small. */
int sssp_parse_edge_list(const char* text, uint64_t len, uint64_t* n, uint64_t* m,
                         uint64_t* edges, uint64_t cap, uint64_t* err_line, char* err,
                         uint64_t err_cap);

#ifdef __cplusplus
}
#endif
#endif
