// host_parse.cpp -- the reference's edge-list text parser (graph.hpp:90-170,
// parse_edge_list_text) on all host threads: sssp_parse_edge_list in
// include/sssp_graph_gen.h.  Same accepted language, same first error (line
// number and message) as the sequential reference:
//   * '#' lines and blank lines skipped; fields split on ' ' / '\t'; trailing
//     ' ', '\t', '\r' trimmed (CRLF);
//   * header '<n> <m>', then lines '<u> <v> <w>' with the reference's checks
//     in its order (field count, from_chars integers, range, self-loop,
//     negative weight, weight > kMaxWeight, more edges than declared);
//   * the error reported is the one at the LOWEST line, as a sequential scan
//     throws at its first failing line.
// The header is parsed sequentially; the body is split into newline-aligned
// chunks parsed in parallel (line numbers from a parallel newline count), and
// the edges are copied to the caller's buffer in order.
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <new>
#include <string>
#include <string_view>
#include <vector>

#include "host_narrow.h"

namespace sssp_b200 {
namespace {

constexpr uint64_t kNoLine = ~0ull;
constexpr uint64_t kMaxWeight = 0xFFFFFFFFull;  // weight.hpp:18

struct Err {
  uint64_t line = kNoLine;
  std::string what;
  void set(uint64_t l, std::string w) {
    if (l < line) {
      line = l;
      what = std::move(w);
    }
  }
};

std::string_view trim(std::string_view s) {  // graph.hpp:92-97
  while (!s.empty() && (s.front() == ' ' || s.front() == '\t')) s.remove_prefix(1);
  while (!s.empty() && (s.back() == ' ' || s.back() == '\t' || s.back() == '\r')) s.remove_suffix(1);
  return s;
}

// up to 4 fields (more are only counted); returns the field count
int split_fields(std::string_view s, std::string_view* f) {
  int k = 0;
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\t')) ++i;
    size_t j = i;
    while (j < s.size() && s[j] != ' ' && s[j] != '\t') ++j;
    if (j > i) {
      if (k < 4) f[k] = s.substr(i, j - i);
      ++k;
    }
    i = j;
  }
  return k;
}

bool parse_ll(std::string_view tok, long long* v) {  // std::from_chars, graph.hpp:104-111
  auto [ptr, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), *v);
  return ec == std::errc{} && ptr == tok.data() + tok.size();
}

std::string malformed(const char* what, std::string_view tok) {
  return std::string("malformed ") + what + " '" + std::string(tok) + "'";
}

// One body line (already trimmed, non-empty, not a comment).  Returns false
// and sets *why on a parse error.
bool body_line(std::string_view line, uint64_t n, uint64_t* u_out, uint64_t* v_out, uint64_t* w_out,
               std::string* why) {
  std::string_view f[4];
  if (split_fields(line, f) != 3) {
    *why = "expected '<u> <v> <w>'";
    return false;
  }
  long long u, v, w;
  if (!parse_ll(f[0], &u)) return *why = malformed("vertex id", f[0]), false;
  if (!parse_ll(f[1], &v)) return *why = malformed("vertex id", f[1]), false;
  if (!parse_ll(f[2], &w)) return *why = malformed("weight", f[2]), false;
  if (u < 0 || v < 0 || (uint64_t)u >= n || (uint64_t)v >= n) return *why = "vertex id out of range", false;
  if (u == v) return *why = "self-loop", false;
  if (w < 0) return *why = "negative weight", false;
  if ((uint64_t)w > kMaxWeight) return *why = "weight out of range", false;
  *u_out = (uint64_t)u;
  *v_out = (uint64_t)v;
  *w_out = (uint64_t)w;
  return true;
}

// Iterates std::getline-style lines of [b, e): fn(line_view_untrimmed, line_no)
template <typename F>
void for_lines(const char* b, const char* e, uint64_t first_line, F&& fn) {
  uint64_t ln = first_line;
  while (b < e) {
    const char* nl = static_cast<const char*>(memchr(b, '\n', (size_t)(e - b)));
    const char* end = nl ? nl : e;
    if (!fn(std::string_view(b, (size_t)(end - b)), ln)) return;
    ++ln;
    b = nl ? nl + 1 : e;
  }
}

}  // namespace

// Returns 0 on success; 1 (parse error: *err_line, err) ; 2 (edge buffer too small).
int parse_edge_list_text(const char* text, uint64_t len, uint64_t* n_out, uint64_t* m_out,
                         uint64_t* edges, uint64_t cap, uint64_t* err_line, std::string* err) {
  const char* const end = text + len;
  // total lines as std::getline counts them (for end-of-input errors)
  uint64_t total_lines = 0;
  for (const char* p = text; p < end;) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(end - p)));
    ++total_lines;
    p = nl ? nl + 1 : end;
  }
  // ---- header, sequentially (graph.hpp:137-147)
  uint64_t n = 0, m = 0, header_line = 0;
  const char* body = end;
  bool seen = false;
  Err e;
  for_lines(text, end, 1, [&](std::string_view raw, uint64_t ln) {
    std::string_view line = trim(raw);
    if (line.empty() || line.front() == '#') return true;
    std::string_view f[4];
    if (split_fields(line, f) != 2) {
      e.set(ln, "expected header '<n> <m>'");
      return false;
    }
    long long a, b;
    if (!parse_ll(f[0], &a)) return e.set(ln, malformed("vertex count", f[0])), false;
    if (!parse_ll(f[1], &b)) return e.set(ln, malformed("edge count", f[1])), false;
    if (a < 0 || b < 0) return e.set(ln, "negative header value"), false;
    n = (uint64_t)a;
    m = (uint64_t)b;
    seen = true;
    header_line = ln;
    body = raw.data() + raw.size() < end ? raw.data() + raw.size() + 1 : end;
    return false;
  });
  if (e.line != kNoLine) {
    *err_line = e.line;
    *err = e.what;
    return 1;
  }
  if (!seen) {
    *err_line = total_lines;
    *err = "missing header";
    return 1;
  }
  *n_out = n;
  *m_out = m;
  if (edges && cap < m) return 2;
  // ---- body, in newline-aligned chunks on every host thread
  const unsigned T = narrow_threads();
  const uint64_t blen = (uint64_t)(end - body);
  std::vector<const char*> cb(T + 1);
  cb[0] = body;
  cb[T] = end;
  for (unsigned t = 1; t < T; ++t) {
    const char* p = body + blen * t / T;
    if (p < cb[t - 1]) p = cb[t - 1];
    const char* nl = p > body ? static_cast<const char*>(memchr(p - 1, '\n', (size_t)(end - (p - 1)))) : p;
    cb[t] = p == body ? body : (nl ? nl + 1 : end);
  }
  std::vector<uint64_t> lines(T, 0);
  parallel_run([&](unsigned t) {  // newlines per chunk -> first line number of every chunk
    uint64_t c = 0;
    for (const char* p = cb[t]; p < cb[t + 1];) {
      const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(cb[t + 1] - p)));
      if (!nl) break;
      ++c;
      p = nl + 1;
    }
    lines[t] = c;
  });
  std::vector<uint64_t> first(T);
  uint64_t acc = 0;
  for (unsigned t = 0; t < T; ++t) {
    first[t] = header_line + 1 + acc;
    acc += lines[t];
  }
  if (!edges) {
    // Header-only call: the caller sizes its buffer from m next, so a header
    // the body does not back (e.g. '1 1000000000' over three lines) must fail
    // HERE with the reference's ParseError instead of a 24 GB allocation.  When
    // the body has exactly m candidate lines the second call validates them.
    std::vector<uint64_t> cand(T, 0);
    parallel_run([&](unsigned t) {
      for_lines(cb[t], cb[t + 1], first[t], [&](std::string_view raw, uint64_t) {
        const std::string_view line = trim(raw);
        if (!line.empty() && line.front() != '#') ++cand[t];
        return true;
      });
    });
    uint64_t c = 0;
    for (uint64_t x : cand) c += x;
    if (c == m) return 0;
    // otherwise the full pass below reports the reference's exact error
  }
  std::vector<std::vector<uint64_t>> local(T);
  std::vector<Err> errs(T);
  parallel_run([&](unsigned t) {
    auto& out = local[t];
    for_lines(cb[t], cb[t + 1], first[t], [&](std::string_view raw, uint64_t ln) {
      std::string_view line = trim(raw);
      if (line.empty() || line.front() == '#') return true;
      uint64_t u, v, w;
      std::string why;
      if (!body_line(line, n, &u, &v, &w, &why)) {
        errs[t].set(ln, why);
        return false;  // lines after this chunk's first error cannot be the answer
      }
      out.push_back(u);
      out.push_back(v);
      out.push_back(w);
      return true;
    });
  });
  // the (m+1)-th edge is 'more edges than declared' (graph.hpp:159-160)
  uint64_t total = 0;
  for (unsigned t = 0; t < T; ++t) {
    e.set(errs[t].line, errs[t].what);
    const uint64_t k = local[t].size() / 3;
    if (total <= m && total + k > m) {  // edge number m (0-based) lives in chunk t
      const uint64_t want = m - total;
      uint64_t seen_e = 0;
      for_lines(cb[t], cb[t + 1], first[t], [&](std::string_view raw, uint64_t ln) {
        std::string_view line = trim(raw);
        if (line.empty() || line.front() == '#') return true;
        if (seen_e++ == want) {
          e.set(ln, "more edges than declared in header");
          return false;
        }
        return true;
      });
    }
    total += k;
  }
  if (e.line != kNoLine) {
    *err_line = e.line;
    *err = e.what;
    return 1;
  }
  if (total != m) {  // graph.hpp:166-168
    *err_line = total_lines;
    *err = "expected " + std::to_string(m) + " edges, found " + std::to_string(total);
    return 1;
  }
  if (!edges) return 0;  // (unreachable: a candidate count != m always errs above)
  std::vector<uint64_t> off(T + 1, 0);
  for (unsigned t = 0; t < T; ++t) off[t + 1] = off[t] + local[t].size();
  parallel_run([&](unsigned t) {
    if (!local[t].empty()) memcpy(edges + off[t], local[t].data(), local[t].size() * 8);
  });
  return 0;
}

}  // namespace sssp_b200

extern "C" int sssp_parse_edge_list(const char* text, uint64_t len, uint64_t* n, uint64_t* m,
                                    uint64_t* edges, uint64_t cap, uint64_t* err_line, char* err,
                                    uint64_t err_cap) {
  if (!text || !n || !m) return 2;  // SSSP_ERR_BAD_ARG
  uint64_t line = 0;
  std::string what;
  int rc;
  try {
    rc = sssp_b200::parse_edge_list_text(text, len, n, m, edges, cap, &line, &what);
  } catch (const std::bad_alloc&) {
    return 4;  // SSSP_ERR_OOM
  }
  if (err_line) *err_line = rc == 1 ? line : 0;
  if (rc == 0) return 0;
  const std::string msg = rc == 1 ? "line " + std::to_string(line) + ": " + what  // ParseError::what()
                                  : std::string("edge buffer smaller than the header's m");
  if (err && err_cap) {
    const size_t k = std::min<size_t>(msg.size(), (size_t)err_cap - 1);
    memcpy(err, msg.data(), k);
    err[k] = 0;
  }
  return 2;  // SSSP_ERR_BAD_ARG (ParseError in the reference)
}
