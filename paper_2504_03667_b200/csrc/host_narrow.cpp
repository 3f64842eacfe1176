// host_narrow.cpp -- host side of the upload: a persistent worker pool and the
// vectorised uint64 -> u8/u16/u32 narrowing of the reference's Graph::adj rows
// (weight.hpp:9-18: UINT64_MAX = no edge).  The e2e cost of a drop-in solve is
// reading the caller's n*n*8 bytes once, so this loop runs at host memory
// bandwidth on every core (runtime-dispatched AVX-512 / AVX2 clones).
#include "host_narrow.h"

#include <immintrin.h>

#include <algorithm>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace sssp_b200 {

namespace {

class Pool {
 public:
  explicit Pool(unsigned n) {
    for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> l(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  unsigned size() const { return (unsigned)workers_.size() + 1; }

  // Runs fn(t) for t in [0, size()); the caller runs t = 0.
  void run(const std::function<void(unsigned)>& fn) {
    {
      std::unique_lock<std::mutex> l(m_);
      fn_ = &fn;
      pending_ = (unsigned)workers_.size();
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> l(m_);
    done_.wait(l, [this] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void loop(unsigned i) {
    unsigned long seen = 0;
    while (true) {
      const std::function<void(unsigned)>* fn;
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        fn = fn_;
      }
      (*fn)(i + 1);
      {
        std::lock_guard<std::mutex> l(m_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(unsigned)>* fn_ = nullptr;
  unsigned pending_ = 0;
  unsigned long gen_ = 0;
  bool stop_ = false;
};

Pool& pool() {
  static Pool p([] {
    const unsigned h = std::thread::hardware_concurrency();
    return std::max(1u, std::min(h ? h : 1u, 64u)) - 1;
  }());
  return p;
}

// One row segment: narrow, and fold max finite / min finite / range overflow.
template <typename W>
__attribute__((target_clones("arch=skylake-avx512", "avx2", "default"))) void narrow_seg(
    const uint64_t* __restrict__ x, W* __restrict__ o, uint64_t len, uint64_t fmax, uint64_t winf,
    uint64_t* mx_io, uint64_t* mn_io, uint64_t* over_io) {
  uint64_t mx = *mx_io, mn = *mn_io, over = 0;
  for (uint64_t j = 0; j < len; ++j) {
    const uint64_t v = x[j];
    const bool inf = v == ~0ull;
    o[j] = (W)(inf ? winf : v);
    mx = std::max<uint64_t>(mx, inf ? 0ull : v);
    mn = std::min<uint64_t>(mn, v);  // INF is the maximum: never lowers mn
    over |= (uint64_t)(!inf & (v > fmax));
  }
  *mx_io = mx;
  *mn_io = mn;
  *over_io |= over;
}

// Explicit AVX-512 form of narrow_seg: 8 weights per step (vpcmpuq for INF,
// blend, vpmovq{b,w,d} narrowing store, vpmaxuq / vpminuq / vpcmpuq folds).
// The compiler's clone of the scalar loop ran at ~5 GB/s per core; this one
// streams at the core's share of host memory bandwidth.
template <typename W>
__attribute__((target("avx512f,avx512vl,avx512bw"))) void narrow_seg_avx512(
    const uint64_t* __restrict__ x, W* __restrict__ o, uint64_t len, uint64_t fmax, uint64_t winf,
    uint64_t* mx_io, uint64_t* mn_io, uint64_t* over_io) {
  const __m512i ones = _mm512_set1_epi64(-1), vfmax = _mm512_set1_epi64((long long)fmax),
                vwinf = _mm512_set1_epi64((long long)winf);
  __m512i vmx = _mm512_set1_epi64((long long)*mx_io), vmn = _mm512_set1_epi64((long long)*mn_io);
  __mmask8 over = 0;
  uint64_t j = 0;
  for (; j + 8 <= len; j += 8) {
    const __m512i v = _mm512_loadu_si512(reinterpret_cast<const void*>(x + j));
    const __mmask8 inf = _mm512_cmpeq_epu64_mask(v, ones);
    const __m512i nv = _mm512_mask_blend_epi64(inf, v, vwinf);
    if constexpr (sizeof(W) == 1) {
      _mm_storel_epi64(reinterpret_cast<__m128i*>(o + j), _mm512_cvtepi64_epi8(nv));
    } else if constexpr (sizeof(W) == 2) {
      _mm_storeu_si128(reinterpret_cast<__m128i*>(o + j), _mm512_cvtepi64_epi16(nv));
    } else if constexpr (sizeof(W) == 4) {
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(o + j), _mm512_cvtepi64_epi32(nv));
    } else {  // uint64 (wide encoding): a copy with the folds
      _mm512_storeu_si512(reinterpret_cast<void*>(o + j), nv);
    }
    vmx = _mm512_mask_max_epu64(vmx, (__mmask8)~inf, vmx, v);
    vmn = _mm512_min_epu64(vmn, v);  // INF is the maximum: never lowers mn
    over |= _mm512_mask_cmpgt_epu64_mask((__mmask8)~inf, v, vfmax);
  }
  uint64_t mx = _mm512_reduce_max_epu64(vmx), mn = _mm512_reduce_min_epu64(vmn);
  uint64_t ov = over ? 1u : 0u;
  for (; j < len; ++j) {
    const uint64_t v = x[j];
    const bool isinf = v == ~0ull;
    o[j] = (W)(isinf ? winf : v);
    mx = std::max<uint64_t>(mx, isinf ? 0ull : v);
    mn = std::min<uint64_t>(mn, v);
    ov |= (uint64_t)(!isinf & (v > fmax));
  }
  *mx_io = mx;
  *mn_io = mn;
  *over_io |= ov;
}

bool have_avx512() {
  static const bool yes = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512vl") &&
                          __builtin_cpu_supports("avx512bw");
  return yes;
}

template <typename W>
void narrow_any(const uint64_t* x, W* o, uint64_t len, uint64_t fmax, uint64_t winf, uint64_t* mx,
                uint64_t* mn, uint64_t* over) {
  if (have_avx512()) narrow_seg_avx512<W>(x, o, len, fmax, winf, mx, mn, over);
  else narrow_seg<W>(x, o, len, fmax, winf, mx, mn, over);
}

}  // namespace

unsigned narrow_threads() { return pool().size(); }

void parallel_run(const std::function<void(unsigned)>& fn) { pool().run(fn); }

template <typename W>
NarrowStats narrow_rows(const uint64_t* src, uint64_t ld, uint64_t r0, uint64_t rows,
                        uint64_t cols, uint64_t col_base, W* out) {
  const uint64_t winf = (W)~0ull, fmax = winf - 1;
  const unsigned T = pool().size();
  std::vector<NarrowStats> part(T);
  pool().run([&](unsigned t) {
    NarrowStats s;
    const uint64_t a = r0 + rows * t / T, b = r0 + rows * (t + 1) / T;
    for (uint64_t r = a; r < b; ++r) {
      const uint64_t* row = src + r * ld;
      W* o = out + (r - r0) * cols;
      // the diagonal (weight 0, graph.hpp:37-44) is excluded from the min
      const uint64_t diag = (r >= col_base && r < col_base + cols) ? r - col_base : cols;
      narrow_any<W>(row, o, diag, fmax, winf, &s.max_w, &s.min_w, &s.overflow);
      if (diag < cols) {
        o[diag] = (W)(row[diag] == ~0ull ? winf : row[diag]);
        s.max_w = std::max<uint64_t>(s.max_w, row[diag] == ~0ull ? 0ull : row[diag]);
        s.overflow |= (uint64_t)(row[diag] != ~0ull && row[diag] > fmax);
        narrow_any<W>(row + diag + 1, o + diag + 1, cols - diag - 1, fmax, winf, &s.max_w,
                      &s.min_w, &s.overflow);
      }
    }
    part[t] = s;
  });
  NarrowStats all;
  for (const auto& s : part) {
    all.max_w = std::max(all.max_w, s.max_w);
    all.min_w = std::min(all.min_w, s.min_w);
    all.overflow |= s.overflow;
  }
  return all;
}

template NarrowStats narrow_rows<uint8_t>(const uint64_t*, uint64_t, uint64_t, uint64_t, uint64_t,
                                          uint64_t, uint8_t*);
template NarrowStats narrow_rows<uint16_t>(const uint64_t*, uint64_t, uint64_t, uint64_t, uint64_t,
                                           uint64_t, uint16_t*);
template NarrowStats narrow_rows<uint64_t>(const uint64_t*, uint64_t, uint64_t, uint64_t, uint64_t,
                                           uint64_t, uint64_t*);
template NarrowStats narrow_rows<uint32_t>(const uint64_t*, uint64_t, uint64_t, uint64_t, uint64_t,
                                           uint64_t, uint32_t*);

}  // namespace sssp_b200
