// Host-side helpers of the host-buffer pipeline: a persistent worker pool and
// the survivor compaction of received words (AVX-512 VBMI2 compress-store
// with a scalar fallback).  Erased symbols are ignored by the decoder
// (rs.py:130-134, batch.py:139-143), so only the survivors cross PCIe.
#include "lch_host.h"

#include <immintrin.h>

#include <algorithm>
#include <cstdint>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace lch {

struct HostPool::Impl {
  std::vector<std::thread> workers;
  std::mutex mu;
  std::condition_variable cv, done_cv;
  const std::function<void(int64_t, int64_t)> *job = nullptr;
  int64_t n = 0, grain = 1, next = 0;
  int active = 0;
  uint64_t generation = 0;
  bool stop = false;

  void work_loop() {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return stop || generation != seen; });
      if (stop) return;
      seen = generation;
      ++active;
      for (;;) {
        if (next >= n) break;
        const int64_t lo = next, hi = std::min(n, lo + grain);
        next = hi;
        lk.unlock();
        (*job)(lo, hi);
        lk.lock();
      }
      if (--active == 0) done_cv.notify_all();
    }
  }
};

HostPool::HostPool(int threads) : impl_(new Impl) {
  if (threads < 1) threads = 1;
  for (int i = 0; i < threads; ++i) impl_->workers.emplace_back([this] { impl_->work_loop(); });
}

HostPool::~HostPool() {
  {
    std::lock_guard<std::mutex> lk(impl_->mu);
    impl_->stop = true;
  }
  impl_->cv.notify_all();
  for (auto &t : impl_->workers) t.join();
  delete impl_;
}

void HostPool::run(int64_t n, int64_t grain, const std::function<void(int64_t, int64_t)> &fn) {
  if (n <= 0) return;
  std::unique_lock<std::mutex> lk(impl_->mu);
  impl_->job = &fn;
  impl_->n = n;
  impl_->grain = std::max<int64_t>(1, grain);
  impl_->next = 0;
  impl_->active = 0;
  ++impl_->generation;
  impl_->cv.notify_all();
  // the calling thread works too
  for (;;) {
    if (impl_->next >= impl_->n) break;
    const int64_t lo = impl_->next, hi = std::min(impl_->n, lo + impl_->grain);
    impl_->next = hi;
    lk.unlock();
    fn(lo, hi);
    lk.lock();
  }
  impl_->done_cv.wait(lk, [&] { return impl_->active == 0 && impl_->next >= impl_->n; });
  impl_->job = nullptr;
}

int HostPool::size() const { return int(impl_->workers.size()) + 1; }

namespace {

__attribute__((target("avx512f,avx512bw,avx512vbmi2"))) void compact_row_avx512(
    const uint16_t *src, const uint32_t *erased, int64_t n, uint16_t *dst) {
  // Survivors are compressed in registers and collected into whole 64-byte
  // lines that leave with non-temporal stores when dst is 64-byte aligned
  // (the page-locked staging rows are): the lines are not read for ownership
  // first, which saves host memory bandwidth the DMA engines share.
  if (reinterpret_cast<uintptr_t>(dst) & 63) {
    uint16_t *o = dst;
    for (int64_t w = 0; w < n / 32; ++w) {
      const __mmask32 keep = ~erased[w];
      const __m512i v = _mm512_loadu_si512(reinterpret_cast<const void *>(src + 32 * w));
      _mm512_mask_compressstoreu_epi16(o, keep, v);
      o += __builtin_popcount(keep);
    }
    return;
  }
  // idx[j] = j for lanes below the pending count p, 32 + (j - p) above it:
  // permutex2var(pend, idx, c) appends c behind the p pending symbols
  const __m512i iota = _mm512_set_epi16(31, 30, 29, 28, 27, 26, 25, 24, 23, 22, 21, 20, 19, 18, 17, 16,
                                        15, 14, 13, 12, 11, 10, 9, 8, 7, 6, 5, 4, 3, 2, 1, 0);
  __m512i pend = _mm512_setzero_si512();
  int np = 0;
  uint16_t *o = dst;
  for (int64_t w = 0; w < n / 32; ++w) {
    const __mmask32 keep = ~erased[w];
    const int cnt = __builtin_popcount(keep);
    const __m512i v = _mm512_loadu_si512(reinterpret_cast<const void *>(src + 32 * w));
    const __m512i c = _mm512_maskz_compress_epi16(keep, v);
    const __m512i pv = _mm512_set1_epi16(short(np));
    // lanes >= np take c[j - np] (index 32 + j - np selects the second table)
    const __m512i idx = _mm512_mask_add_epi16(iota, _mm512_cmpge_epu16_mask(iota, pv), iota,
                                              _mm512_sub_epi16(_mm512_set1_epi16(32), pv));
    const __m512i merged = _mm512_permutex2var_epi16(pend, idx, c);
    if (np + cnt >= 32) {
      _mm512_stream_si512(reinterpret_cast<__m512i *>(o), merged);
      o += 32;
      // the rest of c (from index 32 - np) becomes the pending prefix
      const int used = 32 - np;
      pend = _mm512_permutexvar_epi16(_mm512_add_epi16(iota, _mm512_set1_epi16(short(used))), c);
      np = cnt - used;
    } else {
      pend = merged;
      np += cnt;
    }
  }
  if (np) _mm512_mask_storeu_epi16(o, __mmask32((1u << np) - 1u), pend);
  _mm_sfence();
}

void compact_row_scalar(const uint16_t *src, const uint32_t *erased, int64_t n, uint16_t *dst) {
  uint16_t *o = dst;
  for (int64_t j = 0; j < n; ++j)
    if (!((erased[j >> 5] >> (j & 31)) & 1u)) *o++ = src[j];
}

bool have_vbmi2() {
  static const bool v = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                        __builtin_cpu_supports("avx512vbmi2");
  return v;
}

}  // namespace

void compact_rows(HostPool &pool, const uint16_t *rx, int64_t stride, const uint32_t *erased, int64_t n,
                  int64_t rows, uint16_t *out, int64_t out_stride) {
  const bool vec = have_vbmi2() && n % 32 == 0;
  pool.run(rows, std::max<int64_t>(1, rows / (4 * pool.size())), [&](int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; ++r) {
      if (vec)
        compact_row_avx512(rx + r * stride, erased, n, out + r * out_stride);
      else
        compact_row_scalar(rx + r * stride, erased, n, out + r * out_stride);
    }
  });
}

}  // namespace lch
