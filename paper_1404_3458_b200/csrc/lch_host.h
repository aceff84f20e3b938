// Host-side helpers of the host-buffer pipeline (lch_host.cpp).
#pragma once

#include <cstdint>
#include <functional>

namespace lch {

// Persistent worker pool; run() splits [0, n) into grains over the workers
// and the calling thread and returns when all are done.
class HostPool {
 public:
  explicit HostPool(int threads);
  ~HostPool();
  HostPool(const HostPool &) = delete;
  HostPool &operator=(const HostPool &) = delete;
  void run(int64_t n, int64_t grain, const std::function<void(int64_t, int64_t)> &fn);
  int size() const;

 private:
  struct Impl;
  Impl *impl_;
};

// out row r = the survivors (bit j of `erased` clear) of rx row r, in order.
void compact_rows(HostPool &pool, const uint16_t *rx, int64_t stride, const uint32_t *erased, int64_t n,
                  int64_t rows, uint16_t *out, int64_t out_stride);

}  // namespace lch
