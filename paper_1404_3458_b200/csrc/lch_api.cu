// C ABI (include/lch.h): context, pass planner and the codec pipelines.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/lch.h"
#include "lch_host.h"
#include "lch_kernels.h"
#include "lch_tables.h"

using namespace lch;

struct lch_ctx {
  Tables t;
  int max_lg_h = 0;
  bool dev_ready = false;
  int device = -1;
  uint16_t *d_w_hat = nullptr, *d_b_prod = nullptr, *d_b_prod_inv = nullptr;
  uint16_t *d_exp = nullptr, *d_log = nullptr;
  uint16_t *d_b_lo = nullptr;  // b_prod[j mod 2^(r-1)] for j < 2^r (decode derivative)
  uint32_t *d_fwht_log = nullptr;
  int64_t launches = 0;
  size_t scratch_limit = size_t(4) << 30;
  std::vector<std::pair<int64_t, uint16_t *>> enc_tabs;  // encode-by-decode tables per k
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;         // host-buffer pipeline copy streams
  std::vector<std::pair<size_t, void *>> pinned;          // page-locked staging slots
  std::unique_ptr<HostPool> pool;                          // host workers (survivor compaction)
  cudaEvent_t ring_ev[16] = {};                            // upload_small ring slots
  // per staging slot: the last H2D copy that reads it (host_pipeline waits on
  // it before refilling the slot, also across calls)
  std::vector<cudaEvent_t> stage_ev;
  cudaMemPool_t mempool = nullptr;                         // private stream-ordered scratch pool
  // host-buffer pipeline: persistent device slots (grow-only; inputs at
  // k * 2 + a, outputs at 8 + k) and their events, kept across calls so the
  // copies of one call overlap the tail of the previous one
  std::vector<std::pair<size_t, void *>> pipe_dev;
  cudaEvent_t pipe_in_ready[4] = {}, pipe_in_free[4] = {}, pipe_out_free[4] = {};
  bool host_strict = false;  // host inputs read in stream order (lch_set_host_ordering)
  cudaEvent_t last_h2d = nullptr;  // the pipeline's most recent H2D copy (one of pipe_in_ready)
  uint64_t h2d_bytes = 0, d2h_bytes = 0;  // bytes the host pipeline queued (lch_host_copy_bytes)
  std::vector<cudaEvent_t> trace_ev;  // LCH_PIPE_TRACE: stage events of the host pipeline calls
  std::vector<size_t> trace_calls;    // first event of each call
  size_t ring_next = 0;
  std::mutex mu;
  std::mutex host_mu;  // serialises the host-buffer entry points (shared staging, pool)
};

namespace {

#define LCH_TRY(expr)              \
  do {                             \
    int rc_ = (expr);              \
    if (rc_ != LCH_OK) return rc_; \
  } while (0)

int cu(cudaError_t e) {
  if (e == cudaSuccess) return LCH_OK;
  static const bool verbose = std::getenv("LCH_VERBOSE_ERRORS") != nullptr;
  if (verbose) std::fprintf(stderr, "liblch: CUDA error %d: %s\n", int(e), cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? LCH_ENOMEM : LCH_ECUDA;
}

template <class T>
int upload(T *&dst, const std::vector<T> &src) {
  if (src.empty()) return LCH_OK;
  LCH_TRY(cu(cudaMalloc(&dst, src.size() * sizeof(T))));
  return cu(cudaMemcpy(dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
}

int ensure_device(lch_ctx *c) {
  std::lock_guard<std::mutex> g(c->mu);
  if (c->dev_ready) {
    // a context's tables live on the device that was current at first use
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) return LCH_ECUDA;
    return cur == c->device ? LCH_OK : LCH_EINVAL;
  }
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return LCH_ECUDA;
  }
  LCH_TRY(cu(cudaGetDevice(&c->device)));
  LCH_TRY(upload(c->d_w_hat, c->t.w_hat));
  LCH_TRY(upload(c->d_b_prod, c->t.b_prod));
  LCH_TRY(upload(c->d_b_prod_inv, c->t.b_prod_inv));
  LCH_TRY(upload(c->d_exp, c->t.exp));
  LCH_TRY(upload(c->d_log, c->t.log));
  LCH_TRY(upload(c->d_fwht_log, c->t.fwht_log));
  if (c->t.max_h == c->t.order) {
    std::vector<uint16_t> blo(c->t.order);
    for (uint32_t j = 0; j < c->t.order; ++j) blo[j] = c->t.b_prod[j & (c->t.order / 2 - 1)];
    LCH_TRY(upload(c->d_b_lo, blo));
  }
  // the context's own stream-ordered pool keeps freed scratch mapped (no
  // re-mapping per call) without touching the process-wide default pool
  cudaMemPoolProps pp = {};
  pp.allocType = cudaMemAllocationTypePinned;
  pp.location.type = cudaMemLocationTypeDevice;
  pp.location.id = c->device;
  LCH_TRY(cu(cudaMemPoolCreate(&c->mempool, &pp)));
  uint64_t thr = ~0ull;
  LCH_TRY(cu(cudaMemPoolSetAttribute(c->mempool, cudaMemPoolAttrReleaseThreshold, &thr)));
  c->dev_ready = true;
  return LCH_OK;
}

// Stream-ordered scratch allocation freed at scope exit.
struct Scratch {
  cudaStream_t s;
  cudaMemPool_t pool;
  std::vector<void *> ptrs;
  Scratch(const lch_ctx *c, cudaStream_t st) : s(st), pool(c->mempool) {}
  ~Scratch() {
    for (void *p : ptrs) cudaFreeAsync(p, s);
  }
  template <class T>
  int alloc(T *&p, size_t count) {
    void *v = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = pool ? cudaMallocFromPoolAsync(&v, count * sizeof(T), pool, s)
                         : cudaMallocAsync(&v, count * sizeof(T), s);
    if (e != cudaSuccess) return cu(e);
    ptrs.push_back(v);
    p = static_cast<T *>(v);
    return LCH_OK;
  }
};

// ---------------------------------------------------------------------------
// planner: group a sequence of per-level ops into tile passes of <= TPB_MAX
// distinct position bits, in order.

struct LOp {
  int kind;
  int level;
  uint32_t hs;
  const uint16_t *table;
  int64_t tab_stride = 0;  // per stripe-group table rows (packet layout)
};

struct Plan {
  std::vector<LOp> pre, bf, post;  // scalings before, butterflies, scalings after
  std::vector<int> bits;           // sorted tile bits
  bool empty() const { return pre.empty() && bf.empty() && post.empty(); }
};

bool low_bits_only(const std::vector<int> &bits, int tpb) {
  for (int b : bits)
    if (b >= tpb) return false;
  return true;
}

// Group ops into passes: each pass = [scalings] [butterflies on <= TPB_MAX
// distinct bits] [scalings].  The first/last pass touching a raw uint16
// buffer must tile the contiguous low bits; empty transpose passes are added
// when the op sequence starts/ends on high bits.
std::vector<Plan> plan_passes(const std::vector<LOp> &ops, int lgH, bool raw_in, bool raw_out) {
  const int tpb = std::min(TPB_MAX, lgH);
  std::vector<Plan> out;
  Plan cur;
  auto has = [](const std::vector<int> &v, int b) { return std::find(v.begin(), v.end(), b) != v.end(); };
  auto flush = [&]() {
    out.push_back(cur);
    cur = Plan();
  };
  for (const LOp &op : ops) {
    if (op.kind == OP_SCALE) {
      if (cur.bf.empty()) {
        if (int(cur.pre.size()) == MAXSCALE) flush();
        cur.pre.push_back(op);
      } else {
        if (int(cur.post.size()) == MAXSCALE) flush();
        (cur.bf.empty() ? cur.pre : cur.post).push_back(op);
      }
      continue;
    }
    if (!cur.post.empty()) flush();
    if (!has(cur.bits, op.level) && int(cur.bits.size()) == tpb) flush();
    if (int(cur.bf.size()) == MAXOPS) flush();
    if (!has(cur.bits, op.level)) cur.bits.push_back(op.level);
    cur.bf.push_back(op);
  }
  if (!cur.empty() || out.empty()) out.push_back(cur);
  if (raw_in && !low_bits_only(out.front().bits, tpb)) out.insert(out.begin(), Plan());
  if (raw_out && !low_bits_only(out.back().bits, tpb)) out.push_back(Plan());
  for (size_t i = 0; i < out.size(); ++i) {
    Plan &p = out[i];
    const bool raw = (i == 0 && raw_in) || (i + 1 == out.size() && raw_out);
    if (raw) {
      p.bits.clear();
      for (int b = 0; b < tpb; ++b) p.bits.push_back(b);
    } else {
      for (int b = 0; int(p.bits.size()) < tpb && b < lgH; ++b)
        if (!has(p.bits, b)) p.bits.push_back(b);
    }
    std::sort(p.bits.begin(), p.bits.end());
  }
  return out;
}

// Butterflies of a pass -> radix-4 rounds over <= 2 local tile bits.
int build_rounds(const Plan &pl, PassParams &p) {
  const int tpb = int(pl.bits.size());
  auto local = [&](int level) {
    return int(std::find(pl.bits.begin(), pl.bits.end(), level) - pl.bits.begin());
  };
  p.nops = 0;
  p.nrounds = 0;
  PassRound cur{};
  cur.m0 = cur.m1 = -1;
  auto close = [&]() -> int {
    if (cur.m0 < 0) return LCH_OK;
    if (p.nrounds == MAXROUNDS) return LCH_EINVAL;
    if (cur.m1 < 0 && tpb >= 2)
      for (int b = 0; b < tpb; ++b)
        if (b != cur.m0) { cur.m1 = b; break; }
    cur.nw = 0;
    for (int b = 0; b < tpb; ++b)
      if (b != cur.m0 && b != cur.m1) cur.obit[cur.nw++] = b;
    for (int w = 0; w < NWARP; ++w) {
      int q = 0;
      for (int j = 0; j < cur.nw; ++j) q |= ((w >> j) & 1) << cur.obit[j];
      cur.q0w[w] = uint8_t(q);
    }
    cur.op_end = p.nops;
    // a pair's factor depends on the position bits above its level only
    // (transform.py:123), so both pairs of an op share it when the round's
    // other bit is a lower level
    for (int o = cur.op_begin; o < cur.op_end; ++o) {
      PassOp &op = p.ops[o];
      const int other = op.m == 0 ? cur.m1 : cur.m0;
      op.shared = (other >= 0 && pl.bits[other] < op.level) ? 1 : 0;
    }
    const int nr = cur.op_end - cur.op_begin;
    cur.shape = 0;
    if (cur.m1 >= 0 && nr == 1 && p.ops[cur.op_begin].m == 0) cur.shape = 1;
    if (cur.m1 >= 0 && nr == 2 && p.ops[cur.op_begin].m == 0 && p.ops[cur.op_begin + 1].m == 1)
      cur.shape = 2;
    p.rounds[p.nrounds++] = cur;
    cur = PassRound{};
    cur.m0 = cur.m1 = -1;
    return LCH_OK;
  };
  // Count the distinct-bit runs; with an odd number of levels the FIRST round
  // takes a single level so the last round (which overlaps the next tile's
  // loads) keeps two.
  int nlev = 0;
  {
    int prev = -1;
    for (const LOp &op : pl.bf)
      if (local(op.level) != prev) ++nlev, prev = local(op.level);
  }
  bool single_first = (nlev % 2) == 1 && nlev > 1;
  for (const LOp &op : pl.bf) {
    const int mb = local(op.level);
    if (cur.m0 < 0) {
      cur.m0 = mb;
      cur.op_begin = p.nops;
    } else if (mb != cur.m0 && cur.m1 < 0 && !single_first) {
      cur.m1 = mb;
    } else if ((mb != cur.m0 && mb != cur.m1) ||
               (mb == cur.m0 && cur.m1 >= 0 && p.nops > cur.op_begin &&
                p.ops[p.nops - 1].m == 1)) {
      // new round: a third bit, or a return from m1 to m0 (rounds are m0* m1*)
      LCH_TRY(close());
      single_first = false;
      cur.m0 = mb;
      cur.op_begin = p.nops;
    }
    PassOp &o = p.ops[p.nops++];
    o.kind = op.kind;
    o.level = op.level;
    o.hs = op.hs;
    o.table = nullptr;
    o.shared = 0;
    o.m = (mb == cur.m0) ? 0 : 1;
    o.mloc = mb;
  }
  return close();
}

void fill_bits(const std::vector<int> &bits, int lgH, int *gbit, int &nnb, int *nbit) {
  for (size_t m = 0; m < bits.size(); ++m) gbit[m] = bits[m];
  nnb = 0;
  for (int b = 0; b < lgH; ++b)
    if (std::find(bits.begin(), bits.end(), b) == bits.end()) nbit[nnb++] = b;
}

RawIO make_raw(uint16_t *ptr, int64_t stride, int64_t pkt = 0, int64_t npos = 0,
               int64_t pos_lo = 0, int64_t pos_hi = int64_t(1) << 40) {
  RawIO io{};
  io.ptr = ptr;
  io.row_stride = stride;
  io.pkt = pkt;
  io.npos = npos;
  io.pos_lo = pos_lo;
  io.pos_hi = pos_hi;
  io.vec = (reinterpret_cast<uintptr_t>(ptr) % 16 == 0) && (stride % 8 == 0);
  io.al4 = (reinterpret_cast<uintptr_t>(ptr) % 4 == 0) && (stride % 2 == 0);
  return io;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    else
      cudaGetLastError();
  });
  return fn;
}

// TMA view of a row-major raw input for the pass kernel's raw tiles:
// {8 symbols, chunks of 8 positions over [pos_lo, min(pos_hi, 2^lgH)), rows},
// boxes {8, 1, 256}: one chunk of 256 rows, [row][16 B] in shared memory.  False (use the register path) unless 16-byte aligned.
bool make_raw_tma(const RawIO &io, int64_t batch, int lgH, CUtensorMap *m) {
  if (io.pkt || !io.vec || io.pos_lo % 8) return false;
  const int64_t hi = std::min<int64_t>(io.pos_hi, int64_t(1) << lgH);
  if (hi <= io.pos_lo || (hi - io.pos_lo) % 8 || batch <= 0 || batch >= (int64_t(1) << 31)) return false;
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  // dims ordered by stride: {symbol in chunk, chunk, row}
  const cuuint64_t dims[3] = {8, cuuint64_t((hi - io.pos_lo) / 8), cuuint64_t(batch)};
  const cuuint64_t strides[2] = {16, cuuint64_t(io.row_stride) * 2};
  const cuuint32_t box[3] = {8, 1, 256};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, io.ptr, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int R, uint32_t POLY>
int run_plan(lch_ctx *c, const std::vector<Plan> &plan, int lgH, int64_t batch, const RawIO *raw_in,
             const uint4 *bs_in, const RawIO *raw_out, uint4 *work, cudaStream_t s,
             uint4 *gt_out = nullptr, int gt_lgH = 0, int64_t pkt = 0) {
  const int ngroups = int((batch + GROUP - 1) / GROUP);
  for (size_t i = 0; i < plan.size(); ++i) {
    const Plan &pl = plan[i];
    PassParams p;
    std::memset(&p, 0, sizeof(p));
    LCH_TRY(build_rounds(pl, p));
    p.npre = int(pl.pre.size());
    p.npost = int(pl.post.size());
    for (int o = 0; o < p.npre; ++o)
      p.pre[o] = PassOp{OP_SCALE, 0, 0, 0, 0u, pl.pre[o].table, pl.pre[o].tab_stride, 0};
    for (int o = 0; o < p.npost; ++o)
      p.post[o] = PassOp{OP_SCALE, 0, 0, 0, 0u, pl.post[o].table, pl.post[o].tab_stride, 0};
    p.tpb = int(pl.bits.size());
    p.lgH = lgH;
    fill_bits(pl.bits, lgH, p.gbit, p.nnb, p.nbit);
    {
      std::vector<int> sb(pl.bits);
      std::sort(sb.begin(), sb.end());
      for (size_t m = 0; m < sb.size(); ++m) p.ins_mask[m] = (1u << sb[m]) - 1u;
    }
    p.lgnt = lgH - p.tpb;
    p.batch = batch;
    p.ngroups = ngroups;
    p.pkt = pkt;
    const bool first = i == 0, last = i + 1 == plan.size();
    p.in_mode = (first && raw_in) ? IO_RAW : IO_BS;
    p.out_mode = (last && raw_out) ? IO_RAW : IO_BS;
    if (p.in_mode == IO_RAW) {
      p.raw_in = *raw_in;
      // TMA raw tiles: R = 16, tile = the 32 positions 32t .. 32t+31
      bool low5 = R == 16 && p.tpb == 5;
      for (int m = 0; m < p.tpb; ++m) low5 = low5 && p.gbit[m] == m;
      static const bool no_tma = std::getenv("LCH_NO_RAW_TMA") != nullptr;
      p.raw_tma = (low5 && !no_tma && make_raw_tma(p.raw_in, batch, lgH, &p.tm_in)) ? 1 : 0;
      // packet layout: bulk copies of the 2 KB lane runs (window in whole tiles)
      const RawIO &ri = p.raw_in;
      p.raw_bulk = (low5 && !no_tma && ri.pkt >= GROUP && ri.pkt % GROUP == 0 && ri.pos_lo % 32 == 0 &&
                    (std::min<int64_t>(ri.pos_hi, int64_t(1) << lgH) - ri.pos_lo) % 32 == 0 &&
                    reinterpret_cast<uintptr_t>(ri.ptr) % 16 == 0) ? 1 : 0;
    }
    if (p.out_mode == IO_RAW) {
      p.raw_out = *raw_out;
      // prefetch of the merge's survivor chunks (decode output tiles of 32
      // positions starting at position 0; the merge source indexed by
      // absolute position)
      const RawIO &o = p.raw_out;
      bool low5 = R == 16 && p.tpb == 5 && o.pkt == 0 && o.pos_lo == 0 && o.merge_src && !o.pinv_log;
      for (int m = 0; m < p.tpb; ++m) low5 = low5 && p.gbit[m] == m;
      static const bool no_tma = std::getenv("LCH_NO_RAW_TMA") != nullptr;
      if (low5 && !no_tma) {
        RawIO ms = make_raw(const_cast<uint16_t *>(o.merge_src), o.merge_stride, 0, 0, 0, o.pos_hi);
        p.merge_tma = make_raw_tma(ms, batch, lgH, &p.tm_merge) ? 1 : 0;
      }
    }
    p.bs_in = (first && bs_in) ? bs_in : work;
    p.bs_out = work;
    p.w_hat = c->d_w_hat;
    p.taps = c->t.poly & (c->t.order - 1u);
    if (last && gt_out) {
      p.gt_out = gt_out;
      p.gt_lgH = gt_lgH;
    }
    {
      static const int dbg =
          std::getenv("LCH_DBG_PASS") ? int(std::strtoul(std::getenv("LCH_DBG_PASS"), nullptr, 0)) : 0;
      p.dbg = dbg;
    }
    for (int l = 0; l <= c->t.levels && l < 17; ++l) p.w_hat_off[l] = c->t.w_hat_off[l];
    LCH_TRY(cu(launch_pass<R, POLY>(p, ngroups, s)));
    c->launches++;
  }
  return LCH_OK;
}

size_t bs_bytes(int R, int64_t batch, int lgH) {
  const int64_t ngroups = (batch + GROUP - 1) / GROUP;
  return size_t(ngroups) * (size_t(1) << lgH) * 32 * R * 4;
}

// Derivative gather over the position bits `bits` (all except those already
// summed), in passes of <= GMAXB bits; `special` (or -1) is the top bit
// handled as c * (y[j] + y[j | 2^special]) (decode: folded top inverse level).
template <int R, uint32_t POLY>
int run_gather(lch_ctx *c, const uint4 *y, uint4 *t, int lgH_in, int lgH_out, int64_t batch,
               std::vector<int> bits, int special, uint32_t cconst, const uint4 *t_in,
               cudaStream_t s) {
  const int ngroups = int((batch + GROUP - 1) / GROUP);
  std::sort(bits.begin(), bits.end());
  if (special >= 0) bits.erase(std::remove(bits.begin(), bits.end(), special), bits.end());
  // shared memory holds the y tile over the summed bits (one lane-word)
  auto need = [&](size_t nb) { return (size_t(1) << nb) * R * 4; };
  size_t maxb = 0;
  while (maxb < size_t(GMAXB) && need(maxb + 1) <= GATHER_SMEM_MAX) ++maxb;
  // fewest passes, then balanced sizes so no pass degenerates into tiny tiles
  const size_t npass = bits.empty() ? (special >= 0 ? 1 : 0) : (bits.size() + maxb - 1) / maxb;
  std::vector<std::vector<int>> groups;
  for (size_t i = 0, pi = 0; pi < npass; ++pi) {
    const size_t sz = (bits.size() - i + (npass - pi) - 1) / (npass - pi);
    groups.emplace_back(bits.begin() + long(i), bits.begin() + long(i + sz));
    i += sz;
  }
  bool first = true;
  for (auto grp : groups) {
    GatherParams p;
    std::memset(&p, 0, sizeof(p));
    p.taps = c->t.poly & (c->t.order - 1u);
    p.sb = (first && special >= 0) ? special : -1;
    p.c = cconst;
    p.nbits = int(grp.size());
    // lane-words per CTA: ~1024 position-words per CTA within the smem budget
    p.lwpc = 0;
    while (p.lwpc < 5 && (need(grp.size()) << (p.lwpc + 1)) <= GATHER_SMEM_MAX && (p.nbits + p.lwpc) < 10)
      ++p.lwpc;
    // chunk-major blocks: one lane-word per CTA would read half sectors
    if (p.lwpc == 0 && (need(grp.size()) << 1) <= GATHER_SMEM_CAP) {
      p.lwpc = 1;
      // A 10-bit group (the decode's gather) would need a 128 KB tile, one
      // CTA per SM, whose load and compute phases do not overlap.  Instead the
      // top 3 summed bits leave the tile -- the partners y[j | 2^bit] of the
      // outputs with that bit clear stream from global memory and hit in L2,
      // because the CTAs of the neighbouring tiles run at the same time --
      // and the tile takes 8 lane-words: 64 KB, two CTAs per SM, 128
      // contiguous bytes per position and chunk.  Measured (4096 x 2^15
      // outputs): 338 -> 233 us, DRAM reads unchanged (0.84-0.88 GB).
      // LCH_GATHER_DIRECT / LCH_GATHER_LW override (0 / 1: the old shape).
      static const int nd_env = [] {
        const char *e = getenv("LCH_GATHER_DIRECT");
        return e ? atoi(e) : 3;
      }();
      static const int lw_env = [] {
        const char *e = getenv("LCH_GATHER_LW");
        return e ? atoi(e) : 3;
      }();
      int nd = std::min({nd_env, 4, int(grp.size()) - 1});
      if (nd < 0 || grp.back() >= lgH_out) nd = 0;  // output bits only
      for (int d = 0; d < nd; ++d) {
        p.dbits[p.ndirect++] = grp.back();
        grp.pop_back();
      }
      if (nd > 0) p.lwpc = std::max(1, std::min(5, lw_env));
      p.nbits = int(grp.size());
    }
    p.lgH_in = lgH_in;
    p.lgH_out = lgH_out;
    std::vector<int> tile_and_special = grp;
    fill_bits(grp, lgH_in, p.bits, p.nnb, p.nbit);
    p.y = y;
    p.t_in = first ? t_in : t;
    p.t_out = t;
    LCH_TRY(cu(launch_gather<R, POLY>(p, ngroups, s)));
    c->launches++;
    first = false;
  }
  if (first) {  // nothing to sum: T = T_in or 0
    if (t_in) return cu(cudaMemcpyAsync(t, t_in, bs_bytes(R, batch, lgH_out), cudaMemcpyDeviceToDevice, s));
    return cu(cudaMemsetAsync(t, 0, bs_bytes(R, batch, lgH_out), s));
  }
  return LCH_OK;
}

template <class Fn>
int dispatch(lch_ctx *c, Fn &&fn) {
  if (c->t.r == 16 && c->t.poly == 0x1100Bu)
    return fn(std::integral_constant<int, 16>{}, std::integral_constant<uint32_t, 0x1100Bu>{});
  if (c->t.r == 8 && c->t.poly == 0x11Du)
    return fn(std::integral_constant<int, 8>{}, std::integral_constant<uint32_t, 0x11Du>{});
  // any other primitive polynomial: the runtime-taps instances
  if (c->t.r == 16) return fn(std::integral_constant<int, 16>{}, std::integral_constant<uint32_t, 0u>{});
  return fn(std::integral_constant<int, 8>{}, std::integral_constant<uint32_t, 0u>{});
}

uint32_t hs_of(const lch_ctx *c, int level, uint32_t shift) {
  return shift ? c->t.eval_w_hat(level, shift) : 0u;
}

struct DecodeEpi {
  const uint16_t *rx = nullptr;
  int64_t rx_stride = 0;
  uint16_t *phi = nullptr;
  uint16_t *pinv_log = nullptr;
  uint32_t k = 0;
  bool pinv_val = false;  // out: the locator wrote 1 / Pi' values (r = 16 kernel), not logs
};

int locator_impl(lch_ctx *c, const uint32_t *bits, int64_t np, uint16_t *loc_out, uint16_t *log_out,
                 cudaStream_t s, DecodeEpi *epi = nullptr) {
  const int r = c->t.r;
  const size_t n = size_t(1) << r;
  const bool aligned = !epi || (reinterpret_cast<uintptr_t>(epi->rx) % 16 == 0 &&
                                reinterpret_cast<uintptr_t>(epi->phi) % 16 == 0 && epi->rx_stride % 8 == 0);
  // one CTA per pattern: used when there are enough patterns to fill the GPU
  // (a single pattern runs faster as 4 grid-wide radix-2^8 passes)
  if (r == 16 && c->t.poly == 0x1100Bu && aligned && np >= 32) {
    FwhtParams p;
    std::memset(&p, 0, sizeof(p));
    p.nvec = np;
    p.lgn = r;
    p.mod = c->t.m;
    p.bits = bits;
    p.post_mul = c->d_fwht_log;
    p.exp = c->d_exp;
    p.loc_out = loc_out;
    p.log_out = log_out;
    if (epi) {
      p.bits_e = bits;
      p.rx = epi->rx;
      p.rx_stride = epi->rx_stride;
      p.log = c->d_log;
      p.phi = epi->phi;
      p.pinv_log = epi->pinv_log;
      p.k = epi->k;
      epi->pinv_val = true;
    }
    LCH_TRY(cu(launch_locator16(p, s)));
    c->launches++;
    return LCH_OK;
  }
  Scratch sc(c, s);
  uint32_t *buf = nullptr;
  LCH_TRY(sc.alloc(buf, size_t(np) * n));
  const int ngrp = (r + 7) / 8;
  for (int rep = 0; rep < 2; ++rep) {
    for (int gi = 0; gi < ngrp; ++gi) {
      FwhtParams p;
      std::memset(&p, 0, sizeof(p));
      p.data = buf;
      p.nvec = np;
      p.lgn = r;
      p.b0 = gi * 8;
      p.tb = std::min(8, r - p.b0);
      p.mod = c->t.m;
      if (rep == 0 && gi == 0) p.bits = bits;
      if (rep == 0 && gi == ngrp - 1) p.post_mul = c->d_fwht_log;
      if (rep == 1 && gi == ngrp - 1) {
        p.exp = c->d_exp;
        p.loc_out = loc_out;
        p.log_out = log_out;
        if (epi) {
          p.bits_e = bits;
          p.rx = epi->rx;
          p.rx_stride = epi->rx_stride;
          p.log = c->d_log;
          p.phi = epi->phi;
          p.pinv_log = epi->pinv_log;
          p.k = epi->k;
        }
      }
      LCH_TRY(cu(launch_fwht(p, s)));
      c->launches++;
    }
  }
  return LCH_OK;
}

}  // namespace

// ---------------------------------------------------------------------------

extern "C" {

const char *lch_version(void) { return "lch-b200 0.1 (sm_100a, bit-sliced)"; }

const char *lch_strerror(int code) {
  switch (code) {
    case LCH_OK: return "ok";
    case LCH_EINVAL: return "invalid argument";
    case LCH_ETOOMANY: return "too many erasures";
    case LCH_ENOTPRIM: return "reduction polynomial is not primitive";
    case LCH_ECUDA: return "CUDA error or no CUDA device";
    case LCH_ENOMEM: return "out of memory";
    case LCH_EUNSUPPORTED: return "unsupported configuration";
    case LCH_EZERODIV: return "division by zero";
    default: return "unknown error";
  }
}

int lch_init(int r, uint32_t poly, int max_lg_h, lch_ctx **out) {
  return lch_init_alpha(r, poly, 2u, max_lg_h, out);
}

int lch_init_alpha(int r, uint32_t poly, uint32_t alpha, int max_lg_h, lch_ctx **out) {
  if (!out) return LCH_EINVAL;
  *out = nullptr;
  if (max_lg_h < 0 || max_lg_h > 16) return LCH_EINVAL;
  lch_ctx *c = new (std::nothrow) lch_ctx();
  if (!c) return LCH_ENOMEM;
  int rc = build_tables(r, poly, 1u << max_lg_h, c->t, alpha);
  if (rc != LCH_OK) {
    delete c;
    return rc;
  }
  c->max_lg_h = max_lg_h;
  *out = c;
  return LCH_OK;
}

void lch_destroy(lch_ctx *c) {
  if (!c) return;
  if (c->dev_ready) {
    cudaFree(c->d_w_hat);
    cudaFree(c->d_b_prod);
    cudaFree(c->d_b_prod_inv);
    cudaFree(c->d_exp);
    cudaFree(c->d_log);
    cudaFree(c->d_fwht_log);
    cudaFree(c->d_b_lo);
    for (auto &e : c->enc_tabs) cudaFree(e.second);
    if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
    if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
    for (auto &e : c->pinned)
      if (e.second) cudaFreeHost(e.second);
    for (cudaEvent_t e : c->ring_ev)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : c->stage_ev)
      if (e) cudaEventDestroy(e);
    cudaDeviceSynchronize();
    for (auto &e : c->pipe_dev)
      if (e.second) cudaFree(e.second);
    for (int k = 0; k < 4; ++k) {
      if (c->pipe_in_ready[k]) cudaEventDestroy(c->pipe_in_ready[k]);
      if (c->pipe_in_free[k]) cudaEventDestroy(c->pipe_in_free[k]);
      if (c->pipe_out_free[k]) cudaEventDestroy(c->pipe_out_free[k]);
    }
    if (c->mempool) {
      cudaDeviceSynchronize();
      cudaMemPoolDestroy(c->mempool);
    }
  }
  delete c;
}

int lch_get_tables(const lch_ctx *c, uint16_t *log, uint16_t *exp, uint16_t *w_hat,
                   uint16_t *w_prime, uint16_t *b_prod, uint16_t *b_prod_inv, uint32_t *fwht_log,
                   uint16_t *w_on_basis, uint16_t *w_norm) {
  if (!c) return LCH_EINVAL;
  const Tables &t = c->t;
  if (log) std::memcpy(log, t.log.data(), t.order * 2);
  if (exp) std::memcpy(exp, t.exp.data(), t.m * 2);
  if (w_hat && !t.w_hat.empty()) std::memcpy(w_hat, t.w_hat.data(), t.w_hat.size() * 2);
  if (w_prime) std::memcpy(w_prime, t.w_prime.data(), t.r * 2);
  if (b_prod) std::memcpy(b_prod, t.b_prod.data(), t.max_h * 2);
  if (b_prod_inv) std::memcpy(b_prod_inv, t.b_prod_inv.data(), t.max_h * 2);
  if (fwht_log) std::memcpy(fwht_log, t.fwht_log.data(), t.order * 4);
  if (w_on_basis) std::memcpy(w_on_basis, t.w_on_basis.data(), t.r * t.r * 2);
  if (w_norm) std::memcpy(w_norm, t.w_norm.data(), t.r * 2);
  return LCH_OK;
}

int64_t lch_launch_count(const lch_ctx *c) { return c ? c->launches : 0; }

}  // extern "C"

// ---------------------------------------------------------------------------
// Layouts and lane chunking.
//
// Row layout (packet_len == 0): lane b = row b, symbol j at ptr[b * stride + j].
// Packet layout (packet_len = P > 0, P % 1024 == 0): lane b = (stripe group
// b / P, packet offset b % P), symbol j at ptr[((b / P) * stride + j) * P + b % P];
// the stride counts positions per stripe group.  Each 1024-lane bit-sliced
// group then lies inside one stripe group, so per-group tables are uniform.

static int check_layout(const void *p, int64_t batch, int64_t pkt) {
  if (pkt < 0) return LCH_EINVAL;
  if (pkt == 0) return LCH_OK;
  if (pkt % GROUP || batch % pkt) return LCH_EINVAL;
  if (p && reinterpret_cast<uintptr_t>(p) % 16) return LCH_EINVAL;
  return LCH_OK;
}

static RawIO make_io(const uint16_t *ptr, int64_t stride, int64_t pkt) {
  uint16_t *q = const_cast<uint16_t *>(ptr);
  return pkt ? make_raw(q, 0, pkt, stride) : make_raw(q, stride);
}

// pointer to position j of lane 0
static uint16_t *at_pos(const uint16_t *ptr, int64_t j, int64_t pkt) {
  return const_cast<uint16_t *>(ptr) + (pkt ? j * pkt : j);
}

// the same I/O descriptor for the lanes starting at b0
static RawIO shift_io(RawIO io, int64_t b0) {
  if (io.pkt) {
    const int64_t g0 = b0 / io.pkt;
    io.ptr += g0 * io.npos * io.pkt;
    if (io.merge_src) io.merge_src += g0 * io.merge_stride * io.pkt;
    if (io.merge_bits) io.merge_bits += g0 * io.bits_stride;
  } else {
    io.ptr += b0 * io.row_stride;
    if (io.merge_src) io.merge_src += b0 * io.merge_stride;
    if (io.merge_bits) io.merge_bits += b0 * io.bits_stride;
    if (io.pinv_log) io.pinv_log += b0 * io.pinv_stride;
  }
  return io;
}

static size_t bs_lane_bytes(int R, int lgH) { return (size_t(1) << lgH) * size_t(R) / 8; }

// lanes per chunk so that `lane_bytes` of scratch per lane fit the budget
static int64_t chunk_lanes(const lch_ctx *c, int64_t batch, int64_t pkt, size_t lane_bytes) {
  const int64_t unit = pkt ? pkt : GROUP;
  int64_t ch = lane_bytes ? int64_t(c->scratch_limit / lane_bytes) : batch;
  ch = std::max<int64_t>(unit, ch / unit * unit);
  return std::min(ch, batch);
}

static int ceil_lg(int64_t k) {
  int l = 0;
  while ((int64_t(1) << l) < k) ++l;
  return l;
}

// Erasure pipeline with per-position tables shared by a batch (or by each
// stripe group: row stride *_stride per group), rs.py:130-148:
//   Phi = rx * pi_row -> n-point inverse -> derivative -> 2^lg_out-point
//   forward -> * pinv, written to out_io's window (merging survivors when
//   out_io.merge_src is set).  For lg_out <= r - 1 the XOR-only top inverse
//   level is folded into the derivative gather (T_j = W'_(r-1)(y_j + y_(j+n/2))
//   + sum_(l<r-1, bit l of j clear) y_(j|2^l), y_j = B_(j mod n/2) x_j); for
//   lg_out = r (k > n/2, or encode-by-decode) the plain schedule runs.
template <int R, uint32_t POLY>
static int erasure_core(lch_ctx *c, const RawIO &in0, const RawIO &out0, const uint16_t *pi_row,
                        int64_t pi_stride, const uint16_t *pinv, int64_t pinv_stride, int lg_out,
                        int64_t batch, int64_t pkt, cudaStream_t s) {
  const int r = c->t.r;
  const bool folded = lg_out <= r - 1;
  const int64_t ch = chunk_lanes(c, batch, pkt, bs_lane_bytes(R, r) + 2 * bs_lane_bytes(R, lg_out));
  Scratch sc(c, s);
  uint4 *x = nullptr, *t = nullptr, *t1 = nullptr;
  LCH_TRY(sc.alloc(x, bs_bytes(R, ch, r) / 16));
  LCH_TRY(sc.alloc(t, bs_bytes(R, ch, lg_out) / 16));
  LCH_TRY(sc.alloc(t1, bs_bytes(R, ch, lg_out) / 16));
  for (int64_t b0 = 0; b0 < batch; b0 += ch) {
    const int64_t nb = std::min(ch, batch - b0);
    const int64_t g0 = pkt ? b0 / pkt : 0;
    RawIO in_io = shift_io(in0, b0), out_io = shift_io(out0, b0);
    std::vector<LOp> a = {{OP_SCALE, 0, 0, pi_row + g0 * pi_stride, pi_stride}};
    const int ninv = folded ? r - 1 : r;
    for (int i = 0; i < ninv; ++i) a.push_back({OP_INV, i, 0u, nullptr});
    a.push_back({OP_SCALE, 0, 0, folded ? c->d_b_lo : c->d_b_prod});
    auto plan_a = plan_passes(a, r, true, false);
    // the last inverse pass also sums the gather over its own tile bits
    LCH_TRY((run_plan<R, POLY>(c, plan_a, r, nb, &in_io, nullptr, nullptr, x, s, t1, lg_out, pkt)));
    std::vector<int> rest;
    const auto &lb = plan_a.back().bits;
    for (int b = 0; b < ninv; ++b)
      if (std::find(lb.begin(), lb.end(), b) == lb.end()) rest.push_back(b);
    if (folded) rest.push_back(r - 1);
    LCH_TRY((run_gather<R, POLY>(c, x, t, r, lg_out, nb, rest, folded ? r - 1 : -1,
                                 folded ? c->t.w_prime[r - 1] : 0u, t1, s)));
    std::vector<LOp> b = {{OP_SCALE, 0, 0, c->d_b_prod_inv}};
    for (int i = lg_out - 1; i >= 0; --i) b.push_back({OP_FWD, i, 0u, nullptr});
    b.push_back({OP_SCALE, 0, 0, pinv + g0 * pinv_stride, pinv_stride});
    LCH_TRY((run_plan<R, POLY>(c, plan_passes(b, lg_out, false, true), lg_out, nb, nullptr, t, &out_io,
                               t, s, nullptr, 0, pkt)));
  }
  return LCH_OK;
}

// per-pattern erasure counts (host), from host_counts or a device reduction
static int pattern_counts(lch_ctx *c, const uint32_t *bits, int64_t np, int words,
                          const int64_t *host_counts, std::vector<int64_t> &counts,
                          cudaStream_t s) {
  counts.assign(size_t(np), 0);
  if (host_counts) {
    std::memcpy(counts.data(), host_counts, sizeof(int64_t) * size_t(np));
    return LCH_OK;
  }
  Scratch sc(c, s);
  int64_t *dc = nullptr;
  LCH_TRY(sc.alloc(dc, size_t(np)));
  LCH_TRY(cu(launch_count_bits(bits, np, words, dc, s)));
  c->launches++;
  LCH_TRY(cu(cudaMemcpyAsync(counts.data(), dc, sizeof(int64_t) * size_t(np), cudaMemcpyDeviceToHost, s)));
  return cu(cudaStreamSynchronize(s));
}

// locator logs -> pi_row [np][n] and pinv [np][kf] (rs.py:125-148)
static int erasure_tables(lch_ctx *c, const uint32_t *bits, int64_t np, int64_t kf, Scratch &sc,
                          uint16_t *&pi_row, uint16_t *&pinv, cudaStream_t s) {
  const int64_t n = int64_t(c->t.order);
  uint16_t *logs = nullptr;
  LCH_TRY(sc.alloc(logs, size_t(np * n)));
  LCH_TRY(sc.alloc(pi_row, size_t(np * n)));
  LCH_TRY(sc.alloc(pinv, size_t(np * kf)));
  LCH_TRY(locator_impl(c, bits, np, nullptr, logs, s));
  LCH_TRY(cu(launch_decode_rows(logs, bits, c->d_exp, c->t.m, uint32_t(n), uint32_t(kf), pi_row, pinv,
                                np, s)));
  c->launches++;
  return LCH_OK;
}

static int transform_impl(lch_ctx *c, uint16_t *data, int64_t batch, int64_t stride, int lg_h,
                          uint32_t shift, int64_t pkt, void *stream, bool inverse) {
  if (!c || lg_h < 0 || lg_h > c->max_lg_h || batch < 0) return LCH_EINVAL;
  if (shift >= c->t.order) return LCH_EINVAL;
  LCH_TRY(check_layout(data, batch, pkt));
  const int64_t h = int64_t(1) << lg_h;
  if (stride < h) return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  if (batch == 0 || lg_h == 0) return LCH_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<LOp> ops;
  if (inverse)
    for (int i = 0; i < lg_h; ++i) ops.push_back({OP_INV, i, hs_of(c, i, shift), nullptr});
  else
    for (int i = lg_h - 1; i >= 0; --i) ops.push_back({OP_FWD, i, hs_of(c, i, shift), nullptr});
  return dispatch(c, [&](auto RC, auto PC) -> int {
    constexpr int R = decltype(RC)::value;
    constexpr uint32_t P = decltype(PC)::value;
    auto plan = plan_passes(ops, lg_h, true, true);
    const int64_t ch = plan.size() > 1 ? chunk_lanes(c, batch, pkt, bs_lane_bytes(R, lg_h)) : batch;
    Scratch sc(c, s);
    uint4 *work = nullptr;
    if (plan.size() > 1) LCH_TRY(sc.alloc(work, bs_bytes(R, ch, lg_h) / 16));
    const RawIO io0 = make_io(data, stride, pkt);
    for (int64_t b0 = 0; b0 < batch; b0 += ch) {
      RawIO io = shift_io(io0, b0);
      LCH_TRY((run_plan<R, P>(c, plan, lg_h, std::min(ch, batch - b0), &io, nullptr, &io, work, s,
                              nullptr, 0, pkt)));
    }
    return LCH_OK;
  });
}

// Small GF(2^8) batches (fewer than one 1024-codeword bit-sliced group): one
// CTA per codeword (lch_small.cu), a single launch per encode / decode.
static bool small8_ok(const lch_ctx *c, int64_t batch, int64_t pkt) {
  return c->t.r == 8 && c->t.poly == 0x11Du && pkt == 0 && batch > 0 && batch < GROUP &&
         c->max_lg_h == 8 && !std::getenv("LCH_NO_SMALL8");
}

static Small8Params small8_params(const lch_ctx *c) {
  Small8Params p;
  std::memset(&p, 0, sizeof(p));
  p.max_h = int(c->t.max_h);
  p.log = c->d_log;
  p.exp = c->d_exp;
  p.w_hat = c->d_w_hat;
  p.b_prod = c->d_b_prod;
  p.b_prod_inv = c->d_b_prod_inv;
  p.fwht_log = c->d_fwht_log;
  return p;
}

// Systematic encode for power-of-two k (rs.py:85-96).
// Code length 2^lg_n (<= the field size): parity blocks at shifts k, 2k, ...
// (a sub-code of a longer one evaluates the same polynomials on its first
// 2^lg_n points, so the shift constants are the field's).
static int encode_pow2(lch_ctx *c, const uint16_t *msg, int64_t stride_in, uint16_t *parity,
                       int64_t stride_out, int64_t batch, int lg_k, int64_t pkt, cudaStream_t s,
                       int lg_n = -1) {
  if (lg_n < 0) lg_n = c->t.r;
  const int64_t k = int64_t(1) << lg_k, nb = (int64_t(1) << lg_n) / k;
  if (nb == 1) return LCH_OK;
  if (small8_ok(c, batch, pkt) && lg_n == c->t.r) {
    Small8Params p = small8_params(c);
    p.mode = 0;
    p.k = int(k);
    p.lg_k = lg_k;
    p.batch = batch;
    p.in = msg;
    p.in_stride = stride_in;
    p.out = parity;
    p.out_stride = stride_out;
    for (int64_t blk = 1; blk < nb; ++blk)
      for (int i = 0; i < lg_k; ++i) p.hs[blk * 8 + i] = uint8_t(hs_of(c, i, uint32_t(blk * k)));
    LCH_TRY(cu(launch_small8(p, s)));
    c->launches++;
    return LCH_OK;
  }
  if (lg_k == 0) {
    // 1-point transforms are the identity: every parity symbol is the message
    const int64_t rows = pkt ? batch / pkt : batch, w = pkt ? pkt : 1;
    const size_t sp_out = size_t(pkt ? stride_out * pkt : stride_out) * 2;
    const size_t sp_in = size_t(pkt ? stride_in * pkt : stride_in) * 2;
    for (int64_t i = 1; i < nb; ++i)
      LCH_TRY(cu(cudaMemcpy2DAsync(at_pos(parity, i - 1, pkt), sp_out, msg, sp_in, size_t(w) * 2,
                                   size_t(rows), cudaMemcpyDeviceToDevice, s)));
    return LCH_OK;
  }
  return dispatch(c, [&](auto RC, auto PC) -> int {
    constexpr int R = decltype(RC)::value;
    constexpr uint32_t P = decltype(PC)::value;
    Scratch sc(c, s);
    const RawIO in0 = make_io(msg, stride_in, pkt);
    // rs.py:91 coefficients by a k-point inverse at shift 0
    std::vector<LOp> inv;
    for (int i = 0; i < lg_k; ++i) inv.push_back({OP_INV, i, 0u, nullptr});
    if (nb == 2) {
      // rs.py:93-95 with one parity block: fuse inverse and forward(shift k)
      // The top inverse level and the first forward level act on the same
      // pairs: v' = u + v, u' = u + f1 v', then u'' = u' + f2 v', v'' = u'' + v',
      // i.e. one multiply by f1 + f2 = W^_top(0) + W^_top(k) (the table parts
      // cancel) -- one op, and every round of the middle pass stays a
      // straight-line one.
      std::vector<LOp> ops(inv.begin(), inv.end() - (lg_k > 0 ? 1 : 0));
      if (lg_k > 0) ops.push_back({OP_INVFWD, lg_k - 1, hs_of(c, lg_k - 1, uint32_t(k)), nullptr});
      for (int i = lg_k - 2; i >= 0; --i) ops.push_back({OP_FWD, i, hs_of(c, i, uint32_t(k)), nullptr});
      auto plan = plan_passes(ops, lg_k, true, true);
      const int64_t ch = plan.size() > 1 ? chunk_lanes(c, batch, pkt, bs_lane_bytes(R, lg_k)) : batch;
      uint4 *work = nullptr;
      if (plan.size() > 1) LCH_TRY(sc.alloc(work, bs_bytes(R, ch, lg_k) / 16));
      const RawIO out0 = make_io(parity, stride_out, pkt);
      for (int64_t b0 = 0; b0 < batch; b0 += ch) {
        RawIO in_io = shift_io(in0, b0), out_io = shift_io(out0, b0);
        LCH_TRY((run_plan<R, P>(c, plan, lg_k, std::min(ch, batch - b0), &in_io, nullptr, &out_io, work,
                                s, nullptr, 0, pkt)));
      }
      return LCH_OK;
    }
    const int64_t ch = chunk_lanes(c, batch, pkt, 2 * bs_lane_bytes(R, lg_k));
    uint4 *coef = nullptr, *work = nullptr;
    LCH_TRY(sc.alloc(coef, bs_bytes(R, ch, lg_k) / 16));
    LCH_TRY(sc.alloc(work, bs_bytes(R, ch, lg_k) / 16));
    for (int64_t b0 = 0; b0 < batch; b0 += ch) {
      const int64_t bn = std::min(ch, batch - b0);
      RawIO in_io = shift_io(in0, b0);
      LCH_TRY((run_plan<R, P>(c, plan_passes(inv, lg_k, true, false), lg_k, bn, &in_io, nullptr,
                              nullptr, coef, s, nullptr, 0, pkt)));
      for (int64_t blk = 1; blk < nb; ++blk) {
        std::vector<LOp> fwd;
        const uint32_t shift = uint32_t(blk * k);
        for (int i = lg_k - 1; i >= 0; --i) fwd.push_back({OP_FWD, i, hs_of(c, i, shift), nullptr});
        RawIO out_io = shift_io(make_io(at_pos(parity, (blk - 1) * k, pkt), stride_out, pkt), b0);
        LCH_TRY((run_plan<R, P>(c, plan_passes(fwd, lg_k, false, true), lg_k, bn, nullptr, coef,
                                &out_io, work, s, nullptr, 0, pkt)));
      }
    }
    return LCH_OK;
  });
}

// Encode-by-erasure-decode tables for E = [k, n): pi_row [n], pinv [n]
// (cached per k on the context).
static int encode_tables(lch_ctx *c, int64_t k, const uint16_t *&pi_row, const uint16_t *&pinv,
                         cudaStream_t s) {
  const int64_t n = int64_t(c->t.order);
  {
    std::lock_guard<std::mutex> g(c->mu);
    for (auto &e : c->enc_tabs)
      if (e.first == k) {
        pi_row = e.second;
        pinv = e.second + n;
        return LCH_OK;
      }
  }
  const int words = int(std::max<int64_t>(n / 32, 1));
  std::vector<uint32_t> hb(size_t(words), 0u);
  for (int64_t j = k; j < n; ++j) hb[size_t(j >> 5)] |= 1u << (j & 31);
  uint16_t *tab = nullptr;
  LCH_TRY(cu(cudaMalloc(&tab, size_t(2 * n) * 2)));
  int rc;
  {
    Scratch sc(c, s);
    uint32_t *db = nullptr;
    uint16_t *pr = nullptr, *pv = nullptr;
    rc = sc.alloc(db, size_t(words));
    if (rc == LCH_OK) rc = cu(cudaMemcpyAsync(db, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice, s));
    if (rc == LCH_OK) rc = erasure_tables(c, db, 1, n, sc, pr, pv, s);
    if (rc == LCH_OK) rc = cu(cudaMemcpyAsync(tab, pr, size_t(n) * 2, cudaMemcpyDeviceToDevice, s));
    if (rc == LCH_OK) rc = cu(cudaMemcpyAsync(tab + n, pv, size_t(n) * 2, cudaMemcpyDeviceToDevice, s));
  }
  if (rc == LCH_OK) rc = cu(cudaStreamSynchronize(s));
  if (rc != LCH_OK) {
    cudaFree(tab);
    return rc;
  }
  std::lock_guard<std::mutex> g(c->mu);
  c->enc_tabs.push_back({k, tab});
  pi_row = tab;
  pinv = tab + n;
  return LCH_OK;
}

// ---------------------------------------------------------------------------
// Systematic encode for any k ("a first-class codec"): the
// codeword is the evaluation of the degree < k interpolant f of the message
// (the code of SURVEY H6), computed by recursion on the binary expansion of k
// instead of erasure decoding.  With h = n/2 and k > h, f = A + X_h R where
// deg A < h: X_h vanishes on [0, h) and is 1 on [h, n) (normalised subspace
// polynomial), so A interpolates m on [0, h), its values on [h, n) are the
// parity of the power-of-two code (2h, h) (rs.encode), and R is the degree
// < k - h interpolant of m - A on [h, k), a smaller instance of the same
// problem on the coset [h, n).  Parity = A + R on [k, n).  For k < h not a
// power of two the first 2^ceil(lg k) values are completed recursively and
// then encoded as a power-of-two code.  Every step is a power-of-two encode
// (the fused pass-kernel plans) or an XOR of arrays.

struct View {
  uint16_t *p;
  int64_t s;  // row stride (row layout) or positions per stripe group (packet layout)
};

static View vsub(View v, int64_t j0, int64_t pkt) { return View{at_pos(v.p, j0, pkt), v.s}; }

static int vtemp(Scratch &sc, int64_t batch, int64_t len, View &v) {
  LCH_TRY(sc.alloc(v.p, size_t(std::max<int64_t>(batch * len, 1))));
  v.s = len;
  return LCH_OK;
}

// out = a ^ b (b.p == nullptr: copy) over positions [0, len)
static int vxor(lch_ctx *c, View out, View a, View b, int64_t batch, int64_t len, int64_t pkt,
                cudaStream_t s) {
  if (len <= 0 || batch <= 0) return LCH_OK;
  c->launches++;
  return cu(launch_xor_views(out.p, out.s, a.p, a.s, b.p, b.s, batch, len, pkt, s));
}

static int ilog2(int64_t x) {
  int l = 0;
  while ((int64_t(1) << (l + 1)) <= x) ++l;
  return l;
}

// values on [K, np) of the degree < K interpolant of v on [0, K)
static int solve_interp(lch_ctx *c, View v, View out, int64_t batch, int64_t np, int64_t K,
                        int64_t pkt, cudaStream_t s, Scratch &sc) {
  if (K >= np) return LCH_OK;
  if ((K & (K - 1)) == 0)
    return encode_pow2(c, v.p, v.s, out.p, out.s, batch, ilog2(K), pkt, s, ilog2(np));
  const int64_t h = np / 2;
  if (K > h) {
    View a{}, diff{}, sub{};
    LCH_TRY(vtemp(sc, batch, h, a));
    LCH_TRY(encode_pow2(c, v.p, v.s, a.p, a.s, batch, ilog2(h), pkt, s, ilog2(np)));  // A on [h, np)
    LCH_TRY(vtemp(sc, batch, K - h, diff));
    LCH_TRY(vxor(c, diff, vsub(v, h, pkt), a, batch, K - h, pkt, s));  // m - A on [h, K)
    LCH_TRY(vtemp(sc, batch, np - K, sub));
    LCH_TRY(solve_interp(c, diff, sub, batch, h, K - h, pkt, s, sc));  // R on [K, np)
    return vxor(c, out, vsub(a, K - h, pkt), sub, batch, np - K, pkt, s);
  }
  int64_t t = 1;
  while (t < K) t <<= 1;
  View full{};
  LCH_TRY(vtemp(sc, batch, t, full));
  LCH_TRY(vxor(c, full, v, View{nullptr, 0}, batch, K, pkt, s));
  LCH_TRY(solve_interp(c, v, vsub(full, K, pkt), batch, t, K, pkt, s, sc));
  LCH_TRY(vxor(c, out, vsub(full, K, pkt), View{nullptr, 0}, batch, t - K, pkt, s));
  if (t < np)
    LCH_TRY(encode_pow2(c, full.p, full.s, at_pos(out.p, t - K, pkt), out.s, batch, ilog2(t), pkt, s,
                        ilog2(np)));
  return LCH_OK;
}

static int encode_general(lch_ctx *c, const uint16_t *msg, int64_t stride_in, uint16_t *parity,
                          int64_t stride_out, int64_t batch, int64_t k, int64_t pkt, cudaStream_t s) {
  const int64_t n = int64_t(c->t.order);
  // temporaries: ~2n symbols per lane at the top level of the recursion
  const int64_t ch = chunk_lanes(c, batch, pkt, size_t(4 * n));
  for (int64_t b0 = 0; b0 < batch; b0 += ch) {
    const int64_t nb = std::min(ch, batch - b0);
    const int64_t off_in = pkt ? (b0 / pkt) * stride_in * pkt : b0 * stride_in;
    const int64_t off_out = pkt ? (b0 / pkt) * stride_out * pkt : b0 * stride_out;
    Scratch sc(c, s);
    LCH_TRY(solve_interp(c, View{const_cast<uint16_t *>(msg) + off_in, stride_in},
                         View{parity + off_out, stride_out}, nb, n, k, pkt, s, sc));
  }
  return LCH_OK;
}

static int encode_any(lch_ctx *c, const uint16_t *msg, int64_t stride_in, uint16_t *parity,
                      int64_t stride_out, int64_t batch, int64_t k, int64_t pkt, void *stream) {
  if (!c || batch < 0) return LCH_EINVAL;
  const int64_t n = int64_t(c->t.order);
  if (k < 1 || k > n) return LCH_EINVAL;
  LCH_TRY(check_layout(msg, batch, pkt));
  LCH_TRY(check_layout(parity, batch, pkt));
  if (stride_in < k || (k < n && stride_out < n - k)) return LCH_EINVAL;
  const bool pow2 = (k & (k - 1)) == 0;
  if (pow2 && ceil_lg(k) > c->max_lg_h) return LCH_EINVAL;  // rs.py:162-163
  if (!pow2 && c->max_lg_h < c->t.r) return LCH_EINVAL;      // n-point transforms
  LCH_TRY(ensure_device(c));
  if (batch == 0 || k == n) return LCH_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (pow2) return encode_pow2(c, msg, stride_in, parity, stride_out, batch, ceil_lg(k), pkt, s);
  if (!std::getenv("LCH_ENCODE_BY_DECODE"))
    return encode_general(c, msg, stride_in, parity, stride_out, batch, k, pkt, s);
  // encode-by-erasure-decode (same codeword; kept for cross-checks)
  const uint16_t *pi_row = nullptr, *pinv = nullptr;
  LCH_TRY(encode_tables(c, k, pi_row, pinv, s));
  RawIO in_io = make_io(msg, stride_in, pkt);
  in_io.pos_hi = k;  // positions >= k (erased) read as zero
  RawIO out_io = make_io(parity, stride_out, pkt);
  out_io.pos_lo = k;  // parity = positions [k, n)
  out_io.pos_hi = n;
  return dispatch(c, [&](auto RC, auto PC) -> int {
    constexpr int R = decltype(RC)::value;
    constexpr uint32_t P = decltype(PC)::value;
    return erasure_core<R, P>(c, in_io, out_io, pi_row, 0, pinv, 0, c->t.r, batch, pkt, s);
  });
}

// Decode with one erasure pattern per row (rs.decode row by row): batched
// locator whose epilogue writes phi = rx * Pi_bar (rs.py:130-134) and
// -log Pi' (rs.py:141-148); the shared transform pipeline without the
// per-position scaling; the output epilogue divides erased symbols by Pi'.
static int decode_per_codeword(lch_ctx *c, const uint16_t *rx, int64_t stride_in,
                               const uint32_t *bits, uint16_t *out, int64_t stride_out,
                               int64_t batch, int64_t k, cudaStream_t s) {
  const int r = c->t.r;
  const int64_t n = int64_t(c->t.order);
  const int lgo = std::max(ceil_lg(k), 1);
  const int64_t kf = int64_t(1) << lgo;  // forward length (first kf outputs)
  const bool folded = lgo <= r - 1;      // k > n/2: the unfolded schedule (see erasure_core)
  return dispatch(c, [&](auto RC, auto PC) -> int {
    constexpr int R = decltype(RC)::value;
    constexpr uint32_t P = decltype(PC)::value;
    Scratch sc(c, s);
    uint16_t *phi = nullptr, *pinv_log = nullptr;
    LCH_TRY(sc.alloc(phi, size_t(batch) * size_t(stride_in)));
    LCH_TRY(sc.alloc(pinv_log, size_t(batch) * size_t(kf)));
    DecodeEpi epi;
    epi.rx = rx;
    epi.rx_stride = stride_in;  // phi is written with the received words' row stride
    epi.phi = phi;
    epi.pinv_log = pinv_log;
    epi.k = uint32_t(kf);  // bound and row stride of pinv_log
    LCH_TRY(locator_impl(c, bits, batch, nullptr, nullptr, s, &epi));
    const int64_t ch = chunk_lanes(c, batch, 0, bs_lane_bytes(R, r) + 2 * bs_lane_bytes(R, lgo));
    uint4 *x = nullptr, *t = nullptr, *t1 = nullptr;
    LCH_TRY(sc.alloc(x, bs_bytes(R, ch, r) / 16));
    LCH_TRY(sc.alloc(t, bs_bytes(R, ch, lgo) / 16));
    LCH_TRY(sc.alloc(t1, bs_bytes(R, ch, lgo) / 16));
    const RawIO in0 = make_raw(phi, stride_in);
    RawIO out0 = make_raw(out, stride_out);
    out0.pos_hi = k;
    out0.merge_src = rx;
    out0.merge_stride = stride_in;
    out0.merge_bits = bits;
    out0.bits_stride = n / 32;
    out0.pinv_log = pinv_log;
    out0.pinv_stride = kf;
    out0.pinv_val = epi.pinv_val ? 1 : 0;
    out0.log_tab = c->d_log;
    out0.exp_tab = c->d_exp;
    out0.mord = c->t.m;
    out0.vec = out0.vec && (reinterpret_cast<uintptr_t>(rx) % 16 == 0) && (stride_in % 8 == 0);
    for (int64_t b0 = 0; b0 < batch; b0 += ch) {
      const int64_t nb = std::min(ch, batch - b0);
      RawIO in_io = shift_io(in0, b0), out_io = shift_io(out0, b0);
      std::vector<LOp> a;
      const int ninv = folded ? r - 1 : r;
      for (int i = 0; i < ninv; ++i) a.push_back({OP_INV, i, 0u, nullptr});
      a.push_back({OP_SCALE, 0, 0, folded ? c->d_b_lo : c->d_b_prod});
      auto plan_a = plan_passes(a, r, true, false);
      LCH_TRY((run_plan<R, P>(c, plan_a, r, nb, &in_io, nullptr, nullptr, x, s, t1, lgo)));
      std::vector<int> rest;
      const auto &lb = plan_a.back().bits;
      for (int b = 0; b < ninv; ++b)
        if (std::find(lb.begin(), lb.end(), b) == lb.end()) rest.push_back(b);
      if (folded) rest.push_back(r - 1);
      LCH_TRY((run_gather<R, P>(c, x, t, r, lgo, nb, rest, folded ? r - 1 : -1,
                                folded ? c->t.w_prime[r - 1] : 0u, t1, s)));
      std::vector<LOp> b = {{OP_SCALE, 0, 0, c->d_b_prod_inv}};
      for (int i = lgo - 1; i >= 0; --i) b.push_back({OP_FWD, i, 0u, nullptr});
      LCH_TRY((run_plan<R, P>(c, plan_passes(b, lgo, false, true), lgo, nb, nullptr, t, &out_io, t, s)));
    }
    return LCH_OK;
  });
}

static int decode_any(lch_ctx *c, const uint16_t *rx, int64_t stride_in, const uint32_t *bits,
                      int shared, uint16_t *out, int64_t stride_out, int64_t batch, int64_t k,
                      int64_t pkt, const int64_t *host_counts, void *stream) {
  if (!c || batch < 0 || !bits) return LCH_EINVAL;
  const int r = c->t.r;
  const int64_t n = int64_t(c->t.order);
  if (k < 1 || k > n) return LCH_EINVAL;
  LCH_TRY(check_layout(rx, batch, pkt));
  LCH_TRY(check_layout(out, batch, pkt));
  if (stride_in < n || stride_out < k) return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  if (batch == 0) return LCH_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int words = int(std::max<int64_t>(n / 32, 1));
  const int64_t np = shared ? 1 : (pkt ? batch / pkt : batch);
  std::vector<int64_t> counts;
  LCH_TRY(pattern_counts(c, bits, np, words, host_counts, counts, s));
  int64_t maxc = 0;
  for (int64_t v : counts) maxc = std::max(maxc, v);
  if (maxc > n - k) return LCH_ETOOMANY;  // rs.py:121-123
  if (maxc == 0) {                        // rs.py:119-120
    const int64_t rows = pkt ? batch / pkt : batch, w = pkt ? k * pkt : k;
    const size_t sp_out = size_t(pkt ? stride_out * pkt : stride_out) * 2;
    const size_t sp_in = size_t(pkt ? stride_in * pkt : stride_in) * 2;
    return cu(cudaMemcpy2DAsync(out, sp_out, rx, sp_in, size_t(w) * 2, size_t(rows),
                                cudaMemcpyDeviceToDevice, s));
  }
  if (c->max_lg_h < r) return LCH_EINVAL;  // n-point transforms (transform.py:63-64)
  if (small8_ok(c, batch, pkt)) {
    Small8Params p = small8_params(c);
    p.mode = 1;
    p.k = int(k);
    p.batch = batch;
    p.in = rx;
    p.in_stride = stride_in;
    p.out = out;
    p.out_stride = stride_out;
    p.bits = bits;
    p.bits_stride = shared ? 0 : words;
    LCH_TRY(cu(launch_small8(p, s)));
    c->launches++;
    return LCH_OK;
  }
  if (!shared && !pkt) {
    // phi (n symbols) + -log Pi' + the bit-sliced intermediates per codeword
    const int64_t ch = chunk_lanes(c, batch, 0, size_t(n) * 2 * 4);
    for (int64_t b0 = 0; b0 < batch; b0 += ch)
      LCH_TRY(decode_per_codeword(c, rx + b0 * stride_in, stride_in, bits + b0 * words, out + b0 * stride_out,
                                  stride_out, std::min(ch, batch - b0), k, s));
    return LCH_OK;
  }
  const int lgo = std::max(ceil_lg(k), 1);
  const int64_t kf = int64_t(1) << lgo;
  Scratch sc(c, s);
  uint16_t *pi_row = nullptr, *pinv = nullptr;
  // rs.py:125 locator values, one per pattern
  LCH_TRY(erasure_tables(c, bits, np, kf, sc, pi_row, pinv, s));
  const RawIO in_io = make_io(rx, stride_in, pkt);
  RawIO out_io = make_io(out, stride_out, pkt);
  out_io.pos_hi = k;
  out_io.merge_src = rx;
  out_io.merge_stride = stride_in;
  out_io.merge_bits = bits;
  out_io.bits_stride = shared ? 0 : words;
  if (!pkt) out_io.vec = out_io.vec && (reinterpret_cast<uintptr_t>(rx) % 16 == 0) && (stride_in % 8 == 0);
  return dispatch(c, [&](auto RC, auto PC) -> int {
    constexpr int R = decltype(RC)::value;
    constexpr uint32_t P = decltype(PC)::value;
    return erasure_core<R, P>(c, in_io, out_io, pi_row, shared ? 0 : n, pinv, shared ? 0 : kf, lgo, batch,
                              pkt, s);
  });
}

extern "C" {

int lch_forward(lch_ctx *c, uint16_t *data, int64_t batch, int64_t stride, int lg_h, uint32_t shift,
                int64_t packet_len, void *stream) {
  return transform_impl(c, data, batch, stride, lg_h, shift, packet_len, stream, false);
}

int lch_inverse(lch_ctx *c, uint16_t *data, int64_t batch, int64_t stride, int lg_h, uint32_t shift,
                int64_t packet_len, void *stream) {
  return transform_impl(c, data, batch, stride, lg_h, shift, packet_len, stream, true);
}

int lch_derivative(lch_ctx *c, const uint16_t *in, uint16_t *out, int64_t batch, int64_t stride,
                   int lg_h, int64_t packet_len, void *stream) {
  if (!c || lg_h < 0 || lg_h > c->max_lg_h || batch < 0) return LCH_EINVAL;
  LCH_TRY(check_layout(in, batch, packet_len));
  LCH_TRY(check_layout(out, batch, packet_len));
  const int64_t h = int64_t(1) << lg_h, pkt = packet_len;
  if (stride < h) return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  if (batch == 0) return LCH_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (lg_h == 0) {
    const int64_t rows = pkt ? batch / pkt : batch, w = pkt ? pkt : 1;
    return cu(cudaMemset2DAsync(out, size_t(pkt ? stride * pkt : stride) * 2, 0, size_t(w) * 2,
                                size_t(rows), s));
  }
  return dispatch(c, [&](auto RC, auto PC) -> int {
    constexpr int R = decltype(RC)::value;
    constexpr uint32_t P = decltype(PC)::value;
    const int64_t ch = chunk_lanes(c, batch, pkt, 2 * bs_lane_bytes(R, lg_h));
    Scratch sc(c, s);
    uint4 *x = nullptr, *t = nullptr;
    LCH_TRY(sc.alloc(x, bs_bytes(R, ch, lg_h) / 16));
    LCH_TRY(sc.alloc(t, bs_bytes(R, ch, lg_h) / 16));
    const RawIO in0 = make_io(in, stride, pkt), out0 = make_io(out, stride, pkt);
    std::vector<int> all;
    for (int b = 0; b < lg_h; ++b) all.push_back(b);
    for (int64_t b0 = 0; b0 < batch; b0 += ch) {
      const int64_t nb = std::min(ch, batch - b0);
      RawIO in_io = shift_io(in0, b0), out_io = shift_io(out0, b0);
      // derivative.py:56 scale by B_i, :60-70 gather-XOR, :73-76 scale by B_j^-1
      std::vector<LOp> pre = {{OP_SCALE, 0, 0, c->d_b_prod}};
      LCH_TRY((run_plan<R, P>(c, plan_passes(pre, lg_h, true, false), lg_h, nb, &in_io, nullptr,
                              nullptr, x, s)));
      LCH_TRY((run_gather<R, P>(c, x, t, lg_h, lg_h, nb, all, -1, 0u, nullptr, s)));
      std::vector<LOp> post = {{OP_SCALE, 0, 0, c->d_b_prod_inv}};
      LCH_TRY((run_plan<R, P>(c, plan_passes(post, lg_h, false, true), lg_h, nb, nullptr, t, &out_io,
                              t, s)));
    }
    return LCH_OK;
  });
}

int lch_fwht(lch_ctx *c, uint32_t *data, int64_t batch, int lg_n, uint32_t modulus, void *stream) {
  if (!c || lg_n < 0 || lg_n > 24 || batch < 0 || modulus == 0) return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  if (batch == 0) return LCH_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int b0 = 0;
  do {
    FwhtParams p;
    std::memset(&p, 0, sizeof(p));
    p.data = data;
    p.nvec = batch;
    p.lgn = lg_n;
    p.b0 = b0;
    p.tb = std::min(8, lg_n - b0);
    p.mod = modulus;
    LCH_TRY(cu(launch_fwht(p, s)));
    c->launches++;
    b0 += 8;
  } while (b0 < lg_n);
  return LCH_OK;
}

int lch_locator(lch_ctx *c, const uint32_t *bits, int64_t np, uint16_t *loc_out, uint16_t *log_out,
                void *stream) {
  if (!c || np < 0 || !bits) return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  if (np == 0) return LCH_OK;
  return locator_impl(c, bits, np, loc_out, log_out, static_cast<cudaStream_t>(stream));
}

int lch_encode(lch_ctx *c, const uint16_t *msg, int64_t stride_in, uint16_t *parity,
               int64_t stride_out, int64_t batch, int lg_k, int64_t packet_len, void *stream) {
  if (!c || lg_k < 0 || lg_k > c->t.r) return LCH_EINVAL;
  return encode_any(c, msg, stride_in, parity, stride_out, batch, int64_t(1) << lg_k, packet_len,
                    stream);
}

int lch_encode_k(lch_ctx *c, const uint16_t *msg, int64_t stride_in, uint16_t *parity,
                 int64_t stride_out, int64_t batch, int64_t k, int64_t packet_len, void *stream) {
  return encode_any(c, msg, stride_in, parity, stride_out, batch, k, packet_len, stream);
}

int lch_decode(lch_ctx *c, const uint16_t *rx, int64_t stride_in, const uint32_t *bits, int shared,
               uint16_t *out, int64_t stride_out, int64_t batch, int lg_k, int64_t packet_len,
               const int64_t *host_counts, void *stream) {
  if (!c || lg_k < 0 || lg_k > c->t.r) return LCH_EINVAL;
  if (lg_k > c->max_lg_h) return LCH_EINVAL;
  return decode_any(c, rx, stride_in, bits, shared, out, stride_out, batch, int64_t(1) << lg_k,
                    packet_len, host_counts, stream);
}

int lch_decode_k(lch_ctx *c, const uint16_t *rx, int64_t stride_in, const uint32_t *bits, int shared,
                 uint16_t *out, int64_t stride_out, int64_t batch, int64_t k, int64_t packet_len,
                 const int64_t *host_counts, void *stream) {
  return decode_any(c, rx, stride_in, bits, shared, out, stride_out, batch, k, packet_len, host_counts,
                    stream);
}

// ---------------------------------------------------------------------------
// Host-buffer pipeline: chunks of rows (codewords, or stripe groups in packet
// layout) stream H2D on one stream, through the codec on the caller's
// stream, and D2H on a third, NS slots deep, so the copies of chunk i +- 1
// overlap the kernels of chunk i.  Everything is ordered after the work
// already queued on `stream`, and `stream` waits for the last copy.

}  // extern "C"

namespace {

struct HostArray {
  const uint8_t *src = nullptr;  // host input (or null)
  uint8_t *dst = nullptr;        // host output (or null)
  size_t row_bytes = 0;          // bytes copied per row
  size_t pitch = 0;              // host bytes between rows
  // optional host stage: fills rows [r0, r0 + nr) into a page-locked staging
  // buffer (row_bytes per row) that is then copied instead of src
  std::function<void(int64_t r0, int64_t nr, uint8_t *staging)> prep;
  // with both prep and src set, a chunk goes either through prep (row_bytes
  // per row) or straight from src (raw_row_bytes per row); `choose` picks per
  // chunk (true = raw), given whether the H2D stream is idle
  size_t raw_row_bytes = 0;
  std::function<bool(int64_t chunk_index, bool h2d_idle)> choose;
};

// grow-only page-locked staging buffers of the context
uint8_t *pinned_buffer(lch_ctx *c, size_t idx, size_t bytes) {
  std::lock_guard<std::mutex> g(c->mu);
  if (c->pinned.size() <= idx) c->pinned.resize(idx + 1, {0, nullptr});
  auto &e = c->pinned[idx];
  if (e.first < bytes) {
    if (e.second) cudaFreeHost(e.second);
    e.second = nullptr;
    e.first = 0;
    if (cudaHostAlloc(&e.second, bytes, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    e.first = bytes;
  }
  return static_cast<uint8_t *>(e.second);
}

// Small host -> device uploads through a ring of page-locked slots: an
// asynchronous copy from pageable memory would serialise the stream with
// the host (and with work queued before the call).
int upload_small(lch_ctx *c, void *dst, const void *src, size_t bytes, cudaStream_t s) {
  constexpr size_t SLOT = size_t(1) << 20;
  if (bytes > SLOT) return cu(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
  size_t slot;
  {
    std::lock_guard<std::mutex> g(c->mu);
    slot = c->ring_next++ % 16;
  }
  uint8_t *ring = pinned_buffer(c, 1000, 16 * SLOT);  // one allocation for all slots
  if (!ring) return LCH_ENOMEM;
  uint8_t *stg = ring + slot * SLOT;
  cudaEvent_t &ev = c->ring_ev[slot];
  if (ev) LCH_TRY(cu(cudaEventSynchronize(ev)));
  else LCH_TRY(cu(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)));
  std::memcpy(stg, src, bytes);
  LCH_TRY(cu(cudaMemcpyAsync(dst, stg, bytes, cudaMemcpyHostToDevice, s)));
  return cu(cudaEventRecord(ev, s));
}

HostPool &host_pool(lch_ctx *c) {
  std::lock_guard<std::mutex> g(c->mu);
  if (!c->pool) {
    // share the host cores between the ranks of one node (torchrun exports
    // LOCAL_WORLD_SIZE); LCH_HOST_THREADS overrides
    unsigned hc = std::thread::hardware_concurrency();
    if (!hc) hc = 1;
    const char *lws = std::getenv("LOCAL_WORLD_SIZE");
    const unsigned ranks = lws ? unsigned(std::max(1, std::atoi(lws))) : 1u;
    unsigned nt = std::max(1u, std::min(hc / ranks, 16u));
    if (const char *ov = std::getenv("LCH_HOST_THREADS")) nt = unsigned(std::max(1, std::atoi(ov)));
    c->pool.reset(new HostPool(int(nt) - 1));
  }
  return *c->pool;
}

int host_streams(lch_ctx *c) {
  std::lock_guard<std::mutex> g(c->mu);
  if (!c->s_h2d) LCH_TRY(cu(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking)));
  if (!c->s_d2h) LCH_TRY(cu(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking)));
  return LCH_OK;
}

// ins: host inputs copied per chunk; out: the host output; compute(d_ins,
// d_out, row0, rows) runs the codec on the caller's stream.
// raw: the chunk's first input came straight from src (HostArray::choose)
using ChunkFn = std::function<int(const std::vector<const uint8_t *> &, uint8_t *, int64_t, int64_t, bool raw)>;

// grow-only device buffers of the pipeline slots (kept across calls)
uint8_t *pipe_buffer(lch_ctx *c, size_t idx, size_t bytes) {
  std::lock_guard<std::mutex> g(c->mu);
  if (c->pipe_dev.size() <= idx) c->pipe_dev.resize(idx + 1, {0, nullptr});
  auto &e = c->pipe_dev[idx];
  if (e.first < bytes) {
    if (e.second) {
      cudaDeviceSynchronize();  // an earlier call may still use the old buffer
      cudaFree(e.second);
    }
    e.second = nullptr;
    e.first = 0;
    if (cudaMalloc(&e.second, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    e.first = bytes;
  }
  return static_cast<uint8_t *>(e.second);
}

int host_pipeline(lch_ctx *c, cudaStream_t s, int64_t rows, int64_t chunk,
                  const std::vector<HostArray> &ins, const HostArray &out, const ChunkFn &compute) {
  constexpr int NS = 4;
  LCH_TRY(host_streams(c));
  const int ni = int(ins.size());
  if (ni > 2) return LCH_EINVAL;
  std::vector<uint8_t *> din(size_t(NS) * ni, nullptr), dout(NS, nullptr);
  for (int k = 0; k < NS; ++k) {
    for (int a = 0; a < ni; ++a) {
      din[size_t(k) * ni + a] =
          pipe_buffer(c, size_t(k) * 2 + a, std::max(ins[a].row_bytes, ins[a].raw_row_bytes) * size_t(chunk));
      if (!din[size_t(k) * ni + a]) return LCH_ENOMEM;
    }
    dout[k] = pipe_buffer(c, 8 + size_t(k), out.row_bytes * size_t(chunk));
    if (!dout[k]) return LCH_ENOMEM;
    for (cudaEvent_t *e : {&c->pipe_in_ready[k], &c->pipe_in_free[k], &c->pipe_out_free[k]})
      if (!*e) LCH_TRY(cu(cudaEventCreateWithFlags(e, cudaEventDisableTiming)));
  }
  // The slots and their events persist in the context: a slot's input buffer
  // is refilled once the codec of its previous chunk ran (in_free), its output
  // buffer once the previous D2H copy ran (out_free) -- in this call or in an
  // earlier one still in flight.  Host inputs are read right away (they are
  // complete when the call is made) unless the context asks for stream order.
  if (c->host_strict) {
    cudaEvent_t entry = nullptr;
    LCH_TRY(cu(cudaEventCreateWithFlags(&entry, cudaEventDisableTiming)));
    cudaError_t e1 = cudaEventRecord(entry, s);
    cudaError_t e2 = cudaStreamWaitEvent(c->s_h2d, entry, 0);
    cudaEventDestroy(entry);  // released once the recorded work completes
    LCH_TRY(cu(e1));
    LCH_TRY(cu(e2));
  }
  const int64_t nchunks = (rows + chunk - 1) / chunk;
  // LCH_PIPE_TRACE=1: per-chunk stage timestamps, printed by
  // lch_release_host_buffers (diagnostics; no synchronisation in the calls)
  static const bool trace = std::getenv("LCH_PIPE_TRACE") != nullptr;
  auto mark = [&](cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    c->trace_ev.push_back(e);
  };
  if (trace) c->trace_calls.push_back(c->trace_ev.size());
  mark(s);
  for (int64_t i = 0; i < nchunks; ++i) {
    const int k = int(i % NS);
    const int64_t r0 = i * chunk, nr = std::min(chunk, rows - r0);
    // input slot k is reusable once the codec of its previous chunk has consumed it
    LCH_TRY(cu(cudaStreamWaitEvent(c->s_h2d, c->pipe_in_free[k], 0)));
    std::vector<const uint8_t *> dptr(static_cast<size_t>(ni), nullptr);
    bool raw = false;
    for (int a = 0; a < ni; ++a) {
      const HostArray &h = ins[a];
      uint8_t *d = din[size_t(k) * ni + a];
      if (a == 0 && h.prep && h.src && h.choose) {
        // the H2D stream is idle when its last recorded copy has completed
        const bool idle = !c->last_h2d || cudaEventQuery(c->last_h2d) == cudaSuccess;
        cudaGetLastError();
        raw = h.choose(i, idle);
      }
      c->h2d_bytes += uint64_t(raw && a == 0 ? h.raw_row_bytes : h.row_bytes) * uint64_t(nr);
      if (raw && a == 0) {
        LCH_TRY(cu(cudaMemcpy2DAsync(d, h.raw_row_bytes, h.src + size_t(r0) * h.pitch, h.pitch, h.raw_row_bytes,
                                     size_t(nr), cudaMemcpyHostToDevice, c->s_h2d)));
      } else if (h.prep) {
        // the staging slot is free once the last H2D copy out of it has run --
        // in this call (chunk i - NS) or in an earlier call still in flight
        const size_t si = size_t(k) * ni + a;
        uint8_t *stg = pinned_buffer(c, si, h.row_bytes * size_t(chunk));
        if (!stg) return LCH_ENOMEM;
        cudaEvent_t sev = nullptr;
        {
          std::lock_guard<std::mutex> g(c->mu);
          if (c->stage_ev.size() <= si) c->stage_ev.resize(si + 1, nullptr);
          if (!c->stage_ev[si]) LCH_TRY(cu(cudaEventCreateWithFlags(&c->stage_ev[si], cudaEventDisableTiming)));
          sev = c->stage_ev[si];
        }
        LCH_TRY(cu(cudaEventSynchronize(sev)));
        h.prep(r0, nr, stg);
        LCH_TRY(cu(cudaMemcpyAsync(d, stg, h.row_bytes * size_t(nr), cudaMemcpyHostToDevice, c->s_h2d)));
        LCH_TRY(cu(cudaEventRecord(sev, c->s_h2d)));
      } else {
        LCH_TRY(cu(cudaMemcpy2DAsync(d, h.row_bytes, h.src + size_t(r0) * h.pitch, h.pitch, h.row_bytes,
                                     size_t(nr), cudaMemcpyHostToDevice, c->s_h2d)));
      }
      dptr[size_t(a)] = d;
    }
    mark(c->s_h2d);
    LCH_TRY(cu(cudaEventRecord(c->pipe_in_ready[k], c->s_h2d)));
    c->last_h2d = c->pipe_in_ready[k];
    LCH_TRY(cu(cudaStreamWaitEvent(s, c->pipe_in_ready[k], 0)));
    // output slot k is reusable once the D2H copy of its previous chunk has run
    LCH_TRY(cu(cudaStreamWaitEvent(s, c->pipe_out_free[k], 0)));
    const int crc = compute(dptr, dout[k], r0, nr, raw);
    if (crc != LCH_OK) return crc;
    mark(s);
    LCH_TRY(cu(cudaEventRecord(c->pipe_in_free[k], s)));
    LCH_TRY(cu(cudaStreamWaitEvent(c->s_d2h, c->pipe_in_free[k], 0)));
    LCH_TRY(cu(cudaMemcpy2DAsync(out.dst + size_t(r0) * out.pitch, out.pitch, dout[k], out.row_bytes,
                                 out.row_bytes, size_t(nr), cudaMemcpyDeviceToHost, c->s_d2h)));
    c->d2h_bytes += uint64_t(out.row_bytes) * uint64_t(nr);
    mark(c->s_d2h);
    LCH_TRY(cu(cudaEventRecord(c->pipe_out_free[k], c->s_d2h)));
  }
  // the caller's stream sees the outputs: it waits for the last copies
  for (int64_t i = std::max<int64_t>(0, nchunks - NS); i < nchunks; ++i)
    LCH_TRY(cu(cudaStreamWaitEvent(s, c->pipe_out_free[i % NS], 0)));
  return LCH_OK;
}

// Default rows per chunk: ~64 MiB of the larger per-row transfer, and in row
// layout whole bit-sliced groups of 1024 codewords (a partial group costs the
// kernels as much as a full one) once the batch has several.
int64_t default_chunk(int64_t rows, size_t row_bytes, int64_t pkt) {
  int64_t chunk = std::max<int64_t>(1, int64_t((size_t(64) << 20) / std::max<size_t>(row_bytes, 1)));
  if (!pkt && rows >= 2 * GROUP) chunk = std::max<int64_t>(GROUP, chunk / GROUP * GROUP);
  return chunk;
}

int64_t popcount_words(const uint32_t *w, int64_t n) {
  int64_t c = 0;
  for (int64_t i = 0; i < n; ++i) c += __builtin_popcount(w[i]);
  return c;
}

}  // namespace

extern "C" {

int lch_encode_host(lch_ctx *c, const uint16_t *host_msg, int64_t stride_in, uint16_t *host_parity,
                    int64_t stride_out, int64_t batch, int64_t k, int64_t packet_len, int64_t chunk,
                    void *stream) {
  if (!c || !host_msg || batch < 0 || chunk < 0 || packet_len < 0) return LCH_EINVAL;
  std::lock_guard<std::mutex> hg(c->host_mu);
  const int64_t n = int64_t(c->t.order), pkt = packet_len;
  if (k < 1 || k > n || stride_in < k || (k < n && (!host_parity || stride_out < n - k))) return LCH_EINVAL;
  if (pkt && (pkt % GROUP || batch % pkt)) return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  if (batch == 0 || k == n) return LCH_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // rows: codewords, or stripe groups of pkt lanes
  const int64_t rows = pkt ? batch / pkt : batch, lanes_per_row = pkt ? pkt : 1;
  const size_t in_row = size_t(k * lanes_per_row) * 2, out_row = size_t((n - k) * lanes_per_row) * 2;
  if (chunk == 0) chunk = default_chunk(rows, std::max(in_row, out_row), pkt);
  chunk = std::min(chunk, rows);
  std::vector<HostArray> ins(1);
  ins[0].src = reinterpret_cast<const uint8_t *>(host_msg);
  ins[0].row_bytes = in_row;
  ins[0].pitch = size_t(stride_in * lanes_per_row) * 2;
  HostArray out;
  out.dst = reinterpret_cast<uint8_t *>(host_parity);
  out.row_bytes = out_row;
  out.pitch = size_t(stride_out * lanes_per_row) * 2;
  return host_pipeline(c, s, rows, chunk, ins, out,
                       [&](const std::vector<const uint8_t *> &d, uint8_t *o, int64_t, int64_t nr, bool) {
                         return encode_any(c, reinterpret_cast<const uint16_t *>(d[0]), k,
                                           reinterpret_cast<uint16_t *>(o), n - k, nr * lanes_per_row, k,
                                           pkt, stream);
                       });
}

int lch_decode_host(lch_ctx *c, const uint16_t *host_rx, int64_t stride_in, const uint32_t *host_bits,
                    int shared, uint16_t *host_out, int64_t stride_out, int64_t batch, int64_t k,
                    int64_t packet_len, int64_t chunk, void *stream) {
  if (!c || !host_rx || !host_bits || !host_out || batch < 0 || chunk < 0 || packet_len < 0)
    return LCH_EINVAL;
  std::lock_guard<std::mutex> hg(c->host_mu);
  const int64_t n = int64_t(c->t.order), pkt = packet_len;
  if (k < 1 || k > n || stride_in < n || stride_out < k) return LCH_EINVAL;
  if (pkt && (pkt % GROUP || batch % pkt)) return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  if (batch == 0) return LCH_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t words = std::max<int64_t>(n / 32, 1);
  const int64_t rows = pkt ? batch / pkt : batch, lanes_per_row = pkt ? pkt : 1;
  // erasure counts from the host bitmasks (no device round trip)
  const int64_t npat = shared ? 1 : rows;
  std::vector<int64_t> counts(static_cast<size_t>(npat), 0);
  for (int64_t i = 0; i < npat; ++i) {
    counts[size_t(i)] = popcount_words(host_bits + i * words, words);
    if (counts[size_t(i)] > n - k) return LCH_ETOOMANY;  // rs.py:121-123
  }
  Scratch sc(c, s);
  uint32_t *d_shared = nullptr;
  if (shared) {
    LCH_TRY(sc.alloc(d_shared, size_t(words)));
    LCH_TRY(upload_small(c, d_shared, host_bits, size_t(words) * 4, s));
  }
  const size_t in_row = size_t(n * lanes_per_row) * 2, out_row = size_t(k * lanes_per_row) * 2;
  if (chunk == 0) chunk = default_chunk(rows, in_row / 2, pkt);
  chunk = std::min(chunk, rows);
  // LCH_COMPACT = all | none | alt | auto (default): which chunks of a
  // shared-pattern decode are compacted on the host (below)
  const char *cmode_env = std::getenv("LCH_COMPACT");
  const std::string cmode = std::getenv("LCH_NO_COMPACT") ? "none" : (cmode_env ? cmode_env : "auto");
  if (shared && !pkt && n >= 32 && cmode != "none") {
    // Only the survivors need to cross PCIe: the host compacts each row
    // (AVX-512 compress-store on the worker pool) into page-locked staging,
    // the device expands the rows back (erased positions read as zero; the
    // decoder ignores them, rs.py:130-134).  Compaction trades PCIe bytes for
    // host memory traffic (it reads the row and writes the survivors before
    // the DMA reads them again), so it is decided per chunk: a chunk is
    // compacted while the H2D stream still has copies to run (the host work
    // then hides behind them) and sent as it is when the stream has run dry.
    const int64_t surv = n - counts[0];
    std::vector<int32_t> rank(static_cast<size_t>(n), -1);
    for (int64_t j = 0, r = 0; j < n; ++j)
      if (!((host_bits[j >> 5] >> (j & 31)) & 1u)) rank[size_t(j)] = int32_t(r++);
    int32_t *d_rank = nullptr;
    LCH_TRY(sc.alloc(d_rank, size_t(n)));
    LCH_TRY(upload_small(c, d_rank, rank.data(), size_t(n) * 4, s));
    HostPool &pool = host_pool(c);
    const size_t crow = size_t(std::max<int64_t>(surv, 1)) * 2;
    std::vector<HostArray> cins(1);
    cins[0].row_bytes = crow;
    cins[0].prep = [&](int64_t r0, int64_t nr, uint8_t *stg) {
      compact_rows(pool, host_rx + r0 * stride_in, stride_in, host_bits, n, nr,
                   reinterpret_cast<uint16_t *>(stg), std::max<int64_t>(surv, 1));
    };
    if (cmode != "all") {
      cins[0].src = reinterpret_cast<const uint8_t *>(host_rx);
      cins[0].pitch = size_t(stride_in) * 2;
      cins[0].raw_row_bytes = size_t(n) * 2;
      cins[0].choose = [&](int64_t ci, bool idle) { return cmode == "alt" ? (ci & 1) != 0 : idle; };
    }
    HostArray cout;
    cout.dst = reinterpret_cast<uint8_t *>(host_out);
    cout.row_bytes = size_t(k) * 2;
    cout.pitch = size_t(stride_out) * 2;
    return host_pipeline(c, s, rows, chunk, cins, cout,
                         [&](const std::vector<const uint8_t *> &d, uint8_t *o, int64_t, int64_t nr, bool raw) {
                           if (raw)  // the chunk arrived as it is: rows of n symbols
                             return decode_any(c, reinterpret_cast<const uint16_t *>(d[0]), n, d_shared, 1,
                                               reinterpret_cast<uint16_t *>(o), k, nr, k, 0, counts.data(), stream);
                           Scratch cs(c, s);
                           uint16_t *full = nullptr;
                           LCH_TRY(cs.alloc(full, size_t(nr) * size_t(n)));
                           LCH_TRY(cu(launch_expand_rows(reinterpret_cast<const uint16_t *>(d[0]),
                                                         std::max<int64_t>(surv, 1), d_rank, full, n, nr, s)));
                           c->launches++;
                           return decode_any(c, full, n, d_shared, 1, reinterpret_cast<uint16_t *>(o), k, nr,
                                             k, 0, counts.data(), stream);
                         });
  }
  int64_t min_erased = counts.empty() ? 0 : counts[0];
  for (int64_t v : counts) min_erased = std::min(min_erased, v);
  // packing pays only when a large share of the packets is erased (the host
  // copy of the survivors then costs less than moving the erased ones)
  if (pkt && 5 * min_erased >= 2 * n && cmode != "none") {
    // Packet layout (stripe groups): erasures are whole packets, so only the
    // surviving packets cross PCIe -- the host packs them (memcpy per packet
    // on the worker pool) into page-locked staging, the device scatters them
    // back to their positions (erased packets read as zero).
    int64_t minc = counts[0];
    for (int64_t v : counts) minc = std::min(minc, v);
    const int64_t msurv = std::max<int64_t>(n - minc, 1);
    const size_t pkt_bytes = size_t(pkt) * 2;
    HostPool &pool = host_pool(c);
    std::vector<HostArray> cins(1);
    cins[0].row_bytes = size_t(msurv) * pkt_bytes;
    cins[0].prep = [&](int64_t r0, int64_t nr, uint8_t *stg) {
      for (int64_t g = r0; g < r0 + nr; ++g) {
        const uint32_t *gb = host_bits + (shared ? 0 : g * words);
        const uint8_t *src = reinterpret_cast<const uint8_t *>(host_rx) + size_t(g) * size_t(stride_in) * pkt_bytes;
        uint8_t *dst = stg + size_t(g - r0) * size_t(msurv) * pkt_bytes;
        // block prefix of survivors, then copy blocks of positions in parallel
        constexpr int64_t BLK = 256;
        const int64_t nblk = (n + BLK - 1) / BLK;
        std::vector<int64_t> pre(static_cast<size_t>(nblk) + 1, 0);
        for (int64_t bI = 0; bI < nblk; ++bI) {
          int64_t cnt = 0;
          for (int64_t j = bI * BLK; j < std::min(n, (bI + 1) * BLK); ++j) cnt += !((gb[j >> 5] >> (j & 31)) & 1u);
          pre[size_t(bI) + 1] = pre[size_t(bI)] + cnt;
        }
        pool.run(nblk, 1, [&](int64_t lo, int64_t hi) {
          for (int64_t bI = lo; bI < hi; ++bI) {
            int64_t q = pre[size_t(bI)];
            for (int64_t j = bI * BLK; j < std::min(n, (bI + 1) * BLK); ++j)
              if (!((gb[j >> 5] >> (j & 31)) & 1u))
                std::memcpy(dst + size_t(q++) * pkt_bytes, src + size_t(j) * pkt_bytes, pkt_bytes);
          }
        });
      }
    };
    HostArray cout;
    cout.dst = reinterpret_cast<uint8_t *>(host_out);
    cout.row_bytes = size_t(k) * pkt_bytes;
    cout.pitch = size_t(stride_out) * pkt_bytes;
    return host_pipeline(c, s, rows, chunk, cins, cout,
                         [&](const std::vector<const uint8_t *> &d, uint8_t *o, int64_t r0, int64_t nr, bool) {
                           Scratch cs(c, s);
                           const int64_t npat = shared ? 1 : nr;
                           std::vector<int32_t> rank(size_t(npat) * size_t(n), -1);
                           for (int64_t g = 0; g < npat; ++g) {
                             const uint32_t *gb = host_bits + (shared ? 0 : (r0 + g) * words);
                             for (int64_t j = 0, q = 0; j < n; ++j)
                               if (!((gb[j >> 5] >> (j & 31)) & 1u)) rank[size_t(g * n + j)] = int32_t(q++);
                           }
                           int32_t *d_rank = nullptr;
                           uint32_t *d_bits = d_shared;
                           uint16_t *full = nullptr;
                           LCH_TRY(cs.alloc(d_rank, rank.size()));
                           LCH_TRY(upload_small(c, d_rank, rank.data(), rank.size() * 4, s));
                           if (!shared) {
                             LCH_TRY(cs.alloc(d_bits, size_t(nr * words)));
                             LCH_TRY(upload_small(c, d_bits, host_bits + r0 * words, size_t(nr * words) * 4, s));
                           }
                           LCH_TRY(cs.alloc(full, size_t(nr) * size_t(n) * size_t(pkt)));
                           LCH_TRY(cu(launch_expand_packets(reinterpret_cast<const uint16_t *>(d[0]), msurv, d_rank,
                                                            shared ? 0 : n, full, n, pkt, nr, s)));
                           c->launches++;
                           return decode_any(c, full, n, d_bits, shared, reinterpret_cast<uint16_t *>(o), k,
                                             nr * pkt, k, pkt, counts.data() + (shared ? 0 : r0), stream);
                         });
  }
  std::vector<HostArray> ins(shared ? 1 : 2);
  ins[0].src = reinterpret_cast<const uint8_t *>(host_rx);
  ins[0].row_bytes = in_row;
  ins[0].pitch = size_t(stride_in * lanes_per_row) * 2;
  if (!shared) {
    ins[1].src = reinterpret_cast<const uint8_t *>(host_bits);
    ins[1].row_bytes = ins[1].pitch = size_t(words) * 4;
  }
  HostArray out;
  out.dst = reinterpret_cast<uint8_t *>(host_out);
  out.row_bytes = out_row;
  out.pitch = size_t(stride_out * lanes_per_row) * 2;
  return host_pipeline(c, s, rows, chunk, ins, out,
                       [&](const std::vector<const uint8_t *> &d, uint8_t *o, int64_t r0, int64_t nr, bool) {
                         const uint32_t *bits = shared ? d_shared : reinterpret_cast<const uint32_t *>(d[1]);
                         return decode_any(c, reinterpret_cast<const uint16_t *>(d[0]), n, bits, shared,
                                           reinterpret_cast<uint16_t *>(o), k, nr * lanes_per_row, k, pkt,
                                           counts.data() + (shared ? 0 : r0), stream);
                       });
}

int lch_compact_rows(lch_ctx *c, const uint16_t *host_rx, int64_t stride, const uint32_t *host_bits,
                     int64_t n, int64_t rows, uint16_t *host_out, int64_t out_stride) {
  if (!c || !host_rx || !host_bits || !host_out || n < 0 || rows < 0 || stride < n) return LCH_EINVAL;
  compact_rows(host_pool(c), host_rx, stride, host_bits, n, rows, host_out, out_stride);
  return LCH_OK;
}

int lch_set_host_ordering(lch_ctx *c, int stream_ordered) {
  if (!c) return LCH_EINVAL;
  std::lock_guard<std::mutex> hg(c->host_mu);
  c->host_strict = stream_ordered != 0;
  return LCH_OK;
}

int lch_host_copy_bytes(lch_ctx *c, uint64_t *h2d, uint64_t *d2h) {
  if (!c) return LCH_EINVAL;
  std::lock_guard<std::mutex> hg(c->host_mu);
  if (h2d) *h2d = c->h2d_bytes;
  if (d2h) *d2h = c->d2h_bytes;
  return LCH_OK;
}

int lch_release_host_buffers(lch_ctx *c) {
  if (!c) return LCH_EINVAL;
  std::lock_guard<std::mutex> hg(c->host_mu);
  if (!c->dev_ready) return LCH_OK;
  LCH_TRY(ensure_device(c));
  LCH_TRY(cu(cudaDeviceSynchronize()));
  std::lock_guard<std::mutex> g(c->mu);
  if (!c->trace_ev.empty()) {  // LCH_PIPE_TRACE: ms since the first call's entry
    for (size_t ci = 0; ci < c->trace_calls.size(); ++ci) {
      const size_t b = c->trace_calls[ci], e = ci + 1 < c->trace_calls.size() ? c->trace_calls[ci + 1] : c->trace_ev.size();
      std::fprintf(stderr, "call %zu:", ci);
      for (size_t i = b + 1; i < e; ++i) {
        float ms = 0;
        cudaEventElapsedTime(&ms, c->trace_ev[0], c->trace_ev[i]);
        std::fprintf(stderr, " %s%.2f", (i - b - 1) % 3 == 0 ? "| h2d " : (i - b - 1) % 3 == 1 ? "cmp " : "d2h ", ms);
      }
      std::fprintf(stderr, "\n");
    }
    for (cudaEvent_t e : c->trace_ev) cudaEventDestroy(e);
    c->trace_ev.clear();
    c->trace_calls.clear();
  }
  for (auto &e : c->pipe_dev) {
    if (e.second) cudaFree(e.second);
    e = {0, nullptr};
  }
  for (auto &e : c->pinned) {
    if (e.second) cudaFreeHost(e.second);
    e = {0, nullptr};
  }
  return LCH_OK;
}

int lch_set_scratch_limit(lch_ctx *c, uint64_t bytes) {
  if (!c || bytes == 0) return LCH_EINVAL;
  c->scratch_limit = size_t(bytes);
  return LCH_OK;
}

int lch_gen_symbols(lch_ctx *c, uint64_t seed, uint64_t cw0, int64_t batch, int64_t len, uint16_t *out,
                    int64_t stride, void *stream) {
  if (!c || batch < 0 || len < 0 || stride < len) return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  if (batch == 0 || len == 0) return LCH_OK;
  c->launches++;
  return cu(launch_gen_symbols(seed, cw0, batch, len, c->t.m, out, stride,
                               static_cast<cudaStream_t>(stream)));
}

int lch_gen_packets(lch_ctx *c, uint64_t seed, uint64_t cw0, int64_t batch, int64_t len, uint16_t *out,
                    int64_t n_pos, int64_t packet_len, void *stream) {
  if (!c || batch < 0 || len < 0 || n_pos < len || packet_len <= 0 || batch % packet_len) return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  if (batch == 0 || len == 0) return LCH_OK;
  c->launches++;
  return cu(launch_gen_packets(seed, cw0, batch, len, c->t.m, out, n_pos, packet_len,
                               static_cast<cudaStream_t>(stream)));
}

int lch_pointwise_mul(lch_ctx *c, const uint16_t *a, const uint16_t *b, uint16_t *out, int64_t count,
                      void *stream) {
  if (!c || count < 0 || (count && (!a || !b || !out))) return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  if (count == 0) return LCH_OK;
  c->launches++;
  // r = 16 with the reference polynomial: the table-free product (gf16_mul)
  const bool clmul = c->t.r == 16 && c->t.poly == 0x1100Bu;
  return cu(launch_pointwise_mul(a, b, out, count, clmul ? nullptr : c->d_log, c->d_exp, c->t.m,
                                 static_cast<cudaStream_t>(stream)));
}

int lch_derivative_direct(lch_ctx *c, const uint16_t *in, uint16_t *out, int64_t batch, int64_t row_stride,
                          int lg_h, void *stream) {
  if (!c || batch < 0 || lg_h < 0 || lg_h > c->max_lg_h || row_stride < (int64_t(1) << lg_h) ||
      (batch && (!in || !out)) || (batch && in == out))
    return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  if (batch == 0) return LCH_OK;
  WPrime wp{};
  for (int l = 0; l < c->t.r && l < 16; ++l) wp.w[l] = c->t.w_prime[l];
  wp.r = c->t.r;
  wp.poly = c->t.poly;
  c->launches++;
  return cu(launch_derivative_direct(in, out, batch, row_stride, lg_h, wp, static_cast<cudaStream_t>(stream)));
}

// ---- shard-file layouts (shardfile.py:109-140) ----------------------------

int lch_stripes_to_packets(lch_ctx *c, const uint8_t *file, int64_t len, int r, int64_t k,
                           uint16_t *packets, int64_t packet_len, void *stream) {
  if (!c || len < 0 || (r != 8 && r != 16) || k < 1 || packet_len < 1 || (len && !file) || !packets)
    return LCH_EINVAL;
  const int w = r / 8;
  const int64_t S = (len + k * w - 1) / (k * w);
  if (packet_len < S) return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  c->launches++;
  return cu(launch_stripes_to_packets(file, len, w, k, S, packets, packet_len,
                                      static_cast<cudaStream_t>(stream)));
}

int lch_packets_to_stripes(lch_ctx *c, const uint16_t *packets, int64_t packet_len, int r, int64_t k,
                           uint8_t *file, int64_t len, void *stream) {
  if (!c || len < 0 || (r != 8 && r != 16) || k < 1 || packet_len < 1 || !packets || (len && !file))
    return LCH_EINVAL;
  const int w = r / 8;
  if (packet_len < (len + k * w - 1) / (k * w)) return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  if (len == 0) return LCH_OK;
  c->launches++;
  return cu(launch_packets_to_stripes(packets, packet_len, k, w, file, len, static_cast<cudaStream_t>(stream)));
}

int lch_payload_to_packets(lch_ctx *c, const uint8_t *payload, int64_t rows, int64_t stripes, int r,
                           uint16_t *packets, int64_t packet_len, void *stream) {
  if (!c || rows < 0 || stripes < 0 || (r != 8 && r != 16) || packet_len < stripes || !packets) return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  if (rows == 0) return LCH_OK;
  c->launches++;
  return cu(launch_payload_packets(payload, packets, rows, stripes, packet_len, r / 8, 1, nullptr, nullptr,
                                   static_cast<cudaStream_t>(stream)));
}

int lch_packets_to_payload(lch_ctx *c, const uint16_t *packets, int64_t packet_len, int64_t rows,
                           int64_t stripes, int r, uint8_t *payload, void *stream) {
  if (!c || rows < 0 || stripes < 0 || (r != 8 && r != 16) || packet_len < stripes || !packets) return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  if (rows == 0 || stripes == 0) return LCH_OK;
  c->launches++;
  return cu(launch_payload_packets(nullptr, nullptr, rows, stripes, packet_len, r / 8, 0, payload, packets,
                                   static_cast<cudaStream_t>(stream)));
}

int lch_gen_keys(lch_ctx *c, uint64_t seed, uint64_t cw0, int64_t batch, int64_t len, int64_t *keys,
                 void *stream) {
  if (!c || batch < 0 || len < 0) return LCH_EINVAL;
  LCH_TRY(ensure_device(c));
  if (batch == 0 || len == 0) return LCH_OK;
  c->launches++;
  return cu(launch_gen_keys(seed, cw0, batch, len, keys, static_cast<cudaStream_t>(stream)));
}

}  // extern "C"
