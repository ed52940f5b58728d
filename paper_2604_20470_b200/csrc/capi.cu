// C-ABI entry points (include/dynrad.h): grid/config helpers, sparse
// attention forward, mask utilities, host-buffer convenience.  The mask
// builder entry points live in mask_build.cu.
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.hpp"
#include "plan.hpp"
#include "tmap.hpp"

// Pull in the kernel definitions (single translation unit keeps template
// instantiation and the launch sites together).
#include "attn_f32.cu"
#include "attn_sm100_db.cu"
#include "attn_sm100_rp.cu"
#include "csr.cu"
#include "random_batch.cu"

namespace rp {

static thread_local std::string t_err;

// ----------------------------------------------------- stage profiling --
namespace {
struct StageRec {
  int stage;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
std::atomic<bool> g_prof_on{false};
std::vector<StageRec> g_prof_recs;
std::vector<std::pair<int, cudaEvent_t>> g_prof_open;
}  // namespace
bool profiling_on() { return g_prof_on.load(std::memory_order_relaxed); }
void stage_begin(int stage, cudaStream_t s) {
  if (!profiling_on()) return;
  cudaEvent_t e;
  RP_CUDA(cudaEventCreate(&e));
  RP_CUDA(cudaEventRecord(e, s));
  std::lock_guard<std::mutex> lock(g_prof_mu);
  g_prof_open.emplace_back(stage, e);
}
void stage_end(int stage, cudaStream_t s) {
  if (!profiling_on()) return;
  cudaEvent_t e;
  RP_CUDA(cudaEventCreate(&e));
  RP_CUDA(cudaEventRecord(e, s));
  std::lock_guard<std::mutex> lock(g_prof_mu);
  for (auto it = g_prof_open.rbegin(); it != g_prof_open.rend(); ++it)
    if (it->first == stage) {
      g_prof_recs.push_back({stage, it->second, e});
      g_prof_open.erase(std::next(it).base());
      return;
    }
  cudaEventDestroy(e);
}
std::atomic<long long> g_launches{0};
void set_error(const std::string& msg) { t_err = msg; }

void require_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    throw CudaError("no CUDA device available (dynrad has no CPU fallback)");
  // stream-ordered scratch (static Fisher-Yates batches reach GBs) stays
  // mapped between calls: measured 1.5-8.7 s -> 107 ms for a static Wan build
  keep_pool_memory();
}

static int sm_count() {
  int dev = 0, n = 0;
  RP_CUDA(cudaGetDevice(&dev));
  RP_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

static void check_tensor(const rp_tensor* t, const char* name) {
  if (!t || !t->data) throw std::invalid_argument(std::string("tensor ") + name + ": null");
  if (t->tokens < 1 || t->heads < 1 || t->head_dim < 1)
    throw std::invalid_argument("feature batch: empty dimensions");
  if (t->dtype != RP_F32 && t->dtype != RP_BF16)
    throw std::invalid_argument(std::string("tensor ") + name + ": dtype must be f32 or bf16");
}

// Unit order of the stage-(d) kernels.  Natural (head-major, rows ascending):
// the 148 concurrently running CTAs work on consecutive block rows of one
// head, whose lists overlap, so K/V tiles are shared through L2.  LPT
// (rows by descending list length, DYNRAD_ORDER=lpt) balances the tail but
// scatters concurrent rows over the whole sequence: measured 8-9 % slower
// at the Wan shape (56.5-57.4 % vs 61.9 % of peak).  The row_order argument
// is therefore a hint that is used only under DYNRAD_ORDER=lpt.
static bool use_lpt_order() {
  static const bool lpt = [] {
    const char* e = std::getenv("DYNRAD_ORDER");
    return e && std::strcmp(e, "lpt") == 0;
  }();
  return lpt;
}

// Stage-(d) kernel.  "db" (attn_sm100_db.cu): one query tile per CTA, score
// tile double-buffered in TMEM, Q in TMEM, two softmax warps per row.  "rp"
// (attn_sm100_rp.cu): block-row pairs of one head sharing every K/V tile
// over their union list.  DYNRAD_K6=db|rp forces one; the default (auto) is
// db while one head's K + V fit in half of L2 and rp above that (measured in
// round 2, bench inputs: Wan 75.8 k tokens, 38.8 MB per head: db 22.0 ms vs
// rp 23.4-23.8 ms; Hunyuan 219.6 k tokens, 112 MB: db 107 ms vs rp 101 ms;
// DESIGN.md section 8).
// Measured alternatives (incl. round 2's two-tile ping-pong "pp") live in
// tools/experiments/k6_variants/.
enum class K6Variant { kAuto, kDB, kRP };
static K6Variant k6_forced() {
  static const K6Variant v = [] {
    const char* e = std::getenv("DYNRAD_K6");
    if (e && std::strcmp(e, "db") == 0) return K6Variant::kDB;
    if (e && std::strcmp(e, "rp") == 0) return K6Variant::kRP;
    return K6Variant::kAuto;
  }();
  return v;
}
// The auto rule's threshold in MiB of K + V per head (DYNRAD_K6_RP_MIN_MB,
// default 64: half of L2); tests lower it to run the auto path on small grids.
static double k6_rp_min_bytes() {
  static const double b = [] {
    const char* e = std::getenv("DYNRAD_K6_RP_MIN_MB");
    return (e ? std::atof(e) : 64.0) * (1 << 20);
  }();
  return b;
}
static K6Variant k6_variant(int64_t padded_tokens, int head_dim) {
  const K6Variant f = k6_forced();
  if (f != K6Variant::kAuto) return f;
  const double kv_head_bytes = 4.0 * static_cast<double>(padded_tokens) * head_dim;
  return kv_head_bytes > k6_rp_min_bytes() ? K6Variant::kRP : K6Variant::kDB;
}
static const char* k6_kernel_name(int64_t padded_tokens, int head_dim, int block_size) {
  if (block_size == 64)
    return head_dim == 64 ? "bsfa_fwd_db_kernel<64, quadrant mask>"
                          : "bsfa_fwd_db_kernel<128, quadrant mask>";
  if (k6_variant(padded_tokens, head_dim) == K6Variant::kRP)
    return head_dim == 64 ? "bsfa_fwd_rp_kernel<64>" : "bsfa_fwd_rp_kernel<128>";
  return head_dim == 64 ? "bsfa_fwd_db_kernel<64>" : "bsfa_fwd_db_kernel<128>";
}

// Large-shared-memory opt-in is a per-(kernel, device) attribute: remember
// which devices each kernel was prepared on (bit = device ordinal).
void prepare_kernel(const void* fn, int smem, void (*check)(const void*)) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, uint64_t>> done;
  int dev = 0;
  RP_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = uint64_t{1} << (dev & 63);
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : done)
    if (e.first == fn) {
      if (e.second & bit) return;
      if (check) check(fn);
      RP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      e.second |= bit;
      return;
    }
  if (check) check(fn);
  RP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  done.emplace_back(fn, bit);
}

static void launch_attention(const rp_grid& g, const rp_tensor& q, const rp_tensor& k,
                             const rp_tensor& v, rp_tensor& o, const int32_t* row_ptr,
                             const int32_t* col_idx, const int32_t* row_order, float scale,
                             cudaStream_t stream, int* err_flag,
                             const uint8_t* soft_bits = nullptr, double eps = 0.0) {
  // soft_bits != null: soft mask (masked_attention, attention.cpp:59-81) over
  // dense row lists; the block bit selects the log1p(eps) / log(eps) offset
  const int d = q.head_dim;
  if (!use_lpt_order()) row_order = nullptr;
  const float user_scale = scale;
  if (scale <= 0.f) scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
  if (q.dtype == RP_BF16) {
    if (g.block_size != 128 && g.block_size != 64)
      throw std::invalid_argument("sparse attention (bf16): block_size must be 64 or 128");
    if (d != 64 && d != 128)
      throw std::invalid_argument("sparse attention (bf16): head_dim must be 64 or 128");
    for (const rp_tensor* t : {&q, &k, &v, static_cast<const rp_tensor*>(&o)})
      if (t->token_stride % 8 || t->head_stride % 8)
        throw std::invalid_argument("sparse attention (bf16): strides must be multiples of 8");
    const CUtensorMap mq = make_map_bf16(q), mk = make_map_bf16(k), mv = make_map_bf16(v);
    const K6Variant variant = k6_variant(g.padded_tokens, d);
    // The kernels re-balance registers between warpgroups with setmaxnreg;
    // that only works if the launch allocates the full 168 x 384 pool.
    auto check_regs = [](const void* fn) {
      cudaFuncAttributes fa;
      RP_CUDA(cudaFuncGetAttributes(&fa, fn));
      if (fa.numRegs * attn2::kThreads < 2 * 128 * 208 + 128 * 88)
        throw CudaError("K6 compiled with too few registers for its setmaxnreg plan");
    };
    auto launch = [&](const void* fn, int smem, int grid, int threads, auto&& go) {
      prepare_kernel(fn, smem, check_regs);
      go(grid, threads, smem);
      RP_LAUNCHED();
    };
    const float soft_delta = soft_bits ? static_cast<float>((std::log(eps) - std::log1p(eps)) /
                                                            static_cast<double>(scale))
                                       : 0.f;
    if (g.block_size == 64) {
      // B = 64: the 128-row tensor-core tiles walk the merged
      // lists of two 64-block rows; every tile carries its four 64 x 64
      // quadrant bits and the db kernel masks the quadrants a thread's 64
      // keys fall in (each softmax thread owns one 64-key half of a row).
      if (soft_bits)
        throw std::invalid_argument("soft-mask attention (bf16): block_size must be 128");
      const int64_t nb = g.blocks_per_dim, ns = (nb + 1) / 2;
      int32_t *scnt = nullptr, *srow = nullptr, *scol = nullptr;
      uint8_t* qm = nullptr;
      RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scnt), sizeof(int32_t) * (ns + 1), stream));
      RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&srow), sizeof(int32_t) * (ns + 1), stream));
      RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scol), sizeof(int32_t) * ns * ns, stream));
      RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&qm), ns * ns, stream));
      const unsigned qg = static_cast<unsigned>((ns + 127) / 128);
      csr::quad_kernel<false><<<qg, 128, 0, stream>>>(row_ptr, col_idx, nb, ns, scnt, nullptr,
                                                       nullptr, nullptr);
      RP_LAUNCHED();
      csr::scan_kernel<<<1, 1024, 0, stream>>>(scnt, ns, srow, nullptr);
      RP_LAUNCHED();
      csr::quad_kernel<true><<<qg, 128, 0, stream>>>(row_ptr, col_idx, nb, ns, nullptr, srow,
                                                      scol, qm);
      RP_LAUNCHED();
      attn2::Params p{};
      p.row_ptr = srow;
      p.col_idx = scol;
      p.row_order = nullptr;
      p.n_rows = static_cast<int>(ns);
      p.heads = q.heads;
      p.n_units = static_cast<long long>(q.heads) * ns;
      p.out = static_cast<__nv_bfloat16*>(o.data);
      p.out_tok_stride = o.token_stride;
      p.out_head_stride = o.head_stride;
      p.scale_log2 = scale * 1.4426950408889634f;
      p.qmask = qm;
      p.out_rows = g.padded_tokens;
      const int grid = static_cast<int>(std::min<long long>(p.n_units, sm_count()));
      if (d == 128) {
        launch(reinterpret_cast<const void*>(attn2::bsfa_fwd_db_kernel<128, true>),
               attn2::Layout<128>::kSmemBytes, grid, attn2::kThreads, [&](int gr, int th, int sm) {
                 attn2::bsfa_fwd_db_kernel<128, true><<<gr, th, sm, stream>>>(mq, mk, mv, p);
               });
      } else {
        launch(reinterpret_cast<const void*>(attn2::bsfa_fwd_db_kernel<64, true>),
               attn2::Layout<64>::kSmemBytes, grid, attn2::kThreads, [&](int gr, int th, int sm) {
                 attn2::bsfa_fwd_db_kernel<64, true><<<gr, th, sm, stream>>>(mq, mk, mv, p);
               });
      }
      if (err_flag) {
        csr::empty_row_flag_kernel<<<static_cast<unsigned>((nb + 255) / 256), 256, 0, stream>>>(
            row_ptr, nb, err_flag);
        RP_LAUNCHED();
      }
      for (void* ptr : {static_cast<void*>(scnt), static_cast<void*>(srow),
                        static_cast<void*>(scol), static_cast<void*>(qm)})
        RP_CUDA(cudaFreeAsync(ptr, stream));
      return;
    }
    if (variant == K6Variant::kRP) {
      // union block lists of the row pairs (2p, 2p+1)
      const int n_rows = static_cast<int>(g.blocks_per_dim);
      const int n_pairs = (n_rows + 1) / 2;
      const size_t cap = static_cast<size_t>(n_pairs) * n_rows;
      int32_t *pcnt = nullptr, *prow = nullptr, *pcol = nullptr;
      uint8_t* pflag = nullptr;
      RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&pcnt), sizeof(int32_t) * (n_pairs + 1), stream));
      RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&prow), sizeof(int32_t) * (n_pairs + 1), stream));
      RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&pcol), sizeof(int32_t) * 2 * cap, stream));
      RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&pflag), cap, stream));
      if (n_rows <= 32 * attn3::kPairWords && !std::getenv("DYNRAD_RP_SERIAL_LISTS")) {
        const unsigned wg = static_cast<unsigned>((n_pairs + attn3::kPairWarps - 1) /
                                                  attn3::kPairWarps);
        attn3::pair_lists_warp_kernel<false><<<wg, 32 * attn3::kPairWarps, 0, stream>>>(
            row_ptr, col_idx, n_rows, n_pairs, pcnt, nullptr, nullptr, nullptr);
        RP_LAUNCHED();
        csr::scan_kernel<<<1, 1024, 0, stream>>>(pcnt, n_pairs, prow, nullptr);
        RP_LAUNCHED();
        attn3::pair_lists_warp_kernel<true><<<wg, 32 * attn3::kPairWarps, 0, stream>>>(
            row_ptr, col_idx, n_rows, n_pairs, nullptr, prow, pcol, pflag);
        RP_LAUNCHED();
      } else {
        const unsigned pg = static_cast<unsigned>((n_pairs + 127) / 128);
        attn3::pair_count_kernel<<<pg, 128, 0, stream>>>(row_ptr, col_idx, n_rows, n_pairs, pcnt);
        RP_LAUNCHED();
        csr::scan_kernel<<<1, 1024, 0, stream>>>(pcnt, n_pairs, prow, nullptr);
        RP_LAUNCHED();
        attn3::pair_fill_kernel<<<pg, 128, 0, stream>>>(row_ptr, col_idx, n_rows, n_pairs, prow,
                                                       pcol, pflag);
        RP_LAUNCHED();
      }
      attn3::Params p;
      p.row_ptr = row_ptr;
      p.prow_ptr = prow;
      p.pcol = pcol;
      p.pflag = pflag;
      p.porder = nullptr;
      p.n_rows = n_rows;
      p.n_pairs = n_pairs;
      p.heads = q.heads;
      p.n_units = static_cast<long long>(q.heads) * n_pairs;
      p.out = static_cast<__nv_bfloat16*>(o.data);
      p.out_tok_stride = o.token_stride;
      p.out_head_stride = o.head_stride;
      p.scale_log2 = scale * 1.4426950408889634f;
      p.col_idx = col_idx;
      p.soft_bits = soft_bits;
      p.soft_row_bytes = g.row_bytes;
      p.soft_delta = soft_delta;
      const int grid = static_cast<int>(std::min<long long>(p.n_units, sm_count()));
      auto rp_launch = [&](const void* fn, int smem, auto kern) {
        launch(fn, smem, grid, attn3::kThreads, [&](int gr, int th, int sm) {
          kern<<<gr, th, sm, stream>>>(mq, mk, mv, p);
        });
      };
      if (d == 128) {
        if (soft_bits)
          rp_launch(reinterpret_cast<const void*>(attn3::bsfa_fwd_rp_kernel<128, true>),
                    attn3::Layout<128>::kSmemBytes, attn3::bsfa_fwd_rp_kernel<128, true>);
        else
          rp_launch(reinterpret_cast<const void*>(attn3::bsfa_fwd_rp_kernel<128>),
                    attn3::Layout<128>::kSmemBytes, attn3::bsfa_fwd_rp_kernel<128>);
      } else {
        if (soft_bits)
          rp_launch(reinterpret_cast<const void*>(attn3::bsfa_fwd_rp_kernel<64, true>),
                    attn3::Layout<64>::kSmemBytes, attn3::bsfa_fwd_rp_kernel<64, true>);
        else
          rp_launch(reinterpret_cast<const void*>(attn3::bsfa_fwd_rp_kernel<64>),
                    attn3::Layout<64>::kSmemBytes, attn3::bsfa_fwd_rp_kernel<64>);
      }
      if (err_flag) {  // rp zero-fills empty rows without flagging them
        csr::empty_row_flag_kernel<<<static_cast<unsigned>((g.blocks_per_dim + 255) / 256), 256,
                                     0, stream>>>(row_ptr, g.blocks_per_dim, err_flag);
        RP_LAUNCHED();
      }
      for (void* ptr : {static_cast<void*>(pcnt), static_cast<void*>(prow),
                        static_cast<void*>(pcol), static_cast<void*>(pflag)})
        RP_CUDA(cudaFreeAsync(ptr, stream));
      return;
    }
    {
      // "db": one query tile per CTA, score tile double-buffered in TMEM
      attn2::Params p{};
      p.row_ptr = row_ptr;
      p.col_idx = col_idx;
      p.row_order = use_lpt_order() ? row_order : nullptr;
      p.n_rows = static_cast<int>(g.blocks_per_dim);
      p.heads = q.heads;
      p.n_units = static_cast<long long>(q.heads) * p.n_rows;
      p.out = static_cast<__nv_bfloat16*>(o.data);
      p.out_tok_stride = o.token_stride;
      p.out_head_stride = o.head_stride;
      p.scale_log2 = scale * 1.4426950408889634f;
      p.soft_bits = soft_bits;
      p.soft_row_bytes = g.row_bytes;
      p.soft_delta = soft_delta;
      // Exchange-free rescale protocol (DYNRAD_DB_LAG=1): a per-head max |k|
      // pre-pass (one read of K) bounds every logit, so units whose bound
      // stays within 2^64 of their first block's max decide rescales two
      // steps late from the halves' block sums, without the per-step
      // exchange barrier (attn_sm100_db.cu).
      static const bool lag_on = [] {
        const char* e = std::getenv("DYNRAD_DB_LAG");
        return e && std::strcmp(e, "1") == 0;
      }();
      float* kmax = nullptr;
      if (lag_on && !soft_bits && k.head_dim % 8 == 0 && k.heads <= 64) {
        RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&kmax), sizeof(float) * k.heads, stream));
        RP_CUDA(cudaMemsetAsync(kmax, 0, sizeof(float) * k.heads, stream));
        attn2::kmax_kernel<<<sm_count() * 2, 256, 0, stream>>>(
            static_cast<const __nv_bfloat16*>(k.data), k.tokens, k.heads, k.head_dim,
            k.token_stride, k.head_stride, kmax);
        RP_LAUNCHED();
        p.kmax_head = kmax;
      }
      const int grid = static_cast<int>(std::min<long long>(p.n_units, sm_count()));
      if (d == 128) {
        launch(reinterpret_cast<const void*>(attn2::bsfa_fwd_db_kernel<128>),
               attn2::Layout<128>::kSmemBytes, grid, attn2::kThreads, [&](int gr, int th, int sm) {
                 attn2::bsfa_fwd_db_kernel<128><<<gr, th, sm, stream>>>(mq, mk, mv, p);
               });
      } else {
        launch(reinterpret_cast<const void*>(attn2::bsfa_fwd_db_kernel<64>),
               attn2::Layout<64>::kSmemBytes, grid, attn2::kThreads, [&](int gr, int th, int sm) {
                 attn2::bsfa_fwd_db_kernel<64><<<gr, th, sm, stream>>>(mq, mk, mv, p);
               });
      }
      if (kmax) RP_CUDA(cudaFreeAsync(kmax, stream));
      if (err_flag) {
        // db zero-fills empty rows without flagging them: flag from the CSR
        csr::empty_row_flag_kernel<<<static_cast<unsigned>((g.blocks_per_dim + 255) / 256), 256,
                                     0, stream>>>(row_ptr, g.blocks_per_dim, err_flag);
        RP_LAUNCHED();
      }
      return;
    }
  } else {
    if (d > attn32::kMaxD)
      throw std::invalid_argument("sparse attention (f32): head_dim must be <= 128");
    attn32::Params p;
    p.q = static_cast<const float*>(q.data);
    p.k = static_cast<const float*>(k.data);
    p.v = static_cast<const float*>(v.data);
    p.out = static_cast<float*>(o.data);
    p.q_ts = q.token_stride; p.q_hs = q.head_stride;
    p.k_ts = k.token_stride; p.k_hs = k.head_stride;
    p.v_ts = v.token_stride; p.v_hs = v.head_stride;
    p.o_ts = o.token_stride; p.o_hs = o.head_stride;
    p.tokens = q.tokens;
    p.padded = g.padded_tokens;
    p.block = g.block_size;
    p.heads = q.heads;
    p.d = d;
    p.row_ptr = row_ptr;
    p.col_idx = col_idx;
    p.scale = user_scale > 0.f ? static_cast<double>(user_scale)
                               : 1.0 / std::sqrt(static_cast<double>(d));
    p.error_flag = err_flag;
    p.soft_bits = soft_bits;
    p.soft_row_bytes = g.row_bytes;
    p.log_active = soft_bits ? std::log1p(eps) : 0.0;
    p.log_inactive = soft_bits ? std::log(eps) : 0.0;
    dim3 grid(static_cast<unsigned>((g.padded_tokens + attn32::kRows - 1) / attn32::kRows),
              static_cast<unsigned>(q.heads));
    attn32::attn_f32_kernel<<<grid, attn32::kThreads, 0, stream>>>(p);
    RP_LAUNCHED();
  }
}

static void launch_csr(const rp_grid& g, const uint8_t* bits, int32_t* row_ptr, int32_t* col_idx,
                       int64_t col_cap, int32_t* row_order, int64_t* nnz, int32_t* counts,
                       cudaStream_t stream) {
  const int64_t n = g.blocks_per_dim;
  const int threads = 256;
  const unsigned warps_grid = static_cast<unsigned>((n * 32 + threads - 1) / threads);
  csr::row_count_kernel<<<warps_grid, threads, 0, stream>>>(bits, n, g.row_bytes, counts);
  RP_LAUNCHED();
  csr::scan_kernel<<<1, 1024, 0, stream>>>(counts, n, row_ptr, nnz);
  RP_LAUNCHED();
  csr::fill_kernel<<<warps_grid, threads, 0, stream>>>(bits, n, g.row_bytes, row_ptr, col_idx,
                                                       col_cap);
  RP_LAUNCHED();
  if (row_order) {
    csr::order_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(counts, n,
                                                                                  row_order);
    RP_LAUNCHED();
  }
}

// Host-buffer entry point plumbing: two non-blocking copy streams (H2D, D2H)
// per process, and a stream-ordered pool that keeps its memory between calls
// (the default release threshold returns every byte at each synchronize, so
// multi-GB staging buffers would be re-mapped on every call).
struct HostStreams {
  cudaStream_t in = nullptr, out = nullptr;
};
HostStreams& host_streams() {
  // one pair per device (streams belong to the device current at creation)
  static std::mutex mu;
  static HostStreams per_dev[64];
  int dev = 0;
  RP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  HostStreams& x = per_dev[dev & 63];
  if (!x.in) {
    RP_CUDA(cudaStreamCreateWithFlags(&x.in, cudaStreamNonBlocking));
    RP_CUDA(cudaStreamCreateWithFlags(&x.out, cudaStreamNonBlocking));
  }
  return x;
}
void keep_pool_memory() {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  const uint64_t bit = uint64_t{1} << (dev & 63);
  if (done.load() & bit) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    // keep up to 32 GiB (a static Wan / Hunyuan mask build's Fisher-Yates
    // scratch, the host-buffer layer's Q/K/V/O staging); release above that
    // so the rest of the process (torch's allocator) keeps its memory
    const char* e = std::getenv("DYNRAD_POOL_KEEP_GB");
    uint64_t thr = uint64_t(e ? std::atoll(e) : 32) << 30;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done.fetch_or(bit);
}
// Head chunks of the host-buffer pipeline (DYNRAD_E2E_CHUNKS, default 8:
// measured 54.0 ms at 4 chunks, 47.5 ms at 8 for the Wan layer).
int e2e_chunks() {
  static const int n = [] {
    const char* e = std::getenv("DYNRAD_E2E_CHUNKS");
    const int v = e ? std::atoi(e) : 8;
    return v > 0 ? v : 8;
  }();
  return n;
}

// Head-chunk sizes of the host-buffer pipelines: e2e_chunks() chunks of
// ceil(heads / chunks) (at least min_first heads each), the last one split
// into halves (5 -> 3, 1, 1): the exposed tail is the last piece's kernel
// plus its D2H copy, so it is kept small (DYNRAD_E2E_TAPER=0: no split).
std::vector<int> head_chunks(int heads, int min_first) {
  static const bool taper = [] {
    const char* e = std::getenv("DYNRAD_E2E_TAPER");
    return !(e && std::atoi(e) == 0);
  }();
  const int chunks = std::max(1, std::min(heads, e2e_chunks()));
  const int per = std::max((heads + chunks - 1) / chunks, min_first);
  std::vector<int> out;
  for (int h0 = 0; h0 < heads; h0 += per) out.push_back(std::min(per, heads - h0));
  if (taper && out.size() > 1) {
    int last = out.back();
    out.pop_back();
    while (last > 1) {
      const int a = (last + 1) / 2;
      out.push_back(a);
      last -= a;
    }
    if (last > 0) out.push_back(last);
  }
  return out;
}

}  // namespace rp

using namespace rp;

extern "C" {

const char* rp_last_error(void) { return t_err.c_str(); }

void rp_profile_stages(int enable) {
  std::lock_guard<std::mutex> lock(g_prof_mu);
  for (auto& r : g_prof_recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof_recs.clear();
  for (auto& o : g_prof_open) cudaEventDestroy(o.second);
  g_prof_open.clear();
  g_prof_on.store(enable != 0);
}

rp_status rp_profile_read(double* total_ms, int64_t* count, int n) {
  return guarded([&] {
    std::lock_guard<std::mutex> lock(g_prof_mu);
    for (int i = 0; i < n; ++i) {
      total_ms[i] = 0.0;
      count[i] = 0;
    }
    for (auto& r : g_prof_recs) {
      if (r.stage < 0 || r.stage >= n) continue;
      RP_CUDA(cudaEventSynchronize(r.b));
      float ms = 0.f;
      RP_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      total_ms[r.stage] += ms;
      ++count[r.stage];
    }
  });
}
const char* rp_version(void) { return "dynrad-b200 0.1 (sm_100a)"; }
int64_t rp_kernel_launch_count(void) { return g_launches.load(); }
#ifdef RP_TRACE
int rp_debug_trace(void* host) {
  return cudaMemcpyFromSymbol(host, attn2::g_trace, sizeof(attn2::g_trace)) == cudaSuccess ? 0 : 1;
}
#endif

rp_status rp_make_grid(int nf, int nt, int bs, rp_grid* out) {
  return guarded([&] {
    rp_grid g{};
    g.n_frames = nf;
    g.tokens_per_frame = nt;
    g.block_size = bs;
    check_grid(&g);
    g.total_tokens = static_cast<int64_t>(nf) * nt;
    g.padded_tokens = (g.total_tokens + bs - 1) / bs * bs;
    g.blocks_per_dim = g.padded_tokens / bs;
    g.row_bytes = (g.blocks_per_dim + 7) / 8;
    *out = g;
  });
}

void rp_config_defaults(rp_config* c) {
  c->mode = RP_STATIC_RATIO;
  c->decay_factor = 1.0;
  c->long_range_factor = 1.0;
  c->split_epsilon = 1e-6;
  c->mask_threshold = 0.75;
  c->col_threshold = 0.20;
  c->near_param = 0.25;
  c->far_param = 0.55;
  c->fallback_k = 1;
}

rp_status rp_config_validate(const rp_config* c) {
  return guarded([&] { plan::validate(*c); });
}

rp_status rp_frame_pair_info(const rp_grid* g, const rp_config* c, int i, int j,
                             rp_frame_pair* out) {
  return guarded([&] {
    check_grid(g);
    if (i < 0 || j < 0 || i >= g->n_frames || j >= g->n_frames)
      throw std::out_of_range("frame_pair: frame outside grid");
    const int64_t t = std::llabs(static_cast<long long>(i) - j);
    rp_frame_pair f{};
    f.width = plan::window_width(i, j, *c, *g);
    f.retained = plan::frame_retained(t, *c, *g) ? 1 : 0;
    f.pair_count = f.retained ? plan::band_pairs(g->tokens_per_frame, f.width) : 0;
    f.tier = plan::distance_tier(i, j, *c, *g);
    f.split_factor = t >= 1 ? plan::split_factor(t, *c, *g) : 1;
    if (c->mode == RP_STATIC_RATIO)
      f.retention_or_threshold = f.tier == 0 ? 1.0 : (f.tier == 1 ? c->near_param : c->far_param);
    else
      f.retention_or_threshold = f.tier == 0 ? -std::numeric_limits<double>::infinity()
                                             : (f.tier == 1 ? c->near_param : c->far_param);
    *out = f;
  });
}

static void sparse_attention_entry(const rp_grid* g, const rp_tensor* q, const rp_tensor* k,
                                   const rp_tensor* v, rp_tensor* o, const int32_t* row_ptr,
                                   const int32_t* col_idx, const int32_t* row_order,
                                   float softmax_scale, int* err_flag, rp_stream stream) {
  require_device();
  check_grid(g);
  check_tensor(q, "q");
  check_tensor(k, "k");
  check_tensor(v, "v");
  check_tensor(o, "o");
  if (k->tokens != q->tokens || v->tokens != q->tokens || k->heads != q->heads ||
      v->heads != q->heads || k->head_dim != q->head_dim || v->head_dim != q->head_dim ||
      k->dtype != q->dtype || v->dtype != q->dtype || o->dtype != q->dtype)
    throw std::invalid_argument("feature batch: queries/keys/values shape mismatch");
  if (g->padded_tokens < q->tokens)
    throw std::invalid_argument("masked attention: mask smaller than batch");
  if (o->tokens < g->padded_tokens || o->heads != q->heads || o->head_dim != q->head_dim)
    throw std::invalid_argument("masked attention: output must be [S', heads, head_dim]");
  if (!row_ptr || !col_idx) throw std::invalid_argument("masked attention: null row lists");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  stage_begin(kStageAttention, s);
  launch_attention(*g, *q, *k, *v, *o, row_ptr, col_idx, row_order, softmax_scale, s, err_flag);
  stage_end(kStageAttention, s);
}

rp_status rp_sparse_attention_fwd(const rp_grid* g, const rp_tensor* q, const rp_tensor* k,
                                  const rp_tensor* v, rp_tensor* o, const int32_t* row_ptr,
                                  const int32_t* col_idx, const int32_t* row_order,
                                  float softmax_scale, rp_stream stream) {
  return guarded([&] {
    sparse_attention_entry(g, q, k, v, o, row_ptr, col_idx, row_order, softmax_scale, nullptr,
                           stream);
  });
}

rp_status rp_sparse_attention_fwd_checked(const rp_grid* g, const rp_tensor* q,
                                          const rp_tensor* k, const rp_tensor* v, rp_tensor* o,
                                          const int32_t* row_ptr, const int32_t* col_idx,
                                          const int32_t* row_order, float softmax_scale,
                                          int* err_flag_dev, rp_stream stream) {
  return guarded([&] {
    sparse_attention_entry(g, q, k, v, o, row_ptr, col_idx, row_order, softmax_scale,
                           err_flag_dev, stream);
  });
}

rp_status rp_random_batch(int64_t tokens, int heads, int head_dim, uint64_t seed,
                          int first_head, rp_tensor* q, rp_tensor* k, rp_tensor* v,
                          rp_stream stream) {
  return guarded([&] {
    require_device();
    if (tokens < 1 || heads < 1 || head_dim < 1)
      throw std::invalid_argument("feature batch: empty dimensions");
    if (head_dim % 8) throw std::invalid_argument("random_batch: head_dim must be a multiple of 8");
    if (first_head < 0) throw std::invalid_argument("random_batch: first_head must be >= 0");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    rp_tensor* dst[3] = {q, k, v};
    for (int role = 1; role <= 3; ++role) {
      rp_tensor* t = dst[role - 1];
      if (!t) continue;
      if (!t->data || t->tokens < tokens || t->heads < heads || t->head_dim != head_dim ||
          (t->dtype != RP_F32 && t->dtype != RP_BF16) || t->token_stride % 8 ||
          t->head_stride % 8)
        throw std::invalid_argument("random_batch: output tensor shape / dtype / stride");
      const int64_t n = tokens * heads * (head_dim / 8);
      const unsigned grid = static_cast<unsigned>((n + 255) / 256);
      if (t->dtype == RP_BF16)
        feat::random_batch_kernel<true><<<grid, 256, 0, s>>>(
            tokens, heads, head_dim, seed, static_cast<uint64_t>(role), first_head, t->data,
            t->token_stride, t->head_stride);
      else
        feat::random_batch_kernel<false><<<grid, 256, 0, s>>>(
            tokens, heads, head_dim, seed, static_cast<uint64_t>(role), first_head, t->data,
            t->token_stride, t->head_stride);
      RP_LAUNCHED();
    }
  });
}

const char* rp_attention_kernel(const rp_grid* g, int dtype, int head_dim) {
  if (dtype != RP_BF16) return "attn_f32_kernel";
  return k6_kernel_name(g ? g->padded_tokens : 0, head_dim, g ? g->block_size : 128);
}

rp_status rp_mask_to_csr(const rp_grid* g, const uint8_t* bits, int32_t* row_ptr,
                         int32_t* col_idx, int64_t col_cap, int32_t* row_order, int64_t* nnz,
                         rp_stream stream) {
  return guarded([&] {
    require_device();
    check_grid(g);
    if (!bits || !row_ptr || !col_idx) throw std::invalid_argument("mask_to_csr: null buffer");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int32_t* counts = nullptr;
    RP_CUDA(cudaMallocAsync(&counts, sizeof(int32_t) * (g->blocks_per_dim + 1), s));
    stage_begin(kStageCsr, s);
    launch_csr(*g, bits, row_ptr, col_idx, col_cap, row_order, nnz, counts, s);
    stage_end(kStageCsr, s);
    RP_CUDA(cudaFreeAsync(counts, s));
  });
}

rp_status rp_expand_mask(const rp_grid* g, const uint8_t* bits, uint8_t* token_bits,
                         rp_stream stream) {
  return guarded([&] {
    require_device();
    check_grid(g);
    const int64_t tok = g->padded_tokens, trb = (tok + 7) / 8;
    const int64_t total = tok * trb;
    csr::expand_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0,
                         reinterpret_cast<cudaStream_t>(stream)>>>(
        bits, g->blocks_per_dim, g->row_bytes, g->block_size, tok, trb, token_bits);
    RP_LAUNCHED();
  });
}

rp_status rp_mask_sparsity(const rp_grid* g, const uint8_t* bits, int64_t* active,
                           double* sparsity, rp_stream stream) {
  return guarded([&] {
    require_device();
    check_grid(g);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    unsigned long long* d = nullptr;
    RP_CUDA(cudaMallocAsync(&d, sizeof(unsigned long long), s));
    RP_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), s));
    const int64_t n = g->blocks_per_dim * g->row_bytes;
    csr::popcount_kernel<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 1024)), 256,
                           0, s>>>(bits, n, d);
    RP_LAUNCHED();
    unsigned long long h = 0;
    RP_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
    RP_CUDA(cudaFreeAsync(d, s));
    if (active) *active = static_cast<int64_t>(h);
    if (sparsity)
      *sparsity = 1.0 - static_cast<double>(h) /
                            (static_cast<double>(g->blocks_per_dim) * g->blocks_per_dim);
  });
}

}  // extern "C"

namespace rp {
// Host-buffer attention (exact: soft == false; soft mask with eps otherwise).
static void host_attention(const rp_grid* g, const uint8_t* mask_bits_host, const void* q_host,
                           const void* k_host, const void* v_host, int dtype, int64_t tokens,
                           int heads, int head_dim, void* o_host, rp_stream stream, bool soft,
                           double eps) {
    require_device();
    check_grid(g);
    if (tokens < 1 || heads < 1 || head_dim < 1)
      throw std::invalid_argument("feature batch: empty dimensions");
    if (g->padded_tokens < tokens)
      throw std::invalid_argument("masked attention: mask smaller than batch");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const size_t es = dtype == RP_BF16 ? 2 : 4;
    const size_t row_in = static_cast<size_t>(heads) * head_dim * es;  // bytes per token
    const size_t in_bytes = static_cast<size_t>(tokens) * row_in;
    const size_t out_bytes = static_cast<size_t>(g->padded_tokens) * row_in;
    const size_t mask_bytes = static_cast<size_t>(g->blocks_per_dim * g->row_bytes);
    const int64_t nb = g->blocks_per_dim;
    keep_pool_memory();
    uint8_t *dq = nullptr, *dk = nullptr, *dv = nullptr, *dout = nullptr, *dm = nullptr;
    int32_t *rp_ = nullptr, *ci = nullptr, *ro = nullptr, *cnt = nullptr;
    int* flag = nullptr;
    struct Free {
      cudaStream_t s;
      std::vector<void*> ptrs;
      ~Free() {
        for (void* p : ptrs)
          if (p) cudaFreeAsync(p, s);
      }
    } fr{s, {}};
    auto alloc = [&](auto** p, size_t b) {
      RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(p), b, s));
      fr.ptrs.push_back(*p);
    };
    alloc(&dm, mask_bytes);
    alloc(&rp_, sizeof(int32_t) * (nb + 1));
    alloc(&ci, sizeof(int32_t) * nb * nb);
    alloc(&ro, sizeof(int32_t) * nb);
    alloc(&cnt, sizeof(int32_t) * (nb + 1));
    alloc(&flag, sizeof(int));
    RP_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
    RP_CUDA(cudaMemcpyAsync(dm, mask_bits_host, mask_bytes, cudaMemcpyHostToDevice, s));
    if (soft) {
      csr::dense_lists_kernel<<<static_cast<unsigned>((nb * nb + 255) / 256), 256, 0, s>>>(nb, rp_, ci);
      RP_LAUNCHED();
      ro = nullptr;
    } else {
      // Row lists first: an empty row is a domain_error in the reference
      // (attention.cpp:85-86), detected before any feature is moved.
      launch_csr(*g, dm, rp_, ci, nb * nb, ro, nullptr, cnt, s);
      std::vector<int32_t> hcnt(static_cast<size_t>(nb) + 1);
      RP_CUDA(cudaMemcpyAsync(hcnt.data(), rp_, sizeof(int32_t) * (nb + 1),
                              cudaMemcpyDeviceToHost, s));
      RP_CUDA(cudaStreamSynchronize(s));
      for (int64_t r = 0; r < nb; ++r)
        if (hcnt[r + 1] == hcnt[r])
          throw std::domain_error("masked attention: row has no active key");
    }
    alloc(&dq, in_bytes);
    alloc(&dk, in_bytes);
    alloc(&dv, in_bytes);
    alloc(&dout, out_bytes);
    // Head-chunk pipeline over three streams: H2D of chunk c+1 and D2H of
    // chunk c-1 run under the kernel of chunk c (PCIe is full duplex).
    const std::vector<int> sizes = head_chunks(heads, 1);
    HostStreams& hs = host_streams();
    cudaEvent_t start_ev;
    RP_CUDA(cudaEventCreateWithFlags(&start_ev, cudaEventDisableTiming));
    RP_CUDA(cudaEventRecord(start_ev, s));  // allocations above are ordered on s
    RP_CUDA(cudaStreamWaitEvent(hs.in, start_ev, 0));
    std::vector<cudaEvent_t> evs;
    auto event = [&]() {
      cudaEvent_t e;
      RP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      evs.push_back(e);
      return e;
    };
    int h0 = 0;
    for (const int hc : sizes) {
      const size_t off = static_cast<size_t>(h0) * head_dim * es;
      h0 += hc;
      const size_t w = static_cast<size_t>(hc) * head_dim * es;
      for (auto pr : {std::make_pair(dq, q_host), std::make_pair(dk, k_host),
                      std::make_pair(dv, v_host)})
        RP_CUDA(cudaMemcpy2DAsync(pr.first + off, row_in,
                                  static_cast<const uint8_t*>(pr.second) + off, row_in, w,
                                  static_cast<size_t>(tokens), cudaMemcpyHostToDevice, hs.in));
      cudaEvent_t in_done = event();
      RP_CUDA(cudaEventRecord(in_done, hs.in));
      RP_CUDA(cudaStreamWaitEvent(s, in_done, 0));
      const int64_t ts = static_cast<int64_t>(heads) * head_dim;
      rp_tensor tq{dq + off, dtype, tokens, hc, head_dim, ts, head_dim};
      rp_tensor tk = tq, tv = tq;
      tk.data = dk + off;
      tv.data = dv + off;
      rp_tensor to = tq;
      to.data = dout + off;
      to.tokens = g->padded_tokens;
      launch_attention(*g, tq, tk, tv, to, rp_, ci, ro, 0.f, s, flag, soft ? dm : nullptr, eps);
      cudaEvent_t k_done = event();
      RP_CUDA(cudaEventRecord(k_done, s));
      RP_CUDA(cudaStreamWaitEvent(hs.out, k_done, 0));
      RP_CUDA(cudaMemcpy2DAsync(static_cast<uint8_t*>(o_host) + off, row_in, dout + off, row_in,
                                w, static_cast<size_t>(g->padded_tokens),
                                cudaMemcpyDeviceToHost, hs.out));
    }
    cudaEvent_t out_done = event();
    RP_CUDA(cudaEventRecord(out_done, hs.out));
    RP_CUDA(cudaStreamWaitEvent(s, out_done, 0));  // frees below are ordered after the copies
    RP_CUDA(cudaStreamSynchronize(s));
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    cudaEventDestroy(start_ev);
}

static void rethrow(rp_status st) {
  const std::string m = t_err;
  switch (st) {
    case RP_OK: return;
    case RP_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case RP_OUT_OF_RANGE: throw std::out_of_range(m);
    case RP_DOMAIN_ERROR: throw std::domain_error(m);
    case RP_RUNTIME_ERROR: throw std::runtime_error(m);
    default: throw CudaError(m);
  }
}

// One attention layer from host buffers (rp_sparse_layer_host): Q/K/V are
// copied in by head chunks over a dedicated H2D stream; the mask is built by
// the plan from the first chunk (which holds the scoring heads) as soon as
// it lands, row lists follow, and each chunk's attention runs as its inputs
// arrive while the previous chunk's output is copied out on a D2H stream.
static void layer_host(rp_plan plan, const rp_grid* g, const void* q_host, const void* k_host,
                       const void* v_host, int dtype, int64_t tokens, int heads, int head_dim,
                       int n_score_heads, void* o_host, uint8_t* mask_out, rp_stream stream) {
  require_device();
  check_grid(g);
  if (!plan) throw std::invalid_argument("sparse layer: null plan");
  if (tokens < 1 || heads < 1 || head_dim < 1)
    throw std::invalid_argument("feature batch: empty dimensions");
  if (g->padded_tokens < tokens)
    throw std::invalid_argument("masked attention: mask smaller than batch");
  if (n_score_heads < 0 || n_score_heads > heads)
    throw std::invalid_argument("sparse layer: n_score_heads must be in [0, heads]");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t es = dtype == RP_BF16 ? 2 : 4;
  const size_t row_in = static_cast<size_t>(heads) * head_dim * es;
  const size_t in_bytes = static_cast<size_t>(tokens) * row_in;
  const size_t out_bytes = static_cast<size_t>(g->padded_tokens) * row_in;
  const size_t mask_bytes = static_cast<size_t>(g->blocks_per_dim * g->row_bytes);
  const int64_t nb = g->blocks_per_dim;
  keep_pool_memory();
  uint8_t *dq = nullptr, *dk = nullptr, *dv = nullptr, *dout = nullptr, *dm = nullptr;
  int32_t *rp_ = nullptr, *ci = nullptr, *cnt = nullptr;
  int* flag = nullptr;
  struct Free {
    cudaStream_t s;
    std::vector<void*> ptrs;
    ~Free() {
      for (void* p : ptrs)
        if (p) cudaFreeAsync(p, s);
    }
  } fr{s, {}};
  auto alloc = [&](auto** p, size_t b) {
    RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(p), b, s));
    fr.ptrs.push_back(*p);
  };
  alloc(&dm, mask_bytes);
  alloc(&rp_, sizeof(int32_t) * (nb + 1));
  alloc(&ci, sizeof(int32_t) * nb * nb);
  alloc(&cnt, sizeof(int32_t) * (nb + 1));
  alloc(&flag, sizeof(int));
  alloc(&dq, in_bytes);
  alloc(&dk, in_bytes);
  alloc(&dv, in_bytes);
  alloc(&dout, out_bytes);
  RP_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
  const std::vector<int> sizes = head_chunks(heads, n_score_heads);
  HostStreams& hs = host_streams();
  std::vector<cudaEvent_t> evs;
  auto event = [&]() {
    cudaEvent_t e;
    RP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    evs.push_back(e);
    return e;
  };
  struct Destroy {
    std::vector<cudaEvent_t>& v;
    ~Destroy() {
      for (cudaEvent_t e : v) cudaEventDestroy(e);
    }
  } destroy{evs};
  cudaEvent_t start_ev = event();
  RP_CUDA(cudaEventRecord(start_ev, s));  // allocations above are ordered on s
  RP_CUDA(cudaStreamWaitEvent(hs.in, start_ev, 0));
  const int64_t ts = static_cast<int64_t>(heads) * head_dim;
  // Issue order per chunk: H2D(c), [c == 0: mask + row lists], attention(c),
  // D2H(c) -- interleaved so both copy directions stay busy (queueing every
  // H2D first measured 63 ms instead of 47 ms for the Wan layer).
  int c = 0, h0 = 0;
  for (const int hc : sizes) {
    const size_t off = static_cast<size_t>(h0) * head_dim * es;
    const size_t w = static_cast<size_t>(hc) * head_dim * es;
    auto h2d = [&](uint8_t* dst, const void* src, size_t o, size_t bytes) {
      RP_CUDA(cudaMemcpy2DAsync(dst + o, row_in, static_cast<const uint8_t*>(src) + o, row_in,
                                bytes, static_cast<size_t>(tokens), cudaMemcpyHostToDevice, hs.in));
    };
    // chunk 0: the scoring heads' Q/K go first, so stages (a)-(c) start
    // while the rest of the chunk is still in flight
    const int hs0 = c == 0 ? std::min(n_score_heads, hc) : 0;
    const size_t ws = static_cast<size_t>(hs0) * head_dim * es;
    if (hs0 > 0) {
      h2d(dq, q_host, off, ws);
      h2d(dk, k_host, off, ws);
      cudaEvent_t score_in = event();
      RP_CUDA(cudaEventRecord(score_in, hs.in));
      RP_CUDA(cudaStreamWaitEvent(s, score_in, 0));
    }
    if (w > ws) {
      h2d(dq, q_host, off + ws, w - ws);
      h2d(dk, k_host, off + ws, w - ws);
    }
    h2d(dv, v_host, off, w);
    cudaEvent_t in_done = event();
    RP_CUDA(cudaEventRecord(in_done, hs.in));
    if (c == 0) {
      // stages (a)-(c) from the first chunk (it holds the scoring heads)
      if (hs0 == 0) RP_CUDA(cudaStreamWaitEvent(s, in_done, 0));
      rp_tensor tq{dq, dtype, tokens, hc, head_dim, ts, head_dim};
      rp_tensor tk = tq;
      tk.data = dk;
      rethrow(rp_plan_build_mask(plan, n_score_heads ? &tq : nullptr,
                                 n_score_heads ? &tk : nullptr, n_score_heads, dm, nullptr,
                                 stream));
      stage_begin(kStageCsr, s);
      launch_csr(*g, dm, rp_, ci, nb * nb, nullptr, nullptr, cnt, s);
      csr::empty_row_flag_kernel<<<static_cast<unsigned>((nb + 255) / 256), 256, 0, s>>>(
          rp_, nb, flag);
      RP_LAUNCHED();
      stage_end(kStageCsr, s);
      if (mask_out)
        RP_CUDA(cudaMemcpyAsync(mask_out, dm, mask_bytes, cudaMemcpyDeviceToHost, s));
    }
    RP_CUDA(cudaStreamWaitEvent(s, in_done, 0));
    rp_tensor cq{dq + off, dtype, tokens, hc, head_dim, ts, head_dim};
    rp_tensor ck = cq, cv = cq, co = cq;
    ck.data = dk + off;
    cv.data = dv + off;
    co.data = dout + off;
    co.tokens = g->padded_tokens;
    stage_begin(kStageAttention, s);
    launch_attention(*g, cq, ck, cv, co, rp_, ci, nullptr, 0.f, s, nullptr);
    stage_end(kStageAttention, s);
    cudaEvent_t k_done = event();
    RP_CUDA(cudaEventRecord(k_done, s));
    RP_CUDA(cudaStreamWaitEvent(hs.out, k_done, 0));
    RP_CUDA(cudaMemcpy2DAsync(static_cast<uint8_t*>(o_host) + off, row_in, dout + off, row_in, w,
                              static_cast<size_t>(g->padded_tokens), cudaMemcpyDeviceToHost,
                              hs.out));
    h0 += hc;
    ++c;
  }
  int hflag = 0;
  cudaEvent_t out_done = event();
  RP_CUDA(cudaEventRecord(out_done, hs.out));
  RP_CUDA(cudaStreamWaitEvent(s, out_done, 0));
  RP_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  RP_CUDA(cudaStreamSynchronize(s));
  if (hflag) throw std::domain_error("masked attention: row has no active key");
}

static void check_epsilon(double eps) {
  if (!(eps > 0.0)) throw std::invalid_argument("masked attention: epsilon must be positive");
}
}  // namespace rp

extern "C" {

rp_status rp_masked_attention_exact_host(const rp_grid* g, const uint8_t* mask_bits_host,
                                         const void* q_host, const void* k_host,
                                         const void* v_host, int dtype, int64_t tokens,
                                         int heads, int head_dim, void* o_host,
                                         rp_stream stream) {
  return guarded([&] {
    host_attention(g, mask_bits_host, q_host, k_host, v_host, dtype, tokens, heads, head_dim,
                   o_host, stream, false, 0.0);
  });
}

rp_status rp_sparse_layer_host(rp_plan plan, const rp_grid* g, const void* q_host,
                               const void* k_host, const void* v_host, int dtype, int64_t tokens,
                               int heads, int head_dim, int n_score_heads, void* o_host,
                               uint8_t* mask_bits_host_out, rp_stream stream) {
  return guarded([&] {
    layer_host(plan, g, q_host, k_host, v_host, dtype, tokens, heads, head_dim, n_score_heads,
               o_host, mask_bits_host_out, stream);
  });
}

rp_status rp_masked_attention_host(const rp_grid* g, const uint8_t* mask_bits_host,
                                   const void* q_host, const void* k_host, const void* v_host,
                                   int dtype, int64_t tokens, int heads, int head_dim,
                                   double epsilon, void* o_host, rp_stream stream) {
  return guarded([&] {
    check_epsilon(epsilon);
    host_attention(g, mask_bits_host, q_host, k_host, v_host, dtype, tokens, heads, head_dim,
                   o_host, stream, true, epsilon);
  });
}

rp_status rp_soft_attention_fwd(const rp_grid* g, const rp_tensor* q, const rp_tensor* k,
                                const rp_tensor* v, rp_tensor* o, const uint8_t* mask_bits_dev,
                                double epsilon, float softmax_scale, rp_stream stream) {
  return guarded([&] {
    require_device();
    check_grid(g);
    check_epsilon(epsilon);
    check_tensor(q, "q");
    check_tensor(k, "k");
    check_tensor(v, "v");
    check_tensor(o, "o");
    if (k->tokens != q->tokens || v->tokens != q->tokens || k->heads != q->heads ||
        v->heads != q->heads || k->head_dim != q->head_dim || v->head_dim != q->head_dim ||
        k->dtype != q->dtype || v->dtype != q->dtype || o->dtype != q->dtype)
      throw std::invalid_argument("feature batch: queries/keys/values shape mismatch");
    if (g->padded_tokens < q->tokens)
      throw std::invalid_argument("masked attention: mask smaller than batch");
    if (o->tokens < g->padded_tokens || o->heads != q->heads || o->head_dim != q->head_dim)
      throw std::invalid_argument("masked attention: output must be [S', heads, head_dim]");
    if (!mask_bits_dev) throw std::invalid_argument("masked attention: null mask");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t nb = g->blocks_per_dim;
    int32_t *rp_ = nullptr, *ci = nullptr;
    RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rp_), sizeof(int32_t) * (nb + 1), s));
    RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ci), sizeof(int32_t) * nb * nb, s));
    csr::dense_lists_kernel<<<static_cast<unsigned>((nb * nb + 255) / 256), 256, 0, s>>>(nb, rp_, ci);
    RP_LAUNCHED();
    launch_attention(*g, *q, *k, *v, *o, rp_, ci, nullptr, softmax_scale, s, nullptr,
                     mask_bits_dev, epsilon);
    RP_CUDA(cudaFreeAsync(rp_, s));
    RP_CUDA(cudaFreeAsync(ci, s));
  });
}

}  // extern "C"
