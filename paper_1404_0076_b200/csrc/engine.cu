// engine.cu — kernels and the C ABI of libinetb200 (see include/inet_b200.h).
//
// Host side: a context owns one device, one stream and device buffers that
// are grown (never shrunk) and reused across calls, so a repeated reduction
// does no cudaMalloc. A batch of nets is laid out as per-net slabs of equal
// capacity; one CTA reduces one net (device.cuh), the grid covers the batch.
// If any net overflows its arena the batch is re-run with doubled capacity.
#include <new>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/inet_b200.h"
#include "device.cuh"
#include "ordered.cuh"
#include "finalize.cuh"
#include "host.h"
#include "jit.h"

#include <cstdlib>
#include <map>
#include <tuple>

using inetdev::NetCtl;
using inetdev::NetDesc;

namespace {

using inetdev::Shape;

using inetdev::kTierC;
using inetdev::kTierG;
using inetdev::kTierM;
using inetdev::kTierS;
using inetdev::plan_smem;

template <int kBlock, int kTier>
__global__ void __launch_bounds__(kBlock) reduce_kernel(const NetDesc* __restrict__ nets, uint32_t n_nets,
                                                        const uint32_t* __restrict__ blob, Shape sh) {
  extern __shared__ __align__(16) uint32_t smem[];
  __shared__ NetDesc sd;
  inetdev::reduce_body<kBlock, kTier>(nets, n_nets, blob, sh, smem, sd);
}

template <int kBlock>
__global__ void __launch_bounds__(kBlock) reduce_cluster_kernel(const NetDesc* __restrict__ nets, uint32_t n_nets,
                                                                const uint32_t* __restrict__ blob, Shape sh) {
  extern __shared__ __align__(16) uint32_t smem[];
  __shared__ NetDesc sd;
  inetdev::reduce_cluster_body<kBlock>(nets, n_nets, blob, sh, smem, sd);
}

template <int kBlock>
__global__ void __launch_bounds__(kBlock) reduce_grid_kernel(const NetDesc* __restrict__ nets, uint32_t n_nets,
                                                             const uint32_t* __restrict__ blob, Shape sh) {
  extern __shared__ __align__(16) uint32_t smem[];
  __shared__ NetDesc sd;
  inetdev::reduce_grid_body<kBlock>(nets, n_nets, blob, sh, smem, sd);
}

// Tier R (ordered.cuh): the reference's list order, one CTA per net.
template <int kBlock>
__global__ void __launch_bounds__(kBlock) reduce_ordered_kernel(const NetDesc* __restrict__ nets, uint32_t n_nets,
                                                                const uint32_t* __restrict__ blob, Shape sh) {
  extern __shared__ __align__(16) uint32_t smem[];
  __shared__ NetDesc sd;
  __shared__ inetdev::RShared rs;
  inetdev::reduce_ordered_body<kBlock>(nets, n_nets, blob, sh, smem, sd, rs);
}

using KernelFn = void (*)(const NetDesc*, uint32_t, const uint32_t*, Shape);

KernelFn pick_cluster_kernel(uint32_t threads) {
  switch (threads) {
    case 64:
      return reduce_cluster_kernel<64>;
    case 128:
      return reduce_cluster_kernel<128>;
    case 256:
      return reduce_cluster_kernel<256>;
    case 512:
      return reduce_cluster_kernel<512>;
    default:
      return reduce_cluster_kernel<1024>;
  }
}

template <int kTier>
KernelFn pick_kernel_t(uint32_t threads) {
  switch (threads) {
    case 64:
      return reduce_kernel<64, kTier>;
    case 128:
      return reduce_kernel<128, kTier>;
    case 256:
      return reduce_kernel<256, kTier>;
    case 512:
      return reduce_kernel<512, kTier>;
    default:
      return reduce_kernel<1024, kTier>;
  }
}

KernelFn pick_kernel(uint32_t threads, int tier) {
  if (tier == inetdev::kTierR)
    return threads <= 256 ? reduce_ordered_kernel<256> : threads <= 512 ? reduce_ordered_kernel<512> : reduce_ordered_kernel<1024>;
  if (tier == kTierC) return pick_cluster_kernel(threads);
  if (tier == inetdev::kTierX) return threads <= 256 ? reduce_grid_kernel<256> : reduce_grid_kernel<512>;
  if (tier == kTierS) return pick_kernel_t<kTierS>(threads);
  if (tier == kTierM) return pick_kernel_t<kTierM>(threads);
  return pick_kernel_t<kTierG>(threads);
}

}  // namespace

// Words per net of the rule histogram (>= 128 so development builds can append
// their phase timers after the counts).
inline uint32_t hist_stride(const struct inet_ctx* c);

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t want) {
    if (want <= bytes) return 0;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (cudaMalloc(&p, want) != cudaSuccess) return -1;
    bytes = want;
    return 0;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

// Page-locked host buffer (grow-only): result copies run at full PCIe/C2C speed.
struct PinnedU32 {
  uint32_t* p = nullptr;
  size_t n = 0, cap = 0;
  bool pinned = false;
  void release() {
    if (p) {
      if (pinned)
        cudaFreeHost(p);
      else
        std::free(p);
    }
    p = nullptr;
    cap = 0;
  }
  ~PinnedU32() { release(); }
  void resize(size_t want) {
    if (want > cap) {
      release();
      const size_t bytes = std::max<size_t>(want, 1) * 4;
      pinned = cudaHostAlloc(reinterpret_cast<void**>(&p), bytes, cudaHostAllocDefault) == cudaSuccess;
      if (!pinned) {
        cudaGetLastError();
        p = static_cast<uint32_t*>(std::malloc(bytes));  // plain memory still works, just slower
      }
      cap = want;
    }
    n = want;
  }
  void assign(const uint32_t* b, const uint32_t* e) {
    resize(static_cast<size_t>(e - b));
    if (e != b) std::memcpy(p, b, static_cast<size_t>(e - b) * 4);
  }
  uint32_t& operator[](size_t i) { return p[i]; }
  const uint32_t& operator[](size_t i) const { return p[i]; }
  uint32_t* data() { return p; }
  const uint32_t* data() const { return p; }
  bool empty() const { return n == 0; }
  size_t size() const { return n; }
};

struct inet_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // rules
  std::vector<uint32_t> blob;
  DevBuf d_blob;
  uint32_t n_labels = 0, n_rules = 0, smem_bytes = 0;
  // batch input (host copies)
  uint32_t n_nets = 0;
  PinnedU32 agents, eqs, iface;  // page-locked: the upload is an asynchronous copy
  std::vector<uint32_t> n_vars;
  std::vector<uint64_t> agent_off, eq_off, iface_off;
  uint32_t max_in_agents = 0, max_in_eqs = 0, max_in_vars = 0;
  bool input_resident = false;
  // device state
  DevBuf d_in_agents, d_in_eqs, d_in_iface, d_desc, d_agents, d_vslot, d_aring, d_vring, d_queue, d_stats, d_resid, d_ctl, d_hist,
      d_defer, d_gs, d_rbuf, d_fin, d_stamps;
  bool grid_tier = false;  // the next layout is for tier X (global rings + grid state)
  bool ordered_tier = false;  // the next layout is for tier R (list and stream arrays)
  uint32_t cap_list = 0, cap_out = 0;  // tier R: equations per list / per output stream
  size_t r_bytes = 0;                  // tier R: bytes of one net's arrays (layout)
  uint32_t cap_def = 0;  // deferred equations per net and round (reference loop mode)
  bool count_rules = false;
  std::vector<uint32_t> h_hist;
  uint64_t io_h2d = 0, io_d2h = 0;
  uint32_t cap_agents = 0, cap_vars = 0, cap_queue = 0, cap_rounds = 0;
  uint32_t rows_hint = 0;  // LoopStats rows per net the last run needed (see rows_cap)
  int tier = kTierG;  // tier of the last successful run
  uint32_t cluster_g = 1;  // CTAs per net of the last run (tier C)
  // a single net promoted from one CTA to a cluster: the tier M prefix that
  // ran up to the promotion threshold (replayed by inet_batch_rerun)
  bool promoted = false;
  uint32_t promote_ints = 1u << 19;  // env INET_B200_PROMOTE overrides
  // the state tier M handed over, applied to the next layout (tier C resumes from it)
  struct Resume {
    bool on = false;
    uint32_t agents = 0, vars = 0, pending = 0, round_base = 0;
    uint64_t ints = 0, comms = 0;
    int32_t parked = 0;
  } resume;
  Shape promo_shape{};
  uint32_t promo_cap_def = 0;
  float promo_ms = 0;
  Shape shape{};
  bool collect_stats = false;
  bool reduced = false;
  // results (host)
  std::vector<NetCtl> ctl;
  std::vector<inet_net_stats> stats;
  PinnedU32 h_agents;                 // per-net slab prefixes [n_nets * agent_pitch * 4]
  // Tier S batches write their results (the device-finalized normal forms, or
  // the arena for the host to finalize) straight into page-locked host memory
  // the device addresses directly, so no copy follows the kernel: the nets
  // of a wave write theirs while the next wave computes.
  PinnedU32 h_zc;                     // [n_nets * cap_agents * 4]
  bool zc_next = false;               // the next layout puts tier S results in h_zc
  bool zc_used = false;               // the last run's results are in h_zc (pitch cap_agents)
  PinnedU32 h_resid;                  // [n_nets * resid_pitch * 2]
  PinnedU32 h_desc;                   // layout(): the descriptor table's host staging
  PinnedU32 h_ctl;                    // the control blocks' host staging
  uint32_t agent_pitch = 0, resid_pitch = 0;
  std::vector<uint32_t> h_rounds;     // [n_nets * rows_pitch * 4]
  uint32_t rows_pitch = 1;
  std::vector<inethost::NormalForm> results;
  std::vector<uint8_t> finalized;
  // rule-set specialised kernels (jit.cpp), keyed by (tier, block size)
  int jit_mode = 1;  // 0 = prebuilt interpreter only
  bool last_jit = false;
  uint32_t last_threads = 0;  // CTA size of the last launch
  std::string jit_log;
  std::map<std::tuple<int, uint32_t, int>, std::pair<cudaLibrary_t, cudaKernel_t>> jit_kernels;
  int jit_style = -1;  // -1: per tier (measured defaults); env INET_B200_JITSTYLE overrides
  bool dev_final = true;  // tier S finalizes nets on the device; env INET_B200_DEVFINAL=0 disables
  std::vector<uint32_t> dev_rows;  // per net: device-finalized normal-form agents + 1 (0: host finalize)
  uint32_t text_net = INET_NONE;   // inet_batch_print: the net whose text is cached
  std::string text;
  std::vector<std::string> texts;  // inet_batch_print_all: every net's text (kept for the second call)
  bool exact_code = true;  // rule-set kernel variant with reference-loop (deferred equation) code
  bool var_order = false;  // stamps: var = var keyed in the reference's id order (single-CTA tiers)
};

inline uint32_t hist_stride(const inet_ctx* c) { return std::max(c->n_rules, 128u); }
// the last run's agent records on the host (pitch agent_pitch records per net)
inline const uint32_t* host_agents(const inet_ctx& c) { return c.zc_used ? c.h_zc.data() : c.h_agents.data(); }

#define CUDA_TRY(expr)                                                                         \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess) {                                                                   \
      std::fprintf(stderr, "inet_b200: %s failed: %s\n", #expr, cudaGetErrorString(_e));    \
      return INET_ERR_CUDA;                                                                    \
    }                                                                                          \
  } while (0)

extern "C" {

const char* inet_strerror(int status) {
  switch (status) {
    case INET_OK:
      return "ok";
    case INET_ERR_NO_RULE:
      return "no rule for active pair";
    case INET_ERR_LOOP_CAP:
      return "loop cap exceeded";
    case INET_ERR_ARENA:
      return "device arena exhausted";
    case INET_ERR_CUDA:
      return "CUDA runtime error";
    case INET_ERR_ARG:
      return "invalid argument";
    case INET_ERR_UNSUPPORTED:
      return "net or rule set exceeds a device-engine limit";
    case INET_ERR_NO_DEVICE:
      return "no CUDA device";
    case INET_ERR_STATE:
      return "call order violated";
    case INET_ERR_NAME:
      return "a variable occurs more than twice";
    default:
      return "unknown status";
  }
}

void inet_abi_sizes(size_t* cfg_bytes, size_t* stats_bytes) {
  if (cfg_bytes) *cfg_bytes = sizeof(inet_cfg);
  if (stats_bytes) *stats_bytes = sizeof(inet_net_stats);
}

int inet_ctx_create(int device, inet_ctx** out) {
  try {
    if (!out) return INET_ERR_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return INET_ERR_NO_DEVICE;
    if (device < 0 || device >= n) return INET_ERR_ARG;
    CUDA_TRY(cudaSetDevice(device));
    auto* c = new inet_ctx();
    c->device = device;
    if (const char* e = std::getenv("INET_B200_JIT")) c->jit_mode = std::atoi(e);
    if (const char* e = std::getenv("INET_B200_JITSTYLE")) c->jit_style = std::atoi(e);
    if (const char* e = std::getenv("INET_B200_PROMOTE")) c->promote_ints = static_cast<uint32_t>(std::atol(e));
    if (const char* e = std::getenv("INET_B200_DEVFINAL")) c->dev_final = std::atoi(e) != 0;
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess) {
      delete c;
      return INET_ERR_CUDA;
    }
    *out = c;
    return INET_OK;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

void inet_ctx_destroy(inet_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  for (DevBuf* b : {&c->d_blob, &c->d_in_agents, &c->d_in_eqs, &c->d_desc, &c->d_agents, &c->d_vslot, &c->d_aring,
                    &c->d_vring, &c->d_queue, &c->d_stats, &c->d_resid, &c->d_ctl, &c->d_hist, &c->d_defer, &c->d_gs, &c->d_rbuf, &c->d_fin, &c->d_stamps})
    b->release();
  for (auto& kv : c->jit_kernels) cudaLibraryUnload(kv.second.first);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int inet_device_info(inet_ctx* c, int* sm_count, int* clock_khz, char* name, size_t name_len) {
  try {
    if (!c) return INET_ERR_ARG;
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, c->device));
    if (sm_count) *sm_count = prop.multiProcessorCount;
    if (clock_khz) cudaDeviceGetAttribute(clock_khz, cudaDevAttrClockRate, c->device);
    if (name && name_len) {
      std::strncpy(name, prop.name, name_len - 1);
      name[name_len - 1] = 0;
    }
    return INET_OK;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_rules_load(inet_ctx* c, const uint32_t* blob, size_t n_words) {
  try {
    if (!c || !blob || n_words < 4) return INET_ERR_ARG;
    int st = inethost::validate_rule_blob(blob, n_words);
    if (st != INET_OK) return st;
    CUDA_TRY(cudaSetDevice(c->device));
    if (c->blob.size() != n_words || !std::equal(c->blob.begin(), c->blob.end(), blob)) {
      for (auto& kv : c->jit_kernels) cudaLibraryUnload(kv.second.first);
      c->jit_kernels.clear();
    }
    c->blob.assign(blob, blob + n_words);
    c->n_labels = blob[1];
    c->n_rules = blob[2];
    c->smem_bytes = static_cast<uint32_t>((n_words - 4) * 4);
    if (c->d_blob.ensure(n_words * 4)) return INET_ERR_CUDA;
    CUDA_TRY(cudaMemcpyAsync(c->d_blob.p, blob, n_words * 4, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return INET_OK;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_batch_load(inet_ctx* c, uint32_t n_nets, const uint32_t* agents, const uint64_t* agent_off,
                    const uint32_t* eqs, const uint64_t* eq_off, const uint32_t* iface, const uint64_t* iface_off,
                    const uint32_t* n_vars) {
  try {
    if (!c || n_nets == 0 || !agent_off || !eq_off || !iface_off || !n_vars) return INET_ERR_ARG;
    if (c->blob.empty()) return INET_ERR_STATE;
    c->n_nets = n_nets;
    c->agent_off.assign(agent_off, agent_off + n_nets + 1);
    c->eq_off.assign(eq_off, eq_off + n_nets + 1);
    c->iface_off.assign(iface_off, iface_off + n_nets + 1);
    c->n_vars.assign(n_vars, n_vars + n_nets);
    c->agents.assign(agents, agents + 4 * agent_off[n_nets]);
    c->eqs.assign(eqs, eqs + 2 * eq_off[n_nets]);
    c->iface.assign(iface, iface + iface_off[n_nets]);
    c->max_in_agents = c->max_in_eqs = c->max_in_vars = 0;
    for (uint32_t i = 0; i < n_nets; ++i) {
      const uint64_t na = agent_off[i + 1] - agent_off[i], ne = eq_off[i + 1] - eq_off[i];
      if (na >= INET_VAR_BIT || ne >= INET_VAR_BIT || n_vars[i] >= INET_VAR_BIT - 1) return INET_ERR_UNSUPPORTED;
      c->max_in_agents = std::max<uint32_t>(c->max_in_agents, static_cast<uint32_t>(na));
      c->max_in_eqs = std::max<uint32_t>(c->max_in_eqs, static_cast<uint32_t>(ne));
      c->max_in_vars = std::max<uint32_t>(c->max_in_vars, n_vars[i]);
    }
    int st = inethost::validate_nets(*c);
    if (st != INET_OK) return st;
    c->input_resident = false;
    c->reduced = false;
    c->results.clear();
    c->finalized.clear();
    return INET_OK;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

}  // extern "C"

namespace {

int upload_input(inet_ctx* c) {
  const size_t na = c->agents.size() * 4, ne = c->eqs.size() * 4, ni = c->iface.size() * 4;
  if (c->d_in_agents.ensure(std::max<size_t>(na, 16)) || c->d_in_eqs.ensure(std::max<size_t>(ne, 8)) ||
      c->d_in_iface.ensure(std::max<size_t>(ni, 4)))
    return INET_ERR_CUDA;
  if (na) CUDA_TRY(cudaMemcpyAsync(c->d_in_agents.p, c->agents.data(), na, cudaMemcpyHostToDevice, c->stream));
  if (ne) CUDA_TRY(cudaMemcpyAsync(c->d_in_eqs.p, c->eqs.data(), ne, cudaMemcpyHostToDevice, c->stream));
  if (ni) CUDA_TRY(cudaMemcpyAsync(c->d_in_iface.p, c->iface.data(), ni, cudaMemcpyHostToDevice, c->stream));
  c->input_resident = true;
  c->io_h2d += na + ne + ni;
  return INET_OK;
}

// Size the per-net global slabs and write the descriptor table.
int layout(inet_ctx* c, uint32_t cap_agents, uint32_t cap_vars, uint32_t cap_queue, uint32_t cap_rounds) {
  const uint32_t n = c->n_nets;
  c->cap_agents = cap_agents;
  c->cap_vars = cap_vars;
  c->cap_queue = cap_queue;
  c->cap_rounds = cap_rounds;
  const size_t N = n;
  uint4* zc = nullptr;  // tier S results in mapped host memory (see h_zc)
  if (c->zc_next && N * cap_agents * 16 <= (size_t(1) << 30)) {  // (larger batches copy after the kernel)
    c->h_zc.resize(N * cap_agents * 4);
    void* dp = nullptr;
    if (c->h_zc.pinned && cudaHostGetDevicePointer(&dp, c->h_zc.data(), 0) == cudaSuccess)
      zc = static_cast<uint4*>(dp);
    else
      cudaGetLastError();
  }
  c->zc_used = zc != nullptr;
  if (c->d_agents.ensure(N * cap_agents * 16) || c->d_vslot.ensure(N * cap_vars * 4) ||
      c->d_queue.ensure(N * 2 * cap_queue * 8) || c->d_resid.ensure(N * cap_vars * 8) ||
      c->d_ctl.ensure(N * sizeof(NetCtl)) || c->d_desc.ensure(N * sizeof(NetDesc)) ||
      (cap_rounds && c->d_stats.ensure(N * cap_rounds * 16)) ||
      (c->count_rules && c->d_hist.ensure(N * hist_stride(c) * 4)) ||
      (c->cap_def && c->d_defer.ensure(N * 2 * c->cap_def * 8)) ||
      (c->grid_tier && (c->d_aring.ensure(size_t(cap_agents) * 4) || c->d_vring.ensure(size_t(cap_vars) * 4) ||
                        c->d_gs.ensure(sizeof(inetdev::GridState) + 4096 * 4))))
    return INET_ERR_CUDA;
  c->r_bytes = c->ordered_tier ? inetdev::r_carve(nullptr, cap_agents, cap_vars, c->cap_list, c->cap_out, nullptr) : 0;
  if (c->ordered_tier && c->d_rbuf.ensure(N * c->r_bytes)) return INET_ERR_CUDA;
  if (c->var_order && c->d_stamps.ensure(N * cap_vars * 8)) return INET_ERR_CUDA;
  if (c->grid_tier) CUDA_TRY(cudaMemsetAsync(c->d_gs.p, 0, sizeof(inetdev::GridState) + 4096 * 4, c->stream));
  if (c->count_rules) CUDA_TRY(cudaMemsetAsync(c->d_hist.p, 0, N * hist_stride(c) * 4, c->stream));
  // descriptors staged in page-locked memory (a pageable source would make
  // the copy a staged, synchronous one on every launch)
  static_assert(sizeof(NetDesc) % 4 == 0, "NetDesc words");
  c->h_desc.resize(N * sizeof(NetDesc) / 4);
  NetDesc* desc = reinterpret_cast<NetDesc*>(c->h_desc.data());
  for (uint32_t i = 0; i < n; ++i) {
    NetDesc& d = desc[i];
    std::memset(&d, 0, sizeof(d));
    d.agents = (zc ? zc : static_cast<uint4*>(c->d_agents.p)) + size_t(i) * cap_agents;
    d.vslot = static_cast<uint32_t*>(c->d_vslot.p) + size_t(i) * cap_vars;
    d.queue = static_cast<uint2*>(c->d_queue.p) + size_t(i) * 2 * cap_queue;
    d.stats = cap_rounds ? static_cast<uint4*>(c->d_stats.p) + size_t(i) * cap_rounds : nullptr;
    d.residual = static_cast<uint2*>(c->d_resid.p) + size_t(i) * cap_vars;
    d.ctl = static_cast<NetCtl*>(c->d_ctl.p) + i;
    d.rule_hist = c->count_rules ? static_cast<uint32_t*>(c->d_hist.p) + size_t(i) * hist_stride(c) : nullptr;
    d.cap_agents = cap_agents;
    d.cap_vars = cap_vars;
    d.cap_queue = cap_queue;
    d.cap_rounds = cap_rounds;
    if (c->grid_tier) {
      d.g_aring = static_cast<uint32_t*>(c->d_aring.p);
      d.g_vring = static_cast<uint32_t*>(c->d_vring.p);
      d.gs = static_cast<inetdev::GridState*>(c->d_gs.p);
    }
    d.deferred = c->cap_def ? static_cast<uint2*>(c->d_defer.p) + size_t(i) * 2 * c->cap_def : nullptr;
    d.cap_def = c->cap_def;
    d.in_agents = static_cast<const uint4*>(c->d_in_agents.p) + c->agent_off[i];
    d.in_eqs = static_cast<const uint2*>(c->d_in_eqs.p) + c->eq_off[i];
    d.n_in_agents = static_cast<uint32_t>(c->agent_off[i + 1] - c->agent_off[i]);
    d.n_in_eqs = static_cast<uint32_t>(c->eq_off[i + 1] - c->eq_off[i]);
    d.n_in_vars = c->n_vars[i];
    d.in_iface = static_cast<const uint32_t*>(c->d_in_iface.p) + c->iface_off[i];
    d.n_iface = static_cast<uint32_t>(c->iface_off[i + 1] - c->iface_off[i]);
    d.dev_final = c->dev_final ? 1u : 0u;
    for (uint64_t e = c->eq_off[i]; e < c->eq_off[i + 1]; ++e)  // an input active pair (round 1 is not a no-op loop)
      if (!(c->eqs[2 * e] & INET_VAR_BIT) && !(c->eqs[2 * e + 1] & INET_VAR_BIT)) {
        d.dev_final |= inetdev::kInputActive;
        break;
      }
    if (c->var_order) d.stamps = static_cast<unsigned long long*>(c->d_stamps.p) + size_t(i) * cap_vars;
    if (c->resume.on && n == 1) {
      // resume from tier M's hand-over: its arena, slot table and pending equations
      d.in_agents = d.agents;
      d.in_eqs = d.queue;
      d.n_in_agents = c->resume.agents;
      d.n_in_eqs = c->resume.pending;
      d.n_in_vars = c->resume.vars;
      d.resume = 1;
      d.round_base = c->resume.round_base;
      d.base_ints = c->resume.ints;
      d.base_comms = c->resume.comms;
      d.base_parked = c->resume.parked;
    }
  }
  CUDA_TRY(cudaMemcpyAsync(c->d_desc.p, desc, N * sizeof(NetDesc), cudaMemcpyHostToDevice, c->stream));
  return INET_OK;
}

// Tier M queue (pairs per round): its round counters keep pushes and freed
// variables in 16-bit halves of one word (device.cuh kPush2), so a round may
// queue at most 65,535 pairs: pairs x (equations per rule + 1) must stay below
// that (5,120 for every rule set with up to 11 equations per rule).
uint32_t tier_m_queue(const inet_ctx* c) {
  const uint32_t pair_words = (c->n_labels * c->n_labels + 1) / 2;
  uint32_t max_eq = 0;
  for (uint32_t r = 0; r < c->n_rules; ++r) max_eq = std::max(max_eq, (c->blob[4 + pair_words + r * 16] >> 8) & 0xFFu);
  return std::min<uint32_t>(5120u, 65535u / (max_eq + 1u)) & ~3u;
}

uint32_t auto_threads(const inet_ctx* c, const inet_cfg* cfg) {
  if (cfg && cfg->threads) {
    uint32_t t = cfg->threads;
    if (t <= 64) return 64;
    if (t <= 128) return 128;
    if (t <= 256) return 256;
    if (t <= 512) return 512;
    return 1024;
  }
  // measured on 2..4096 x A(3,6) (profiles/r02x_style_sweep.txt): 128 threads
  // once there are more nets than ~3 per SM (style 0 past ~768 nets, style 1
  // below), 256 below that; single nets 256 (fib(18): 2.72 ms vs 3.21 at 1024)
  return c->n_nets > 400 ? 128u : 256u;
}

// Rule-code style of the rule-set kernels (jit.cpp): tier C and X fixed; tier S
// by load — the uniform style 1 (selects, one memory phase per warp) is ~30 %
// faster per round while few nets share an SM (latency-bound: a warp no longer
// runs one dependent chain per rule present in it), the straight-line style 0
// once the SMs are full (issue-bound: 36.1 vs 45.3 ms for 4096 x A(3,6));
// profiles/r02x_style_sweep.txt.
// Tier M (single nets): both codes, chosen per warp (style 3: the cases while a
// warp's pairs span at most two rules, the uniform code otherwise) — fib(18)'s
// narrow rounds keep the cases (2.46 ms; 2.97 with style 1), the wide rounds of
// A(3,8)'s tier M prefix get the uniform code (profiles/r02ad_style_adaptive.txt).
int default_style(int tier) { return tier == kTierC ? 1 : tier == inetdev::kTierX ? 2 : tier == kTierM ? 3 : 0; }

int tier_style(const inet_ctx* c, int tier) {
  if (c->jit_style >= 0) return c->jit_style;
  if (tier == kTierS) return c->n_nets <= 768 ? 1 : 0;
  return default_style(tier);
}

// CTA size of tier R for a few nets (env INET_B200_RTHREADS overrides; measured).
uint32_t tier_r_threads(const inet_cfg* cfg) {
  if (cfg && cfg->threads) return cfg->threads <= 256 ? 256u : cfg->threads <= 512 ? 512u : 1024u;
  if (const char* e = std::getenv("INET_B200_RTHREADS")) return static_cast<uint32_t>(std::atoi(e));
  return 512u;
}

// CTA size of tier C (one CTA per SM of the cluster).
uint32_t cluster_threads(const inet_cfg* cfg) {
  const uint32_t t = cfg && cfg->threads ? cfg->threads : 256;
  if (t <= 64) return 64;
  if (t <= 128) return 128;
  if (t <= 256) return 256;
  if (t <= 512) return 512;
  return 1024;
}

// One attempt at the current capacities and tier: one kernel launch, timed.
// Rule-set specialised kernel for (tier, threads), compiled on first use;
// nullptr when NVRTC is unavailable or compilation failed (then the prebuilt
// interpreter runs).
const void* jit_kernel(inet_ctx* c, int tier, uint32_t threads) {
  if (!c->jit_mode) return nullptr;
  // code style per tier: straight-line cases where the rewrite is issue-bound
  // (S, M, G); a uniform memory phase where remote latency dominates (C)
  const int style = tier_style(c, tier);
  // per-round rows compiled in only when this layout records them (cap_rounds)
  const bool rows = c->cap_rounds != 0;
  const auto key = std::make_tuple(tier, threads,
                                   style + (c->exact_code ? 16 : 0) + (c->count_rules ? 32 : 0) + (c->var_order ? 64 : 0) +
                                       (rows ? 128 : 0));
  auto it = c->jit_kernels.find(key);
  if (it != c->jit_kernels.end()) return reinterpret_cast<const void*>(it->second.second);
  const std::string src =
      inetjit::kernel_source(c->blob.data(), c->blob.size(), tier, threads, style, c->exact_code, c->count_rules,
                             c->var_order, rows);
  std::vector<char> cubin;
  if (inetjit::compile_cubin(src, cubin, c->jit_log) != 0) {
    std::fprintf(stderr, "inet_b200: rule-set JIT unavailable, using the prebuilt kernels: %s\n", c->jit_log.c_str());
    c->jit_mode = 0;
    return nullptr;
  }
  cudaLibrary_t lib;
  cudaKernel_t k;
  if (cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
      cudaLibraryGetKernel(&k, lib, "inet_jit_kernel") != cudaSuccess) {
    cudaGetLastError();
    std::fprintf(stderr, "inet_b200: could not load the JIT cubin, using the prebuilt kernels\n");
    c->jit_mode = 0;
    return nullptr;
  }
  c->jit_kernels[key] = {lib, k};
  return reinterpret_cast<const void*>(k);
}

int launch(inet_ctx* c, const inet_cfg* cfg, Shape sh, int tier, float* ms) {
  if (tier == inetdev::kTierR) {
    sh.rbuf = static_cast<uint8_t*>(c->d_rbuf.p);
    sh.rbuf_stride = c->r_bytes;
    sh.cap_list = c->cap_list;
    sh.cap_out = c->cap_out;
  }
  const uint32_t threads = tier == kTierC                ? cluster_threads(cfg)
                           : tier == inetdev::kTierX     ? 256u
                           : tier == inetdev::kTierR     ? (c->n_nets > 64 ? 256u : tier_r_threads(cfg))
                                                         : auto_threads(c, cfg);
  sh.threads = threads;
  const void* jk = tier == inetdev::kTierR ? nullptr : jit_kernel(c, tier, threads);
  const void* fn = jk ? jk : reinterpret_cast<const void*>(pick_kernel(threads, tier));
  c->last_jit = jk != nullptr;
  c->last_threads = threads;
  const size_t smem = tier == inetdev::kTierR ? (size_t(inetdev::align4(sh.rule_words)) + 16u * threads) * 4
                                              : size_t(plan_smem(sh, tier).words) * 4;
  int dev_sms = 0, max_optin = 0;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c->device);
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
  if (smem + sizeof(NetDesc) > size_t(max_optin)) return INET_ERR_UNSUPPORTED;
  CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const NetDesc* a_nets = static_cast<const NetDesc*>(c->d_desc.p);
  uint32_t a_n = c->n_nets;
  const uint32_t* a_blob = static_cast<const uint32_t*>(c->d_blob.p);
  void* args[] = {&a_nets, &a_n, &a_blob, &sh};
  if (tier == kTierC) {
    // one cluster of G CTAs per net (G > 8 needs the non-portable opt-in)
    const uint32_t G = c->cluster_g;
    if (G > 8) CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(G * c->n_nets);
    lc.blockDim = dim3(threads);
    lc.dynamicSmemBytes = smem;
    lc.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    int n_clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&n_clusters, fn, &lc) != cudaSuccess || n_clusters < 1) {
      cudaGetLastError();
      return INET_ERR_UNSUPPORTED;
    }
    CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
    CUDA_TRY(cudaLaunchKernelExC(&lc, fn, args));
  } else if (tier == inetdev::kTierX) {
    // the whole GPU on one net: every CTA resident (cooperative launch)
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, static_cast<int>(threads), smem);
    if (per_sm < 1) return INET_ERR_UNSUPPORTED;
    const uint32_t grid = std::min<uint32_t>(uint32_t(dev_sms) * uint32_t(per_sm), 4096u);
    CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
    const cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(threads), args, smem, c->stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      if (std::getenv("INET_B200_DEBUG"))
        std::fprintf(stderr, "inet_b200: tier X launch failed (%s), grid %u\n", cudaGetErrorString(e), grid);
      return INET_ERR_UNSUPPORTED;
    }
  } else {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, static_cast<int>(threads), smem);
    uint32_t grid = std::max(1, dev_sms * std::max(per_sm, 1));
    grid = std::min(grid, c->n_nets);
    CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
    CUDA_TRY(cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, smem, c->stream));
  }
  CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
  CUDA_TRY(cudaEventSynchronize(c->ev1));
  CUDA_TRY(cudaEventElapsedTime(ms, c->ev0, c->ev1));
  return INET_OK;
}

// Tier M runs that may hand a net over to the cluster tier are laid out with
// the cluster's capacities (16 CTAs x 4096 agents / variables) plus room for
// the pending equations, so the hand-over reuses the same device buffers.
constexpr uint32_t kPromoCapAgents = 16u * 4096u;
constexpr uint32_t kPromoCapVars = 16u * 4096u;
constexpr uint32_t kPromoCapQueue = 16384u;

void set_resume(inet_ctx* c, const NetCtl& m) {
  c->resume.on = true;
  c->resume.agents = m.agent_bump;
  c->resume.vars = m.var_bump;
  c->resume.pending = m.n_residual;
  c->resume.round_base = m.rounds - 1;
  c->resume.ints = m.interactions;
  c->resume.comms = m.communications;
  c->resume.parked = static_cast<int32_t>(m.parked_total);
}

Shape base_shape(const inet_ctx* c, uint32_t max_loops) {
  Shape sh{};
  sh.max_rounds = max_loops;
  sh.rule_words = static_cast<uint32_t>(c->blob.size() - 4);
  sh.n_labels = c->n_labels;
  return sh;
}

// Per-net capacity of the LoopStats rows buffer. The reference keeps one row
// per loop (up to max_loops + 1); a batch of nets with the default cap of a
// million loops would need tens of GB, so the first attempt gets a share of a
// fixed budget (2^24 rows = 256 MB over all nets, at least 1,024 per net) and
// a run whose nets needed more rows is repeated once with exactly that many
// (c->rows_hint, set by run()). Rows past 2^22 per net are not recorded.
constexpr uint32_t kRowsBudget = 1u << 24;
constexpr uint32_t kRowsMax = 1u << 22;

uint32_t rows_cap(const inet_ctx* c, uint32_t max_loops) {
  const uint32_t want = static_cast<uint32_t>(std::min<uint64_t>(uint64_t(max_loops) + 1u, kRowsMax));
  const uint32_t share = std::max<uint32_t>(1024u, kRowsBudget / std::max<uint32_t>(c->n_nets, 1u));
  return std::min(want, std::max(share, c->rows_hint));
}

int run_once(inet_ctx* c, const inet_cfg* cfg, float* device_ms, bool fetch);
int finish_run(inet_ctx* c, bool fetch);

// Tier X: finalize the net on the device (finalize.cuh). On success the
// preorder records replace the arena prefix and the resolved interface goes
// to residual[k].x — the layout tier S's device finalize leaves — and the
// control block says so (pad[1] = records + 1, pad[2] = interface terms);
// otherwise nothing changes and the host finalizes from the arena.
int device_finalize_x(inet_ctx* c) {
  NetCtl& k = c->ctl[0];
  const uint32_t n = std::min(k.agent_bump, c->cap_agents), nv = std::min(k.var_bump, c->cap_vars);
  const uint32_t m = k.n_residual, ni = static_cast<uint32_t>(c->iface_off[1] - c->iface_off[0]);
  if (n == 0 || n >= (1u << 29) || ni == 0 || ni > 4096 || m > c->cap_vars) return INET_OK;
  uint32_t lohi[2];
  CUDA_TRY(cudaMemcpyAsync(lohi, static_cast<const char*>(c->d_gs.p) + offsetof(inetdev::GridState, fin_lo_a), 8,
                           cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t E = 2 * size_t(n);
  const size_t bytes = al(size_t(nv) * 4) * 2 + al(size_t(n) * 4) * 2 + al(size_t(n) * 16) * 2 + al(ni * 4) * 2 +
                       al(E * 8) * 2 + 256;
  if (c->d_fin.ensure(bytes)) return INET_ERR_CUDA;
  uint8_t* p = static_cast<uint8_t*>(c->d_fin.p);
  auto take = [&](size_t b) {
    uint8_t* q = p;
    p += al(b);
    return q;
  };
  inetfin::FinArgs f{};
  f.agents = static_cast<const uint4*>(c->d_agents.p);
  f.n = n;
  f.resid = static_cast<const uint2*>(c->d_resid.p);
  f.m = m;
  f.iface = static_cast<const uint32_t*>(c->d_in_iface.p);
  f.ni = ni;
  f.nv = nv;
  f.ring = static_cast<const uint32_t*>(c->d_aring.p);
  f.ring_mask = c->shape.ring_a - 1;
  f.lo = lohi[0];
  f.hi = lohi[1];
  f.val = reinterpret_cast<uint32_t*>(take(size_t(nv) * 4));
  f.used = reinterpret_cast<uint32_t*>(take(size_t(nv) * 4));
  f.dead = reinterpret_cast<uint32_t*>(take(size_t(n) * 4));
  f.parent = reinterpret_cast<uint32_t*>(take(size_t(n) * 4));
  f.res = reinterpret_cast<uint4*>(take(size_t(n) * 16));
  f.out = reinterpret_cast<uint4*>(take(size_t(n) * 16));
  f.res_iface = reinterpret_cast<uint32_t*>(take(ni * 4));
  f.out_iface = reinterpret_cast<uint32_t*>(take(ni * 4));
  f.rk[0] = reinterpret_cast<unsigned long long*>(take(E * 8));
  f.rk[1] = reinterpret_cast<unsigned long long*>(take(E * 8));
  f.flag = reinterpret_cast<uint32_t*>(take(16));
  CUDA_TRY(cudaMemsetAsync(f.flag, 0, 8, c->stream));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  const dim3 grid(static_cast<uint32_t>(sms) * 8), block(256);
  inetfin::fin_init<<<grid, block, 0, c->stream>>>(f);
  inetfin::fin_mark<<<grid, block, 0, c->stream>>>(f);
  inetfin::fin_resolve<<<grid, block, 0, c->stream>>>(f);
  inetfin::fin_unused<<<grid, block, 0, c->stream>>>(f);
  inetfin::fin_tour<<<grid, block, 0, c->stream>>>(f);
  int cur = 0;
  for (size_t span = 1; span < E; span *= 2) {  // ceil(log2 E) pointer-jumping steps
    inetfin::fin_jump<<<grid, block, 0, c->stream>>>(f.rk[cur], f.rk[cur ^ 1], static_cast<uint32_t>(E));
    cur ^= 1;
  }
  inetfin::fin_write<<<grid, block, 0, c->stream>>>(f, f.rk[cur]);
  CUDA_TRY(cudaGetLastError());
  uint32_t flag[2];
  CUDA_TRY(cudaMemcpyAsync(flag, f.flag, 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (flag[0]) return INET_OK;  // not a forest: the host finalizes
  const uint32_t total = flag[1];
  CUDA_TRY(cudaMemcpyAsync(c->d_agents.p, f.out, size_t(total) * 16, cudaMemcpyDeviceToDevice, c->stream));
  CUDA_TRY(cudaMemcpy2DAsync(c->d_resid.p, 8, f.out_iface, 4, 4, ni, cudaMemcpyDeviceToDevice, c->stream));
  k.pad[1] = total + 1;
  k.pad[2] = ni;
  return INET_OK;
}

int run(inet_ctx* c, const inet_cfg* cfg, float* device_ms, bool fetch) {
  if (!c) return INET_ERR_STATE;
  c->rows_hint = 0;
  int st = run_once(c, cfg, device_ms, fetch);
  if (c->collect_stats && !c->stats.empty()) {
    uint32_t need = 0;
    for (const auto& s : c->stats) need = std::max(need, s.rounds);
    need = std::min(need, kRowsMax);
    if (need > c->cap_rounds) {  // some net's rows did not fit: once more with room for all of them
      c->rows_hint = need;
      st = run_once(c, cfg, device_ms, fetch);
    }
  }
  return st;
}

int run_once(inet_ctx* c, const inet_cfg* cfg, float* device_ms, bool fetch) {
  if (!c || c->n_nets == 0 || c->blob.empty()) return INET_ERR_STATE;
  CUDA_TRY(cudaSetDevice(c->device));
  if (!c->input_resident) {
    int st = upload_input(c);
    if (st) return st;
  }
  const uint32_t max_loops = cfg ? cfg->max_loops : 1000000u;
  c->collect_stats = cfg && cfg->collect_stats;
  c->count_rules = cfg && cfg->count_rules;
  const uint32_t cap_rounds = c->collect_stats ? rows_cap(c, max_loops) : 0u;
  const uint32_t retries = cfg && cfg->max_retries ? cfg->max_retries : 8;
  float ms = 0;
  c->ctl.assign(c->n_nets, NetCtl{});
  auto any_oom = [&]() {
    for (uint32_t i = 0; i < c->n_nets; ++i)
      if (c->ctl[i].err == INET_ERR_ARENA) return true;
    return false;
  };
  auto fetch_ctl = [&]() -> int {
    static_assert(sizeof(NetCtl) % 4 == 0, "NetCtl words");
    c->h_ctl.resize(size_t(c->n_nets) * sizeof(NetCtl) / 4);
    CUDA_TRY(cudaMemcpyAsync(c->h_ctl.data(), c->d_ctl.p, c->n_nets * sizeof(NetCtl), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    std::memcpy(c->ctl.data(), c->h_ctl.data(), c->n_nets * sizeof(NetCtl));
    c->io_d2h += c->n_nets * sizeof(NetCtl);
    c->io_h2d += c->n_nets * sizeof(NetDesc);
    return INET_OK;
  };
  const bool user_caps = cfg && (cfg->cap_agents || cfg->cap_vars);
  // Reference loop mode: the rule-set kernel is first run without the
  // deferred-equation code (smaller and faster); it stops at the first merge
  // that leaves a var-headed equation (kNeedExact), and only then is the net
  // rerun with the full kernel. Nets whose merges only form active pairs (all
  // Ackermann nets) never need it, and their rounds are the reference's loops.
  const bool exact = cfg && cfg->exact_loops;
  bool with_defer = exact && !c->jit_mode;  // the prebuilt kernels always carry the code
  // Tier R: the reference's list order (ordered.cuh), capacities doubled on overflow.
  const bool ordered = cfg && (cfg->reference_order || cfg->validate_phases);
  // stamps (reference-ordered var = var keys) run on the single-CTA tiers only
  c->var_order = !ordered && cfg && cfg->var_order;
  if (ordered) {
    c->resume.on = false;  // a hand-over of an earlier single-net run must not leak into this layout
    c->promoted = false;
    const uint32_t pair_words = (c->n_labels * c->n_labels + 1) / 2;
    uint32_t max_fresh = 0;
    for (uint32_t r = 0; r < c->n_rules; ++r) max_fresh = std::max(max_fresh, (c->blob[4 + pair_words + r * 16] >> 16) & 0xFFu);
    uint32_t ca = cfg->cap_agents ? cfg->cap_agents : (c->n_nets == 1 ? (1u << 16) : 4096u);
    uint32_t cv = cfg->cap_vars ? cfg->cap_vars : (c->n_nets == 1 ? (1u << 16) : 4096u);
    uint32_t cl = c->n_nets == 1 ? (1u << 14) : 2048u;
    ca = std::max(ca, 2 * c->max_in_agents + 64);
    cv = std::max(cv, 2 * c->max_in_vars + 64);
    cl = std::max(cl, 2 * c->max_in_eqs + 64);
    bool done = false;
    for (uint32_t attempt = 0; !done; ++attempt) {
      Shape sh = base_shape(c, max_loops);
      sh.max_fresh = max_fresh;
      sh.validate = cfg->validate_phases ? 1u : 0u;
      c->ordered_tier = true;
      c->cap_list = cl;
      c->cap_out = 2 * cl;
      c->cap_def = 0;
      int st = layout(c, ca, cv, 1, cap_rounds);
      if (st == INET_OK) st = launch(c, cfg, sh, inetdev::kTierR, &ms);
      c->ordered_tier = false;
      if (st) return st;
      fetch_ctl();
      c->tier = inetdev::kTierR;
      c->shape = sh;
      if (!any_oom()) done = true;
      else if (attempt + 1 >= retries || uint64_t(ca) * 2 >= INET_VAR_BIT || uint64_t(cv) * 2 >= INET_VAR_BIT ||
               uint64_t(cl) * 4 >= INET_VAR_BIT)
        break;
      ca *= 2;
      cv *= 2;
      cl *= 2;
    }
  }
  for (int pass = 0; pass < 2 && !ordered; ++pass) {
  c->exact_code = with_defer || !c->jit_mode;
  bool done = false;
  c->promoted = false;
  c->promo_ms = 0;
  c->resume.on = false;
  // Try the shared-memory tiers first; a net that overflows sends the whole
  // launch to the next tier (S or M, then G with doubling capacities).
  auto attempt_tier = [&](int tier, const Shape& sh0, uint32_t ca, uint32_t cv, uint32_t cq) -> int {
    Shape sh = sh0;
    sh.exact = exact && c->exact_code ? 1u : 0u;
    sh.detect_vh = exact && !c->exact_code ? 1u : 0u;
    // deferred equations per round: the round's queue size is a safe bound in
    // practice; an overflow reports ARENA and the next attempt grows it
    c->cap_def = sh.exact ? (tier == kTierC ? c->cluster_g * 1024u : std::max<uint32_t>(256u, tier == kTierG ? cq : sh.res_queue))
                       : 0u;
    int st = layout(c, ca, cv, cq, cap_rounds);
    if (st) return st;
    st = launch(c, cfg, sh, tier, &ms);
    if (st) return st;
    fetch_ctl();
    c->tier = tier;
    c->shape = sh;
    if (std::getenv("INET_B200_DEBUG"))
      std::fprintf(stderr, "inet_b200: attempt tier %d caps %u/%u/%u: %.3f ms, net 0 status 0x%x (%u, %u)\n", tier, ca, cv,
                   cq, ms, c->ctl[0].err, c->ctl[0].err_a, c->ctl[0].err_b);
    return INET_OK;
  };
  if (!user_caps && c->n_nets > 1 && c->max_in_agents <= 512 && c->max_in_vars <= 512) {
    for (uint32_t cap : {1024u, 2048u}) {
      Shape sh = base_shape(c, max_loops);
      sh.res_agents = cap;
      sh.res_vars = cap;
      sh.res_queue = cap / 2;
      sh.ring_a = cap;
      sh.ring_v = cap;
      if (const char* e = std::getenv("INET_B200_SCAP")) {  // development: agents,vars,queue,ring
        unsigned a = 0, v = 0, q = 0, rg = 0;
        if (std::sscanf(e, "%u,%u,%u,%u", &a, &v, &q, &rg) == 4 && cap == 1024u) {
          sh.res_agents = a;
          sh.res_vars = v;
          sh.res_queue = q;
          sh.ring_a = sh.ring_v = rg;
        }
      }
      c->zc_next = c->dev_final;
      int st = attempt_tier(kTierS, sh, sh.res_agents, sh.res_vars, 1);
      c->zc_next = false;
      if (st == INET_OK && !any_oom()) {
        done = true;
        break;
      }
      if (st != INET_OK && st != INET_ERR_UNSUPPORTED) return st;
    }
  }
  // Large single nets: a cluster of G CTAs sharing their shared memory (tier C).
  // Its arenas are fixed by shared memory; a net that outgrows them falls
  // through to the single-CTA tiers.
  // auto (0): a single net starts on one CTA (tier M, lowest per-round cost);
  // past 2^19 interactions tier M hands it over — arena, slot table, pending
  // equations, rounds and totals — and a 16-CTA cluster (tier C) resumes it
  // from there, which wins once rounds are wide. 1 forces one CTA per net.
  if (const char* e = std::getenv("INET_B200_SINGLE_S"); e && !done && c->n_nets == 1 && !user_caps) {
    // development: a single net on tier S with these capacities (agents,vars,queue,ring)
    unsigned a = 0, v = 0, q = 0, rg = 0;
    if (std::sscanf(e, "%u,%u,%u,%u", &a, &v, &q, &rg) == 4) {
      Shape sh = base_shape(c, max_loops);
      sh.res_agents = a;
      sh.res_vars = v;
      sh.res_queue = q;
      sh.ring_a = sh.ring_v = rg;
      const int st = attempt_tier(kTierS, sh, a, v, 1);
      if (st == INET_OK && !any_oom()) done = true;
      else if (st != INET_OK && st != INET_ERR_UNSUPPORTED) return st;
    }
  }
  uint32_t want_g = cfg ? cfg->ctas_per_net : 0;
  if (c->var_order) want_g = 1;  // no cluster or whole-GPU tier: one CTA, tier M then G
  if (!done && want_g == 0 && c->n_nets == 1 && !user_caps) {
    want_g = 16;
    if (c->max_in_agents < 32768 && c->max_in_vars < 16384) {
      Shape sh = base_shape(c, max_loops);
      sh.res_vars = 14336;
      sh.res_queue = tier_m_queue(c);
      sh.ring_a = 8192;
      sh.ring_v = 8192;
      sh.promote_ints = c->promote_ints;
      // capacities that also fit the cluster tier, so the hand-over needs no copy
      int st = attempt_tier(kTierM, sh, kPromoCapAgents, kPromoCapVars, kPromoCapQueue);
      if (st == INET_OK && !any_oom() && c->ctl[0].err != inetdev::kPromote) {
        done = true;
      } else if (st == INET_OK && c->ctl[0].err == inetdev::kPromote) {
        c->promoted = true;  // its time counts towards the reduction
        c->promo_shape = c->shape;
        c->promo_cap_def = c->cap_def;
        c->promo_ms = ms;
        set_resume(c, c->ctl[0]);
      } else if (st != INET_OK && st != INET_ERR_UNSUPPORTED) {
        return st;
      }
    }
  }
  if (!done && want_g >= 2 && want_g <= 16 && c->n_nets <= 64) {
    uint32_t G = 2;  // a power of two (ids are owned round-robin: owner = id & (G - 1))
    while (G * 2 <= std::min<uint32_t>(want_g, 16)) G *= 2;
    Shape sh = base_shape(c, max_loops);
    sh.res_agents = 4096;
    sh.res_vars = 4096;
    sh.res_queue = 256;  // pairs one CTA can deal to one CTA per round
    sh.ring_a = 4096;
    sh.ring_v = 4096;
    c->cluster_g = G;
    int st = attempt_tier(kTierC, sh, G * sh.res_agents, G * sh.res_vars, 1);
    if (st == INET_OK && !any_oom()) done = true;
    else if (st != INET_OK && st != INET_ERR_UNSUPPORTED) return st;
    if (!done) {
      c->resume.on = false;  // the single-CTA tiers below start over from the input
      c->promoted = false;
    }
  }
  // Single nets too large for a cluster (or ctas_per_net > 16): the whole GPU
  // (tier X), capacities doubled on overflow.
  if (!done && c->n_nets == 1 && (cfg ? cfg->ctas_per_net : 0) != 1 && !c->var_order) {
    uint32_t ca = cfg && cfg->cap_agents ? cfg->cap_agents : (1u << 20);
    uint32_t cv = cfg && cfg->cap_vars ? cfg->cap_vars : (1u << 20);
    ca = std::max(ca, c->max_in_agents + 64);
    cv = std::max(cv, c->max_in_vars + 64);
    for (uint32_t attempt = 0; !done; ++attempt) {
      uint32_t ra = 1, rv = 1;
      while (ra < ca) ra *= 2;
      while (rv < cv) rv *= 2;
      Shape sh = base_shape(c, max_loops);
      sh.ring_a = ra;
      sh.ring_v = rv;
      c->grid_tier = true;
      int st = attempt_tier(inetdev::kTierX, sh, ra, rv, ra / 2 + 1);
      c->grid_tier = false;
      if (st == INET_ERR_UNSUPPORTED) break;
      if (st) return st;
      if (!any_oom()) {
        done = true;
        break;
      }
      if (attempt + 1 >= retries || uint64_t(ra) * 2 >= INET_VAR_BIT) break;
      ca = ra * 2;
      cv = rv * 2;
    }
  }
  if (!done && !user_caps && c->n_nets <= 148 && c->max_in_agents < 32768 && c->max_in_vars < 16384) {
    Shape sh = base_shape(c, max_loops);
    sh.res_vars = 14336;
    sh.res_queue = tier_m_queue(c);
    sh.ring_a = 8192;
    sh.ring_v = 8192;
    int st = attempt_tier(kTierM, sh, 65535, sh.res_vars, 1);
    if (st == INET_OK && !any_oom()) done = true;
    else if (st != INET_OK && st != INET_ERR_UNSUPPORTED) return st;
  }
  uint32_t ca = cfg && cfg->cap_agents ? cfg->cap_agents : 0;
  uint32_t cv = cfg && cfg->cap_vars ? cfg->cap_vars : 0;
  if (!ca) ca = c->n_nets == 1 ? (1u << 20) : 4096u;
  if (!cv) cv = c->n_nets == 1 ? (1u << 20) : 8192u;
  ca = std::max(ca, c->max_in_agents + 64);
  cv = std::max(cv, c->max_in_vars + 64);
  for (uint32_t attempt = 0; !done; ++attempt) {
    Shape sh = base_shape(c, max_loops);
    sh.ring_a = c->n_nets == 1 ? 8192 : 1024;
    sh.ring_v = c->n_nets == 1 ? 8192 : 1024;
    int st = attempt_tier(kTierG, sh, ca, cv, ca / 2 + 1);
    if (st) return st;
    if (!any_oom() || attempt + 1 >= retries) break;
    if (uint64_t(ca) * 2 >= INET_VAR_BIT || uint64_t(cv) * 2 >= INET_VAR_BIT) break;
    ca *= 2;
    cv *= 2;
  }
  if (!exact || c->exact_code) break;
  bool need = false;
  for (uint32_t i = 0; i < c->n_nets; ++i) need |= c->ctl[i].err == inetdev::kNeedExact;
  if (!need) break;
  with_defer = true;
  }
  if (c->promoted && c->tier != kTierC) c->promoted = false;  // the cluster fell through: no prefix
  if (device_ms) *device_ms = ms + (c->promoted ? c->promo_ms : 0.0f);
  if (fetch && c->dev_final && c->tier == inetdev::kTierX && c->n_nets == 1 && c->ctl[0].err == 0) {
    const int st = device_finalize_x(c);
    if (st) return st;
  }
  return finish_run(c, fetch);
}

// Per-net statistics from the fetched control blocks and, with fetch, the
// result arrays (arena prefixes, residual equations, rows) of the last launch.
int finish_run(inet_ctx* c, bool fetch) {
  c->stats.assign(c->n_nets, inet_net_stats{});
  c->dev_rows.assign(c->n_nets, 0);
  int first = INET_OK;
  for (uint32_t i = 0; i < c->n_nets; ++i) {
    const NetCtl& k = c->ctl[i];
    if ((c->tier == kTierS || c->tier == inetdev::kTierX) && k.err == 0) c->dev_rows[i] = k.pad[1];
    inet_net_stats& s = c->stats[i];
    s.interactions = k.interactions;
    s.communications = k.communications;
    s.rounds = k.rounds;
    s.status = k.err;
    s.err_label_a = k.err_a;
    s.err_label_b = k.err_b;
    s.agent_hw = std::min(k.agent_bump, c->cap_agents);
    s.var_hw = std::min(k.var_bump, c->cap_vars);
    s.n_residual = k.n_residual;
    s.cap_agents = c->cap_agents;
    s.cap_vars = c->cap_vars;
    s.tier = static_cast<uint32_t>(c->tier);
    s.jit = c->last_jit ? 1u : 0u;
    s.sm_mhz = k.pad[0];
    s.device_final = c->dev_rows[i] ? 1u : 0u;
    s.threads = c->last_threads;
    if (first == INET_OK && k.err) first = static_cast<int>(k.err);
  }
  c->reduced = true;
  c->text_net = INET_NONE;
  c->texts.clear();
  c->results.assign(c->n_nets, inethost::NormalForm{});
  c->finalized.assign(c->n_nets, 0);
  if (fetch) {
    // results: agent slabs up to the high-water, residual equations, round rows
    // (nets finalized on the device: their compacted normal form and interface)
    uint32_t max_hw = 0, max_res = 0;
    for (uint32_t i = 0; i < c->n_nets; ++i) {
      const inet_net_stats& s = c->stats[i];
      const bool dev = c->dev_rows[i] != 0;
      max_hw = std::max(max_hw, dev ? c->dev_rows[i] - 1 : s.agent_hw);
      max_res = std::max(max_res, dev ? c->ctl[i].pad[2] : s.n_residual);
    }
    // strided copies of each slab's used prefix
    c->agent_pitch = c->zc_used ? c->cap_agents : std::max(max_hw, 1u);
    c->resid_pitch = std::max(max_res, 1u);
    if (!c->zc_used) c->h_agents.resize(size_t(c->n_nets) * c->agent_pitch * 4);
    c->h_resid.resize(size_t(c->n_nets) * c->resid_pitch * 2);
    if (max_hw && !c->zc_used)
      CUDA_TRY(cudaMemcpy2DAsync(c->h_agents.data(), size_t(c->agent_pitch) * 16, c->d_agents.p,
                                 size_t(c->cap_agents) * 16, size_t(max_hw) * 16, c->n_nets, cudaMemcpyDeviceToHost,
                                 c->stream));
    if (max_res)
      CUDA_TRY(cudaMemcpy2DAsync(c->h_resid.data(), size_t(c->resid_pitch) * 8, c->d_resid.p, size_t(c->cap_vars) * 8,
                                 size_t(max_res) * 8, c->n_nets, cudaMemcpyDeviceToHost, c->stream));
    if (c->collect_stats) {
      uint32_t max_r = 0;
      for (auto& s : c->stats) max_r = std::max(max_r, std::min(s.rounds, c->cap_rounds));
      c->rows_pitch = std::max(max_r, 1u);  // host copy: only the rows some net used
      c->h_rounds.resize(size_t(c->n_nets) * c->rows_pitch * 4);
      if (max_r)
        CUDA_TRY(cudaMemcpy2DAsync(c->h_rounds.data(), size_t(c->rows_pitch) * 16, c->d_stats.p,
                                   size_t(c->cap_rounds) * 16, size_t(max_r) * 16, c->n_nets,
                                   cudaMemcpyDeviceToHost, c->stream));
    }
    if (c->count_rules) {
      c->h_hist.resize(size_t(c->n_nets) * hist_stride(c));
      CUDA_TRY(cudaMemcpyAsync(c->h_hist.data(), c->d_hist.p, c->h_hist.size() * 4, cudaMemcpyDeviceToHost, c->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->io_d2h += size_t(c->n_nets) * (size_t(max_hw) * 16 + size_t(max_res) * 8);
    if (c->collect_stats) {
      uint32_t max_r = 0;
      for (auto& s : c->stats) max_r = std::max(max_r, std::min(s.rounds, c->cap_rounds));
      c->io_d2h += size_t(c->n_nets) * max_r * 16;
    }
  }
  return first;
}

}  // namespace

extern "C" {

int inet_batch_reduce(inet_ctx* c, const inet_cfg* cfg, float* device_ms) {
  try {
    if (!c) return INET_ERR_ARG;
    c->input_resident = false;
    c->io_h2d = c->io_d2h = 0;
    return run(c, cfg, device_ms, true);
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_batch_rerun(inet_ctx* c, const inet_cfg* cfg, float* device_ms) {
  try {
    if (!c || !c->reduced) return INET_ERR_STATE;
    // same tier, shape and capacities as the successful run: no growth expected
    inet_cfg k = cfg ? *cfg : inet_cfg{1000000u, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    c->count_rules = k.count_rules != 0;
    CUDA_TRY(cudaSetDevice(c->device));
    const uint32_t cap_rounds = k.collect_stats ? rows_cap(c, k.max_loops) : 0u;
    float pre_ms = 0;
    if (c->promoted) {
      // replay the single-CTA prefix up to the promotion threshold, then the cluster run
      const uint32_t ca = c->cap_agents, cv = c->cap_vars, cq = c->cap_queue, cd = c->cap_def;
      c->cap_def = c->promo_cap_def;
      c->resume.on = false;
      int st = layout(c, kPromoCapAgents, kPromoCapVars, kPromoCapQueue, cap_rounds);
      if (st) return st;
      Shape ps = c->promo_shape;
      ps.max_rounds = k.max_loops;
      st = launch(c, &k, ps, kTierM, &pre_ms);
      if (st) return st;
      NetCtl m;
      CUDA_TRY(cudaMemcpy(&m, c->d_ctl.p, sizeof(NetCtl), cudaMemcpyDeviceToHost));
      if (m.err != inetdev::kPromote) return INET_ERR_STATE;
      set_resume(c, m);
      c->cap_def = cd;
      c->cap_agents = ca;
      c->cap_vars = cv;
      c->cap_queue = cq;
    }
    c->grid_tier = c->tier == inetdev::kTierX;
    c->ordered_tier = c->tier == inetdev::kTierR;
    c->zc_next = c->tier == kTierS && c->dev_final && c->n_nets > 1;
    int st = layout(c, c->cap_agents, c->cap_vars, c->cap_queue, cap_rounds);
    c->grid_tier = false;
    c->ordered_tier = false;
    c->zc_next = false;
    if (st) return st;
    Shape sh = c->shape;
    sh.max_rounds = k.max_loops;
    float ms = 0;
    st = launch(c, &k, sh, c->tier, &ms);
    if (st) return st;
    if (device_ms) *device_ms = ms + pre_ms;
    return INET_OK;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_batch_collect(inet_ctx* c) {
  try {
    if (!c || !c->reduced) return INET_ERR_STATE;
    CUDA_TRY(cudaSetDevice(c->device));
    c->ctl.assign(c->n_nets, NetCtl{});
    CUDA_TRY(cudaMemcpy(c->ctl.data(), c->d_ctl.p, c->n_nets * sizeof(NetCtl), cudaMemcpyDeviceToHost));
    c->collect_stats = c->cap_rounds != 0;
    return finish_run(c, true);
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_batch_stats(inet_ctx* c, uint32_t net, inet_net_stats* out) {
  try {
    if (!c || !out) return INET_ERR_ARG;
    if (!c->reduced) return INET_ERR_STATE;
    if (net >= c->n_nets) return INET_ERR_ARG;
    *out = c->stats[net];
    return INET_OK;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_jit_compile(const uint32_t* blob, size_t n_words, int tier, uint32_t threads, char* log, size_t log_len) {
  try {
    if (!blob || n_words < 4) return INET_ERR_ARG;
    if (int st = inethost::validate_rule_blob(blob, n_words)) return st;
    std::vector<char> cubin;
    std::string msg;
    int style = default_style(tier);
    if (const char* e = std::getenv("INET_B200_JITSTYLE")) style = std::atoi(e);
    bool exact_code = true;
    if (const char* e = std::getenv("INET_B200_EXACTCODE")) exact_code = std::atoi(e) != 0;
    const int rc =
        inetjit::compile_cubin(inetjit::kernel_source(blob, n_words, tier, threads, style, exact_code), cubin, msg);
    if (log && log_len) {
      std::strncpy(log, msg.c_str(), log_len - 1);
      log[log_len - 1] = 0;
    }
    return rc == 0 ? INET_OK : INET_ERR_UNSUPPORTED;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_jit_precompile(const uint32_t* blob, size_t n_words, int tier, uint32_t threads, uint32_t flags, char* log,
                        size_t log_len) {
  try {
    if (!blob || n_words < 4) return INET_ERR_ARG;
    if (int st = inethost::validate_rule_blob(blob, n_words)) return st;
    if (tier < kTierS || tier > inetdev::kTierX) return INET_ERR_ARG;
    // as jit_kernel picks it, or flags bits 8-11 = style + 1; bit 3: without per-round rows
    const int style = (flags >> 8) & 15u ? static_cast<int>(((flags >> 8) & 15u) - 1u) : default_style(tier);
    std::string msg;
    const int rc = inetjit::precompile(
        inetjit::kernel_source(blob, n_words, tier, threads, style, (flags & 1u) != 0, (flags & 2u) != 0,
                               (flags & 4u) != 0, (flags & 8u) == 0),
        msg);
    if (log && log_len) {
      std::strncpy(log, msg.c_str(), log_len - 1);
      log[log_len - 1] = 0;
    }
    return rc == 0 ? INET_OK : INET_ERR_UNSUPPORTED;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_set_jit(inet_ctx* c, int mode) {
  try {
    if (!c) return INET_ERR_ARG;
    c->jit_mode = mode ? 1 : 0;
    return INET_OK;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_batch_rule_counts(inet_ctx* c, uint32_t net, uint64_t* counts, uint32_t n_rules) {
  try {
    if (!c || !counts) return INET_ERR_ARG;
    if (!c->reduced || !c->count_rules || c->h_hist.empty()) return INET_ERR_STATE;
    if (net >= c->n_nets) return INET_ERR_ARG;
    const uint32_t R = hist_stride(c);
    for (uint32_t r = 0; r < n_rules; ++r) counts[r] = r < R ? c->h_hist[size_t(net) * R + r] : 0;
    return INET_OK;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_batch_io_bytes(inet_ctx* c, uint64_t* h2d, uint64_t* d2h) {
  try {
    if (!c) return INET_ERR_ARG;
    if (h2d) *h2d = c->io_h2d;
    if (d2h) *d2h = c->io_d2h;
    return INET_OK;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_batch_totals(inet_ctx* c, uint64_t* interactions, uint64_t* communications, uint32_t* max_rounds,
                      uint32_t* n_failed) {
  try {
    if (!c) return INET_ERR_ARG;
    if (!c->reduced) return INET_ERR_STATE;
    uint64_t ti = 0, tc = 0;
    uint32_t mr = 0, nf = 0;
    for (auto& s : c->stats) {
      ti += s.interactions;
      tc += s.communications;
      mr = std::max(mr, s.rounds);
      nf += s.status != INET_OK;
    }
    if (interactions) *interactions = ti;
    if (communications) *communications = tc;
    if (max_rounds) *max_rounds = mr;
    if (n_failed) *n_failed = nf;
    return INET_OK;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_batch_rounds(inet_ctx* c, uint32_t net, uint32_t* rows, uint32_t* n_rows) {
  try {
    if (!c || !n_rows) return INET_ERR_ARG;
    if (!c->reduced) return INET_ERR_STATE;
    if (net >= c->n_nets) return INET_ERR_ARG;
    if (!c->collect_stats) {
      *n_rows = 0;
      return INET_OK;
    }
    const uint32_t n = std::min(c->stats[net].rounds, c->cap_rounds);
    if (!rows) {
      *n_rows = n;
      return INET_OK;
    }
    const uint32_t m = std::min(n, *n_rows);
    std::memcpy(rows, c->h_rounds.data() + size_t(net) * c->rows_pitch * 4, size_t(m) * 16);
    *n_rows = m;
    return INET_OK;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_batch_finalize(inet_ctx* c, uint32_t net, uint32_t n_threads) {
  try {
    if (!c) return INET_ERR_ARG;
    if (!c->reduced) return INET_ERR_STATE;
    return inethost::finalize_batch(*c, net, n_threads);
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_batch_print(inet_ctx* c, uint32_t net, const char* const* names, const uint8_t* arity, uint32_t n_labels,
                     char* buf, size_t cap, size_t* len) {
  try {
    if (!c || !len || (n_labels && (!names || !arity))) return INET_ERR_ARG;
    if (!c->reduced || net >= c->n_nets || !c->finalized[net]) return INET_ERR_STATE;
    if (c->text_net != net) {
      const inethost::NormalForm& nf = c->results[net];
      c->text_net = INET_NONE;
      const int st = inethost::print_flat(nf.agent_data(), nf.n_agents(), nf.iface.data(),
                                          static_cast<uint32_t>(nf.iface.size()), nf.eqs.data(),
                                          static_cast<uint32_t>(nf.eqs.size() / 2), names, arity, n_labels, c->text);
      if (st) return st;
      c->text_net = net;
    }
    return inethost::copy_text(c->text, buf, cap, len);
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_batch_stats_all(inet_ctx* c, inet_net_stats* out, uint32_t n) {
  try {
    if (!c || !out) return INET_ERR_ARG;
    if (!c->reduced) return INET_ERR_STATE;
    if (n != c->n_nets) return INET_ERR_ARG;
    std::memcpy(out, c->stats.data(), size_t(n) * sizeof(inet_net_stats));
    return INET_OK;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_batch_result_counts(inet_ctx* c, uint32_t* n_agents, uint32_t* n_iface, uint32_t* n_eqs, uint32_t n) {
  try {
    if (!c) return INET_ERR_ARG;
    if (!c->reduced) return INET_ERR_STATE;
    if (n != c->n_nets) return INET_ERR_ARG;
    for (uint32_t i = 0; i < n; ++i) {
      const bool ok = c->finalized[i] != 0;
      const inethost::NormalForm& nf = c->results[i];
      if (n_agents) n_agents[i] = ok ? nf.n_agents() : 0u;
      if (n_iface) n_iface[i] = ok ? static_cast<uint32_t>(nf.iface.size()) : 0u;
      if (n_eqs) n_eqs[i] = ok ? static_cast<uint32_t>(nf.eqs.size() / 2) : 0u;
    }
    return INET_OK;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_batch_print_all(inet_ctx* c, const char* const* names, const uint8_t* arity, uint32_t n_labels,
                         uint32_t n_threads, char* buf, size_t cap, uint64_t* offsets, size_t* len) {
  try {
    if (!c || !len || (n_labels && (!names || !arity))) return INET_ERR_ARG;
    if (!c->reduced) return INET_ERR_STATE;
    if (!buf || c->texts.size() != c->n_nets) {
      // print every finalized net (in parallel over host threads); failed nets print empty
      c->texts.assign(c->n_nets, std::string());
      const int st = inethost::parallel_for(c->n_nets, n_threads, [&](uint32_t i) -> int {
        if (!c->finalized[i]) return INET_OK;
        const inethost::NormalForm& nf = c->results[i];
        return inethost::print_flat(nf.agent_data(), nf.n_agents(), nf.iface.data(), static_cast<uint32_t>(nf.iface.size()),
                                    nf.eqs.data(), static_cast<uint32_t>(nf.eqs.size() / 2), names, arity, n_labels,
                                    c->texts[i]);
      });
      if (st) return st;
    }
    size_t total = 0;
    for (const auto& t : c->texts) total += t.size();
    *len = total;
    if (!buf || cap < total) return INET_OK;  // size query: call again with a buffer of *len bytes
    size_t pos = 0;
    for (uint32_t i = 0; i < c->n_nets; ++i) {
      if (offsets) offsets[i] = pos;
      std::memcpy(buf + pos, c->texts[i].data(), c->texts[i].size());
      pos += c->texts[i].size();
    }
    if (offsets) offsets[c->n_nets] = pos;
    c->texts.clear();
    return INET_OK;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

int inet_batch_result(inet_ctx* c, uint32_t net, const uint32_t** agents, uint32_t* n_agents, const uint32_t** iface,
                      uint32_t* n_iface, const uint32_t** eqs, uint32_t* n_eqs) {
  try {
    if (!c) return INET_ERR_ARG;
    if (!c->reduced || net >= c->n_nets || !c->finalized[net]) return INET_ERR_STATE;
    const inethost::NormalForm& nf = c->results[net];
    if (agents) *agents = nf.agent_data();
    if (n_agents) *n_agents = nf.n_agents();
    if (iface) *iface = nf.iface.data();
    if (n_iface) *n_iface = static_cast<uint32_t>(nf.iface.size());
    if (eqs) *eqs = nf.eqs.data();
    if (n_eqs) *n_eqs = static_cast<uint32_t>(nf.eqs.size() / 2);
    return INET_OK;
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

}  // extern "C"

// ---------------------------------------------------------------------------
// glue used by host.cpp (kept here because it needs the ctx layout)

namespace inethost {

int validate_nets(const inet_ctx& c) {
  const uint32_t L = c.n_labels;
  for (uint32_t i = 0; i < c.n_nets; ++i) {
    const uint64_t a0 = c.agent_off[i], a1 = c.agent_off[i + 1];
    const uint32_t na = static_cast<uint32_t>(a1 - a0), nv = c.n_vars[i];
    auto ok_ref = [&](uint32_t r) {
      if (r == INET_NONE) return false;
      if (r & INET_VAR_BIT) return (r & ~INET_VAR_BIT) < nv;
      return r < na;
    };
    for (uint64_t a = a0; a < a1; ++a) {
      const uint32_t* rec = &c.agents[4 * a];
      if (rec[0] >= L) return INET_ERR_UNSUPPORTED;
      for (int k = 1; k < 4; ++k)
        if (rec[k] != INET_NONE && !ok_ref(rec[k])) return INET_ERR_ARG;
    }
    for (uint64_t e = c.eq_off[i]; e < c.eq_off[i + 1]; ++e)
      if (!ok_ref(c.eqs[2 * e]) || !ok_ref(c.eqs[2 * e + 1])) return INET_ERR_ARG;
    for (uint64_t k = c.iface_off[i]; k < c.iface_off[i + 1]; ++k)
      if (!ok_ref(c.iface[k])) return INET_ERR_ARG;
  }
  return INET_OK;
}

int finalize_batch(inet_ctx& c, uint32_t net, uint32_t n_threads) {
  auto one = [&](uint32_t i) -> int {
    const inet_net_stats& s = c.stats[i];
    if (s.status != INET_OK) return static_cast<int>(s.status);
    if (const uint32_t rows = i < c.dev_rows.size() ? c.dev_rows[i] : 0u) {
      // finalized on the device: copy out the compacted normal form
      NormalForm& nf = c.results[i];
      const uint32_t* ag = host_agents(c) + size_t(i) * c.agent_pitch * 4;
      const uint32_t* rs = c.h_resid.data() + size_t(i) * c.resid_pitch * 2;
      const uint32_t ni = static_cast<uint32_t>(c.iface_off[i + 1] - c.iface_off[i]);
      nf.agents.clear();
      nf.ext_agents = ag;
      nf.ext_n = rows - 1;
      nf.iface.resize(ni);
      for (uint32_t k = 0; k < ni; ++k) nf.iface[k] = rs[2 * k];
      nf.eqs.clear();
      c.finalized[i] = 1;
      return INET_OK;
    }
    NetView v;
    v.agents = host_agents(c) + size_t(i) * c.agent_pitch * 4;
    v.n_agents = s.agent_hw;
    v.residual = c.h_resid.data() + size_t(i) * c.resid_pitch * 2;
    v.n_residual = s.n_residual;
    v.iface = c.iface.data() + c.iface_off[i];
    v.n_iface = static_cast<uint32_t>(c.iface_off[i + 1] - c.iface_off[i]);
    v.n_vars = s.var_hw;
    int st = finalize_net(v, c.results[i]);
    if (st == INET_OK) c.finalized[i] = 1;
    return st;
  };
  if (net != INET_NONE) {
    if (net >= c.n_nets) return INET_ERR_ARG;
    return one(net);
  }
  // nets the device finalized only need their pointers set: no worker threads
  // for them (spawning 16 threads costs more than the whole loop)
  uint32_t host_nets = 0;
  for (uint32_t i = 0; i < c.n_nets; ++i) host_nets += i >= c.dev_rows.size() || c.dev_rows[i] == 0;
  if (host_nets == 0) {
    int first = INET_OK;
    for (uint32_t i = 0; i < c.n_nets; ++i) {
      const int st = one(i);
      if (st != INET_OK && first == INET_OK) first = st;
    }
    return first;
  }
  return parallel_for(c.n_nets, n_threads, one);
}

}  // namespace inethost
