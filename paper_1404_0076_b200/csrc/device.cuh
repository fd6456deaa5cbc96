// device.cuh — device-side data model and the per-net reduction loop.
//
// One CTA owns one net and runs the reference's main loop
// (engine.py:204-223) to the fixpoint inside a single launch:
//
//   round r:  every queued active pair is rewritten by its rule
//             (interaction_phase, engine.py:77-134 + core.py:281-304);
//             every right-hand-side equation that is not active is linked
//             through the variable-slot table at once (communication_phase,
//             engine.py:137-166), to a fixpoint, so merges that produce new
//             active pairs feed round r+1 directly;
//             one __syncthreads() ends the round.
//
// The sort + reduce_by_key of the reference (and of the paper's Thrust
// pipeline) is replaced by an exchange on vslot[x]: the first whole-side
// occurrence of x parks its other side there, the second takes it and forms
// the merged equation (reduce_by_key's merge lambda, engine.py:161-165).
// var=var equations are keyed by the smaller id as in engine.py:150-153.
//
// Because a net never leaves its CTA, every counter (queue tail, allocators,
// statistics) and both free rings live in shared memory. Three residency
// tiers share this code (chosen per launch by the host, falling back S -> G
// or M -> G when a net outgrows its shared-memory arena):
//
//   S  agents, variable slots, queues in shared memory (small nets: the
//      4096 x A(3,6) batch, several CTAs per SM);
//   M  variable slots and queues in shared memory, agents in global memory
//      (one large net per SM, e.g. A(3,10)); the exchanges that link
//      variables are shared-memory atomics, the only L2 round trip per
//      interaction is the read of the two agents;
//   G  everything but the counters and rings in global memory (unbounded).
//
// Tiers S and M pack an active pair into one 32-bit queue word (two 16-bit
// agent indices) and keep 16-bit free rings, so their arenas are capped at
// 65,535 agents.
//
// Memory: agents are 16-byte records {label, port0..2}. The two agents of an
// active pair are dead after the rewrite; their slots are reused in place for
// the first two right-hand-side agents, others come from a round-phased free
// ring (ids freed in round r become allocatable in round r+1), then from a
// bump pointer. Variable ids are recycled the same way once both occurrences
// have met. A full ring drops the id (it is simply never reused).
#pragma once
#ifndef __CUDACC_RTC__
#include <cstdint>
#endif

#include "../../include/inet_b200.h"

namespace inetdev {

constexpr uint32_t kVar = INET_VAR_BIT;
constexpr uint32_t kNone = INET_NONE;
constexpr int kEnvFresh = 6;
constexpr int kEnvNew = 14;
constexpr int kEnvNone = 22;
constexpr int kEnvSize = 23;  // sources 0..22 (22 = none)
constexpr int kRuleWords = 16;
constexpr int kFastEq = 4;  // rhs equations linked with overlapped exchanges

enum : int { kTierS = 0, kTierM = 1, kTierG = 2 };

template <int kTier>
struct Traits {
  using Ring = uint16_t;
  static constexpr bool kEnvSmem = false;           // per-thread source table in shared memory
  static constexpr bool kEnvLocal = kTier == kTierS;  // per-thread source table in local memory (L1)
  static constexpr bool kAgentsSmem = kTier == kTierS;
  static constexpr bool kSlotsSmem = true;
  static constexpr bool kPacked = true;
};
template <>
struct Traits<kTierG> {
  using Ring = uint32_t;
  static constexpr bool kEnvSmem = false;
  static constexpr bool kEnvLocal = false;
  static constexpr bool kAgentsSmem = false;
  static constexpr bool kSlotsSmem = false;
  static constexpr bool kPacked = false;
};

// Counters of the running round, bumped by every thread while it works.
struct RoundCtr {
  uint32_t qcount;  // active pairs queued for the next round
  uint32_t atake;   // agent ring entries taken
  uint32_t afree;   // agents offered to the ring
  uint32_t vtake;
  uint32_t vfree;
  uint32_t ints;
  uint32_t comms;
  int32_t parked;   // delta of parked equations
  uint32_t err;     // any failure in this round
  uint32_t pad[3];
};

// Parameters of the next round, written by the last warp to finish a round
// (before the round's barrier) and read by every thread after it.
struct Header {
  uint32_t n;       // active pairs in the queue
  uint32_t stop;    // leave the loop
  uint32_t lo_a, hi_a, lo_v, hi_v;  // ring windows allocatable in this round
  uint32_t pad[2];
};

// Shared-memory control block of the net a CTA is reducing.
struct Ctl {
  RoundCtr ctr;
  Header hdr;
  uint32_t done_warps;
  uint32_t agent_bump;
  uint32_t var_bump;
  uint32_t err_code;
  uint32_t err_a;
  uint32_t err_b;
  uint32_t rounds;
  int32_t parked_total;
  unsigned long long t_prev;
  unsigned long long tot_i;
  unsigned long long tot_c;
  uint32_t scratch[34];
};

// Global result block of one net (read by the host).
struct NetCtl {
  uint32_t agent_bump;
  uint32_t var_bump;
  uint32_t err;
  uint32_t err_a;
  uint32_t err_b;
  uint32_t rounds;
  uint32_t n_residual;
  uint32_t parked_total;
  unsigned long long interactions;
  unsigned long long communications;
  uint32_t pad[4];
};

// Per-net device view of its private global arrays.
struct NetDesc {
  uint4* agents;       // cap_agents (tiers M/G arena; tier S result copy)
  uint32_t* vslot;     // cap_vars (tier G)
  uint2* queue;        // 2 * cap_queue (tier G)
  uint4* stats;        // cap_rounds rows {ints, comms, live, ns} or null
  uint2* residual;     // cap_vars
  NetCtl* ctl;
  uint32_t* rule_hist; // interactions per rule (accounting runs) or null
  uint32_t cap_agents, cap_vars, cap_queue, cap_rounds;
  // initial contents (device copies of the caller's flat arrays)
  const uint4* in_agents;
  const uint2* in_eqs;
  uint32_t n_in_agents, n_in_eqs, n_in_vars, pad;
};

// Launch-wide shape: ring sizes and the shared-memory capacities.
struct Shape {
  uint32_t ring_a, ring_v;        // powers of two
  uint32_t res_agents;            // tier S agents in shared memory
  uint32_t res_vars;              // tiers S/M variable slots in shared memory
  uint32_t res_queue;             // tiers S/M queue words per buffer
  uint32_t max_rounds;
  uint32_t rule_words;            // pair table + rule records (words)
  uint32_t n_labels;
  uint32_t threads;               // CTA size
  uint32_t pad;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#ifdef INET_TIMING
// Development build only: per-phase clock64 totals (tools/phase_timing.py).
#define INET_TMARK(c, k)                  \
  do {                                    \
    const long long _t = clock64();       \
    (c).tm[k] += _t - (c).tlast;          \
    (c).tlast = _t;                       \
  } while (0)
#else
#define INET_TMARK(c, k) \
  do {                   \
  } while (0)
#endif

template <class T>
__device__ __forceinline__ T vload(const T* p) {
  return *reinterpret_cast<const volatile T*>(p);
}

// Thread-private view of the running round.
template <int kTier>
struct Round {
  using Ring = typename Traits<kTier>::Ring;
  const NetDesc* d;
  Ctl* ctl;
  uint4* agents;
  uint32_t* vslot;
  Ring* aring;
  Ring* vring;
  uint32_t* env;  // this thread's column of the shared source table (stride blockDim)
  void* out;
  RoundCtr* cur;
  const uint16_t* pair;
  const uint32_t* rules;
  uint32_t n_labels;
  uint32_t cap_agents, cap_vars, cap_queue;
  uint32_t amask, vmask;
  uint32_t lo_a, hi_a, lo_v, hi_v;  // ring windows available this round
  uint32_t ints, comms;
  int32_t parked;
  bool failed;
#ifdef INET_TIMING
  long long tm[8];
  long long tlast;
#endif
};

template <int kTier>
__device__ __forceinline__ void fail(Round<kTier>& c, uint32_t code, uint32_t a = 0, uint32_t b = 0) {
  c.failed = true;
  c.cur->err = 1u;
  if (atomicCAS(&c.ctl->err_code, 0u, code) == 0u) {
    c.ctl->err_a = a;
    c.ctl->err_b = b;
  }
}

// A contiguous claim on a free ring: ids j < got are ring[(pos + j) & mask],
// the rest come from the bump pointer (bump + j - got).
struct Claim {
  uint32_t pos, got, bump;
};

template <int kTier>
__device__ __forceinline__ bool alloc_vars(Round<kTier>& c, uint32_t nf, Claim& k) {
  k.pos = k.got = k.bump = 0;
  if (nf == 0) return true;
  const uint32_t t = atomicAdd(&c.cur->vtake, nf);
  const uint32_t avail = c.hi_v - c.lo_v;
  k.pos = c.lo_v + t;
  if (t < avail) k.got = min(avail - t, nf);
  if (k.got < nf) {
    const uint32_t need = nf - k.got;
    k.bump = atomicAdd(&c.ctl->var_bump, need);
    if (k.bump + need > c.cap_vars) {
      fail(c, INET_ERR_ARENA, 1);
      return false;
    }
  }
  return true;
}

template <int kTier>
__device__ __forceinline__ bool alloc_agents(Round<kTier>& c, uint32_t n, Claim& k) {
  k.pos = k.got = k.bump = 0;
  if (n == 0) return true;
  const uint32_t t = atomicAdd(&c.cur->atake, n);
  const uint32_t avail = c.hi_a - c.lo_a;
  k.pos = c.lo_a + t;
  if (t < avail) k.got = min(avail - t, n);
  if (k.got < n) {
    const uint32_t need = n - k.got;
    k.bump = atomicAdd(&c.ctl->agent_bump, need);
    if (k.bump + need > c.cap_agents) {
      fail(c, INET_ERR_ARENA, 0);
      return false;
    }
  }
  return true;
}

template <int kTier>
__device__ __forceinline__ void free_agent(Round<kTier>& c, uint32_t a) {
  const uint32_t f = atomicAdd(&c.cur->afree, 1u);
  const uint32_t pos = c.hi_a + f;
  if (pos - c.lo_a <= c.amask) c.aring[pos & c.amask] = a;  // else dropped
}

template <int kTier>
__device__ __forceinline__ void free_var(Round<kTier>& c, uint32_t x) {
  const uint32_t f = atomicAdd(&c.cur->vfree, 1u);
  const uint32_t pos = c.hi_v + f;
  if (pos - c.lo_v <= c.vmask) c.vring[pos & c.vmask] = x;
}

template <int kTier>
__device__ __forceinline__ void push_active(Round<kTier>& c, uint32_t l, uint32_t r) {
  const uint32_t p = atomicAdd(&c.cur->qcount, 1u);
  if (p >= c.cap_queue) {
    fail(c, INET_ERR_ARENA, 2);
    return;
  }
  if constexpr (Traits<kTier>::kPacked)
    static_cast<uint32_t*>(c.out)[p] = (l << 16) | r;  // both < 65536 in tiers S/M
  else
    static_cast<uint2*>(c.out)[p] = make_uint2(l, r);
}

// Key and parked value of a non-active equation: var=var keys on the smaller id.
__device__ __forceinline__ void key_of(uint32_t l, uint32_t r, uint32_t& key, uint32_t& val) {
  const bool lv = (l & kVar) != 0, rv = (r & kVar) != 0;
  if (lv && rv) {
    key = l < r ? l : r;
    val = l < r ? r : l;
  } else if (lv) {
    key = l;
    val = r;
  } else {
    key = r;
    val = l;
  }
}

// Finish an exchange on slot x that returned `old`; continue linking the
// merged equation {x = old, x = val} -> old = val until it parks or is active.
template <int kTier>
__device__ __forceinline__ void settle(Round<kTier>& c, uint32_t x, uint32_t old, uint32_t val) {
  while (true) {
    if (old == kNone) {
      c.parked += 1;
      return;
    }
    c.vslot[x] = kNone;  // x is dead: both occurrences met
    c.comms += 1;
    c.parked -= 1;
    free_var(c, x);
    const uint32_t l = old, r = val;
    if (((l | r) & kVar) == 0) {
      push_active(c, l, r);
      return;
    }
    uint32_t key;
    key_of(l, r, key, val);
    x = key & ~kVar;
    old = atomicExch(&c.vslot[x], val);
  }
}

template <int kTier>
__device__ __forceinline__ void link(Round<kTier>& c, uint32_t l, uint32_t r) {
  if (((l | r) & kVar) == 0) {
    push_active(c, l, r);
    return;
  }
  uint32_t key, val;
  key_of(l, r, key, val);
  const uint32_t x = key & ~kVar;
  settle(c, x, atomicExch(&c.vslot[x], val), val);
}

#ifdef INET_JIT
// Helpers of the generated rewrites: allocation with compile-time counts into
// registers, and the first half of link() (push or exchange key).
template <uint32_t N, int kTier>
__device__ __forceinline__ bool jit_alloc_vars(Round<kTier>& c, uint32_t (&f)[N]) {
  Claim k;
  if (!alloc_vars(c, N, k)) return false;
#pragma unroll
  for (uint32_t j = 0; j < N; ++j)
    f[j] = kVar | (j < k.got ? static_cast<uint32_t>(c.vring[(k.pos + j) & c.vmask]) : k.bump + (j - k.got));
  return true;
}

template <uint32_t N, int kTier>
__device__ __forceinline__ bool jit_alloc_agents(Round<kTier>& c, uint32_t (&g)[N]) {
  Claim k;
  if (!alloc_agents(c, N, k)) return false;
#pragma unroll
  for (uint32_t j = 0; j < N; ++j)
    g[j] = j < k.got ? static_cast<uint32_t>(c.aring[(k.pos + j) & c.amask]) : k.bump + (j - k.got);
  return true;
}

// Active pair -> queue (returns false); otherwise the slot key and the parked value.
template <int kTier>
__device__ __forceinline__ bool jit_prep(Round<kTier>& c, uint32_t l, uint32_t r, uint32_t& x, uint32_t& val) {
  if (((l | r) & kVar) == 0) {
    push_active(c, l, r);
    return false;
  }
  uint32_t key;
  key_of(l, r, key, val);
  x = key & ~kVar;
  return true;
}

// Rule-set specialised rewrite, generated per rule set by csrc/jit.cpp: one
// straight-line case per rule with every source known at compile time.
template <int kTier>
__device__ __forceinline__ void jit_apply(Round<kTier>& c, uint32_t rule, const uint4& A, const uint4& B, uint32_t l,
                                          uint32_t r);
#endif

// Rewrite one active pair (find_rule + instantiate, core.py:281-312).
template <int kTier>
__device__ __forceinline__ void interact(Round<kTier>& c, uint32_t l, uint32_t r) {
  INET_TMARK(c, 0);
  uint4 A = c.agents[l];
  uint4 B = c.agents[r];
  const uint32_t t = c.pair[A.x * c.n_labels + B.x];
  INET_TMARK(c, 1);
  if (t == 0xFFFFu) {
    fail(c, INET_ERR_NO_RULE, A.x, B.x);
    return;
  }
  if (t & 1u) {
    const uint4 tmp = A;
    A = B;
    B = tmp;
    const uint32_t u = l;
    l = r;
    r = u;
  }
  if (c.d->rule_hist) atomicAdd(&c.d->rule_hist[t >> 1], 1u);
#ifdef INET_JIT
  jit_apply<kTier>(c, t >> 1, A, B, l, r);
  c.ints += 1;
  INET_TMARK(c, 4);
  return;
#endif
  const uint32_t* R = c.rules + (t >> 1) * kRuleWords;
  const uint32_t hdr = R[0];
  const uint32_t nn = hdr & 0xFFu, ne = (hdr >> 8) & 0xFFu, nf = (hdr >> 16) & 0xFFu;
  Claim fv, na;
  if (!alloc_vars(c, nf, fv)) return;
  if (!alloc_agents(c, nn > 2 ? nn - 2 : 0, na)) return;
  INET_TMARK(c, 2);
  auto fresh = [&](uint32_t j) -> uint32_t {
    return kVar | (j < fv.got ? static_cast<uint32_t>(c.vring[(fv.pos + j) & c.vmask]) : fv.bump + (j - fv.got));
  };
  auto extra = [&](uint32_t q) -> uint32_t {
    return q < na.got ? static_cast<uint32_t>(c.aring[(na.pos + q) & c.amask]) : na.bump + (q - na.got);
  };
  uint32_t env_l[Traits<kTier>::kEnvLocal ? kEnvSize : 1];
  if constexpr (Traits<kTier>::kEnvLocal) {
    // Small nets (tier S): a per-thread table in local memory; with several
    // CTAs per SM this measured faster than resolving sources by branches.
    env_l[0] = A.y;
    env_l[1] = A.z;
    env_l[2] = A.w;
    env_l[3] = B.y;
    env_l[4] = B.z;
    env_l[5] = B.w;
    for (uint32_t j = 0; j < nf; ++j) env_l[kEnvFresh + j] = fresh(j);
    env_l[kEnvNew] = l;
    env_l[kEnvNew + 1] = r;
    for (uint32_t q = 0; q + 2 < nn; ++q) env_l[kEnvNew + 2 + q] = extra(q);
    env_l[kEnvNone] = kNone;
  }
  if constexpr (Traits<kTier>::kEnvSmem) {
    // Source table in shared memory, one column per thread: every rule source
    // then resolves with a single LDS.
    uint32_t* E = c.env;
    const uint32_t bd = blockDim.x;
    E[0] = A.y;
    E[bd] = A.z;
    E[2 * bd] = A.w;
    E[3 * bd] = B.y;
    E[4 * bd] = B.z;
    E[5 * bd] = B.w;
    for (uint32_t j = 0; j < nf; ++j) E[(kEnvFresh + j) * bd] = fresh(j);
    E[kEnvNew * bd] = l;
    E[(kEnvNew + 1) * bd] = r;
    for (uint32_t q = 0; q + 2 < nn; ++q) E[(kEnvNew + 2 + q) * bd] = extra(q);
  }
  // Resolve a rule source (include/inet_b200.h) to a term ref.
  auto src = [&](uint32_t s) -> uint32_t {
    if constexpr (Traits<kTier>::kEnvSmem) {
      return c.env[s * blockDim.x];
    } else if constexpr (Traits<kTier>::kEnvLocal) {
      return env_l[s];
    } else {
      if (s < 3) return s == 0 ? A.y : (s == 1 ? A.z : A.w);
      if (s < 6) return s == 3 ? B.y : (s == 4 ? B.z : B.w);
      if (s < 14) return fresh(s - kEnvFresh);
      if (s < 22) {
        const uint32_t m = s - kEnvNew;
        if (m < 2) return m == 0 ? l : r;
        return extra(m - 2);
      }
      return kNone;
    }
  };
  for (uint32_t m = 0; m < nn; ++m) {
    const uint32_t w = R[1 + m];
    c.agents[src(kEnvNew + m)] = make_uint4(w & 0xFFu, src((w >> 8) & 0xFFu), src((w >> 16) & 0xFFu), src(w >> 24));
  }
  if (nn < 2) free_agent(c, r);
  if (nn < 1) free_agent(c, l);
  INET_TMARK(c, 3);
  // Link the rhs: issue the first exchange of every equation back to back so
  // their latencies overlap, then settle each.
  uint32_t xs[kFastEq], olds[kFastEq], vals[kFastEq];
#pragma unroll
  for (int e = 0; e < kFastEq; ++e) {
    xs[e] = kNone;
    if (e < static_cast<int>(ne)) {
      const uint32_t h = (R[9 + (e >> 1)] >> ((e & 1) * 16)) & 0xFFFFu;
      const uint32_t el = src(h & 0xFFu), er = src(h >> 8);
      if (((el | er) & kVar) == 0) {
        push_active(c, el, er);
      } else {
        uint32_t key;
        key_of(el, er, key, vals[e]);
        xs[e] = key & ~kVar;
        olds[e] = atomicExch(&c.vslot[xs[e]], vals[e]);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < kFastEq; ++e)
    if (xs[e] != kNone) settle(c, xs[e], olds[e], vals[e]);
  for (uint32_t e = kFastEq; e < ne; ++e) {
    const uint32_t h = (R[9 + (e >> 1)] >> ((e & 1) * 16)) & 0xFFFFu;
    link(c, src(h & 0xFFu), src(h >> 8));
  }
  c.ints += 1;
  INET_TMARK(c, 4);
}

// Block-wide exclusive prefix of a 0/1 flag; returns the total.
__device__ __forceinline__ uint32_t block_scan_flag(bool flag, uint32_t* warp_tot, uint32_t* my_off) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t nw = (blockDim.x + 31u) >> 5;
  const uint32_t bal = __ballot_sync(0xFFFFFFFFu, flag);
  const uint32_t below = __popc(bal & ((1u << lane) - 1u));
  if (lane == 0) warp_tot[warp] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (uint32_t w = 0; w < nw; ++w) {
      const uint32_t v = warp_tot[w];
      warp_tot[w] = s;
      s += v;
    }
    warp_tot[32] = s;
  }
  __syncthreads();
  *my_off = warp_tot[warp] + below;
  const uint32_t total = warp_tot[32];
  __syncthreads();
  return total;
}

// Shared-memory plan (32-bit words):
//   rule table | Ctl | agent ring | var ring | [S: agents] | [S,M: slots] | [S,M: 2 queues]
struct SmemPlan {
  uint32_t ctl_off, aring_off, vring_off, agents_off, slots_off, queue_off, env_off, words;
};

__host__ __device__ inline uint32_t align4(uint32_t w) { return (w + 3u) & ~3u; }

__host__ __device__ inline SmemPlan plan_smem(const Shape& sh, int tier) {
  const uint32_t ring_bytes = tier == kTierG ? 4u : 2u;
  SmemPlan p;
  p.ctl_off = align4(sh.rule_words);
  p.aring_off = p.ctl_off + align4(sizeof(Ctl) / 4);
  p.vring_off = p.aring_off + align4((sh.ring_a * ring_bytes + 3) / 4);
  p.agents_off = p.vring_off + align4((sh.ring_v * ring_bytes + 3) / 4);
  p.slots_off = p.agents_off + (tier == kTierS ? 4 * sh.res_agents : 0);
  p.queue_off = p.slots_off + (tier != kTierG ? align4(sh.res_vars) : 0);
  p.env_off = p.queue_off + (tier != kTierG ? align4(2 * sh.res_queue) : 0);
  p.words = p.env_off;  // (shared source table disabled: measured slower than registers)
  return p;
}

// Reduce one net to its fixpoint; the whole CTA cooperates.
template <int kTier>
__device__ void run_net(const NetDesc& d, const Shape& sh, const uint16_t* pair, const uint32_t* rules,
                        uint32_t* smem) {
  using T = Traits<kTier>;
  using Ring = typename T::Ring;
  const SmemPlan plan = plan_smem(sh, kTier);
  Ctl* ctl = reinterpret_cast<Ctl*>(smem + plan.ctl_off);
  Round<kTier> c;
  c.d = &d;
  c.ctl = ctl;
  c.aring = reinterpret_cast<Ring*>(smem + plan.aring_off);
  c.vring = reinterpret_cast<Ring*>(smem + plan.vring_off);
  c.amask = sh.ring_a - 1;
  c.vmask = sh.ring_v - 1;
  c.pair = pair;
  c.rules = rules;
  c.n_labels = sh.n_labels;
  void* q0;
  uint32_t qstride;  // queue buffer stride in items
  if constexpr (T::kAgentsSmem) {
    c.agents = reinterpret_cast<uint4*>(smem + plan.agents_off);
    c.cap_agents = sh.res_agents;
  } else {
    c.agents = d.agents;
    c.cap_agents = d.cap_agents;
  }
  if constexpr (T::kSlotsSmem) {
    c.vslot = smem + plan.slots_off;
    c.cap_vars = sh.res_vars;
    q0 = smem + plan.queue_off;
    c.cap_queue = sh.res_queue;
  } else {
    c.vslot = d.vslot;
    c.cap_vars = d.cap_vars;
    q0 = d.queue;
    c.cap_queue = d.cap_queue;
  }
  if constexpr (T::kPacked) c.cap_agents = min(c.cap_agents, 65535u);
  qstride = c.cap_queue;
  // ---- init: private copy of the input agents, empty slots, zero counters
  const bool fits = d.n_in_agents <= c.cap_agents && d.n_in_vars <= c.cap_vars;
  for (uint32_t i = threadIdx.x; i < c.cap_vars; i += blockDim.x) c.vslot[i] = kNone;
  if (fits)
    for (uint32_t i = threadIdx.x; i < d.n_in_agents; i += blockDim.x) c.agents[i] = d.in_agents[i];
  {
    uint32_t* w = reinterpret_cast<uint32_t*>(ctl);
    for (uint32_t i = threadIdx.x; i < sizeof(Ctl) / 4; i += blockDim.x) w[i] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ctl->agent_bump = d.n_in_agents;
    ctl->var_bump = d.n_in_vars;
    ctl->hdr.n = d.n_in_eqs;
    ctl->t_prev = globaltimer();
    ctl->rounds = 1;
    if (!fits) {
      ctl->err_code = INET_ERR_ARENA;
      ctl->hdr.stop = 1;
    } else if (d.n_in_eqs == 0) {  // one no-op loop (engine.py:222-223)
      ctl->hdr.stop = 1;
      if (d.stats && d.cap_rounds) d.stats[0] = make_uint4(0, 0, 0, 0);
    } else if (sh.max_rounds == 0) {  // loop 1 > max_loops (engine.py:205-207)
      ctl->err_code = INET_ERR_LOOP_CAP;
      ctl->hdr.stop = 1;
    }
  }
  __syncthreads();
  c.failed = false;
  c.cur = &ctl->ctr;
  c.env = smem + plan.env_off + threadIdx.x;
  if constexpr (T::kEnvSmem) c.env[(kEnvSize - 1) * blockDim.x] = kNone;  // (disabled tier option)
#ifdef INET_TIMING
  for (int i = 0; i < 8; ++i) c.tm[i] = 0;
  c.tlast = clock64();
#endif
  const uint32_t n_warps = (blockDim.x + 31u) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  for (uint32_t r = 1;; ++r) {
    const Header h = ctl->hdr;
    if (h.stop) break;
    const uint32_t n = h.n;
    c.lo_a = h.lo_a;
    c.hi_a = h.hi_a;
    c.lo_v = h.lo_v;
    c.hi_v = h.hi_v;
    c.ints = c.comms = 0;
    c.parked = 0;
    if (r == 1) {
      // the input equations, in any class (communication_phase's first pass)
      c.out = T::kPacked ? static_cast<void*>(static_cast<uint32_t*>(q0) + qstride)
                         : static_cast<void*>(static_cast<uint2*>(q0) + qstride);
      for (uint32_t i = threadIdx.x; i < n && !c.failed; i += blockDim.x) {
        const uint2 eq = d.in_eqs[i];
        if (((eq.x | eq.y) & kVar) == 0)
          interact(c, eq.x, eq.y);
        else
          link(c, eq.x, eq.y);
      }
    } else if constexpr (T::kPacked) {
      const uint32_t* in = static_cast<const uint32_t*>(q0) + ((r - 1) & 1u) * qstride;
      c.out = static_cast<uint32_t*>(q0) + (r & 1u) * qstride;
      for (uint32_t i = threadIdx.x; i < n && !c.failed; i += blockDim.x) {
        const uint32_t w = in[i];
        interact(c, w >> 16, w & 0xFFFFu);
      }
    } else {
      const uint2* in = static_cast<const uint2*>(q0) + ((r - 1) & 1u) * qstride;
      c.out = static_cast<uint2*>(q0) + (r & 1u) * qstride;
      for (uint32_t i = threadIdx.x; i < n && !c.failed; i += blockDim.x) {
        const uint2 eq = in[i];
        interact(c, eq.x, eq.y);
      }
    }
    INET_TMARK(c, 5);
    const uint32_t wi = __reduce_add_sync(0xFFFFFFFFu, c.ints);
    const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, c.comms);
    const int32_t wp = __reduce_add_sync(0xFFFFFFFFu, c.parked);
    __syncwarp();
    uint32_t last = 0;
    if (lane == 0) {
      if (wi) atomicAdd(&c.cur->ints, wi);
      if (wc) atomicAdd(&c.cur->comms, wc);
      if (wp) atomicAdd(&c.cur->parked, wp);
#ifndef INET_NO_FENCE
      __threadfence_block();
#endif
      last = atomicAdd(&ctl->done_warps, 1u) == n_warps - 1;
    }
    if (last) {
      // every other warp has finished round r: close it and open round r+1
#ifndef INET_NO_FENCE
      __threadfence_block();
#endif
      RoundCtr k;
      {
        const volatile uint32_t* src = reinterpret_cast<const volatile uint32_t*>(&ctl->ctr);
        uint32_t* dst = reinterpret_cast<uint32_t*>(&k);
#pragma unroll
        for (int i = 0; i < static_cast<int>(sizeof(RoundCtr) / 4); ++i) dst[i] = src[i];
      }
      Header nh;
      nh.pad[0] = nh.pad[1] = 0;
      // frees of round r were kept while they fit the ring (against its old window)
      const uint32_t wa = min(k.afree, sh.ring_a - (h.hi_a - h.lo_a));
      const uint32_t wv = min(k.vfree, sh.ring_v - (h.hi_v - h.lo_v));
      nh.lo_a = h.lo_a + min(k.atake, h.hi_a - h.lo_a);
      nh.hi_a = h.hi_a + wa;
      nh.lo_v = h.lo_v + min(k.vtake, h.hi_v - h.lo_v);
      nh.hi_v = h.hi_v + wv;
      nh.n = k.qcount;
      nh.stop = 0;
      const int32_t parked = ctl->parked_total + k.parked;
      ctl->parked_total = parked;
      ctl->tot_i += k.ints;
      ctl->tot_c += k.comms;
#ifdef INET_NO_TIMER
      const unsigned long long now = 0;
#else
      const unsigned long long now = globaltimer();
#endif
      if (d.stats && r - 1 < d.cap_rounds)
        d.stats[r - 1] = make_uint4(k.ints, k.comms, k.qcount + static_cast<uint32_t>(parked),
                                    static_cast<uint32_t>(now - ctl->t_prev));
      ctl->t_prev = now;
      ctl->rounds = r + 1;
      if (k.err) {
        nh.stop = 1;
      } else if (k.qcount == 0) {
        // the trailing no-op loop the reference records (engine.py:222-223)
        nh.stop = 1;
        if (d.stats && r < d.cap_rounds) d.stats[r] = make_uint4(0, 0, static_cast<uint32_t>(parked), 0);
      } else if (r + 1 > sh.max_rounds) {  // engine.py:205-207
        nh.stop = 1;
        atomicCAS(&ctl->err_code, 0u, static_cast<uint32_t>(INET_ERR_LOOP_CAP));
      }
      ctl->ctr = RoundCtr{};
      ctl->hdr = nh;
      ctl->done_warps = 0;
    }
    INET_TMARK(c, 6);
    __syncthreads();
    INET_TMARK(c, 7);
  }
#ifdef INET_TIMING
  if (d.rule_hist)
    for (int i = 0; i < 8; ++i)
      atomicAdd(reinterpret_cast<unsigned long long*>(d.rule_hist) + 32 + i, static_cast<unsigned long long>(c.tm[i]));
#endif
  __syncthreads();
  // ---- results: residual parked equations in variable-id order, arena copy
  const uint32_t hw = min(ctl->var_bump, c.cap_vars);
  uint32_t base = 0;
  for (uint32_t c0 = 0; c0 < hw; c0 += blockDim.x) {
    const uint32_t x = c0 + threadIdx.x;
    const uint32_t v = x < hw ? c.vslot[x] : kNone;
    uint32_t off;
    const uint32_t tot = block_scan_flag(v != kNone, ctl->scratch, &off);
    if (v != kNone && base + off < d.cap_vars) d.residual[base + off] = make_uint2(kVar | x, v);
    base += tot;
  }
  const uint32_t ahw = min(ctl->agent_bump, c.cap_agents);
  if constexpr (T::kAgentsSmem) {
    const uint32_t n_copy = min(ahw, d.cap_agents);
    for (uint32_t i = threadIdx.x; i < n_copy; i += blockDim.x) d.agents[i] = c.agents[i];
  }
  if (threadIdx.x == 0) {
    NetCtl* g = d.ctl;
    g->agent_bump = ahw;
    g->var_bump = hw;
    g->err = ctl->err_code;
    g->err_a = ctl->err_a;
    g->err_b = ctl->err_b;
    g->rounds = ctl->rounds;
    g->interactions = ctl->tot_i;
    g->communications = ctl->tot_c;
    g->n_residual = base;
    g->parked_total = static_cast<uint32_t>(ctl->parked_total);
    if ((ahw > d.cap_agents || hw > d.cap_vars) && g->err == 0) g->err = INET_ERR_ARENA;
  }
  __syncthreads();
}

// Kernel body shared by the prebuilt kernels (engine.cu) and the rule-set
// specialised ones (jit.cpp): load the rule table into shared memory, then
// reduce the CTA's nets one after the other.
template <int kBlock, int kTier>
__device__ __forceinline__ void reduce_body(const NetDesc* __restrict__ nets, uint32_t n_nets,
                                            const uint32_t* __restrict__ blob, const Shape& sh, uint32_t* smem,
                                            NetDesc& sd) {
  for (uint32_t i = threadIdx.x; i < sh.rule_words; i += kBlock) smem[i] = blob[4 + i];
  const uint32_t pair_words = (sh.n_labels * sh.n_labels + 1) / 2;
  const uint16_t* pair = reinterpret_cast<const uint16_t*>(smem);
  const uint32_t* rules = smem + pair_words;
  for (uint32_t net = blockIdx.x; net < n_nets; net += gridDim.x) {
    __syncthreads();
    if (threadIdx.x == 0) sd = nets[net];
    __syncthreads();
    run_net<kTier>(sd, sh, pair, rules, smem);
  }
}

}  // namespace inetdev
