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
// Memory: agents are 16-byte records {label, port0..2}. The two agents of an
// active pair are dead after the rewrite; their slots are reused in place for
// the first two right-hand-side agents, others come from a round-phased free
// ring, then from a bump pointer. Variable ids are recycled the same way once
// both occurrences have met.
#pragma once
#include <cstdint>

#include "../../include/inet_b200.h"

namespace inetdev {

constexpr uint32_t kVar = INET_VAR_BIT;
constexpr uint32_t kNone = INET_NONE;
constexpr int kEnvFresh = 6;
constexpr int kEnvNew = 14;
constexpr int kEnvNone = 22;
constexpr int kEnvSize = 24;
constexpr int kRuleWords = 16;

// Counters of one round; three rotate so that round r writes ctr[r%3] while
// every thread reads the finished ctr[(r-1)%3] and thread 0 clears ctr[(r+1)%3].
struct RoundCtr {
  uint32_t qcount;  // active pairs queued for the next round
  uint32_t atake;   // agent ring entries taken
  uint32_t afree;   // agents freed into the ring
  uint32_t vtake;
  uint32_t vfree;
  uint32_t ints;
  uint32_t comms;
  int32_t parked;   // delta of parked equations
  uint32_t err;     // any failure in this round (read by all threads next round)
  uint32_t pad[7];
};

struct NetCtl {
  RoundCtr ctr[3];
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

// Per-net device view; all arrays are private to the net.
struct NetDesc {
  uint4* agents;       // cap_agents
  uint32_t* vslot;     // cap_vars, kNone = no parked side
  uint32_t* aring;     // amask+1 >= cap_agents
  uint32_t* vring;     // vmask+1 >= cap_vars
  uint2* queue;        // 2 * cap_queue (double buffer)
  uint4* stats;        // cap_rounds rows {ints, comms, live, ns} or null
  uint2* residual;     // cap_vars
  NetCtl* ctl;
  uint32_t* rule_hist;  // interactions per rule (accounting runs) or null
  uint32_t cap_agents, cap_vars, cap_queue, cap_rounds;
  uint32_t amask, vmask;
  // initial contents (device copies of the caller's flat arrays)
  const uint4* in_agents;
  const uint2* in_eqs;
  uint32_t n_in_agents, n_in_eqs, n_in_vars, pad;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t vload(const uint32_t* p) { return *reinterpret_cast<const volatile uint32_t*>(p); }

// Thread-private view of the running round.
struct Round {
  const NetDesc* d;
  uint4* agents;
  uint32_t* vslot;
  RoundCtr* cur;
  uint2* out;
  const uint16_t* pair;
  const uint32_t* rules;
  uint32_t n_labels;
  uint32_t lo_a, hi_a, lo_v, hi_v;  // ring windows available this round
  uint32_t ints, comms;
  int32_t parked;
  bool failed;
};

__device__ __forceinline__ void fail(Round& c, uint32_t code, uint32_t a = 0, uint32_t b = 0) {
  c.failed = true;
  c.cur->err = 1u;
  if (atomicCAS(&c.d->ctl->err, 0u, code) == 0u) {
    c.d->ctl->err_a = a;
    c.d->ctl->err_b = b;
  }
}

__device__ __forceinline__ bool alloc_vars(Round& c, uint32_t nf, uint32_t* out) {
  if (nf == 0) return true;
  const uint32_t t = atomicAdd(&c.cur->vtake, nf);
  const uint32_t avail = c.hi_v - c.lo_v;
  uint32_t got = 0;
  if (t < avail) got = min(avail - t, nf);
  for (uint32_t j = 0; j < got; ++j) out[j] = kVar | c.d->vring[(c.lo_v + t + j) & c.d->vmask];
  if (got < nf) {
    const uint32_t need = nf - got;
    const uint32_t b = atomicAdd(&c.d->ctl->var_bump, need);
    if (b + need > c.d->cap_vars) {
      fail(c, INET_ERR_ARENA, 1);
      return false;
    }
    for (uint32_t j = 0; j < need; ++j) out[got + j] = kVar | (b + j);
  }
  return true;
}

__device__ __forceinline__ bool alloc_agents(Round& c, uint32_t n, uint32_t* out) {
  const uint32_t t = atomicAdd(&c.cur->atake, n);
  const uint32_t avail = c.hi_a - c.lo_a;
  uint32_t got = 0;
  if (t < avail) got = min(avail - t, n);
  for (uint32_t j = 0; j < got; ++j) out[j] = c.d->aring[(c.lo_a + t + j) & c.d->amask];
  if (got < n) {
    const uint32_t need = n - got;
    const uint32_t b = atomicAdd(&c.d->ctl->agent_bump, need);
    if (b + need > c.d->cap_agents) {
      fail(c, INET_ERR_ARENA, 0);
      return false;
    }
    for (uint32_t j = 0; j < need; ++j) out[got + j] = b + j;
  }
  return true;
}

__device__ __forceinline__ void free_agent(Round& c, uint32_t a) {
  const uint32_t f = atomicAdd(&c.cur->afree, 1u);
  c.d->aring[(c.hi_a + f) & c.d->amask] = a;
}

__device__ __forceinline__ void free_var(Round& c, uint32_t x) {
  const uint32_t f = atomicAdd(&c.cur->vfree, 1u);
  c.d->vring[(c.hi_v + f) & c.d->vmask] = x;
}

__device__ __forceinline__ void push_active(Round& c, uint32_t l, uint32_t r) {
  const uint32_t p = atomicAdd(&c.cur->qcount, 1u);
  if (p >= c.d->cap_queue) {
    fail(c, INET_ERR_ARENA, 2);
    return;
  }
  c.out[p] = make_uint2(l, r);
}

// Link one equation: park it on its variable or merge with the parked
// partner, repeating on the merged equation until it is active or parked.
__device__ __forceinline__ void link(Round& c, uint32_t l, uint32_t r) {
  while (true) {
    const bool lv = (l & kVar) != 0, rv = (r & kVar) != 0;
    if (!lv && !rv) {
      push_active(c, l, r);
      return;
    }
    uint32_t key, val;
    if (lv && rv) {
      key = l < r ? l : r;  // smaller id is the key (engine.py:150-153)
      val = l < r ? r : l;
    } else if (lv) {
      key = l;
      val = r;
    } else {
      key = r;
      val = l;
    }
    const uint32_t x = key & ~kVar;
    const uint32_t old = atomicExch(&c.vslot[x], val);
    if (old == kNone) {
      c.parked += 1;
      return;
    }
    // second occurrence: {x = old, x = val} -> old = val; x is dead
    c.vslot[x] = kNone;
    c.comms += 1;
    c.parked -= 1;
    free_var(c, x);
    l = old;
    r = val;
  }
}

// Rewrite one active pair (find_rule + instantiate, core.py:281-312).
__device__ __forceinline__ void interact(Round& c, uint32_t l, uint32_t r) {
  uint4 A = c.agents[l];
  uint4 B = c.agents[r];
  const uint32_t t = c.pair[A.x * c.n_labels + B.x];
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
  const uint32_t* R = c.rules + (t >> 1) * kRuleWords;
  const uint32_t hdr = R[0];
  const uint32_t nn = hdr & 0xFFu, ne = (hdr >> 8) & 0xFFu, nf = (hdr >> 16) & 0xFFu;
  uint32_t env[kEnvSize];
  env[0] = A.y;
  env[1] = A.z;
  env[2] = A.w;
  env[3] = B.y;
  env[4] = B.z;
  env[5] = B.w;
  env[kEnvNone] = kNone;
  if (!alloc_vars(c, nf, env + kEnvFresh)) return;
  env[kEnvNew] = l;
  env[kEnvNew + 1] = r;
  if (nn > 2 && !alloc_agents(c, nn - 2, env + kEnvNew + 2)) return;
  for (uint32_t m = 0; m < nn; ++m) {
    const uint32_t w = R[1 + m];
    c.agents[env[kEnvNew + m]] =
        make_uint4(w & 0xFFu, env[(w >> 8) & 0xFFu], env[(w >> 16) & 0xFFu], env[w >> 24]);
  }
  if (nn < 2) free_agent(c, r);
  if (nn < 1) free_agent(c, l);
  for (uint32_t e = 0; e < ne; ++e) {
    const uint32_t h = (R[9 + (e >> 1)] >> ((e & 1u) * 16u)) & 0xFFFFu;
    link(c, env[h & 0xFFu], env[h >> 8]);
  }
  c.ints += 1;
}

// Copy a net's input into its private arrays and reset its counters.
__device__ void init_net(const NetDesc& d) {
  for (uint32_t i = threadIdx.x; i < d.cap_vars; i += blockDim.x) d.vslot[i] = kNone;
  for (uint32_t i = threadIdx.x; i < d.n_in_agents; i += blockDim.x) d.agents[i] = d.in_agents[i];
  for (uint32_t i = threadIdx.x; i < d.n_in_eqs; i += blockDim.x) d.queue[i] = d.in_eqs[i];
  uint32_t* ctl = reinterpret_cast<uint32_t*>(d.ctl);
  for (uint32_t i = threadIdx.x; i < sizeof(NetCtl) / 4; i += blockDim.x) ctl[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    d.ctl->ctr[0].qcount = d.n_in_eqs;
    d.ctl->agent_bump = d.n_in_agents;
    d.ctl->var_bump = d.n_in_vars;
  }
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

// Reduce one net to its fixpoint; the whole CTA cooperates.
__device__ void run_net(const NetDesc& d, const uint16_t* pair, const uint32_t* rules, uint32_t n_labels,
                        uint32_t max_rounds, uint32_t* scratch) {
  init_net(d);
  __syncthreads();
  NetCtl* ctl = d.ctl;
  Round c;
  c.d = &d;
  c.agents = d.agents;
  c.vslot = d.vslot;
  c.pair = pair;
  c.rules = rules;
  c.n_labels = n_labels;
  c.lo_a = c.hi_a = c.lo_v = c.hi_v = 0;
  c.failed = false;
  // thread-0 bookkeeping
  unsigned long long t_prev = 0, tot_i = 0, tot_c = 0;
  int32_t parked_total = 0;
  uint32_t r = 1;
  for (;; ++r) {
    const RoundCtr* prev = &ctl->ctr[(r - 1) % 3];
    const uint32_t n = vload(&prev->qcount);
    const uint32_t p_atake = vload(&prev->atake), p_afree = vload(&prev->afree);
    const uint32_t p_vtake = vload(&prev->vtake), p_vfree = vload(&prev->vfree);
    c.lo_a += min(p_atake, c.hi_a - c.lo_a);
    c.hi_a += p_afree;
    c.lo_v += min(p_vtake, c.hi_v - c.lo_v);
    c.hi_v += p_vfree;
    // errors of round r-1 are read from its (now frozen) counters so that
    // every thread takes the same exit at the same round
    const uint32_t err = vload(&prev->err);
    if (threadIdx.x == 0) {
      const unsigned long long now = globaltimer();
      if (r > 1) {
        const uint32_t pi = vload(&prev->ints), pc = vload(&prev->comms);
        parked_total += static_cast<int32_t>(vload(reinterpret_cast<const uint32_t*>(&prev->parked)));
        tot_i += pi;
        tot_c += pc;
        if (d.stats && r - 2 < d.cap_rounds)
          d.stats[r - 2] = make_uint4(pi, pc, n + static_cast<uint32_t>(parked_total),
                                      static_cast<uint32_t>(now - t_prev));
      }
      t_prev = now;
      RoundCtr* nxt = &ctl->ctr[(r + 1) % 3];
      *nxt = RoundCtr{};
    }
    if (err) break;
    if (r > max_rounds) {  // engine.py:205-207
      if (threadIdx.x == 0) atomicCAS(&ctl->err, 0u, static_cast<uint32_t>(INET_ERR_LOOP_CAP));
      break;
    }
    if (n == 0) {
      // the trailing no-op loop the reference records (engine.py:222-223)
      if (threadIdx.x == 0 && d.stats && r - 1 < d.cap_rounds)
        d.stats[r - 1] = make_uint4(0, 0, static_cast<uint32_t>(parked_total), 0);
      break;
    }
    c.cur = &ctl->ctr[r % 3];
    const uint2* in = d.queue + ((r - 1) & 1u) * d.cap_queue;
    c.out = d.queue + (r & 1u) * d.cap_queue;
    c.ints = c.comms = 0;
    c.parked = 0;
    for (uint32_t i = threadIdx.x; i < n && !c.failed; i += blockDim.x) {
      const uint2 eq = in[i];
      if (((eq.x | eq.y) & kVar) == 0)
        interact(c, eq.x, eq.y);
      else
        link(c, eq.x, eq.y);  // round 1 only: input equations that are not active
    }
    const uint32_t wi = __reduce_add_sync(0xFFFFFFFFu, c.ints);
    const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, c.comms);
    const int32_t wp = __reduce_add_sync(0xFFFFFFFFu, c.parked);
    if ((threadIdx.x & 31u) == 0) {
      if (wi) atomicAdd(&c.cur->ints, wi);
      if (wc) atomicAdd(&c.cur->comms, wc);
      if (wp) atomicAdd(&c.cur->parked, wp);
    }
    __syncthreads();
  }
  // residual parked equations, in variable-id order
  __syncthreads();
  const uint32_t hw = min(vload(&ctl->var_bump), d.cap_vars);
  uint32_t base = 0;
  for (uint32_t c0 = 0; c0 < hw; c0 += blockDim.x) {
    const uint32_t x = c0 + threadIdx.x;
    const uint32_t v = x < hw ? d.vslot[x] : kNone;
    uint32_t off;
    const uint32_t tot = block_scan_flag(v != kNone, scratch, &off);
    if (v != kNone) d.residual[base + off] = make_uint2(kVar | x, v);
    base += tot;
  }
  if (threadIdx.x == 0) {
    ctl->rounds = r;
    ctl->interactions = tot_i;
    ctl->communications = tot_c;
    ctl->n_residual = base;
    ctl->parked_total = static_cast<uint32_t>(parked_total);
  }
}

}  // namespace inetdev
