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

// Reference loop mode code (deferred equations). The rule-set kernels are
// compiled with and without it: nets whose merges only ever form active pairs
// (all Ackermann nets) run the smaller kernel and get the same rounds.
// Per-rule interaction counts (accounting runs): the rule-set kernels are
// built with or without them (INET_COUNT_RULES 0/1); the prebuilt kernels
// check at run time.
#ifndef INET_COUNT_RULES
#define INET_COUNT_RULES 1
#endif
#ifndef INET_EXACT_CODE
#define INET_EXACT_CODE 1
#endif
// Reference-ordered var = var keys (single-CTA tiers): every variable carries
// a 64-bit stamp {loop of creation, creating interaction, bound-variable
// index}; the rule-set kernels are built with or without the code.
#ifndef INET_STAMPS
#define INET_STAMPS 1
#endif

namespace inetdev {

constexpr uint32_t kVar = INET_VAR_BIT;
constexpr uint32_t kNone = INET_NONE;
constexpr int kEnvFresh = 6;
constexpr int kEnvNew = 14;
constexpr int kEnvNone = 22;
constexpr int kEnvSize = 23;  // sources 0..22 (22 = none)
constexpr int kRuleWords = 16;
constexpr int kFastEq = 4;  // rhs equations linked with overlapped exchanges
constexpr uint32_t kMbox = 64;  // tier C: ids one CTA can mail to one owner per round (then direct frees)

enum : int { kTierS = 0, kTierM = 1, kTierG = 2, kTierC = 3, kTierX = 4 };

template <int kTier>
struct Traits {
  using Ring = uint16_t;
  static constexpr bool kCompact = kTier == kTierS;   // 8-byte agents with 16-bit refs in shared memory
  static constexpr bool kEnvSmem = false;           // per-thread source table in shared memory
  static constexpr bool kEnvLocal = kTier == kTierS;  // per-thread source table in local memory (L1)
  static constexpr bool kAgentsSmem = kTier == kTierS;
  static constexpr bool kSlotsSmem = true;
  static constexpr bool kPacked = true;
};
template <>
struct Traits<kTierG> {
  using Ring = uint32_t;
  static constexpr bool kCompact = false;
  static constexpr bool kEnvSmem = false;
  static constexpr bool kEnvLocal = false;
  static constexpr bool kAgentsSmem = false;
  static constexpr bool kSlotsSmem = false;
  static constexpr bool kPacked = false;
};
// Tier C: one net on a thread-block cluster; agents, slots and queues in
// global memory (L2-resident), rings and round counters per CTA.
template <>
struct Traits<kTierC> : Traits<kTierG> {};
// Tier X: one net on the whole GPU (one CTA per SM slot, cooperative launch);
// everything, counters included, in global memory (L2-resident).
template <>
struct Traits<kTierX> : Traits<kTierG> {};

// Counters of the running round, bumped by every thread while it works.
// (Tier C reads {qcount, ints, comms, parked} of every CTA with one 16-byte
// distributed-shared-memory load, so they lead.)
constexpr uint32_t kErrBit = 0x80000000u;  // in qcount: a failure in this round
constexpr uint32_t kAgentCache = 4096;     // tier M: shared-memory agent-record cache entries
struct RoundCtr {
  uint32_t qcount;  // active pairs queued for the next round (| kErrBit on failure)
  uint32_t ints;
  uint32_t comms;
  int32_t parked;   // delta of parked equations
  uint32_t atake;   // agent ring entries taken
  uint32_t afree;   // agents offered to the ring
  uint32_t vtake;
  uint32_t vfree;
  uint32_t dcount;  // merged equations deferred to the next round (reference loop mode)
  uint32_t vh;      // a merge left a var-headed equation (kernels without INET_EXACT_CODE)
  uint32_t pad[2];
};

// Parameters of the next round, written by the last warp to finish a round
// (before the round's barrier) and read by every thread after it.
struct Header {
  uint32_t n;       // active pairs in the queue
  uint32_t stop;    // leave the loop
  uint32_t lo_a, hi_a, lo_v, hi_v;  // ring windows allocatable in this round
  uint32_t nd;      // deferred equations to link first (reference loop mode)
  uint32_t pad;
};

// Shared-memory control block of the net a CTA is reducing.
struct Ctl {
  RoundCtr ctr3[3];  // tiers S/M/G: round r counts into set r % 3 (cleared two rounds ahead)
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
  uint32_t fpos_a, fpos_v;  // tier C: ring positions handed to freers (monotonic)
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
  uint32_t pad[4];  // pad[0]: effective SM clock (MHz) over the reduction
};

// Effective SM clock between two (clock64, globaltimer) samples, in MHz.
__device__ __forceinline__ uint32_t clock_mhz(long long c0, unsigned long long g0) {
  const long long dc = clock64() - c0;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const unsigned long long dg = t - g0;
  return dg ? static_cast<uint32_t>(static_cast<unsigned long long>(dc) * 1000ull / dg) : 0u;
}

// Tier X: the control block of a net reduced by the whole grid.
struct GridState {
  Ctl ctl;
  RoundCtr ctr3[3];
  uint32_t bar_count, bar_gen;
  uint32_t fin_lo_a, fin_hi_a;  // the agent ring window at the end (its entries are the dead agents)
  uint32_t blk_res[1];  // per-block residual counts follow (gridDim.x words)
};

// Per-net device view of its private global arrays. (Pointers first, then
// 64-bit, then 32-bit fields: no padding — every CTA keeps a copy in shared
// memory, and tier S packs 10 CTAs per SM.)
struct NetDesc {
  uint4* agents;       // cap_agents (tiers M/G arena; tier S result copy)
  uint32_t* vslot;     // cap_vars (tier G)
  uint2* queue;        // 2 * cap_queue (tier G)
  uint4* stats;        // cap_rounds rows {ints, comms, live, ns} or null
  uint2* residual;     // cap_vars
  NetCtl* ctl;
  uint32_t* rule_hist; // interactions per rule (accounting runs) or null
  // initial contents (device copies of the caller's flat arrays)
  const uint4* in_agents;
  const uint2* in_eqs;
  // reference loop mode: equations a merge left var-headed wait for the next
  // round's communication, [2 parities][cap_def] (tier C: [2][G][cap_def / G])
  uint2* deferred;
  // tier X: global free rings and the net's global control block
  uint32_t* g_aring;
  uint32_t* g_vring;
  struct GridState* gs;
  // device-side finalize (tier S): the net's interface; dev_final enables it
  const uint32_t* in_iface;
  // reference-ordered var = var keys: one stamp per variable id (null: off)
  unsigned long long* stamps;
  // tier C resuming a net that tier M handed over (its arena, slot table and
  // pending equations are the inputs): the totals already done
  unsigned long long base_ints, base_comms;
  uint32_t cap_agents, cap_vars, cap_queue, cap_rounds;
  uint32_t n_in_agents, n_in_eqs, n_in_vars;
  uint32_t cap_def;
  uint32_t resume, round_base;  // (tier C resume: the rounds already done)
  int32_t base_parked;
  uint32_t n_iface, dev_final;  // dev_final: bit 0 device-side finalize (tier S), bit 1 kInputActive
};
constexpr uint32_t kInputActive = 2u;  // NetDesc::dev_final: an input equation is an active pair

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
  uint32_t exact;                 // 1: reference loop mode (merged var-headed equations wait a round)
  uint32_t promote_ints;          // tier M: give the net up to the cluster tier past this many interactions
  uint32_t detect_vh;             // stop with kNeedExact at the first var-headed merge (exact requested,
                                  // kernel without INET_EXACT_CODE)
  uint32_t max_fresh;             // tier R: RuleSet.max_fresh (the reference's fresh-id block per equation)
  uint32_t validate;              // tier R: name discipline after every phase (EngineConfig.validate_phases)
  uint32_t cap_list, cap_out;     // tier R: equations per list / per output stream
  uint8_t* rbuf;                  // tier R: net i's arrays start at rbuf + i * rbuf_stride (ordered.cuh)
  unsigned long long rbuf_stride;
};

// Internal statuses (never returned to callers): a single-CTA run that outgrew
// it; a run without reference-loop code that met a var-headed merge.
constexpr uint32_t kPromote = 0x100u;
constexpr uint32_t kNeedExact = 0x101u;

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Per-round rows (EvalResult.loops): the rule-set kernels are compiled with or
// without them (jit.cpp kernel_source); the prebuilt kernels decide at run time.
#ifndef INET_ROWS
#define INET_ROWS 1
#endif

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

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t lane, uint32_t& total) {
  uint32_t inc = v;
#pragma unroll
  for (uint32_t o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += t;
  }
  total = __shfl_sync(0xFFFFFFFFu, inc, 31);
  return inc - v;
}

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
  uint4* acache;  // tier M: cache of agent records, [kAgentCache]
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
  uint32_t a_base, v_base, stride;  // tier C: bump sequence s -> id base + stride * s
  uint32_t rank, gshift;            // tier C: this CTA's rank in the cluster, log2 G
  uint2* dout;                      // reference loop mode: this round's deferred equations (null: fixpoint)
  uint32_t cap_def;
  uint32_t* outc;                   // tier C: ids mailed this round per owner: agents [0,16), vars [16,32)
  uint32_t* mbox_a;                 // tier C: mailboxes of this round, [src][kMbox] (owner's layout)
  uint32_t* mbox_v;
  uint2* inq;                       // tier C: next round's input queues, [producer][qj] (consumer's layout)
  uint32_t qj;
  uint32_t ints, comms;
  int32_t parked;
  bool failed;
#if INET_STAMPS
  unsigned long long* stamps;       // reference-ordered var = var keys (null: off)
  uint32_t round, cid;              // the running round; the interaction being rewritten (its A agent)
#endif
#ifdef INET_TIMING
  long long tm[8];
  long long tlast;
#endif
#ifdef INET_TRACE
  long long tr[8];
#endif
};

#ifdef INET_TRACE
__device__ unsigned int inet_trace_count;
#ifndef INET_TRACE_R0
#define INET_TRACE_R0 2
#endif
#define INET_TR(c, k) ((c).tr[k] = clock64())
#else
#define INET_TR(c, k) \
  do {                \
  } while (0)
#endif

template <int kTier>
__device__ __forceinline__ void fail(Round<kTier>& c, uint32_t code, uint32_t a = 0, uint32_t b = 0) {
  c.failed = true;
  atomicOr(&c.cur->qcount, kErrBit);
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

// Id of the s-th bump allocation. Tier C interleaves the CTAs of a cluster
// (CTA k owns base + k + G*s), so ids stay dense without a shared counter.
template <int kTier>
__device__ __forceinline__ uint32_t bump_agent(const Round<kTier>& c, uint32_t s) {
  if constexpr (kTier == kTierC) return c.a_base + c.stride * s;
  else return s;
}
template <int kTier>
__device__ __forceinline__ uint32_t bump_var(const Round<kTier>& c, uint32_t s) {
  if constexpr (kTier == kTierC) return c.v_base + c.stride * s;
  else return s;
}


// ---- thread-block-cluster primitives (tier C) ------------------------------
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, uint32_t rank) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  return ra;
}
__device__ __forceinline__ uint32_t dsmem_atom_add(const void* p, uint32_t rank, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared::cluster.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(dsmem_addr(p, rank)), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void dsmem_red_add(const void* p, uint32_t rank, uint32_t v) {
  asm volatile("red.shared::cluster.add.u32 [%0], %1;" ::"r"(dsmem_addr(p, rank)), "r"(v) : "memory");
}
__device__ __forceinline__ void dsmem_st(const void* p, uint32_t rank, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(dsmem_addr(p, rank)), "r"(v) : "memory");
}
__device__ __forceinline__ void dsmem_st4(const void* p, uint32_t rank, uint4 v) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dsmem_addr(p, rank)), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint32_t dsmem_ld(const void* p, uint32_t rank) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(dsmem_addr(p, rank)) : "memory");
  return v;
}

// Tier C free: an id goes back to the ring of the CTA that owns it
// (owner = id mod G), at a position drawn from the owner's monotonic counter;
// the owner's per-round count makes it allocatable from the next round on.
// A CTA never owns more ids than its ring holds, so nothing is dropped.
template <int kTier>
__device__ __forceinline__ void free_owned(Round<kTier>& c, uint32_t id, uint32_t* fpos, uint32_t* ring, uint32_t mask,
                                           uint32_t* cnt, uint32_t* outc, uint32_t* mbox, uint32_t* slots) {
  const uint32_t k = id & (c.stride - 1);
  if (k == c.rank) {
    if (slots) slots[id >> c.gshift] = kNone;  // a dead variable's slot, cleared by its owner
    const uint32_t pos = atomicAdd(fpos, 1u);
    ring[pos & mask] = id;
    atomicAdd(cnt, 1u);
    return;
  }
  // mail it: a local counter and one remote store; the owner moves its mail
  // into its ring next round (allocatable the round after)
#ifdef INET_NO_MBOX
  const uint32_t p = kMbox;
#else
  const uint32_t p = atomicAdd(&outc[k], 1u);
#endif
  if (p < kMbox) {
    dsmem_st(&mbox[c.rank * kMbox + p], k, id);
    return;
  }
  const uint32_t pos = dsmem_atom_add(fpos, k, 1u);  // mailbox full: straight into the owner's ring
  if (slots) dsmem_st(&slots[id >> c.gshift], k, kNone);
  dsmem_st(&ring[pos & mask], k, id);
  dsmem_red_add(cnt, k, 1u);
}

// ---- agent and variable-slot access -----------------------------------------
// Tiers S/M/G address one array; tier C spreads both over the cluster's shared
// memory (id -> CTA id & (G-1), slot id >> log2 G).
__device__ __forceinline__ uint4 dsmem_ld4(const void* p, uint32_t rank) {
  uint4 v;
  asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(dsmem_addr(p, rank))
               : "memory");
  return v;
}
__device__ __forceinline__ uint2 dsmem_ld2(const void* p, uint32_t rank) {
  uint2 v;
  asm volatile("ld.shared::cluster.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(dsmem_addr(p, rank)) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t dsmem_exch(const void* p, uint32_t rank, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared::cluster.exch.b32 %0, [%1], %2;" : "=r"(old) : "r"(dsmem_addr(p, rank)), "r"(v) : "memory");
  return old;
}

// Tier S keeps agents as 8 bytes {label, p0 | p1, p2} with 16-bit refs
// (its arenas hold < 32768 ids, the top one unused, so a variable is
// 0x8000 | id and 0xFFFF is none), which fits more nets per SM.
// Tier S keeps references inside the kernel in a sign-extended form: variable
// x is 0xFFFF8000 | x (bit 31 still marks a variable, kNone is still all ones,
// agents are plain indices), so the 16-bit halves of the 8-byte agent records
// convert with one sign extension or one byte permute per port. Every
// other tier uses the standard form (INET_VAR_BIT | x). Conversions happen only
// where tier S meets global memory: the input, the residual equations and the
// arena / normal-form copies.
template <int kTier>
__device__ __forceinline__ constexpr uint32_t vtag() {
  return kTier == kTierS ? 0xFFFF8000u : kVar;
}
template <int kTier>
__device__ __forceinline__ uint32_t ref_in(uint32_t r) {  // standard -> internal
  if constexpr (kTier == kTierS) return (r != kNone && (r & kVar)) ? (r | 0xFFFF8000u) : r;
  else return r;
}
template <int kTier>
__device__ __forceinline__ uint32_t ref_out(uint32_t r) {  // internal -> standard
  if constexpr (kTier == kTierS) return (r != kNone && (r & kVar)) ? (kVar | (r & 0x7FFFu)) : r;
  else return r;
}
template <int kTier>
__device__ __forceinline__ uint4 agent_in(const uint4& v) {
  return make_uint4(v.x, ref_in<kTier>(v.y), ref_in<kTier>(v.z), ref_in<kTier>(v.w));
}
template <int kTier>
__device__ __forceinline__ uint4 agent_out(const uint4& v) {
  return make_uint4(v.x, ref_out<kTier>(v.y), ref_out<kTier>(v.z), ref_out<kTier>(v.w));
}
__device__ __forceinline__ uint32_t sext16(uint32_t h) {  // low 16 bits, sign-extended
  return static_cast<uint32_t>(static_cast<int32_t>(h << 16) >> 16);
}
__device__ __forceinline__ uint2 pack_agent_s(const uint4& v) {
  return make_uint2(__byte_perm(v.x, v.y, 0x5410), __byte_perm(v.z, v.w, 0x5410));
}
__device__ __forceinline__ uint4 unpack_agent_s(const uint2& w) {
  return make_uint4(w.x & 0xFFFFu, sext16(w.x >> 16), sext16(w.y), sext16(w.y >> 16));
}

// Tier M keeps its arena in global memory, and a record written in one round
// is read in the next by another thread: past the round barrier that load
// goes to L2 (~700 cycles on a narrow round's critical path,
// profiles/r02al_round_trace.txt). Every store therefore also goes to a
// direct-mapped shared-memory cache of records, tagged in the label word's
// high half (label < 2^16, id < 2^16: tag = id / kAgentCache + 1, 0 = empty);
// a load that finds its tag there does not touch global memory. The global
// arena stays complete (write-through), so the hand-over to a cluster and the
// host finalize read it as before.
template <int kTier>
__device__ __forceinline__ uint4 ld_agent(const Round<kTier>& c, uint32_t a) {
  if constexpr (kTier == kTierC) return dsmem_ld4(c.agents + (a >> c.gshift), a & (c.stride - 1));
  else if constexpr (Traits<kTier>::kCompact) return unpack_agent_s(reinterpret_cast<const uint2*>(c.agents)[a]);
  else if constexpr (kTier == kTierM) {
    const uint4 e = c.acache[a & (kAgentCache - 1u)];
    if ((e.x >> 16) == (a / kAgentCache) + 1u) return make_uint4(e.x & 0xFFFFu, e.y, e.z, e.w);
    return c.agents[a];
  } else return c.agents[a];
}
template <int kTier>
__device__ __forceinline__ void st_agent(const Round<kTier>& c, uint32_t a, const uint4& v) {
  if constexpr (kTier == kTierC) dsmem_st4(c.agents + (a >> c.gshift), a & (c.stride - 1), v);
  else if constexpr (Traits<kTier>::kCompact) reinterpret_cast<uint2*>(c.agents)[a] = pack_agent_s(v);
  else if constexpr (kTier == kTierM) {
    c.agents[a] = v;
    c.acache[a & (kAgentCache - 1u)] = make_uint4(v.x | (((a / kAgentCache) + 1u) << 16), v.y, v.z, v.w);
  } else c.agents[a] = v;
}
template <int kTier>
__device__ __forceinline__ uint32_t exch_slot(const Round<kTier>& c, uint32_t x, uint32_t v) {
  if constexpr (kTier == kTierC) return dsmem_exch(c.vslot + (x >> c.gshift), x & (c.stride - 1), v);
  else return atomicExch(&c.vslot[x], v);
}
template <int kTier>
__device__ __forceinline__ void st_slot(const Round<kTier>& c, uint32_t x, uint32_t v) {
  if constexpr (kTier == kTierC) dsmem_st(c.vslot + (x >> c.gshift), x & (c.stride - 1), v);
  else c.vslot[x] = v;
}

// Ring claims of a round. Tiers S and M count both in one word (agents in the
// low half, variables in the high half: a round takes fewer than 2^16 of
// either), so a rewrite that needs both claims them with one shared-memory
// atomic — same-address atomics serialise per lane, and the counters are the
// batch kernel's busiest shared-memory traffic.
template <int kTier>
constexpr bool kTake2 = kTier == kTierS || kTier == kTierM;
template <int kTier>
__device__ __forceinline__ uint32_t take_vars(Round<kTier>& c, uint32_t n) {
  if constexpr (kTake2<kTier>) return atomicAdd(&c.cur->atake, n << 16) >> 16;
  else return atomicAdd(&c.cur->vtake, n);
}
template <int kTier>
__device__ __forceinline__ uint32_t take_agents(Round<kTier>& c, uint32_t n) {
  if constexpr (kTake2<kTier>) return atomicAdd(&c.cur->atake, n) & 0xFFFFu;
  else return atomicAdd(&c.cur->atake, n);
}

template <int kTier>
__device__ __forceinline__ bool alloc_vars(Round<kTier>& c, uint32_t nf, Claim& k) {
  k.pos = k.got = k.bump = 0;
  if (nf == 0) return true;
  const uint32_t t = take_vars(c, nf);
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
  const uint32_t t = take_agents(c, n);
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

// atomicAdd(p, 1) shared by the converged lanes of the warp: one atomic per
// warp (tier X counters are global and hot).
__device__ __forceinline__ uint32_t agg_add(uint32_t* p) {
  const uint32_t m = __activemask();
  const uint32_t lane = threadIdx.x & 31u, leader = __ffs(m) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(p, static_cast<uint32_t>(__popc(m)));
  base = __shfl_sync(m, base, leader);
  return base + __popc(m & ((1u << lane) - 1u));
}

template <int kTier>
__device__ __forceinline__ void free_agent(Round<kTier>& c, uint32_t a) {
  if constexpr (kTier == kTierC) {
    free_owned(c, a, &c.ctl->fpos_a, reinterpret_cast<uint32_t*>(c.aring), c.amask, &c.cur->afree, c.outc, c.mbox_a,
               static_cast<uint32_t*>(nullptr));
    return;
  }
  const uint32_t f = kTier == kTierX ? agg_add(&c.cur->afree) : atomicAdd(&c.cur->afree, 1u);
  const uint32_t pos = c.hi_a + f;
  if (pos - c.lo_a <= c.amask) c.aring[pos & c.amask] = a;  // else dropped
}

// Tiers S and M count queued pairs in the low half of vfree (freed variables
// in the high half; a round queues and frees fewer than 2^16 of each), so a
// merge that frees its variable and queues the active pair it formed takes
// one shared-memory atomic. qcount then only carries the failure bit.
template <int kTier>
constexpr bool kPush2 = kTier == kTierS || kTier == kTierM;

template <int kTier>
__device__ __forceinline__ void ring_var(Round<kTier>& c, uint32_t x, uint32_t f) {
  const uint32_t pos = c.hi_v + f;
  if (pos - c.lo_v <= c.vmask) c.vring[pos & c.vmask] = x;
}

template <int kTier>
__device__ __forceinline__ void free_var(Round<kTier>& c, uint32_t x) {
  if constexpr (kTier == kTierC) {
    free_owned(c, x, &c.ctl->fpos_v, reinterpret_cast<uint32_t*>(c.vring), c.vmask, &c.cur->vfree, c.outc + 16,
               c.mbox_v, c.vslot);
    return;
  }
  if constexpr (kPush2<kTier>) {
    ring_var(c, x, atomicAdd(&c.cur->vfree, 1u << 16) >> 16);
    return;
  }
  ring_var(c, x, kTier == kTierX ? agg_add(&c.cur->vfree) : atomicAdd(&c.cur->vfree, 1u));
}

__device__ __forceinline__ void dsmem_st2(const void* p, uint32_t rank, uint2 v) {
  asm volatile("st.shared::cluster.v2.u32 [%0], {%1, %2};" ::"r"(dsmem_addr(p, rank)), "r"(v.x), "r"(v.y) : "memory");
}

// Queue an active pair. Tier C deals a CTA's pairs round-robin over the
// cluster (the p-th to CTA (p + rank) mod G, slot p / G) straight into the
// consumer's shared memory, so next round every CTA reads its pairs locally.
template <int kTier>
__device__ __forceinline__ void queue_at(Round<kTier>& c, uint32_t p, uint32_t l, uint32_t r) {  // tiers S/M/G/X
  if (p >= c.cap_queue) {
    fail(c, INET_ERR_ARENA, 2);
    return;
  }
  if constexpr (Traits<kTier>::kPacked)
    static_cast<uint32_t*>(c.out)[p] = (l << 16) | r;  // both < 65536 in tiers S/M
  else
    static_cast<uint2*>(c.out)[p] = make_uint2(l, r);
}

template <int kTier>
__device__ __forceinline__ void push_active(Round<kTier>& c, uint32_t l, uint32_t r) {
  if constexpr (kPush2<kTier>) {
    queue_at(c, atomicAdd(&c.cur->vfree, 1u) & 0xFFFFu, l, r);
    return;
  }
  const uint32_t p = kTier == kTierX ? agg_add(&c.cur->qcount) : atomicAdd(&c.cur->qcount, 1u);
  if constexpr (kTier == kTierC) {
    const uint32_t s = (p & ~kErrBit) >> c.gshift;
    if (s >= c.qj) {
      fail(c, INET_ERR_ARENA, 2);
      return;
    }
    dsmem_st2(&c.inq[c.rank * c.qj + s], (p + c.rank) & (c.stride - 1), make_uint2(l, r));
    return;
  }
  queue_at(c, p, l, r);
}

// Warp-collective push: every lane calls it, lanes with `pu` push (l, r).
template <int kTier>
__device__ __forceinline__ void warp_push(Round<kTier>& c, bool pu, uint32_t l, uint32_t r) {
  if constexpr (kTier == kTierC) {
    if (pu) push_active(c, l, r);
    return;
  }
  const uint32_t m = __ballot_sync(0xFFFFFFFFu, pu);
  if (!m) return;
  const uint32_t lane = threadIdx.x & 31u, leader = __ffs(m) - 1;
  uint32_t base = 0;
  if (lane == leader)
    base = kPush2<kTier> ? atomicAdd(&c.cur->vfree, static_cast<uint32_t>(__popc(m))) & 0xFFFFu
                         : atomicAdd(&c.cur->qcount, static_cast<uint32_t>(__popc(m)));
  base = __shfl_sync(0xFFFFFFFFu, base, leader);
  if (!pu) return;
  const uint32_t p = base + __popc(m & ((1u << lane) - 1u));
  if (p >= c.cap_queue) {
    fail(c, INET_ERR_ARENA, 2);
    return;
  }
  if constexpr (Traits<kTier>::kPacked)
    static_cast<uint32_t*>(c.out)[p] = (l << 16) | r;
  else
    static_cast<uint2*>(c.out)[p] = make_uint2(l, r);
}

// A variable's stamp: {round of creation : 24 | creating interaction : 32 |
// bound-variable index : 8}; input variables {0 | dense id | 0}. The
// reference numbers fresh variables base_L + i * max_fresh + j (engine.py:93,
// 122): by loop, then list position of the creating equation, then j. Stamps
// decide every comparison except two variables made in the same round by
// different interactions, whose order is their creators' list positions —
// that case stops the net with INET_ERR_ORDER and the host reruns it on tier R.
constexpr uint32_t kOrderUndecided = INET_ERR_ORDER;

template <int kTier>
__device__ __forceinline__ void stamp_store(const Round<kTier>& c, uint32_t x, uint32_t j) {
#if INET_STAMPS
  if (c.stamps)
    c.stamps[x & ~vtag<kTier>()] =
        (static_cast<unsigned long long>(c.round) << 40) | (static_cast<unsigned long long>(c.cid) << 8) | j;
#endif
}
// One fence after a rewrite's stamps: ordered before the exchange that may hand
// a fresh variable to another thread this round.
template <int kTier>
__device__ __forceinline__ void stamp_publish(const Round<kTier>& c) {
#if INET_STAMPS
  if (c.stamps) __threadfence_block();
#endif
}

// Key and parked value of a non-active equation: var=var keys on the smaller
// id (engine.py:150-153) — with stamps, the smaller reference id.
template <int kTier>
__device__ __forceinline__ void key_of(Round<kTier>& c, uint32_t l, uint32_t r, uint32_t& key, uint32_t& val) {
  const bool lv = (l & kVar) != 0, rv = (r & kVar) != 0;
  if (lv && rv) {
    bool l_first = l < r;
#if INET_STAMPS
    if (c.stamps) {
      __threadfence_block();  // (after the exchange that delivered a variable made this round)
      const unsigned long long a = c.stamps[l & ~vtag<kTier>()], b = c.stamps[r & ~vtag<kTier>()];
      const unsigned long long la = a >> 40, lb = b >> 40;
      if (la != lb || la == 0 || (a >> 8) == (b >> 8)) {
        l_first = a < b;
      } else {
        fail(c, kOrderUndecided, 0, 0);  // same round, different creators: tier R decides
      }
    }
#endif
    key = l_first ? l : r;
    val = l_first ? r : l;
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
    // x is dead: both occurrences met. Tier C leaves the slot to its owner,
    // which clears it locally when the id comes back to its ring (no remote store).
    if constexpr (kTier != kTierC) st_slot(c, x, kNone);
    c.comms += 1;
    c.parked -= 1;
    const uint32_t l = old, r = val;
    if constexpr (kPush2<kTier>) {
      if (((l | r) & kVar) == 0) {  // free x and queue (l, r): one atomic
        const uint32_t w = atomicAdd(&c.cur->vfree, (1u << 16) | 1u);
        ring_var(c, x, w >> 16);
        queue_at(c, w & 0xFFFFu, l, r);
        return;
      }
      ring_var(c, x, atomicAdd(&c.cur->vfree, 1u << 16) >> 16);
    } else {
      free_var(c, x);
      if (((l | r) & kVar) == 0) {
        push_active(c, l, r);
        return;
      }
    }
#if INET_EXACT_CODE
    if (c.dout) {
      // reference loop mode: the merged equation communicates next round, as
      // it would in the reference's next communication_phase (engine.py:137-166).
      // (Kept minimal — settle is inlined at every equation of every rule; a
      // full buffer is reported when the round closes.)
      c.dout[min(atomicAdd(&c.cur->dcount, 1u), c.cap_def - 1)] = make_uint2(l, r);
      c.parked += 1;  // live until linked
      return;
    }
#else
    c.cur->vh = 1u;  // noted; a run that wants reference loops restarts with the full kernel
#endif
    uint32_t key;
    key_of(c, l, r, key, val);
    x = key & ~vtag<kTier>();
    old = exch_slot(c, x, val);
  }
}

template <int kTier>
__device__ __forceinline__ void link(Round<kTier>& c, uint32_t l, uint32_t r) {
  if (((l | r) & kVar) == 0) {
    push_active(c, l, r);
    return;
  }
  uint32_t key, val;
  key_of(c, l, r, key, val);
  const uint32_t x = key & ~vtag<kTier>();
  settle(c, x, exch_slot(c, x, val), val);
}

#ifdef INET_JIT
// Helpers of the generated rewrites: allocation with compile-time counts into
// registers, and the first half of link() (push or exchange key).
template <uint32_t N, int kTier>
__device__ __forceinline__ bool jit_alloc_vars(Round<kTier>& c, uint32_t (&f)[N]) {
  Claim k;
  if (!alloc_vars(c, N, k)) return false;
#pragma unroll
  for (uint32_t j = 0; j < N; ++j) {
    f[j] = vtag<kTier>() | (j < k.got ? static_cast<uint32_t>(c.vring[(k.pos + j) & c.vmask]) : bump_var(c, k.bump + (j - k.got)));
    stamp_store(c, f[j], j);
  }
  stamp_publish(c);
  return true;
}

template <uint32_t N, int kTier>
__device__ __forceinline__ bool jit_alloc_agents(Round<kTier>& c, uint32_t (&g)[N]) {
  Claim k;
  if (!alloc_agents(c, N, k)) return false;
#pragma unroll
  for (uint32_t j = 0; j < N; ++j)
    g[j] = j < k.got ? static_cast<uint32_t>(c.aring[(k.pos + j) & c.amask]) : bump_agent(c, k.bump + (j - k.got));
  return true;
}

// Runtime counts (n <= N): ids land in f[0..n), the rest are untouched.
template <uint32_t N, int kTier>
__device__ __forceinline__ bool jit_alloc_vars_n(Round<kTier>& c, uint32_t n, uint32_t (&f)[N]) {
  Claim k;
  if (!alloc_vars(c, n, k)) return false;
#pragma unroll
  for (uint32_t j = 0; j < N; ++j)
    if (j < n) {
      f[j] = vtag<kTier>() | (j < k.got ? static_cast<uint32_t>(c.vring[(k.pos + j) & c.vmask]) : bump_var(c, k.bump + (j - k.got)));
      stamp_store(c, f[j], j);
    }
  stamp_publish(c);
  return true;
}

template <uint32_t N, int kTier>
__device__ __forceinline__ bool jit_alloc_agents_n(Round<kTier>& c, uint32_t n, uint32_t (&g)[N]) {
  Claim k;
  if (!alloc_agents(c, n, k)) return false;
#pragma unroll
  for (uint32_t j = 0; j < N; ++j)
    if (j < n)
      g[j] = j < k.got ? static_cast<uint32_t>(c.aring[(k.pos + j) & c.amask]) : bump_agent(c, k.bump + (j - k.got));
  return true;
}

// Warp-collective allocation for the rule-set kernels: every lane asks for nf
// fresh variables and nx extra agents; one lane claims the warp's total on
// each ring (two independent atomics), overflow goes to the bump pointers.
// Returns false on every lane if an arena is exhausted.
template <uint32_t MF, uint32_t MX, int kTier>
__device__ __forceinline__ bool jit_warp_alloc(Round<kTier>& c, uint32_t nf, uint32_t nx, uint32_t (&f)[MF],
                                               uint32_t (&g)[MX]) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t tot_f, tot_x;
  const uint32_t ex_f = warp_excl_scan(nf, lane, tot_f);
  const uint32_t ex_x = warp_excl_scan(nx, lane, tot_x);
  if ((tot_f | tot_x) == 0) return true;
  const uint32_t av_v = c.hi_v - c.lo_v, av_a = c.hi_a - c.lo_a;
  uint32_t tv = 0, ta = 0, bv = 0, ba = 0, ok = 1;
  if (lane == 0) {
    if constexpr (kTake2<kTier>) {
      const uint32_t w = atomicAdd(&c.cur->atake, (tot_f << 16) | tot_x);
      tv = w >> 16;
      ta = w & 0xFFFFu;
    } else {
      if (tot_f) tv = atomicAdd(&c.cur->vtake, tot_f);
      if (tot_x) ta = atomicAdd(&c.cur->atake, tot_x);
    }
    const uint32_t ov = tv + tot_f > av_v ? tv + tot_f - max(tv, av_v) : 0u;
    const uint32_t oa = ta + tot_x > av_a ? ta + tot_x - max(ta, av_a) : 0u;
    if (ov) {
      bv = atomicAdd(&c.ctl->var_bump, ov);
      if (bv + ov > c.cap_vars) {
        fail(c, INET_ERR_ARENA, 1);
        ok = 0;
      }
    }
    if (oa) {
      ba = atomicAdd(&c.ctl->agent_bump, oa);
      if (ba + oa > c.cap_agents) {
        fail(c, INET_ERR_ARENA, 0);
        ok = 0;
      }
    }
  }
  if (!__shfl_sync(0xFFFFFFFFu, ok, 0)) {
    c.failed = true;
    return false;
  }
  tv = __shfl_sync(0xFFFFFFFFu, tv, 0);
  ta = __shfl_sync(0xFFFFFFFFu, ta, 0);
  bv = __shfl_sync(0xFFFFFFFFu, bv, 0);
  ba = __shfl_sync(0xFFFFFFFFu, ba, 0);
  const uint32_t fb_v = max(tv, av_v), fb_a = max(ta, av_a);  // first bumped take index
#pragma unroll
  for (uint32_t j = 0; j < MF; ++j)
    if (j < nf) {
      const uint32_t q = tv + ex_f + j;
      f[j] = vtag<kTier>() | (q < av_v ? static_cast<uint32_t>(c.vring[(c.lo_v + q) & c.vmask]) : bump_var(c, bv + (q - fb_v)));
    }
#pragma unroll
  for (uint32_t j = 0; j < MX; ++j)
    if (j < nx) {
      const uint32_t q = ta + ex_x + j;
      g[j] = q < av_a ? static_cast<uint32_t>(c.aring[(c.lo_a + q) & c.amask]) : bump_agent(c, ba + (q - fb_a));
    }
  return true;
}

// Rule-set specialised rewrites, generated per rule set by csrc/jit.cpp.
template <int kTier>
__device__ __forceinline__ void jit_warp(Round<kTier>& c, bool valid, uint32_t l, uint32_t r);
template <int kTier>
__device__ __forceinline__ void jit_apply(Round<kTier>& c, uint32_t rule, const uint4& A, const uint4& B, uint32_t l,
                                          uint32_t r);

// Both claims of a rewrite with their ring atomics issued back to back.
template <uint32_t MF, uint32_t MX, int kTier>
__device__ __forceinline__ bool jit_alloc_both(Round<kTier>& c, uint32_t nf, uint32_t nx, uint32_t (&f)[MF],
                                               uint32_t (&g)[MX]) {
  if ((nf | nx) == 0) return true;
  uint32_t tv = 0, ta = 0;
  if constexpr (kTake2<kTier>) {
    const uint32_t w = atomicAdd(&c.cur->atake, (nf << 16) | nx);
    tv = w >> 16;
    ta = w & 0xFFFFu;
  } else {
    tv = nf ? atomicAdd(&c.cur->vtake, nf) : 0u;
    ta = nx ? atomicAdd(&c.cur->atake, nx) : 0u;
  }
  const uint32_t av_v = c.hi_v - c.lo_v, av_a = c.hi_a - c.lo_a;

  const uint32_t gv = tv < av_v ? min(av_v - tv, nf) : 0u, ga = ta < av_a ? min(av_a - ta, nx) : 0u;
  uint32_t bv = 0, ba = 0;
  if (gv < nf) {
    bv = atomicAdd(&c.ctl->var_bump, nf - gv);
    if (bv + (nf - gv) > c.cap_vars) {
      fail(c, INET_ERR_ARENA, 1);
      return false;
    }
  }
  if (ga < nx) {
    ba = atomicAdd(&c.ctl->agent_bump, nx - ga);
    if (ba + (nx - ga) > c.cap_agents) {
      fail(c, INET_ERR_ARENA, 0);
      return false;
    }
  }
  // only the claimed ring entries are read (predicated loads, still issued back
  // to back): an entry past the claim may be being written by a freer this round
  uint32_t rv[MF], ra[MX];
#pragma unroll
  for (uint32_t j = 0; j < MF; ++j) rv[j] = j < gv ? static_cast<uint32_t>(c.vring[(c.lo_v + tv + j) & c.vmask]) : 0u;
#pragma unroll
  for (uint32_t j = 0; j < MX; ++j) ra[j] = j < ga ? static_cast<uint32_t>(c.aring[(c.lo_a + ta + j) & c.amask]) : 0u;
#pragma unroll
  for (uint32_t j = 0; j < MF; ++j) f[j] = vtag<kTier>() | (j < gv ? rv[j] : bump_var(c, bv + (j - gv)));
#pragma unroll
  for (uint32_t j = 0; j < MX; ++j) g[j] = j < ga ? ra[j] : bump_agent(c, ba + (j - ga));
#if INET_STAMPS
  if (c.stamps && nf) {
#pragma unroll
    for (uint32_t j = 0; j < MF; ++j)
      if (j < nf) stamp_store(c, f[j], j);
    stamp_publish(c);
  }
#endif
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
  key_of(c, l, r, key, val);
  x = key & ~vtag<kTier>();
  return true;
}

#endif

// Rewrite one active pair (find_rule + instantiate, core.py:281-312).
template <int kTier>
__device__ __forceinline__ void interact(Round<kTier>& c, uint32_t l, uint32_t r) {
  INET_TMARK(c, 0);
  INET_TR(c, 1);
  uint4 A = ld_agent(c, l);
  uint4 B = ld_agent(c, r);
  const uint32_t t = c.pair[A.x * c.n_labels + B.x];
  INET_TMARK(c, 1);
  INET_TR(c, 2);
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
#if !defined(INET_CTIMING) && INET_COUNT_RULES
  if (c.d->rule_hist) atomicAdd(&c.d->rule_hist[t >> 1], 1u);
#endif
#if INET_STAMPS
  c.cid = l;  // identifies this interaction in its fresh variables' stamps
#endif
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
  INET_TR(c, 3);
  auto fresh = [&](uint32_t j) -> uint32_t {
    return vtag<kTier>() | (j < fv.got ? static_cast<uint32_t>(c.vring[(fv.pos + j) & c.vmask]) : bump_var(c, fv.bump + (j - fv.got)));
  };
  auto extra = [&](uint32_t q) -> uint32_t {
    return q < na.got ? static_cast<uint32_t>(c.aring[(na.pos + q) & c.amask]) : bump_agent(c, na.bump + (q - na.got));
  };
#if INET_STAMPS
  if (c.stamps && nf) {
    for (uint32_t j = 0; j < nf; ++j) stamp_store(c, fresh(j), j);
    stamp_publish(c);
  }
#endif
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
    st_agent(c, src(kEnvNew + m), make_uint4(w & 0xFFu, src((w >> 8) & 0xFFu), src((w >> 16) & 0xFFu), src(w >> 24)));
  }
  if (nn < 2) free_agent(c, r);
  if (nn < 1) free_agent(c, l);
  INET_TMARK(c, 3);
  INET_TR(c, 4);
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
        key_of(c, el, er, key, vals[e]);
        xs[e] = key & ~vtag<kTier>();
        olds[e] = exch_slot(c, xs[e], vals[e]);
      }
    }
  }
  INET_TR(c, 5);
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

#ifdef INET_JIT_WARP
constexpr bool kWarpRewrite = true;
#else
constexpr bool kWarpRewrite = false;
#endif

// Warp-collective entry: every lane of the warp calls it; lanes with `valid`
// rewrite their pair. The rule-set kernels run the whole warp through one
// specialised rewrite (jit_warp); the interpreter handles lanes one by one.
template <int kTier>
__device__ __forceinline__ void interact_w(Round<kTier>& c, bool valid, uint32_t l, uint32_t r) {
#ifdef INET_JIT_WARP
  jit_warp<kTier>(c, valid, l, r);
#else
  if (valid) interact(c, l, r);
#endif
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
  uint32_t ctl_off, aring_off, vring_off, agents_off, slots_off, queue_off, env_off, cagent_off, words;
  uint32_t acache_off;  // tier M: agent-record cache
  uint32_t outc_off, inbox_off, mbox_off;  // tier C
};

__host__ __device__ inline uint32_t align4(uint32_t w) { return (w + 3u) & ~3u; }

// Shared-memory plan (32-bit words):
//   S: rules | Ctl | u16 rings | agents | slots | 2 packed queues
//   M: rules | Ctl | u16 rings | slots | 2 packed queues | agent cache (agents global)
//   G: rules | Ctl | u32 rings                                   (rest global)
//   C: rules | Ctl | u32 rings | 3 counter sets | 3 mail counts | 3 inboxes |
//      2x2 mailboxes | slots | 2 input queues [16][res_queue] | agents
//      (this CTA's share of the cluster-wide arrays)
__host__ __device__ inline SmemPlan plan_smem(const Shape& sh, int tier) {
  const uint32_t ring_bytes = tier >= kTierG ? 4u : 2u;
  SmemPlan p;
  p.ctl_off = align4(sh.rule_words);
  p.aring_off = p.ctl_off + align4(sizeof(Ctl) / 4);
  const bool smem_rings = tier != kTierX;  // tier X keeps its rings in global memory
  p.vring_off = p.aring_off + (smem_rings ? align4((sh.ring_a * ring_bytes + 3) / 4) : 0);
  p.agents_off = p.vring_off + (smem_rings ? align4((sh.ring_v * ring_bytes + 3) / 4) : 0);
  p.outc_off = p.inbox_off = p.mbox_off = 0;
  if (tier == kTierC) {
    p.outc_off = p.agents_off + align4(3 * sizeof(RoundCtr) / 4);
    p.inbox_off = p.outc_off + 3 * 32;
    p.mbox_off = p.inbox_off + 3 * 16 * 8;
    p.slots_off = p.mbox_off + 2 * 2 * 16 * kMbox;
    p.queue_off = p.slots_off + align4(sh.res_vars);
    p.env_off = p.queue_off + 2 * 16 * sh.res_queue * 2;
    p.cagent_off = p.env_off;
    p.words = p.cagent_off + 4 * sh.res_agents;
    return p;
  }
  p.slots_off = p.agents_off + (tier == kTierS ? 2 * sh.res_agents : 0);  // compact 8-byte agents
  const bool res_slots = tier != kTierG;
  p.queue_off = p.slots_off + (res_slots ? align4(sh.res_vars) : 0);
  p.env_off = p.queue_off + (res_slots ? align4(2 * sh.res_queue) : 0);
  p.cagent_off = p.env_off;
  p.words = p.cagent_off;
  p.acache_off = 0;
  if (tier == kTierM) {
    p.acache_off = align4(p.words);
    p.words = p.acache_off + 4 * kAgentCache;
  }
  return p;
}

// Device-side finalize of a tier S net whose arena is still in shared memory
// (restates engine.finalize, src/inet/engine.py:287-362, and the preorder
// compaction of host.cpp finalize_net, for the nets where every parked
// equation is eliminated). A parked equation x = t (slot[x] = t) has the
// other occurrence of x in the interface or in an agent port; walking the net
// from the interface roots in preorder (port 0 first), every variable met
// whose slot is set is replaced by its value (following var-valued chains), so
// each equation is consumed at its variable's other occurrence exactly as the
// reference's elimination does. When the walk consumes every parked equation
// the substituted net is a tree whose preorder is the host's compaction order:
// records go to d.agents[0, nf), the interface to d.residual[i].x, and nf + 1
// is returned. Otherwise (an equation left over: a cycle or a part not
// reachable from the interface; a shared agent; an interface longer than 32;
// scratch that does not fit) nothing is written and 0 is returned: the host
// finalizes from the arena copy as before.
// Scratch, all free once the loop has stopped: the queues hold the DFS stack,
// the agent ring the preorder list, the variable ring the remap table.
constexpr uint32_t kConsumed = 0x40000000u;  // finalize_smem: a parked equation already applied

template <int kTier>
__device__ uint32_t finalize_smem(const Round<kTier>& c, const NetDesc& d, Ctl* ctl, const SmemPlan& plan,
                                  uint32_t* smem, const Shape& sh, uint32_t hw, uint32_t ahw, uint32_t n_parked) {
  uint32_t* const ifc = ctl->scratch;  // the resolved interface (<= 32 refs); scratch[33]: verdict
  uint32_t* const stack = smem + plan.queue_off;
  uint16_t* const order = reinterpret_cast<uint16_t*>(smem + plan.aring_off);
  uint16_t* const remap = reinterpret_cast<uint16_t*>(smem + plan.vring_off);
  const uint32_t ni = d.n_iface;
  const bool fits = ctl->err_code == 0 && ni <= 32 && 2 * sh.res_queue >= ahw + 3 && sh.ring_a >= ahw &&
                    sh.ring_v >= ahw && ahw < 0xFFFFu;
  __syncthreads();  // the residual scan's last use of ctl->scratch
  if (!fits) return 0;
  for (uint32_t i = threadIdx.x; i < ahw; i += blockDim.x) remap[i] = 0xFFFFu;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t consumed = 0, nf = 0, sp = 0;
    bool ok = true;
    // the value a reference stands for once the parked equations are applied;
    // a consumed slot keeps its value, marked (a variable is met at most once)
    auto resolve = [&](uint32_t t) {
      for (uint32_t guard = 0; t != kNone && (t & kVar) && guard <= n_parked; ++guard) {
        const uint32_t x = t & ~vtag<kTier>();
        const uint32_t v = x < hw ? c.vslot[x] : kNone;
        if (v == kNone) break;
        if (v & kConsumed) {
          ok = false;
          break;
        }
        c.vslot[x] = v | kConsumed;
        consumed += 1;
        t = v;
      }
      return t;
    };
    for (uint32_t i = 0; i < ni && ok; ++i) {
      const uint32_t root = resolve(ref_in<kTier>(d.in_iface[i]));
      ifc[i] = root;
      if (root == kNone || (root & kVar)) continue;
      stack[sp++] = root;
      while (sp) {
        const uint32_t a = stack[--sp];
        if (a >= ahw || remap[a] != 0xFFFFu) {  // shared agent: not a tree
          ok = false;
          break;
        }
        remap[a] = static_cast<uint16_t>(nf);
        order[nf++] = static_cast<uint16_t>(a);
        const uint4 A = ld_agent(c, a);
        const uint4 R = make_uint4(A.x, resolve(A.y), resolve(A.z), resolve(A.w));
        if (sp + 3 > 2 * sh.res_queue) {
          ok = false;
          break;
        }
        if (R.w != kNone && !(R.w & kVar)) stack[sp++] = R.w;
        if (R.z != kNone && !(R.z & kVar)) stack[sp++] = R.z;
        if (R.y != kNone && !(R.y & kVar)) stack[sp++] = R.y;
      }
    }
    ctl->scratch[33] = ok && consumed == n_parked ? nf + 1 : 0u;
  }
  __syncthreads();
  const uint32_t rows = ctl->scratch[33];
  if (!rows) return 0;
  // the agents themselves are left untouched (a failed attempt must leave the
  // arena as the host finalize expects it): ports are resolved again here
  auto map = [&](uint32_t t) {
    for (uint32_t guard = 0; t != kNone && (t & kVar) && guard <= n_parked; ++guard) {
      const uint32_t x = t & ~vtag<kTier>();
      const uint32_t v = x < hw ? c.vslot[x] : kNone;
      if (v == kNone) break;
      t = v & ~kConsumed;
    }
    return (t == kNone || (t & kVar)) ? ref_out<kTier>(t) : static_cast<uint32_t>(remap[t]);
  };
  for (uint32_t j = threadIdx.x; j < rows - 1; j += blockDim.x) {
    const uint4 A = ld_agent(c, order[j]);
    d.agents[j] = make_uint4(A.x, map(A.y), map(A.z), map(A.w));
  }
  if (threadIdx.x < ni) d.residual[threadIdx.x] = make_uint2(map(ifc[threadIdx.x]), 0u);
  return rows;
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
  c.acache = reinterpret_cast<uint4*>(smem + plan.acache_off);
  if constexpr (kTier == kTierM)
    for (uint32_t i = threadIdx.x; i < kAgentCache; i += blockDim.x) c.acache[i] = make_uint4(0, 0, 0, 0);
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
  const long long clk0 = clock64();
  const unsigned long long gt0 = globaltimer();
  // ---- init: private copy of the input agents, empty slots, zero counters
  const bool fits = d.n_in_agents <= c.cap_agents && d.n_in_vars <= c.cap_vars;
  for (uint32_t i = threadIdx.x; i < c.cap_vars; i += blockDim.x) c.vslot[i] = kNone;
  if (fits)
    for (uint32_t i = threadIdx.x; i < d.n_in_agents; i += blockDim.x) st_agent(c, i, agent_in<kTier>(d.in_agents[i]));
  {
    uint32_t* w = reinterpret_cast<uint32_t*>(ctl);
    for (uint32_t i = threadIdx.x; i < sizeof(Ctl) / 4; i += blockDim.x) w[i] = 0;
  }
  __syncthreads();
  // Round state, kept identically by every thread: each thread closes every
  // round itself from the round's counters, so a round ends with one barrier
  // and no serial bookkeeping warp.
  bool stop = false;
  uint32_t stop_err = 0;
  if (threadIdx.x == 0) {
    ctl->agent_bump = d.n_in_agents;
    ctl->var_bump = d.n_in_vars;
  }
  if (!fits) {
    stop = true;
    stop_err = INET_ERR_ARENA;
  } else if (sh.max_rounds == 0) {  // loop 1 > max_loops (engine.py:205-207), even for the no-op loop
    stop = true;
    stop_err = INET_ERR_LOOP_CAP;
  } else if (d.n_in_eqs == 0) {  // one no-op loop (engine.py:222-223)
    stop = true;
    if (threadIdx.x == 0 && d.stats && d.cap_rounds) d.stats[0] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  c.failed = false;
#if INET_STAMPS
  c.stamps = d.stamps;
  c.round = 0;
  c.cid = 0;
  if (c.stamps)  // input variables: {round 0 | dense id}, dense ids are in the input's id order
    for (uint32_t x = threadIdx.x; x < d.n_in_vars; x += blockDim.x) c.stamps[x] = static_cast<unsigned long long>(x) << 8;
  __syncthreads();
#endif
  c.env = smem + plan.env_off + threadIdx.x;
  if constexpr (T::kEnvSmem) c.env[(kEnvSize - 1) * blockDim.x] = kNone;  // (disabled tier option)
#ifdef INET_TIMING
  for (int i = 0; i < 8; ++i) c.tm[i] = 0;
  c.tlast = clock64();
#endif
  const uint32_t lane = threadIdx.x & 31u;
  c.cap_def = d.cap_def;
  // Per-round totals are only needed for the per-round rows; otherwise each
  // thread keeps its own running totals, summed once after the loop. (Tier
  // M's hand-over threshold counts queued pairs instead: the pairs queued in
  // round r are exactly the interactions of round r + 1.)
  const bool per_round = INET_ROWS && d.stats != nullptr;
  unsigned long long tot_q = 0;
  c.ints = c.comms = 0;
  c.parked = 0;
  uint32_t lo_a = 0, hi_a = 0, lo_v = 0, hi_v = 0, n = d.n_in_eqs, nd = 0, rounds = 1;
  int32_t parked_tot = 0;
  unsigned long long tot_i = 0, tot_c = 0, t_prev = globaltimer();
  // counter sets r % 3 (this round), (r + 1) % 3 (cleared now), (r + 2) % 3
  // (read by the previous round's close), rotated as pointers
  RoundCtr *cur = &ctl->ctr3[1], *nxt = &ctl->ctr3[2], *old = &ctl->ctr3[0];
  // queue buffers: this round's input and output, swapped every round
  char* q_in = static_cast<char*>(q0);
  char* q_out = static_cast<char*>(q0) + size_t(qstride) * (T::kPacked ? 4u : 8u);
  const bool input_active = (d.dev_final & kInputActive) != 0;
  const bool detect_vh = !INET_EXACT_CODE && sh.detect_vh;
#ifdef INET_TRACE
  long long tr_top = 0;
  uint32_t tr_items = 0;
#endif
  for (uint32_t r = 1; !stop; ++r) {
#ifdef INET_TRACE
    tr_top = clock64();
    tr_items = 0;
#endif
    c.cur = cur;
#if INET_STAMPS
    c.round = r;
#endif
    c.lo_a = lo_a;
    c.hi_a = hi_a;
    c.lo_v = lo_v;
    c.hi_v = hi_v;
    if (per_round) {
      c.ints = c.comms = 0;
      c.parked = 0;
    }
    if (threadIdx.x < sizeof(RoundCtr) / 4) reinterpret_cast<uint32_t*>(nxt)[threadIdx.x] = 0;
    c.dout = INET_EXACT_CODE && sh.exact ? d.deferred + (r & 1u) * d.cap_def : nullptr;
    c.out = q_out;
    if (INET_EXACT_CODE && nd) {
      // equations merged last round that are still var-headed: this round's
      // communication links them (reference loop mode)
      const uint2* din = d.deferred + ((r - 1) & 1u) * d.cap_def;
      for (uint32_t i = threadIdx.x; i < nd && !c.failed; i += blockDim.x) {
        const uint2 eq = din[i];
        c.parked -= 1;
        link(c, eq.x, eq.y);
      }
    }
    if (r == 1) {
      // the input equations, in any class (communication_phase's first pass)
      c.out = T::kPacked ? static_cast<void*>(static_cast<uint32_t*>(q0) + qstride)
                         : static_cast<void*>(static_cast<uint2*>(q0) + qstride);
      if constexpr (kWarpRewrite) {
        for (uint32_t b = threadIdx.x & ~31u; b < n; b += blockDim.x) {
          const uint32_t i = b + lane;
          const bool v = i < n && !c.failed;
          const uint2 eq = v ? make_uint2(ref_in<kTier>(d.in_eqs[i].x), ref_in<kTier>(d.in_eqs[i].y)) : make_uint2(0, 0);
          const bool act = v && ((eq.x | eq.y) & kVar) == 0;
          interact_w(c, act, eq.x, eq.y);
          if (v && !act && !c.failed) link(c, eq.x, eq.y);
        }
      } else {
        for (uint32_t i = threadIdx.x; i < n && !c.failed; i += blockDim.x) {
          const uint2 eq = make_uint2(ref_in<kTier>(d.in_eqs[i].x), ref_in<kTier>(d.in_eqs[i].y));
          if (((eq.x | eq.y) & kVar) == 0)
            interact(c, eq.x, eq.y);
          else
            link(c, eq.x, eq.y);
        }
      }
    } else if constexpr (T::kPacked) {
      const uint32_t* in = reinterpret_cast<const uint32_t*>(q_in);
      if constexpr (kWarpRewrite) {
        for (uint32_t b = threadIdx.x & ~31u; b < n; b += blockDim.x) {
          const uint32_t i = b + lane;
          const bool v = i < n && !c.failed;
          const uint32_t w = v ? in[i] : 0u;
          interact_w(c, v, w >> 16, w & 0xFFFFu);
        }
      } else {
        for (uint32_t i = threadIdx.x; i < n && !c.failed; i += blockDim.x) {
          INET_TR(c, 0);
          const uint32_t w = in[i];
          interact(c, w >> 16, w & 0xFFFFu);
#ifdef INET_TRACE
          c.tr[6] = clock64();
          tr_items += 1;
#endif
        }
      }
    } else {
      const uint2* in = reinterpret_cast<const uint2*>(q_in);
      if constexpr (kWarpRewrite) {
        for (uint32_t b = threadIdx.x & ~31u; b < n; b += blockDim.x) {
          const uint32_t i = b + lane;
          const bool v = i < n && !c.failed;
          const uint2 eq = v ? in[i] : make_uint2(0, 0);
          interact_w(c, v, eq.x, eq.y);
        }
      } else {
        for (uint32_t i = threadIdx.x; i < n && !c.failed; i += blockDim.x) {
          const uint2 eq = in[i];
          interact(c, eq.x, eq.y);
        }
      }
    }
    INET_TMARK(c, 5);
    if (per_round) {
      const uint32_t wi = __reduce_add_sync(0xFFFFFFFFu, c.ints);
      const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, c.comms);
      const int32_t wp = __reduce_add_sync(0xFFFFFFFFu, c.parked);
      if (lane == 0) {
        if (wi) atomicAdd(&cur->ints, wi);
        if (wc) atomicAdd(&cur->comms, wc);
        if (wp) atomicAdd(&cur->parked, wp);
      }
    }
    INET_TMARK(c, 6);
#ifdef INET_TRACE
    const long long tr_arr = clock64();
#endif
    __syncthreads();
    INET_TMARK(c, 7);
#ifdef INET_TRACE
    {  // development: one line per thread with pairs (and thread 0) in rounds [R0, R0 + 3)
      const long long tr_exit = clock64();
      if (r >= INET_TRACE_R0 && r < INET_TRACE_R0 + 3 && (tr_items || threadIdx.x == 0) && blockIdx.x == 0)
        printf("MT r=%u t=%u items=%u n=%u start=%lld q+ag=%lld pair=%lld alloc=%lld recs=%lld exissue=%lld settle=%lld "
               "tail=%lld arrive=%lld exit=%lld\n",
               r, threadIdx.x, tr_items, n, tr_items ? c.tr[0] - tr_top : 0ll, tr_items ? c.tr[2] - c.tr[0] : 0ll,
               tr_items ? c.tr[2] - c.tr[1] : 0ll, tr_items ? c.tr[3] - c.tr[2] : 0ll, tr_items ? c.tr[4] - c.tr[3] : 0ll,
               tr_items ? c.tr[5] - c.tr[4] : 0ll, tr_items ? c.tr[6] - c.tr[5] : 0ll,
               tr_items ? tr_arr - c.tr[6] : 0ll, tr_arr - tr_top, tr_exit - tr_top);
    }
#endif
    // ---- close round r (every thread, same values)
    const RoundCtr k = *cur;
    bool round_failed = (k.qcount & kErrBit) != 0;
    const uint32_t q = kPush2<kTier> ? (k.vfree & 0xFFFFu) : (k.qcount & ~kErrBit);
#if INET_EXACT_CODE
    if (k.dcount > d.cap_def) {
      round_failed = true;
      if (threadIdx.x == 0 && atomicCAS(&ctl->err_code, 0u, static_cast<uint32_t>(INET_ERR_ARENA)) == 0u) ctl->err_a = 3;
    }
#endif
    // frees of round r were kept while they fit the ring (against its old window)
    const uint32_t wa = min(k.afree, sh.ring_a - (hi_a - lo_a));
    const uint32_t wv = min(kPush2<kTier> ? (k.vfree >> 16) : k.vfree, sh.ring_v - (hi_v - lo_v));
    const uint32_t atake = kTake2<kTier> ? (k.atake & 0xFFFFu) : k.atake;
    const uint32_t vtake = kTake2<kTier> ? (k.atake >> 16) : k.vtake;
    lo_a += min(atake, hi_a - lo_a);
    hi_a += wa;
    lo_v += min(vtake, hi_v - lo_v);
    hi_v += wv;
    if (per_round) {
      parked_tot += k.parked;
      tot_i += k.ints;
      tot_c += k.comms;
    }
    {
      RoundCtr* t = cur;
      cur = nxt;
      nxt = old;
      old = t;
      char* u = q_in;
      q_in = q_out;
      q_out = u;
    }
    if (per_round && threadIdx.x == 0) {
#ifdef INET_NO_TIMER
      const unsigned long long now = 0;
#else
      const unsigned long long now = globaltimer();
#endif
      if (r - 1 < d.cap_rounds)
        d.stats[r - 1] = make_uint4(k.ints, k.comms, q + static_cast<uint32_t>(parked_tot),
                                    static_cast<uint32_t>(now - t_prev));
      t_prev = now;
    }
    // a round that had no pairs and whose deferred equations all parked was
    // itself the reference's trailing no-op loop (exact mode: the last loop can
    // be communication only); no second trailing row then
    const bool was_noop = (r > 1 ? n == 0 : !input_active) && q == 0 &&
                          (INET_EXACT_CODE ? k.dcount : 0u) == 0;
    rounds = was_noop ? r : r + 1;
    n = q;
    nd = INET_EXACT_CODE ? k.dcount : 0u;
    if (round_failed) {
      stop = true;
    } else if (detect_vh && k.vh) {
      stop = true;  // the host reruns the net with reference-loop code
      stop_err = kNeedExact;
    } else if (was_noop) {
      stop = true;  // this round was the trailing no-op loop (its row is written)
    } else if (r + 1 > sh.max_rounds) {  // engine.py:205-207 (checked before every loop, the no-op one too)
      stop = true;
      stop_err = INET_ERR_LOOP_CAP;
    } else if (q == 0 && nd == 0) {
      // the trailing no-op loop the reference records (engine.py:222-223)
      stop = true;
      if (per_round && threadIdx.x == 0 && r < d.cap_rounds)
        d.stats[r] = make_uint4(0, 0, static_cast<uint32_t>(parked_tot), 0);
    } else if (kTier == kTierM && sh.promote_ints && (tot_q += q) >= sh.promote_ints) {
      stop = true;  // a large net: the host hands it over to a cluster
      stop_err = kPromote;
    }
  }
  if (threadIdx.x == 0) {
    if (stop_err) atomicCAS(&ctl->err_code, 0u, stop_err);
    ctl->rounds = rounds;
    ctl->tot_i = tot_i;
    ctl->tot_c = tot_c;
    ctl->parked_total = parked_tot;
    ctl->hdr.n = n;
    ctl->hdr.nd = nd;
  }
  if (!per_round) {
    __syncthreads();
    const uint32_t wi = __reduce_add_sync(0xFFFFFFFFu, c.ints);
    const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, c.comms);
    const int32_t wp = __reduce_add_sync(0xFFFFFFFFu, c.parked);
    if (lane == 0) {
      if (wi) atomicAdd(&ctl->tot_i, static_cast<unsigned long long>(wi));
      if (wc) atomicAdd(&ctl->tot_c, static_cast<unsigned long long>(wc));
      if (wp) atomicAdd(&ctl->parked_total, wp);
    }
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
  const bool handed = kTier == kTierM && ctl->err_code == kPromote;
  if constexpr (kTier == kTierM) {
    if (handed) {
      // handing the net over to a cluster (tier C resumes it): the slot table,
      // then the next round's pairs followed by its deferred equations
      const uint32_t r = ctl->rounds - 1, n = ctl->hdr.n, nd = ctl->hdr.nd;
      for (uint32_t x = threadIdx.x; x < hw; x += blockDim.x) d.vslot[x] = c.vslot[x];
      const uint32_t* pq = static_cast<const uint32_t*>(q0) + (r & 1u) * qstride;
      const uint2* pd = d.deferred + (r & 1u) * d.cap_def;
      for (uint32_t i = threadIdx.x; i < n + nd && i < d.cap_queue; i += blockDim.x)
        d.queue[i] = i < n ? make_uint2(pq[i] >> 16, pq[i] & 0xFFFFu) : pd[i - n];
      base = n + nd;
      if (base > d.cap_queue && threadIdx.x == 0) ctl->err_code = INET_ERR_ARENA;
      __syncthreads();
    }
  }
  for (uint32_t c0 = 0; c0 < hw && !handed; c0 += blockDim.x) {
    const uint32_t x = c0 + threadIdx.x;
    const uint32_t v = x < hw ? c.vslot[x] : kNone;
    uint32_t off;
    const uint32_t tot = block_scan_flag(v != kNone, ctl->scratch, &off);
    if (v != kNone && base + off < d.cap_vars) d.residual[base + off] = make_uint2(kVar | x, ref_out<kTier>(v));
    base += tot;
  }
  const uint32_t ahw = min(ctl->agent_bump, c.cap_agents);
  uint32_t nf_rows = 0;  // device-finalized normal form: agents + 1 (0: the host finalizes)
  if constexpr (kTier == kTierS) {
    if ((d.dev_final & 1u) && !handed) nf_rows = finalize_smem(c, d, ctl, plan, smem, sh, hw, ahw, base);
  }
  if constexpr (T::kAgentsSmem) {
    const uint32_t n_copy = nf_rows ? 0u : min(ahw, d.cap_agents);
    for (uint32_t i = threadIdx.x; i < n_copy; i += blockDim.x) d.agents[i] = agent_out<kTier>(ld_agent(c, i));
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
    g->pad[0] = clock_mhz(clk0, gt0);
    g->pad[1] = nf_rows;
    g->pad[2] = nf_rows ? d.n_iface : 0u;
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


// ---------------------------------------------------------------------------
// Tier C: one net reduced by a thread-block cluster of G CTAs (one per SM),
// all of its state in the cluster's distributed shared memory.
//
// The round structure is the one of run_net, spread over G SMs:
//   * agent and variable ids are owned round-robin: id i lives at index
//     i >> log2 G of CTA i & (G-1). Agent loads/stores and slot exchanges are
//     ld/st/atom.shared::cluster (~0.2 us remote, local ones stay on the SM);
//     nothing on the round path touches global memory;
//   * every CTA allocates only ids it owns (its rings and bump pointer), and a
//     freed id goes back to its owner's ring (free_owned), so the per-CTA
//     arenas stay balanced whatever the work split;
//   * every CTA appends the pairs it creates to its own shared-memory queue;
//     the next round, CTA k takes the pairs whose global index is k mod G,
//     reading them from their producer's queue;
//   * a round closes with __syncthreads, a push of the CTA's counters
//     {pairs queued, interactions, merges, parked delta} into every CTA's
//     inbox, and one cluster barrier (release/acquire); after it every warp
//     scans the inbox locally to split the next round;
//   * the counters rotate over three sets (round r counts into set r%3, its
//     readers use it between barriers r and r+1, it is cleared in round r+2).
// Thread 0 of CTA 0 keeps the running totals and writes the per-round row.
// At the fixpoint the CTAs write their shares back to the global arrays,
// where the residual equations are compacted in variable-id order.

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_index() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

#ifdef INET_CTIMING
// Development build: critical-path split of a tier C round, per CTA (thread
// 0's clock for the barrier, CTA maxima for work and arrival), summed over
// rounds into the rule-histogram area (tools/cluster_timing.py).
#define CT_MARK(k)                                                            \
  do {                                                                        \
    const long long _t = clock64();                                           \
    if ((k) == 0) ct_t0 = _t;                                                 \
    if ((k) == 1) atomicMax(&ct_max[0], static_cast<unsigned long long>(_t - ct_t0)); \
    if ((k) == 2) atomicMax(&ct_max[1], static_cast<unsigned long long>(_t - ct_t0)); \
    if ((k) == 3 && threadIdx.x == 0) {                                       \
      ct_sum[0] += ct_max[0];                                                 \
      ct_sum[1] += ct_max[1] - ct_max[0];                                     \
      ct_sum[2] += _t - ct_t0 - ct_max[1];                                    \
      ct_max[0] = ct_max[1] = 0;                                              \
    }                                                                         \
    if ((k) == 0 && threadIdx.x == 0 && ct_t3) ct_sum[3] += _t - ct_t3;       \
    if ((k) == 3) ct_t3 = _t;                                                 \
  } while (0)
#else
#define CT_MARK(k) \
  do {             \
  } while (0)
#endif

template <int kBlock>
__device__ void run_net_cluster(const NetDesc& d, const Shape& sh, const uint16_t* pair, const uint32_t* rules,
                                uint32_t* smem) {
  constexpr int kTier = kTierC;
  const SmemPlan plan = plan_smem(sh, kTier);
  Ctl* ctl = reinterpret_cast<Ctl*>(smem + plan.ctl_off);
  RoundCtr* ctr3 = reinterpret_cast<RoundCtr*>(smem + plan.agents_off);
  uint32_t* const outc3 = smem + plan.outc_off;                          // [3][32] ids mailed per owner
  uint4* const inbox = reinterpret_cast<uint4*>(smem + plan.inbox_off);  // [3][16][2] counters per source CTA
  uint32_t* const mbox = smem + plan.mbox_off;                           // [2 parity][2 kind][16 src][kMbox]
  uint4* const lagents = reinterpret_cast<uint4*>(smem + plan.cagent_off);
  uint32_t* const lslots = smem + plan.slots_off;
  uint2* const lqueue = reinterpret_cast<uint2*>(smem + plan.queue_off);  // [2 parity][16 producer][res_queue]
  const uint32_t G = cluster_size(), rank = cluster_rank();
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  Round<kTier> c;
  c.d = &d;
  c.ctl = ctl;
  c.aring = smem + plan.aring_off;
  c.vring = smem + plan.vring_off;
  c.amask = sh.ring_a - 1;
  c.vmask = sh.ring_v - 1;
  c.pair = pair;
  c.rules = rules;
  c.n_labels = sh.n_labels;
  c.agents = lagents;
  c.vslot = lslots;
  // Ids are owned round-robin: CTA k owns k, k+G, k+2G, ... (inputs included)
  // and keeps id k+G*s at index s of its shared-memory arrays.
  c.stride = G;
  c.gshift = __ffs(G) - 1;
  c.rank = rank;
  c.a_base = rank;
  c.v_base = rank;
  auto owned_below = [&](uint32_t n) -> uint32_t { return n > rank ? (n - rank + G - 1) / G : 0u; };
  c.cap_agents = min(sh.res_agents, sh.ring_a);
  c.cap_vars = min(sh.res_vars, sh.ring_v);
  const uint32_t s0_a = owned_below(d.n_in_agents), s0_v = owned_below(d.n_in_vars);
  const uint32_t cap_q = sh.res_queue;  // pairs one producer can deal to one consumer per round
  c.cap_queue = cap_q;
  c.qj = cap_q;
  c.cap_def = d.cap_def / G;
  const long long clk0 = clock64();
  const unsigned long long gt0 = globaltimer();
  // ---- init: this CTA's share of the input agents, empty slots, zero counters
  const bool fits = s0_a <= c.cap_agents && s0_v <= c.cap_vars && uint64_t(G) * c.cap_agents <= d.cap_agents &&
                    uint64_t(G) * c.cap_vars <= d.cap_vars;
  for (uint32_t i = threadIdx.x; i < c.cap_vars; i += kBlock)
    lslots[i] = d.resume && i < s0_v ? d.vslot[rank + G * i] : kNone;
  if (fits)
    for (uint32_t i = threadIdx.x; i < s0_a; i += kBlock) lagents[i] = d.in_agents[rank + G * i];
  {
    uint32_t* w = reinterpret_cast<uint32_t*>(ctl);
    for (uint32_t i = threadIdx.x; i < sizeof(Ctl) / 4; i += kBlock) w[i] = 0;
    w = reinterpret_cast<uint32_t*>(ctr3);
    for (uint32_t i = threadIdx.x; i < plan.mbox_off - plan.agents_off; i += kBlock) w[i] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ctl->agent_bump = s0_a;
    ctl->var_bump = s0_v;
  }
#ifdef INET_CTIMING
  __shared__ unsigned long long ct_max[2];
  unsigned long long ct_sum[4] = {0, 0, 0, 0};
  long long ct_t0 = clock64(), ct_t3 = 0;
  if (threadIdx.x == 0) ct_max[0] = ct_max[1] = 0;
#endif
  cluster_barrier();
  c.failed = false;
#if INET_STAMPS
  c.stamps = nullptr;  // (single-CTA tiers only)
  c.round = c.cid = 0;
#endif
  uint32_t lo_a = 0, hi_a = 0, lo_v = 0, hi_v = 0;
  // running totals: thread 0 of CTA 0
  unsigned long long tot_i = d.base_ints, tot_c = d.base_comms, t_prev = globaltimer();
  int32_t parked_tot = d.base_parked;
  const uint32_t rb = d.round_base;  // rounds done before this launch (resume)
  uint32_t N = d.n_in_eqs, excl = 0, rounds = 1, stop_err = 0;
  bool stop = false, mail_any = false;
  const bool writer = rank == 0 && threadIdx.x == 0;
  // per-round totals only for the per-round rows; otherwise per-thread
  // running totals, summed once after the loop
  const bool per_round = INET_ROWS && d.stats != nullptr;
  c.ints = c.comms = 0;
  c.parked = 0;
  if (!fits) {
    stop = true;
    stop_err = INET_ERR_ARENA;
  } else if (sh.max_rounds == 0) {  // loop 1 > max_loops (engine.py:205-207), even for the no-op loop
    stop = true;
    stop_err = INET_ERR_LOOP_CAP;
  } else if (N == 0) {  // one no-op loop (engine.py:222-223)
    stop = true;
    if (writer && d.stats && d.cap_rounds) d.stats[0] = make_uint4(0, 0, 0, 0);
  }
  for (uint32_t r = 1; !stop; ++r) {
    RoundCtr* cur = &ctr3[r % 3];
    c.cur = cur;
    c.lo_a = lo_a;
    c.hi_a = hi_a;
    c.lo_v = lo_v;
    c.hi_v = hi_v;
    if (per_round) {
      c.ints = c.comms = 0;
      c.parked = 0;
    }
    c.inq = lqueue + (r & 1u) * 16 * cap_q;
    c.dout = INET_EXACT_CODE && sh.exact ? d.deferred + ((r & 1u) * G + rank) * c.cap_def : nullptr;
    c.outc = outc3 + (r % 3) * 32;
    c.mbox_a = mbox + (r & 1u) * 2 * 16 * kMbox;
    c.mbox_v = c.mbox_a + 16 * kMbox;
    if (threadIdx.x < 32) {
      if (threadIdx.x < sizeof(RoundCtr) / 4) reinterpret_cast<uint32_t*>(&ctr3[(r + 1) % 3])[threadIdx.x] = 0;
      outc3[((r + 1) % 3) * 32 + threadIdx.x] = 0;
    }
    // mail of round r-1: move the ids other CTAs freed for this one into its rings
    // (the top warps do it; pairs go to the low threads first)
    if (r > 1 && mail_any) {
      const uint32_t ma = lane < G ? min(inbox[((r - 1) % 3) * 32 + 2 * lane + 1].x, kMbox) : 0u;
      const uint32_t mv = lane < G ? min(inbox[((r - 1) % 3) * 32 + 2 * lane + 1].y, kMbox) : 0u;
      const uint32_t ta = __reduce_add_sync(0xFFFFFFFFu, ma), tv = __reduce_add_sync(0xFFFFFFFFu, mv);
      const uint32_t* pm = mbox + ((r - 1) & 1u) * 2 * 16 * kMbox;
      const uint32_t nw = kBlock / 32;
      // only the warps that copy need the per-source offsets
      uint32_t xa = 0, xv = 0, dummy;
      if ((nw - 1 - warp) * 32 < ta + tv) {
        xa = warp_excl_scan(ma, lane, dummy);
        xv = warp_excl_scan(mv, lane, dummy);
      }
      for (uint32_t eb = (nw - 1 - warp) * 32; eb < ta + tv; eb += kBlock) {
        const uint32_t e = eb + lane;
        const bool is_a = e < ta;
        const uint32_t q = is_a ? e : e - ta;
        uint32_t j = 0;
#pragma unroll
        for (uint32_t step = 8; step; step >>= 1) {
          const uint32_t cand = j + step;
          const uint32_t ea = __shfl_sync(0xFFFFFFFFu, xa, cand & 31u);
          const uint32_t ev = __shfl_sync(0xFFFFFFFFu, xv, cand & 31u);
          if (cand < G && (is_a ? ea : ev) <= q) j = cand;
        }
        const uint32_t eja = __shfl_sync(0xFFFFFFFFu, xa, j), ejv = __shfl_sync(0xFFFFFFFFu, xv, j);
        const uint32_t ej = is_a ? eja : ejv;
        if (e < ta + tv) {
          const uint32_t id = pm[(is_a ? 0u : 16u * kMbox) + j * kMbox + (q - ej)];
          if (is_a) {
            const uint32_t pos = atomicAdd(&ctl->fpos_a, 1u);
            c.aring[pos & c.amask] = id;
            atomicAdd(&cur->afree, 1u);
          } else {
            lslots[id >> c.gshift] = kNone;  // the variable died last round; its slot is ours to clear
            const uint32_t pos = atomicAdd(&ctl->fpos_v, 1u);
            c.vring[pos & c.vmask] = id;
            atomicAdd(&cur->vfree, 1u);
          }
        }
      }
    }
    if (INET_EXACT_CODE && r > 1 && sh.exact) {
      // this CTA's equations merged last round that are still var-headed
      const uint32_t nd = ctr3[(r - 1) % 3].dcount;
      const uint2* din = d.deferred + (((r - 1) & 1u) * G + rank) * c.cap_def;
      for (uint32_t i = threadIdx.x; i < nd && !c.failed; i += kBlock) {
        const uint2 eq = din[i];
        c.parked -= 1;
        link(c, eq.x, eq.y);
      }
    }
    if (r == 1) {
      // the input equations, in any class (communication_phase's first pass)
      for (uint32_t mb = threadIdx.x & ~31u; rank + G * mb < N; mb += kBlock) {
        const uint32_t i = rank + G * (mb + lane);
        const bool v = i < N && !c.failed;
        const uint2 eq = v ? d.in_eqs[i] : make_uint2(0, 0);
        const bool act = v && ((eq.x | eq.y) & kVar) == 0;
        interact_w(c, act, eq.x, eq.y);
        if (v && !act && !c.failed) {
          if (d.resume) c.parked -= 1;  // a handed-over deferred equation was counted live
          link(c, eq.x, eq.y);
        }
      }
    } else {
      // this CTA's pairs: producer j dealt it n_j of them, in slots [0, n_j) of queue j
      const uint2* in = lqueue + ((r - 1) & 1u) * 16 * cap_q;
      for (uint32_t mb = threadIdx.x & ~31u; mb < N; mb += kBlock) {
        const uint32_t i = mb + lane;
        // segment j of global index i: the last j with excl_j <= i
        uint32_t j = 0;
#pragma unroll
        for (uint32_t step = 8; step; step >>= 1) {
          const uint32_t cand = j + step;
          const uint32_t e = __shfl_sync(0xFFFFFFFFu, excl, cand & 31u);
          if (cand < G && e <= i) j = cand;
        }
        const uint32_t ej = __shfl_sync(0xFFFFFFFFu, excl, j);
        const bool v = i < N && !c.failed;
#ifdef INET_TRACE
        c.tr[6] = c.tr[7] = 0;
#endif
        INET_TR(c, 0);
        const uint2 e = v ? in[j * cap_q + (i - ej)] : make_uint2(0, 0);
        interact_w(c, v, e.x, e.y);
        if (v) {
#ifdef INET_TRACE
          {
            const long long t6 = clock64();
            if (r >= INET_TRACE_R0 && r < INET_TRACE_R0 + 2 && ((threadIdx.x & 31u) == 0 || (c.tr[6] != 0)) &&
                atomicAdd(&inet_trace_count, 1u) < 1200u)
              printf("TR r=%u k=%u t=%u q+ag=%lld pair=%lld alloc=%lld recs+ex+wr+free=%lld push=%lld settle=%lld recs=%lld exissue=%lld\n",
                     r, rank, threadIdx.x, c.tr[2] - c.tr[0], c.tr[2] - c.tr[1], c.tr[3] - c.tr[2], c.tr[4] - c.tr[3],
                     c.tr[5] - c.tr[4], t6 - c.tr[5], c.tr[6] - c.tr[3], c.tr[7] - c.tr[6]);
          }
#endif
        }
      }
    }
    CT_MARK(1);
    if (per_round) {
      const uint32_t wi = __reduce_add_sync(0xFFFFFFFFu, c.ints);
      const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, c.comms);
      const int32_t wp = __reduce_add_sync(0xFFFFFFFFu, c.parked);
      if (lane == 0) {
        if (wi) atomicAdd(&cur->ints, wi);
        if (wc) atomicAdd(&cur->comms, wc);
        if (wp) atomicAdd(&cur->parked, wp);
      }
    }
    // every CTA pushes its round counters into every CTA's inbox
    __syncthreads();
#if INET_EXACT_CODE
    if (threadIdx.x == 0 && cur->dcount > c.cap_def) {  // deferred buffer overflowed
      if (atomicCAS(&ctl->err_code, 0u, static_cast<uint32_t>(INET_ERR_ARENA)) == 0u) ctl->err_a = 3;
      atomicOr(&cur->qcount, kErrBit);
    }
    __syncthreads();
#endif
    if (threadIdx.x < G) {
      const uint32_t k = threadIdx.x;
      uint4* dst = &inbox[(r % 3) * 32 + 2 * rank];
      dsmem_st4(dst, k, make_uint4(cur->qcount, cur->ints, cur->comms, static_cast<uint32_t>(cur->parked)));
      dsmem_st4(dst + 1, k, make_uint4(c.outc[k], c.outc[16 + k], cur->dcount, cur->vh));
    }
    CT_MARK(2);
    cluster_barrier();
    CT_MARK(3);
    // ---- round r is closed on every CTA: its counters are in the local inbox
    uint4 w = make_uint4(0, 0, 0, 0);
    if (lane < G) w = inbox[(r % 3) * 32 + 2 * lane];
    const bool err_any = __any_sync(0xFFFFFFFFu, (w.x & kErrBit) != 0);
    w.x &= ~kErrBit;
    const uint32_t total = __reduce_add_sync(0xFFFFFFFFu, w.x);  // pairs queued cluster-wide
    const uint4 w2 = lane < G ? inbox[(r % 3) * 32 + 2 * lane + 1] : make_uint4(0, 0, 0, 0);
    const bool deferred_any = __any_sync(0xFFFFFFFFu, w2.z != 0);
    mail_any = __any_sync(0xFFFFFFFFu, (w2.x | w2.y) != 0);  // mail for this CTA, moved next round
    const bool vh_any = sh.detect_vh && __any_sync(0xFFFFFFFFu, w2.w != 0);
    // pairs producer `lane` dealt to this CTA: its p-th went to CTA (p + lane) mod G
    uint32_t mine;
    {
      const uint32_t dd = (rank - lane) & (G - 1);
      const uint32_t nj = lane < G && w.x > dd ? ((w.x - dd - 1) >> c.gshift) + 1 : 0u;
      excl = warp_excl_scan(nj, lane, mine);
    }
    {
      // ids freed to this CTA in round r become allocatable (nothing is dropped)
      const uint32_t atake = cur->atake, afree = cur->afree, vtake = cur->vtake, vfree = cur->vfree;
      lo_a += min(atake, hi_a - lo_a);
      hi_a += afree;
      lo_v += min(vtake, hi_v - lo_v);
      hi_v += vfree;
    }
    if (rank == 0 && warp == 0) {
      const uint32_t ri = __reduce_add_sync(0xFFFFFFFFu, w.y);
      const uint32_t rc = __reduce_add_sync(0xFFFFFFFFu, w.z);
      const int32_t rp = __reduce_add_sync(0xFFFFFFFFu, static_cast<int32_t>(w.w));
      if (lane == 0) {
        tot_i += ri;
        tot_c += rc;
        parked_tot += rp;
        if (per_round) {
#ifdef INET_NO_TIMER
          const unsigned long long now = 0;
#else
          const unsigned long long now = globaltimer();
#endif
          if (rb + r - 1 < d.cap_rounds)
            d.stats[rb + r - 1] = make_uint4(ri, rc, total + static_cast<uint32_t>(parked_tot),
                                             static_cast<uint32_t>(now - t_prev));
          t_prev = now;
          if (!err_any && total == 0 && !deferred_any && rb + r < d.cap_rounds)
            d.stats[rb + r] = make_uint4(0, 0, static_cast<uint32_t>(parked_tot), 0);
        }
      }
    }
    CT_MARK(0);
    rounds = r + 1;
    N = mine;
    if (err_any) {
      stop = true;
    } else if (vh_any) {
      stop = true;  // the host reruns the net with reference-loop code
      stop_err = kNeedExact;
    } else if (rb + r + 1 > sh.max_rounds) {  // engine.py:205-207 (the no-op loop too)
      stop = true;
      stop_err = INET_ERR_LOOP_CAP;
    } else if (total == 0 && !deferred_any) {
      stop = true;  // the trailing no-op loop the reference records (engine.py:222-223)
    }
  }
#ifdef INET_CTIMING
  if (threadIdx.x == 0 && d.rule_hist)
    for (int i = 0; i < 4; ++i)
      atomicAdd(reinterpret_cast<unsigned long long*>(d.rule_hist) + 32 + i, ct_sum[i]);
#endif
  if (!per_round) {  // this CTA's totals (ctl->tot_* are unused by the loop of this tier)
    const uint32_t wi = __reduce_add_sync(0xFFFFFFFFu, c.ints);
    const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, c.comms);
    const int32_t wp = __reduce_add_sync(0xFFFFFFFFu, c.parked);
    if (lane == 0) {
      if (wi) atomicAdd(&ctl->tot_i, static_cast<unsigned long long>(wi));
      if (wc) atomicAdd(&ctl->tot_c, static_cast<unsigned long long>(wc));
      if (wp) atomicAdd(&ctl->parked_total, wp);
    }
  }
  // ---- results. High-water marks of the interleaved id spaces.
  uint32_t a_hw = d.n_in_agents, v_hw = d.n_in_vars;
  uint32_t e_code = 0, e_a = 0, e_b = 0;
  if (lane < G) {
    const uint32_t ab = dsmem_ld(&ctl->agent_bump, lane), vb = dsmem_ld(&ctl->var_bump, lane);
    if (ab) a_hw = max(a_hw, lane + G * (min(ab, c.cap_agents) - 1) + 1);
    if (vb) v_hw = max(v_hw, lane + G * (min(vb, c.cap_vars) - 1) + 1);
    e_code = dsmem_ld(&ctl->err_code, lane);
    e_a = dsmem_ld(&ctl->err_a, lane);
    e_b = dsmem_ld(&ctl->err_b, lane);
  }
  a_hw = min(__reduce_max_sync(0xFFFFFFFFu, a_hw), d.cap_agents);
  v_hw = min(__reduce_max_sync(0xFFFFFFFFu, v_hw), d.cap_vars);
  const uint32_t e_mask = __ballot_sync(0xFFFFFFFFu, e_code != 0);
  const uint32_t e_src = e_mask ? __ffs(e_mask) - 1 : 0;
  e_code = __shfl_sync(0xFFFFFFFFu, e_code, e_src);
  e_a = __shfl_sync(0xFFFFFFFFu, e_a, e_src);
  e_b = __shfl_sync(0xFFFFFFFFu, e_b, e_src);
  // variables that died in the last round and were mailed here: clear their slots
  if (!stop_err && rounds >= 2) {
    const uint32_t rl = rounds - 1;
    const uint32_t* pm = mbox + (rl & 1u) * 2 * 16 * kMbox + 16 * kMbox;
    for (uint32_t e = threadIdx.x; e < 16 * kMbox; e += kBlock) {
      const uint32_t src = e / kMbox, q = e % kMbox;
      if (src < G && q < min(inbox[(rl % 3) * 32 + 2 * src + 1].y, kMbox)) lslots[pm[e] >> c.gshift] = kNone;
    }
    __syncthreads();
  }
  // write this CTA's share of the agents and slots back to the global arrays
  {
    const uint32_t na = min(ctl->agent_bump, c.cap_agents), nv = min(ctl->var_bump, c.cap_vars);
    for (uint32_t i = threadIdx.x; i < na; i += kBlock) d.agents[rank + G * i] = lagents[i];
    for (uint32_t i = threadIdx.x; i < nv; i += kBlock) d.vslot[rank + G * i] = lslots[i];
    // ids below the high-water mark that this CTA never handed out read as free
    const uint32_t nv_hw = owned_below(v_hw);
    for (uint32_t i = nv + threadIdx.x; i < nv_hw; i += kBlock) d.vslot[rank + G * i] = kNone;
  }
  cluster_barrier();
  // residual parked equations in variable-id order: CTA k compacts slice k
  const uint32_t s_lo = static_cast<uint32_t>(uint64_t(v_hw) * rank / G);
  const uint32_t s_hi = static_cast<uint32_t>(uint64_t(v_hw) * (rank + 1) / G);
  uint32_t mine = 0;
  for (uint32_t x = s_lo + threadIdx.x; x < s_hi; x += kBlock) mine += d.vslot[x] != kNone;
  mine = __reduce_add_sync(0xFFFFFFFFu, mine);
  if (threadIdx.x == 0) ctl->scratch[33] = 0;
  __syncthreads();
  if (lane == 0 && mine) atomicAdd(&ctl->scratch[33], mine);
  cluster_barrier();
  uint32_t n_res;
  {
    const uint32_t cnt = lane < G ? dsmem_ld(&ctl->scratch[33], lane) : 0;
    const uint32_t ex = warp_excl_scan(cnt, lane, n_res);
    uint32_t base = __shfl_sync(0xFFFFFFFFu, ex, rank);
    for (uint32_t c0 = s_lo; c0 < s_hi; c0 += kBlock) {
      const uint32_t x = c0 + threadIdx.x;
      const uint32_t v = x < s_hi ? d.vslot[x] : kNone;
      uint32_t off;
      const uint32_t tot = block_scan_flag(v != kNone, ctl->scratch, &off);
      if (v != kNone && base + off < d.cap_vars) d.residual[base + off] = make_uint2(kVar | x, v);
      base += tot;
    }
  }
  if (writer && !per_round) {
    for (uint32_t k = 0; k < G; ++k) {
      const uint32_t* ti = reinterpret_cast<const uint32_t*>(&ctl->tot_i);
      const uint32_t* tc = reinterpret_cast<const uint32_t*>(&ctl->tot_c);
      tot_i += dsmem_ld(ti, k) | (static_cast<unsigned long long>(dsmem_ld(ti + 1, k)) << 32);
      tot_c += dsmem_ld(tc, k) | (static_cast<unsigned long long>(dsmem_ld(tc + 1, k)) << 32);
      parked_tot += static_cast<int32_t>(dsmem_ld(&ctl->parked_total, k));
    }
  }
  if (writer) {
    NetCtl* g = d.ctl;
    g->agent_bump = a_hw;
    g->var_bump = v_hw;
    g->err = stop_err ? stop_err : e_code;
    g->err_a = stop_err ? 0 : e_a;
    g->err_b = stop_err ? 0 : e_b;
    g->rounds = rb + rounds;
    g->interactions = tot_i;
    g->communications = tot_c;
    g->n_residual = n_res;
    g->parked_total = static_cast<uint32_t>(parked_tot);
    g->pad[0] = clock_mhz(clk0, gt0);
  }
  cluster_barrier();  // no CTA leaves while another may still read its shared memory
}

// Kernel body of tier C: cluster i reduces net i.
template <int kBlock>
__device__ __forceinline__ void reduce_cluster_body(const NetDesc* __restrict__ nets, uint32_t n_nets,
                                                    const uint32_t* __restrict__ blob, const Shape& sh,
                                                    uint32_t* smem, NetDesc& sd) {
  for (uint32_t i = threadIdx.x; i < sh.rule_words; i += kBlock) smem[i] = blob[4 + i];
  const uint32_t pair_words = (sh.n_labels * sh.n_labels + 1) / 2;
  const uint16_t* pair = reinterpret_cast<const uint16_t*>(smem);
  const uint32_t* rules = smem + pair_words;
  const uint32_t net = cluster_index();
  if (threadIdx.x == 0 && net < n_nets) sd = nets[net];
  __syncthreads();
  if (net < n_nets) run_net_cluster<kBlock>(sd, sh, pair, rules, smem);
}


// ---------------------------------------------------------------------------
// Tier X: one net reduced by the whole GPU. Nets too large for a cluster's
// shared memory (wide L-system nets: 10^5-10^6 redexes per round) keep the
// single-CTA tier G's global-memory layout, but every CTA of a cooperative
// grid takes a slice of each round; the round counters, free rings and bump
// pointers are global (warp-aggregated atomics), and a grid barrier closes
// the round (its gpu-scope fence also invalidates L1, so agents and queue
// words written by other SMs in the round are read fresh from L2).

__device__ __forceinline__ void grid_barrier(GridState* g) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t gen = *reinterpret_cast<volatile uint32_t*>(&g->bar_gen);
    __threadfence();
    if (atomicAdd(&g->bar_count, 1u) == gridDim.x - 1) {
      g->bar_count = 0;
      __threadfence();
      atomicAdd(&g->bar_gen, 1u);
    } else {
      while (*reinterpret_cast<volatile uint32_t*>(&g->bar_gen) == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

template <int kBlock>
__device__ void run_net_grid(const NetDesc& d, const Shape& sh, const uint16_t* pair, const uint32_t* rules,
                             uint32_t* smem) {
  constexpr int kTier = kTierX;
  GridState* const g = d.gs;
  Ctl* const ctl = &g->ctl;
  Round<kTier> c;
  c.d = &d;
  c.ctl = ctl;
  c.aring = d.g_aring;
  c.vring = d.g_vring;
  c.amask = sh.ring_a - 1;
  c.vmask = sh.ring_v - 1;
  c.pair = pair;
  c.rules = rules;
  c.n_labels = sh.n_labels;
  c.agents = d.agents;
  c.vslot = d.vslot;
  c.cap_agents = d.cap_agents;
  c.cap_vars = d.cap_vars;
  c.cap_queue = d.cap_queue;
  c.cap_def = d.cap_def;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t gtid = blockIdx.x * kBlock + threadIdx.x, gthreads = gridDim.x * kBlock;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  const long long clk0 = clock64();
  const unsigned long long gt0 = globaltimer();
  const bool fits = d.n_in_agents <= c.cap_agents && d.n_in_vars <= c.cap_vars;
  // ---- init (the host zeroed the grid state)
  for (uint32_t i = gtid; i < c.cap_vars; i += gthreads) c.vslot[i] = kNone;
  if (fits)
    for (uint32_t i = gtid; i < d.n_in_agents; i += gthreads) c.agents[i] = d.in_agents[i];
  if (lead) {
    ctl->agent_bump = d.n_in_agents;
    ctl->var_bump = d.n_in_vars;
  }
  bool stop = false;
  uint32_t stop_err = 0;
  if (!fits) {
    stop = true;
    stop_err = INET_ERR_ARENA;
  } else if (sh.max_rounds == 0) {
    stop = true;
    stop_err = INET_ERR_LOOP_CAP;
  } else if (d.n_in_eqs == 0) {
    stop = true;
    if (lead && d.stats && d.cap_rounds) d.stats[0] = make_uint4(0, 0, 0, 0);
  }
  __shared__ uint32_t red3[3];
  __shared__ uint32_t scan_scratch[34];
  grid_barrier(g);
  c.failed = false;
#if INET_STAMPS
  c.stamps = nullptr;  // (single-CTA tiers only)
  c.round = c.cid = 0;
#endif
  uint32_t lo_a = 0, hi_a = 0, lo_v = 0, hi_v = 0, n = d.n_in_eqs, rounds = 1;
  int32_t parked_tot = 0;
  unsigned long long tot_i = 0, tot_c = 0, t_prev = globaltimer();
  uint2* const Q = d.queue;
  // per-round totals only for the per-round rows (every block's atomics on
  // three global counters each round otherwise)
  const bool per_round = INET_ROWS && d.stats != nullptr;
  c.ints = c.comms = 0;
  c.parked = 0;
  for (uint32_t r = 1; !stop; ++r) {
    RoundCtr* cur = &g->ctr3[r % 3];
    c.cur = cur;
    c.lo_a = lo_a;
    c.hi_a = hi_a;
    c.lo_v = lo_v;
    c.hi_v = hi_v;
    if (per_round) {
      c.ints = c.comms = 0;
      c.parked = 0;
    }
    c.dout = nullptr;
    c.out = Q + (r & 1u) * c.cap_queue;
    if (blockIdx.x == 0 && threadIdx.x < sizeof(RoundCtr) / 4)
      reinterpret_cast<uint32_t*>(&g->ctr3[(r + 1) % 3])[threadIdx.x] = 0;
    if (threadIdx.x < 3) red3[threadIdx.x] = 0;
    if (r == 1) {
      for (uint32_t b = gtid & ~31u; b < n; b += gthreads) {
        const uint32_t i = b + lane;
        const bool v = i < n && !c.failed;
        const uint2 eq = v ? d.in_eqs[i] : make_uint2(0, 0);
        const bool act = v && ((eq.x | eq.y) & kVar) == 0;
        interact_w(c, act, eq.x, eq.y);
        if (v && !act && !c.failed) link(c, eq.x, eq.y);
      }
    } else {
      const uint2* in = Q + ((r - 1) & 1u) * c.cap_queue;
      for (uint32_t b = gtid & ~31u; b < n; b += gthreads) {
        const uint32_t i = b + lane;
        const bool v = i < n && !c.failed;
        const uint2 e = v ? in[i] : make_uint2(0, 0);
        interact_w(c, v, e.x, e.y);
      }
    }
    if (per_round) {
      const uint32_t wi = __reduce_add_sync(0xFFFFFFFFu, c.ints);
      const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, c.comms);
      const int32_t wp = __reduce_add_sync(0xFFFFFFFFu, c.parked);
      __syncthreads();  // red3 cleared
      if (lane == 0) {
        if (wi) atomicAdd(&red3[0], wi);
        if (wc) atomicAdd(&red3[1], wc);
        if (wp) atomicAdd(&red3[2], static_cast<uint32_t>(wp));
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        if (red3[0]) atomicAdd(&cur->ints, red3[0]);
        if (red3[1]) atomicAdd(&cur->comms, red3[1]);
        if (red3[2]) atomicAdd(&cur->parked, static_cast<int32_t>(red3[2]));
      }
    }
    grid_barrier(g);
    // ---- close round r (every thread, same values)
    const RoundCtr k = *cur;
    const bool round_failed = (k.qcount & kErrBit) != 0;
    const uint32_t q = k.qcount & ~kErrBit;
    const uint32_t wa = min(k.afree, sh.ring_a - (hi_a - lo_a));
    const uint32_t wv = min(k.vfree, sh.ring_v - (hi_v - lo_v));
    lo_a += min(k.atake, hi_a - lo_a);
    hi_a += wa;
    lo_v += min(k.vtake, hi_v - lo_v);
    hi_v += wv;
    parked_tot += k.parked;
    tot_i += k.ints;
    tot_c += k.comms;
    if (per_round && lead) {
      const unsigned long long now = globaltimer();
      if (r - 1 < d.cap_rounds)
        d.stats[r - 1] = make_uint4(k.ints, k.comms, q + static_cast<uint32_t>(parked_tot),
                                    static_cast<uint32_t>(now - t_prev));
      t_prev = now;
    }
    rounds = r + 1;
    n = q;
    if (round_failed) {
      stop = true;
    } else if (sh.detect_vh && k.vh) {
      stop = true;
      stop_err = kNeedExact;
    } else if (r + 1 > sh.max_rounds) {  // engine.py:205-207 (the no-op loop too)
      stop = true;
      stop_err = INET_ERR_LOOP_CAP;
    } else if (q == 0) {
      stop = true;
      if (per_round && lead && r < d.cap_rounds) d.stats[r] = make_uint4(0, 0, static_cast<uint32_t>(parked_tot), 0);
    } else if (q > c.cap_queue) {
      stop = true;
      stop_err = INET_ERR_ARENA;
    }
  }
  if (lead && stop_err) atomicCAS(&ctl->err_code, 0u, stop_err);
  if (!per_round) {  // the run's totals, once
    const uint32_t wi = __reduce_add_sync(0xFFFFFFFFu, c.ints);
    const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, c.comms);
    const int32_t wp = __reduce_add_sync(0xFFFFFFFFu, c.parked);
    if (lane == 0) {
      if (wi) atomicAdd(&ctl->tot_i, static_cast<unsigned long long>(wi));
      if (wc) atomicAdd(&ctl->tot_c, static_cast<unsigned long long>(wc));
      if (wp) atomicAdd(&ctl->parked_total, wp);
    }
  }
  grid_barrier(g);
  if (!per_round) {  // (L2 reads: the atomics bypassed this SM's L1)
    tot_i = __ldcg(&ctl->tot_i);
    tot_c = __ldcg(&ctl->tot_c);
    parked_tot = __ldcg(&ctl->parked_total);
  }
  // ---- results: residual parked equations in variable-id order (two passes)
  const uint32_t v_hw = min(ctl->var_bump, c.cap_vars), a_hw = min(ctl->agent_bump, c.cap_agents);
  const uint32_t per = (v_hw + gridDim.x - 1) / gridDim.x;
  const uint32_t s_lo = min(blockIdx.x * per, v_hw), s_hi = min(s_lo + per, v_hw);
  uint32_t mine = 0;
  for (uint32_t x = s_lo + threadIdx.x; x < s_hi; x += kBlock) mine += c.vslot[x] != kNone;
  mine = __reduce_add_sync(0xFFFFFFFFu, mine);
  if (threadIdx.x == 0) red3[0] = 0;
  __syncthreads();
  if (lane == 0 && mine) atomicAdd(&red3[0], mine);
  __syncthreads();
  if (threadIdx.x == 0) g->blk_res[blockIdx.x] = red3[0];
  grid_barrier(g);
  uint32_t base = 0, n_res = 0;
  for (uint32_t b = threadIdx.x; b < gridDim.x; b += kBlock) {
    const uint32_t v = g->blk_res[b];
    n_res += v;
    if (b < blockIdx.x) base += v;
  }
  // block-wide sums of base / n_res
  base = __reduce_add_sync(0xFFFFFFFFu, base);
  n_res = __reduce_add_sync(0xFFFFFFFFu, n_res);
  __shared__ uint32_t sums[2][32];
  if (lane == 0) {
    sums[0][warp] = base;
    sums[1][warp] = n_res;
  }
  __syncthreads();
  base = 0;
  n_res = 0;
  for (uint32_t w = 0; w < kBlock / 32; ++w) {
    base += sums[0][w];
    n_res += sums[1][w];
  }
  __syncthreads();
  for (uint32_t c0 = s_lo; c0 < s_hi; c0 += kBlock) {
    const uint32_t x = c0 + threadIdx.x;
    const uint32_t v = x < s_hi ? c.vslot[x] : kNone;
    uint32_t off;
    const uint32_t tot = block_scan_flag(v != kNone, scan_scratch, &off);
    if (v != kNone && base + off < d.cap_vars) d.residual[base + off] = make_uint2(kVar | x, v);
    base += tot;
  }
  if (lead) {
    NetCtl* o = d.ctl;
    o->agent_bump = a_hw;
    o->var_bump = v_hw;
    o->err = ctl->err_code;
    o->err_a = ctl->err_a;
    o->err_b = ctl->err_b;
    o->rounds = rounds;
    o->interactions = tot_i;
    o->communications = tot_c;
    o->n_residual = n_res;
    o->parked_total = static_cast<uint32_t>(parked_tot);
    o->pad[0] = clock_mhz(clk0, gt0);
    if ((ctl->agent_bump > d.cap_agents || ctl->var_bump > d.cap_vars) && o->err == 0) o->err = INET_ERR_ARENA;
    o->pad[1] = 0;  // (set by the host after a device-side finalize)
    o->pad[2] = 0;
    g->fin_lo_a = lo_a;  // for the device-side finalize (finalize.cuh)
    g->fin_hi_a = hi_a;
  }
}

template <int kBlock>
__device__ __forceinline__ void reduce_grid_body(const NetDesc* __restrict__ nets, uint32_t n_nets,
                                                 const uint32_t* __restrict__ blob, const Shape& sh, uint32_t* smem,
                                                 NetDesc& sd) {
  for (uint32_t i = threadIdx.x; i < sh.rule_words; i += kBlock) smem[i] = blob[4 + i];
  const uint32_t pair_words = (sh.n_labels * sh.n_labels + 1) / 2;
  const uint16_t* pair = reinterpret_cast<const uint16_t*>(smem);
  const uint32_t* rules = smem + pair_words;
  if (threadIdx.x == 0) sd = nets[0];
  __syncthreads();
  if (n_nets >= 1) run_net_grid<kBlock>(sd, sh, pair, rules, smem);
}

}  // namespace inetdev
