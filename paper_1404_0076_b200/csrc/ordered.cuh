// ordered.cuh — tier R: the reference's evaluation order on the device.
//
// The fast tiers (device.cuh) link variables by exchanges on a slot table, so
// the order in which two equations meet is the order of arrival. Everything
// the reference *counts* is schedule-free (uniform confluence) except where
// its own list order decides: which variable keys a var = var equation (the
// smaller id, engine.py:150-153) — and with it the loop in which a merge
// happens, total_communications and the LoopStats rows —, the orientation of
// a merged pair (engine.py:161-165), the first failing pair of a loop
// (engine.py:88-92) and, through the order of the residual equations, where
// finalize cuts a cyclic normal form (engine.py:313-355).
//
// Tier R keeps the reference's equation list itself, in its order, and runs
// each loop exactly as engine.py:106-166 defines it:
//
//   interaction  every active entry i of E_L is rewritten; its fresh variables
//                get the reference's ids base + i * max_fresh + j (engine.py:93,
//                122), kept per variable as a 64-bit `refid`; the outputs go,
//                in list order, to three streams — agent=agent (P, the next
//                list's head), parked singles whose key is unchanged (A, still
//                sorted from the previous loop) and everything else (B);
//   communication  B is normalised (var left, smaller refid left) and stably
//                sorted by key refid (rank counting in shared memory for a
//                small stream, an LSD radix sort otherwise); A and B are
//                merged by (key, list position) along a merge path (each
//                thread walks its chunk of A); runs of equal keys fold as
//                reduce_by_key does (a run x=t, x=u -> t = u; longer runs keep
//                the last two right-hand sides, like the reference's fold);
//   next list    P ++ folded runs.
//
// Every phase is block-wide (one CTA per net, global memory arrays, L2
// resident), deterministic, and ordered by block scans over contiguous
// per-thread chunks, so agent and variable ids are reproducible too. The
// residual list handed to the host finalize is the reference's final list,
// same order and orientation, so even cyclic normal forms print identically.
// With `sh.validate` the name discipline (engine.py:169-183) is checked after
// both phases of every loop, on the device.
#pragma once
#include "device.cuh"

namespace inetdev {

constexpr int kTierR = 5;
constexpr uint32_t kRPos = 8;  // list position p of output k of entry i: i * kRPos + k (k < INET_MAX_EQ)

// Per-net tier R arrays, carved from one buffer (host and device agree on the layout).
struct RArrays {
  unsigned long long* refid;    // [V]  reference id of each device variable
  uint32_t* aring;              // [ra] free agent ids (power of two)
  uint32_t* vring;              // [rv] free variable ids
  uint2* E[2];                  // [Lc] the equation list, double-buffered
  uint8_t* F[2];                // [Lc] 1: an unmerged single of the last communication (key unchanged)
  unsigned long long* akey;     // [Lc] stream A: key refid, list position, equation
  uint32_t* apos;
  uint2* aeq;
  unsigned long long* bkey[2];  // [Oc] stream B, double-buffered for the radix sort
  uint32_t* bpos[2];
  uint2* beq[2];
  unsigned long long* skey;     // [Lc + Oc] the sorted eligible equations
  uint2* seq;
  uint32_t* vcount;             // [V] name discipline (validate)
  uint8_t* alive;               // [A] live agents (validate)
};

__host__ __device__ inline uint32_t pow2_at_least(uint32_t x) {
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

__host__ __device__ inline size_t r_align(size_t b) { return (b + 255) & ~size_t(255); }

// Carve the per-net buffer (base may be null: returns the byte count).
__host__ __device__ inline size_t r_carve(uint8_t* base, uint32_t A, uint32_t V, uint32_t Lc, uint32_t Oc, RArrays* out) {
  size_t off = 0;
  auto take = [&](size_t bytes) -> uint8_t* {
    uint8_t* p = base ? base + off : nullptr;
    off += r_align(bytes);
    return p;
  };
  RArrays r;
  r.refid = reinterpret_cast<unsigned long long*>(take(size_t(V) * 8));
  r.aring = reinterpret_cast<uint32_t*>(take(size_t(pow2_at_least(A)) * 4));
  r.vring = reinterpret_cast<uint32_t*>(take(size_t(pow2_at_least(V)) * 4));
  for (int k = 0; k < 2; ++k) {
    r.E[k] = reinterpret_cast<uint2*>(take(size_t(Lc) * 8));
    r.F[k] = take(Lc);
  }
  r.akey = reinterpret_cast<unsigned long long*>(take(size_t(Lc) * 8));
  r.apos = reinterpret_cast<uint32_t*>(take(size_t(Lc) * 4));
  r.aeq = reinterpret_cast<uint2*>(take(size_t(Lc) * 8));
  for (int k = 0; k < 2; ++k) {
    r.bkey[k] = reinterpret_cast<unsigned long long*>(take(size_t(Oc) * 8));
    r.bpos[k] = reinterpret_cast<uint32_t*>(take(size_t(Oc) * 4));
    r.beq[k] = reinterpret_cast<uint2*>(take(size_t(Oc) * 8));
  }
  r.skey = reinterpret_cast<unsigned long long*>(take((size_t(Lc) + Oc) * 8));
  r.seq = reinterpret_cast<uint2*>(take((size_t(Lc) + Oc) * 8));
  r.vcount = reinterpret_cast<uint32_t*>(take(size_t(V) * 4));
  r.alive = take(A);
  if (out) *out = r;
  return off;
}

// Block-wide exclusive scan of K counters per thread (blockDim a multiple of
// 32). v becomes the exclusive prefix, tot the block totals. sm: K * 33 words.
template <int K>
__device__ __forceinline__ void block_scan_k(uint32_t (&v)[K], uint32_t (&tot)[K], uint32_t* sm) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t inc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    inc[k] = v[k];
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, inc[k], o);
      if (lane >= o) inc[k] += t;
    }
  }
  if (lane == 31)
#pragma unroll
    for (int k = 0; k < K; ++k) sm[k * 32 + warp] = inc[k];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint32_t w0 = lane < nw ? sm[k * 32 + lane] : 0u;
      uint32_t w = w0;
#pragma unroll
      for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, w, o);
        if (lane >= o) w += t;
      }
      sm[k * 32 + lane] = w - w0;
      if (lane == 31) sm[K * 32 + k] = w;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    v[k] = inc[k] - v[k] + sm[k * 32 + warp];
    tot[k] = sm[K * 32 + k];
  }
  __syncthreads();
}

__device__ __forceinline__ void chunk_of(uint32_t n, uint32_t& lo, uint32_t& hi) {
  const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
  lo = min(n, threadIdx.x * per);
  hi = min(n, lo + per);
}

__device__ __forceinline__ bool r_is_var(uint32_t t) { return (t & kVar) != 0; }

constexpr uint32_t kSmallB = 256;  // stream B sorted in shared memory up to this size
constexpr uint32_t kRB = 4;        // list entries whose loads are batched (interaction passes)
constexpr uint32_t kRW = 8;        // sorted keys a thread prefetches for the fold

// Shared state of the running loop (one copy per CTA).
struct RShared {
  uint32_t scan[8 * 33 + 8];
  unsigned long long kmin, kmax;
  uint32_t err_i;                // first failing active entry (NoRuleForPair)
  unsigned long long bad_var;    // smallest refid occurring more than twice (validate)
  uint32_t flag;
  // a small stream B, sorted in shared memory
  unsigned long long sb_key[kSmallB];
  uint32_t sb_pos[kSmallB];
  uint2 sb_eq[kSmallB];
};

// Source k of a rule template -> term ref (include/inet_b200.h source coding).
struct RRewrite {
  uint4 A, B;
  uint32_t l, r;
  uint32_t fresh[INET_MAX_FRESH];
  uint32_t extra[INET_MAX_NEW];
  __device__ __forceinline__ uint32_t src(uint32_t s) const {
    if (s < 3) return s == 0 ? A.y : (s == 1 ? A.z : A.w);
    if (s < 6) return s == 3 ? B.y : (s == 4 ? B.z : B.w);
    if (s < 14) return fresh[s - kEnvFresh];
    if (s < 22) {
      const uint32_t m = s - kEnvNew;
      return m == 0 ? l : (m == 1 ? r : extra[m - 2]);
    }
    return kNone;
  }
  // Is source s an agent? (before the ids are known: new agents always are)
  __device__ __forceinline__ bool src_is_agent(uint32_t s) const {
    if (s < 6) return !r_is_var(s < 3 ? (s == 0 ? A.y : (s == 1 ? A.z : A.w)) : (s == 3 ? B.y : (s == 4 ? B.z : B.w)));
    if (s < 14) return false;
    return s < 22;
  }
};

// Normalise a var-headed equation as communication_phase does (engine.py:147-159):
// var left; var = var with the smaller reference id left. Returns the key refid.
__device__ __forceinline__ unsigned long long r_normalise(const RArrays& R, uint2& e) {
  const bool lv = r_is_var(e.x), rv = r_is_var(e.y);
  if (lv && rv) {
    const unsigned long long a = R.refid[e.x & ~kVar], b = R.refid[e.y & ~kVar];
    if (b < a) {
      e = make_uint2(e.y, e.x);
      return b;
    }
    return a;
  }
  if (!lv) e = make_uint2(e.y, e.x);
  return R.refid[e.x & ~kVar];
}

// Sort a small stream B (n <= kSmallB) into shared memory: each item's rank is
// the number of items with a smaller key, or an equal key earlier in the
// stream (B is written in list order, so this is the stable order).
__device__ void r_sort_small(const RArrays& R, uint32_t n, RShared& S) {
  unsigned long long k = 0;
  uint32_t p = 0;
  uint2 e = make_uint2(0, 0);
  const uint32_t b = threadIdx.x;
  if (b < n) {
    k = R.bkey[0][b];
    p = R.bpos[0][b];
    e = R.beq[0][b];
    S.sb_key[b] = k;
  }
  __syncthreads();
  uint32_t rank = 0;
  if (b < n)
    for (uint32_t j = 0; j < n; ++j) {
      const unsigned long long kj = S.sb_key[j];
      rank += kj < k || (kj == k && j < b);
    }
  __syncthreads();
  if (b < n) {
    S.sb_key[rank] = k;
    S.sb_pos[rank] = p;
    S.sb_eq[rank] = e;
  }
  __syncthreads();
}

// Stable LSD radix sort of stream B by key (4-bit digits over the key range).
// Returns the buffer index holding the sorted stream.
__device__ int r_sort_b(const RArrays& R, uint32_t n, RShared& S, uint32_t* hist) {
  if (n < 2) return 0;
  unsigned long long lo = ~0ull, hi = 0;
  uint32_t a, b;
  chunk_of(n, a, b);
  for (uint32_t i = a; i < b; ++i) {
    const unsigned long long k = R.bkey[0][i];
    lo = min(lo, k);
    hi = max(hi, k);
  }
  if (threadIdx.x == 0) {
    S.kmin = ~0ull;
    S.kmax = 0;
  }
  __syncthreads();
  if (b > a) {
    atomicMin(&S.kmin, lo);
    atomicMax(&S.kmax, hi);
  }
  __syncthreads();
  const unsigned long long kmin = S.kmin, span = S.kmax - S.kmin;
  const uint32_t bits = span ? 64 - __clzll(static_cast<long long>(span)) : 0;
  int cur = 0;
  const uint32_t T = blockDim.x;
  for (uint32_t sh = 0; sh < bits; sh += 4) {
    for (uint32_t j = threadIdx.x; j < 16 * T; j += T) hist[j] = 0;
    __syncthreads();
    for (uint32_t i = a; i < b; ++i) hist[((R.bkey[cur][i] - kmin) >> sh & 15u) * T + threadIdx.x] += 1;
    __syncthreads();
    // exclusive scan of hist (digit-major, thread-minor): 16 consecutive words per thread
    uint32_t v[1] = {0}, tot[1];
    for (uint32_t j = 0; j < 16; ++j) v[0] += hist[threadIdx.x * 16 + j];
    block_scan_k<1>(v, tot, S.scan);
    uint32_t run = v[0];
    for (uint32_t j = 0; j < 16; ++j) {
      const uint32_t w = hist[threadIdx.x * 16 + j];
      hist[threadIdx.x * 16 + j] = run;
      run += w;
    }
    __syncthreads();
    for (uint32_t i = a; i < b; ++i) {
      const unsigned long long k = R.bkey[cur][i];
      const uint32_t dst = hist[((k - kmin) >> sh & 15u) * T + threadIdx.x]++;
      R.bkey[cur ^ 1][dst] = k;
      R.bpos[cur ^ 1][dst] = R.bpos[cur][i];
      R.beq[cur ^ 1][dst] = R.beq[cur][i];
    }
    __syncthreads();
    cur ^= 1;
  }
  return cur;
}

// Number of items of a (key, pos)-sorted array strictly before (k, p).
__device__ __forceinline__ uint32_t r_rank(const unsigned long long* key, const uint32_t* pos, uint32_t n,
                                           unsigned long long k, uint32_t p) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const unsigned long long km = key[mid];
    if (km < k || (km == k && pos[mid] < p))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// Name discipline over the whole net: interface, list sides and every live
// agent's ports (each live agent sits in exactly one term). Sets S.bad_var to
// the smallest refid of a variable occurring more than twice.
__device__ void r_check_names(const NetDesc& d, const RArrays& R, RShared& S, const uint2* E, uint32_t nE,
                              const uint2* extra, uint32_t n_extra, const uint2* extra2, uint32_t n_extra2,
                              uint32_t n_vars, uint32_t n_agents) {
  for (uint32_t x = threadIdx.x; x < n_vars; x += blockDim.x) R.vcount[x] = 0;
  __syncthreads();
  auto count = [&](uint32_t t) {
    if (t != kNone && r_is_var(t)) atomicAdd(&R.vcount[t & ~kVar], 1u);
  };
  for (uint32_t i = threadIdx.x; i < d.n_iface; i += blockDim.x) count(d.in_iface[i]);
  for (uint32_t i = threadIdx.x; i < nE; i += blockDim.x) {
    count(E[i].x);
    count(E[i].y);
  }
  for (uint32_t i = threadIdx.x; i < n_extra; i += blockDim.x) {
    count(extra[i].x);
    count(extra[i].y);
  }
  for (uint32_t i = threadIdx.x; i < n_extra2; i += blockDim.x) {
    count(extra2[i].x);
    count(extra2[i].y);
  }
  for (uint32_t a = threadIdx.x; a < n_agents; a += blockDim.x)
    if (R.alive[a]) {
      const uint4 g = d.agents[a];
      count(g.y);
      count(g.z);
      count(g.w);
    }
  __syncthreads();
  for (uint32_t x = threadIdx.x; x < n_vars; x += blockDim.x)
    if (R.vcount[x] > 2) atomicMin(&S.bad_var, R.refid[x]);
  __syncthreads();
}

#ifdef INET_RTIMING
// Development build: clock64 per phase of a tier R loop, thread 0's view
// (after each phase's barrier), summed into the rule-histogram area
// (tools/rtier_timing.py).
#define RT_MARK(k)                       \
  do {                                   \
    if (threadIdx.x == 0) {              \
      const long long _t = clock64();    \
      rt[k] += _t - rt_last;             \
      rt_last = _t;                      \
    }                                    \
  } while (0)
#else
#define RT_MARK(k) \
  do {             \
  } while (0)
#endif

// Reduce one net in the reference's order (see the file comment).
__device__ void run_net_ordered(const NetDesc& d, const Shape& sh, uint32_t net, const uint16_t* pair,
                                const uint32_t* rules, uint32_t* hist, RShared& S) {
  RArrays R;
  r_carve(sh.rbuf + net * sh.rbuf_stride, d.cap_agents, d.cap_vars, sh.cap_list, sh.cap_out, &R);
  const uint32_t T = blockDim.x;
  const uint32_t A = d.cap_agents, V = d.cap_vars, Lc = sh.cap_list, Oc = sh.cap_out;
  const uint32_t amask = pow2_at_least(A) - 1, vmask = pow2_at_least(V) - 1;
  const long long clk0 = clock64();
  const unsigned long long gt0 = globaltimer();
  uint32_t err = 0, err_a = 0, err_b = 0;
  if (d.n_in_agents > A || d.n_in_vars > V || d.n_in_eqs > Lc) err = INET_ERR_ARENA;
  if (!err) {
    for (uint32_t i = threadIdx.x; i < d.n_in_agents; i += T) d.agents[i] = d.in_agents[i];
    for (uint32_t i = threadIdx.x; i < d.n_in_vars; i += T) R.refid[i] = i;  // input ids keep their order
    for (uint32_t i = threadIdx.x; i < d.n_in_eqs; i += T) {
      R.E[0][i] = d.in_eqs[i];
      R.F[0][i] = 0;
    }
    if (sh.validate)
      for (uint32_t i = threadIdx.x; i < A; i += T) R.alive[i] = i < d.n_in_agents;
  }
  __syncthreads();
  uint32_t nE = d.n_in_eqs, cur = 0;
  uint32_t agent_bump = d.n_in_agents, var_bump = d.n_in_vars;
  uint32_t lo_a = 0, hi_a = 0, lo_v = 0, hi_v = 0;  // ring windows (positions, mod size)
  unsigned long long base = d.n_in_vars;              // fresh refids start after the input ids
  unsigned long long tot_i = 0, tot_c = 0;
  uint32_t loop = 0;
  unsigned long long t_prev = gt0;
  const uint32_t max_fresh = sh.max_fresh;
#ifdef INET_RTIMING
  long long rt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, rt_last = clock64();
#endif
  while (!err) {
    loop += 1;
    if (loop > sh.max_rounds) {  // engine.py:205-207, before every loop
      err = INET_ERR_LOOP_CAP;
      break;
    }
    const uint2* E = R.E[cur];
    const uint8_t* F = R.F[cur];
    uint2* En = R.E[cur ^ 1];
    uint8_t* Fn = R.F[cur ^ 1];
    if (threadIdx.x == 0) {
      S.err_i = INET_NONE;
      S.bad_var = ~0ull;
    }
    __syncthreads();
    // ---- interaction, pass 1: per-thread counts of every output stream
    uint32_t lo, hi;
    chunk_of(nE, lo, hi);
    // 0 P outputs, 1 A outputs, 2 B outputs, 3 agents taken, 4 agents freed, 5 variables taken, 6 active
    uint32_t cnt[7] = {0, 0, 0, 0, 0, 0, 0};
    // entries are processed in batches of kRB whose loads are all issued before
    // any is used: one L2 round trip per batch instead of one per entry
    for (uint32_t i0 = lo; i0 < hi; i0 += kRB) {
      uint2 ev[kRB];
      uint8_t fv[kRB];
      uint4 av[kRB], bv[kRB];
#pragma unroll
      for (uint32_t k = 0; k < kRB; ++k) {
        ev[k] = i0 + k < hi ? E[i0 + k] : make_uint2(kVar, kVar);
        fv[k] = i0 + k < hi ? F[i0 + k] : 0;
      }
#pragma unroll
      for (uint32_t k = 0; k < kRB; ++k) {
        const bool act = !r_is_var(ev[k].x) && !r_is_var(ev[k].y);
        av[k] = act ? d.agents[ev[k].x] : make_uint4(0, 0, 0, 0);
        bv[k] = act ? d.agents[ev[k].y] : make_uint4(0, 0, 0, 0);
      }
      bool failed = false;
#pragma unroll
      for (uint32_t k = 0; k < kRB; ++k) {
        const uint32_t i = i0 + k;
        if (i >= hi || failed) continue;
        const uint2 e = ev[k];
        if (r_is_var(e.x) || r_is_var(e.y)) {
          cnt[fv[k] ? 1 : 2] += 1;
          continue;
        }
        RRewrite w;
        w.A = av[k];
        w.B = bv[k];
        const uint32_t t = pair[w.A.x * sh.n_labels + w.B.x];
        if (t == 0xFFFFu) {
          atomicMin(&S.err_i, i);
          failed = true;  // later entries of this chunk cannot be the first failure
          continue;
        }
        if (t & 1u) {
          const uint4 tmp = w.A;
          w.A = w.B;
          w.B = tmp;
        }
        const uint32_t* Rr = rules + (t >> 1) * kRuleWords;
        const uint32_t hdr = Rr[0];
        const uint32_t nn = hdr & 0xFFu, ne = (hdr >> 8) & 0xFFu, nf = (hdr >> 16) & 0xFFu;
        for (uint32_t q = 0; q < ne; ++q) {
          const uint32_t h = (Rr[9 + (q >> 1)] >> ((q & 1) * 16)) & 0xFFFFu;
          const bool act = w.src_is_agent(h & 0xFFu) && w.src_is_agent(h >> 8);
          cnt[act ? 0 : 2] += 1;
        }
        cnt[3] += nn > 2 ? nn - 2 : 0;
        cnt[4] += nn < 2 ? 2 - nn : 0;
        cnt[5] += nf;
        cnt[6] += 1;
      }
      if (failed) break;
    }
    uint32_t off[7], tot[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) off[k] = cnt[k];
    block_scan_k<7>(off, tot, S.scan);
    if (S.err_i != INET_NONE) {  // find_rule raised on the first failing entry (engine.py:88-92)
      const uint2 e = E[S.err_i];
      err = INET_ERR_NO_RULE;
      err_a = d.agents[e.x].x;
      err_b = d.agents[e.y].x;
      break;
    }
    RT_MARK(0);
    const uint32_t nP = tot[0], nA = tot[1], nB = tot[2], n_act = tot[6];
    const uint32_t av_a = hi_a - lo_a, av_v = hi_v - lo_v;
    const uint32_t bump_a = tot[3] > av_a ? tot[3] - av_a : 0u, bump_v = tot[5] > av_v ? tot[5] - av_v : 0u;
    if (nP > Lc || nA > Lc || nB > Oc || agent_bump + bump_a > A || var_bump + bump_v > V) {
      err = INET_ERR_ARENA;
      break;
    }
    // ---- interaction, pass 2: rewrite in list order, emit the three streams
    for (uint32_t i0 = lo; i0 < hi; i0 += kRB) {
      uint2 ev[kRB];
      uint8_t fv[kRB];
      uint4 av[kRB], bv[kRB];
      unsigned long long kv[kRB];
#pragma unroll
      for (uint32_t k = 0; k < kRB; ++k) {
        ev[k] = i0 + k < hi ? E[i0 + k] : make_uint2(kVar, kVar);
        fv[k] = i0 + k < hi ? F[i0 + k] : 0;
      }
#pragma unroll
      for (uint32_t k = 0; k < kRB; ++k) {
        const bool act = !r_is_var(ev[k].x) && !r_is_var(ev[k].y);
        av[k] = act ? d.agents[ev[k].x] : make_uint4(0, 0, 0, 0);
        bv[k] = act ? d.agents[ev[k].y] : make_uint4(0, 0, 0, 0);
        // a parked single keeps its key (normalised last loop: var left)
        kv[k] = !act && fv[k] && i0 + k < hi ? R.refid[ev[k].x & ~kVar] : 0ull;
      }
#pragma unroll
      for (uint32_t k = 0; k < kRB; ++k) {
        const uint32_t i = i0 + k;
        if (i >= hi) continue;
        uint2 e = ev[k];
        const uint32_t opos = i * kRPos;
        if (r_is_var(e.x) || r_is_var(e.y)) {
          if (fv[k]) {
            R.aeq[off[1]] = e;
            R.akey[off[1]] = kv[k];
            R.apos[off[1]] = opos;
            off[1] += 1;
          } else {
            const unsigned long long key = r_normalise(R, e);
            R.beq[0][off[2]] = e;
            R.bkey[0][off[2]] = key;
            R.bpos[0][off[2]] = opos;
            off[2] += 1;
          }
          continue;
        }
        RRewrite w;
        w.l = e.x;
        w.r = e.y;
        w.A = av[k];
        w.B = bv[k];
        const uint32_t t = pair[w.A.x * sh.n_labels + w.B.x];
        if (t & 1u) {  // orient as the rule's pattern (core.py:287-298)
          const uint4 tmp = w.A;
          w.A = w.B;
          w.B = tmp;
          w.l = e.y;
          w.r = e.x;
        }
#if INET_COUNT_RULES
        if (d.rule_hist) atomicAdd(&d.rule_hist[t >> 1], 1u);
#endif
        const uint32_t* Rr = rules + (t >> 1) * kRuleWords;
        const uint32_t hdr = Rr[0];
        const uint32_t nn = hdr & 0xFFu, ne = (hdr >> 8) & 0xFFu, nf = (hdr >> 16) & 0xFFu;
        for (uint32_t j = 0; j < nf; ++j) {  // fresh ids: base + i * max_fresh + j (engine.py:93)
          const uint32_t q = off[5] + j;
          const uint32_t x = q < av_v ? R.vring[(lo_v + q) & vmask] : var_bump + (q - av_v);
          R.refid[x] = base + static_cast<unsigned long long>(i) * max_fresh + j;
          w.fresh[j] = kVar | x;
        }
        off[5] += nf;
        for (uint32_t m = 2; m < nn; ++m) {
          const uint32_t q = off[3] + (m - 2);
          w.extra[m - 2] = q < av_a ? R.aring[(lo_a + q) & amask] : agent_bump + (q - av_a);
          if (sh.validate) R.alive[w.extra[m - 2]] = 1;
        }
        off[3] += nn > 2 ? nn - 2 : 0;
        for (uint32_t m = 0; m < nn; ++m) {
          const uint32_t tw = Rr[1 + m];
          d.agents[w.src(kEnvNew + m)] =
              make_uint4(tw & 0xFFu, w.src((tw >> 8) & 0xFFu), w.src((tw >> 16) & 0xFFu), w.src(tw >> 24));
        }
        for (uint32_t m = nn; m < 2; ++m) {  // consumed agents not reused in place
          const uint32_t a = m == 0 ? w.l : w.r;
          R.aring[(hi_a + off[4]) & amask] = a;
          off[4] += 1;
          if (sh.validate) R.alive[a] = 0;
        }
        for (uint32_t q = 0; q < ne; ++q) {
          const uint32_t h = (Rr[9 + (q >> 1)] >> ((q & 1) * 16)) & 0xFFFFu;
          uint2 o = make_uint2(w.src(h & 0xFFu), w.src(h >> 8));
          if (!r_is_var(o.x) && !r_is_var(o.y)) {
            En[off[0]] = o;
            off[0] += 1;
          } else {
            const unsigned long long key = r_normalise(R, o);
            R.beq[0][off[2]] = o;
            R.bkey[0][off[2]] = key;
            R.bpos[0][off[2]] = opos + q;
            off[2] += 1;
          }
        }
      }
    }
    __syncthreads();
    RT_MARK(1);
    base += static_cast<unsigned long long>(nE) * max_fresh;  // reserve(len(eqs) * max_fresh), engine.py:122
    agent_bump += bump_a;
    var_bump += bump_v;
    const uint32_t took_a = min(tot[3], av_a), took_v = min(tot[5], av_v);
    lo_a += took_a;
    hi_a += tot[4];
    lo_v += took_v;
    if (sh.validate) {  // after the interaction phase (engine.py:210-211)
      r_check_names(d, R, S, En, nP, R.aeq, nA, R.beq[0], nB, var_bump, agent_bump);
      if (S.bad_var != ~0ull) {
        err = INET_ERR_NAME;
        err_a = static_cast<uint32_t>(S.bad_var);
        err_b = static_cast<uint32_t>(S.bad_var >> 32);
        break;
      }
    }
    // ---- communication: sort B by key (stable), merge with A, fold runs
    const unsigned long long* bk;
    const uint32_t* bp;
    const uint2* be;
    if (nB <= kSmallB && T >= kSmallB) {
      r_sort_small(R, nB, S);
      bk = S.sb_key;
      bp = S.sb_pos;
      be = S.sb_eq;
    } else {
      const int sb = r_sort_b(R, nB, S, hist);
      bk = R.bkey[sb];
      bp = R.bpos[sb];
      be = R.beq[sb];
    }
    RT_MARK(2);
    // merge path: thread t merges its chunk of A with the B items that sort
    // before the chunk's end (A is sorted from the last loop, keys unique)
    chunk_of(nA, lo, hi);
    if (nA == 0) {
      for (uint32_t b = threadIdx.x; b < nB; b += T) {
        R.skey[b] = bk[b];
        R.seq[b] = be[b];
      }
    } else if (lo < hi) {
      const uint32_t jb = lo == 0 ? 0u : r_rank(bk, bp, nB, R.akey[lo], R.apos[lo]);
      const uint32_t je = hi == nA ? nB : r_rank(bk, bp, nB, R.akey[hi], R.apos[hi]);
      uint32_t i = lo, j = jb;
      unsigned long long ka = R.akey[i];
      uint32_t pa = R.apos[i];
      while (i < hi || j < je) {
        bool take_b = j < je;
        if (take_b && i < hi) take_b = bk[j] < ka || (bk[j] == ka && bp[j] < pa);
        if (take_b) {
          R.skey[i + j] = bk[j];
          R.seq[i + j] = be[j];
          ++j;
        } else {
          R.skey[i + j] = ka;
          R.seq[i + j] = R.aeq[i];
          ++i;
          if (i < hi) {
            ka = R.akey[i];
            pa = R.apos[i];
          }
        }
      }
    }
    __syncthreads();
    RT_MARK(3);
    const uint32_t nS = nA + nB;
    chunk_of(nS, lo, hi);
    // this chunk's keys and their neighbours, loaded once (a run of equal keys is
    // at most a few long: a neighbour past the window is read directly)
    unsigned long long kw[kRW + 2];
#pragma unroll
    for (uint32_t k = 0; k < kRW + 2; ++k) {
      const uint32_t p = lo + k - 1;  // kw[k] = skey[lo - 1 + k]
      kw[k] = (lo + k >= 1 && p < nS && lo + k <= hi + 1 && k < kRW + 2) ? R.skey[p] : ~0ull;
    }
    const uint32_t n_kw = min(kRW + 2, hi - lo + 2);  // kw[0, n_kw) hold skey[lo - 1, lo - 1 + n_kw)
    auto key_at = [&](uint32_t p) -> unsigned long long {
      const uint32_t k = p + 1 - lo;
      return p + 1 >= lo && k < n_kw ? kw[k] : R.skey[p];
    };
    uint32_t c2[2] = {0, 0};  // 0 runs, 1 variables freed
    for (uint32_t p = lo; p < hi; ++p)
      if (p == 0 || key_at(p - 1) != key_at(p)) {
        c2[0] += 1;
        c2[1] += p + 1 < nS && key_at(p + 1) == key_at(p);
      }
    uint32_t t2[2];
    block_scan_k<2>(c2, t2, S.scan);
    const uint32_t runs = t2[0];
    if (nP + runs > Lc) {
      err = INET_ERR_ARENA;
      break;
    }
    for (uint32_t p = lo; p < hi; ++p) {
      if (p != 0 && key_at(p - 1) == key_at(p)) continue;
      uint32_t q = p + 1;
      while (q < nS && key_at(q) == key_at(p)) ++q;
      const uint32_t out = nP + c2[0];
      c2[0] += 1;
      if (q - p == 1) {
        En[out] = R.seq[p];
        Fn[out] = 1;
      } else {
        // reduce_by_key's fold of merge(a, b) = Equation(a.rhs, b.rhs) (engine.py:161-165)
        En[out] = make_uint2(R.seq[q - 2].y, R.seq[q - 1].y);
        Fn[out] = 0;
        R.vring[(hi_v + c2[1]) & vmask] = R.seq[p].x & ~kVar;  // the key variable is consumed
        c2[1] += 1;
      }
    }
    for (uint32_t i = threadIdx.x; i < nP; i += T) Fn[i] = 0;
    __syncthreads();
    RT_MARK(4);
    hi_v += t2[1];
    const uint32_t comms = nS - runs;
    nE = nP + runs;
    cur ^= 1;
    tot_i += n_act;
    tot_c += comms;
    if (sh.validate) {  // after the communication phase (engine.py:213-214)
      r_check_names(d, R, S, R.E[cur], nE, nullptr, 0, nullptr, 0, var_bump, agent_bump);
      if (S.bad_var != ~0ull) {
        err = INET_ERR_NAME;
        err_a = static_cast<uint32_t>(S.bad_var);
        err_b = static_cast<uint32_t>(S.bad_var >> 32);
        break;
      }
    }
    if (threadIdx.x == 0 && d.stats && loop - 1 < d.cap_rounds) {
      const unsigned long long now = globaltimer();
      d.stats[loop - 1] = make_uint4(n_act, comms, nE, static_cast<uint32_t>(min(now - t_prev, 0xFFFFFFFFull)));
      t_prev = now;
    }
    RT_MARK(5);
    if (n_act == 0 && comms == 0) break;  // engine.py:222-223
  }
#ifdef INET_RTIMING
  if (threadIdx.x == 0 && d.rule_hist)
    for (int k = 0; k < 8; ++k)
      atomicAdd(reinterpret_cast<unsigned long long*>(d.rule_hist) + 32 + k, static_cast<unsigned long long>(rt[k]));
#endif
  __syncthreads();
  // ---- results: the final list is the residual input of finalize, in order
  const bool fits = nE <= V;
  if (!err && fits)
    for (uint32_t i = threadIdx.x; i < nE; i += T) d.residual[i] = R.E[cur][i];
  if (threadIdx.x == 0) {
    NetCtl* g = d.ctl;
    g->agent_bump = agent_bump;
    g->var_bump = var_bump;
    g->err = err ? err : (fits ? 0u : static_cast<uint32_t>(INET_ERR_ARENA));
    g->err_a = err_a;
    g->err_b = err_b;
    g->rounds = loop;
    g->interactions = tot_i;
    g->communications = tot_c;
    g->n_residual = nE;
    g->parked_total = nE;
    g->pad[0] = clock_mhz(clk0, gt0);
    g->pad[1] = 0;
    g->pad[2] = 0;
  }
  __syncthreads();
}

template <int kBlock>
__device__ __forceinline__ void reduce_ordered_body(const NetDesc* __restrict__ nets, uint32_t n_nets,
                                                    const uint32_t* __restrict__ blob, const Shape& sh, uint32_t* smem,
                                                    NetDesc& sd, RShared& S) {
  for (uint32_t i = threadIdx.x; i < sh.rule_words; i += kBlock) smem[i] = blob[4 + i];
  const uint32_t pair_words = (sh.n_labels * sh.n_labels + 1) / 2;
  const uint16_t* pair = reinterpret_cast<const uint16_t*>(smem);
  const uint32_t* rules = smem + pair_words;
  uint32_t* hist = smem + align4(sh.rule_words);  // 16 * kBlock words
  for (uint32_t net = blockIdx.x; net < n_nets; net += gridDim.x) {
    __syncthreads();
    if (threadIdx.x == 0) sd = nets[net];
    __syncthreads();
    run_net_ordered(sd, sh, net, pair, rules, hist, S);
  }
}

}  // namespace inetdev
