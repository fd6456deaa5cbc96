// finalize.cuh — device-side finalize of a net reduced on the whole GPU (tier X).
//
// The reference finishes with a sequential pass (engine.finalize,
// src/inet/engine.py:287-362): every parked equation x = t is eliminated by
// splicing t into x's other occurrence. For a normal form that is a forest
// hanging off the interface, that is exactly: replace each variable whose
// parked value is known by that value (following var-valued chains), then
// lay the trees out in preorder from the interface roots (port 0 first) — the
// host's finalize_walk (host.cpp) does it with one sequential DFS, which for a
// wide net (lsystem(26): 376K agents, 196K parked equations) costs more than
// the reduction itself. Here it is data-parallel:
//
//   resolve   every live agent's ports through the parked values (each parked
//             equation may be consumed once) and claim each agent child's
//             parent slot (a child claimed twice is a shared subterm);
//   check     every parked equation consumed, every live agent has a parent;
//   tour      Euler tour of the forest: down-edge D(c) -> D(first child) or
//             U(c); up-edge U(c) -> D(next sibling) or U(parent); roots are
//             chained in interface order;
//   rank      Wyllie pointer jumping gives each edge the number of down-edges
//             from it to the end; preorder(c) = total - rank(D(c)); a cycle
//             (agents whose parent chain never reaches a root) shows up as a
//             total below the live count;
//   write     records in preorder with agent ports renumbered, and the
//             resolved interface.
//
// Anything outside that shape (a cycle, a shared agent, an equation left
// over) sets the failure flag and the host finalizes from the arena as before.
#pragma once
#include "device.cuh"

namespace inetfin {

using inetdev::kNone;
using inetdev::kVar;
constexpr uint32_t kRootBit = 0x80000000u;  // parent word: kRootBit | interface index, else (agent << 2) | port
constexpr uint32_t kEnd = 0xFFFFFFFFu;

struct FinArgs {
  const uint4* agents;  // arena [0, n)
  uint32_t n;
  const uint2* resid;   // parked equations (VAR | x, t)
  uint32_t m;
  const uint32_t* iface;
  uint32_t ni;
  uint32_t nv;          // variable ids < nv
  const uint32_t* ring;  // free agent ring: entries [lo, hi) are dead agents
  uint32_t ring_mask, lo, hi;
  uint32_t* val;        // [nv] parked value of x
  uint32_t* used;       // [nv] 1 once consumed
  uint32_t* dead;       // [n]
  uint32_t* parent;     // [n]
  uint4* res;           // [n] resolved records
  uint32_t* res_iface;  // [ni]
  unsigned long long* rk[2];  // [2n] (rank << 32) | next edge
  uint4* out;           // [n] preorder records
  uint32_t* out_iface;  // [ni]
  uint32_t* flag;       // [0] failure, [1] live agents
};

__device__ __forceinline__ void fail(const FinArgs& f) { atomicOr(&f.flag[0], 1u); }

__device__ __forceinline__ uint32_t resolve(const FinArgs& f, uint32_t t) {
  for (uint32_t guard = 0; t != kNone && (t & kVar) && guard <= f.m; ++guard) {
    const uint32_t x = t & ~kVar;
    if (x >= f.nv) break;
    const uint32_t w = f.val[x];
    if (w == kNone) break;
    if (atomicExch(&f.used[x], 1u) != 0u) {  // a parked equation spliced twice: not a forest
      fail(f);
      return kNone;
    }
    t = w;
  }
  return t;
}

__global__ void fin_init(FinArgs f) {
  const uint32_t N = max(f.n, f.nv);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    if (i < f.nv) {
      f.val[i] = kNone;
      f.used[i] = 0;
    }
    if (i < f.n) {
      f.dead[i] = 0;
      f.parent[i] = kNone;
    }
  }
}

__global__ void fin_mark(FinArgs f) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t q = f.lo + blockIdx.x * blockDim.x + threadIdx.x; q - f.lo < f.hi - f.lo; q += stride) {
    const uint32_t a = f.ring[q & f.ring_mask];
    if (a < f.n) f.dead[a] = 1;
  }
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < f.m; e += stride) {
    const uint2 r = f.resid[e];
    const uint32_t x = r.x & ~kVar;
    if (!(r.x & kVar) || x >= f.nv) fail(f);
    else f.val[x] = r.y;
  }
}

__device__ __forceinline__ void claim(const FinArgs& f, uint32_t t, uint32_t who) {
  if (t == kNone || (t & kVar)) return;
  if (t >= f.n || f.dead[t] || atomicCAS(&f.parent[t], kNone, who) != kNone) fail(f);
}

__global__ void fin_resolve(FinArgs f) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t a = blockIdx.x * blockDim.x + threadIdx.x; a < f.n; a += stride) {
    if (f.dead[a]) continue;
    const uint4 g = f.agents[a];
    const uint4 r = make_uint4(g.x, resolve(f, g.y), resolve(f, g.z), resolve(f, g.w));
    f.res[a] = r;
    claim(f, r.y, (a << 2) | 0u);
    claim(f, r.z, (a << 2) | 1u);
    claim(f, r.w, (a << 2) | 2u);
    atomicAdd(&f.flag[1], 1u);
  }
  if (blockIdx.x == 0)
    for (uint32_t i = threadIdx.x; i < f.ni; i += blockDim.x) {
      const uint32_t t = resolve(f, f.iface[i]);
      f.res_iface[i] = t;
      claim(f, t, kRootBit | i);
    }
}

__device__ __forceinline__ uint32_t port(const uint4& r, uint32_t k) { return k == 0 ? r.y : (k == 1 ? r.z : r.w); }
__device__ __forceinline__ bool is_agent(uint32_t t) { return t != kNone && !(t & kVar); }

__global__ void fin_tour(FinArgs f) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < f.n; c += stride) {
    if (f.dead[c]) {
      f.rk[0][2 * c] = f.rk[0][2 * c + 1] = kEnd;
      continue;
    }
    if (f.parent[c] == kNone) fail(f);  // a live agent nothing points to
    const uint4 r = f.res[c];
    uint32_t fc = kNone;
    for (uint32_t k = 0; k < 3 && fc == kNone; ++k)
      if (is_agent(port(r, k))) fc = port(r, k);
    const uint32_t d_next = fc != kNone ? 2 * fc : 2 * c + 1;
    uint32_t u_next = kEnd;
    const uint32_t p = f.parent[c];
    if (p != kNone && (p & kRootBit)) {
      for (uint32_t i = (p & ~kRootBit) + 1; i < f.ni && u_next == kEnd; ++i)
        if (is_agent(f.res_iface[i])) u_next = 2 * f.res_iface[i];
    } else if (p != kNone) {
      const uint32_t a = p >> 2;
      const uint4 ra = f.res[a];
      for (uint32_t k = (p & 3u) + 1; k < 3 && u_next == kEnd; ++k)
        if (is_agent(port(ra, k))) u_next = 2 * port(ra, k);
      if (u_next == kEnd) u_next = 2 * a + 1;
    }
    f.rk[0][2 * c] = (1ull << 32) | d_next;
    f.rk[0][2 * c + 1] = u_next;
  }
}

__global__ void fin_unused(FinArgs f) {  // a parked equation the resolution never reached
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < f.nv; x += gridDim.x * blockDim.x)
    if (f.val[x] != kNone && !f.used[x]) fail(f);
}

// One pointer-jumping step: rank(e) += rank(next(e)), next(e) = next(next(e)).
__global__ void fin_jump(const unsigned long long* __restrict__ in, unsigned long long* __restrict__ out, uint32_t E) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const unsigned long long v = in[e];
    const uint32_t nx = static_cast<uint32_t>(v);
    if (nx == kEnd) {
      out[e] = v;
      continue;
    }
    const unsigned long long w = in[nx];
    out[e] = (((v >> 32) + (w >> 32)) << 32) | static_cast<uint32_t>(w);
  }
}

__global__ void fin_write(FinArgs f, const unsigned long long* __restrict__ rk) {
  uint32_t head = kEnd;  // the first interface root that is an agent starts the tour
  for (uint32_t i = 0; i < f.ni && head == kEnd; ++i)
    if (is_agent(f.res_iface[i])) head = f.res_iface[i];
  const uint32_t total = head == kEnd ? 0u : static_cast<uint32_t>(rk[2 * head] >> 32);
  if (blockIdx.x == 0 && threadIdx.x == 0 && total != f.flag[1]) fail(f);  // a cycle off the tour
  auto pre = [&](uint32_t t) -> uint32_t { return is_agent(t) ? total - static_cast<uint32_t>(rk[2 * t] >> 32) : t; };
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < f.n; c += stride) {
    if (f.dead[c]) continue;
    const uint32_t p = pre(c);
    if (p >= f.n) {
      fail(f);
      continue;
    }
    const uint4 r = f.res[c];
    f.out[p] = make_uint4(r.x, pre(r.y), pre(r.z), pre(r.w));
  }
  if (blockIdx.x == 0)
    for (uint32_t i = threadIdx.x; i < f.ni; i += blockDim.x) f.out_iface[i] = pre(f.res_iface[i]);
}

}  // namespace inetfin
