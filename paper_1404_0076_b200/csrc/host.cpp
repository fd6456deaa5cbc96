// host.cpp — sequential cleanup of a reduced net on flat arrays.
//
// finalize_flat restates engine.finalize (src/inet/engine.py:287-362): after
// the device loop stops, the remaining equations are parked var-headed
// equations whose variable's other occurrence is nested (inside an agent) or
// in the interface. Every such equation x = t is eliminated by writing t into
// the other occurrence of x, in the reference's queue order (equations in
// order; an equation whose top-level slot received a term is re-queued).
// An equation is kept when the other occurrence of x lies inside the
// equation itself (a cycle, or x = x).
//
// The reference decides "inside the equation itself" with a DFS of the other
// side (engine.py:275-284, 337). Here each agent carries the container it was
// found in and containers are merged with union-find when a term is spliced,
// so the test is O(alpha) instead of O(term size) and the whole pass is linear
// even for an 8,190-deep Ackermann(3,10) result chain in any order.
#include <new>
#include "host.h"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <sched.h>
#include <unordered_map>

namespace inethost {

namespace {

constexpr uint32_t kNone = INET_NONE;
constexpr uint32_t kVar = INET_VAR_BIT;

inline bool is_var(uint32_t r) { return r != kNone && (r & kVar); }

struct Finalizer {
  uint32_t* ag;  // 4 words per agent
  uint32_t na;
  uint32_t* ifc;
  uint32_t ni;
  uint32_t* eq;  // 2 words per equation
  uint32_t ne;
  uint32_t nv;
  // cells: [0,ni) interface, [ni, ni+2ne) equation sides, then 3 ports per agent
  std::vector<uint32_t> occ;     // 2 cells per variable
  std::vector<uint32_t> owner;   // container of each agent
  std::vector<uint32_t> parent;  // union-find over containers [0, ni+ne)
  std::vector<uint8_t> alive;
  std::vector<uint32_t> fifo;

  uint32_t eq_cell(uint32_t e, uint32_t s) const { return ni + 2 * e + s; }
  uint32_t port_cell(uint32_t a, uint32_t k) const { return ni + 2 * ne + 3 * a + k; }
  bool is_eq_cell(uint32_t c) const { return c >= ni && c < ni + 2 * ne; }
  bool is_port_cell(uint32_t c) const { return c >= ni + 2 * ne; }
  uint32_t& cell(uint32_t c) {
    if (c < ni) return ifc[c];
    if (c < ni + 2 * ne) return eq[c - ni];
    const uint32_t p = c - ni - 2 * ne;
    return ag[4 * (p / 3) + 1 + p % 3];
  }
  uint32_t find(uint32_t k) {
    while (parent[k] != k) {
      parent[k] = parent[parent[k]];
      k = parent[k];
    }
    return k;
  }
  uint32_t container_of(uint32_t c) {
    if (c < ni) return c;
    if (c < ni + 2 * ne) return ni + (c - ni) / 2;
    return find(owner[(c - ni - 2 * ne) / 3]);
  }

  // Record occurrences and owners below one root cell.
  std::vector<uint32_t> stack;  // scan work list, reused across roots

  int scan(uint32_t root_cell, uint32_t container) {
    stack.clear();
    stack.push_back(root_cell);
    while (!stack.empty()) {
      const uint32_t c = stack.back();
      stack.pop_back();
      const uint32_t t = cell(c);
      if (t == kNone) continue;
      if (t & kVar) {
        const uint32_t x = t & ~kVar;
        if (x >= nv) return INET_ERR_ARG;
        if (occ[2 * x] == kNone)
          occ[2 * x] = c;
        else if (occ[2 * x + 1] == kNone)
          occ[2 * x + 1] = c;
        else
          return INET_ERR_ARG;  // name discipline broken (NameDisciplineError)
        continue;
      }
      if (t >= na) return INET_ERR_ARG;
      if (owner[t] != kNone) return INET_ERR_ARG;  // shared agent: not a tree
      owner[t] = container;
      for (uint32_t k = 0; k < 3; ++k)
        if (ag[4 * t + 1 + k] != kNone) stack.push_back(port_cell(t, k));
    }
    return INET_OK;
  }

  int run() {
    occ.assign(size_t(nv) * 2, kNone);
    owner.assign(na, kNone);
    parent.resize(ni + ne);
    for (uint32_t k = 0; k < ni + ne; ++k) parent[k] = k;
    alive.assign(ne, 1);
    for (uint32_t i = 0; i < ni; ++i)
      if (int st = scan(i, i)) return st;
    for (uint32_t e = 0; e < ne; ++e)
      for (uint32_t s = 0; s < 2; ++s)
        if (int st = scan(eq_cell(e, s), ni + e)) return st;

    // FIFO of equations to visit (the reference's queue discipline)
    std::vector<uint32_t>& queue = fifo;
    queue.clear();
    for (uint32_t e = 0; e < ne; ++e) queue.push_back(e);
    for (size_t head = 0; head < queue.size();) {
      const uint32_t e = queue[head++];
      if (!alive[e]) continue;
      for (uint32_t side = 0; side < 2; ++side) {
        const uint32_t v = eq[2 * e + side];
        if (!is_var(v)) continue;
        const uint32_t x = v & ~kVar;
        const uint32_t self = eq_cell(e, side);
        uint32_t target = kNone;
        for (uint32_t j = 0; j < 2; ++j) {
          const uint32_t o = occ[2 * x + j];
          if (o == kNone || o == self) continue;
          if (is_eq_cell(o) && !alive[(o - ni) / 2]) continue;  // stale slot of a consumed equation
          target = o;
          break;
        }
        if (target == kNone) continue;
        // the other occurrence must not be inside this very equation
        if (target == eq_cell(e, 1 - side)) continue;
        if (is_port_cell(target) && container_of(target) == ni + e) continue;
        const uint32_t rep = eq[2 * e + 1 - side];
        alive[e] = 0;
        cell(target) = rep;
        if (is_var(rep)) {
          const uint32_t y = rep & ~kVar;
          for (uint32_t j = 0; j < 2; ++j)
            if (occ[2 * y + j] == eq_cell(e, 1 - side)) occ[2 * y + j] = target;
        } else {
          parent[ni + e] = container_of(target);
        }
        occ[2 * x] = occ[2 * x + 1] = kNone;
        if (is_eq_cell(target)) {
          const uint32_t f = (target - ni) / 2;
          if (alive[f]) queue.push_back(f);
        }
        break;
      }
    }
    return INET_OK;
  }
};

}  // namespace

int validate_rule_blob(const uint32_t* blob, size_t n_words) {
  if (blob[0] != INET_RULES_MAGIC) return INET_ERR_ARG;
  const uint32_t L = blob[1], R = blob[2];
  if (L == 0 || L > INET_MAX_LABELS || R > INET_MAX_RULES) return INET_ERR_UNSUPPORTED;
  const size_t pair_words = (size_t(L) * L + 1) / 2;
  if (n_words != 4 + pair_words + size_t(R) * 16) return INET_ERR_ARG;
  const uint16_t* pair = reinterpret_cast<const uint16_t*>(blob + 4);
  for (size_t i = 0; i < size_t(L) * L; ++i)
    if (pair[i] != 0xFFFFu && (pair[i] >> 1) >= R) return INET_ERR_ARG;
  const uint32_t* rules = blob + 4 + pair_words;
  for (uint32_t r = 0; r < R; ++r) {
    const uint32_t* w = rules + 16 * r;
    const uint32_t nn = w[0] & 0xFF, ne = (w[0] >> 8) & 0xFF, nf = (w[0] >> 16) & 0xFF;
    if (nn > INET_MAX_NEW || ne > INET_MAX_EQ || nf > INET_MAX_FRESH) return INET_ERR_UNSUPPORTED;
    auto src_ok = [&](uint32_t s) {
      if (s < 6) return true;
      if (s < 14) return s - 6 < nf;
      if (s < 22) return s - 14 < nn;
      return s == 22;
    };
    for (uint32_t m = 0; m < nn; ++m) {
      if ((w[1 + m] & 0xFF) >= L) return INET_ERR_ARG;
      for (int k = 1; k < 4; ++k)
        if (!src_ok((w[1 + m] >> (8 * k)) & 0xFF)) return INET_ERR_ARG;
    }
    for (uint32_t e = 0; e < ne; ++e) {
      const uint32_t h = (w[9 + e / 2] >> ((e & 1) * 16)) & 0xFFFF;
      if (!src_ok(h & 0xFF) || !src_ok(h >> 8) || (h & 0xFF) == 22 || (h >> 8) == 22) return INET_ERR_ARG;
    }
  }
  return INET_OK;
}

int finalize_flat(uint32_t* agents, uint32_t n_agents, uint32_t* iface, uint32_t n_iface, uint32_t* eqs,
                  uint32_t n_eqs, uint32_t n_vars, uint8_t* alive) {
  Finalizer f{};
  f.ag = agents;
  f.na = n_agents;
  f.ifc = iface;
  f.ni = n_iface;
  f.eq = eqs;
  f.ne = n_eqs;
  f.nv = n_vars;
  int st = f.run();
  if (st) return st;
  if (alive) std::copy(f.alive.begin(), f.alive.end(), alive);
  return INET_OK;
}

namespace {

// Fast path of finalize_net (the host twin of the device's finalize_smem):
// walk the net from the interface in preorder, replacing every variable whose
// parked equation is known by that equation's other side at the variable's
// other occurrence — where the reference's elimination writes it. When the
// walk consumes every parked equation and meets no agent twice, the result is
// the one the general pass produces (tests/test_gpu_finalize.py compares the
// two); otherwise return false and the general pass runs.
bool finalize_walk(const NetView& v, NormalForm& out, std::vector<uint32_t>& val, std::vector<uint32_t>& remap,
                   std::vector<uint32_t>& order, std::vector<uint32_t>& stack, std::vector<uint32_t>& ports) {
  constexpr uint32_t kUsed = 0xFFFFFFFEu;  // a parked equation already applied
  val.assign(v.n_vars, kNone);
  for (uint32_t e = 0; e < v.n_residual; ++e) {
    const uint32_t x = v.residual[2 * e], t = v.residual[2 * e + 1];
    if (!is_var(x) || (x & ~kVar) >= v.n_vars || t == kUsed || val[x & ~kVar] != kNone) return false;
    val[x & ~kVar] = t;
  }
  uint32_t consumed = 0;
  bool ok = true;
  auto resolve = [&](uint32_t t) {
    for (uint32_t guard = 0; is_var(t) && guard <= v.n_residual; ++guard) {
      const uint32_t x = t & ~kVar;
      if (x >= v.n_vars) {
        ok = false;
        break;
      }
      const uint32_t w = val[x];
      if (w == kNone) break;
      if (w == kUsed) {
        ok = false;
        break;
      }
      val[x] = kUsed;
      consumed += 1;
      t = w;
    }
    return t;
  };
  remap.assign(v.n_agents, kNone);
  order.clear();
  ports.clear();
  out.iface.resize(v.n_iface);
  for (uint32_t i = 0; i < v.n_iface && ok; ++i) {
    const uint32_t root = resolve(v.iface[i]);
    out.iface[i] = root;
    if (root == kNone || is_var(root)) continue;
    stack.clear();
    stack.push_back(root);
    while (!stack.empty() && ok) {
      const uint32_t a = stack.back();
      stack.pop_back();
      if (a >= v.n_agents || remap[a] != kNone) {
        ok = false;
        break;
      }
      remap[a] = static_cast<uint32_t>(order.size());
      order.push_back(a);
      const uint32_t* rec = v.agents + 4 * size_t(a);
      const uint32_t p0 = resolve(rec[1]), p1 = resolve(rec[2]), p2 = resolve(rec[3]);
      ports.push_back(p0);
      ports.push_back(p1);
      ports.push_back(p2);
      if (p2 != kNone && !is_var(p2)) stack.push_back(p2);
      if (p1 != kNone && !is_var(p1)) stack.push_back(p1);
      if (p0 != kNone && !is_var(p0)) stack.push_back(p0);
    }
  }
  if (!ok || consumed != v.n_residual) return false;
  auto map_ref = [&](uint32_t t) { return (t == kNone || is_var(t)) ? t : remap[t]; };
  out.agents.resize(order.size() * 4);
  for (size_t j = 0; j < order.size(); ++j) {
    out.agents[4 * j] = v.agents[4 * size_t(order[j])];
    for (int k = 0; k < 3; ++k) out.agents[4 * j + 1 + k] = map_ref(ports[3 * j + k]);
  }
  for (uint32_t i = 0; i < v.n_iface; ++i) out.iface[i] = map_ref(out.iface[i]);
  out.eqs.clear();
  return true;
}

}  // namespace

int finalize_net(const NetView& v, NormalForm& out) {
  // per-thread scratch, reused across the nets a worker finalizes (a batch of
  // 4096 nets would otherwise spend most of its time in the allocator)
  struct Scratch {
    std::vector<uint32_t> ag, ifc, eq, remap, order, stack;
    Finalizer f{};
  };
  thread_local Scratch sc;
  out.ext_agents = nullptr;
  out.ext_n = 0;
  // (INET_B200_HOSTWALK=0 forces the general pass: the tests compare the two)
  const char* walk_env = std::getenv("INET_B200_HOSTWALK");
  if ((!walk_env || std::atoi(walk_env) != 0) && finalize_walk(v, out, sc.remap, sc.order, sc.stack, sc.eq, sc.ifc))
    return INET_OK;
  std::vector<uint32_t>& ag = sc.ag;
  std::vector<uint32_t>& ifc = sc.ifc;
  std::vector<uint32_t>& eq = sc.eq;
  out.ext_agents = nullptr;
  out.ext_n = 0;
  ag.assign(v.agents, v.agents + size_t(v.n_agents) * 4);
  ifc.assign(v.iface, v.iface + v.n_iface);
  eq.assign(v.residual, v.residual + size_t(v.n_residual) * 2);
  Finalizer& f = sc.f;
  f.ag = ag.data();
  f.na = v.n_agents;
  f.ifc = ifc.data();
  f.ni = v.n_iface;
  f.eq = eq.data();
  f.ne = v.n_residual;
  f.nv = v.n_vars;
  int st = f.run();
  if (st) return st;
  // compact the reachable normal form in preorder
  std::vector<uint32_t>& remap = sc.remap;
  std::vector<uint32_t>& order = sc.order;
  std::vector<uint32_t>& stack = sc.stack;
  remap.assign(v.n_agents, kNone);
  order.clear();
  stack.clear();
  auto visit = [&](uint32_t root) {
    if (root == kNone || (root & kVar)) return;
    stack.push_back(root);
    while (!stack.empty()) {
      const uint32_t a = stack.back();
      stack.pop_back();
      remap[a] = static_cast<uint32_t>(order.size());
      order.push_back(a);
      for (int k = 2; k >= 0; --k) {
        const uint32_t t = ag[4 * a + 1 + k];
        if (t != kNone && !(t & kVar)) stack.push_back(t);
      }
    }
  };
  for (uint32_t i = 0; i < v.n_iface; ++i) visit(ifc[i]);
  for (uint32_t e = 0; e < v.n_residual; ++e)
    if (f.alive[e]) {
      visit(eq[2 * e]);
      visit(eq[2 * e + 1]);
    }
  auto map_ref = [&](uint32_t t) { return (t == kNone || (t & kVar)) ? t : remap[t]; };
  out.agents.resize(order.size() * 4);
  for (size_t j = 0; j < order.size(); ++j) {
    const uint32_t a = order[j];
    out.agents[4 * j] = ag[4 * a];
    for (int k = 1; k < 4; ++k) out.agents[4 * j + k] = map_ref(ag[4 * a + k]);
  }
  out.iface.resize(v.n_iface);
  for (uint32_t i = 0; i < v.n_iface; ++i) out.iface[i] = map_ref(ifc[i]);
  out.eqs.clear();
  for (uint32_t e = 0; e < v.n_residual; ++e)
    if (f.alive[e]) {
      out.eqs.push_back(map_ref(eq[2 * e]));
      out.eqs.push_back(map_ref(eq[2 * e + 1]));
    }
  return INET_OK;
}

// Cores this process may run on (the affinity mask, not the machine's count:
// a container pinned to 16 of 224 cores must not spawn 224 threads).
uint32_t usable_cores() {
  cpu_set_t set;
  CPU_ZERO(&set);
  if (sched_getaffinity(0, sizeof(set), &set) == 0) return std::max(1, CPU_COUNT(&set));
  return std::max(1u, std::thread::hardware_concurrency());
}

int parallel_for(uint32_t n, uint32_t n_threads, const std::function<int(uint32_t)>& fn) {
  static const uint32_t cores = usable_cores();
  if (n_threads == 0) n_threads = cores;
  n_threads = std::min(n_threads, std::max(1u, n / 16));  // at least 16 items per thread
  n_threads = std::min(n_threads, n);
  std::atomic<uint32_t> next{0};
  std::atomic<int> first{INET_OK};
  auto worker = [&]() {
    for (;;) {
      const uint32_t i = next.fetch_add(1);
      if (i >= n) return;
      const int st = fn(i);
      int expect = INET_OK;
      if (st != INET_OK) first.compare_exchange_strong(expect, st);
    }
  };
  if (n_threads <= 1) {
    worker();
  } else {
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < n_threads; ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
  }
  return first.load();
}


// ---------------------------------------------------------------------------
// Canonical printer (restates lang.print_configuration, src/inet/lang.py:333-396,
// with core.iter_vars order, core.py:96-104): equations oriented so that the
// smaller structural skeleton (lang.py:347-360) is on the left, stably sorted
// by (smaller, larger) skeleton, variables named x0, x1, ... in first-occurrence
// preorder over the interface then the sorted equations, terms printed as
// `Name` / `Name(c0,c1)`. Works on a flat normal form (preorder agents whose
// refs index the same array), so large results print without building terms.
namespace {

struct Printer {
  const uint32_t* ag;
  uint32_t na;
  const char* const* names;
  const uint8_t* arity;
  uint32_t nl;
  uint64_t budget;  // agents a walk may visit (a tree visits each once)
  std::vector<uint32_t>* st;      // walk stack (per thread, reused across nets)
  const std::vector<uint32_t>* nlen;  // strlen of every label name

  bool agent_ok(uint32_t a) const { return a < na && ag[4 * a] < nl; }

  // structural skeleton: Name( children ) with ? for variables
  bool skeleton(uint32_t root, std::string& out) {
    std::vector<uint32_t>& s = *st;
    s.clear();
    s.push_back(root);
    uint64_t seen = 0;
    while (!s.empty()) {
      const uint32_t t = s.back();
      s.pop_back();
      if (t == kNone - 1) {
        out.push_back(')');
        continue;
      }
      if (t == kNone) return false;
      if (t & kVar) {
        out.push_back('?');
        continue;
      }
      if (!agent_ok(t) || ++seen > budget) return false;
      const uint32_t lab = ag[4 * t];
      out.append(names[lab], (*nlen)[lab]);
      out.push_back('(');
      s.push_back(kNone - 1);
      for (int k = int(arity[lab]) - 1; k >= 0; --k) s.push_back(ag[4 * t + 1 + k]);
    }
    return true;
  }

  // Prints one term; a variable gets its number at its first occurrence in
  // printing order (interface terms, then the sorted equations left to right),
  // which is core.iter_vars' first-occurrence preorder — numbering and printing
  // in one walk.
  bool term(uint32_t root, std::unordered_map<uint32_t, uint32_t>& ids, std::string& out) {
    std::vector<uint32_t>& s = *st;
    s.clear();
    s.push_back(root);
    uint64_t seen = 0;
    char num[12];
    while (!s.empty()) {
      const uint32_t t = s.back();
      s.pop_back();
      if (t == kNone - 1) {
        out.push_back(')');
        continue;
      }
      if (t == kNone - 2) {
        out.push_back(',');
        continue;
      }
      if (t == kNone) return false;
      if (t & kVar) {
        const uint32_t next = static_cast<uint32_t>(ids.size());
        uint32_t id = ids.emplace(t & ~kVar, next).first->second;
        char* e = num + sizeof(num);
        char* b = e;
        do {
          *--b = static_cast<char>('0' + id % 10u);
          id /= 10u;
        } while (id);
        out.push_back('x');
        out.append(b, static_cast<size_t>(e - b));
        continue;
      }
      if (!agent_ok(t) || ++seen > budget) return false;
      const uint32_t lab = ag[4 * t];
      out.append(names[lab], (*nlen)[lab]);
      const uint32_t n = arity[lab];
      if (n == 0) continue;
      out.push_back('(');
      s.push_back(kNone - 1);
      for (int k = int(n) - 1; k >= 0; --k) {
        s.push_back(ag[4 * t + 1 + k]);
        if (k) s.push_back(kNone - 2);
      }
    }
    return true;
  }
};

}  // namespace

int print_flat(const uint32_t* agents, uint32_t n_agents, const uint32_t* iface, uint32_t n_iface,
               const uint32_t* eqs, uint32_t n_eqs, const char* const* names, const uint8_t* arity,
               uint32_t n_labels, std::string& out) {
  // per-thread scratch, reused across the nets a worker prints
  thread_local std::vector<uint32_t> stack;
  thread_local std::vector<uint32_t> nlen;
  thread_local std::unordered_map<uint32_t, uint32_t> ids;
  nlen.resize(n_labels);
  for (uint32_t l = 0; l < n_labels; ++l) {
    if (!names[l] || arity[l] > 3) return INET_ERR_ARG;
    nlen[l] = static_cast<uint32_t>(std::strlen(names[l]));
  }
  Printer p{agents, n_agents, names, arity, n_labels, uint64_t(n_agents) + 1, &stack, &nlen};
  // orientation and order of the equations
  struct Eq {
    uint32_t l, r;
    std::string a, b;  // (smaller, larger) skeleton
  };
  std::vector<Eq> es(n_eqs);
  for (uint32_t e = 0; e < n_eqs; ++e) {
    std::string sl, sr;
    if (!p.skeleton(eqs[2 * e], sl) || !p.skeleton(eqs[2 * e + 1], sr)) return INET_ERR_ARG;
    if (sl <= sr)
      es[e] = Eq{eqs[2 * e], eqs[2 * e + 1], std::move(sl), std::move(sr)};
    else
      es[e] = Eq{eqs[2 * e + 1], eqs[2 * e], std::move(sr), std::move(sl)};
  }
  std::stable_sort(es.begin(), es.end(), [](const Eq& x, const Eq& y) {
    const int c = x.a.compare(y.a);
    return c != 0 ? c < 0 : x.b < y.b;
  });
  ids.clear();
  out.clear();
  out.reserve(size_t(n_agents) * 3 + 16);
  out.append("net");
  if (n_iface) out.push_back(' ');
  for (uint32_t i = 0; i < n_iface; ++i) {
    if (i) out.append(", ");
    if (!p.term(iface[i], ids, out)) return INET_ERR_ARG;
  }
  out.append(" : ");
  for (size_t k = 0; k < es.size(); ++k) {
    if (k) out.append(", ");
    if (!p.term(es[k].l, ids, out)) return INET_ERR_ARG;
    out.append(" = ");
    if (!p.term(es[k].r, ids, out)) return INET_ERR_ARG;
  }
  out.push_back(';');  // "net ... : ;" when no equation is left
  return INET_OK;
}

int copy_text(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (buf && cap) std::memcpy(buf, s.data(), std::min(cap, s.size()));
  return INET_OK;
}
}  // namespace inethost

extern "C" int inet_finalize_flat(uint32_t* agents, uint32_t n_agents, uint32_t* iface, uint32_t n_iface,
                                  uint32_t* eqs, uint32_t n_eqs, uint32_t n_vars, uint8_t* alive) {
  try {
    if ((n_agents && !agents) || (n_iface && !iface) || (n_eqs && !eqs)) return INET_ERR_ARG;
    return inethost::finalize_flat(agents, n_agents, iface, n_iface, eqs, n_eqs, n_vars, alive);
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}

extern "C" int inet_print_flat(const uint32_t* agents, uint32_t n_agents, const uint32_t* iface, uint32_t n_iface,
                               const uint32_t* eqs, uint32_t n_eqs, const char* const* names, const uint8_t* arity,
                               uint32_t n_labels, char* buf, size_t cap, size_t* len) {
  try {
    if ((n_agents && !agents) || (n_iface && !iface) || (n_eqs && !eqs) || (n_labels && (!names || !arity)) || !len)
      return INET_ERR_ARG;
    std::string text;
    const int st = inethost::print_flat(agents, n_agents, iface, n_iface, eqs, n_eqs, names, arity, n_labels, text);
    if (st) return st;
    return inethost::copy_text(text, buf, cap, len);
  } catch (const std::bad_alloc&) {
    return INET_ERR_ARENA;  // host allocation failed: reported, never thrown across the C ABI
  } catch (...) {
    return INET_ERR_ARG;
  }
}
