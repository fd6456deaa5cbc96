// inet_oracle.cpp — CPU restatement of the reference reducer. TEST INFRASTRUCTURE ONLY.
//
// This file is the parity checker and the CPU baseline. Only tests/, the
// smoke() entry point and bench.py's cpu_baseline / --impl reference legs may
// load it; the product (paper_1404_0076_b200) never does.
//
// It restates, step for step and with the reference's exact variable ids,
// the bulk-synchronous evaluator of /root/reference/pkg/src/inet:
//
//   evaluate             engine.py:186-228   loop, cap check, (0,0) stop
//   interaction_phase    engine.py:106-134   fresh block base + i*max_fresh,
//                                            slot order, stable compaction
//   _fill_slots          engine.py:77-103    find_rule / instantiate per eq
//   instantiate          core.py:281-304     orientation, pattern binding,
//                                            bound_vars -> fresh ids in order
//   communication_phase  engine.py:137-166   var-left normalisation, smaller
//                                            id left for var=var, stable sort
//                                            by left id, reduce_by_key merge
//   reduce_by_key        engine.py:59-74
//   finalize             engine.py:287-362   queue order, DFS containment test
//
// Terms are int64 refs: >= 0 agent index, < 0 variable -(id+1). Agents are
// immutable once built; the two agents of an active pair are recycled after
// the rewrite (they are unreachable in the reference too), which changes no
// observable result. The rule table is the same blob the device consumes
// (include/inet_b200.h), so the restatement shares no code with the engine
// beyond that documented format.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <deque>
#include <vector>

namespace {

constexpr int64_t kNoTerm = INT64_MIN;
constexpr uint32_t kMagic = 0x31524E49u;

enum Status { OK = 0, NO_RULE = 1, LOOP_CAP = 2, SLOT_OVERFLOW = 9, BAD_INPUT = 5 };

inline bool is_var(int64_t t) { return t < 0 && t != kNoTerm; }
inline int64_t var_id(int64_t t) { return -(t + 1); }
inline int64_t mk_var(int64_t id) { return -(id + 1); }

struct Rule {
  uint32_t n_new, n_eq, n_fresh;
  uint32_t agent[8];
  uint16_t eq[8];
};

struct Rules {
  uint32_t L = 0;
  std::vector<uint16_t> pair;
  std::vector<Rule> rule;
  uint32_t max_rhs = 0, max_fresh = 0;
  bool load(const uint32_t* b, size_t n) {
    if (n < 4 || b[0] != kMagic) return false;
    L = b[1];
    const uint32_t R = b[2];
    const size_t pw = (size_t(L) * L + 1) / 2;
    if (n != 4 + pw + size_t(R) * 16) return false;
    pair.assign(reinterpret_cast<const uint16_t*>(b + 4), reinterpret_cast<const uint16_t*>(b + 4) + size_t(L) * L);
    rule.resize(R);
    for (uint32_t r = 0; r < R; ++r) {
      const uint32_t* w = b + 4 + pw + 16 * r;
      Rule& x = rule[r];
      x.n_new = w[0] & 0xFF;
      x.n_eq = (w[0] >> 8) & 0xFF;
      x.n_fresh = (w[0] >> 16) & 0xFF;
      for (int m = 0; m < 8; ++m) x.agent[m] = w[1 + m];
      for (int e = 0; e < 8; ++e) x.eq[e] = (w[9 + e / 2] >> ((e & 1) * 16)) & 0xFFFF;
      max_rhs = std::max(max_rhs, x.n_eq);
      max_fresh = std::max(max_fresh, x.n_fresh);
    }
    return true;
  }
};

struct Arena {
  std::vector<int64_t> rec;  // 4 per agent: label, port0..2
  std::vector<int64_t> free_list;
  int64_t alloc() {
    if (!free_list.empty()) {
      const int64_t a = free_list.back();
      free_list.pop_back();
      return a;
    }
    rec.resize(rec.size() + 4, kNoTerm);
    return int64_t(rec.size() / 4 - 1);
  }
  int64_t label(int64_t a) const { return rec[4 * a]; }
  int64_t port(int64_t a, int k) const { return rec[4 * a + 1 + k]; }
};

struct Eq {
  int64_t l, r;
};

struct Result {
  int status = OK;
  int64_t err_a = -1, err_b = -1;
  int64_t interactions = 0, communications = 0, loops = 0;
  std::vector<int64_t> rows;  // 3 per loop: interactions, communications, live
  double wall_s = 0;
  // final configuration, compacted (preorder agents, refs local)
  std::vector<int64_t> f_agents, f_iface, f_eqs;
};

struct Oracle {
  Rules rules;
  Arena ar;
  std::vector<Eq> eqs;
  std::vector<int64_t> iface;

  // instantiate (core.py:281-304) into out; returns false on NoRuleForPair
  bool interact(const Eq& eq, int64_t fresh_base, std::vector<Eq>& out, Result& res) {
    int64_t A = eq.l, B = eq.r;
    const int64_t la = ar.label(A), lb = ar.label(B);
    const uint16_t t = rules.pair[size_t(la) * rules.L + size_t(lb)];
    if (t == 0xFFFF) {
      res.status = NO_RULE;
      res.err_a = la;
      res.err_b = lb;
      return false;
    }
    if (t & 1) std::swap(A, B);
    const Rule& R = rules.rule[t >> 1];
    int64_t env[24];
    for (int k = 0; k < 3; ++k) {
      env[k] = ar.port(A, k);
      env[3 + k] = ar.port(B, k);
    }
    for (uint32_t j = 0; j < R.n_fresh; ++j) env[6 + j] = mk_var(fresh_base + j);
    env[22] = kNoTerm;
    // the pattern agents are unreachable after the rewrite: recycle them
    ar.free_list.push_back(B);
    ar.free_list.push_back(A);
    for (uint32_t m = 0; m < R.n_new; ++m) env[14 + m] = ar.alloc();
    for (uint32_t m = 0; m < R.n_new; ++m) {
      const uint32_t w = R.agent[m];
      int64_t* rec = &ar.rec[4 * env[14 + m]];
      rec[0] = w & 0xFF;
      rec[1] = env[(w >> 8) & 0xFF];
      rec[2] = env[(w >> 16) & 0xFF];
      rec[3] = env[w >> 24];
    }
    for (uint32_t e = 0; e < R.n_eq; ++e) out.push_back({env[R.eq[e] & 0xFF], env[R.eq[e] >> 8]});
    return true;
  }

  void run(int64_t slot_count, int64_t max_loops, bool collect, Result& res) {
    const auto t0 = std::chrono::steady_clock::now();
    if (slot_count >= 0 && uint64_t(slot_count) < rules.max_rhs) {
      res.status = SLOT_OVERFLOW;
      return;
    }
    // FreshIdAllocator(config.max_var_id() + 1)  (engine.py:196)
    int64_t next_id = 0;
    auto note = [&](int64_t t) {
      if (is_var(t)) next_id = std::max(next_id, var_id(t) + 1);
    };
    for (size_t a = 0; a < ar.rec.size() / 4; ++a)
      for (int k = 0; k < 3; ++k) note(ar.port(int64_t(a), k));
    for (auto& e : eqs) {
      note(e.l);
      note(e.r);
    }
    for (auto t : iface) note(t);
    const int64_t max_fresh = rules.max_fresh;
    std::vector<Eq> out, pass, elig, merged;
    std::vector<std::pair<int64_t, uint32_t>> keyed;
    int64_t loop = 0;
    for (;;) {
      ++loop;
      if (loop > max_loops) {
        res.status = LOOP_CAP;
        break;
      }
      // interaction phase: reserve len(eqs)*max_fresh ids, then in order
      const int64_t base = next_id;
      next_id += int64_t(eqs.size()) * max_fresh;
      out.clear();
      int64_t ints = 0;
      for (size_t i = 0; i < eqs.size(); ++i) {
        const Eq& eq = eqs[i];
        if (eq.l >= 0 && eq.r >= 0) {
          if (!interact(eq, base + int64_t(i) * max_fresh, out, res)) break;
          ++ints;
        } else {
          out.push_back(eq);
        }
      }
      if (res.status != OK) break;
      // communication phase
      pass.clear();
      elig.clear();
      for (const Eq& eq : out) {
        const bool lv = is_var(eq.l), rv = is_var(eq.r);
        if (lv && rv)
          elig.push_back(var_id(eq.r) < var_id(eq.l) ? Eq{eq.r, eq.l} : eq);
        else if (lv)
          elig.push_back(eq);
        else if (rv)
          elig.push_back({eq.r, eq.l});
        else
          pass.push_back(eq);
      }
      keyed.resize(elig.size());
      for (size_t k = 0; k < elig.size(); ++k) keyed[k] = {var_id(elig[k].l), uint32_t(k)};
      std::sort(keyed.begin(), keyed.end());  // (key, position): stable by construction
      merged.clear();
      int64_t last = -1;
      bool have = false;
      for (auto& kp : keyed) {
        const Eq& x = elig[kp.second];
        if (have && kp.first == last) {
          merged.back() = {merged.back().r, x.r};
        } else {
          merged.push_back(x);
          last = kp.first;
          have = true;
        }
      }
      const int64_t comms = int64_t(elig.size()) - int64_t(merged.size());
      eqs.swap(pass);
      eqs.insert(eqs.end(), merged.begin(), merged.end());
      res.interactions += ints;
      res.communications += comms;
      if (collect) {
        res.rows.push_back(ints);
        res.rows.push_back(comms);
        res.rows.push_back(int64_t(eqs.size()));
      }
      res.loops = loop;
      if (ints == 0 && comms == 0) break;
    }
    if (res.status == OK) finalize(res);
    res.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }

  // ---- finalize (engine.py:287-362) --------------------------------------
  // cells: interface [0,ni), equation sides [ni, ni+2ne), ports of agent a at
  // ni + 2ne + 3a + k. The reference keys containers by Python identity; here
  // a cell id plays that role.
  void finalize(Result& res) {
    const int64_t ni = int64_t(iface.size()), ne = int64_t(eqs.size());
    const int64_t na = int64_t(ar.rec.size() / 4);
    auto cell = [&](int64_t c) -> int64_t& {
      if (c < ni) return iface[size_t(c)];
      if (c < ni + 2 * ne) {
        Eq& e = eqs[size_t((c - ni) / 2)];
        return ((c - ni) & 1) ? e.r : e.l;
      }
      const int64_t p = c - ni - 2 * ne;
      return ar.rec[size_t(4 * (p / 3) + 1 + p % 3)];
    };
    std::vector<std::vector<int64_t>> occ;  // var id -> cells, discovery order
    std::vector<int64_t> ids;               // dense index per var id
    auto occ_of = [&](int64_t id) -> std::vector<int64_t>& {
      if (id >= int64_t(ids.size())) ids.resize(size_t(id) + 1, -1);
      if (ids[size_t(id)] < 0) {
        ids[size_t(id)] = int64_t(occ.size());
        occ.emplace_back();
      }
      return occ[size_t(ids[size_t(id)])];
    };
    auto scan = [&](int64_t root) {  // _to_mutable's traversal
      std::vector<int64_t> st{root};
      while (!st.empty()) {
        const int64_t c = st.back();
        st.pop_back();
        const int64_t t = cell(c);
        if (t == kNoTerm) continue;
        if (is_var(t)) {
          occ_of(var_id(t)).push_back(c);
          continue;
        }
        for (int k = 0; k < 3; ++k)
          if (ar.port(t, k) != kNoTerm) st.push_back(ni + 2 * ne + 3 * t + k);
      }
    };
    for (int64_t i = 0; i < ni; ++i) scan(i);
    for (int64_t e = 0; e < ne; ++e) {
      scan(ni + 2 * e);
      scan(ni + 2 * e + 1);
    }
    (void)na;
    std::vector<uint8_t> alive(size_t(ne), 1);
    auto contains_var = [&](int64_t term, int64_t id) {  // engine.py:275-284
      std::vector<int64_t> st{term};
      while (!st.empty()) {
        const int64_t t = st.back();
        st.pop_back();
        if (t == kNoTerm) continue;
        if (is_var(t)) {
          if (var_id(t) == id) return true;
        } else {
          for (int k = 0; k < 3; ++k) st.push_back(ar.port(t, k));
        }
      }
      return false;
    };
    std::deque<int64_t> queue;
    for (int64_t e = 0; e < ne; ++e) queue.push_back(e);
    while (!queue.empty()) {
      const int64_t e = queue.front();
      queue.pop_front();
      if (!alive[size_t(e)]) continue;
      for (int side = 0; side < 2; ++side) {
        const int64_t self = ni + 2 * e + side;
        const int64_t v = cell(self);
        if (!is_var(v)) continue;
        std::vector<int64_t>& slots = occ_of(var_id(v));
        int64_t target = -1;
        for (int64_t o : slots) {
          if (o == self) continue;
          if (o >= ni && o < ni + 2 * ne && !alive[size_t((o - ni) / 2)]) continue;
          target = o;
          break;
        }
        if (target < 0) continue;
        const int64_t other = ni + 2 * e + (1 - side);
        if (target == other || contains_var(cell(other), var_id(v))) continue;
        const int64_t rep = cell(other);
        alive[size_t(e)] = 0;
        cell(target) = rep;
        if (is_var(rep)) {
          for (int64_t& s : occ_of(var_id(rep)))
            if (s == other) {
              s = target;
              break;
            }
        }
        slots.clear();
        if (target >= ni && target < ni + 2 * ne) {
          const int64_t f = (target - ni) / 2;
          if (alive[size_t(f)]) queue.push_back(f);
        }
        break;
      }
    }
    // compact: preorder numbering of reachable agents
    std::vector<int64_t> remap(ar.rec.size() / 4, -1);
    std::vector<int64_t> order;
    auto visit = [&](int64_t root) {
      if (root < 0) return;
      std::vector<int64_t> st{root};
      while (!st.empty()) {
        const int64_t a = st.back();
        st.pop_back();
        remap[size_t(a)] = int64_t(order.size());
        order.push_back(a);
        for (int k = 2; k >= 0; --k) {
          const int64_t t = ar.port(a, k);
          if (t >= 0) st.push_back(t);
        }
      }
    };
    for (int64_t i = 0; i < ni; ++i) visit(iface[size_t(i)]);
    for (int64_t e = 0; e < ne; ++e)
      if (alive[size_t(e)]) {
        visit(eqs[size_t(e)].l);
        visit(eqs[size_t(e)].r);
      }
    auto map_ref = [&](int64_t t) { return t >= 0 ? remap[size_t(t)] : t; };
    res.f_agents.clear();
    for (int64_t a : order) {
      res.f_agents.push_back(ar.label(a));
      for (int k = 0; k < 3; ++k) res.f_agents.push_back(map_ref(ar.port(a, k)));
    }
    res.f_iface.clear();
    for (int64_t t : iface) res.f_iface.push_back(map_ref(t));
    res.f_eqs.clear();
    for (int64_t e = 0; e < ne; ++e)
      if (alive[size_t(e)]) {
        res.f_eqs.push_back(map_ref(eqs[size_t(e)].l));
        res.f_eqs.push_back(map_ref(eqs[size_t(e)].r));
      }
  }
};

}  // namespace

extern "C" {

// Run the reference algorithm on one net. Agent records are 4 int64 {label,
// port0..2} with kNoTerm (INT64_MIN) for unused ports; refs >= 0 are agents,
// < 0 variables -(id+1) with the caller's original ids. slot_count < 0 means
// None. Returns an opaque handle (never null) holding the result.
void* oracle_run(const uint32_t* blob, size_t blob_words, const int64_t* agents, int64_t n_agents,
                 const int64_t* eqs, int64_t n_eqs, const int64_t* iface, int64_t n_iface, int64_t slot_count,
                 int64_t max_loops, int collect) {
  auto* res = new Result();
  Oracle o;
  if (!o.rules.load(blob, blob_words)) {
    res->status = BAD_INPUT;
    return res;
  }
  o.ar.rec.assign(agents, agents + 4 * n_agents);
  o.eqs.resize(size_t(n_eqs));
  for (int64_t i = 0; i < n_eqs; ++i) o.eqs[size_t(i)] = {eqs[2 * i], eqs[2 * i + 1]};
  o.iface.assign(iface, iface + n_iface);
  o.run(slot_count, max_loops, collect != 0, *res);
  return res;
}

int oracle_status(void* h, int64_t* out6) {
  auto* r = static_cast<Result*>(h);
  out6[0] = r->interactions;
  out6[1] = r->communications;
  out6[2] = r->loops;
  out6[3] = r->err_a;
  out6[4] = r->err_b;
  out6[5] = int64_t(r->wall_s * 1e9);
  return r->status;
}

int64_t oracle_rows(void* h, int64_t* rows) {
  auto* r = static_cast<Result*>(h);
  if (rows) std::memcpy(rows, r->rows.data(), r->rows.size() * sizeof(int64_t));
  return int64_t(r->rows.size() / 3);
}

// sizes[3] = {n_agents, n_iface, n_eqs}; buffers may be null to query sizes
void oracle_final(void* h, int64_t* sizes, int64_t* agents, int64_t* iface, int64_t* eqs) {
  auto* r = static_cast<Result*>(h);
  sizes[0] = int64_t(r->f_agents.size() / 4);
  sizes[1] = int64_t(r->f_iface.size());
  sizes[2] = int64_t(r->f_eqs.size() / 2);
  if (agents) std::memcpy(agents, r->f_agents.data(), r->f_agents.size() * sizeof(int64_t));
  if (iface) std::memcpy(iface, r->f_iface.data(), r->f_iface.size() * sizeof(int64_t));
  if (eqs) std::memcpy(eqs, r->f_eqs.data(), r->f_eqs.size() * sizeof(int64_t));
}

void oracle_free(void* h) { delete static_cast<Result*>(h); }

}  // extern "C"
