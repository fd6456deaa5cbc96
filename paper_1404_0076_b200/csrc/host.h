// host.h — host-side helpers of libinetb200: rule-blob validation, the
// sequential finalize (engine.py:287-362) on flat arrays, and a tiny
// parallel-for used to finalize a batch of nets on all host cores.
#pragma once
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "../../include/inet_b200.h"

struct inet_ctx;

namespace inethost {

// Finalized normal form of one net: preorder agent records (4 words), interface
// refs, surviving equations (2 words). Refs index these arrays; variable ids are
// the device's.
struct NormalForm {
  std::vector<uint32_t> agents;
  std::vector<uint32_t> iface;
  std::vector<uint32_t> eqs;
  // finalized on the device: the agent records stay in the context's
  // page-locked result buffer (valid until the next reduction)
  const uint32_t* ext_agents = nullptr;
  uint32_t ext_n = 0;
  const uint32_t* agent_data() const { return ext_agents ? ext_agents : agents.data(); }
  uint32_t n_agents() const { return ext_agents ? ext_n : static_cast<uint32_t>(agents.size() / 4); }
};

// Read-only view of one reduced net as fetched from the device.
struct NetView {
  const uint32_t* agents;    // arena prefix, 4 words per agent
  uint32_t n_agents;
  const uint32_t* residual;  // parked equations {Var(x), other side}
  uint32_t n_residual;
  const uint32_t* iface;
  uint32_t n_iface;
  uint32_t n_vars;           // exclusive bound of variable ids
};

int validate_rule_blob(const uint32_t* blob, size_t n_words);
int validate_nets(const inet_ctx& c);

// In-place finalize on mutable flat arrays; alive[e] = 1 for surviving equations.
int finalize_flat(uint32_t* agents, uint32_t n_agents, uint32_t* iface, uint32_t n_iface, uint32_t* eqs,
                  uint32_t n_eqs, uint32_t n_vars, uint8_t* alive);

// Canonical text of a flat normal form (lang.print_configuration).
int print_flat(const uint32_t* agents, uint32_t n_agents, const uint32_t* iface, uint32_t n_iface,
               const uint32_t* eqs, uint32_t n_eqs, const char* const* names, const uint8_t* arity,
               uint32_t n_labels, std::string& out);
int copy_text(const std::string& s, char* buf, size_t cap, size_t* len);

// finalize + compaction of one fetched net.
int finalize_net(const NetView& v, NormalForm& out);
int finalize_batch(inet_ctx& c, uint32_t net, uint32_t n_threads);

// Run fn(i) for i in [0, n) on up to n_threads threads; returns the first error.
int parallel_for(uint32_t n, uint32_t n_threads, const std::function<int(uint32_t)>& fn);

}  // namespace inethost
