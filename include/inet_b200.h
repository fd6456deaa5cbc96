/*
 * inet_b200.h — C ABI of the B200 interaction-net reducer.
 *
 * This is the drop-in boundary for the reference's hot path
 *   inet.engine.evaluate(config, rules, cfg) -> EvalResult
 *   (/root/reference/pkg/src/inet/engine.py:186-228)
 * and its helpers interaction_phase / communication_phase / reduce_by_key /
 * finalize (engine.py:59-166, 287-362). The Python host module
 * paper_1404_0076_b200.engine binds these entry points with ctypes; the
 * reference-side binding a maintainer would add is shown in INTEGRATION.md.
 *
 * Everything is plain C: 32-bit words, host pointers and sizes. No CUDA or
 * torch types cross the boundary.
 *
 * Flat formats
 * ------------
 * term ref   u32. Bit 31 set: variable, id = low 31 bits. Otherwise an index
 *            into the agent array. INET_NONE (0xFFFFFFFF) = no term.
 * agent      4 x u32 {label, port0, port1, port2}; unused ports INET_NONE.
 *            (arity <= 3; every shipped program has arity <= 2.)
 * equation   2 x u32 {lhs ref, rhs ref}.
 * rule blob  see "Rule blob" below; built by
 *            paper_1404_0076_b200.flat.compile_rules from a RuleSet
 *            (the reference's Rule/RuleSet, core.py:158-251).
 *
 * Rule blob (u32 words)
 * ---------------------
 *   [0] INET_RULES_MAGIC  [1] n_labels (<= 64)  [2] n_rules (<= 256)  [3] 0
 *   pair table: n_labels*n_labels u16 entries packed two per word,
 *     entry[la*n_labels+lb] = 0xFFFF (no rule) or (rule << 1 | swap), where
 *     swap means the equation's lhs plays the rule's lhs_b
 *     (core.py:287-298: orientation of instantiate).
 *   n_rules records of 16 words:
 *     w0        n_new | n_eq << 8 | n_fresh << 16
 *     w1..w8    new agent m: label | src0 << 8 | src1 << 16 | src2 << 24
 *     w9..w12   rhs equation e: (srcL | srcR << 8) in 16-bit half (e & 1)
 *               of word 9 + e/2
 *   source codes: 0..2 port k of lhs_a, 3..5 port k of lhs_b,
 *     6..13 fresh variable j (bound_vars order, core.py:195-204),
 *     14..21 new agent m, 22 none.
 */
#ifndef INET_B200_H
#define INET_B200_H

#ifndef __CUDACC_RTC__
#include <stddef.h>
#include <stdint.h>
#else
typedef unsigned int uint32_t;
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef int int32_t;
typedef unsigned long long uint64_t;
typedef unsigned long size_t;
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define INET_NONE 0xFFFFFFFFu
#define INET_VAR_BIT 0x80000000u
#define INET_RULES_MAGIC 0x31524E49u /* "INR1" */
#define INET_MAX_ARITY 3
#define INET_MAX_LABELS 64
#define INET_MAX_RULES 256
#define INET_MAX_NEW 8
#define INET_MAX_EQ 8
#define INET_MAX_FRESH 8

/* Status codes. Mirrors the reference's error classes (errors.py:46-65). */
enum inet_status {
  INET_OK = 0,
  INET_ERR_NO_RULE = 1,      /* NoRuleForPair(a, b)       engine.py:92 / core.py:307-312 */
  INET_ERR_LOOP_CAP = 2,     /* LoopCapExceeded(max)      engine.py:205-207 */
  INET_ERR_ARENA = 3,        /* agent / variable / queue arena exhausted at max size */
  INET_ERR_CUDA = 4,         /* CUDA runtime failure */
  INET_ERR_ARG = 5,          /* bad argument / malformed blob */
  INET_ERR_UNSUPPORTED = 6,  /* exceeds a device-engine limit */
  INET_ERR_NO_DEVICE = 7,    /* no CUDA device visible */
  INET_ERR_STATE = 8,        /* call order violated (e.g. fetch before reduce) */
  INET_ERR_NAME = 9,         /* NameDisciplineError       engine.py:169-183 (validate_phases); the
                                variable's reference id in err_label_a (low) / err_label_b (high) */
  INET_ERR_ORDER = 10        /* var_order: two variables made in one loop by different interactions met
                                in a var = var equation; only the reference's list order (tier R,
                                reference_order = 1) decides which keys it */
};

typedef struct inet_ctx inet_ctx;

/* Knobs of one reduction; EngineConfig (engine.py:35-48) maps onto it. */
typedef struct inet_cfg {
  uint32_t max_loops;     /* LoopCapExceeded when round > max_loops */
  uint32_t collect_stats; /* record per-round rows (LoopStats) */
  uint32_t threads;       /* CTA size per net; 0 = auto */
  uint32_t ctas_per_net;  /* 0 = auto: a single net starts on one CTA, moves to a 16-CTA cluster past
                             2^19 interactions, and to the whole GPU if it outgrows the cluster;
                             1 = one CTA per net; 2..16 = that cluster size; > 16 = the whole GPU */
  uint32_t cap_agents;    /* initial per-net agent arena; 0 = auto (grows on overflow) */
  uint32_t cap_vars;      /* initial per-net variable table; 0 = auto (grows on overflow) */
  uint32_t max_retries;   /* arena doublings before INET_ERR_ARENA; 0 = default */
  uint32_t count_rules;   /* per-rule interaction histogram (accounting runs only) */
  uint32_t exact_loops;   /* 1: reference loop semantics — an equation a merge leaves var-headed
                             communicates in the next round (engine.py:137-166), so rounds and
                             LoopStats rows are the reference's loops; 0: link to a fixpoint
                             within the round (fewer rounds) */
  uint32_t reference_order; /* 1: tier R — the reference's equation list, in its order (var = var
                               keys, merge orientation, first failing pair and residual order
                               exactly as engine.py:106-166); 0: the fast tiers */
  uint32_t validate_phases; /* 1: name discipline checked after both phases of every loop
                               (engine.py:210-214); implies reference_order */
  uint32_t var_order;       /* 1: the fast single-CTA tiers key var = var equations by the reference's
                               variable ids (per-variable stamps: loop, creating interaction, bound
                               index); INET_ERR_ORDER when that does not decide */
} inet_cfg;

/* Per-net outcome. */
typedef struct inet_net_stats {
  uint64_t interactions;   /* EvalResult.total_interactions */
  uint64_t communications; /* EvalResult.total_communications */
  uint32_t rounds;         /* rounds incl. the trailing no-op round (= len(loops)) */
  uint32_t status;         /* inet_status of this net */
  uint32_t err_label_a;    /* NoRuleForPair labels, equation orientation */
  uint32_t err_label_b;
  uint32_t agent_hw;       /* arena high-water (agents ever addressed) */
  uint32_t var_hw;         /* variable-table high-water */
  uint32_t n_residual;     /* parked equations at the fixpoint (input of finalize) */
  uint32_t cap_agents;     /* capacities the successful run used */
  uint32_t cap_vars;
  uint32_t tier;           /* residency tier used: 0 S (shared), 1 M (mixed), 2 G (global), 3 C (cluster), 4 X (whole GPU),
                              5 R (reference order) */
  uint32_t jit;            /* 1 if the rule-set specialised kernel ran (else the interpreter) */
  uint32_t sm_mhz;         /* effective SM clock over this net's reduction (clock64 / globaltimer) */
  uint32_t device_final;   /* 1 if the normal form was finalized on the device (tier S), else the host did */
  uint32_t threads;        /* CTA size (threads per net, per CTA of a cluster) of the kernel that ran */
} inet_net_stats;

/* Context: one device, one stream, device buffers reused across calls.
 * Replaces the per-call ThreadPoolExecutor of evaluate (engine.py:201, 224-226). */
int inet_ctx_create(int device, inet_ctx** out);
void inet_ctx_destroy(inet_ctx* ctx);
const char* inet_strerror(int status);
/* sizeof(inet_cfg) and sizeof(inet_net_stats) as compiled into the library,
 * so a binding can check its struct layouts (no device needed). */
void inet_abi_sizes(size_t* cfg_bytes, size_t* stats_bytes);
/* Device properties for reporting: SM count and clock (kHz). */
int inet_device_info(inet_ctx* ctx, int* sm_count, int* clock_khz, char* name, size_t name_len);

/* Rule-set specialised kernels (NVRTC, compiled on first use and cached):
 * mode 1 = use when available (default; env INET_B200_JIT=0 disables), 0 = the
 * prebuilt table interpreter only. */
int inet_set_jit(inet_ctx* ctx, int mode);
/* Compile (or fetch from cache) the specialised kernel for a rule blob without
 * a device; returns INET_OK or INET_ERR_UNSUPPORTED with the NVRTC log. */
int inet_jit_compile(const uint32_t* blob, size_t n_words, int tier, uint32_t threads, char* log, size_t log_len);

/* Build time: compile the specialised kernel of (rule blob, tier, CTA size)
 * into the package's kernels/ directory next to the library, where every
 * later process finds it without running NVRTC (the shipped programs are
 * precompiled by the package build). flags: bit 0 reference-loop code
 * (deferred equations), bit 1 per-rule counters, bit 2 reference-ordered
 * var = var keys (stamps), bit 3 without per-round rows (collect_stats off),
 * bits 8-11 code style + 1 (0: the tier's default). */
int inet_jit_precompile(const uint32_t* blob, size_t n_words, int tier, uint32_t threads, uint32_t flags, char* log,
                        size_t log_len);

/* Upload a compiled rule set. Replaces RuleSet.lookup / find_rule / instantiate
 * (core.py:241-242, 281-312): the per-equation dictionary lookup and tree
 * rebuild become one table lookup and a template expansion on the device. */
int inet_rules_load(inet_ctx* ctx, const uint32_t* blob, size_t n_words);

/*
 * Load a batch of nets (n_nets >= 1). The Configuration argument of evaluate
 * (engine.py:186-189; core.py:135-155) in flat form; n_nets == 1 is evaluate
 * itself, n_nets > 1 is the new batch API. Net i owns
 *   agents[4*agent_off[i] .. 4*agent_off[i+1])   its agents (local indices)
 *   eqs[2*eq_off[i] .. 2*eq_off[i+1])             its equations
 *   iface[iface_off[i] .. iface_off[i+1])         its interface refs (host only)
 *   n_vars[i]                                     variables 0..n_vars[i]-1 in use
 * All refs are net-local. Data is copied; the caller keeps ownership.
 */
int inet_batch_load(inet_ctx* ctx, uint32_t n_nets, const uint32_t* agents, const uint64_t* agent_off,
                    const uint32_t* eqs, const uint64_t* eq_off, const uint32_t* iface,
                    const uint64_t* iface_off, const uint32_t* n_vars);

/*
 * Reduce every loaded net to its fixpoint on the device (the loop of
 * evaluate, engine.py:204-223: interaction_phase engine.py:106-134 and
 * communication_phase + reduce_by_key engine.py:59-74, 137-166). The whole
 * interaction / communication loop runs inside one persistent kernel with no
 * host synchronisation per round (replaces engine.py:204-223). Host buffers
 * were copied by inet_batch_load; this call performs H2D, the kernel(s),
 * overflow retries and the D2H of results. *device_ms is the CUDA-event time
 * of the reduction kernel(s) of the final, successful attempt.
 * Returns the first non-OK net status, or INET_OK.
 */
int inet_batch_reduce(inet_ctx* ctx, const inet_cfg* cfg, float* device_ms);

/* Same, but only the device part (inputs already resident from a previous
 * inet_batch_reduce of the same batch): re-initialise device state from the
 * resident copy and run the kernel. For device-timed benchmarking. */
int inet_batch_rerun(inet_ctx* ctx, const inet_cfg* cfg, float* device_ms);

/* EvalResult.total_interactions / total_communications and the error of net i
 * (engine.py:51-56; errors.py:46-56). */
/* Fetch the outcome of the last launch (after inet_batch_rerun, which only
 * times it): per-net statistics and results, as inet_batch_reduce leaves them. */
int inet_batch_collect(inet_ctx* ctx);
int inet_batch_stats(inet_ctx* ctx, uint32_t net, inet_net_stats* out);
/* Interactions per rule of net i (needs cfg.count_rules); counts[n_rules]. */
int inet_batch_rule_counts(inet_ctx* ctx, uint32_t net, uint64_t* counts, uint32_t n_rules);
/* Host<->device bytes moved by the last inet_batch_reduce (inputs, results). */
int inet_batch_io_bytes(inet_ctx* ctx, uint64_t* h2d, uint64_t* d2h);
/* Aggregate over all nets (sum of interactions/communications, max rounds). */
int inet_batch_totals(inet_ctx* ctx, uint64_t* interactions, uint64_t* communications, uint32_t* max_rounds,
                      uint32_t* n_failed);

/* EvalResult.loops (LoopStats rows, profile.py:16-22; engine.py:215-221).
 * Per-round rows of net i: 4 words per round {interactions, communications,
 * live_equations, elapsed_ns}. Two-call protocol: rows==NULL returns count. */
int inet_batch_rounds(inet_ctx* ctx, uint32_t net, uint32_t* rows, uint32_t* n_rows);

/*
 * finalize (engine.py:287-362) of net i: splice every parked
 * equation into the other occurrence of its variable, in the reference's
 * queue order, then compact the reachable normal form. Runs on host threads
 * (all nets in parallel when net == INET_NONE).
 */
int inet_batch_finalize(inet_ctx* ctx, uint32_t net, uint32_t n_threads);

/* EvalResult.final (engine.py:227-228) of net i after finalize: pointers stay valid until the next
 * load/reduce/finalize on this context. Agents are in preorder (children
 * after parents), refs are local to these arrays; variable ids are the
 * device's (input ids 0..n_vars-1 are preserved, fresh ids >= n_vars). */
/* Whole-batch forms of inet_batch_stats / the result sizes / inet_batch_print
 * (one call instead of one per net). inet_batch_print_all prints every
 * finalized net with n_threads host threads (0 = all cores): a first call with
 * buf = NULL returns the total length in *len; the second writes the texts
 * back to back with offsets[n_nets + 1] delimiting them. */
int inet_batch_stats_all(inet_ctx* ctx, inet_net_stats* out, uint32_t n_nets);
int inet_batch_result_counts(inet_ctx* ctx, uint32_t* n_agents, uint32_t* n_iface, uint32_t* n_eqs, uint32_t n_nets);
int inet_batch_print_all(inet_ctx* ctx, const char* const* names, const uint8_t* arity, uint32_t n_labels,
                         uint32_t n_threads, char* buf, size_t cap, uint64_t* offsets, size_t* len);
int inet_batch_result(inet_ctx* ctx, uint32_t net, const uint32_t** agents, uint32_t* n_agents,
                      const uint32_t** iface, uint32_t* n_iface, const uint32_t** eqs, uint32_t* n_eqs);

/*
 * Stand-alone finalize on caller buffers (engine.finalize, engine.py:287, flat):
 * agents/iface/eqs are modified in place; alive[e] receives 1 for equations
 * that survive. n_vars bounds variable ids.
 */
int inet_finalize_flat(uint32_t* agents, uint32_t n_agents, uint32_t* iface, uint32_t n_iface, uint32_t* eqs,
                       uint32_t n_eqs, uint32_t n_vars, uint8_t* alive);

/*
 * Canonical text of a normal form: lang.print_configuration (src/inet/lang.py:
 * 333-396) — equations oriented by structural skeleton (lang.py:347-365) and
 * stably sorted, variables renamed x0, x1, ... in first-occurrence preorder
 * (core.iter_vars, core.py:96-104). names[l] / arity[l] describe label l (the
 * rule blob's numbering). Writes min(cap, len) bytes (no terminating NUL) and
 * the full length to *len; call again with a larger buffer when *len > cap.
 * inet_print_flat prints flat arrays in the inet_batch_result layout (agents in
 * any order, refs index the agent array); inet_batch_print prints a finalized
 * net of the context without building terms on the host.
 */
int inet_print_flat(const uint32_t* agents, uint32_t n_agents, const uint32_t* iface, uint32_t n_iface,
                    const uint32_t* eqs, uint32_t n_eqs, const char* const* names, const uint8_t* arity,
                    uint32_t n_labels, char* buf, size_t cap, size_t* len);
int inet_batch_print(inet_ctx* ctx, uint32_t net, const char* const* names, const uint8_t* arity,
                     uint32_t n_labels, char* buf, size_t cap, size_t* len);

#ifdef __cplusplus
}
#endif

#endif /* INET_B200_H */
