// jit.h — rule-set specialised kernels (see jit.cpp).
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace inetjit {

// CUDA source of the per-rule rewrites (jit_apply) for a rule blob.
std::string generate_rules(const uint32_t* blob, size_t n_words, int style = 0);
// Complete translation unit: device code + rewrites + one kernel `inet_jit_kernel`.
// style: 0 straight-line cases, 1 per-lane uniform memory phase, 2 warp-collective
std::string kernel_source(const uint32_t* blob, size_t n_words, int tier, uint32_t block, int style = 0,
                          bool exact_code = true, bool count_rules = true, bool stamps = false, bool rows = true);
// NVRTC loadable?
bool available();
// Compile (or fetch from the on-disk cache) to an sm_100a cubin; 0 on success.
int compile_cubin(const std::string& source, std::vector<char>& cubin, std::string& log);
// Compile into the package's kernels/ directory (build time), skipping caches.
int precompile(const std::string& source, std::string& log);

}  // namespace inetjit
