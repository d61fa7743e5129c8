// Host-side FSM learner (PAPER §2.3): tabular N-step Q-learning.  Internal to
// libedbatch.so; the ABI is ed_fsm_learn in include/ed_batch.h.
#pragma once
#include <stdint.h>

#include <map>
#include <utility>
#include <vector>

#include "ed_batch.h"

namespace ed {

// One instance graph with local node ids; node inputs only (dependencies).
struct RlGraph {
  int32_t n = 0;
  std::vector<int32_t> type;
  std::vector<int32_t> pred_off, preds;  // distinct node inputs (CSR)
};

struct RlResult {
  std::map<std::pair<std::vector<int32_t>, int32_t>, double> q;  // (state key, action) -> Q
  std::map<std::vector<int32_t>, int32_t> table;                  // state key -> greedy action
  std::vector<std::pair<int64_t, int64_t>> checkpoints;           // (episode, greedy batch total)
  int64_t episodes = 0, final_batches = 0, lower_bound = 0;
};

// Returns 0 on success, -1 on a bad config.
int rl_train(const std::vector<RlGraph> &graphs, int num_types, const ed_rl_config_t &cfg, RlResult *out);

// Type of every batch of Alg. 1 run with the sufficient-condition chooser: argmax over the
// ready types of |Frontier_a(G_t)| / |Frontier(G^a_t)|, ties to the larger ready count, then the
// lower type id.
std::vector<int32_t> sc_type_sequence(const RlGraph &g, int num_types);

}  // namespace ed
