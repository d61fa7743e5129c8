// PQ-tree memory layout planner (PAPER §3.2, Alg. 2-6, App. C) over node-output rows.
#pragma once
#include <stdint.h>

#include <vector>

#include "ed_batch.h"

namespace ed {

struct LayoutInput {
  int64_t V;
  const std::vector<int32_t> *gtype, *in_off, *in_idx;             // merged graph
  const std::vector<int32_t> *batch_type, *batch_off, *members;    // Alg. 1 schedule
  const std::vector<ed_op_type_t> *types;
};

// Returns row_of_node (size V) or an empty vector if the planner is unavailable.
std::vector<int32_t> plan_layout_pq(const LayoutInput &in);

}  // namespace ed
