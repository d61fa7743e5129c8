#include "ed_layout.h"

namespace ed {

std::vector<int32_t> plan_layout_pq(const LayoutInput &) { return {}; }

}  // namespace ed
