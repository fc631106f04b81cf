// K4: batched window greedy (placeholder until the kernel lands).
#include "roam_internal.h"

extern "C" int rm_greedy_windows(RmGraph*, int32_t, const int64_t*, const int32_t*, const int64_t*,
                                 const int32_t*, const int64_t*, const int32_t*, int32_t*, int64_t*,
                                 int32_t*, int32_t*, void*) {
  return roam::fail(RM_ERR_CAPACITY, "rm_greedy_windows: not built yet");
}
