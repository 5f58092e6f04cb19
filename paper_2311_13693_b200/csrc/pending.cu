// Entry points whose device implementations land in later milestones.
#include "common.cuh"
using namespace xtsg;
extern "C" {
int32_t xtsg_plan_compress_factors(xtsg_plan*, const double*, const double*, const double*, int64_t, int64_t,
                                   int64_t, void*, int32_t, void*) {
  return guard([] { throw Status(XTSG_E_INTERNAL, "not implemented yet"); });
}
int32_t xtsg_plan_compress_coo(xtsg_plan*, const int32_t*, const int32_t*, const int32_t*, const float*, int64_t,
                               void*, int32_t, void*) {
  return guard([] { throw Status(XTSG_E_INTERNAL, "not implemented yet"); });
}
}
