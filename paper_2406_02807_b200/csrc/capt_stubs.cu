// Temporary: device construct / filter land in capt_build.cu / capt_filter.cu.
#include "capt_internal.cuh"
using namespace capt;
extern "C" int capt_filter_cloud(int, int, const float*, int64_t, double, int, const double*,
                                 double, uint32_t, float*, int64_t*, void*) {
  return fail(CAPT_EINVAL, "capt_filter_cloud not built yet");
}
