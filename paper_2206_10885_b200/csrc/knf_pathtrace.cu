// knf_pathtrace.cu -- placeholder; replaced by the device path tracer.
#include "knf_engine.h"

using namespace knf;

struct knf_scene_s {
  int device;
};

extern "C" {
int knf_scene_create(const KnfObject*, int32_t, const double*, int, knf_scene_t* out) {
  if (out) *out = nullptr;
  return fail(KNF_E_UNSUPPORTED, "path tracer not built yet");
}
int knf_scene_destroy(knf_scene_t sc) {
  delete sc;
  return 0;
}
int knf_rng_uniform(uint64_t, const uint64_t*, const uint64_t*, const uint64_t*, int64_t, double*, int, int, void*) {
  return fail(KNF_E_UNSUPPORTED, "path tracer not built yet");
}
int knf_pathtrace(knf_scene_t, const KnfCamera*, int32_t, uint64_t, int32_t, int32_t, int, int, double*, int, void*) {
  return fail(KNF_E_UNSUPPORTED, "path tracer not built yet");
}
int knf_trace_paths(knf_scene_t, const double*, const double*, const uint64_t*, int64_t, uint64_t, uint64_t, int32_t,
                    double*, int, void*) {
  return fail(KNF_E_UNSUPPORTED, "path tracer not built yet");
}
}
