// adaptis_inst_onef1b.cu — instantiations of the segment kernel for ADAPTIS_ONEF1B
// (one translation unit per policy so that nvcc builds them in parallel).
#include "adaptis_seg.cuh"

namespace adaptis {

template <int V, typename T>
static KFn pick_fb_onef1b(bool fallback, bool trace) {
  if constexpr (!std::is_floating_point<T>::value)
    if (trace) return (KFn)seg_kernel<ADAPTIS_ONEF1B, V, T, true, true>;
  return fallback ? (KFn)seg_kernel<ADAPTIS_ONEF1B, V, T, true> : (KFn)seg_kernel<ADAPTIS_ONEF1B, V, T, false>;
}
template <typename T>
static KFn pick_v_onef1b(int v, bool fb, bool tr) {
  switch (v) {
    case 1: return pick_fb_onef1b<1, T>(fb, tr);
    case 2: return pick_fb_onef1b<2, T>(fb, tr);
    case 3: return pick_fb_onef1b<3, T>(fb, tr);
    default: return pick_fb_onef1b<4, T>(fb, tr);
  }
}
KFn pick_policy_onef1b(int tick, int v, bool fb, bool tr) {
  if (tick == kTickI64) return pick_v_onef1b<int64_t>(v, fb, tr);
  if (tick == kTickF32) return pick_v_onef1b<float>(v, fb, tr);
  return pick_v_onef1b<int32_t>(v, fb, tr);
}

}  // namespace adaptis
