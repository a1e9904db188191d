// adaptis_inst_zb.cu — instantiations of the segment kernel for ADAPTIS_ZB
// (one translation unit per policy so that nvcc builds them in parallel).
#include "adaptis_seg.cuh"

namespace adaptis {

template <int V, typename T>
static KFn pick_fb_zb(bool fallback, bool trace) {
  if constexpr (!std::is_floating_point<T>::value)
    if (trace) return (KFn)seg_kernel<ADAPTIS_ZB, V, T, true, true>;
  return fallback ? (KFn)seg_kernel<ADAPTIS_ZB, V, T, true> : (KFn)seg_kernel<ADAPTIS_ZB, V, T, false>;
}
template <typename T>
static KFn pick_v_zb(int v, bool fb, bool tr) {
  switch (v) {
    case 1: return pick_fb_zb<1, T>(fb, tr);
    case 2: return pick_fb_zb<2, T>(fb, tr);
    case 3: return pick_fb_zb<3, T>(fb, tr);
    default: return pick_fb_zb<4, T>(fb, tr);
  }
}
KFn pick_policy_zb(int tick, int v, bool fb, bool tr) {
  if (tick == kTickI64) return pick_v_zb<int64_t>(v, fb, tr);
  if (tick == kTickF32) return pick_v_zb<float>(v, fb, tr);
  return pick_v_zb<int32_t>(v, fb, tr);
}

}  // namespace adaptis
