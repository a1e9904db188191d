// adaptis_inst_list.cu — instantiations of the segment kernel for explicit
// per-device task orders (ADAPTIS_LIST / ADAPTIS_LIST_FUSED, reading R30).
#include "adaptis_seg.cuh"

namespace adaptis {

template <int POLICY, int V, typename T>
static KFn pick_fb_list(bool fallback, bool trace) {
  if (trace) return (KFn)seg_kernel<POLICY, V, T, true, true>;
  return fallback ? (KFn)seg_kernel<POLICY, V, T, true> : (KFn)seg_kernel<POLICY, V, T, false>;
}
template <int POLICY, typename T>
static KFn pick_v_list(int v, bool fb, bool tr) {
  switch (v) {
    case 1: return pick_fb_list<POLICY, 1, T>(fb, tr);
    case 2: return pick_fb_list<POLICY, 2, T>(fb, tr);
    case 3: return pick_fb_list<POLICY, 3, T>(fb, tr);
    default: return pick_fb_list<POLICY, 4, T>(fb, tr);
  }
}
// integer ticks only (adaptis_eval_lists rejects the FP32 cost mode)
KFn pick_policy_list(int tick, int v, bool fb, bool tr, bool fused) {
  if (fused) {
    if (tick == kTickI64) return pick_v_list<ADAPTIS_LIST_FUSED, int64_t>(v, fb, tr);
    return pick_v_list<ADAPTIS_LIST_FUSED, int32_t>(v, fb, tr);
  }
  if (tick == kTickI64) return pick_v_list<ADAPTIS_LIST, int64_t>(v, fb, tr);
  return pick_v_list<ADAPTIS_LIST, int32_t>(v, fb, tr);
}

}  // namespace adaptis
