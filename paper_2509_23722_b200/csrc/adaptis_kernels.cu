// adaptis_kernels.cu — launchers of the segment kernels (adaptis_seg.cuh,
// instantiated per policy in adaptis_inst_*.cu) and the R29 accounting kernel.
#include "adaptis_seg.cuh"

namespace adaptis {

// ------------------------------------------------------------------------------
static WarpLayout host_layout(const SegLaunch& s, bool gring) {
  const int tsz = s.tick == kTickI64 ? 8 : 4;
  const int rsz = s.tick == kTickI64 ? (int)sizeof(Rec<int64_t>)
                : s.tick == kTickF32 ? (int)sizeof(Rec<float>) : (int)sizeof(Rec<int32_t>);
  const int gsz = s.policy != ADAPTIS_GREEDY ? 0
                : s.tick == kTickI64 ? (int)sizeof(GAux<int64_t>)
                : s.tick == kTickF32 ? (int)sizeof(GAux<float>) : (int)sizeof(GAux<int32_t>);
  return warp_layout(s.S, s.G, s.v, s.ring_k, tsz, rsz, gring, gsz);
}

size_t smem_bytes(const SegLaunch& s, bool fallback) {
  const WarpLayout l = host_layout(s, fallback);
  return l.prefix_bytes(s.L) + (size_t)kWarpsPerCta * l.per_warp;
}

// report launches with a trace (R29) use the global-ring kernel instantiated
// with TRACE (integer ticks only); every other launch keeps its hot kernel.
// The instantiations live in one translation unit per policy (adaptis_inst_*.cu).
static KFn pick(const SegLaunch& s, bool fb) {
  const bool tr = s.trace != nullptr;
  switch (s.policy) {
    case ADAPTIS_GPIPE: return pick_policy_gpipe(s.tick, s.v, fb, tr);
    case ADAPTIS_ONEF1B: return pick_policy_onef1b(s.tick, s.v, fb, tr);
    case ADAPTIS_ZB: return pick_policy_zb(s.tick, s.v, fb, tr);
    case ADAPTIS_LIST: return pick_policy_list(s.tick, s.v, fb, tr, false);
    case ADAPTIS_LIST_FUSED: return pick_policy_list(s.tick, s.v, fb, tr, true);
    default: return pick_policy_greedy(s.tick, s.v, fb, tr);
  }
}

// ---- R29 communication accounting: one thread per (candidate, device)
__global__ void comm_account_kernel(const TraceEntry* __restrict__ trace, const int* __restrict__ trace_n,
                                    int cap, int p, uint64_t n, int64_t* __restrict__ report) {
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= n * (uint64_t)p) return;
  const uint64_t o = gid / p;
  const int d = (int)(gid % p);
  int64_t* rep = report + o * 5 * p;
  const int64_t Td = rep[d];
  const TraceEntry* base = trace + o * p * (size_t)cap;
  int ptr[ADAPTIS_MAX_P], len[ADAPTIS_MAX_P];
  for (int l = 0; l < p; ++l) {
    ptr[l] = 0;
    const int k = trace_n[o * p + l];
    len[l] = k < cap ? k : cap;
  }
  const TraceEntry* own = base + (size_t)d * cap;
  // transfers incident to d: d's own outputs to other devices, and every
  // device's outputs to d; each device's trace is in execution order, so every
  // stream is sorted by transfer start (= producer finish): a p-way merge
  auto relevant = [&](int l, const TraceEntry& e) {
    return e.oc > 0 && e.tgt >= 0 && (l == d ? e.tgt != d : e.tgt == d);
  };
  int64_t comm = 0, exposed = 0, u0 = 0, u1 = -1;
  int ci = 0;  // first compute interval of d that may still overlap a union segment
  auto flush = [&]() {  // |[u0, u1] clipped to [0, Td] minus d's compute intervals|
    const int64_t a = u0 < 0 ? 0 : u0, b = u1 < Td ? u1 : Td;
    if (b <= a) return;
    while (ci < len[d] && own[ci].fin <= a) ++ci;
    int64_t covered = 0;
    for (int j = ci; j < len[d] && own[j].start < b; ++j) {
      const int64_t x = own[j].start > a ? own[j].start : a;
      const int64_t y = own[j].fin < b ? own[j].fin : b;
      if (y > x) covered += y - x;
    }
    exposed += (b - a) - covered;
  };
  for (;;) {
    int best = -1;
    int64_t bs = 0;
    for (int l = 0; l < p; ++l) {
      while (ptr[l] < len[l] && !relevant(l, base[(size_t)l * cap + ptr[l]])) ++ptr[l];
      if (ptr[l] < len[l]) {
        const int64_t st = base[(size_t)l * cap + ptr[l]].fin;
        if (best < 0 || st < bs) { best = l; bs = st; }
      }
    }
    if (best < 0) break;
    const TraceEntry& e = base[(size_t)best * cap + ptr[best]];
    ++ptr[best];
    const int64_t a = e.fin, b = e.fin + e.oc;
    comm += e.oc;
    if (u1 < 0 || a > u1) {  // a new disjoint union segment
      if (u1 >= 0) flush();
      u0 = a; u1 = b;
    } else if (b > u1) {
      u1 = b;
    }
  }
  if (u1 >= 0) flush();
  rep[3 * p + d] = comm;
  rep[4 * p + d] = exposed;
}

int launch_comm_account(const TraceEntry* trace, const int* trace_n, int trace_cap, int p,
                        uint64_t n, int64_t* report, void* stream) {
  if (n == 0) return 0;
  const uint64_t threads = n * (uint64_t)p;
  const unsigned grid = (unsigned)((threads + 127) / 128);
  comm_account_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(trace, trace_n, trace_cap, p, n, report);
  return (int)cudaGetLastError();
}

int occupancy_ctas_per_sm(const SegLaunch& s, bool fallback) {
  KFn f = pick(s, fallback);
  const size_t sm = smem_bytes(s, fallback);
  if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
    return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, kWarpsPerCta * 32, sm) != cudaSuccess)
    return 0;
  return n;
}

int launch_segment(const DevTables& t, const SegLaunch& s, int num_sms, void* stream,
                   bool fallback, unsigned grid_limit) {
  KFn f = pick(s, fallback);
  const size_t sm = smem_bytes(s, fallback);
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return (int)e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, kWarpsPerCta * 32, sm);
  if (e != cudaSuccess) return (int)e;
  if (per_sm < 1) return (int)cudaErrorInvalidConfiguration;
  unsigned grid = (unsigned)num_sms * (unsigned)per_sm;
  const uint64_t warps_needed = (s.n_pos + s.G - 1) / s.G;
  const uint64_t ctas_needed = (warps_needed + kWarpsPerCta - 1) / kWarpsPerCta;
  if (ctas_needed < grid) grid = (unsigned)(ctas_needed ? ctas_needed : 1);
  if (grid_limit && grid > grid_limit) grid = grid_limit;
  f<<<grid, kWarpsPerCta * 32, sm, (cudaStream_t)stream>>>(t, s);
  return (int)cudaGetLastError();
}

// ---- memory timeline (R35): one thread per (plan, device) walks the device's
// trace in execution order; F allocates act + stash at its start, B frees act
// (+ stash when fused) at its end, W frees stash at its end (R16)
__global__ void mem_timeline_kernel(const TraceEntry* __restrict__ trace, const int* __restrict__ trace_n,
                                    int cap_t, int p, uint64_t n, const int16_t* __restrict__ cuts,
                                    const int32_t* __restrict__ plan_info, const int64_t* __restrict__ pre,
                                    int L, int64_t cap, adaptis_mem_point* __restrict__ points, int pcap,
                                    int* __restrict__ npts, int64_t* __restrict__ first) {
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= n * (uint64_t)p) return;
  const uint64_t o = gid / p;
  const int d = (int)(gid % p);
  const int info = plan_info[o];
  const int v = info & 15, placement = (info >> 4) & 15;
  const bool fused = (info >> 8) & 1;
  const int S = p * v;
  const int16_t* c = cuts + o * (ADAPTIS_MAX_S + 1);
  auto col = [&](int k, int a, int b) { return pre[(size_t)k * (L + 1) + b] - pre[(size_t)k * (L + 1) + a]; };
  int64_t stat = 0;
  for (int s = 0; s < S; ++s)
    if (dev_of(placement, p, s) == d) stat += col(kColWG, c[s], c[s + 1]);
  adaptis_mem_point* out = points + gid * (size_t)pcap;
  int k = 0;
  int64_t bytes = stat, fv = -1;
  out[k].time = 0; out[k].bytes = bytes; ++k;
  if (bytes > cap) fv = 0;
  const int nt = min(trace_n[gid], cap_t);
  const TraceEntry* tr = trace + gid * (size_t)cap_t;
  for (int i = 0; i < nt && k < pcap; ++i) {
    const TraceEntry e = tr[i];
    const int s = e.stage;
    const int64_t act = col(kColAct, c[s], c[s + 1]), sta = col(kColStash, c[s], c[s + 1]);
    int64_t delta, t;
    if (e.kind == 0) { delta = act + sta; t = e.start; }
    else if (e.kind == 1) { delta = -(act + (fused ? sta : 0)); t = e.fin; }
    else { delta = -sta; t = e.fin; }
    bytes += delta;
    out[k].time = t; out[k].bytes = bytes; ++k;
    if (fv < 0 && bytes > cap) fv = t;
  }
  npts[gid] = k;
  first[gid] = fv;
}

int launch_mem_timeline(const TraceEntry* trace, const int* trace_n, int trace_cap, int p, uint64_t n,
                        const int16_t* cuts, const int32_t* plan_info, const int64_t* pre, int L,
                        int64_t cap, adaptis_mem_point* points, int pcap, int* npts, int64_t* first,
                        void* stream) {
  if (n == 0) return 0;
  const uint64_t threads = n * (uint64_t)p;
  const unsigned grid = (unsigned)((threads + 127) / 128);
  mem_timeline_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(trace, trace_n, trace_cap, p, n, cuts, plan_info,
                                                              pre, L, cap, points, pcap, npts, first);
  return (int)cudaGetLastError();
}

}  // namespace adaptis
