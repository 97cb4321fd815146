// loadtrace.cu — the schedule's load post-passes on the device, one CTA per
// traced candidate:
//   compute_idle_avgs   (sim.cpp:670-702)  idle_avg of every assignment
//   compute_load_trace  (sim.cpp:975-991)  the (time, active) step function
//   busy_time, LoadTrace::integral (sim.cpp:71-87)
//
// Layout: the detail/schedule kernels leave (proc, start, end) by task id
// (proc < 0: not a scheduled leaf).  The CTA collects one 64-bit key per
// start and per end event -- the non-negative time's bit pattern shifted left
// by one, the low bit set for an end -- so one ascending sort of the keys
// orders the events by time (bit patterns of non-negative doubles order like
// the values), and the low bit carries the +1 / -1 of each event.  A bitonic
// sort runs in shared memory (global scratch when the keys do not fit).  Two
// block scans give every group of equal times its index and the running
// active count at its last event.  The reference's sums are left folds, so
// the cumulative idle integral, the load integral and the busy time run as
// serial loops on three threads in the reference's order (plain IEEE adds and
// multiplies: the library is built with --fmad=false); each assignment's
// idle average is then an independent binary search over the step times.
#include <cuda_runtime.h>

#include <cub/block/block_scan.cuh>

#include <cstdint>
#include <vector>

#include "trace.h"

namespace hx {
namespace {

constexpr int LT_THREADS = 1024;

__device__ __forceinline__ unsigned long long ev_key(double t, bool is_end) {
  const double c = t == 0.0 ? 0.0 : t;  // one key for +0 and -0 (equal in the reference's grouping)
  return ((unsigned long long)__double_as_longlong(c) << 1) | (is_end ? 1ull : 0ull);
}
__device__ __forceinline__ double ev_time(unsigned long long k) { return __longlong_as_double((long long)(k >> 1)); }

__global__ void __launch_bounds__(LT_THREADS) load_trace_kernel(
    const int32_t* __restrict__ proc, const double* __restrict__ start, const double* __restrict__ end, int nid,
    int P, unsigned long long* gkeys, int key_cap, double* times, int32_t* active, double* cum, double* idle,
    double* scal) {
  extern __shared__ unsigned long long s_keys[];
  using Scan = cub::BlockScan<int, LT_THREADS>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int s_n, s_g;
  const int tid = threadIdx.x;
  const size_t q = blockIdx.x;
  proc += q * nid;
  start += q * nid;
  end += q * nid;
  times += q * nid;
  active += q * nid;
  cum += q * nid;
  idle += q * nid;
  scal += q * 4;
  unsigned long long* keys = gkeys ? gkeys + q * (size_t)key_cap : s_keys;
  if (tid == 0) s_n = 0;
  __syncthreads();
  // events (any order: they are sorted next)
  for (int i = tid; i < nid; i += LT_THREADS) {
    idle[i] = 0.0;
    if (proc[i] < 0) continue;
    const int at = atomicAdd(&s_n, 2);
    if (at + 1 < key_cap) {
      keys[at] = ev_key(start[i], false);
      keys[at + 1] = ev_key(end[i], true);
    }
  }
  __syncthreads();
  const int n = s_n;
  if (n > key_cap) {  // more scheduled leaves than the slot holds: not a trace this engine wrote
    if (tid == 0) scal[0] = -1.0;
    return;
  }
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = n + tid; i < m; i += LT_THREADS) keys[i] = ~0ull;
  __syncthreads();
  // bitonic sort, ascending
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < m; i += LT_THREADS) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long a = keys[i], b = keys[l];
          if ((a > b) == ((i & k) == 0)) {
            keys[i] = b;
            keys[l] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  // groups of equal times: index = heads so far - 1; active = running sum of
  // the deltas at the group's last event
  int carry_g = 0, carry_a = 0;
  for (int base = 0; base < n; base += LT_THREADS) {
    const int i = base + tid;
    const bool in = i < n;
    const unsigned long long t2 = in ? keys[i] >> 1 : 0ull;
    const int head = in && (i == 0 || (keys[i - 1] >> 1) != t2) ? 1 : 0;
    const int d = in ? ((keys[i] & 1ull) ? -1 : 1) : 0;
    int hs, ds, htot, dtot;
    Scan(scan_tmp).InclusiveSum(head, hs, htot);
    __syncthreads();
    Scan(scan_tmp).InclusiveSum(d, ds, dtot);
    __syncthreads();
    if (in && (i == n - 1 || (keys[i + 1] >> 1) != t2)) {
      const int g = carry_g + hs - 1;
      times[g] = ev_time(keys[i]);
      active[g] = carry_a + ds;
    }
    carry_g += htot;
    carry_a += dtot;
  }
  if (tid == 0) s_g = carry_g;
  __syncthreads();
  const int G = s_g;
  // the reference's left folds
  if (tid == 0) {  // cumulative idle integral up to each step time
    double c = 0.0;
    if (G > 0) cum[0] = 0.0;
    for (int i = 1; i < G; ++i) {
      c = c + (P - active[i - 1]) * (times[i] - times[i - 1]);
      cum[i] = c;
    }
  } else if (tid == 32) {  // LoadTrace::integral
    double s = 0.0;
    for (int i = 0; i + 1 < G; ++i) s += active[i] * (times[i + 1] - times[i]);
    scal[2] = s;
  } else if (tid == 64) {  // busy_time over the assignments in task-id order
    double s = 0.0;
    for (int i = 0; i < nid; ++i)
      if (proc[i] >= 0) s += end[i] - start[i];
    scal[1] = s;
  }
  __syncthreads();
  // idle_avg of each assignment: idle integral over [start, end) / duration
  auto idle_up_to = [&](double t) -> double {
    int lo = 0, hi = G;  // first step time > t (std::upper_bound)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (times[mid] > t) hi = mid;
      else lo = mid + 1;
    }
    if (lo == 0) return 0.0;
    const int k = lo - 1;
    return cum[k] + (P - active[k]) * (t - times[k]);
  };
  for (int i = tid; i < nid; i += LT_THREADS) {
    if (proc[i] < 0) continue;
    const double a = start[i], b = end[i];
    const double dur = b - a;
    idle[i] = dur > 0 ? (idle_up_to(b) - idle_up_to(a)) / dur : 0.0;
  }
  if (tid == 0) {
    scal[0] = (double)G;
    scal[3] = (double)(n / 2);
  }
}

}  // namespace

size_t load_trace_scratch_bytes(int nid, int B) {
  int cap = 1;
  while (cap < nid) cap <<= 1;
  const size_t per = (size_t)nid * (8 + 4 + 8 + 8) + 4 * 8;
  const size_t keys = (size_t)cap * 8 > LOAD_TRACE_SMEM ? (size_t)cap * 8 : 0;
  return (size_t)B * (per + keys) + 256 * 6;
}

int load_trace_device(const int32_t* proc, const double* start, const double* end, int nid, int B, int P,
                      void* scratch, cudaStream_t st, std::vector<TraceLogs*>& out) {
  int cap = 1;
  while (cap < nid) cap <<= 1;
  const bool in_smem = (size_t)cap * 8 <= LOAD_TRACE_SMEM;
  auto carve = [&](size_t bytes) {
    uint8_t* p = (uint8_t*)scratch;
    scratch = p + ((bytes + 255) & ~(size_t)255);
    return (void*)p;
  };
  double* times = (double*)carve((size_t)B * nid * 8);
  int32_t* active = (int32_t*)carve((size_t)B * nid * 4);
  double* cum = (double*)carve((size_t)B * nid * 8);
  double* idle = (double*)carve((size_t)B * nid * 8);
  double* scal = (double*)carve((size_t)B * 4 * 8);
  unsigned long long* gkeys = in_smem ? nullptr : (unsigned long long*)carve((size_t)B * cap * 8);
  const size_t smem = in_smem ? (size_t)cap * 8 : 0;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(load_trace_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return HESP_E_CUDA;
  load_trace_kernel<<<B, LT_THREADS, smem, st>>>(proc, start, end, nid, P, gkeys, cap, times, active, cum, idle, scal);
  if (cudaGetLastError() != cudaSuccess) return HESP_E_CUDA;
  std::vector<double> hs((size_t)B * 4);
  if (cudaMemcpyAsync(hs.data(), scal, hs.size() * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return HESP_E_CUDA;
  for (int b = 0; b < B; ++b) {
    TraceLogs* L = out[b];
    if (!L) continue;
    const int G = (int)hs[4 * b];
    if (G < 0) return HESP_E_LIMIT;
    L->steps_time.resize(G);
    L->steps_active.resize(G);
    L->idle.resize(nid);
    L->busy = hs[4 * b + 1];
    L->integral = hs[4 * b + 2];
    if (cudaMemcpyAsync(L->steps_time.data(), times + (size_t)b * nid, (size_t)G * 8, cudaMemcpyDeviceToHost, st) !=
            cudaSuccess ||
        cudaMemcpyAsync(L->steps_active.data(), active + (size_t)b * nid, (size_t)G * 4, cudaMemcpyDeviceToHost,
                        st) != cudaSuccess ||
        cudaMemcpyAsync(L->idle.data(), idle + (size_t)b * nid, (size_t)nid * 8, cudaMemcpyDeviceToHost, st) !=
            cudaSuccess)
      return HESP_E_CUDA;
    L->has_load = true;
  }
  return cudaStreamSynchronize(st) == cudaSuccess ? HESP_OK : HESP_E_CUDA;
}

}  // namespace hx
