// verify.cu — schedule validation on the device:
// the four checks of the reference's verify_schedule (sim.cpp:857-973),
// designed as independent data-parallel passes over one traced candidate.
//
//   (a) overlap   one CTA per processor: its assignments ranked by
//                 (start, task) in shared memory, adjacent pairs compared;
//   (b) edges     one warp per leaf: every predecessor in the engine's
//                 closure-equivalent relation (E2) checked; a
//                 violated pair is reported only if it is a covering pair of
//                 the dependence order (no longer path), which is exactly the
//                 reference's transitively reduced TaskGraph::edges();
//   (c) coherence one warp per read: the writes of the read block's base tile
//                 (every region except the root's lies inside one tile) give
//                 the fragment grid; lanes take the cells, find the freshest
//                 write before the read and look for a local copy, the
//                 initial data, or a transfer into the space that arrived in
//                 time, over the transfers of the same (space, tile);
//   (d) capacity  one warp: a segmented prefix sum of the residency log per
//                 space.
// Each violation is a record (kind, ordering keys); the host sorts the
// records into the reference's report order (processor id / edge order /
// task id and read index / log order) and formats its messages.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>

#include "engine_types.h"
#include "hesp_engine.h"
#include "problem.h"
#include "trace.h"

namespace hx {
namespace {

struct Viol {
  int32_t kind;  // 0 overlap, 1 edge, 2 read, 3 capacity
  int32_t key1, key2;
  int32_t a, b, c;
  double t;
};

struct VRegion {
  int32_t row, col, rows, cols;
};

__device__ __forceinline__ bool vcontains(const VRegion& o, const VRegion& i) {
  return i.row >= o.row && i.col >= o.col && i.row + i.rows <= o.row + o.rows && i.col + i.cols <= o.col + o.cols;
}
__device__ __forceinline__ bool voverlap(const VRegion& a, const VRegion& b) {
  return a.row < b.row + b.rows && b.row < a.row + a.rows && a.col < b.col + b.cols && b.col < a.col + a.cols;
}
__device__ __forceinline__ int vclamp(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ void emit(Viol* out, int* nout, int cap, Viol v) {
  const int k = atomicAdd(nout, 1);
  if (k < cap) out[k] = v;
}

// (a) one CTA per processor; smem: n_p x (start, end, task, rank)
__global__ void vfy_overlap(const int32_t* __restrict__ task, const int32_t* __restrict__ proc,
                            const double* __restrict__ st, const double* __restrict__ en, int na, double eps,
                            Viol* out, int* nout, int cap) {
  extern __shared__ unsigned char sm[];
  __shared__ int cnt;
  const int p = blockIdx.x;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  // this processor's assignments (order irrelevant: ranked below)
  int maxn = 0;
  for (int i = threadIdx.x; i < na; i += blockDim.x)
    if (proc[i] == p) atomicAdd(&cnt, 1);
  __syncthreads();
  maxn = cnt;
  double* s0 = (double*)sm;
  double* s1 = s0 + maxn;
  int32_t* tk = (int32_t*)(s1 + maxn);
  int32_t* ord = tk + maxn;
  __syncthreads();
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < na; i += blockDim.x)
    if (proc[i] == p) {
      const int k = atomicAdd(&cnt, 1);
      s0[k] = st[i];
      s1[k] = en[i];
      tk[k] = task[i];
    }
  __syncthreads();
  // rank by (start, task): list sorted by start (sim.cpp:865-866)
  for (int i = threadIdx.x; i < maxn; i += blockDim.x) {
    int r = 0;
    for (int j = 0; j < maxn; ++j) r += s0[j] < s0[i] || (s0[j] == s0[i] && tk[j] < tk[i]);
    ord[r] = i;
  }
  __syncthreads();
  for (int r = 1 + threadIdx.x; r < maxn; r += blockDim.x) {
    const int prev = ord[r - 1], cur = ord[r];
    if (s0[cur] < s1[prev] - eps) emit(out, nout, cap, Viol{0, p, r, tk[prev], tk[cur], 0, 0.0});
  }
}

// (b) one warp per leaf (program rank v): candidate violated pairs (u, v)
__global__ void vfy_edges(const int32_t* __restrict__ leaves, const int32_t* __restrict__ poff,
                          const int32_t* __restrict__ pcnt, const int32_t* __restrict__ preds,
                          const int32_t* __restrict__ rank_of, const int32_t* __restrict__ aproc,
                          const double* __restrict__ ast, const double* __restrict__ aen, int n, double eps,
                          Viol* out, int* nout, int cap) {
  const int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= n) return;
  const int dst = leaves[v];
  for (int q = lane; q < pcnt[v]; q += 32) {
    const int src = preds[poff[v] + q];
    const int u = rank_of[src];
    if (u < 0) continue;
    const bool missing = aproc[src] < 0 || aproc[dst] < 0;
    if (missing || ast[dst] < aen[src] - eps) emit(out, nout, cap, Viol{1, u, v, src, dst, missing ? 1 : 0, 0.0});
  }
}

// (c) one warp per (leaf, read slot).  The fragment grid's lines are kept as
// bitmaps over the read's extent (offsets 0..cols / 0..rows) in shared
// memory -- duplicates cost nothing -- and expanded to sorted line lists.
constexpr int VW = 4;          // warps per CTA
constexpr int VDIST = 512;     // distinct grid lines per axis (overflow is reported)
__global__ void __launch_bounds__(VW * 32) vfy_reads(
    const int32_t* __restrict__ rd_task, const int32_t* __restrict__ rd_k, const int32_t* __restrict__ rd_blk,
    const int32_t* __restrict__ rd_space, const double* __restrict__ rd_start, const int32_t* __restrict__ rd_tile,
    int nreads, const VRegion* __restrict__ breg,
    // writes by tile (CSR; task-id order inside a tile); the last bucket holds regions spanning tiles
    const int32_t* __restrict__ w_off, const VRegion* __restrict__ w_reg, const double* __restrict__ w_end,
    const int32_t* __restrict__ w_space, int ntile_buckets,
    // transfers by (dst space, tile) (CSR), same spanning bucket per space
    const int32_t* __restrict__ x_off, const VRegion* __restrict__ x_reg, const double* __restrict__ x_end,
    int main_space, double eps, int bm_words, Viol* out, int* nout, int cap) {
  extern __shared__ uint32_t vsm[];  // per warp: x bitmap, y bitmap (bm_words each), x list, y list (VDIST each)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * VW + w;
  if (r >= nreads) return;
  uint32_t* bx = vsm + (size_t)w * (2 * bm_words + 2 * VDIST);
  uint32_t* by = bx + bm_words;
  int* xu = (int*)(by + bm_words);
  int* yu = xu + VDIST;
  const VRegion rr = breg[rd_blk[r]];
  const int space = rd_space[r];
  const double a = rd_start[r];
  const int T = rd_tile[r];
  const int span = ntile_buckets - 1;  // bucket of tile-spanning regions
  // the writes to scan: the read's tile and the spanning bucket (a spanning
  // read -- the root -- scans every bucket)
  const int b0 = T < 0 ? 0 : T, b1 = T < 0 ? span : T;
  auto for_buckets = [&](auto&& f) {
    for (int bk = b0; bk <= b1; ++bk) f(bk);
    if (T >= 0) f(span);
  };
  const int wx = (rr.cols >> 5) + 1, wy = (rr.rows >> 5) + 1;  // bitmap words in use
  for (int k = lane; k < wx; k += 32) bx[k] = 0;
  for (int k = lane; k < wy; k += 32) by[k] = 0;
  __syncwarp();
  if (lane == 0) {
    atomicOr(&bx[0], 1u);
    atomicOr(&bx[rr.cols >> 5], 1u << (rr.cols & 31));
    atomicOr(&by[0], 1u);
    atomicOr(&by[rr.rows >> 5], 1u << (rr.rows & 31));
  }
  // every overlapping write's edges, clamped to the read (sim.cpp:908-916)
  for_buckets([&](int bk) {
    for (int i = w_off[bk] + lane; i < w_off[bk + 1]; i += 32) {
      const VRegion wr = w_reg[i];
      if (!voverlap(wr, rr)) continue;
      const int x0 = vclamp(wr.col, rr.col, rr.col + rr.cols) - rr.col;
      const int x1 = vclamp(wr.col + wr.cols, rr.col, rr.col + rr.cols) - rr.col;
      const int y0 = vclamp(wr.row, rr.row, rr.row + rr.rows) - rr.row;
      const int y1 = vclamp(wr.row + wr.rows, rr.row, rr.row + rr.rows) - rr.row;
      atomicOr(&bx[x0 >> 5], 1u << (x0 & 31));
      atomicOr(&bx[x1 >> 5], 1u << (x1 & 31));
      atomicOr(&by[y0 >> 5], 1u << (y0 & 31));
      atomicOr(&by[y1 >> 5], 1u << (y1 & 31));
    }
  });
  __syncwarp();
  // sorted distinct lines: word-wise popcount prefix sums
  auto expand = [&](const uint32_t* bm, int words, int origin, int* list) -> int {
    int n = 0;
    for (int base = 0; base < words; base += 32) {
      const int k = base + lane;
      const uint32_t m = k < words ? bm[k] : 0u;
      const int c = __popc(m);
      int incl = c;
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      int at = n + incl - c;
      for (uint32_t mm = m; mm; mm &= mm - 1, ++at)
        if (at < VDIST) list[at] = origin + 32 * k + (__ffs((int)mm) - 1);
      n += __shfl_sync(0xffffffffu, incl, 31);
    }
    return n;
  };
  const int nxu = expand(bx, wx, rr.col, xu);
  const int nyu = expand(by, wy, rr.row, yu);
  __syncwarp();
  if (nxu > VDIST || nyu > VDIST) {
    if (lane == 0) emit(out, nout, cap, Viol{-1, 0, 0, rd_task[r], 0, 0, 0.0});
    return;
  }
  // ---- cells: freshest write before the read, then a copy that is fresh here
  const int ncell = (nxu - 1) * (nyu - 1);
  bool bad = false;
  for (int c = lane; c < ncell && !bad; c += 32) {
    const int yi = c / (nxu - 1), xi = c - yi * (nxu - 1);
    const VRegion cell{yu[yi], xu[xi], yu[yi + 1] - yu[yi], xu[xi + 1] - xu[xi]};
    double wend = -1.0;
    int wsp = main_space;
    // ties on the end time go to the earliest task id (strict >, task-id order)
    for_buckets([&](int bk) {
      for (int i = w_off[bk]; i < w_off[bk + 1]; ++i) {
        const double e = w_end[i];
        if (e > a + eps) continue;
        if (!vcontains(w_reg[i], cell)) continue;
        if (e > wend) {
          wend = e;
          wsp = w_space[i];
        }
      }
    });
    bool ok = (wend >= 0.0 && wsp == space) || (wend < 0.0 && space == main_space);
    if (!ok) {
      const double lower = wend > 0.0 ? wend : 0.0;
      const int xb0 = space * ntile_buckets;
      auto scan = [&](int bk) {
        for (int i = x_off[xb0 + bk]; i < x_off[xb0 + bk + 1] && !ok; ++i) {
          const double e = x_end[i];
          if (e <= a + eps && e >= lower - eps && vcontains(x_reg[i], cell)) ok = true;
        }
      };
      for_buckets(scan);
    }
    bad = !ok;
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0)
    emit(out, nout, cap, Viol{2, rd_task[r], rd_k[r], rd_task[r], rd_blk[r], space, 0.0});
}

// (d) one warp: used bytes per space after every residency change, in log order
__global__ void vfy_capacity(const int32_t* __restrict__ sp, const int64_t* __restrict__ delta,
                             const double* __restrict__ t, int n, const int64_t* __restrict__ cap_b, int S, Viol* out,
                             int* nout, int cap) {
  const int lane = threadIdx.x & 31;
  long long carry[MAXS];
  for (int q = 0; q < MAXS; ++q) carry[q] = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const int s = i < n ? sp[i] : -1;
    const long long d = i < n ? (long long)delta[i] : 0;
    for (int q = 0; q < S; ++q) {
      long long v = s == q ? d : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const long long u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      const long long used = carry[q] + v;
      if (s == q) {
        if (used > cap_b[q]) emit(out, nout, cap, Viol{3, i, 0, q, 0, 0, t[i]});
        if (used < 0) emit(out, nout, cap, Viol{3, i, 1, q, 0, 0, t[i]});
      }
      carry[q] += __shfl_sync(0xffffffffu, v, 31);
    }
  }
}

template <class T>
struct DBuf {
  T* p = nullptr;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  bool put(const std::vector<T>& v, cudaStream_t st) {
    if (cudaMalloc(&p, (v.empty() ? 1 : v.size()) * sizeof(T)) != cudaSuccess) return false;
    return v.empty() || cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st) == cudaSuccess;
  }
};

}  // namespace

int verify_trace_device(const Problem& P, const TraceGraph& g, const hesp_trace& tr, cudaStream_t st,
                        std::vector<std::string>& out) {
  out.clear();
  const double eps = 1e-9 * std::max(1.0, tr.outcome.makespan);
  const int na = tr.n_assign, n = (int)g.leaves.size();
  // assignments by task id (the trace may have been edited by the caller)
  int maxid = 0;
  for (int i = 0; i < na; ++i) maxid = std::max(maxid, tr.assignments[i].task);
  for (int v = 0; v < n; ++v) maxid = std::max(maxid, g.leaves[v]);
  const int ids = maxid + 1;
  std::vector<int32_t> a_task(na), a_proc(na), rank_of(ids, -1), aproc(ids, -1);
  std::vector<double> a_st(na), a_en(na), ast(ids, 0.0), aen(ids, 0.0);
  for (int i = 0; i < na; ++i) {
    const hesp_assignment& a = tr.assignments[i];
    a_task[i] = a.task;
    a_proc[i] = a.proc;
    a_st[i] = a.start;
    a_en[i] = a.end;
    aproc[a.task] = a.proc;
    ast[a.task] = a.start;
    aen[a.task] = a.end;
  }
  for (int v = 0; v < n; ++v) rank_of[g.leaves[v]] = v;
  // base tile of a region (row-major over the n/base_b grid); -1 = spans tiles
  const long long bb = P.base_b;
  const int G = (int)(P.n / bb);
  auto tile_of = [&](const Region& r) -> int {
    if (r.rows <= 0 || r.cols <= 0) return -1;
    const long long r0 = r.row / bb, c0 = r.col / bb;
    if ((r.row + r.rows - 1) / bb != r0 || (r.col + r.cols - 1) / bb != c0) return -1;
    return (int)(r0 * G + c0);
  };
  const int NT = G * G + 1;  // tile buckets + the spanning bucket
  auto bucket = [&](const Region& r) {
    const int t = tile_of(r);
    return t < 0 ? NT - 1 : t;
  };
  // writes (one per assigned leaf), by bucket, task-id order within a bucket
  std::vector<int32_t> w_off(NT + 1, 0), w_space, order;
  std::vector<VRegion> w_reg;
  std::vector<double> w_end;
  {
    std::vector<std::pair<int, int>> key;  // (bucket, task) -> assignment index
    std::vector<int> aidx;
    for (int i = 0; i < na; ++i) {
      const int id = tr.assignments[i].task;
      if (id >= ids || rank_of[id] < 0) continue;
      const TaskMeta& m = g.meta[rank_of[id]];
      key.push_back({bucket(g.bregion[m.blk[m.nrd]]), id});
      aidx.push_back(i);
    }
    std::vector<int> idx(key.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = (int)i;
    std::sort(idx.begin(), idx.end(), [&](int x, int y) { return key[x] < key[y]; });
    for (int k : idx) {
      const hesp_assignment& a = tr.assignments[aidx[k]];
      const TaskMeta& m = g.meta[rank_of[a.task]];
      const Region rg = g.bregion[m.blk[m.nrd]];
      w_reg.push_back({rg.row, rg.col, rg.rows, rg.cols});
      w_end.push_back(a.end);
      w_space.push_back(P.proc_space[a.proc]);
      ++w_off[key[k].first + 1];
    }
    for (int b = 0; b < NT; ++b) w_off[b + 1] += w_off[b];
  }
  // transfers by (dst space, bucket)
  const int S = P.S;
  std::vector<int32_t> x_off((size_t)S * NT + 1, 0);
  std::vector<VRegion> x_reg;
  std::vector<double> x_end;
  {
    std::vector<std::pair<long long, int>> key;
    for (int i = 0; i < tr.n_xfer; ++i) {
      const hesp_transfer& x = tr.transfers[i];
      const Region xr = x.has_fragment ? Region{x.frag_row, x.frag_col, x.frag_rows, x.frag_cols} : g.bregion[x.block];
      key.push_back({(long long)x.dst_space * NT + bucket(xr), i});
    }
    std::sort(key.begin(), key.end());
    for (auto& [k, i] : key) {
      const hesp_transfer& x = tr.transfers[i];
      const Region xr = x.has_fragment ? Region{x.frag_row, x.frag_col, x.frag_rows, x.frag_cols} : g.bregion[x.block];
      x_reg.push_back({xr.row, xr.col, xr.rows, xr.cols});
      x_end.push_back(x.end);
      ++x_off[k + 1];
    }
    for (size_t b = 0; b + 1 < x_off.size(); ++b) x_off[b + 1] += x_off[b];
  }
  // reads: every (assigned leaf, read slot), task-id order
  std::vector<int32_t> rd_task, rd_k, rd_blk, rd_space, rd_tile;
  std::vector<double> rd_start;
  for (int i = 0; i < na; ++i) {
    const hesp_assignment& a = tr.assignments[i];
    if (a.task >= ids || rank_of[a.task] < 0) continue;
    const TaskMeta& m = g.meta[rank_of[a.task]];
    for (int k = 0; k < m.nrd; ++k) {
      rd_task.push_back(a.task);
      rd_k.push_back(k);
      rd_blk.push_back(m.blk[k]);
      rd_space.push_back(P.proc_space[a.proc]);
      rd_start.push_back(a.start);
      rd_tile.push_back(tile_of(g.bregion[m.blk[k]]));
    }
  }
  std::vector<VRegion> breg(g.bregion.size());
  for (size_t b = 0; b < breg.size(); ++b) breg[b] = {g.bregion[b].row, g.bregion[b].col, g.bregion[b].rows, g.bregion[b].cols};
  std::vector<int32_t> r_sp(tr.n_res);
  std::vector<int64_t> r_d(tr.n_res), capb(P.cap, P.cap + MAXS);
  std::vector<double> r_t(tr.n_res);
  for (int i = 0; i < tr.n_res; ++i) {
    r_sp[i] = tr.residency[i].space;
    r_d[i] = tr.residency[i].delta_bytes;
    r_t[i] = tr.residency[i].time;
  }
  // ---- device
  DBuf<int32_t> d_atask, d_aproc, d_leaves, d_poff, d_pcnt, d_preds, d_rank, d_aprocid, d_woff, d_wsp, d_xoff, d_rdt,
      d_rdk, d_rdb, d_rds, d_rdtile, d_rsp;
  DBuf<double> d_ast0, d_aen0, d_ast, d_aen, d_wend, d_xend, d_rdst, d_rt;
  DBuf<VRegion> d_breg, d_wreg, d_xreg;
  DBuf<int64_t> d_rd, d_cap;
  bool ok = d_atask.put(a_task, st) && d_aproc.put(a_proc, st) && d_ast0.put(a_st, st) && d_aen0.put(a_en, st) &&
            d_leaves.put(g.leaves, st) && d_poff.put(g.poff, st) && d_pcnt.put(g.pcnt, st) && d_preds.put(g.preds, st) &&
            d_rank.put(rank_of, st) && d_aprocid.put(aproc, st) && d_ast.put(ast, st) && d_aen.put(aen, st) &&
            d_breg.put(breg, st) && d_woff.put(w_off, st) && d_wreg.put(w_reg, st) && d_wend.put(w_end, st) &&
            d_wsp.put(w_space, st) && d_xoff.put(x_off, st) && d_xreg.put(x_reg, st) && d_xend.put(x_end, st) &&
            d_rdt.put(rd_task, st) && d_rdk.put(rd_k, st) && d_rdb.put(rd_blk, st) && d_rds.put(rd_space, st) &&
            d_rdst.put(rd_start, st) && d_rdtile.put(rd_tile, st) && d_rsp.put(r_sp, st) && d_rd.put(r_d, st) &&
            d_rt.put(r_t, st) && d_cap.put(capb, st);
  if (!ok) return HESP_E_CUDA;
  int cap = 1 << 16;
  Viol* d_out = nullptr;
  int* d_n = nullptr;
  std::vector<Viol> viols;
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (cudaMalloc(&d_out, (size_t)cap * sizeof(Viol)) != cudaSuccess || cudaMalloc(&d_n, sizeof(int)) != cudaSuccess ||
        cudaMemsetAsync(d_n, 0, sizeof(int), st) != cudaSuccess)
      return HESP_E_CUDA;
    // (a): shared memory sized by the busiest processor
    std::vector<int> per(P.P > 0 ? P.P : 1, 0);
    for (int i = 0; i < na; ++i)
      if (a_proc[i] >= 0 && a_proc[i] < P.P) ++per[a_proc[i]];
    const int mx = *std::max_element(per.begin(), per.end());
    const size_t smem = (size_t)mx * (8 + 8 + 4 + 4) + 16;
    cudaFuncSetAttribute(vfy_overlap, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (P.P > 0 && na > 0 && smem <= 200 * 1024)
      vfy_overlap<<<P.P, 256, smem, st>>>(d_atask.p, d_aproc.p, d_ast0.p, d_aen0.p, na, eps, d_out, d_n, cap);
    if (n > 0)
      vfy_edges<<<(n + 7) / 8, 256, 0, st>>>(d_leaves.p, d_poff.p, d_pcnt.p, d_preds.p, d_rank.p, d_aprocid.p, d_ast.p,
                                             d_aen.p, n, eps, d_out, d_n, cap);
    const int nreads = (int)rd_task.size();
    if (nreads > 0) {
      // bitmap words for the largest read extent
      int ext = 0;
      for (int b : rd_blk) ext = std::max(ext, std::max(g.bregion[b].rows, g.bregion[b].cols));
      const int bm_words = (ext >> 5) + 1;
      const size_t rsmem = (size_t)VW * (2 * bm_words + 2 * VDIST) * 4;
      if (rsmem > 200 * 1024) {
        set_last_error("verify: read extent too large for the device bitmaps");
        return HESP_E_LIMIT;
      }
      cudaFuncSetAttribute(vfy_reads, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem);
      vfy_reads<<<(nreads + VW - 1) / VW, VW * 32, rsmem, st>>>(d_rdt.p, d_rdk.p, d_rdb.p, d_rds.p, d_rdst.p, d_rdtile.p,
                                                               nreads, d_breg.p, d_woff.p, d_wreg.p, d_wend.p, d_wsp.p, NT,
                                                               d_xoff.p, d_xreg.p, d_xend.p, P.main_space, eps, bm_words,
                                                               d_out, d_n, cap);
    }
    if (tr.n_res > 0) vfy_capacity<<<1, 32, 0, st>>>(d_rsp.p, d_rd.p, d_rt.p, tr.n_res, d_cap.p, S, d_out, d_n, cap);
    int nv = 0;
    ok = cudaGetLastError() == cudaSuccess && cudaMemcpyAsync(&nv, d_n, sizeof(int), cudaMemcpyDeviceToHost, st) == cudaSuccess &&
         cudaStreamSynchronize(st) == cudaSuccess;
    if (ok && nv > cap) {  // too many violations for the record buffer: once more with room for all
      cudaFree(d_out);
      cudaFree(d_n);
      cap = nv;
      continue;
    }
    if (ok) {
      viols.resize(nv);
      ok = nv == 0 || (cudaMemcpy(viols.data(), d_out, (size_t)nv * sizeof(Viol), cudaMemcpyDeviceToHost) == cudaSuccess);
    }
    cudaFree(d_out);
    cudaFree(d_n);
    if (!ok) return HESP_E_CUDA;
    break;
  }
  for (const Viol& v : viols)
    if (v.kind < 0) {
      set_last_error("verify: a read's fragment grid exceeds the device scratch (VDIST lines per axis)");
      return HESP_E_LIMIT;
    }
  // (b) keep only covering pairs: (u, v) with no path of length >= 2 in the
  // dependence order (ranks strictly increase along every edge)
  std::vector<Viol> keep;
  std::vector<std::vector<int>> succ;
  std::vector<int> seen;
  int stamp = 0;
  for (const Viol& v : viols) {
    if (v.kind != 1) {
      keep.push_back(v);
      continue;
    }
    if (succ.empty()) {
      succ.assign(n, {});
      for (int w = 0; w < n; ++w)
        for (int q = 0; q < g.pcnt[w]; ++q) {
          const int u = rank_of[g.preds[g.poff[w] + q]];
          if (u >= 0) succ[u].push_back(w);
        }
      seen.assign(n, 0);
    }
    ++stamp;
    const int u = v.key1, target = v.key2;
    bool longer = false;
    std::vector<int> stack;
    for (int w : succ[u])
      if (w != target && w < target && seen[w] != stamp) {
        seen[w] = stamp;
        stack.push_back(w);
      }
    while (!stack.empty() && !longer) {
      const int x = stack.back();
      stack.pop_back();
      for (int y : succ[x]) {
        if (y == target) {
          longer = true;
          break;
        }
        if (y < target && seen[y] != stamp) {
          seen[y] = stamp;
          stack.push_back(y);
        }
      }
    }
    if (!longer) keep.push_back(v);
  }
  std::sort(keep.begin(), keep.end(), [](const Viol& x, const Viol& y) {
    if (x.kind != y.kind) return x.kind < y.kind;
    if (x.key1 != y.key1) return x.key1 < y.key1;
    return x.key2 < y.key2;
  });
  for (const Viol& v : keep) {
    switch (v.kind) {
      case 0:
        out.push_back("processor " + std::to_string(v.key1) + ": tasks " + std::to_string(v.a) + " and " +
                      std::to_string(v.b) + " overlap");
        break;
      case 1:
        if (v.c) out.push_back("edge endpoint not scheduled");
        else
          out.push_back("edge " + std::to_string(v.a) + "->" + std::to_string(v.b) +
                        " violated: dst starts before src ends");
        break;
      case 2:
        out.push_back("task " + std::to_string(v.a) + " reads block " + std::to_string(v.b) + " in space " +
                      std::to_string(v.c) + " without a fresh local copy");
        break;
      default:
        out.push_back("space " + std::to_string(v.a) + (v.key2 ? " under-run at t=" : " exceeds capacity at t=") +
                      std::to_string(v.t));
    }
  }
  return HESP_OK;
}

}  // namespace hx
