// trace.h — host side of the full-trace path (hesp_eval_trace /
// hesp_verify_trace): orders the device logs of one simulated candidate the
// way the reference's Engine::run does and derives its post-passes.
#pragma once

#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "engine_types.h"
#include "hesp_engine.h"

namespace hx {

// Graph of the traced candidate, exported by the device (TraceBufs).
struct TraceGraph {
  std::vector<int32_t> leaves;  // program order
  std::vector<TaskMeta> meta;   // per leaf
  std::vector<int32_t> poff, pcnt, preds;
  std::vector<Region> bregion;
  std::vector<int32_t> bisint;
  std::vector<PartEntry> parts;  // clusters by id; merged ones have task < 0
  std::vector<TaskMeta> tmeta;   // by task id
  bool valid = false;
};

// Device logs of one traced candidate, as copied back.
struct TraceLogs {
  std::vector<int32_t> proc;  // by task id (-1: not a scheduled leaf)
  std::vector<double> start, end;
  std::vector<XferLog> xfers;  // emission order
  std::vector<ResLog> res;     // emission order (ties are identical records)
  // load post-passes computed on the device (load_trace_device)
  bool has_load = false;
  std::vector<double> idle;  // idle_avg by task id
  std::vector<double> steps_time;
  std::vector<int32_t> steps_active;
  double busy = 0.0, integral = 0.0;
};

// Load post-passes (compute_idle_avgs, compute_load_trace, busy_time,
// LoadTrace::integral) of B traces on the device (loadtrace.cu): one CTA per
// trace over (proc, start, end) by task id (nid ids per trace, trace b at
// offset b * nid), scratch of load_trace_scratch_bytes(nid, B) device bytes;
// fills out[b] (skipped when null).  HESP_OK, HESP_E_CUDA or HESP_E_LIMIT.
constexpr size_t LOAD_TRACE_SMEM = 160 * 1024;  // sort keys in shared memory up to this size
size_t load_trace_scratch_bytes(int nid, int B);
int load_trace_device(const int32_t* proc, const double* start, const double* end, int nid, int B, int P,
                      void* scratch, cudaStream_t st, std::vector<TraceLogs*>& out);

// Rewrites an exported graph (and the logs' block ids) from the engine's
// internal ids to reference ids (BaseView offsets; identity when all are 0).
void to_reference_ids(TraceGraph& g, TraceLogs* logs, int off_t, int off_b, int off_c);

// Fills the caller's hesp_trace arrays; HESP_OK or HESP_E_LIMIT.
int finish_trace(const Problem& p, const TraceGraph& g, const TraceLogs& logs, hesp_trace* tr,
                 bool schedule_only = false);

// verify_schedule (sim.cpp:857-973) over a hesp_trace and the candidate graph,
// as data-parallel passes on the device (verify.cu); messages in `out`.
// HESP_OK, HESP_E_CUDA or HESP_E_LIMIT.
int verify_trace_device(const Problem& p, const TraceGraph& g, const hesp_trace& tr, cudaStream_t st,
                        std::vector<std::string>& out);

// Critical-path and work lower bounds of the traced graph (fastest type per task).
void trace_bounds(const Problem& p, const TraceGraph& g, double* cp, double* work);

}  // namespace hx

namespace hx {
// Schedule-only traces of B candidates in one launch (one warp each):
// per-candidate graph and (proc, start, end) by task id; outs[b].status != 0
// leaves graphs[b] / logs[b] empty.  HESP_OK or a negative HESP_E_* code.
int schedule_batch(hesp_engine* e, const hesp_cand_desc* descs, int B, std::vector<TraceGraph>& graphs,
                   std::vector<TraceLogs>& logs, std::vector<hesp_outcome>& outs);
}  // namespace hx

// engine internals the host-side solver reads (engine_kernels.cu)
const hx::Problem& hesp_engine_problem(const hesp_engine* e);
const hx::TraceGraph& hesp_engine_last_graph(const hesp_engine* e);

namespace hx {

}  // namespace hx
