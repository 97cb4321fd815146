/* hesp_workload.h — the synthetic candidate workload shared by every arm.
 *
 * A candidate is a sequence of partition (and optionally merge) operations
 * applied, after the base tiling, to a root tiled-Cholesky task:
 *
 *     g = TaskGraph::root_cholesky(n, elem)                  graph.cpp:397
 *     g.partition_task(0, 1.0 / s_base, min_block)           graph.cpp:456  (base tiling)
 *     for op in desc.ops: g.partition_task(op.task, 1.0 / op.s, min_block)
 *                         (or g.merge_cluster(op.task) when op.s == HESP_OP_MERGE)
 *
 * The reference has no candidate generator (its solver is declared only,
 * solver.hpp:57-86), so this header *defines* the workload of BASELINE.json's
 * configs: candidate i draws K ~ U[0, k_max] operations from a
 * splitmix64 stream seeded with (seed ^ i); each operation picks, uniformly by
 * task-id rank, a leaf with b/2 >= min_block and depth < max_depth, and a tile
 * count s from s_choices.  The generator tracks leaf ids, sides and depths
 * exactly as partition_task assigns them (sequential ids, graph.cpp:438; side
 * d/s, graph.cpp:504) so the emitted task ids are valid reference task ids.
 *
 * This is input generation, not the measured path: the oracle harness, the
 * CPU baseline and the GPU engine all consume the same descriptors.
 * Plain C99/C++ with HESP_HD so nvcc and gcc compile the identical code.
 */
#ifndef HESP_WORKLOAD_H
#define HESP_WORKLOAD_H

#include <stdint.h>

#if defined(__CUDACC__)
#define HESP_HD __host__ __device__ inline
#define HESP_NOUNROLL _Pragma("unroll 1")
#else
#define HESP_HD static inline
#define HESP_NOUNROLL
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* TaskKind ordinals, platform.hpp:15 */
enum { HESP_CHOL = 0, HESP_TRSM = 1, HESP_SYRK = 2, HESP_GEMM = 3 };

#define HESP_MAX_OPS 64     /* operations per candidate (solver chains append one per iteration) */
#define HESP_GEN_MAX_OPS 16 /* bound on the generator's k_max */
/* op.s value marking TaskGraph::merge_cluster(op.task) (graph.cpp:521-534);
 * repartition_cluster (graph.cpp:536-539) is a merge followed by a partition
 * of the restored parent. */
#define HESP_OP_MERGE ((int32_t)0x80000000)

typedef struct {
  int32_t task; /* reference task id (must be a leaf when applied); cluster id for a merge */
  int32_t s;    /* requested tile count, applied as p = 1.0 / s; HESP_OP_MERGE = merge */
} hesp_op;

typedef struct {
  int32_t n_ops;
  int32_t reserved;
  hesp_op ops[HESP_MAX_OPS];
} hesp_cand_desc; /* 520 bytes */

typedef struct {
  uint64_t seed;
  int32_t k_max;     /* K ~ U[0, k_max], k_max <= HESP_GEN_MAX_OPS   */
  int32_t max_depth; /* leaves with depth < max_depth are eligible    */
  int64_t min_block; /* grain; also partition_task's min_block       */
  int32_t n_s_choices;
  int32_t s_choices[4];
  int32_t merge_pct; /* per op: % chance of merging a random innermost
                        non-base cluster instead (0 = partitions only) */
} hesp_gen_config;

/* splitmix64, identical to hesp::Rng::next (sim.cpp:59-65). */
HESP_HD uint64_t hesp_splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* splitmix64 finaliser used by the order-independent result hashes. */
HESP_HD uint64_t hesp_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* Snap a requested tile count to a divisor of d with tiles >= min_block,
 * nearest first, coarser on ties: graph.cpp:464-481.  0 == IndivisibleGrain.
 * s0 is computed through p = 1.0/s exactly as the harness passes it. */
HESP_HD int64_t hesp_snap_tiles(int64_t d, int32_t s_req, int64_t min_block) {
  const double p = 1.0 / (double)s_req;
  const double inv = 1.0 / p;
  /* llround without libm: inv is positive and far from .5 ties */
  int64_t r = (int64_t)(inv + 0.5);
  const int64_t s0 = r > 2 ? r : 2;
  const int64_t mb = min_block > 1 ? min_block : 1;
  const int64_t s_hi = d / mb;
  HESP_NOUNROLL for (int64_t delta = 0; delta <= s0 + s_hi; ++delta) {
    int64_t c = s0 - delta;
    if (c >= 2 && c <= s_hi && d % c == 0) return c;
    c = s0 + delta;
    if (c >= 2 && c <= s_hi && d % c == 0) return c;
  }
  return 0;
}

/* Number of sub-tasks emitted by enumerate_partition (graph.cpp:301-392). */
HESP_HD int32_t hesp_member_count(int32_t kind, int32_t s) {
  switch (kind) {
    case HESP_CHOL: return s * (s + 1) * (s + 2) / 6;
    case HESP_TRSM: return s * (s * (s + 1) / 2);
    case HESP_SYRK: return s * (s * (s + 1) / 2);
    default: return s * s * s;
  }
}

/* Kind of the m-th sub-task of a kind/s partition, in the loop order of
 * graph.cpp:313-389 (CHOL k-loop; TRSM j,i,k; SYRK i,j<=i,k; GEMM i,j,k). */
HESP_HD int32_t hesp_member_kind(int32_t kind, int32_t s, int32_t m) {
  if (kind == HESP_CHOL) {
    HESP_NOUNROLL for (int32_t k = 0; k < s; ++k) {
      const int32_t t = s - k - 1; /* trailing tiles below the diagonal */
      if (m == 0) return HESP_CHOL;
      if (m <= t) return HESP_TRSM;
      m -= 1 + t;
      HESP_NOUNROLL for (int32_t i = k + 1; i < s; ++i) {
        const int32_t g = i - k - 1; /* GEMMs before this row's SYRK */
        if (m < g) return HESP_GEMM;
        if (m == g) return HESP_SYRK;
        m -= g + 1;
      }
    }
    return -1;
  }
  if (kind == HESP_TRSM) {
    HESP_NOUNROLL for (int32_t j = 0; j < s; ++j) {
      const int32_t blk = s * (j + 1);
      if (m < blk) return (m % (j + 1)) < j ? HESP_GEMM : HESP_TRSM;
      m -= blk;
    }
    return -1;
  }
  if (kind == HESP_SYRK) {
    HESP_NOUNROLL for (int32_t i = 0; i < s; ++i)
      HESP_NOUNROLL for (int32_t j = 0; j <= i; ++j) {
        if (m < s) return i == j ? HESP_SYRK : HESP_GEMM;
        m -= s;
      }
    return -1;
  }
  return HESP_GEMM;
}

/* Generate candidate `index`.  n_base = leaves of the base tiling (ids
 * 1..n_base, all of side base_b, depth 1, kinds of a CHOL/s_base partition). */
HESP_HD void hesp_generate(const hesp_gen_config* cfg, int32_t s_base, int32_t n_base,
                           int64_t base_b, uint64_t index, hesp_cand_desc* out) {
  struct Range {
    int32_t first, count;
    int64_t b;
    int32_t depth, pkind, s;
    int32_t parent, dead; /* partitioned task; merged away */
  } rg[HESP_GEN_MAX_OPS + 1];
  int32_t removed[HESP_GEN_MAX_OPS];
  int32_t nr = 1, nrem = 0, nops = 0;
  uint64_t st = cfg->seed ^ index;
  const int32_t kmax = cfg->k_max < HESP_GEN_MAX_OPS ? cfg->k_max : HESP_GEN_MAX_OPS;
  const int32_t K = (int32_t)(hesp_splitmix_next(&st) % (uint64_t)(kmax + 1));
  rg[0].first = 1;
  rg[0].count = n_base;
  rg[0].b = base_b;
  rg[0].depth = 1;
  rg[0].pkind = HESP_CHOL;
  rg[0].s = s_base;
  rg[0].parent = 0;
  rg[0].dead = 0;
  int32_t next_id = 1 + n_base;
  HESP_NOUNROLL for (int32_t op = 0; op < K; ++op) {
    if (cfg->merge_pct > 0) {
      /* innermost live clusters created by earlier ops (never the base one) */
      int32_t ninner = 0;
      HESP_NOUNROLL for (int32_t r = 1; r < nr; ++r) {
        int32_t inner = !rg[r].dead;
        HESP_NOUNROLL for (int32_t q = 0; q < nrem && inner; ++q)
          if (removed[q] >= rg[r].first && removed[q] < rg[r].first + rg[r].count) inner = 0;
        ninner += inner;
      }
      if (ninner > 0 && (int32_t)(hesp_splitmix_next(&st) % 100u) < cfg->merge_pct) {
        int32_t k = (int32_t)(hesp_splitmix_next(&st) % (uint64_t)ninner), c = -1;
        HESP_NOUNROLL for (int32_t r = 1; r < nr && c < 0; ++r) {
          int32_t inner = !rg[r].dead;
          HESP_NOUNROLL for (int32_t q = 0; q < nrem && inner; ++q)
            if (removed[q] >= rg[r].first && removed[q] < rg[r].first + rg[r].count) inner = 0;
          if (inner && k-- == 0) c = r;
        }
        out->ops[nops].task = c; /* cluster ids follow partition order: base = 0 */
        out->ops[nops].s = HESP_OP_MERGE;
        ++nops;
        rg[c].dead = 1;
        /* the restored parent is a leaf again */
        int32_t w = 0;
        HESP_NOUNROLL for (int32_t q = 0; q < nrem; ++q)
          if (removed[q] != rg[c].parent) removed[w++] = removed[q];
        nrem = w;
        continue;
      }
    }
    uint64_t total = 0;
    HESP_NOUNROLL for (int32_t r = 0; r < nr; ++r) {
      if (rg[r].dead) continue;
      if (!(rg[r].b / 2 >= cfg->min_block && rg[r].depth < cfg->max_depth)) continue;
      int32_t live = rg[r].count;
      HESP_NOUNROLL for (int32_t q = 0; q < nrem; ++q)
        if (removed[q] >= rg[r].first && removed[q] < rg[r].first + rg[r].count) --live;
      total += (uint64_t)live;
    }
    if (total == 0) break;
    uint64_t pick = hesp_splitmix_next(&st) % total;
    int32_t id = -1, rsel = -1;
    HESP_NOUNROLL for (int32_t r = 0; r < nr && id < 0; ++r) {
      if (rg[r].dead) continue;
      if (!(rg[r].b / 2 >= cfg->min_block && rg[r].depth < cfg->max_depth)) continue;
      int32_t live = rg[r].count;
      HESP_NOUNROLL for (int32_t q = 0; q < nrem; ++q)
        if (removed[q] >= rg[r].first && removed[q] < rg[r].first + rg[r].count) --live;
      if (pick < (uint64_t)live) {
        id = rg[r].first + (int32_t)pick;
        /* removed[] is sorted ascending: skip removed ids at or below id */
        HESP_NOUNROLL for (int32_t q = 0; q < nrem; ++q)
          if (removed[q] >= rg[r].first && removed[q] <= id) ++id;
        rsel = r;
      } else {
        pick -= (uint64_t)live;
      }
    }
    const int32_t s_req =
        cfg->s_choices[hesp_splitmix_next(&st) % (uint64_t)(cfg->n_s_choices > 0 ? cfg->n_s_choices : 1)];
    out->ops[nops].task = id;
    out->ops[nops].s = s_req;
    ++nops;
    const int64_t s = hesp_snap_tiles(rg[rsel].b, s_req, cfg->min_block);
    if (s == 0) break; /* the build reports IndivisibleGrain */
    const int32_t kind = hesp_member_kind(rg[rsel].pkind, rg[rsel].s, id - rg[rsel].first);
    int32_t q = nrem++;
    while (q > 0 && removed[q - 1] > id) {
      removed[q] = removed[q - 1];
      --q;
    }
    removed[q] = id;
    const int32_t cnt = hesp_member_count(kind, (int32_t)s);
    rg[nr].first = next_id;
    rg[nr].count = cnt;
    rg[nr].b = rg[rsel].b / s;
    rg[nr].depth = rg[rsel].depth + 1;
    rg[nr].pkind = kind;
    rg[nr].s = (int32_t)s;
    rg[nr].parent = id;
    rg[nr].dead = 0;
    ++nr;
    next_id += cnt;
  }
  out->n_ops = nops;
  out->reserved = 0;
  HESP_NOUNROLL for (int32_t r = nops; r < HESP_MAX_OPS; ++r) {
    out->ops[r].task = -1;
    out->ops[r].s = 0;
  }
}

/* Order-independent result hashes (sum of mixed terms, wrapping).  Both the
 * oracle harness and the engine fold every assignment / transfer record of a
 * schedule into these, so equality means bit-identical records.  One
 * splitmix finaliser round per record over a rotation/xor combination of
 * every field keeps them cheap on the device. */
HESP_HD uint64_t hesp_rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

HESP_HD uint64_t hesp_assign_term(int32_t task, int32_t proc, uint64_t start_bits,
                                  uint64_t end_bits) {
  return hesp_mix64((start_bits + hesp_rotl64(end_bits, 21)) ^
                    (((uint64_t)(uint32_t)task << 32) | (uint64_t)(uint32_t)proc));
}

HESP_HD uint64_t hesp_xfer_term(int32_t block, int32_t src_space, int32_t dst_space, int64_t bytes,
                                uint64_t start_bits, uint64_t end_bits, int64_t frow, int64_t fcol,
                                int64_t frows, int64_t fcols) {
  const uint64_t id = ((uint64_t)(uint32_t)block << 24) ^ ((uint64_t)(uint32_t)src_space << 16) ^
                      ((uint64_t)(uint32_t)dst_space << 8);
  const uint64_t f = hesp_rotl64(((uint64_t)frow << 32) ^ (uint64_t)(uint32_t)fcol, 7) ^
                     hesp_rotl64(((uint64_t)frows << 32) ^ (uint64_t)(uint32_t)fcols, 29);
  return hesp_mix64((start_bits + hesp_rotl64(end_bits, 21)) ^ hesp_rotl64((uint64_t)bytes, 40) ^ id ^ f);
}

#ifdef __cplusplus
}
#endif

#endif /* HESP_WORKLOAD_H */
