/* nccl_shim.c — TEST INFRASTRUCTURE: a two-process stand-in for
 * ncclAllReduce, so hesp_min_reduce's exchange (the C-ABI cross-GPU winner,
 * engine_kernels.cu) runs with world size 2 on a one-GPU lease.  NCCL itself
 * rejects two ranks on one device; this shim keeps NCCL's calling convention
 * (ncclAllReduce(send, recv, count, ncclInt64, ncclMin|ncclSum, comm, stream))
 * and does the reduction through files in a shared directory.
 *
 * The engine loads it through HESP_NCCL_LIB.  `comm` is a shim_comm made by
 * shim_comm_init(rank, world, dir).  Only int64 MIN / SUM are supported (the
 * only reductions hesp_min_reduce issues). */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

typedef struct {
  int rank, world;
  long seq;
  char dir[512];
} shim_comm;

void* shim_comm_init(int rank, int world, const char* dir) {
  shim_comm* c = (shim_comm*)calloc(1, sizeof(shim_comm));
  c->rank = rank;
  c->world = world;
  snprintf(c->dir, sizeof c->dir, "%s", dir);
  return c;
}

long shim_calls(void* comm) { return ((shim_comm*)comm)->seq; }

const char* ncclGetErrorString(int r) { return r ? "shim error" : "ok"; }

static int write_part(const shim_comm* c, long seq, const int64_t* v, size_t n) {
  char tmp[600], fin[600];
  snprintf(tmp, sizeof tmp, "%s/r%d_s%ld.tmp", c->dir, c->rank, seq);
  snprintf(fin, sizeof fin, "%s/r%d_s%ld.bin", c->dir, c->rank, seq);
  FILE* f = fopen(tmp, "wb");
  if (!f) return 1;
  if (fwrite(v, 8, n, f) != n) return 1;
  fclose(f);
  return rename(tmp, fin) != 0;  /* atomic publish */
}

static int read_part(const shim_comm* c, int rank, long seq, int64_t* v, size_t n) {
  char fin[600];
  snprintf(fin, sizeof fin, "%s/r%d_s%ld.bin", c->dir, rank, seq);
  for (int tries = 0; tries < 600000; ++tries) { /* <= 60 s */
    FILE* f = fopen(fin, "rb");
    if (f) {
      const size_t got = fread(v, 8, n, f);
      fclose(f);
      if (got == n) return 0;
    }
    usleep(100);
  }
  return 1;
}

int ncclAllReduce(const void* send, void* recv, size_t count, int dtype, int op, void* comm,
                  cudaStream_t stream) {
  shim_comm* c = (shim_comm*)comm;
  if (dtype != 4 || (op != 0 && op != 3) || count > 64) return 1; /* ncclInt64; ncclSum / ncclMin */
  int64_t mine[64], other[64], acc[64];
  if (cudaStreamSynchronize(stream) != cudaSuccess) return 1;
  if (cudaMemcpy(mine, send, count * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  const long seq = c->seq++;
  if (write_part(c, seq, mine, count)) return 1;
  memcpy(acc, mine, count * 8);
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    if (read_part(c, r, seq, other, count)) return 1;
    for (size_t i = 0; i < count; ++i) acc[i] = op == 3 ? (other[i] < acc[i] ? other[i] : acc[i]) : acc[i] + other[i];
  }
  /* rank order of the fold is irrelevant: MIN and wrapping SUM commute */
  if (cudaMemcpyAsync(recv, acc, count * 8, cudaMemcpyHostToDevice, stream) != cudaSuccess) return 1;
  return cudaStreamSynchronize(stream) != cudaSuccess;
}
