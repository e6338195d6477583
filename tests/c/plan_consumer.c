/* plan_consumer.c — a plain C99 consumer of include/mpb200.h (no C++, no
 * CUDA headers): loads a .topo, plans GPU0 -> GPU1 and prints the chunk plan
 * as "path offset length seq" lines, the format tests/test_c_consumer.py
 * compares with the oracle.  Runs without a GPU (the planner is host code).
 *
 *   usage: plan_consumer <topo file> <gpu_paths> <host 0|1> <max_chunks> <size>
 */
#include <stdio.h>
#include <stdlib.h>

#include "mpb200.h"

static char* slurp(const char* path) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  fseek(f, 0, SEEK_END);
  long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  char* buf = (char*)malloc((size_t)n + 1);
  if (fread(buf, 1, (size_t)n, f) != (size_t)n) n = 0;
  buf[n] = 0;
  fclose(f);
  return buf;
}

int main(int argc, char** argv) {
  if (argc != 6) {
    fprintf(stderr, "usage: %s topo gpu_paths host max_chunks size\n", argv[0]);
    return 2;
  }
  if (mp_abi_version() != MP_ABI_VERSION) return 3;
  char* text = slurp(argv[1]);
  mp_topology* topo = NULL;
  if (!text || mp_topology_load(text, "c_consumer", &topo) != MP_OK) {
    fprintf(stderr, "topology: %s\n", mp_last_error());
    return 1;
  }
  mp_config cfg = {atoi(argv[2]), atoi(argv[3]), atoi(argv[4]), 1, 16, MP_SHARE_BANDWIDTH};
  mp_path paths[16];
  int32_t np = 0;
  if (mp_plan_paths(topo, 0, 1, &cfg, paths, 16, &np) != MP_OK) {
    fprintf(stderr, "plan: %s\n", mp_last_error());
    return 1;
  }
  uint64_t size = strtoull(argv[5], NULL, 10);
  int32_t nc = 0;
  /* capacity probe: cap 0 reports the needed count (MP_ERR_CAPACITY) */
  int rc = mp_make_chunk_plan(paths, np, size, cfg.max_chunks, NULL, 0, &nc);
  if (rc != MP_OK && rc != MP_ERR_CAPACITY) {
    fprintf(stderr, "chunks: %s\n", mp_last_error());
    return 1;
  }
  mp_chunk* chunks = (mp_chunk*)malloc(sizeof(mp_chunk) * (size_t)(nc > 0 ? nc : 1));
  if (mp_make_chunk_plan(paths, np, size, cfg.max_chunks, chunks, nc, &nc) != MP_OK) {
    fprintf(stderr, "chunks: %s\n", mp_last_error());
    return 1;
  }
  for (int32_t i = 0; i < np; ++i) printf("share %d %.17g\n", paths[i].kind, paths[i].share);
  for (int32_t i = 0; i < nc; ++i)
    printf("%d %llu %llu %d\n", chunks[i].path_index, (unsigned long long)chunks[i].offset,
           (unsigned long long)chunks[i].length, chunks[i].seq);
  free(chunks);
  mp_topology_destroy(topo);
  free(text);
  return 0;
}
