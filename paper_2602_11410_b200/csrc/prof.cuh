// Launch counting and optional CUDA-event bracketing of kernel launches (cadet_prof_* in cadet.h).
#pragma once
#include <cuda_runtime.h>

namespace cadet {
enum ProfClass { PROF_GEMM = 0, PROF_ATTN_FWD = 1, PROF_ATTN_BWD = 2, PROF_OTHER = 3 };
void note_launches(int n);
int prof_begin(int cls, cudaStream_t st);   // returns a slot (or -1 when not profiling this class)
void prof_end(int slot, cudaStream_t st);

struct ProfScope {  // RAII bracket around the launches of one launcher call
  int slot;
  cudaStream_t st;
  ProfScope(int cls, cudaStream_t s, int nlaunch) : slot(prof_begin(cls, s)), st(s) { note_launches(nlaunch); }
  ~ProfScope() { prof_end(slot, st); }
};
}  // namespace cadet
