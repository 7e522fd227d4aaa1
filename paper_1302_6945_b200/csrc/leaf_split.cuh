// Split leaf sweep (pivot chain / basis replay / check), see leaf_split.cu.
#pragma once
#include "leaf.cuh"

enum { SPLIT_DONE = -1, SPLIT_EXACT = -2 };

struct SplitState {
  int* need;           // [sys] round the system is waiting for, DONE or EXACT
  int kcap;            // >= conditions per leaf
  cplx* mu;            // [sys][kcap][P] per-step multipliers
  int* jl;             // [sys][kcap] per-step pivot (-1 = deferred)
  int2* def_try;       // [sys][kcap]
  int2* def_best;      // [sys][kcap]
  int* ndef_try;
  int* ndef_best;
  int* len_try;
  int* len_best;
  int* cd_try;         // [sys][8]
  int* cd_best;        // [sys][8]
  double* factor_try;
  double* factor_best;
  double* res_best;
  int* viol;           // [sys] rescale speculation violated
  int* any_viol;       // [1] sticky: some leaf of some system was handed to the exact kernel
  double* colpart;     // [sys][8][8] per-row column max^2 (row-parallel build)
};

bool leaf_split_supported(const LeafArgs& a);
int leaf_split_launch(const LeafArgs& a, const SplitState& s, int nsys, cudaStream_t st);

// default path (leaf_fast.cu): chain kernel + fused basis / self-check kernel
bool leaf_fast_supported(const LeafArgs& a);
int leaf_fast_launch(const LeafArgs& a, const SplitState& s, int nsys, cudaStream_t st);
