// Leaf serial sweep (ref: pkg/src/toepreg/tanint.py:395-434 _serial_leaf,
// :189-217 _serial_core, :137-186 _Workspace, :262-270 _self_residual,
// :220-259 absorption orders).
#pragma once
#include "common.cuh"

struct LeafArgs {
  // condition data
  const cplx* W;        // current weights [sys][N][rows][P]
  long long w_sys;      // system stride (complex elements)
  long long N;
  int rows, P;
  // leaf node set: offsets o[0..noff) + stride*t, t < M
  long long o0, o1;
  int noff;
  long long stride;
  int M;                // nodes per coset
  int count;            // leaf nodes = noff * M
  int K;                // conditions = rows * count
  int dbound = 0;       // planned structural degree of the leaf basis (0: unknown)
  // absorption orders
  int nattempts;
  int ord_stride[4];    // perm[i] = (i * s) % count   (ord_reverse: use reversed)
  int ord_reverse[4];
  const cplx* twN;      // exp(2 pi i k / N)
  double thr;           // pivot threshold
  double check_tol;     // leaf self-check tolerance (1e-11)
  // per-system state
  int* cd;              // [sys][8] column degrees (in/out)
  cplx* out;            // output cube [sys][P*P][cap]
  long long out_sys;
  int cap;
  cplx* scratch;        // same layout as out, for retry attempts
  int2* defer;          // [sys][dmax] (node, row)
  int* dcount;          // [sys]
  int dmax;
  double* max_scale;    // [sys]
  int* retried;         // [sys]
  int* status;          // [sys]
  double* res_out;      // [sys] best self residual (diagnostic), may be null
  int* len_out;         // [sys] basis length (diagnostic), may be null
  long long* dbg = nullptr;  // [sys][16] clock64 trace (diagnostic), may be null
  const int* only = nullptr; // when set: only systems with only[sys] == -2 run (exact fallback)
  int len_eff = 0;           // coefficients the parent's fused combine reads (0: all)
  int* trim_over = nullptr;  // [sys] the exact kernel counts a basis longer than len_eff here
  int force_viol = 0;        // test hook (TR_TEST_VIOL): system 0 reports a violated speculation here
  int dense = 0;             // fused leaf kernel: every warp has a role (set by launch_fused3)
};

struct SplitState;
// Launch the leaf sweep for every system of the batch (split kernels when a
// SplitState is given and the shape fits, else the exact coupled kernel).
// exact_pass = false: the exact fallback for leaves the split kernels hand over is not
// launched (they are flagged in split->any_viol; the caller re-runs with it).
int leaf_launch(const LeafArgs& a, int nsys, cudaStream_t st, const SplitState* split = nullptr,
                bool exact_pass = true);
// Whether a (P, K) leaf fits the register kernels.
bool leaf_supported(int P, int K);
