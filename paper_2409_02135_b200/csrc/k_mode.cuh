// k_mode.cuh -- body of k_mode<M>.cu: the k_step / k_run instantiations of one step mode.
#pragma once
#define QQA_INST_ONLY
#include "qqa_dispatch.h"

namespace qqa {
template <int M, int CT>
RunKernel run_for(int lanes, int vpl, bool full) {
#define QQA_RCASE(L, V) \
  if (lanes == L && vpl == V) \
    return full ? k_run<L, V, M, (V == 1 ? CT : 256), true> : k_run<L, V, M, (V == 1 ? CT : 256), false>;
  QQA_RCASE(1, 1) QQA_RCASE(2, 1) QQA_RCASE(4, 1) QQA_RCASE(8, 1) QQA_RCASE(16, 1)
  QQA_RCASE(32, 1) QQA_RCASE(32, 2) QQA_RCASE(32, 4)
#undef QQA_RCASE
  return nullptr;
}

template <int M>
StepKernel step_for(int lanes, int vpl, bool full) {
#define QQA_SCASE(L, V) \
  if (lanes == L && vpl == V) return full ? k_step<L, V, M, true> : k_step<L, V, M, false>;
  QQA_SCASE(1, 1) QQA_SCASE(2, 1) QQA_SCASE(4, 1) QQA_SCASE(8, 1) QQA_SCASE(16, 1)
  QQA_SCASE(32, 1) QQA_SCASE(32, 2) QQA_SCASE(32, 4)
#undef QQA_SCASE
  return nullptr;
}

template <int M>
XStepKernel xstep_for(int lanes, int vpl, bool full) {
  if (M & kModeSparseClique) return nullptr;   // fused exchange: modes 0-3 and the weighted 8-11
#define QQA_XCASE(L, V) \
  if (lanes == L && vpl == V) \
    return full ? k_step_x<L, V, (M & 11), true> : k_step_x<L, V, (M & 11), false>;
  QQA_XCASE(1, 1) QQA_XCASE(2, 1) QQA_XCASE(4, 1) QQA_XCASE(8, 1) QQA_XCASE(16, 1)
  QQA_XCASE(32, 1) QQA_XCASE(32, 2) QQA_XCASE(32, 4)
#undef QQA_XCASE
  return nullptr;
}

// k_step_st<lanes, M> (staged state; VPL = 1, FULL shapes, modes 0-3); nullptr otherwise.
template <int M>
StepKernel stage_for(int lanes) {
  if (M & (kModeSparseClique | kModeWeighted)) return nullptr;
#define QQA_TCASE(L) \
  if (lanes == L) return k_step_st<L, (M & 3)>;
  QQA_TCASE(1) QQA_TCASE(2) QQA_TCASE(4) QQA_TCASE(8) QQA_TCASE(16) QQA_TCASE(32)
#undef QQA_TCASE
  return nullptr;
}

// k_step_xs (owner-slotted exchange): the same shapes and modes as k_step_x.
template <int M>
XStepKernel xsstep_for(int lanes, int vpl, bool full) {
  if (M & kModeSparseClique) return nullptr;
#define QQA_XSCASE(L, V) \
  if (lanes == L && vpl == V) \
    return full ? k_step_xs<L, V, (M & 11), true> : k_step_xs<L, V, (M & 11), false>;
  QQA_XSCASE(1, 1) QQA_XSCASE(2, 1) QQA_XSCASE(4, 1) QQA_XSCASE(8, 1) QQA_XSCASE(16, 1)
  QQA_XSCASE(32, 1) QQA_XSCASE(32, 2) QQA_XSCASE(32, 4)
#undef QQA_XSCASE
  return nullptr;
}

template <int M>
RunKernel run_kernel_for(int lanes, int vpl, int cta, bool full) {
  if (M & kModeSparseClique) return nullptr;   // its column sums need a pass between steps: no k_run
  if (vpl == 1 && cta == 1024) return run_for<M, 1024>(lanes, vpl, full);
  if (vpl == 1 && cta == 768) return run_for<M, 768>(lanes, vpl, full);
  return run_for<M, 256>(lanes, vpl, full);
}
}  // namespace qqa
