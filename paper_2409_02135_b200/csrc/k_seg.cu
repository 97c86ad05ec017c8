// k_seg.cu -- the segmented-gather step kernels (k_seg_gather, k_step_seg): VPL = 1, FULL
// shapes, unweighted step modes 0-3.
#define QQA_INST_ONLY
#include "qqa_dispatch.h"

namespace qqa {
namespace {
template <int M>
bool seg_for(int lanes, StepKernel& first, StepKernel& mid, StepKernel& last) {
#define QQA_GCASE(L) \
  if (lanes == L) { first = k_seg_gather<L, true>; mid = k_seg_gather<L, false>; last = k_step_seg<L, M>; return true; }
  QQA_GCASE(1) QQA_GCASE(2) QQA_GCASE(4) QQA_GCASE(8) QQA_GCASE(16) QQA_GCASE(32)
#undef QQA_GCASE
  return false;
}
}  // namespace

bool seg_kernels(int lanes, int mode, StepKernel& first, StepKernel& mid, StepKernel& last) {
  first = mid = last = nullptr;
  switch (mode) {
    case 0: return seg_for<0>(lanes, first, mid, last);
    case 1: return seg_for<1>(lanes, first, mid, last);
    case 2: return seg_for<2>(lanes, first, mid, last);
    case 3: return seg_for<3>(lanes, first, mid, last);
    default: return false;
  }
}
}  // namespace qqa
