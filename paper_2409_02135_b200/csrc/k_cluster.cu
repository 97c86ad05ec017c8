// k_cluster.cu -- instantiations of the one-cluster, shared-memory-resident anneal (k_run_cluster).
#define QQA_INST_ONLY
#include "qqa_dispatch.h"

namespace qqa {
RunKernel cluster_kernel(int mode) {
  switch (mode) {
    case 0: return k_run_cluster<0>;
    case 1: return k_run_cluster<1>;
    case 2: return k_run_cluster<2>;
    case 3: return k_run_cluster<3>;
    default: return nullptr;
  }
}
}  // namespace qqa
