// k_mode9.cu -- k_step / k_run of step mode 9 (bit 0 clamp, bit 1 Langevin noise, bit 3 edge weights).
#include "k_mode.cuh"

namespace qqa {
StepKernel step_kernel_m9(int lanes, int vpl, bool full) { return step_for<9>(lanes, vpl, full); }
RunKernel run_kernel_m9(int lanes, int vpl, int cta, bool full) { return run_kernel_for<9>(lanes, vpl, cta, full); }
XStepKernel xstep_kernel_m9(int lanes, int vpl, bool full) { return xstep_for<9>(lanes, vpl, full); }
XStepKernel xsstep_kernel_m9(int lanes, int vpl, bool full) { return xsstep_for<9>(lanes, vpl, full); }
}  // namespace qqa
