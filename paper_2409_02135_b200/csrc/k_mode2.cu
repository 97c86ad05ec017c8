// k_mode2.cu -- k_step / k_run of step mode 2 (bit 0 clamp, bit 1 Langevin noise).
#include "k_mode.cuh"

namespace qqa {
StepKernel step_kernel_m2(int lanes, int vpl, bool full) { return step_for<2>(lanes, vpl, full); }
RunKernel run_kernel_m2(int lanes, int vpl, int cta, bool full) { return run_kernel_for<2>(lanes, vpl, cta, full); }
XStepKernel xstep_kernel_m2(int lanes, int vpl, bool full) { return xstep_for<2>(lanes, vpl, full); }
XStepKernel xsstep_kernel_m2(int lanes, int vpl, bool full) { return xsstep_for<2>(lanes, vpl, full); }
StepKernel stage_kernel_m2(int lanes) { return stage_for<2>(lanes); }
}  // namespace qqa
