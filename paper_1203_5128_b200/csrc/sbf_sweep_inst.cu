// One K3 sweep instantiation per object (built with -DSBF_R=<r> -DSBF_P=<passes>).
#include "sbf_sweepw.cuh"

namespace sbf {
#define SBF_SCAT2(a, b, c) a##b##_##c
#define SBF_SCAT(a, b, c) SBF_SCAT2(a, b, c)
SweepEntry SBF_SCAT(sweep_entry_, SBF_R, SBF_P)() { return SBF_SWEEP_ENTRY(SBF_R, SBF_P); }
}  // namespace sbf
