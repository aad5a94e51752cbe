// One split-sweep instantiation per object (built with -DSBF_R=<r> -DSBF_P=<passes>).
#include "sbf_split.cuh"

namespace sbf {
#define SBF_CAT2(a, b, c) a##b##_##c
#define SBF_CAT(a, b, c) SBF_CAT2(a, b, c)
SplitEntry SBF_CAT(split_entry_, SBF_R, SBF_P)() { return SBF_SPLIT_ENTRY(SBF_R, SBF_P); }
}  // namespace sbf
