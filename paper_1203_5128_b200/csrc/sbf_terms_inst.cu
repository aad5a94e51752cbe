// One explicit K3 instantiation per object file (parallel build); the
// (R, PASSES, MODE) triple comes from -DSBF_R/-DSBF_P/-DSBF_M.
#include "sbf_terms.cuh"

#define SBF_NAME3(a, b, c) terms_entry_##a##_##b##_##c
#define SBF_NAME(a, b, c) SBF_NAME3(a, b, c)

namespace sbf {
TermsEntry SBF_NAME(SBF_R, SBF_P, SBF_M)() { return SBF_TERMS_ENTRY(SBF_R, SBF_P, SBF_M); }
}  // namespace sbf
