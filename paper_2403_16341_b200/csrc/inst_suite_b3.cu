// Registry instances: suite members 12-14 (problems.py:315-330), fp64.
// (Suite members 9-16 are split over four translation units so the largest
// kernels compile in parallel.)
#include "nlk_registry.cuh"
namespace nlk {
static const Entry kEntries[] = {
    NLK_ENTRY_F64("test23/variably-dimensioned", VariablyDimensioned),
    NLK_ENTRY_F64("test23/broyden-tridiagonal", BroydenTridiagonal<10>),
    NLK_ENTRY_F64("test23/broyden-banded", BroydenBanded),
};
EntryTable registry_suite_b3() { return {kEntries, sizeof(kEntries) / sizeof(kEntries[0])}; }
}  // namespace nlk
