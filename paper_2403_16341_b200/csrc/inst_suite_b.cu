// Registry instances: suite members 9-10 (problems.py:315-330), fp64.
// (Suite members 9-16 are split over four translation units so the largest
// kernels compile in parallel.)
#include "nlk_registry.cuh"
namespace nlk {
static const Entry kEntries[] = {
    NLK_ENTRY_F64("test23/discrete-boundary-value", DiscreteBoundaryValue),
    NLK_ENTRY_F64("test23/discrete-integral", DiscreteIntegral),
};
EntryTable registry_suite_b() { return {kEntries, sizeof(kEntries) / sizeof(kEntries[0])}; }
}  // namespace nlk
