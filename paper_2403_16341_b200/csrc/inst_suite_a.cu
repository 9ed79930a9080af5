// Registry instances: suite members 1-8 (problems.py:300-313), fp64.
#include "nlk_registry.cuh"
namespace nlk {
static const Entry kEntries[] = {
    NLK_ENTRY_F64("test23/rosenbrock", Rosenbrock),
    NLK_ENTRY_F64("test23/powell-singular", PowellSingular),
    NLK_ENTRY_F64("test23/powell-badly-scaled", PowellBadlyScaled),
    NLK_ENTRY_F64("test23/wood", Wood),
    NLK_ENTRY_F64("test23/helical-valley", HelicalValley),
    NLK_ENTRY_F64("test23/watson", Watson),
    NLK_ENTRY_F64("test23/chebyquad", Chebyquad),
    NLK_ENTRY_F64("test23/brown-almost-linear", BrownAlmostLinear),
};
EntryTable registry_suite_a() { return {kEntries, sizeof(kEntries) / sizeof(kEntries[0])}; }
}  // namespace nlk
