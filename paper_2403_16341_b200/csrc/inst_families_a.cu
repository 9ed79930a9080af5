// Registry instances: quadratic (problems.py:376-387) at several n, fp64+fp32.
#include "nlk_registry.cuh"
namespace nlk {
static const Entry kEntries[] = {
    NLK_ENTRY_BOTH("quadratic", Quadratic<1>),
    NLK_ENTRY_BOTH("quadratic", Quadratic<2>),
    NLK_ENTRY_BOTH("quadratic", Quadratic<3>),
    NLK_ENTRY_BOTH("quadratic", Quadratic<4>),
    NLK_ENTRY_BOTH("quadratic", Quadratic<8>),
    NLK_ENTRY_BOTH("generalized_rosenbrock", GeneralizedRosenbrock<2>),
    NLK_ENTRY_BOTH("generalized_rosenbrock", GeneralizedRosenbrock<3>),
    NLK_ENTRY_BOTH("generalized_rosenbrock", GeneralizedRosenbrock<4>),
};
EntryTable registry_families_a() { return {kEntries, sizeof(kEntries) / sizeof(kEntries[0])}; }
}  // namespace nlk
