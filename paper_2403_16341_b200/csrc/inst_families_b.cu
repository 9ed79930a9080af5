// Registry instances: generalized Rosenbrock (problems.py:358-373) N = 8, 10.
#include "nlk_registry.cuh"
namespace nlk {
static const Entry kEntries[] = {
    NLK_ENTRY_BOTH("generalized_rosenbrock", GeneralizedRosenbrock<8>),
    NLK_ENTRY_BOTH("generalized_rosenbrock", GeneralizedRosenbrock<10>),
};
EntryTable registry_families_b() { return {kEntries, sizeof(kEntries) / sizeof(kEntries[0])}; }
}  // namespace nlk
