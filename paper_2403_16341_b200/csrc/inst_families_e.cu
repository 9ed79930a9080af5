// Registry instances: quadratic (problems.py:376-387) at n = 16.
#include "nlk_registry.cuh"
namespace nlk {
static const Entry kEntries[] = {
    NLK_ENTRY_BOTH("quadratic", Quadratic<16>),
};
EntryTable registry_families_e() { return {kEntries, sizeof(kEntries) / sizeof(kEntries[0])}; }
}  // namespace nlk
