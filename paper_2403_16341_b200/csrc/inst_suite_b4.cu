// Registry instances: suite members 15-16 (problems.py:315-330), fp64.
// (Suite members 9-16 are split over four translation units so the largest
// kernels compile in parallel.)
#include "nlk_registry.cuh"
namespace nlk {
static const Entry kEntries[] = {
    NLK_ENTRY_F64("test23/matrix-sqrt-2x2", MatrixSqrt2x2),
    NLK_ENTRY_F64("test23/matrix-sqrt-3x3", MatrixSqrt3x3),
};
EntryTable registry_suite_b4() { return {kEntries, sizeof(kEntries) / sizeof(kEntries[0])}; }
}  // namespace nlk
