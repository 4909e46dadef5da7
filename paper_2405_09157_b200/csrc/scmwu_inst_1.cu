// scmwu_inst_1.cu — explicit instantiations of the persistent kernel (part 1 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SVM, 2, 2, 2)
SCMWU_INST(SC_SVM, 4, 6, 4)
SCMWU_INST(SC_SVM, 8, 10, 4)
SCMWU_INST(SC_SVM, 16, 16, 2)

namespace scmwu {
KernelFn scmwu_lookup_1(int kind, int lpr, int cpl, int nb) {
    SCMWU_MATCH(SC_SVM, 2, 2, 2)
    SCMWU_MATCH(SC_SVM, 4, 6, 4)
    SCMWU_MATCH(SC_SVM, 8, 10, 4)
    SCMWU_MATCH(SC_SVM, 16, 16, 2)
    return nullptr;
}
}  // namespace scmwu
