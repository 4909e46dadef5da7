// scmwu_inst_3.cu — explicit instantiations of the persistent kernel (part 3 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SVM, 2, 4, 2)
SCMWU_INST(SC_SVM, 4, 8, 4)
SCMWU_INST(SC_SVM, 8, 13, 4)
SCMWU_INST(SC_SVM, 32, 12, 2)

namespace scmwu {
KernelFn scmwu_lookup_3(int kind, int lpr, int cpl, int nb) {
    SCMWU_MATCH(SC_SVM, 2, 4, 2)
    SCMWU_MATCH(SC_SVM, 4, 8, 4)
    SCMWU_MATCH(SC_SVM, 8, 13, 4)
    SCMWU_MATCH(SC_SVM, 32, 12, 2)
    return nullptr;
}
}  // namespace scmwu
