// placeholder, replaced by the matrix-free SCM kernels
#include "wcb_internal.cuh"
namespace wcb {
Operator* make_scm_operator(Context*, const wcb_scm_desc*) {
    throw Error{WCB_E_UNSUPPORTED, "SCM operator not built yet"};
}
}
