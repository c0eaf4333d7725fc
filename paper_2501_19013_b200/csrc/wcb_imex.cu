// placeholder for the IMEX plan
#include "wcb_internal.cuh"
extern "C" {
int wcb_imex_plan_create(wcb_operator*, int64_t, const int64_t*, int64_t, const int64_t*,
                         const double*, const wcb_lu*, const wcb_lu*, const double*,
                         const wcb_observer*, wcb_imex_plan**) {
    wcb::set_error("imex not built yet");
    return WCB_E_UNSUPPORTED;
}
int wcb_imex_plan_destroy(wcb_imex_plan*) { return WCB_OK; }
int wcb_imex_plan_run(wcb_imex_plan*, double, const double*, const double*, double, int64_t,
                      double, double, const double*, const double*, double*, double*, double*,
                      wcb_divergence*, wcb_timings*) {
    wcb::set_error("imex not built yet");
    return WCB_E_UNSUPPORTED;
}
}
