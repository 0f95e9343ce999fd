// Temporary: entry points not implemented yet.
#include "common.cuh"
using namespace ifgfb;
extern "C" {
int ifgfb_plan_set_surface(ifgfb_plan*, const ifgfb_surface_desc*) { set_error("not implemented"); return IFGFB_ERR_UNSUPPORTED; }
int ifgfb_plan_set_near(ifgfb_plan*, const ifgfb_near_desc*) { set_error("not implemented"); return IFGFB_ERR_UNSUPPORTED; }
int ifgfb_potentials(ifgfb_plan*, const double*, double*, double*, void*) { set_error("not implemented"); return IFGFB_ERR_UNSUPPORTED; }
int ifgfb_muller_apply(ifgfb_plan*, const double*, double*, void*) { set_error("not implemented"); return IFGFB_ERR_UNSUPPORTED; }
int ifgfb_muller_apply_host(ifgfb_plan*, const double*, double*, void*) { set_error("not implemented"); return IFGFB_ERR_UNSUPPORTED; }
int ifgfb_zdotc(const double*, const double*, int64_t, double*, void*) { return IFGFB_ERR_UNSUPPORTED; }
int ifgfb_dznrm2(const double*, int64_t, double*, void*) { return IFGFB_ERR_UNSUPPORTED; }
int ifgfb_zaxpy(const double*, const double*, double*, int64_t, void*) { return IFGFB_ERR_UNSUPPORTED; }
int ifgfb_zscal_div(double*, const double*, double, int64_t, void*) { return IFGFB_ERR_UNSUPPORTED; }
}
