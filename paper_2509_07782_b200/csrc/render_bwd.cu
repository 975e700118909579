// render_bwd.cu -- K7 backward (replay of the forward march; see render.cu).
#include "gsx_common.cuh"

extern "C" int gsx_render_backward(const void*, const void*, const float*, int64_t,
                                   const gsx_camera*, const gsx_render_cfg*, int64_t, int64_t,
                                   const float*, const float*, const float*, const float*,
                                   const float*, const float*, float*, gsx_dev_status*, void*) {
  return GSX_ERR_ARG;  // not yet implemented
}
