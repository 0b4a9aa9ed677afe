// wm_motif.cu — placeholder until the motif kernel lands.
#include "wm_common.cuh"
namespace wm {
int run_motif(Graph *g, const wm_app *app, const wm_cfg *cfg, wm_result *res, cudaStream_t s) {
  return fail(WM_EINVAL, "motif kernel not built yet");
}
}  // namespace wm
