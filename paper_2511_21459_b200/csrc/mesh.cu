// mixed-resolution Marching Cubes (placeholder until the GPU extractor lands)
#include <cstdlib>
#include "fusion.h"
namespace tsdf {
int extract_mesh(Table* T, double iso, double eps, MeshOut* out) {
  (void)T; (void)iso; (void)eps; (void)out;
  set_error("extract_mesh: not built yet");
  return kValueError;
}
void mesh_free(MeshOut* m) {
  free(m->v); free(m->n); free(m->c); free(m->tri);
}
}  // namespace tsdf
namespace tsdf {
int collapse_vertices(const double*, const double*, const double*, int64_t, const int64_t*,
                      int64_t, double, MeshOut*) {
  set_error("collapse_vertices: not built yet");
  return kValueError;
}
}  // namespace tsdf
