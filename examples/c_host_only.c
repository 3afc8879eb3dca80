/* examples/c_host_only.c — using libvsr from plain C (no Python, no GPU needed):
 * create a scene from a host description, build its BVH on the host (device -1),
 * read the statistics and the exported structure, exercise an error path.
 *
 *   gcc -std=c11 -I include examples/c_host_only.c -L paper_1912_12786_b200 -lvsr \
 *       -Wl,-rpath,paper_1912_12786_b200 -o /tmp/vsr_c && /tmp/vsr_c
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "vsr.h"

#define CHECK(call)                                                            \
  do {                                                                         \
    vsr_status st_ = (call);                                                   \
    if (st_ != VSR_OK) {                                                       \
      fprintf(stderr, "%s failed (%d): %s\n", #call, (int)st_, vsr_last_error()); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

int main(void) {
  /* two unit quads (4 triangles) at z = 1 and z = 2 */
  float v[4 * 9];
  for (int q = 0; q < 2; ++q) {
    float z = 1.0f + (float)q;
    float a[9] = {0, 0, z, 1, 0, z, 1, 1, z};
    float b[9] = {0, 0, z, 1, 1, z, 0, 1, z};
    memcpy(v + (2 * q) * 9, a, sizeof a);
    memcpy(v + (2 * q + 1) * 9, b, sizeof b);
  }
  vsr_scene_desc d;
  memset(&d, 0, sizeof d);
  d.num_tris = 4;
  d.vertices = v;
  d.device = -1; /* host-only: build and export, no GPU */
  vsr_scene* s = NULL;
  CHECK(vsr_scene_create(&d, &s));
  vsr_build_params bp = {1, 16, 1.0f, 1.0f};
  CHECK(vsr_bvh_build(s, &bp));
  vsr_stats st;
  CHECK(vsr_scene_stats(s, &st));
  vsr_bvh_view view;
  memset(&view, 0, sizeof view);
  CHECK(vsr_bvh_export(s, &view)); /* sizes only */
  void* nodes = malloc((size_t)view.num_nodes * 64 + 64);
  view.nodes = nodes;
  view.tris = malloc((size_t)view.num_tris * 48);
  view.sides = malloc((size_t)view.num_tris * 32);
  view.texdescs = malloc((size_t)view.num_textures * 16 + 16);
  view.texels = malloc((size_t)view.num_texels + 1);
  CHECK(vsr_bvh_export(s, &view)); /* copies */
  printf("abi %u tris %u nodes %u leaves %u depth %u root_ref %08x\n", vsr_abi_version(),
         st.num_tris, st.num_nodes, st.num_leaves, st.max_depth, view.root_ref);
  /* a host-only scene cannot be traced: UNSUPPORTED, with a message */
  vsr_status e = vsr_trace(s, NULL, 0, VSR_QUERY_CLOSEST, VSR_ISECT_DEFAULT, NULL, NULL, NULL, NULL);
  vsr_ray r;
  vsr_hit h;
  e = vsr_trace(s, &r, 1, VSR_QUERY_CLOSEST, VSR_ISECT_DEFAULT, NULL, &h, NULL, NULL);
  printf("trace on host-only scene: %d (%s)\n", (int)e, vsr_last_error());
  free(nodes);
  free(view.tris);
  free(view.sides);
  free(view.texdescs);
  free(view.texels);
  CHECK(vsr_destroy(s));
  return (st.num_tris == 4 && st.num_nodes == 3 && e == VSR_ERR_UNSUPPORTED) ? 0 : 2;
}
