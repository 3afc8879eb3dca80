/* examples/c_trace_host.c — tracing from plain C on the GPU (device 0) with host buffers:
 * two stacked unit quads with an alpha texture whose left half is transparent; rays down the
 * z axis through both halves.  vsr_trace_host copies rays in, traces, copies hits out.
 *
 *   gcc -std=c11 -I include examples/c_trace_host.c -L paper_1912_12786_b200 -lvsr \
 *       -Wl,-rpath,paper_1912_12786_b200 -o /tmp/vsr_ct && /tmp/vsr_ct
 */
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "vsr.h"

int main(void) {
  float v[4 * 9];
  float tc[4 * 6];
  for (int q = 0; q < 2; ++q) {
    float z = 1.0f + (float)q;
    float a[9] = {0, 0, z, 1, 0, z, 1, 1, z}, b[9] = {0, 0, z, 1, 1, z, 0, 1, z};
    float ta[6] = {0, 0, 1, 0, 1, 1}, tb[6] = {0, 0, 1, 1, 0, 1};
    memcpy(v + (2 * q) * 9, a, sizeof a);
    memcpy(v + (2 * q + 1) * 9, b, sizeof b);
    memcpy(tc + (2 * q) * 6, ta, sizeof ta);
    memcpy(tc + (2 * q + 1) * 6, tb, sizeof tb);
  }
  /* geometry 0 (near quad): 2x1 texture, alpha 0 on the left texel, 255 on the right;
     geometry 1 (far quad): the implicit opaque texture index 1 */
  uint8_t t0[2 * 4] = {255, 255, 255, 0, 255, 255, 255, 255};
  uint8_t t1[4] = {255, 255, 255, 255};
  vsr_texture_desc tex[2] = {{2, 1, t0}, {1, 1, t1}};
  uint32_t gids[4] = {0, 0, 1, 1};
  vsr_scene_desc d;
  memset(&d, 0, sizeof d);
  d.num_tris = 4;
  d.vertices = v;
  d.geom_ids = gids;
  d.texcoords = tc;
  d.num_textures = 2;
  d.textures = tex;
  d.device = 0;
  vsr_scene* s = NULL;
  if (vsr_scene_create(&d, &s) != VSR_OK || vsr_bvh_build(s, NULL) != VSR_OK) {
    fprintf(stderr, "setup: %s\n", vsr_last_error());
    return 1;
  }
  vsr_ray rays[2] = {{0.25f, 0.5f, 0.0f, 1e-4f, 0, 0, 1, INFINITY},    /* left: transparent */
                     {0.75f, 0.5f, 0.0f, 1e-4f, 0, 0, 1, INFINITY}};   /* right: opaque */
  vsr_hit hits[2];
  if (vsr_trace_host(s, rays, 2, VSR_QUERY_CLOSEST, VSR_ISECT_ALPHA_TEXTURE, NULL, hits, NULL,
                     NULL) != VSR_OK) {
    fprintf(stderr, "trace: %s\n", vsr_last_error());
    return 1;
  }
  printf("left: t=%g prim=%u   right: t=%g prim=%u\n", hits[0].t, hits[0].prim_id, hits[1].t,
         hits[1].prim_id);
  vsr_destroy(s);
  /* the left ray passes the transparent half and stops on the far quad (z = 2) */
  return (hits[0].t == 2.0f && hits[0].prim_id >= 2 && hits[1].t == 1.0f && hits[1].prim_id < 2)
             ? 0 : 2;
}
