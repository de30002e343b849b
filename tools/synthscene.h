/* Synthetic RGB-D input generator for the bench and the tests (NOT part of
 * the product, NOT the oracle): a C restatement of the reference's
 * SyntheticScene::render_frame (proj/src/synthcam.cpp:13-316) — analytic SDF
 * shapes (sphere, box, plane, cylinder), procedural textures (checker, value
 * noise, dots), scene warps (rigid, bend, twist), rigid camera motion,
 * sphere-traced depth + color, optional depth noise.  Checked bit for bit
 * against the reference's own renderer (oracle/_ref) by
 * tests/test_synthscene.py, so the B200 arm and the reference arm of bench.py
 * consume identical frames. */
#pragma once

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SS_SPHERE = 0, SS_BOX = 1, SS_PLANE = 2, SS_CYLINDER = 3 };          /* ShapeType */
enum { SS_CHECKER = 0, SS_NOISE = 1, SS_DOTS = 2 };                          /* TextureType */
enum { SS_WARP_NONE = 0, SS_WARP_RIGID = 1, SS_WARP_BEND = 2, SS_WARP_TWIST = 3 }; /* WarpType */
enum { SS_MAX_SHAPES = 8 };

typedef struct ss_shape { /* ShapeSpec (synthcam.hpp:15-24) */
  int32_t type;
  int32_t reserved_;
  double center[3];
  double radius;
  double half_extents[3];
  double normal[3];
  double offset;
  double axis[3];
  double half_height;
} ss_shape;

typedef struct ss_scene { /* SceneSpec (synthcam.hpp:62-78) */
  int32_t frames;
  int32_t num_shapes;
  double fx, fy, cx, cy;
  int32_t width, height;
  ss_shape shapes[SS_MAX_SHAPES];
  /* TextureSpec */
  int32_t tex_type;
  uint32_t tex_seed;
  double tex_scale;
  double dot_radius;
  /* WarpSpec */
  int32_t warp_type;
  int32_t driver_axis;
  int32_t rot_axis;
  int32_t reserved2_;
  double amplitude;
  double frequency;
  double pivot[3];
  double rotation_axis[3];
  double deg_per_frame;
  double trans_per_frame[3];
  /* CameraSpec */
  double cam_rot_axis[3];
  double cam_deg_per_frame;
  double cam_trans_per_frame[3];
  double t_min, t_max;
  double noise_sigma;
  uint32_t noise_seed;
  int32_t reserved3_;
} ss_scene;

/* SyntheticScene::render_frame(frame): depth (W*H meters, 0 = miss) and color
 * (3*W*H, RGB in [0,255]); threads <= 0 uses all OpenMP threads.  Returns 0,
 * or -1 for an invalid scene (no shapes / bad intrinsics / frames < 1). */
int ss_render(const ss_scene* s, int32_t frame, float* depth, float* color, int32_t threads);
/* SyntheticScene::inverse_warp / warp_phase (ground truth for evaluation) */
void ss_inverse_warp(const ss_scene* s, int32_t frame, const double world[3], double canonical[3]);
double ss_warp_phase(const ss_scene* s, int32_t frame);

#ifdef __cplusplus
}
#endif
