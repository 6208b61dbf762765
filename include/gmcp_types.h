/* Plain-C value types shared by the GMCP B200 C-ABI (include/gmcp_b200.h) and
 * the CPU oracle API (oracle/gmcp_oracle_api.h). No torch, no Eigen, no CUDA
 * types: plain pointers and sizes only.
 *
 * Each struct is the SoA/C restatement of a reference type:
 *   gmcp_surface          <- gmcp::ContactSurface   (proj/include/gmcp/contact_sampling.hpp:219-224)
 *   gmcp_barrier_params   <- gmcp::BarrierParams    (proj/include/gmcp/barrier.hpp:9-19)
 *   gmcp_samples          <- std::vector<gmcp::ContactSample> (contact_sampling.hpp:20-31), SoA
 *   gmcp_pressure_record  <- gmcp::PressureRecord   (contact_energy.hpp:217-223)
 */
#ifndef GMCP_TYPES_H
#define GMCP_TYPES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. The C++ drop-in layer (include/gmcp/b200.hpp) rethrows the
 * matching reference exception type (proj/include/gmcp/core.hpp:25-56). */
enum {
  GMCP_OK = 0,
  GMCP_ERR_INFEASIBLE = 1, /* InfeasibleGapError{sample_id}: a gap is <= 0      */
  GMCP_ERR_DEGENERATE = 2, /* MeshError: degenerate slave triangle / 2D frame     */
  GMCP_ERR_CONFIG = 3,     /* ConfigError: bad parameters / mismatched inputs     */
  GMCP_ERR_SOLVER = 4,     /* SolverError{residual}: Newton / line search / PCG   */
  GMCP_ERR_CUDA = 5,       /* CUDA runtime failure (no CPU fallback exists)       */
  GMCP_ERR_ARG = 6,        /* null pointer / size mismatch at the boundary        */
  GMCP_ERR_PARSE = 7       /* ParseError (scene text)                             */
};

/* Reference SampleType values (contact_sampling.hpp:18). */
enum { GMCP_POINT = 0, GMCP_EDGE = 1, GMCP_FACE = 2 };

/* One side of a contact pair, addressed by global vertex ids into the flat
 * 3N position vector (xyz interleaved, as the reference's VecX). */
typedef struct {
  int32_t n_tris;
  const int32_t* tris;      /* [n_tris][3]                                    */
  int32_t n_edges;
  const int32_t* edges;     /* [n_edges][2], lo < hi, numbered by first use   */
  const int32_t* tri_edges; /* [n_tris][3]                                    */
  int32_t n_verts;
  const int32_t* verts;     /* ascending unique global vertex ids             */
} gmcp_surface;

typedef struct {
  double kappa_face;       /* Pa/m                                    */
  double kappa_edge;       /* < 0: derived (barrier.hpp:25-46)        */
  double kappa_point;      /* < 0: derived                            */
  double eps_max;
  double delta_face;
  double delta_edge;
  double detection_radius; /* < 0: derived = 10 eps_max               */
  int32_t quad_order_face; /* 1..4                                    */
  int32_t quad_order_edge; /* 1..5                                    */
} gmcp_barrier_params;

/* Frozen contact samples in reference order, structure of arrays. Every
 * pointer is caller-owned and sized for n entries (x3 where noted). */
typedef struct {
  int64_t n;
  int8_t* type;    /* GMCP_POINT / GMCP_EDGE / GMCP_FACE        */
  int32_t* slave;  /* [n][3] global vertex ids of slave tri     */
  int32_t* master; /* [n][3] 3 (face) / 2 (edge) / 1 (point), -1 padded */
  double* beta_s;  /* [n][3]                                    */
  double* beta_m;  /* [n][3] (face samples; 0 otherwise)        */
  double* eta;     /* [n]                                       */
  double* weight;  /* [n]                                       */
  double* gamma;   /* [n]                                       */
  double* eps;     /* [n]                                       */
  double* g_ref;   /* [n]                                       */
} gmcp_samples;

typedef struct {
  int64_t sample;     /* index into the sample array            */
  double position[3]; /* slave-side sample point                */
  double radius;      /* hypot(x, y)                            */
  double gap;
  double pressure;
} gmcp_pressure_record;

#ifdef __cplusplus
}
#endif

#endif /* GMCP_TYPES_H */
