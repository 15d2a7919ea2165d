// Device-resident batch of independent environments ("world").
//
// Layout (all fp64 state, SoA, flattened over environments; every per-env
// range is a prefix array `env_*[e] .. env_*[e+1]`):
//   DoF vector x/v/...   env e owns [env_dof[e], env_dof[e+1]); inside an env
//                        the reference layout: soft vertex triples first,
//                        then affine bodies as (p, rows of A)  (ref bodies.py:1-6)
//   soft vertices        vert_dof (index of the x coordinate), vert_mass
//   affine bodies        aff_dof, aff_M (12x12), aff_acc (M⁻¹ f_gravity), aff_ortho (λV)
//   tets                 tet_dof (4 vertex DoF indices), Dm⁻¹ (9), rest volume, μ, λ, model
//   contact slots        slot_aff (kind), slot_dof (soft DoF index | affine body DoF
//                        offset), slot_rest (lever arm), slot_cbody
//   triangles / edges    global slot ids, owning collision body, rest length²
//   collision bodies     rigid / kinematic flags, excluded-partner bitmask (env-local ids)
//   constraints          kinematic AL targets (ref constraints.py:36)
//   candidates           per-env capacity ranges; pairs stored lexicographically
#pragma once

// The engine is built from two translation units compiled in parallel:
// engine.cu (host engine + batched kernels) and fused.cu (the per-env fused
// step kernels). Batched kernels are declared IPC_GLOBAL; in the fused unit
// they become uninstantiated templates, so each kernel is compiled once.
#ifdef IPC_FUSED_TU
#define IPC_GLOBAL template <int = 0> __global__
#else
#define IPC_GLOBAL __global__
#endif
#include <stdint.h>

// Programmatic dependent launch: the engine launches its kernels with
// programmatic stream serialization, so a kernel may be scheduled while its
// predecessor drains; every kernel waits here before touching memory (a no-op
// when launched without the attribute).
__device__ __forceinline__ void ipc_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

namespace ipc {

struct Cands {
  int2* pt;       // (slot, tri)
  int2* ee;       // (edge i, edge j), i < j
  int* gnd;       // slot ids
  int* n_pt;      // [n_env]
  int* n_ee;
  int* n_gnd;
  const long long* pt_off;  // [n_env+1] capacity prefix
  const long long* ee_off;
  const int* gnd_off;       // == env_slot
  int* overflow;            // [1] set when a capacity is exceeded
  int *pre_pt, *pre_ee, *pre_gnd;  // [n_env+1] prefix of counts over flagged envs
  int *need_pt, *need_ee;           // [n_env] unclipped counts of the last broad phase (capacity growth)
};

struct Lags {  // lagged friction (ref friction.py:35)
  int4* slots;      // 4 slots per stencil
  double* gamma;    // 4
  double* tangent;  // 3x2 row-major
  double* lam;
  int* n;           // [n_env]
  const long long* off;  // [n_env+1] capacity prefix (== pt_off + ee_off)
  int* g_slot;      // ground lags
  double* g_lam;
  int* g_n;         // [n_env]
  int *pre, *g_pre;  // [n_env+1] prefix of lag counts
};

struct World {
  int n_env, n_dof, n_vert, n_aff, n_tet, n_slot, n_tri, n_edge, n_cbody, n_cons;
  // env prefix arrays
  const int *env_dof, *env_vert, *env_aff, *env_tet, *env_slot, *env_tri, *env_edge, *env_cbody,
      *env_cons;
  const unsigned char* env_pairs;  // needs_pair_search
  const unsigned char* env_has_ground;
  const double* env_ground_y;
  const double* env_gravity;  // 3 per env
  double *env_dhat, *env_kappa, *env_kappa0, *env_mu, *env_epsv;
  // per-element env ids
  const int *dof_env, *vert_env, *aff_env, *tet_env, *slot_env, *cons_env;
  // state
  double *x, *v, *x_prev, *xhat, *p, *xt, *grad;
  // soft vertices
  const int* vert_dof;
  const double* vert_mass;
  // affine bodies
  const int* aff_dof;
  const double *aff_M, *aff_acc, *aff_ortho;
  // tets
  const int4* tet_dof;
  const double *tet_Dminv, *tet_vol, *tet_mu, *tet_lam;
  const unsigned char* tet_model;
  // slots & primitives
  const unsigned char* slot_aff;
  const int* slot_dof;
  const double* slot_rest;
  const int* slot_cbody;
  const int3* tri_v;
  const int* tri_cbody;
  const int2* edge_v;
  const int* edge_cbody;
  const double* edge_len2;
  const unsigned char *cbody_rigid, *cbody_kin;
  const unsigned long long* cbody_excl;
  const int *cbody_slot, *cbody_tri, *cbody_edge;  // [n_cbody+1] contiguous primitive ranges
  // 32-primitive chunks per body (second culling level of the broad phase)
  int n_tchunk, n_echunk;
  const int *tchunk_p0, *echunk_p0;        // [n_chunk+1] first primitive of each chunk
  const int *cbody_tchunk, *cbody_echunk;  // [n_cbody+1] chunk ranges of each body
  double *tchunk_box, *echunk_box;         // 6 per chunk (lo, hi), refreshed per broad phase
  // LBVHs of large bodies (lbvh.cuh), rebuilt per global broad phase
  int n_tree;
  const int *tree_kind, *tree_p0, *tree_n, *tree_node0, *tree_leaf0;  // [n_tree]
  const int *cbody_tbvh, *cbody_ebvh;  // [n_cbody] tree of the body's triangles / edges, -1: none
  int *bvh_child, *bvh_parent, *bvh_lparent, *bvh_prim;  // 2 per internal node, per node, per leaf, per leaf
  double* bvh_box;                     // 6 per internal node
  // constraints
  const int* cons_aff;
  double *cons_target, *cons_lam, *cons_kappa, *cons_kappa0, *cons_mass, *cons_lastres;
  // world-space slot positions
  double *xw, *xw0, *dxw;
};

// per-environment solver scalars (device)
struct EnvState {
  double *e0, *e_new, *alpha, *alpha_max, *pnorm, *prev_pnorm, *gnorm, *min_s_before, *min_s,
      *res;
  int *small_run, *newton_active, *ls_active, *al_active, *ls_failed, *converged, *newton_iters,
      *ccd_calls, *al_outer, *err, *any;
};

}  // namespace ipc
