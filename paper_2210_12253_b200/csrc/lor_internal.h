// lor_internal.h -- shared declarations of the B200 LOR library (host setup <-> CUDA kernels).
// Not part of the public ABI (include/lor.h).
//
// Vocabulary:
//   * entity slot tau of an element: per-axis class c_a in {0: min side, 1: interior, 2: max side},
//     tau = c_x + 3 c_y (+ 9 c_z).  3D: 27 slots = 8 vertices, 12 edges, 6 faces, 1 interior
//     (tau = 13); 2D: 9 slots (interior tau = 4).  The slot of a lattice point is the coarse entity
//     it lies on (the "join" of two points is the entity whose classes agree where both points
//     sit on the same boundary).
//   * block (s', tau): the dofs of sub-lattice s' (H1: one; ND: edge direction; RT: face normal)
//     that lie on entity tau.  Their global ids are affine in the local lattice coordinates:
//     gid = g0 + sum_a str[a] * x[a]  (App. A numbering, rank-major renumbered).
//   * OSE: "owned shared entity" -- an entity owned by this rank that is shared by > 1 element;
//     its rows are merged from per-element partial rows ("records") held in the scratch.
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

namespace lorb {

enum Space : int { SP_H1 = 0, SP_ND = 1, SP_RT = 2 };

// topology record flags (per element, per slot)
enum : uint8_t {
  TF_MIN = 1,    // this element is the minimal element containing the entity
  TF_OWNED = 2,  // the entity (and its dofs) is owned by this rank
};
// space record flags
enum : uint8_t {
  SF_SHARED = 1,  // rows of this entity are merged from records (valence > 1)
  SF_DEFER = 2,   // owned shared entity with remote contributors: finalized after the exchange
  SF_SEND = 4,    // entity owned by another rank: records go to the send region
};

constexpr int MAX_VALENCE = 16;           // elements sharing a coarse entity (setup check)

// One per element (local elements first, then ghost elements).  3D uses 27 slots, 2D 9.
struct __align__(16) ElemTopo {
  int32_t ent[27];     // global entity id: vertex / edge / face id, element id for the interior
  uint8_t orient[27];  // edge: 1 = local tail has the larger vertex id; face: swap | s1neg<<1 | s2neg<<2
  uint8_t val[27];     // valence (number of elements containing the entity), capped at 255
  uint8_t flags[27];   // TF_*
  uint8_t pad[3];
};
static_assert(sizeof(ElemTopo) == 192, "layout");

// One per LOCAL element per space.
struct __align__(16) ElemSpace {
  int32_t rec[27];     // record base (16-byte-entry records of MAXL entries) of this element's partial
                       // rows of the entity, -1 if the entity's rows are written directly
  int32_t ose[27];     // index into the OSE table (owned shared entities), -1 otherwise
  int32_t ebase[27];   // global id of the first dof of the entity at each slot (this space)
  uint8_t sflags[27];  // SF_*
  uint8_t pad[1];
};
static_assert(sizeof(ElemSpace) % 16 == 0, "layout");

// Owned shared entity (per space)
struct __align__(16) Ose {
  int32_t gid_base;   // global id of the entity's first dof (rows gid_base .. gid_base+nrows-1)
  int32_t nrows;
  int32_t k;          // number of contributing elements (slots)
  int32_t slot_off;   // offset into ose_slots (record base of each slot, element order)
};

// scratch record entry.  A record = one element's partial row of a shared row: entries sorted by
// column; the last entry of the record (index rstride-1) is the header {col = len}.
struct __align__(16) RecEntry {
  int32_t col;
  int32_t bbase;  // base gid of the column's block: equal bases = same block in every element
  double val;
};

}  // namespace lorb
