/* Prints sizeof / offsetof of every struct in include/dbtsdf.h as JSON, so
 * tests can check ctypes mirrors (paper_2509_20081_b200/_native.py and the
 * reference-side shim integration/bitsdf_b200.py) against the header itself. */
#include <stddef.h>
#include <stdio.h>

#include "../../include/dbtsdf.h"

#define F(S, m) printf("\"%s.%s\": [%zu, %zu], ", #S, #m, offsetof(S, m), sizeof(((S*)0)->m))

int main(void) {
  printf("{");
  printf("\"dbt_params\": %zu, \"dbt_stats\": %zu, \"dbt_mc_tables\": %zu, \"dbt_deskew\": %zu, ", sizeof(dbt_params),
         sizeof(dbt_stats), sizeof(dbt_mc_tables), sizeof(dbt_deskew));
  F(dbt_params, h_max); F(dbt_params, t_occ); F(dbt_params, downsample); F(dbt_params, first_return);
  F(dbt_params, flags); F(dbt_params, reserved);
  F(dbt_stats, points_in); F(dbt_stats, points_discarded); F(dbt_stats, voxels_written);
  F(dbt_stats, points_applied); F(dbt_stats, unique_centers); F(dbt_stats, centers_skipped);
  F(dbt_stats, bin_fallbacks); F(dbt_stats, elapsed_ms); F(dbt_stats, device_ms); F(dbt_stats, rows_swept);
  F(dbt_mc_tables, edge_table); F(dbt_mc_tables, tri_table); F(dbt_mc_tables, corner_offsets);
  F(dbt_mc_tables, edge_base); F(dbt_mc_tables, edge_axis);
  F(dbt_deskew, mode); F(dbt_deskew, reserved); F(dbt_deskew, q); F(dbt_deskew, rv); F(dbt_deskew, y0);
  F(dbt_deskew, dy); F(dbt_deskew, t0); F(dbt_deskew, t1); F(dbt_deskew, r1);
  printf("\"end\": 0}\n");
  return 0;
}
