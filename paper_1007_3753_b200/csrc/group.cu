// group.cu — sizing entry points of the group launches (one dictionary per
// solve; see solvers_common.cuh group_kernel / run_group and the header).
#include "solvers_common.cuh"

using namespace ell1;

int32_t ell1_fista_group_team_impl(const ell1_dict_t* D);
int32_t ell1_ist_group_team_impl(const ell1_dict_t* D);
int32_t ell1_palm_group_team_impl(const ell1_dict_t* D);
int32_t ell1_dalm_group_team_impl(const ell1_dict_t* D);
int32_t ell1_gpsr_group_team_impl(const ell1_dict_t* D);
int32_t ell1_tnipm_group_team_impl(const ell1_dict_t* D);
int32_t ell1_homotopy_group_team_impl(const ell1_dict_t* D);

extern "C" size_t ell1_group_args_bytes(int32_t count) {
  return count <= 0 ? 256 : (size_t)count * ELL1_GROUP_ARG_BYTES + 512;
}

extern "C" int32_t ell1_group_team(int32_t solver, const ell1_dict_t* D) {
  if (!dict_ok(D)) return 0;
  switch (solver) {
    case ELL1_SOLVER_CORR:
    case ELL1_SOLVER_POWER: return 1;
    case ELL1_SOLVER_FISTA: return ell1_fista_group_team_impl(D);
    case ELL1_SOLVER_IST: return ell1_ist_group_team_impl(D);
    case ELL1_SOLVER_PALM: return ell1_palm_group_team_impl(D);
    case ELL1_SOLVER_DALM: return ell1_dalm_group_team_impl(D);
    case ELL1_SOLVER_GPSR: return ell1_gpsr_group_team_impl(D);
    case ELL1_SOLVER_TNIPM: return ell1_tnipm_group_team_impl(D);
    case ELL1_SOLVER_HOMOTOPY: return ell1_homotopy_group_team_impl(D);
    default: return 0;
  }
}

extern "C" size_t ell1_group_workspace(int32_t solver, const ell1_dict_t* D, int32_t team) {
  if (!dict_ok(D) || team < 1) return 0;
  switch (solver) {
    case ELL1_SOLVER_CORR: return grid_bytes(team, D->d, 0) + 1024;
    case ELL1_SOLVER_POWER: return grid_bytes(team, D->d, 1) + 3 * align_up(D->ld * 8, 256) + 2048;
    case ELL1_SOLVER_FISTA: return ell1_fista_workspace(D, nullptr, team);
    case ELL1_SOLVER_IST: return ell1_ist_workspace(D, team);
    case ELL1_SOLVER_PALM: return ell1_palm_workspace(D, team);
    case ELL1_SOLVER_DALM: return ell1_dalm_workspace(D, team);
    case ELL1_SOLVER_GPSR: return ell1_gpsr_workspace(D, team);
    case ELL1_SOLVER_TNIPM: return ell1_tnipm_workspace(D, team);
    case ELL1_SOLVER_HOMOTOPY: return ell1_homotopy_workspace(D, team);
    default: return 0;
  }
}
