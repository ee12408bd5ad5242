"""B200-native interior-penalty DG system assembly (drop-in for dgfem::assemble_all)."""
from . import capi, problems  # noqa: F401
