"""Oracle-side metric definitions (§5.1 'Metric', L628-637).

TEST INFRASTRUCTURE. Plain transcriptions of the paper's formulas, used to
check the product's host-side finalize (gml_utilization / gml_fragmentation
and paper_2401_08156_b200.metrics).
"""


def utilization(peak_active: int, peak_reserved: int) -> float:
    """'peak active memory divided by peak reserved memory' (L630);
    (0, 0) -> 1.0."""
    if peak_reserved == 0:
        if peak_active:
            raise ValueError("active exceeds reserved")
        return 1.0
    return peak_active / peak_reserved


def fragmentation(peak_active: int, peak_reserved: int) -> float:
    """'(1 - utilization ratio)' (L629)."""
    return 1.0 - utilization(peak_active, peak_reserved)


def mem_reduction_ratio(reserved, gmlake_reserved) -> float:
    """(sum Reserved - sum GMLakeReserved) / sum Reserved (L633-634)."""
    if len(reserved) != len(gmlake_reserved) or not reserved:
        raise ValueError("workload lists must be non-empty and matched")
    a, b = sum(reserved), sum(gmlake_reserved)
    if a == 0:
        raise ValueError("zero denominator")
    return (a - b) / a
