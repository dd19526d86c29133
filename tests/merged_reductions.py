"""One element-wise producer with three reductions of different lengths
(column sums n=C >= 32, row sums n=R, a full sum n=1): the planner finalizes
all three in ONE launch (blockIdx.y selects the reduction).  Shared by the
CPU plan test and the GPU parity test."""


def merged_reduction_program(R: int, C: int) -> str:
    X = f"<{R} x {C} x f32>"
    return f'''module "mf"
stage raw
func @f: ({X}) -> (<{C} x f32>, <{R} x f32>, f32) {{
'entry(%x: {X}):
    %s = multiply %x: {X}, %x: {X}
    %c = reduce %s: {X} by add along 0
    %r = reduce %s: {X} by add along 1
    %e = exp %x: {X}
    %q = reduce %e: {X} by add along 1
    %t = reduce %q: <{R} x f32> by add along 0
    return (%c: <{C} x f32>, %r: <{R} x f32>, %t: f32)
}}
'''
