for v in '{"mode":"f32"}' '{"mode":"f32","epi_pace":-1}' '{"mode":"f16"}' '{"mode":"f16","epi_pace":-1}'; do bash tools/ncu_metrics.sh "$v"; done
VARIANTS='[{"mode":"f32"},{"mode":"f32","epi_pace":-1},{"mode":"f16"},{"mode":"f16","epi_pace":-1}]' ROUNDS=4 python tools/ab.py
