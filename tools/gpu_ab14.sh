VARIANTS='[{"mode":"f32","config":1},{"mode":"f32","config":8},{"mode":"f16","config":1},{"mode":"f16","config":8}]' ROUNDS=12 REPS=8 python tools/ab.py
VARIANTS='[{"mode":"f32","config":8},{"mode":"f32","config":1},{"mode":"f16","config":8},{"mode":"f16","config":1}]' ROUNDS=12 REPS=8 python tools/ab.py
