# Per-kernel times for every kind x material x precision at scale (default
# engine flags): T4 d=120 (10.4M tets), H8 d=130 (2.2M hexes).
DJG_KIND=T4 DJG_DIVS=120 timeout 900 python tools/ab_models.py NH:4 TI:4 OT:4 MR:4 I57:4 NH:8 TI:8 OT:8 MR:8 I57:8
DJG_KIND=H8 DJG_DIVS=130 timeout 900 python tools/ab_models.py NH:4 TI:4 OT:4 MR:4 I57:4 NH:8 TI:8 OT:8 MR:8 I57:8
