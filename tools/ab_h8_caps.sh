export DJG_KIND=H8 DJG_DIVS=130
A="${@:-NH:4 TI:4 OT:4 MR:4 NH:8 TI:8 OT:8 MR:8}"
echo "== default"; timeout 600 python tools/ab_models.py $A
echo "== full"; DJG_FLAGS=32 timeout 600 python tools/ab_models.py $A
