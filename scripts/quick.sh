bash scripts/abtest.sh "" "-DVP_TEAM_MINB=4"
